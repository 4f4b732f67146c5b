"""B200-native Elixir chunk-memory hot path (arXiv 2212.05339).

Public API (drop-in for the reference runtime's chunk-manager /
chunk-fetcher / hybrid-optimizer, consuming offplan's plan/layout/trace):

    ChunkManager, ChunkFetcher, HybridAdam, LossScaler   (runtime.py)
    pack_chunks, build_chunk_trace, ChunkLayout, ...       (layout.py)
    compile_schedule, simulate, Plan, load_plan, Device    (schedule.py)
    ElixirGPT2, GPT2Config, PRESETS                        (gpt2.py)

Kernels live in libelixir_b200.so (csrc/, include/elixir_b200.h).
"""

from .errors import (ChunkTooSmallError, ElixirCudaError, ExtensionMissingError, InfeasibleCacheError,
                     InfeasibleError, PlannerError, ProfileFormatError, UncommonGraphError, ValidationError)
from .layout import Chunk, ChunkLayout, ChunkMember, ChunkTrace, build_chunk_trace, pack_chunks, waste_rate, working_set_blocks
from .profiles import (AccessTrace, ModelProfile, OperatorNode, ParameterSpec, PrecisionSpec, coarsen_graph,
                       partition_multiuse, synthesize_transformer_profile)
from .memory import chunk_footprint, mixed_precision_states, shared_state_bytes
from .schedule import Device, Plan, Schedule, SimReport, compile_schedule, load_plan, simulate

__all__ = [
    "ChunkTooSmallError", "ElixirCudaError", "ExtensionMissingError", "InfeasibleCacheError", "InfeasibleError",
    "PlannerError", "ProfileFormatError", "UncommonGraphError", "ValidationError",
    "Chunk", "ChunkLayout", "ChunkMember", "ChunkTrace", "build_chunk_trace", "pack_chunks", "waste_rate",
    "working_set_blocks", "AccessTrace", "ModelProfile", "OperatorNode", "ParameterSpec", "PrecisionSpec",
    "coarsen_graph", "partition_multiuse", "synthesize_transformer_profile", "Device", "Plan", "Schedule",
    "SimReport", "compile_schedule", "load_plan", "simulate", "ChunkManager", "ChunkFetcher", "HybridAdam",
    "LossScaler", "ElixirGPT2", "GPT2Config", "PRESETS", "chunk_footprint", "mixed_precision_states",
    "shared_state_bytes",
]

__version__ = "0.1.0"


def __getattr__(name):  # torch-dependent parts load on first use
    if name in ("ChunkManager", "ChunkFetcher", "HybridAdam", "LossScaler"):
        from . import runtime
        return getattr(runtime, name)
    if name in ("ElixirGPT2", "GPT2Config", "PRESETS"):
        from . import gpt2
        return getattr(gpt2, name)
    raise AttributeError(name)
