"""ctypes binding of libelixir_b200.so (include/elixir_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(``make -C paper_2212_05339_b200/csrc``). There is deliberately no fallback:
if the library is missing every hot-path call raises ExtensionMissingError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import (
    ChunkTooSmallError,
    ElixirCudaError,
    ExtensionMissingError,
    InfeasibleCacheError,
    InfeasibleError,
    ValidationError,
)

LIB_PATH = Path(__file__).resolve().parent / "libelixir_b200.so"

# elx_status (include/elixir_b200.h)
OK = 0
ERR_VALIDATION = 100
ERR_INFEASIBLE = 200
ERR_CHUNK_TOO_SMALL = 201
ERR_INFEASIBLE_CACHE = 202
ERR_CUDA = 300

# elx_dtype
F32, BF16, F16 = 0, 1, 2
ADAM_TILE = 4096
MAX_WORLD = 16
# step-scalar block (include/elixir_b200.h, K3)
STEP_SCALARS = 2048
SC_TICKET = 4
SC_PARTIALS = 8
RELEASE_MAX_SEGS = 16
EV_GATHER, EV_REDUCE = 0, 1

c_i32, c_i64, c_f32, c_f64, c_vp = (
    ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p)


class Event(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("pos", c_i32), ("chunk", c_i32), ("block", c_i32),
                ("victim", c_i32), ("issue_pos", c_i32)]


class SimCounters(ctypes.Structure):
    _fields_ = [("gather_ops", c_i64), ("replaced_ops", c_i64), ("reduce_ops", c_i64),
                ("c2g_units", c_i64), ("g2c_units", c_i64), ("peak_rcache_blocks", c_i64),
                ("working_set", c_i64)]


class Member(ctypes.Structure):
    _fields_ = [("ext", c_vp), ("offset", c_i64), ("numel", c_i64), ("ext_dtype", c_i32),
                ("pad_", c_i32)]


class AdamSeg(ctypes.Structure):
    _fields_ = [("p32", c_vp), ("m", c_vp), ("v", c_vp), ("g", c_vp), ("p16", c_vp),
                ("n", c_i64), ("tile0", c_i64), ("g_dtype", c_i32), ("pad_", c_i32)]


class AdamHP(ctypes.Structure):
    _fields_ = [("lr", c_f64), ("beta1", c_f64), ("beta2", c_f64), ("eps", c_f64),
                ("weight_decay", c_f64), ("max_norm", c_f64), ("grad_scale", c_f64),
                ("p16_dtype", c_i32), ("max_ctas", c_i32), ("bc1_table", c_vp), ("bc2s_table", c_vp),
                ("table_len", c_i64)]


class CpuSeg(ctypes.Structure):
    _fields_ = [("p32", c_vp), ("m", c_vp), ("v", c_vp), ("g", c_vp), ("p16", c_vp),
                ("n", c_i64), ("g_dtype", c_i32), ("pad_", c_i32)]


class ReleaseSeg(ctypes.Structure):
    _fields_ = [("g", c_vp), ("src", c_vp * MAX_WORLD), ("n", c_i64)]


# name -> (restype, argtypes)
_SIGNATURES = {
    "elx_abi_version": (c_i32, []),
    "elx_last_error": (ctypes.c_char_p, []),
    "elx_launch_count": (c_i64, []),
    "elx_event_record": (ctypes.c_int, [c_vp, c_vp]),
    "elx_sizeof": (c_i64, [c_i32]),
    "elx_layout_pack": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "elx_schedule": (ctypes.c_int, [c_i32, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "elx_chunk_pack": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_vp, c_i32, c_vp]),
    "elx_chunk_unpack": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_vp]),
    "elx_fetch": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "elx_fetch_ce": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "elx_fetch_ranked": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_vp]),
    "elx_device_barrier": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_vp]),
    "elx_peer_sum_f64": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32, c_vp]),
    "elx_enable_peer_access": (ctypes.c_int, [c_i32]),
    "elx_ipc_open": (ctypes.c_int, [c_vp, c_vp]),
    "elx_ipc_close": (ctypes.c_int, [c_vp]),
    "elx_release": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32, c_i32, c_f32, c_vp, c_vp]),
    "elx_release_batch": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_f32, c_vp, c_vp]),
    "elx_release_geometry": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "elx_adam": (ctypes.c_int, [c_vp, c_i32, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "elx_norm_finalize": (ctypes.c_int, [c_vp, c_f64, c_vp, c_vp]),
    "elx_step_reset": (ctypes.c_int, [c_vp, c_vp]),
    "elx_step_advance": (ctypes.c_int, [c_vp, c_vp]),
    "elx_colsum_workspace": (c_i64, [c_i64, c_i64]),
    "elx_colsum_geometry": (ctypes.c_int, [c_i64, c_i64, c_vp, c_vp]),
    "elx_colsum": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i32, c_i64, c_i64, c_vp, c_vp]),
    "elx_colsum_batched": (ctypes.c_int, [c_i32, c_vp, c_i32, c_vp, c_i32, c_i64, c_i64, c_vp]),
    "elx_xent_fwd": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "elx_xent_bwd": (ctypes.c_int, [c_vp, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "elx_ln_param_grad": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp]),
    "elx_layer_norm_fwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_f32, c_vp]),
    "elx_layer_norm_bwd_dx": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp]),
    "elx_layer_norm_bwd_dx_res": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp]),
    "elx_gelu_fwd": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i64, c_vp]),
    "elx_gelu_bwd": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i64, c_vp]),
    "elx_gelu_bwd_colsum": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i64, c_i64, c_vp]),
    "elx_embedding_bwd": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp]),
    "elx_lt_matmul": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                     c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "elx_lt_matmul_ex": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64,
                                        c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp]),
    "elx_copy_h2d": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "elx_copy_d2h": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "elx_cpu_adam": (ctypes.c_int, [c_vp, c_i32, c_vp, c_i64, c_vp, c_i32]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("ELX_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise ExtensionMissingError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the hot path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.elx_abi_version() != 1:
        raise ExtensionMissingError("libelixir_b200 ABI version mismatch")
    for i, st in enumerate((Event, SimCounters, Member, AdamSeg, AdamHP, CpuSeg, ReleaseSeg)):
        if lib.elx_sizeof(i) != ctypes.sizeof(st):
            raise ExtensionMissingError(f"libelixir_b200 struct {st.__name__} layout mismatch "
                                        f"({lib.elx_sizeof(i)} != {ctypes.sizeof(st)}): rebuild the library")
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map an elx_status to the exception tree (errors.py)."""
    if rc == OK:
        return
    msg = load().elx_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == ERR_CHUNK_TOO_SMALL:
        raise ChunkTooSmallError(msg)
    if rc == ERR_INFEASIBLE_CACHE:
        raise InfeasibleCacheError(msg)
    if rc == ERR_INFEASIBLE:
        raise InfeasibleError(msg)
    if rc == ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == ERR_CUDA:
        raise ElixirCudaError(msg)
    raise RuntimeError(f"unknown elx status {rc}: {msg}")


def launch_count() -> int:
    return int(load().elx_launch_count())
