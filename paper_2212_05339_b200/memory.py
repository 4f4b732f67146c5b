"""Memory contracts of the chunk store (the reference's cost-model sizes).

The planner sizes every placement with three formulas; the runtime's
allocations must honour them, so they are restated here as the contract the
ChunkManager is checked against (`ChunkManager.memory_ledger`):

  * chunk_footprint        — per-GPU bytes of one partitioned chunk plus its
                             paired optimizer chunk, ceil((Lc + Los*Fos)*C / N)
                             (offplan/cost_model.py:147-153)
  * mixed_precision_states — whole-model (parameter, gradient, optimizer
                             state) bytes, (Lc*M, Lc*M, Los*Fos*M)
                             (offplan/cost_model.py:156-167)
  * shared_state_bytes     — the shared (multi-use) parameter's cost:
                             replicated Lc*S plus ceil((Lc + Los*Fos)*S / N)
                             (offplan/search.py:116-126)

Errors follow the reference: ValidationError on non-positive sizes.
"""

from __future__ import annotations

from typing import Any

from .errors import ValidationError
from .profiles import PrecisionSpec


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def chunk_footprint(chunk_length: int, gpus: int, precision: Any = PrecisionSpec()) -> int:
    """Per-GPU bytes of one chunk's compute shard + optimizer shard
    (cost_model.py:147-153)."""
    if chunk_length < 1 or gpus < 1:
        raise ValidationError("chunk_length and gpus must be >= 1")
    return _ceil_div((precision.compute_bytes + precision.optimizer_state_bytes) * chunk_length, gpus)


def mixed_precision_states(model_elements: int, precision: Any = PrecisionSpec()) -> tuple[int, int, int]:
    """(parameter, gradient, optimizer-state) bytes for the whole model
    (cost_model.py:156-167): 2M, 2M, 12M at the default widths."""
    if model_elements < 1:
        raise ValidationError("model_elements must be >= 1")
    lc = precision.compute_bytes
    return lc * model_elements, lc * model_elements, precision.optimizer_state_bytes * model_elements


def shared_state_bytes(shared_elements: int, gpus: int, precision: Any = PrecisionSpec()) -> int:
    """Per-GPU bytes of the shared parameters: the replicated compute copy
    plus this rank's share of compute + optimizer state (search.py:116-126)."""
    if shared_elements <= 0:
        return 0
    lc = precision.compute_bytes
    return lc * shared_elements + _ceil_div((lc + precision.optimizer_state_bytes) * shared_elements, gpus)
