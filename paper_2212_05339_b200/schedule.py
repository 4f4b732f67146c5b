"""rCache schedule: plan input, event program, SimReport-equivalent counters.

The runtime does not re-decide anything at run time: the reference planner's
Plan (offplan/search.py:267-291, loaded from its JSON, search.py:444-474)
fixes chunk length, rCache size and chunk homes, and the native schedule
compiler (elx_schedule, csrc/elx_schedule.cpp) turns the chunk trace into the
exact gather / evict / pin / reduce sequence of offplan.simulate
(rcache_sim.py:87-199). The runtime replays that program and its live
counters must equal the compiled ones (and therefore the reference's).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from enum import Enum
from types import MappingProxyType
from typing import Any, Mapping

import numpy as np

from . import _lib
from .errors import ProfileFormatError, ValidationError
from .profiles import PrecisionSpec

FORMAT_VERSION = 1


class Device(str, Enum):
    GPU = "gpu"
    CPU = "cpu"


@dataclass(frozen=True)
class SimReport:
    """Same fields and meaning as offplan.SimReport (rcache_sim.py:65-84)."""

    gather_ops: int
    gather_bytes: int
    reduce_bytes: int
    g2c_bytes: int
    c2g_bytes: int
    replaced_bytes: int
    peak_rcache_blocks: int
    estimated_offload_seconds: float
    estimated_update_seconds: float
    g2c_shard_bytes: int
    c2g_shard_bytes: int


@dataclass(frozen=True)
class Decision:
    action: str
    benefit: float
    budget_after: float


@dataclass(frozen=True)
class Plan:
    """The planner's output (search.py:267-291)."""

    chunk_length: int
    n_block: int
    chunk_homes: Mapping[int, Device]
    shared_strategy_bytes: int = 0
    shared_param_ids: tuple[str, ...] = ()
    estimates: SimReport | None = None
    decision_trace: tuple[Decision, ...] = ()

    def __post_init__(self) -> None:
        if self.n_block < 1:
            raise ValidationError("n_block must be >= 1")
        object.__setattr__(self, "chunk_homes", MappingProxyType(
            {int(k): Device(v) for k, v in dict(self.chunk_homes).items()}))

    @property
    def gpu_home_chunks(self) -> int:
        return sum(1 for d in self.chunk_homes.values() if d is Device.GPU)


def load_plan(text: str) -> Plan:
    """Parse the reference plan JSON (search.py:422-474 writes it)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ProfileFormatError(f"plan: not valid JSON ({exc})") from None
    if not isinstance(doc, dict) or doc.get("format_version") != FORMAT_VERSION:
        raise ProfileFormatError("plan: format_version: expected 1")
    try:
        est = doc.get("estimates")
        return Plan(
            chunk_length=int(doc["chunk_length"]),
            n_block=int(doc["n_block"]),
            chunk_homes={int(k): Device(v) for k, v in doc["chunk_homes"].items()},
            shared_strategy_bytes=int(doc.get("shared_strategy_bytes", 0)),
            shared_param_ids=tuple(doc.get("shared_param_ids", ())),
            estimates=None if est is None else SimReport(**est),
            decision_trace=tuple(Decision(d["action"], float(d["benefit"]), float(d["budget_after"]))
                                 for d in doc.get("decision_trace", ())),
        )
    except (KeyError, TypeError, ValueError) as exc:
        raise ProfileFormatError(f"plan: malformed field ({exc})") from None


def as_plan(obj: Any) -> Plan:
    """Accept our Plan, an offplan.Plan (duck-typed) or plan JSON text."""
    if isinstance(obj, Plan):
        return obj
    if isinstance(obj, str):
        return load_plan(obj)
    return Plan(obj.chunk_length, obj.n_block,
                {int(k): Device(getattr(v, "value", v)) for k, v in obj.chunk_homes.items()},
                int(getattr(obj, "shared_strategy_bytes", 0)),
                tuple(getattr(obj, "shared_param_ids", ())))


# --------------------------------------------------------------------------
# Compiled event program
# --------------------------------------------------------------------------

EVENT_DTYPE = np.dtype([("kind", np.int32), ("pos", np.int32), ("chunk", np.int32),
                        ("block", np.int32), ("victim", np.int32), ("issue_pos", np.int32)])


@dataclass(frozen=True)
class Schedule:
    n_forward: int
    n_chunks: int
    n_block: int
    events: np.ndarray             # EVENT_DTYPE records, ordered by (pos, emission)
    counters: dict[str, int]       # elx_sim_counters fields
    cpu_home: np.ndarray           # uint8 per chunk

    @property
    def walk_length(self) -> int:
        return 2 * self.n_forward

    def gathers_at(self, pos: int) -> np.ndarray:
        e = self.events
        return e[(e["kind"] == _lib.EV_GATHER) & (e["pos"] == pos)]

    def reduces_at(self, pos: int) -> np.ndarray:
        e = self.events
        return e[(e["kind"] == _lib.EV_REDUCE) & (e["pos"] == pos)]


def _placement_array(trace: Any, n_chunks: int, placement: Mapping[int, Any]) -> np.ndarray:
    ids = sorted(trace.chunk_ids)
    missing = [c for c in ids if c not in placement]
    if missing:
        raise ValidationError(f"placement missing chunk ids {missing}")
    arr = np.zeros(n_chunks, dtype=np.uint8)
    for c, d in placement.items():
        if 0 <= int(c) < n_chunks:
            arr[int(c)] = 1 if Device(getattr(d, "value", d)) is Device.CPU else 0
    return arr


def compile_schedule(trace: Any, n_block: int, placement: Mapping[int, Any],
                     n_chunks: int | None = None) -> Schedule:
    """Compile a ChunkTrace (ours or offplan's) into the rCache event program."""
    lib = _lib.load()
    fwd = [sorted(s) for s in trace.forward]
    if n_chunks is None:
        n_chunks = 1 + max((c for s in fwd for c in s), default=-1)
    ptr = np.zeros(len(fwd) + 1, dtype=np.int32)
    for i, s in enumerate(fwd):
        ptr[i + 1] = ptr[i] + len(s)
    flat = np.ascontiguousarray([c for s in fwd for c in s] or [0], dtype=np.int32)
    home = _placement_array(trace, n_chunks, placement)
    cap = 2 * int(ptr[-1]) + n_chunks + 8  # every walk touch may gather; one reduce per chunk
    events = np.zeros(cap, dtype=EVENT_DTYPE)
    n_ev = ctypes.c_int64(0)
    cnt = _lib.SimCounters()
    rc = lib.elx_schedule(len(fwd), ptr.ctypes.data, flat.ctypes.data, n_chunks, int(n_block),
                          home.ctypes.data if n_chunks else None, events.ctypes.data, cap,
                          ctypes.byref(n_ev), ctypes.byref(cnt))
    _lib.check(rc, "elx_schedule")
    counters = {name: int(getattr(cnt, name)) for name, _ in _lib.SimCounters._fields_}
    return Schedule(len(fwd), n_chunks, int(n_block), events[: n_ev.value].copy(), counters, home)


def report_from_counters(counters: Mapping[str, int], trace: Any, chunk_length: int,
                         placement: Mapping[int, Any], precision: Any = PrecisionSpec(),
                         gpu_count: int = 1, hardware: Any = None) -> SimReport:
    """SimReport from unit counters, with rcache_sim.py:168-199's byte/time rules."""
    cb = precision.compute_bytes * chunk_length
    g2c = counters["g2c_units"] * cb
    c2g = counters["c2g_units"] * cb
    off_s = upd_s = 0.0
    if hardware is not None:
        r = hardware.rates(gpu_count)
        off_s = g2c / r.b_g2c + c2g / r.b_c2g
        os_chunk = precision.optimizer_bytes * chunk_length
        ids = trace.chunk_ids
        n_cpu = sum(1 for c in ids if Device(getattr(placement[c], "value", placement[c])) is Device.CPU)
        upd_s = (len(ids) - n_cpu) * os_chunk / r.v_g + n_cpu * os_chunk / r.v_c
    return SimReport(
        gather_ops=counters["gather_ops"],
        gather_bytes=counters["gather_ops"] * cb,
        reduce_bytes=counters["reduce_ops"] * cb,
        g2c_bytes=g2c,
        c2g_bytes=c2g,
        replaced_bytes=counters["replaced_ops"] * cb,
        peak_rcache_blocks=counters["peak_rcache_blocks"],
        estimated_offload_seconds=off_s,
        estimated_update_seconds=upd_s,
        g2c_shard_bytes=-(-g2c // gpu_count),
        c2g_shard_bytes=-(-c2g // gpu_count),
    )


def simulate(trace: Any, n_block: int, chunk_length: int, placement: Mapping[int, Any],
             precision: Any = PrecisionSpec(), gpu_count: int = 1, hardware: Any = None) -> SimReport:
    """Native equivalent of offplan.simulate (rcache_sim.py:87-199)."""
    if chunk_length < 1:
        raise ValidationError("chunk_length must be >= 1")
    if gpu_count < 1:
        raise ValidationError("gpu_count must be >= 1")
    sched = compile_schedule(trace, n_block, placement)
    return report_from_counters(sched.counters, trace, chunk_length, placement, precision,
                                gpu_count, hardware)
