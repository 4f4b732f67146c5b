"""Chunk layout and chunk-level trace (the chunk store's addressing contract).

Field names follow offplan/chunking.py:25-79 so layouts from either side
compare equal field by field. Packing itself runs in the native library
(elx_layout_pack, csrc/elx_schedule.cpp), which implements the greedy
in-order contract of offplan.pack_chunks (chunking.py:102-138).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from types import MappingProxyType
from typing import Any, Mapping, Sequence

import numpy as np

from . import _lib
from .errors import ValidationError


@dataclass(frozen=True)
class ChunkMember:
    param_id: str
    offset: int
    numel: int


@dataclass(frozen=True)
class Chunk:
    id: int
    length: int
    members: tuple[ChunkMember, ...]

    @property
    def used_elements(self) -> int:
        return sum(m.numel for m in self.members)


@dataclass(frozen=True)
class ChunkLayout:
    chunk_length: int
    chunks: tuple[Chunk, ...]
    param_to_chunk: Mapping[str, int]
    total_elements: int

    def __post_init__(self) -> None:
        object.__setattr__(self, "param_to_chunk", MappingProxyType(dict(self.param_to_chunk)))

    @property
    def n_chunks(self) -> int:
        return len(self.chunks)

    @property
    def aggregate_length(self) -> int:
        return self.n_chunks * self.chunk_length


@dataclass(frozen=True)
class ChunkTrace:
    forward: tuple[frozenset[int], ...]
    backward: tuple[frozenset[int], ...]
    reduce_after: Mapping[int, int]

    def __post_init__(self) -> None:
        object.__setattr__(self, "reduce_after", MappingProxyType(dict(self.reduce_after)))

    @property
    def chunk_ids(self) -> frozenset[int]:
        return frozenset(self.reduce_after)


def pack_chunks(sequence: Sequence[Any], chunk_length: int) -> ChunkLayout:
    """Greedy in-order packing of ``sequence`` (ParameterSpec-like records)."""
    lib = _lib.load()
    n = len(sequence)
    numel = np.ascontiguousarray([int(p.numel) for p in sequence], dtype=np.int64)
    chunk_of = np.zeros(n, dtype=np.int32)
    offset = np.zeros(n, dtype=np.int64)
    n_chunks = ctypes.c_int32(0)
    rc = lib.elx_layout_pack(numel.ctypes.data if n else None, n, int(chunk_length),
                             chunk_of.ctypes.data if n else None, offset.ctypes.data if n else None,
                             ctypes.byref(n_chunks))
    if rc != _lib.OK:
        msg = lib.elx_last_error().decode()
        # Name the parameter, as the reference does (chunking.py:106-111).
        if "#" in msg:
            idx = int(msg.split("#")[1].split()[0])
            msg = msg.replace(f"parameter #{idx}", f"parameter '{sequence[idx].id}'")
        _raise(rc, msg)
    members: list[list[ChunkMember]] = [[] for _ in range(n_chunks.value)]
    for p, c, o in zip(sequence, chunk_of.tolist(), offset.tolist()):
        members[c].append(ChunkMember(p.id, o, int(p.numel)))
    chunks = tuple(Chunk(i, int(chunk_length), tuple(ms)) for i, ms in enumerate(members))
    return ChunkLayout(int(chunk_length), chunks,
                       {p.id: c for p, c in zip(sequence, chunk_of.tolist())},
                       int(numel.sum()) if n else 0)


def _raise(rc: int, msg: str) -> None:
    from .errors import ChunkTooSmallError, InfeasibleCacheError
    if rc == _lib.ERR_CHUNK_TOO_SMALL:
        raise ChunkTooSmallError(msg)
    if rc == _lib.ERR_INFEASIBLE_CACHE:
        raise InfeasibleCacheError(msg)
    raise ValidationError(msg)


def waste_rate(layout: Any) -> float:
    """Padding fraction of the chunk storage (chunking.py:141-146)."""
    total = layout.n_chunks * layout.chunk_length
    return 0.0 if total == 0 else (total - layout.total_elements) / total


def build_chunk_trace(trace: Any, layout: Any) -> ChunkTrace:
    """Coarse parameter nodes -> chunk-id sets; backward mirrors forward and
    reduce_after[c] is c's last backward position (chunking.py:149-170)."""
    mapping = layout.param_to_chunk
    fwd = []
    for node in trace.coarse_ops:
        try:
            fwd.append(frozenset(mapping[pid] for pid in node))
        except KeyError as exc:
            raise ValidationError(
                f"parameter '{exc.args[0]}' in the access trace is not mapped to any chunk") from None
    bwd = tuple(fwd[::-1])
    last: dict[int, int] = {}
    for pos, ids in enumerate(bwd):
        last.update((c, pos) for c in ids)
    return ChunkTrace(tuple(fwd), bwd, last)


def working_set_blocks(trace: Any) -> int:
    """Most chunks any one coarse node needs at once (chunking.py:173-177)."""
    return max((len(s) for s in trace.forward), default=0)
