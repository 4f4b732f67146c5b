"""Rank-to-rank data movement for chunk fetch and gradient release.

Two exchange primitives cover the path:
  * gather  — all-gather of every rank's shard into an rCache block (fetch);
  * scatter — every rank sends segment r of its block to rank r, so that
    rank r holds all N copies of ITS segment; the release kernel (K3) then
    reduces them in fixed rank order in fp32. This is a reduce-scatter whose
    reduction runs in our kernel, giving rank-order-deterministic fp32
    results (NCCL's bf16 reduce-scatter accumulates in bf16 and in ring
    order, which cannot meet the 1e-6 parity bar).

Implementations:
  LocalTransport   world 1 (nothing moves between ranks);
  TorchDistTransport  torch.distributed collectives (NCCL over NVLink on the
                   GPU box; gloo on CPU for the multi-process host tests);
  IpcTransport     in-kernel P2P (the N > 1 default): K2/K3 read peers' HBM
                   through CUDA-IPC mappings opened on the rank's own device,
                   ordered by our device barrier kernel (also runs N processes
                   on one GPU);
  SymmMemTransport the same P2P path over torch symmetric-memory mappings
                   (one GPU per rank), same barrier kernel.
The P2P transports can run K2 on the copy engines (fetch_engine "ce").
Collectives are issued under the caller's current stream, so the comm
stream orders them with the K1-K3 launches around them.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import ValidationError


class LocalTransport:
    world = 1
    rank = 0

    def gather(self, block: torch.Tensor, shard: torch.Tensor) -> None:  # pragma: no cover - not used at world 1
        block[: shard.numel()].copy_(shard)

    def scatter(self, recv: torch.Tensor, block: torch.Tensor) -> None:  # pragma: no cover
        recv.copy_(block)

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        return None

    def barrier(self) -> None:
        return None


class TorchDistTransport:
    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)

    def gather(self, block: torch.Tensor, shard: torch.Tensor) -> None:
        """block[r*S:(r+1)*S] <- rank r's shard (S = shard.numel())."""
        out = block[: self.world * shard.numel()]
        if self.backend == "gloo":  # gloo has no all_gather_into_tensor
            dist.all_gather(list(out.chunk(self.world)), shard, group=self.group)
        else:
            dist.all_gather_into_tensor(out, shard, group=self.group)

    def scatter(self, recv: torch.Tensor, block: torch.Tensor) -> None:
        """recv[r*S:(r+1)*S] <- rank r's block[self.rank*S:(self.rank+1)*S]."""
        dist.all_to_all_single(recv, block[: recv.numel()], group=self.group)

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def barrier(self) -> None:
        dist.barrier(group=self.group)


class SymmMemTransport(TorchDistTransport):
    """In-kernel NVLink path over torch symmetric memory: rCache blocks, GPU-home
    shards and the barrier's signal pads are allocated in symmetric memory; K2
    (fetch) and K3 (release) read peers' HBM through the mapped pointers, and
    the stream-ordered barrier is our own device-numbered kernel
    (elx_device_barrier) over the symmetric pads, so a step captured as a CUDA
    graph replays it. Needs one GPU per rank (symmetric memory refuses ranks
    that share a device)."""

    p2p = True
    graph_safe = True

    def __init__(self, group=None, fetch_engine: str | None = None):
        super().__init__(group)
        import os

        import torch.distributed._symmetric_memory as symm

        from . import kernels

        # K2 on SMs ("sm", the fetch kernel) or on the copy engines ("ce")
        self.fetch_engine = fetch_engine or os.environ.get("ELX_FETCH_ENGINE", "sm")
        self.symm = symm
        self._kernels = kernels
        self.handles = []
        self._group = group if group is not None else dist.group.WORLD
        try:
            symm.enable_symm_mem_for_group(self._group.group_name)
        except Exception:  # newer torch enables it implicitly
            pass
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.pad = self.alloc((self.world + 1,), torch.int32, self.device)
        self.pad_ptrs = self.peer_ptrs(self.pad)

    def alloc(self, shape, dtype, device) -> torch.Tensor:
        t = self.symm.empty(*shape, dtype=dtype, device=device)
        t.zero_()
        return t

    def peer_ptrs(self, t: torch.Tensor) -> list[int]:
        """Device pointers of `t`'s counterpart on every rank (rank order)."""
        if t.numel() == 0:
            return [0] * self.world
        torch.cuda.current_stream(t.device).synchronize()
        h = self.symm.rendezvous(t, self._group)
        self.handles.append(h)
        base = h.buffer_ptrs[self.rank]
        off = t.data_ptr() - base
        return [int(p) + off for p in h.buffer_ptrs]

    def device_barrier(self) -> None:
        """All ranks' current streams reach this point before any continues."""
        self._kernels.device_barrier(self.pad_ptrs, self.rank, 0)


def _ipc_handle(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte cudaIpcMemHandle_t of the caching-allocator segment holding
    `t`, byte offset of t's data in that segment), via torch's own export."""
    st = t.untyped_storage()
    _, handle, _, storage_off, *_ = st._share_cuda_()
    h = bytes(handle)
    # torch's shareable form: [format version byte] + segment type ('c' = cudaMalloc, 'e' = expandable
    # segment) + the 64-byte cudaIpcMemHandle_t for 'c'; a bare 64-byte handle on older versions
    if len(h) > 64 and h[-65:-64] == b"c":
        h = h[-64:]
    if len(h) != 64:
        kind = "expandable segment" if b"e" in h[:2] else f"{len(h)}-byte handle {h[:2]!r}"
        raise ValidationError(f"IpcTransport needs cudaMalloc-backed segments, got a {kind} (unset "
                              "expandable_segments in PYTORCH_CUDA_ALLOC_CONF)")
    return h, int(storage_off) + t.storage_offset() * t.element_size()


class IpcTransport(TorchDistTransport):
    """The in-kernel P2P path over CUDA IPC: shards and rCache blocks are
    ordinary device tensors; every rank exports their allocations' IPC handles
    and maps its peers' with OUR elx_ipc_open on ITS OWN device (lazy peer
    access over NVLink), so each rank process keeps exactly one CUDA context
    (torch's rebuild_cuda_tensor would open the handle under the exporter's
    device and create a context there: eight per process on an 8-GPU node).
    The stream-ordered barrier is our device-numbered elx_device_barrier over
    IPC-mapped int32 signal pads, so a captured CUDA graph replays it. Works for
    ranks on different GPUs and for several processes sharing one GPU (which
    symmetric memory refuses), so the same path runs on the one-GPU test box."""

    p2p = True
    # The barrier numbers itself on the device, so a captured CUDA graph can replay it.
    graph_safe = True

    def __init__(self, group=None, fetch_engine: str | None = None):
        super().__init__(group)
        import os

        from . import kernels

        self.fetch_engine = fetch_engine or os.environ.get("ELX_FETCH_ENGINE", "sm")
        self._kernels = kernels
        self.device = torch.device("cuda", torch.cuda.current_device())
        self._opened: dict[bytes, int] = {}  # peer allocation handle -> base pointer in this process
        # signal pad: one arrival flag per rank + this rank's own barrier count
        self.pad = torch.zeros(self.world + 1, dtype=torch.int32, device=self.device)
        self.pad_ptrs = self.peer_ptrs(self.pad)

    def alloc(self, shape, dtype, device) -> torch.Tensor:
        return torch.zeros(shape, dtype=dtype, device=device)

    def peer_ptrs(self, t: torch.Tensor) -> list[int]:
        """Device pointers of `t`'s counterpart on every rank (rank order),
        usable by kernels on this rank's device."""
        if t.numel() == 0:
            return [0] * self.world
        torch.cuda.current_stream(t.device).synchronize()  # contents initialised before peers map it
        h, off = _ipc_handle(t)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, (t.device.index, h, off), group=self.group)
        ptrs = []
        for r, (dev_index, ph, poff) in enumerate(everyone):
            if r == self.rank:
                ptrs.append(t.data_ptr())
                continue
            if dev_index != t.device.index:
                self._kernels.enable_peer_access(dev_index)
            base = self._opened.get(ph)
            if base is None:
                base = self._opened[ph] = self._kernels.ipc_open(ph)
            ptrs.append(base + poff)
        dist.barrier(group=self.group)  # every rank has mapped before anyone frees or reuses
        return ptrs

    def close(self) -> None:
        """Unmap every peer allocation (call after a final barrier)."""
        for base in self._opened.values():
            self._kernels.ipc_close(base)
        self._opened.clear()

    def device_barrier(self) -> None:
        """All ranks' current streams reach this point before any continues."""
        self._kernels.device_barrier(self.pad_ptrs, self.rank, 0)


def primary_contexts() -> list[int]:
    """Device ordinals on which THIS process holds an active primary CUDA
    context (driver API). One rank process per GPU should report exactly its
    own device."""
    import ctypes

    lib = ctypes.CDLL("libcuda.so.1")
    out = []
    for d in range(torch.cuda.device_count()):
        dev = ctypes.c_int()
        if lib.cuDeviceGet(ctypes.byref(dev), d) != 0:
            continue
        flags, active = ctypes.c_uint(), ctypes.c_int()
        if lib.cuDevicePrimaryCtxGetState(dev, ctypes.byref(flags), ctypes.byref(active)) == 0 and active.value:
            out.append(d)
    return out


def resolve_kind(world_size: int, kind: str | None = None) -> str:
    """The N > 1 transport: "auto" (default) picks the in-kernel P2P path over
    our own IPC mappings ("ipc") when every rank can reach every peer's GPU
    (NVLink / NVSwitch peer access, or ranks sharing a GPU), and the NCCL
    exchange ("nccl") otherwise. Every rank gets the same answer."""
    import os

    kind = kind or os.environ.get("ELX_TRANSPORT", "auto")
    if world_size == 1:
        return "local"
    if kind != "auto":
        return kind
    me = torch.cuda.current_device()
    devs = [None] * world_size
    dist.all_gather_object(devs, me)
    ok = all(d == me or torch.cuda.can_device_access_peer(me, d) for d in devs)
    votes = [None] * world_size
    dist.all_gather_object(votes, ok)
    return "ipc" if all(votes) else "nccl"


def make_transport(world_size: int, kind: str | None = None):
    """kind: "auto" (default; see resolve_kind), "nccl" (torch.distributed
    collectives + K3), "ipc" (in-kernel P2P over our CUDA IPC mappings) or
    "p2p" (in-kernel P2P over torch symmetric memory); env ELX_TRANSPORT."""
    kind = resolve_kind(world_size, kind)
    if kind == "local":
        return LocalTransport()
    if kind == "p2p":
        return SymmMemTransport()
    if kind == "ipc":
        return IpcTransport()
    if kind == "ipc-ce":
        return IpcTransport(fetch_engine="ce")
    if kind == "nccl":
        return TorchDistTransport()
    raise ValueError(f"unknown transport {kind!r}")
