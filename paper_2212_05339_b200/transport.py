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
  SymmMemTransport   in-kernel P2P: K2/K3 read peers' HBM through torch
                   symmetric-memory mappings, symmetric-memory barriers;
  IpcTransport     the same P2P path over CUDA-IPC mappings and our own
                   device barrier kernel (also runs N processes on one GPU).
The P2P transports can run K2 on the copy engines (fetch_engine "ce").
Collectives are issued under the caller's current stream, so the comm
stream orders them with the K1-K3 launches around them.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


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
    """In-kernel NVLink path: rCache blocks and GPU-home shards are allocated
    in torch symmetric memory; K2 (fetch) and K3 (release) read peers' HBM
    through the mapped pointers, ordered by device-side barriers on the comm
    stream. Collectives not on that path (shared-parameter exchange, scalar
    all-reduce, CPU-home segments) stay on NCCL."""

    p2p = True

    def __init__(self, group=None, fetch_engine: str | None = None):
        super().__init__(group)
        import os

        import torch.distributed._symmetric_memory as symm

        # K2 on SMs ("sm", the fetch kernel) or on the copy engines ("ce")
        self.fetch_engine = fetch_engine or os.environ.get("ELX_FETCH_ENGINE", "sm")
        self.symm = symm
        self.handles = []
        self._group = group if group is not None else dist.group.WORLD
        try:
            symm.enable_symm_mem_for_group(self._group.group_name)
        except Exception:  # newer torch enables it implicitly
            pass

    def alloc(self, shape, dtype, device) -> torch.Tensor:
        t = self.symm.empty(*shape, dtype=dtype, device=device)
        t.zero_()
        return t

    def peer_ptrs(self, t: torch.Tensor) -> list[int]:
        """Device pointers of `t`'s counterpart on every rank (rank order)."""
        if t.numel() == 0:
            return [0] * self.world
        h = self.symm.rendezvous(t, self._group)
        self.handles.append(h)
        base = h.buffer_ptrs[self.rank]
        off = t.data_ptr() - base
        return [int(p) + off for p in h.buffer_ptrs]

    def device_barrier(self) -> None:
        """All ranks' comm streams reach this point before any continues."""
        self.handles[0].barrier(channel=0)


class IpcTransport(TorchDistTransport):
    """The same in-kernel P2P path without symmetric memory: shards and
    rCache blocks are ordinary device tensors exported with CUDA IPC (torch's
    CUDA tensor sharing), every rank maps its peers' allocations, and the
    stream-ordered device barrier is our own kernel (elx_device_barrier) over
    IPC-mapped int32 signal pads. Works for ranks on different GPUs (peer
    access over NVLink, enabled explicitly) and for several processes sharing
    one GPU, which symmetric memory refuses — so the P2P path can run in real
    separate processes on the one-GPU test box."""

    p2p = True

    def __init__(self, group=None, fetch_engine: str | None = None):
        super().__init__(group)
        import os

        from . import kernels

        self.fetch_engine = fetch_engine or os.environ.get("ELX_FETCH_ENGINE", "sm")
        self._kernels = kernels
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.peers: list[torch.Tensor] = []  # keep the peer mappings alive
        # signal pad: one arrival flag per rank + this rank's own barrier count
        self.pad = torch.zeros(self.world + 1, dtype=torch.int32, device=self.device)
        self.pad_ptrs = self.peer_ptrs(self.pad)

    def alloc(self, shape, dtype, device) -> torch.Tensor:
        return torch.zeros(shape, dtype=dtype, device=device)

    def peer_ptrs(self, t: torch.Tensor) -> list[int]:
        """Device pointers of `t`'s counterpart on every rank (rank order)."""
        if t.numel() == 0:
            return [0] * self.world
        from torch.multiprocessing.reductions import rebuild_cuda_tensor, reduce_tensor

        torch.cuda.current_stream(t.device).synchronize()  # contents initialised before peers map it
        _, args = reduce_tensor(t)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, (t.device.index, args), group=self.group)
        ptrs = []
        for r, (dev_index, a) in enumerate(everyone):
            if r == self.rank:
                ptrs.append(t.data_ptr())
                continue
            if dev_index != t.device.index:
                self._kernels.enable_peer_access(dev_index)
            peer = rebuild_cuda_tensor(*a)
            self.peers.append(peer)
            ptrs.append(peer.data_ptr())
        torch.cuda.set_device(t.device)
        dist.barrier(group=self.group)  # every rank has mapped before anyone frees or reuses
        return ptrs

    # The barrier numbers itself on the device, so a captured CUDA graph can replay it.
    graph_safe = True

    def device_barrier(self) -> None:
        """All ranks' current streams reach this point before any continues."""
        self._kernels.device_barrier(self.pad_ptrs, self.rank, 0)


def make_transport(world_size: int, kind: str | None = None):
    """kind: "nccl" (default), "p2p" (symmetric memory) or "ipc" (CUDA IPC
    peer mappings + our device barrier); env ELX_TRANSPORT."""
    import os

    if world_size == 1:
        return LocalTransport()
    kind = kind or os.environ.get("ELX_TRANSPORT", "nccl")
    if kind == "p2p":
        return SymmMemTransport()
    if kind == "ipc":
        return IpcTransport()
    return TorchDistTransport()
