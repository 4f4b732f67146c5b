"""Chunk manager, chunk fetcher and hybrid optimizer — the Elixir runtime.

This is the layer the reference leaves as prose (PAPER.md:170-181 chunks and
rCache, :203-206 wrapped operators, :221-238 gradient overwrite and the
paired optimizer chunk, :276-281 prefetch on streams) and whose schedule,
layout and memory contracts it pins in code (chunking.py:102-170,
rcache_sim.py:87-199, cost_model.py:147-153, search.py:116-126).

HBM layout per rank (N = world size, S = shard length = ceil(C/N) rounded up
to 8 elements so every shard starts 16-byte aligned):
  GPU-home chunks  p16 [G, S] compute dtype   (the rank's parameter shard)
                   p32/m/v [G, S] fp32        (paired optimizer chunk)
                   g32 [G, S] fp32            (reduced gradient shard)
  CPU-home chunks  the same five arrays in pinned host memory
  rCache           n_block blocks of N*S compute-dtype elements, when N > 1
                   or some chunk is CPU-homed. At N = 1 a GPU-home chunk's
                   shard IS the whole chunk and is used in place (its gathers
                   move no bytes but are still counted, as simulate counts
                   them).
  shared params    replicated compute copy + fp32 state shard (ZeRO-2
                   treatment, search.py:116-126), outside the chunks
                   (chunking.py:95-98).

All kernels come from libelixir_b200.so (kernels.py); torch is used for
memory, streams, events and collectives.
"""

from __future__ import annotations

import math
import os
import threading
import time
from dataclasses import dataclass
from typing import Any, Mapping, Sequence

import torch

from . import _lib, kernels
from .errors import InfeasibleCacheError, ValidationError
from .schedule import Device, Plan, Schedule, as_plan, compile_schedule, report_from_counters
from .transport import LocalTransport

# NVTX ranges around every fetch, release and optimizer step when ELX_NVTX=1
# (for nsys / ncu --nvtx timelines); a no-op otherwise.
_NVTX = os.environ.get("ELX_NVTX") == "1"


class _nvtx:
    __slots__ = ("name",)

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if _NVTX:
            torch.cuda.nvtx.range_push(self.name)

    def __exit__(self, *exc):
        if _NVTX:
            torch.cuda.nvtx.range_pop()

SHARD_ALIGN = 8  # elements; keeps every shard and rCache segment 16-byte aligned
ELX_TILE = _lib.ADAM_TILE
# (host update, GPU-streamed update) in elements/s, measured on the B200 box
# (plans/hardware_b200_measured.json: v_c = 19.5 GB/s of 4-byte elements;
# pinned PCIe ~55 GB/s each way at 14 B per element and direction).
DEFAULT_UPDATE_RATES = (19.5e9 / 4, 55e9 / 14)


def shard_length(chunk_length: int, world: int) -> int:
    s = -(-chunk_length // world)
    return -(-s // SHARD_ALIGN) * SHARD_ALIGN


@dataclass
class _SharedParam:
    pid: str
    numel: int
    shape: tuple[int, ...]
    shard: int               # Ssh
    full: torch.Tensor       # replicated compute copy [N*Ssh]
    grad: torch.Tensor       # replicated compute-dtype grad accumulator [N*Ssh]
    p16: torch.Tensor        # this rank's compute shard [Ssh] (== full at N=1)
    p32: torch.Tensor
    m: torch.Tensor
    v: torch.Tensor
    g32: torch.Tensor

    def valid(self, rank: int) -> int:
        return max(0, min(self.shard, self.numel - rank * self.shard))


class ChunkManager:
    """Owns every chunk shard, optimizer shard and rCache block of one rank.

    API mirrors the reference concepts: chunks of ``layout.chunk_length``
    elements at the layout's exact member offsets (chunking.py:113-131),
    homes and rCache size from the Plan (search.py:267-291).
    """

    def __init__(self, profile: Any, layout: Any, plan: Any, *, shapes: Mapping[str, Sequence[int]] | None = None,
                 transport=None, device=None, dtype: torch.dtype = torch.bfloat16,
                 shared_padded: Mapping[str, Sequence[int]] | None = None):
        self.plan: Plan = as_plan(plan)
        self.layout = layout
        self.transport = transport or LocalTransport()
        self.world = self.transport.world
        self.rank = self.transport.rank
        self.device = torch.device(device if device is not None else "cuda")
        self.dtype = dtype
        if dtype not in (torch.bfloat16, torch.float16):
            raise ValidationError("compute dtype must be bfloat16 or float16")
        if self.plan.chunk_length != layout.chunk_length:
            raise ValidationError(f"plan chunk_length {self.plan.chunk_length} != layout {layout.chunk_length}")
        n = layout.n_chunks
        ids = set(range(n))
        if set(self.plan.chunk_homes) != ids:
            # cli.py:255-259: a plan and a profile must pack into the same chunk ids.
            raise ValidationError(f"plan chunk ids {sorted(self.plan.chunk_homes)[:8]}... do not match the "
                                  f"layout's {n} chunks")
        self.n_chunks = n
        self.C = layout.chunk_length
        self.S = shard_length(self.C, self.world)
        self.P = self.S * self.world  # physical block length
        self.homes = [self.plan.chunk_homes[c] for c in range(n)]
        self.gpu_ids = [c for c in range(n) if self.homes[c] is Device.GPU]
        self.cpu_ids = [c for c in range(n) if self.homes[c] is Device.CPU]
        self.row = {}
        for i, c in enumerate(self.gpu_ids):
            self.row[c] = i
        for i, c in enumerate(self.cpu_ids):
            self.row[c] = i
        self.used = [sum(m.numel for m in ch.members) for ch in layout.chunks]
        self.members = {m.param_id: (ch.id, m.offset, m.numel) for ch in layout.chunks for m in ch.members}
        shared_ids = [p.id for p in profile.parameters if p.shared]
        self.shapes = {p.id: (tuple(shapes[p.id]) if shapes and p.id in shapes else (p.numel,))
                       for p in profile.parameters}
        for pid, (c, off, numel) in self.members.items():
            if math.prod(self.shapes[pid]) != numel:
                raise ValidationError(f"shape {self.shapes[pid]} of '{pid}' does not hold {numel} elements")

        dev, S = self.device, self.S
        G, H = len(self.gpu_ids), len(self.cpu_ids)
        f32 = torch.float32
        # In-kernel NVLink path: shards and rCache blocks live in symmetric
        # memory so K2/K3 read peers' buffers directly (transport.alloc).
        self.p2p = bool(getattr(self.transport, "p2p", False)) and self.world > 1
        peer_alloc = (lambda shape: self.transport.alloc(shape, dtype, dev)) if self.p2p else \
            (lambda shape: torch.zeros(shape, dtype=dtype, device=dev))
        # ---- GPU-home arenas
        self.p16 = peer_alloc((G, S))  # at N=1, S == P: the whole chunk
        self.p32 = torch.zeros(G, S, dtype=f32, device=dev)
        self.m = torch.zeros(G, S, dtype=f32, device=dev)
        self.v = torch.zeros(G, S, dtype=f32, device=dev)
        # World 1: the reduce-scatter is the identity, so the gradient stays in
        # the compute-dtype chunk; K3 only produces the norm/overflow and K4
        # unscales the compute-dtype gradient in-register (same IEEE ops). No
        # fp32 grad shard: the footprint is exactly chunk_footprint.
        self.fused_w1 = self.world == 1
        self.g32 = torch.zeros(G, 0 if self.fused_w1 else S, dtype=f32, device=dev)
        # ---- CPU-home arenas (pinned)
        pin = torch.cuda.is_available()
        self.h_p16 = torch.zeros(H, S, dtype=dtype, pin_memory=pin)
        self.h_p32 = torch.zeros(H, S, dtype=f32, pin_memory=pin)
        self.h_m = torch.zeros(H, S, dtype=f32, pin_memory=pin)
        self.h_v = torch.zeros(H, S, dtype=f32, pin_memory=pin)
        # host gradient landing buffer: fp32 reduced shard, or (world 1) the
        # compute-dtype gradient — half the D2H bytes
        self.h_g32 = torch.zeros(H, S, dtype=dtype if self.fused_w1 else f32, pin_memory=pin)
        # ---- rCache blocks and release staging
        self.alias = self.world == 1
        need_blocks = self.world > 1 or H > 0
        nb = self.plan.n_block if need_blocks else 0
        self.blocks = peer_alloc((nb, self.P))
        # peer base pointers of the same tensors on every rank (P2P only)
        self.peer_p16 = self.transport.peer_ptrs(self.p16) if self.p2p else None
        self.peer_blocks = self.transport.peer_ptrs(self.blocks) if self.p2p else None
        self.recv = torch.zeros(self.P if self.world > 1 else 0, dtype=dtype, device=dev)
        self.stage32 = torch.zeros(S if (H > 0 and not self.fused_w1) else 0, dtype=f32, device=dev)
        # ---- shared (multi-use) parameters: replicated copy + partitioned state
        self.shared: dict[str, _SharedParam] = {}
        for pid in shared_ids:
            numel = next(p.numel for p in profile.parameters if p.id == pid)
            ssh = shard_length(numel, self.world)
            # The compute copy may be over-allocated so the model can view it
            # with padded rows (e.g. vocab rounded up for aligned GEMMs); the
            # pad is never written (Adam touches valid elements only).
            pad_shape = tuple(shared_padded[pid]) if shared_padded and pid in shared_padded else None
            full_len = max(ssh * self.world, math.prod(pad_shape) if pad_shape else 0)
            full = torch.zeros(full_len, dtype=dtype, device=dev)
            # P2P: the shard peers gather from and the gradient peers reduce from are peer-mapped
            p16 = full[self.rank * ssh:(self.rank + 1) * ssh] if self.world == 1 else peer_alloc((ssh,))
            grad = peer_alloc((ssh * self.world,)) if self.p2p else torch.zeros(ssh * self.world, dtype=dtype,
                                                                                  device=dev)
            self.shared[pid] = _SharedParam(
                pid, numel, self.shapes[pid], ssh, full, grad, p16,
                torch.zeros(ssh, dtype=f32, device=dev), torch.zeros(ssh, dtype=f32, device=dev),
                torch.zeros(ssh, dtype=f32, device=dev),
                torch.zeros(0 if self.world == 1 else ssh, dtype=f32, device=dev))
        self.peer_shared = ({pid: (self.transport.peer_ptrs(sp.p16), self.transport.peer_ptrs(sp.grad))
                             for pid, sp in self.shared.items()} if self.p2p else {})
        # step scalars: [0] sum g^2, [1] overflow flag (elx_release / elx_adam); on the P2P path
        # peer-mapped, so the N-scalar all-reduce is a rank-ordered read of the peers' values
        if self.p2p:
            self.step_scalars = self.transport.alloc((kernels.STEP_SCALARS,), torch.float64, dev)
            self.peer_scalars = self.transport.peer_ptrs(self.step_scalars)
            self._scalar_tmp = torch.zeros(2, dtype=torch.float64, device=dev)
        else:
            self.step_scalars = kernels.new_step_scalars(dev)
            self.peer_scalars = None
        self._bound: dict[int, torch.Tensor] = {}   # chunk -> storage it is bound to
        # CPU-home chunks whose rCache block holds their current parameters (the resident streamed update,
        # HybridAdam.attach_fetcher): their gather copies nothing; cleared whenever the host copies are rewritten
        self.in_block: set[int] = set()
        self._views: dict[str, torch.Tensor] = {}

    def all_reduce_scalars(self) -> None:
        """Sum step_scalars[0:2] (sum of squares, overflow flag) over ranks on
        the current stream: NCCL all-reduce, or on the P2P path barrier ->
        rank-ordered read of every peer's scalars -> barrier -> write back
        (deterministic, no collective library)."""
        if self.world == 1:
            return
        if not self.p2p:
            self.transport.all_reduce_sum(self.step_scalars[:2])
            return
        self.transport.device_barrier()
        kernels.peer_sum_f64(self._scalar_tmp, self.peer_scalars, 2)
        self.transport.device_barrier()  # every rank has read before anyone overwrites
        self.step_scalars[:2].copy_(self._scalar_tmp)

    def gather_shared(self, sp: "_SharedParam") -> None:
        """Rebuild the replicated compute copy of a shared parameter from every
        rank's updated shard (after the optimizer step): NCCL all-gather, or K2
        over the peers' shards after a device barrier on the P2P path."""
        if self.world == 1:
            return
        if not self.p2p:
            self.transport.gather(sp.full[:sp.shard * self.world], sp.p16)
            return
        self.transport.device_barrier()  # every rank's K4 has written its shard
        kernels.fetch(sp.full, self.peer_shared[sp.pid][0], sp.shard, rank=self.rank)

    # ------------------------------------------------------------ sizes
    def valid(self, c: int, rank: int | None = None) -> int:
        """Elements of chunk c that are real parameters inside `rank`'s shard."""
        r = self.rank if rank is None else rank
        return max(0, min(self.S, self.used[c] - r * self.S))

    def memory_report(self) -> dict:
        t = lambda *xs: sum(x.numel() * x.element_size() for x in xs)
        return {
            "gpu_chunk_state_bytes": t(self.p16, self.p32, self.m, self.v),
            "gpu_grad_shard_bytes": t(self.g32),
            "rcache_bytes": t(self.blocks),
            "host_chunk_state_bytes": t(self.h_p16, self.h_p32, self.h_m, self.h_v, self.h_g32),
            "shared_bytes": sum(t(s.full, s.grad, s.p32, s.m, s.v, s.g32) + (0 if self.world == 1 else t(s.p16))
                                for s in self.shared.values()),
        }

    def memory_ledger(self) -> dict:
        """This rank's share of the whole-model states in the contract's terms
        (mixed_precision_states, cost_model.py:156-167): the compute-dtype
        parameter bytes it owns, the gradient bytes (the gradient overwrites
        the parameter's slot in the chunk, so it occupies the
        same bytes; at N > 1 the reduced fp32 shard is extra and listed
        separately) and the fp32 master/m/v bytes. Summed over ranks, every
        element is owned exactly once: params/grads = Lc*M, optimizer =
        Los*Fos*M, the contract's triple."""
        lc = torch.tensor([], dtype=self.dtype).element_size()
        owned = sum(self.valid(c) for c in range(self.n_chunks)) + \
            sum(sp.valid(self.rank) for sp in self.shared.values())
        return {"param_bytes": lc * owned, "grad_bytes": lc * owned, "optimizer_bytes": 12 * owned,
                "reduced_grad_shard_bytes": 0 if self.world == 1 else 4 * owned, "owned_elements": owned}

    # ------------------------------------------------------------ init
    def load_params(self, tensors: Mapping[str, torch.Tensor]) -> None:
        """Pack initial parameters into chunks (K1) and seed the fp32 masters."""
        self.in_block.clear()
        dev = self.device
        tmp16 = torch.empty(self.P, dtype=self.dtype, device=dev)
        tmp32 = torch.empty(self.P, dtype=torch.float32, device=dev)
        lo, hi = self.rank * self.S, (self.rank + 1) * self.S
        for ch in self.layout.chunks:
            mem = []
            for m in ch.members:
                t = tensors[m.param_id]
                if t.numel() != m.numel:
                    raise ValidationError(f"'{m.param_id}' has {t.numel()} elements, layout says {m.numel}")
                mem.append((t.detach().to(dev).reshape(-1), m.offset))
            kernels.chunk_pack(tmp16, mem, used_len=ch.used_elements)
            kernels.chunk_pack(tmp32, mem, used_len=ch.used_elements)
            r = self.row[ch.id]
            if self.homes[ch.id] is Device.GPU:
                if self.alias:
                    self.p16[r].copy_(tmp16)
                else:
                    self.p16[r].copy_(tmp16[lo:hi])
                self.p32[r].copy_(tmp32[lo:hi])
            else:
                self.h_p16[r].copy_(tmp16[lo:hi])
                self.h_p32[r].copy_(tmp32[lo:hi])
        for sp in self.shared.values():
            t = tensors[sp.pid].detach().to(dev).reshape(-1)
            kernels.chunk_pack(sp.full, [(t, 0)], used_len=sp.numel)
            lo_s, hi_s = self.rank * sp.shard, (self.rank + 1) * sp.shard
            kernels.chunk_pack(sp.p32, [(t[lo_s:min(hi_s, sp.numel)], 0)], used_len=max(0, min(hi_s, sp.numel) - lo_s))
            if self.world > 1:
                sp.p16.copy_(sp.full[lo_s:hi_s])
        torch.cuda.synchronize(dev)

    # ------------------------------------------------------------ views
    def home_storage(self, c: int) -> torch.Tensor:
        """N=1 GPU-home chunk storage (used in place)."""
        return self.p16[self.row[c]]

    def bind(self, c: int, storage: torch.Tensor) -> None:
        self._bound[c] = storage
        for m in self.layout.chunks[c].members:
            self._views[m.param_id] = storage[m.offset:m.offset + m.numel].view(self.shapes[m.param_id])

    def unbind(self, c: int) -> None:
        self._bound.pop(c, None)
        for m in self.layout.chunks[c].members:
            self._views.pop(m.param_id, None)

    def storage(self, c: int) -> torch.Tensor:
        try:
            return self._bound[c]
        except KeyError:
            raise InfeasibleCacheError(f"chunk {c} is not resident in the rCache") from None

    def param(self, pid: str) -> torch.Tensor:
        """Current compute-dtype view of a parameter (chunk member or shared)."""
        v = self._views.get(pid)
        if v is not None:
            return v
        sp = self.shared.get(pid)
        if sp is not None:
            return sp.full[:sp.numel].view(sp.shape)
        raise InfeasibleCacheError(f"parameter '{pid}' is not resident (its chunk was not fetched)")

    def padded_param(self, pid: str, shape: Sequence[int]) -> torch.Tensor:
        """A shared parameter viewed with zero padding (see shared_padded)."""
        sp = self.shared[pid]
        n = math.prod(shape)
        if n > sp.full.numel():
            raise ValidationError(f"padded view {tuple(shape)} exceeds the allocation of '{pid}'")
        return sp.full[:n].view(tuple(shape))

    # ------------------------------------------------------------ export
    def master_params(self) -> dict[str, torch.Tensor]:
        """fp32 master values of this rank's shards, reassembled per parameter
        for the members this rank owns completely (world 1: all of them)."""
        out = {}
        for pid, (c, off, numel) in self.members.items():
            lo = self.rank * self.S
            if off < lo or off + numel > lo + self.S:
                continue
            r = self.row[c]
            src = self.p32[r] if self.homes[c] is Device.GPU else self.h_p32[r]
            out[pid] = src[off - lo:off - lo + numel].view(self.shapes[pid]).clone()
        return out


class ChunkFetcher:
    """Replays the compiled rCache program: gathers (with Belady victims and
    one-position prefetch on the comm stream), pins, and releases.

    Live counters carry SimReport's field names and must equal
    offplan.simulate for the same trace/plan (rcache_sim.py:87-199).
    """

    def __init__(self, manager: ChunkManager, trace: Any, *, comm_stream: torch.cuda.Stream | None = None,
                 prefetch: bool = True, inv_scale: float = 1.0):
        self.mgr = manager
        self.trace = trace
        plan = manager.plan
        self.sched: Schedule = compile_schedule(trace, plan.n_block, plan.chunk_homes, manager.n_chunks)
        self.n_fwd = self.sched.n_forward
        self.walk = list(trace.forward) + list(trace.backward)
        self.comm = comm_stream or torch.cuda.Stream(device=manager.device)
        self.prefetch = prefetch
        self.inv_scale = inv_scale
        self.time_release = False     # bench: CUDA events around each release / offload copy
        self.release_events: list = []
        self.fetch_events: list = []      # (start, end, block elements) per GPU-home gather at N > 1
        self.copy_events: list = []
        self.optimizer = None         # HybridAdam whose per-chunk updates gate our reads
        self._fenced = False
        ev = self.sched.events
        W = 2 * self.n_fwd
        self.due = [[] for _ in range(W)]
        self.early = [[] for _ in range(W)]
        self.reduces = [[] for _ in range(W)]
        # no eviction anywhere in the program: every chunk is gathered into the same block each step and that
        # block holds nothing else (HybridAdam.attach_fetcher keeps streamed chunks' state there between steps)
        self.stable_blocks = all(int(e["victim"]) < 0 for e in ev if int(e["kind"]) != _lib.EV_REDUCE)
        self.block_for = {int(e["chunk"]): int(e["block"]) for e in ev if int(e["kind"]) != _lib.EV_REDUCE}
        for e in ev:
            rec = (int(e["chunk"]), int(e["block"]), int(e["victim"]), int(e["pos"]))
            if int(e["kind"]) == _lib.EV_REDUCE:
                self.reduces[int(e["pos"])].append(rec[0])
            elif prefetch and int(e["issue_pos"]) < int(e["pos"]):
                self.early[int(e["issue_pos"])].append(rec)
            else:
                self.due[int(e["pos"])].append(rec)
        self._reset()

    # ------------------------------------------------------------ state
    def _reset(self) -> None:
        for c in list(self.mgr._bound):
            self.mgr.unbind(c)
        self.block_of: dict[int, int] = {}
        self.ready: dict[int, torch.cuda.Event] = {}
        self.last_use: dict[int, torch.cuda.Event] = {}
        self.gathered: set[int] = set()
        self.live = dict(gather_ops=0, replaced_ops=0, reduce_ops=0, c2g_units=0, g2c_units=0,
                         peak_rcache_blocks=0)
        self.bytes_moved = dict(h2d=0, d2h=0, gather=0, scatter=0)
        self.pos = 0
        self._fenced = False
        self.deferred: dict[int, list] = {}
        self._dirty: set[int] = set()   # P2P: blocks released since the last device barrier

    def begin_step(self, after: torch.cuda.Event | None = None) -> None:
        """Start a walk. The comm stream is forked from the compute stream
        (and made to wait on `after`, the previous optimizer step's event):
        every gather of this step reads shards that step's K4 rewrote — on
        every transport, not only P2P — and during a CUDA graph capture the
        fork brings the comm stream into the capture. On the P2P path every
        rank must also have finished its previous optimizer step before anyone
        reads its shards: one device barrier on the comm stream."""
        self._reset()
        self.comm.wait_stream(torch.cuda.current_stream(self.mgr.device))
        if after is not None:
            self.comm.wait_event(after)
        if self.mgr.p2p:
            with torch.cuda.stream(self.comm):
                self.mgr.transport.device_barrier()

    # ------------------------------------------------------------ walk
    def enter(self, pos: int) -> None:
        """Before node `pos` computes: make its chunks resident and bound."""
        if pos != self.pos:
            raise ValidationError(f"walk out of order: expected position {self.pos}, got {pos}")
        for rec in self.deferred.pop(pos, []) + self.due[pos]:
            self._gather(rec)
        opt = self.optimizer
        for rec in self.early[pos]:  # prefetch, up to the schedule's horizon
            c = rec[0]
            if (opt is not None and self.mgr.world == 1 and self.mgr.homes[c] is Device.CPU
                    and c in opt.cpu_ready and not opt.cpu_ready[c].is_set()):
                # its host update is still running: issue at the due position instead of blocking here.
                # Only at world 1: with several ranks the choice depends on host timing, so ranks could
                # issue their gathers (collectives, or barrier-ordered peer reads) in different orders;
                # there _gather blocks on the update instead and the issue order stays the schedule's.
                self.deferred.setdefault(rec[3], []).append(rec)
                continue
            self._gather(rec)
        cur = torch.cuda.current_stream(self.mgr.device)
        opt = self.optimizer
        for c in self.walk[pos]:
            if c not in self.block_of:
                raise InfeasibleCacheError(f"chunk {c} needed at position {pos} is not resident")
            ev = self.ready.pop(c, None)
            if ev is not None:
                cur.wait_event(ev)
            elif opt is not None and self.mgr.alias:
                opt.wait_gpu(c, cur)  # N=1 in-place chunk: its own update must be done
        self.live["peak_rcache_blocks"] = max(self.live["peak_rcache_blocks"], len(self.block_of))

    def after_compute(self, pos: int) -> None:
        """After node `pos` (and, in backward, its gradient write-back)."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.mgr.device))
        for c in self.walk[pos]:
            self.last_use[c] = ev
        if pos >= self.n_fwd and self.reduces[pos]:
            self._release_group(self.reduces[pos], ev)
        self.pos = pos + 1

    # names used by SURVEY.md §8b for the reference runtime's chunk-fetcher
    def fetch(self, pos: int) -> None:
        """Make the chunks of walk position `pos` resident (alias of enter)."""
        self.enter(pos)

    def finish(self) -> torch.cuda.Event:
        """End of the walk: every release is enqueued; returns their event."""
        if self.pos != 2 * self.n_fwd:
            raise ValidationError(f"walk ended at position {self.pos} of {2 * self.n_fwd}")
        done = torch.cuda.Event()
        done.record(self.comm)
        return done

    def counters(self) -> dict:
        return dict(self.live)

    def report(self, precision=None, hardware=None):
        from .profiles import PrecisionSpec
        return report_from_counters(self.live, self.trace, self.mgr.C, self.mgr.plan.chunk_homes,
                                    precision or PrecisionSpec(), self.mgr.world, hardware)

    # ------------------------------------------------------------ events
    def _gather(self, rec) -> None:
        with _nvtx(f"elx.fetch c{rec[0]} b{rec[1]}"):
            self._gather_impl(rec)

    def _gather_impl(self, rec) -> None:
        c, b, victim, pos = rec
        mgr = self.mgr
        if victim >= 0:
            if self.block_of.get(victim) != b:
                raise InfeasibleCacheError(f"schedule desync: victim {victim} not in block {b}")
            del self.block_of[victim]
            mgr.unbind(victim)
        self.block_of[c] = b
        self.live["gather_ops"] += 1
        if c in self.gathered:
            self.live["replaced_ops"] += 1
        self.gathered.add(c)
        cpu = mgr.homes[c] is Device.CPU
        if cpu:
            self.live["c2g_units"] += 1
        if mgr.alias and not cpu:
            mgr.bind(c, mgr.home_storage(c))  # the shard is the whole chunk: no bytes move
            return
        block = mgr.blocks[b]
        comm = self.comm
        opt = self.optimizer
        if cpu and opt is not None:
            opt.wait_offloaded(c, self.comm)  # host shard rewritten by the CPU-home update
        with torch.cuda.stream(comm):
            if victim >= 0 and victim in self.last_use:
                comm.wait_event(self.last_use[victim])
            if not cpu and opt is not None:
                opt.wait_gpu(c, comm)
            if mgr.p2p and b in self._dirty:
                self._barrier()  # peers may still be reading block b's gradients (released since the last barrier)
            seg = block[mgr.rank * mgr.S:(mgr.rank + 1) * mgr.S]
            if self.time_release and not cpu and mgr.world > 1:
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(comm)
            if mgr.p2p and not cpu:
                # K2 over NVLink: read every rank's shard of c straight from its HBM
                es = block.element_size()
                off = mgr.row[c] * mgr.S * es
                kernels.fetch(block, [p + off for p in mgr.peer_p16], mgr.S, stream=comm,
                              engine=getattr(mgr.transport, "fetch_engine", "sm"), rank=mgr.rank)
            elif cpu and c in mgr.in_block:
                pass  # the streamed update wrote this chunk's parameters into its block (attach_fetcher)
            elif cpu:
                if self.time_release:
                    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    c0.record(comm)
                kernels.copy_h2d(seg, mgr.h_p16[mgr.row[c]], stream=comm)
                if self.time_release:
                    c1.record(comm)
                    self.copy_events.append(("h2d", c0, c1, seg.numel() * seg.element_size()))
                self.bytes_moved["h2d"] += seg.numel() * seg.element_size()
                if mgr.world > 1 and mgr.p2p:
                    # every rank has landed its segment of block b; read the others' over peer memory
                    es = block.element_size()
                    off = b * mgr.P * es
                    self._barrier()
                    kernels.fetch(block, [p + off + r * mgr.S * es for r, p in enumerate(mgr.peer_blocks)], mgr.S,
                                  stream=comm, engine=getattr(mgr.transport, "fetch_engine", "sm"), rank=mgr.rank)
                    self._barrier()  # peers may reuse block b (its gradients, later) only after every rank read it
                elif mgr.world > 1:
                    mgr.transport.gather(block, seg)
            else:
                mgr.transport.gather(block, mgr.p16[mgr.row[c]])
            if self.time_release and not cpu and mgr.world > 1:
                f1.record(comm)
                self.fetch_events.append((f0, f1, mgr.P))
            if mgr.world > 1:
                self.bytes_moved["gather"] += (mgr.world - 1) * mgr.S * block.element_size()
            ev = torch.cuda.Event()
            ev.record(comm)
        self.ready[c] = ev
        mgr.bind(c, block)

    def release(self, chunks) -> None:
        """Release chunk(s) now (SURVEY.md §8b `release(chunk)`): the
        reduce-scatter of their gradients, written by the current stream, into
        this rank's fp32 shards with the unscale, the sum of squares and the
        overflow flag — one K3 launch for all of them. The schedule replay
        calls this itself at each chunk's reduce position (after_compute)."""
        cs = [int(chunks)] if isinstance(chunks, int) else [int(c) for c in chunks]
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.mgr.device))
        self._release_group(cs, ev)

    def _barrier(self) -> None:
        """Device barrier on the comm stream (P2P). Every rank has then finished
        its earlier comm work, including its K3 reads of our blocks."""
        self.mgr.transport.device_barrier()
        self._dirty.clear()

    def _release_group(self, cs, grads_written: torch.cuda.Event) -> None:
        with _nvtx(f"elx.release {cs}"):
            self._release_impl(cs, grads_written)

    def _release_impl(self, cs, grads_written: torch.cuda.Event) -> None:
        """Every chunk due at one reduce position (rcache_sim.py:160-167): one
        K3 launch over all of them (per-chunk launches only for CPU-home chunks
        at N > 1, which share the fp32 staging buffer of their D2H). On the P2P
        path one device barrier precedes it (every rank's gradients are in its
        blocks); the blocks are then 'dirty' — peers may still be reading them
        — until the next barrier, which a gather into one of them issues first."""
        mgr = self.mgr
        comm = self.comm
        opt = self.optimizer
        es = mgr.p16.element_size()
        batch, staged = [], []
        for c in cs:
            self.live["reduce_ops"] += 1
            cpu = mgr.homes[c] is Device.CPU
            if cpu:
                self.live["g2c_units"] += 1
                if opt is not None:
                    opt.wait_offloaded(c, self.comm)  # previous update still reading the host grad shard
            (staged if cpu and not mgr.fused_w1 else batch).append(c)
        with torch.cuda.stream(comm):
            comm.wait_event(grads_written)
            if not self._fenced and opt is not None and opt.done_event is not None:
                comm.wait_event(opt.done_event)  # g32 / step scalars free again
                self._fenced = True
            if mgr.p2p:
                self._barrier()
            if self.time_release:  # after the barrier: the K3 launch itself (bus/HBM rate), not the wait
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(comm)
            segs = []
            exchange = mgr.world > 1 and not mgr.p2p
            for c in batch:
                if exchange:
                    # the all-to-all lands every rank's copy of our segment in the ONE receive buffer, so each
                    # chunk's K3 runs before the next chunk's exchange; and every rank joins every collective,
                    # also for a chunk whose tail leaves this rank no valid elements
                    srcs = self._release_srcs(c)
                    if mgr.valid(c) > 0:
                        kernels.release_batch([(mgr.g32[mgr.row[c]], srcs, mgr.valid(c))], mgr.dtype,
                                              self.inv_scale, mgr.step_scalars, stream=comm)
                elif mgr.valid(c) > 0:
                    segs.append((None if mgr.fused_w1 else mgr.g32[mgr.row[c]], self._release_srcs(c), mgr.valid(c)))
            if segs:
                kernels.release_batch(segs, mgr.dtype, self.inv_scale, mgr.step_scalars, stream=comm)
            if self.time_release:
                t1.record(comm)
                self.release_events.append((t0, t1, sum(n for _, _, n in segs)))
            for c in cs:
                if mgr.world > 1:
                    self.bytes_moved["scatter"] += (mgr.world - 1) * mgr.S * es
                if mgr.p2p:
                    self._dirty.add(self.block_of[c])
                n = mgr.valid(c)
                if mgr.homes[c] is not Device.CPU:
                    continue
                if c in staged:  # CPU-home at N > 1: reduce into the fp32 staging shard, then D2H it
                    srcs = self._release_srcs(c)  # a collective on the exchange path: joined even when n == 0
                    if n > 0:
                        kernels.release(mgr.stage32, srcs, n, mgr.dtype, self.inv_scale, mgr.step_scalars,
                                        stream=comm)
                if n == 0:
                    continue
                if opt is not None and c in opt.resident:
                    continue  # its streamed update reads the gradient from the block itself
                src = mgr.storage(c) if mgr.fused_w1 else mgr.stage32
                nbytes = n * src.element_size()
                if self.time_release:
                    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    c0.record(comm)
                kernels.copy_d2h(mgr.h_g32[mgr.row[c]], src, nbytes, stream=comm)
                if self.time_release:
                    c1.record(comm)
                    self.copy_events.append(("d2h", c0, c1, nbytes))
                self.bytes_moved["d2h"] += nbytes

    def _release_srcs(self, c: int) -> list[int]:
        """Per-rank device pointers of this rank's segment of chunk c's gradients."""
        mgr = self.mgr
        storage = mgr.storage(c)
        es = storage.element_size()
        if mgr.world == 1:
            return [storage.data_ptr()]
        if mgr.p2p:
            # K3 over NVLink: segment `rank` of every rank's copy of block b, in rank order
            off = (self.block_of[c] * mgr.P + mgr.rank * mgr.S) * es
            return [p + off for p in mgr.peer_blocks]
        mgr.transport.scatter(mgr.recv, storage)
        return [mgr.recv.data_ptr() + r * mgr.S * es for r in range(mgr.world)]

    def release_shared(self, sp: _SharedParam) -> None:
        """Release of a shared parameter's gradient (after its last use)."""
        mgr = self.mgr
        comm = self.comm
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(mgr.device))
        with torch.cuda.stream(comm):
            comm.wait_event(ev)
            opt = self.optimizer
            if not self._fenced and opt is not None and opt.done_event is not None:
                comm.wait_event(opt.done_event)
                self._fenced = True
            if mgr.world == 1:
                srcs = [sp.grad.data_ptr()]
            elif mgr.p2p:
                # K3 straight over every rank's replicated gradient (segment `rank`); peers may read our
                # gradient until the next barrier (the optimizer step's scalar all-reduce), and it is
                # rewritten only in the next step's backward, after begin_step's barrier
                self._barrier()
                es = sp.grad.element_size()
                srcs = [p + mgr.rank * sp.shard * es for p in mgr.peer_shared[sp.pid][1]]
            else:
                recv = torch.empty_like(sp.grad)
                mgr.transport.scatter(recv, sp.grad)
                recv.record_stream(comm)
                es = recv.element_size()
                srcs = [recv.data_ptr() + r * sp.shard * es for r in range(mgr.world)]
            n = sp.valid(mgr.rank)
            if self.time_release:
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record(comm)
            if n > 0:
                kernels.release(None if mgr.fused_w1 else sp.g32, srcs, n, mgr.dtype, self.inv_scale,
                                mgr.step_scalars, stream=comm)
            if self.time_release:
                t1.record(comm)
                self.release_events.append((t0, t1, n))


class StepStats:
    """Result of one optimizer step; reading it synchronises with the step's
    scalar snapshot only (not the whole device)."""

    def __init__(self, host_slot: torch.Tensor, ready: torch.cuda.Event):
        self._slot, self._ready, self._vals = host_slot, ready, None

    def scalars(self) -> tuple[float, float]:
        if self._vals is None:
            self._ready.synchronize()
            self._vals = (float(self._slot[0]), float(self._slot[1]))
        return self._vals

    @property
    def found_inf(self) -> bool:
        sq, flag = self.scalars()
        return flag != 0.0 or not math.isfinite(sq)

    @property
    def grad_norm(self) -> float:
        sq, _ = self.scalars()
        return math.sqrt(sq) if math.isfinite(sq) else float("inf")

    def __iter__(self):  # (found_inf, grad_norm) unpacking, as the host-sync API returned
        yield self.found_inf
        yield self.grad_norm


class HybridAdam:
    """Chunk-wise fused mixed-precision AdamW: GPU-home shards on the device
    (K4, update rate v_g), CPU-home shards on host threads (elx_cpu_adam,
    rate v_c), with global grad-norm clipping and overflow skip
    (rcache_sim.py:173-184).

    The CPU-home update always runs on a host thread (the GPU keeps going);
    the next step's fetch of a CPU-home chunk waits for that chunk's flag.
    With ``overlap`` the GPU update is also issued per chunk in forward-use
    order on an optimizer stream and the next forward waits per chunk. On
    B200 this measured no gain (the persistent K4 grid holds every SM, so
    the forward's GEMMs queue behind it: 107.95 vs 107.94 ms per step,
    profiles/r01_overlap.md) and it blurs K4's own timing, so the default is
    one K4 launch over all GPU-home shards right after the backward.
    """

    def __init__(self, manager: ChunkManager, *, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.01, max_norm: float | None = 1.0, cpu_threads: int | None = None,
                 overlap: bool = False, device_step: bool = True, cpu_update: str = "split",
                 update_rates: tuple[float, float] | None = None, stream_tile: int = 32 * 2 ** 20,
                 max_grad_norm: float | None = None):
        if max_grad_norm is not None:  # SURVEY.md §8b's name for max_norm
            max_norm = max_grad_norm
        self.mgr = manager
        self.hp = dict(lr=lr, beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay,
                       max_norm=max_norm or 0.0)
        self.cpu_threads = cpu_threads or max(1, min(32, len(os.sched_getaffinity(0))))
        self.overlap = overlap
        m = manager
        # groups in forward-use order: shared params (used by the first node), then chunks by id
        self.groups: list[tuple[object, kernels.AdamTable]] = []
        all_segs = []
        self.gpu_segments: list[tuple[object, tuple]] = []  # (shared pid or chunk id, K4 segment), table order
        for pid, sp in m.shared.items():
            n = sp.valid(m.rank)
            if n > 0:
                seg = (sp.p32, sp.m, sp.v, sp.grad if m.fused_w1 else sp.g32, sp.p16, n)
                all_segs.append(seg)
                self.gpu_segments.append((pid, seg))
                self.groups.append((pid, kernels.AdamTable([seg], m.device)))
        for c in m.gpu_ids:
            r = m.row[c]
            n = m.valid(c)
            if n > 0:
                # world 1: the gradient is read from the chunk itself (bf16) and
                # overwritten in place by the new parameter
                seg = (m.p32[r], m.m[r], m.v[r], m.p16[r] if m.fused_w1 else m.g32[r], m.p16[r], n)
                all_segs.append(seg)
                self.gpu_segments.append((c, seg))
                self.groups.append((c, kernels.AdamTable([seg], m.device)))
        self.table = kernels.AdamTable(all_segs, m.device)  # single-launch form (overlap=False)
        all_cpu = {}
        for c in m.cpu_ids:
            r = m.row[c]
            n = m.valid(c)
            if n > 0:
                all_cpu[c] = (m.h_p32[r], m.h_m[r], m.h_v[r], m.h_g32[r], m.h_p16[r], n)
        # CPU-home updates are split between host threads (elx_cpu_adam, rate
        # v_c) and a GPU-streamed update (H2D p32/m/v/g -> K4 -> D2H
        # p32/m/v/p16 over PCIe) by measured rate: chunks in forward order go
        # to the worker that would finish them first (§8f row 4).
        self._all_cpu, self._cpu_update_mode = all_cpu, cpu_update
        self._rates = update_rates or DEFAULT_UPDATE_RATES
        self._stream_tile = stream_tile
        # streamed chunks whose gradient and parameters stay in their rCache block between steps
        # (attach_fetcher): chunk -> block tensor (mgr.in_block: the block holds the current parameters)
        self.resident: dict[int, torch.Tensor] = {}
        self._assign_cpu_updates(self._rates[0], self._rates[1])
        self.stream = torch.cuda.Stream(device=m.device) if overlap else None
        pin = torch.cuda.is_available()
        # ring of pinned snapshots of the step scalars (read lazily by StepStats / the CPU thread)
        self._host_ring = [torch.zeros(4, dtype=torch.float64, pin_memory=pin) for _ in range(8)]
        self.device_step = device_step
        self.tables = kernels.BiasTables(betas[0], betas[1], m.device) if device_step else None
        self._issued = 0          # step() calls since construction / checkpoint load
        self._step0 = 0           # completed steps at that point
        self._host_steps = 0      # host-mode step counter
        self._cpu_steps = 0       # CPU-home update's own counter (same rule as step_scalars[2])
        self.last_stats = None
        self.cpu_wait_s = 0.0      # host time the runtime blocked on CPU-home updates
        self.cpu_update_s = 0.0    # host time spent in CPU-home updates (on their thread)
        self.adam_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []
        self.stream_events: list[tuple[torch.cuda.Event, torch.cuda.Event]] = []  # streamed update spans
        self.time_adam = False
        self._cap_events: tuple[torch.cuda.Event, torch.cuda.Event] | None = None
        self.done_event: torch.cuda.Event | None = None
        self.grad_scale = 1.0
        self.pending: dict[object, torch.cuda.Event] = {}     # key -> GPU update done
        self._cpu_thread: threading.Thread | None = None
        self._cpu_error: BaseException | None = None

    def _assign_cpu_updates(self, host_rate: float, stream_rate: float) -> None:
        self.cpu_segs, self.stream_segs = {}, {}
        t_host = t_stream = 0.0
        for c in sorted(self._all_cpu):
            n = self._all_cpu[c][5]
            mode = self._cpu_update_mode
            use_stream = mode == "stream" or (mode == "split" and t_stream + n / stream_rate < t_host + n / host_rate)
            if use_stream:
                self.stream_segs[c] = self._all_cpu[c]
                t_stream += n / stream_rate
            else:
                self.cpu_segs[c] = self._all_cpu[c]
                t_host += n / host_rate
        self.cpu_ready: dict[int, threading.Event] = {c: threading.Event() for c in self.cpu_segs}
        for ev in self.cpu_ready.values():
            ev.set()
        self._init_stream_update(self._stream_tile)

    def attach_fetcher(self, fetcher: "ChunkFetcher") -> None:
        """Pair with the fetcher whose releases feed this optimizer (and whose
        gathers wait on its updates). At world 1 with a schedule that never
        evicts (`fetcher.stable_blocks`: each chunk keeps one rCache block,
        gathered into it every step), a streamed CPU-home chunk keeps its
        gradient and its parameters in that block: its release skips the D2H of
        the gradient, the streamed K4 reads the gradient from the block and
        writes the new bf16 parameters over it (as the GPU-home update does in
        the chunk itself), only p32/m/v cross PCIe (12 B each way per element
        instead of 14), and the next gather of the chunk copies nothing. The
        host memory traffic of such an element drops from 32 to 24 B per step
        — host DRAM is the offload path's bound — so the split
        between host threads and the streamed update is re-planned with that
        rate. The chunk's host parameter copy (h_p16) is then not kept current;
        `host_params_current()` writes it back on demand."""
        fetcher.optimizer = self
        m = self.mgr
        if not (m.fused_w1 and fetcher.stable_blocks and self._all_cpu and self._cpu_update_mode != "host"):
            return
        if os.environ.get("ELX_RESIDENT_STREAM", "1") == "0":  # A/B switch: the round-trip form
            return
        # planning rate of the resident streamed worker: 12 instead of 14 B each way per element, times 0.8 —
        # calibrated on the box (4B offload: 4 streamed chunks 14.5-14.6 samples/s vs 5 at 13.3-13.8; 10B: equal
        # at 0.8 and 1.0; 1.3/1.6 worse on both — profiles/r02aj_split_scale.txt); ELX_STREAM_RATE_SCALE overrides
        host_rate, stream_rate = self._rates
        scale = float(os.environ.get("ELX_STREAM_RATE_SCALE", "0.8"))
        self._assign_cpu_updates(host_rate, stream_rate * 14.0 / 12.0 * scale)
        self.resident = {c: m.blocks[fetcher.block_for[c]] for c in self.stream_segs if c in fetcher.block_for}

    def host_params_current(self) -> None:
        """Copy the parameters of resident streamed chunks from their blocks
        back to the host copies (h_p16), after the pending updates."""
        if not self.mgr.in_block:
            return
        self.synchronize()
        torch.cuda.synchronize(self.mgr.device)
        for c in sorted(self.mgr.in_block):
            n = self.stream_segs[c][5]
            self.stream_segs[c][4][:n].copy_(self.resident[c][:n])

    def _init_stream_update(self, tile: int) -> None:
        m = self.mgr
        self.xfer_done: dict[int, torch.cuda.Event] = {}
        self.stream_done: torch.cuda.Event | None = None
        if not self.stream_segs:
            return
        dev = m.device
        T = min(tile, max(seg[5] for seg in self.stream_segs.values()))
        T = -(-T // ELX_TILE) * ELX_TILE
        gdt = m.h_g32.dtype
        self._slots = [dict(p32=torch.empty(T, device=dev), m=torch.empty(T, device=dev),
                            v=torch.empty(T, device=dev), g=torch.empty(T, dtype=gdt, device=dev),
                            p16=torch.empty(T, dtype=m.dtype, device=dev), free=None) for _ in range(2)]
        self._slot_tables: dict[tuple[int, int], kernels.AdamTable] = {}
        self._tile = T
        self.h2d_stream = torch.cuda.Stream(device=dev)
        self.xfer_stream = torch.cuda.Stream(device=dev)
        self.sc_stream = torch.zeros(4, dtype=torch.float64, device=dev)  # K4 reads [0..2] only

    def _resident_table(self, s: int, cnt: int, c: int, a: int) -> kernels.AdamTable:
        """K4 over slot s's p32/m/v with the gradient read from (and the bf16
        parameters written over) elements [a, a+cnt) of chunk c's block."""
        key = ("res", s, cnt, c, a)
        if key not in self._slot_tables:
            sl, blk = self._slots[s], self.resident[c][a:a + cnt]
            self._slot_tables[key] = kernels.AdamTable(
                [(sl["p32"][:cnt], sl["m"][:cnt], sl["v"][:cnt], blk, blk, cnt)], self.mgr.device)
        return self._slot_tables[key]

    def _slot_table(self, s: int, cnt: int) -> kernels.AdamTable:
        key = (s, cnt)
        if key not in self._slot_tables:
            sl = self._slots[s]
            self._slot_tables[key] = kernels.AdamTable(
                [(sl["p32"][:cnt], sl["m"][:cnt], sl["v"][:cnt], sl["g"][:cnt], sl["p16"][:cnt], cnt)], self.mgr.device)
        return self._slot_tables[key]

    def _stream_update(self, cur: torch.cuda.Stream, tabs) -> None:
        """GPU-streamed update of the stream-assigned CPU-home chunks: tiles of
        T elements double-buffered through two HBM slots; H2D on one stream,
        K4 + D2H on another, so loads of tile k+1 overlap the update of tile k."""
        m = self.mgr
        h2d, xfer = self.h2d_stream, self.xfer_stream
        h2d.wait_stream(cur)
        xfer.wait_stream(cur)
        if self.time_adam:  # the streamed worker's span: its first H2D can start here
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(h2d)
        k = 0
        for c in sorted(self.stream_segs):
            p32, mm, vv, g, p16, n = self.stream_segs[c]
            blk = self.resident.get(c)
            for a in range(0, n, self._tile):
                cnt = min(self._tile, n - a)
                s = k % 2
                sl = self._slots[s]
                with torch.cuda.stream(h2d):
                    if sl["free"] is not None:
                        h2d.wait_event(sl["free"])
                    moves = ((p32, sl["p32"]), (mm, sl["m"]), (vv, sl["v"])) + (((g, sl["g"]),) if blk is None else ())
                    for src, dst in moves:
                        kernels.copy_h2d(dst, src[a:a + cnt], stream=h2d)
                    loaded = torch.cuda.Event()
                    loaded.record(h2d)
                with torch.cuda.stream(xfer):
                    xfer.wait_event(loaded)
                    tab = self._slot_table(s, cnt) if blk is None else self._resident_table(s, cnt, c, a)
                    kernels.adam(tab, self.hp, 0 if tabs is not None else self._kstep,
                                 self.sc_stream, m.dtype, stream=xfer, grad_scale=self.grad_scale,
                                 bias_tables=tabs)
                    backs = ((sl["p32"], p32), (sl["m"], mm), (sl["v"], vv)) + (((sl["p16"], p16),) if blk is None else ())
                    for src, dst in backs:
                        kernels.copy_d2h(dst[a:a + cnt], src, cnt * src.element_size(), stream=xfer)
                    free = torch.cuda.Event()
                    free.record(xfer)
                    sl["free"] = free
                k += 1
            ev = torch.cuda.Event()
            ev.record(xfer)
            self.xfer_done[c] = ev
            if blk is not None:
                self.mgr.in_block.add(c)   # the next gather finds the new parameters in the block
        self.stream_done = torch.cuda.Event(enable_timing=self.time_adam)
        self.stream_done.record(xfer)
        if self.time_adam:
            self.stream_events.append((t0, self.stream_done))

    def wait_offloaded(self, c: int, stream: torch.cuda.Stream) -> None:
        """Before touching chunk c's host shards: its previous update must be done
        (host flag for host-updated chunks, stream event for streamed ones)."""
        ev = self.xfer_done.get(c)
        if ev is not None:
            stream.wait_event(ev)
        else:
            self.wait_cpu(c)

    @property
    def gpu_elements(self) -> int:
        return self.table.valid_elements

    @property
    def bytes_per_element(self) -> int:
        """K4 algorithmic bytes per element: p32/m/v read+write (24), the
        gradient read (4 fp32, or 2 compute-dtype at world 1), the compute-dtype
        parameter write (2)."""
        return 24 + (2 if self.mgr.fused_w1 else 4) + 2

    # ------------------------------------------------------------ waits used by the fetcher / model
    def wait_gpu(self, key, stream: torch.cuda.Stream) -> None:
        ev = self.pending.get(key)
        if ev is not None:
            stream.wait_event(ev)

    def wait_cpu(self, c: int) -> None:
        ev = self.cpu_ready.get(c)
        if ev is not None and not ev.is_set():
            t0 = time.perf_counter()
            ev.wait()
            self.cpu_wait_s += time.perf_counter() - t0
        if self._cpu_error is not None:
            raise self._cpu_error

    def synchronize(self, stream: torch.cuda.Stream | None = None) -> None:
        """Make `stream` (default: current) wait for every outstanding update."""
        s = stream or torch.cuda.current_stream(self.mgr.device)
        if self.done_event is not None:
            s.wait_event(self.done_event)
        if self.stream_done is not None:
            s.wait_event(self.stream_done)
        if self._cpu_thread is not None:
            self._cpu_thread.join()
            if self._cpu_error is not None:
                raise self._cpu_error

    # ------------------------------------------------------------ checkpoint
    @property
    def step_count(self) -> int:
        """Completed (non-skipped) optimizer steps — the device counter
        step_scalars[2] is authoritative (reading it synchronises)."""
        if not self.device_step:
            return self._host_steps
        return int(self.mgr.step_scalars[2].item())

    def state_dict(self) -> dict:
        """This rank's fp32 master / m / v shards (GPU-home, CPU-home, shared)
        and the step count — the complete training state of the chunk path."""
        self.synchronize()
        torch.cuda.synchronize(self.mgr.device)
        m = self.mgr
        out = {"step": self.step_count, "world": m.world, "rank": m.rank, "chunk_length": m.C,
               "gpu": {k: getattr(m, k).cpu().clone() for k in ("p32", "m", "v")},
               "cpu": {k: getattr(m, "h_" + k).clone() for k in ("p32", "m", "v")},
               "shared": {pid: {k: getattr(sp, k).cpu().clone() for k in ("p32", "m", "v")}
                          for pid, sp in m.shared.items()}}
        return out

    def load_state_dict(self, state: dict) -> None:
        """Restore masters/moments and rebuild every compute-dtype copy from
        the masters (K4's skip path: p16 <- round(p32); host: elx_cpu_adam)."""
        m = self.mgr
        if state["world"] != m.world or state["rank"] != m.rank or state["chunk_length"] != m.C:
            raise ValidationError("checkpoint was written for a different world/rank/chunk length")
        self.synchronize()
        for k in ("p32", "m", "v"):
            getattr(m, k).copy_(state["gpu"][k])
            getattr(m, "h_" + k).copy_(state["cpu"][k])
            for pid, sp in m.shared.items():
                getattr(sp, k).copy_(state["shared"][pid][k])
        steps = int(state["step"])
        m.in_block.clear()  # the host copies are rebuilt below: the next gathers read them
        self._host_steps = self._cpu_steps = steps
        self._issued = 0
        self._step0 = steps
        sc = torch.tensor([0.0, 1.0, 0.0, 0.0], dtype=torch.float64, device=m.device)  # "skip": restore only
        kernels.adam(self.table, self.hp, max(1, steps), sc, m.dtype)
        host_segs = list(self.cpu_segs.values()) + list(self.stream_segs.values())
        if host_segs:
            kernels.cpu_adam(host_segs, self.hp, max(1, steps), (0.0, 1.0), m.dtype, self.cpu_threads)
        for sp in m.shared.values():
            m.gather_shared(sp)
        m.step_scalars.zero_()
        m.step_scalars[2] = float(steps)
        torch.cuda.synchronize(m.device)

    # ------------------------------------------------------------ step
    def step(self, releases_done: "torch.cuda.Event | float | None" = None, grad_scale: float = 1.0, *,
             loss_scale: float | None = None) -> "StepStats":
        """All-reduce norm/overflow, then update every shard.

        SURVEY.md §8b's form `step(loss_scale) -> (found_inf, grad_norm)` is
        accepted too: a number in the first position (or `loss_scale=`) is the
        loss scale, and grad_scale = 1 / loss_scale (the releases are then
        waited for by synchronising the device).

        Device-step mode (default): no host synchronisation — the overflow
        skip, the clip coefficient and the step number (step_scalars[2]) are
        all read on the device, and the bias corrections come from device
        tables. Returns a StepStats whose found_inf / grad_norm synchronise
        only when read. `releases_done` is the event ChunkFetcher.finish()
        returns (None: synchronise the device); `grad_scale` = 1/loss_scale,
        applied in-register to compute-dtype gradients (world 1)."""
        if isinstance(releases_done, (int, float)):
            releases_done, loss_scale = None, float(releases_done)
        if loss_scale is not None:
            if not loss_scale > 0:
                raise ValidationError("loss_scale must be > 0")
            grad_scale = 1.0 / loss_scale
        with _nvtx("elx.adam"):
            return self._step_impl(releases_done, grad_scale)

    def _step_impl(self, releases_done: torch.cuda.Event | None, grad_scale: float) -> "StepStats":
        self.grad_scale = float(grad_scale)
        m = self.mgr
        dev = m.device
        cur = torch.cuda.current_stream(dev)
        if releases_done is None:
            torch.cuda.synchronize(dev)
        else:
            cur.wait_event(releases_done)
        m.all_reduce_scalars()
        slot = self._host_ring[self._issued % len(self._host_ring)]
        slot.copy_(m.step_scalars[:4], non_blocking=True)
        snap = torch.cuda.Event()
        snap.record(cur)
        stats = StepStats(slot, snap)
        self._issued += 1
        if self._cpu_thread is not None:
            self._cpu_thread.join()
        if self.device_step:
            self.tables.ensure(self._step0 + self._issued)
            kstep = 0
        else:
            found_inf = stats.found_inf
            kstep = max(self._host_steps + (0 if found_inf else 1), 1)
            if not found_inf:
                self._host_steps += 1
        if self.stream_segs:
            self.sc_stream.copy_(m.step_scalars[:4])  # snapshot before the opt stream's step_advance
        opt = self.stream if self.overlap else cur
        if opt is not cur:
            opt.wait_stream(cur)
        tabs = self.tables if self.device_step else None
        capturing = torch.cuda.is_current_stream_capturing()
        if self.time_adam:
            if capturing:  # graph-internal K4 timing: the pair prepared by prepare_graph_timing()
                if self._cap_events is None:
                    raise ValidationError("time_adam under capture needs prepare_graph_timing() first")
                e0, e1 = self._cap_events
                kernels.event_record(e0, opt)
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(opt)
        self.pending = {}
        with torch.cuda.stream(opt):
            if self.overlap:
                for key, table in self.groups:
                    kernels.adam(table, self.hp, kstep, m.step_scalars, m.dtype, stream=opt,
                                 grad_scale=self.grad_scale, bias_tables=tabs)
                    if key in m.shared:
                        m.gather_shared(m.shared[key])
                    ev = torch.cuda.Event()
                    ev.record(opt)
                    self.pending[key] = ev
            else:
                kernels.adam(self.table, self.hp, kstep, m.step_scalars, m.dtype, stream=opt,
                             grad_scale=self.grad_scale, bias_tables=tabs)
                for sp in m.shared.values():
                    m.gather_shared(sp)
            if self.time_adam:
                if capturing:
                    kernels.event_record(e1, opt)
                else:
                    e1.record(opt)
                self.adam_events.append((e0, e1))
            if self.device_step:
                kernels.step_advance(m.step_scalars, stream=opt)
            else:
                kernels.step_reset(m.step_scalars, stream=opt)
            self.done_event = torch.cuda.Event()
            self.done_event.record(opt)
        if self.stream_segs:
            self._kstep = kstep
            self._stream_update(cur, tabs)
        if self.cpu_segs:
            for ev in self.cpu_ready.values():
                ev.clear()
            self._cpu_thread = threading.Thread(target=self._cpu_update, args=(stats,), daemon=True)
            self._cpu_thread.start()
        self.last_stats = stats
        return stats

    def prepare_graph_timing(self) -> tuple[torch.cuda.Event, torch.cuda.Event]:
        """Create the timing-event pair a captured step records around K4 (as
        event-record nodes: each replay re-records them, so
        `e0.elapsed_time(e1)` after a replay is that replay's K4 time)."""
        cur = torch.cuda.current_stream(self.mgr.device)
        pair = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for e in pair:
            e.record(cur)  # creates the CUDA events before any capture starts
        self._cap_events = pair
        return pair

    @property
    def last(self) -> dict:
        s = self.last_stats
        if s is None:
            return dict(found_inf=False, grad_norm=0.0)
        return dict(found_inf=s.found_inf, grad_norm=s.grad_norm)

    def _cpu_update(self, stats: "StepStats") -> None:
        """CPU-home shards in forward order, flagging each chunk when done.
        Runs on a host thread: it waits for this step's scalars (device ->
        pinned copy), not the main thread."""
        try:
            sq, flag = stats.scalars()
            t0 = time.perf_counter()
            skip = flag != 0.0 or not math.isfinite(sq)
            kstep = max(self._cpu_steps + (0 if skip else 1), 1)
            for c in sorted(self.cpu_segs):
                kernels.cpu_adam([self.cpu_segs[c]], self.hp, kstep, (sq, flag), self.mgr.dtype, self.cpu_threads,
                                 grad_scale=self.grad_scale)
                self.cpu_ready[c].set()
            if not skip:
                self._cpu_steps += 1
            self.cpu_update_s += time.perf_counter() - t0
        except BaseException as exc:  # surfaced by wait_cpu / synchronize
            self._cpu_error = exc
            for ev in self.cpu_ready.values():
                ev.set()


class LossScaler:
    """Dynamic loss scale for fp16 (GradScaler convention: halve on overflow,
    double after `growth_interval` clean steps); bf16 uses a static 1.0."""

    def __init__(self, init_scale: float = 65536.0, growth_interval: int = 2000, dynamic: bool = True):
        self.scale = float(init_scale)
        self.growth_interval = growth_interval
        self.dynamic = dynamic
        self._good = 0

    def update(self, found_inf: bool) -> None:
        if not self.dynamic:
            return
        if found_inf:
            self.scale *= 0.5
            self._good = 0
        else:
            self._good += 1
            if self._good >= self.growth_interval:
                self.scale *= 2.0
                self._good = 0
