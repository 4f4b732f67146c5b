"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic:
shard geometry, the transport's gather / scatter / all-reduce semantics that
the fetch (K2) and release (K3) paths rely on, and the end-to-end claim that
(scatter + rank-ordered fp32 reduce on each rank) equals the single-process
oracle reduction of the whole chunk, shard by shard."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import arith
from paper_2212_05339_b200.runtime import shard_length
from paper_2212_05339_b200.transport import TorchDistTransport

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        fn(rank)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, fn, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(WORLD):
        assert res[r] == "ok", res[r]


def _chunk_grads(rank: int, C: int, seed: int = 0) -> np.ndarray:
    """Rank `rank`'s bf16 gradient block for a chunk of length C (bits)."""
    rng = np.random.default_rng(seed * 100 + rank)
    return arith.f32_to_bf16_bits(rng.standard_normal(C).astype(np.float32))


def _gather_case(rank):
    t = TorchDistTransport()
    assert t.world == WORLD and t.rank == rank
    C = 1001
    S = shard_length(C, WORLD)
    assert S % 8 == 0 and S * WORLD >= C
    shards = [torch.from_numpy(_chunk_grads(r, S, 1).view(np.int16)).view(torch.bfloat16) for r in range(WORLD)]
    block = torch.zeros(WORLD * S, dtype=torch.bfloat16)
    t.gather(block, shards[rank].clone())
    want = arith.gather([s.view(torch.int16).numpy().view(np.uint16) for s in shards])
    assert np.array_equal(block.view(torch.int16).numpy().view(np.uint16), want)


def _release_case(rank):
    """scatter + per-rank ordered reduce == oracle reduce of full blocks."""
    t = TorchDistTransport()
    C = 4099
    S = shard_length(C, WORLD)
    P = WORLD * S
    blocks = []
    for r in range(WORLD):
        b = np.zeros(P, np.uint16)
        b[:C] = _chunk_grads(r, C, 2)
        blocks.append(b)
    mine = torch.from_numpy(blocks[rank].view(np.int16)).view(torch.bfloat16)
    recv = torch.zeros(P, dtype=torch.bfloat16)
    t.scatter(recv, mine)
    rb = recv.view(torch.int16).numpy().view(np.uint16)
    segs = [rb[r * S:(r + 1) * S] for r in range(WORLD)]
    for r in range(WORLD):
        assert np.array_equal(segs[r], blocks[r][rank * S:(rank + 1) * S])
    valid = max(0, min(S, C - rank * S))
    g, sq, bad = arith.release([s[:valid] for s in segs], 0.5)
    full, _, _ = arith.release([b[:C] for b in blocks], 0.5)
    assert np.array_equal(g, full[rank * S:rank * S + valid])
    # norm all-reduce across ranks == single-process norm
    tot = torch.tensor([sq, float(bad)], dtype=torch.float64)
    t.all_reduce_sum(tot)
    want = arith.sumsq(full)  # the same quad partials; only the fp64 order differs
    assert tot[0].item() == pytest.approx(want, rel=1e-12)
    assert tot[1].item() == 0.0


def _valid_geometry_case(rank):
    from paper_2212_05339_b200.layout import pack_chunks
    from paper_2212_05339_b200.profiles import ParameterSpec, ModelProfile, OperatorNode
    from paper_2212_05339_b200.runtime import ChunkManager
    from paper_2212_05339_b200.schedule import Plan

    specs = tuple(ParameterSpec(f"p{i}", n) for i, n in enumerate([300, 500, 77, 900, 13]))
    prof = ModelProfile("m", specs, tuple(OperatorNode(f"o{i}", (s.id,)) for i, s in enumerate(specs)))
    lay = pack_chunks(specs, 901)
    plan = Plan(901, lay.n_chunks, {c: "gpu" for c in range(lay.n_chunks)})
    mgr = ChunkManager(prof, lay, plan, transport=TorchDistTransport(), device="cpu")
    S = shard_length(901, WORLD)
    assert mgr.S == S and mgr.P == WORLD * S
    for c, ch in enumerate(lay.chunks):
        tot = [mgr.valid(c, r) for r in range(WORLD)]
        assert sum(tot) == ch.used_elements
        assert mgr.valid(c) == tot[rank]
    # every rank owns the same shard geometry: all-gather of the sizes agrees
    sizes = torch.tensor([mgr.S, mgr.P, lay.n_chunks])
    allsz = [torch.zeros_like(sizes) for _ in range(WORLD)]
    dist.all_gather(allsz, sizes)
    assert all(torch.equal(a, sizes) for a in allsz)


def test_gather_semantics_world2():
    _run(_gather_case)


def test_scatter_release_equals_single_process_oracle_world2():
    _run(_release_case)


def test_shard_geometry_world2():
    _run(_valid_geometry_case)
