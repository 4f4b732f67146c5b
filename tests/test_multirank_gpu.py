"""The N > 1 runtime path on ONE GPU: N ranks run as N threads with a
loopback transport (tests/_refstep.py) that moves bytes exactly as the
NCCL collectives would. Each rank trains on its own batch; the reassembled
fp32 masters must equal the oracle's (per-rank grads reduced in rank order in
fp32, clip, AdamW) bit for bit, and every rank's live counters must equal
simulate. Exercises sharding, rCache gathers with Belady victims and
prefetch, the all-to-all + K3 release, the shared wte all-gather and the
N-scalar all-reduce. The "p2p" variant runs the in-kernel NVLink path (K2
reading peers' shards, K3 reading peers' rCache blocks) with the peers'
buffers emulated by the other rank-threads' tensors on the same GPU."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from _refstep import ReferenceStep, run_ranks
from oracle import layout_ref as L
from paper_2212_05339_b200 import gpt2
from paper_2212_05339_b200.gpt2 import ElixirGPT2, GPT2Config
from paper_2212_05339_b200.runtime import shard_length
from paper_2212_05339_b200.schedule import Plan

pytestmark = pytest.mark.gpu

CFG = GPT2Config(hidden=64, layers=3, heads=4, vocab=389, seq_len=32, batch=2)
HP = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, max_norm=1.0)


def _plan(kind):
    h = CFG.hidden
    C = 4 * h * h + 3 * h * h // 2 + 5  # odd length: shard round-up + padding
    params, ops = L.gpt2_records(CFG.hidden, CFG.layers, CFG.vocab, CFG.seq_len)
    chunks, where = L.pack(L.partition(params, ops)[1], C)
    fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
    n, ws = len(chunks), max(len(s) for s in fwd)
    if kind == "rcache-max":
        return Plan(C, n, {c: "gpu" for c in range(n)}), fwd, red
    if kind == "rcache-min":
        return Plan(C, ws, {c: "gpu" for c in range(n)}), fwd, red
    return Plan(C, ws + 1, {c: ("cpu" if c % 2 == 0 else "gpu") for c in range(n)}), fwd, red


def _batches(world, step, dev):
    out = []
    for r in range(world):
        g = torch.Generator(device=dev).manual_seed(1000 * step + r)
        t = torch.randint(0, CFG.vocab, (CFG.batch, CFG.seq_len + 1), generator=g, device=dev)
        out.append((t[:, :-1].contiguous(), t[:, 1:].contiguous()))
    return out


def _rank_masters(model):
    """This rank's fp32 shards as {pid: (global offset in param, values)}."""
    mgr = model.manager
    out = {}
    lo = mgr.rank * mgr.S
    for pid, (c, off, numel) in mgr.members.items():
        a, b = max(off, lo), min(off + numel, lo + mgr.S)
        if a >= b:
            continue
        r = mgr.row[c]
        src = mgr.p32[r] if mgr.homes[c].value == "gpu" else mgr.h_p32[r]
        out[pid] = (a - off, src[a - lo:b - lo].float().cpu().numpy())
    sp = mgr.shared["wte"]
    n = sp.valid(mgr.rank)
    if n > 0:
        out.setdefault("wte", (mgr.rank * sp.shard, sp.p32[:n].cpu().numpy()))
    return out


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("path", ["exchange", "p2p"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["rcache-max", "rcache-min", "offload"])
def test_multirank_step_parity(cuda, world, kind, path, overlap):
    plan, fwd, red = _plan(kind)
    init = gpt2.init_params(CFG, cuda, seed=11)
    cpu = {c for c, d in plan.chunk_homes.items() if d.value == "cpu"}
    want_cnt, _ = L.simulate(fwd, plan.n_block, cpu, red)
    steps = 2

    def rank_fn(r, transport):
        model = ElixirGPT2(CFG, plan, device=cuda, transport=transport, overlap_update=overlap,
                           init={k: v.clone() for k, v in init.items()}, **HP)
        assert model.manager.S == shard_length(plan.chunk_length, world)
        losses = []
        for s in range(steps):
            tok, tgt = _batches(world, s, cuda)[r]
            losses.append(model.train_step(tok, tgt).item())
        model.synchronize()
        torch.cuda.synchronize()
        live = model.fetcher.counters()
        return losses, _rank_masters(model), live, model

    res = run_ranks(world, rank_fn, p2p=(path == "p2p"))
    if path == "p2p":
        assert res[0][3].manager.p2p
    ref = ReferenceStep(res[0][3], init, HP)
    ref_losses = []
    for s in range(steps):
        ls, _ = ref.step(_batches(world, s, cuda))
        ref_losses.append([x.item() for x in ls])
    for r in range(world):
        assert [ref_losses[s][r] for s in range(steps)] == res[r][0]
        live = res[r][2]
        for k in ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units"):
            assert live[k] == want_cnt[k], (r, k, live, want_cnt)
    # reassemble the sharded masters and compare bit for bit
    covered = {pid: np.zeros(v.size, bool) for pid, v in ref.master.items()}
    for r in range(world):
        for pid, (off, vals) in res[r][1].items():
            want = ref.master[pid][off:off + vals.size]
            assert np.array_equal(vals, want), (r, pid, off)
            covered[pid][off:off + vals.size] = True
    for pid, cov in covered.items():
        assert cov.all(), pid
