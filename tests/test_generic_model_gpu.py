"""The chunk runtime through its public API on a model that is NOT GPT-2:
a stack of residual MLP blocks described by a ModelProfile (one AC group per
block), packed with pack_chunks, scheduled by the plan, trained with
ChunkManager / ChunkFetcher / HybridAdam exactly as a maintainer would wire
them into another training loop ("For a model other than
GPT-2"). The fp32 masters after three steps must equal the CPU oracle's
(rank-ordered release, clip, AdamW) bit for bit, and the live counters must
equal simulate — for an all-GPU plan, a small rCache and a half-offloaded plan.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import arith
from oracle import layout_ref as L
from paper_2212_05339_b200 import (ChunkFetcher, ChunkManager, HybridAdam, build_chunk_trace, coarsen_graph,
                                   kernels, pack_chunks, partition_multiuse)
from paper_2212_05339_b200.profiles import profile_from_records
from paper_2212_05339_b200.schedule import Plan

pytestmark = pytest.mark.gpu

D, BLOCKS, BATCH = 96, 5, 64
HP = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, max_norm=1.0)


def _profile():
    params, ops = [], []
    for i in range(BLOCKS):
        names = [f"b{i}.w1", f"b{i}.b1", f"b{i}.w2", f"b{i}.b2"]
        params += [(names[0], 2 * D * D, False), (names[1], 2 * D, False), (names[2], 2 * D * D, False),
                   (names[3], D, False)]
        ops += [(f"b{i}.fc", names[:2], i), (f"b{i}.proj", names[2:], i)]
    shapes = {}
    for i in range(BLOCKS):
        shapes.update({f"b{i}.w1": (2 * D, D), f"b{i}.b1": (2 * D,), f"b{i}.w2": (D, 2 * D), f"b{i}.b2": (D,)})
    return profile_from_records("mlp-stack", params, ops), shapes


def _block(x, w1, b1, w2, b2):
    return x + F.linear(F.gelu(F.linear(x, w1, b1)), w2, b2)


def _init(shapes, dev):
    g = torch.Generator(device=dev).manual_seed(3)
    return {k: (torch.randn(s, device=dev, generator=g) * (0.05 if len(s) == 2 else 0.01)).to(torch.bfloat16)
            for k, s in shapes.items()}


def _data(dev, step):
    g = torch.Generator(device=dev).manual_seed(100 + step)
    x = torch.randn(BATCH, D, device=dev, generator=g).to(torch.bfloat16)
    y = torch.randn(BATCH, D, device=dev, generator=g).to(torch.bfloat16)
    return x, y


class Trainer:
    """The whole training loop a maintainer writes against the public API."""

    def __init__(self, profile, shapes, plan, init, dev):
        self.access = coarsen_graph(profile)
        _, seq = partition_multiuse(profile)
        self.layout = pack_chunks(seq, plan.chunk_length)
        self.trace = build_chunk_trace(self.access, self.layout)
        self.mgr = ChunkManager(profile, self.layout, plan, shapes=shapes, device=dev)
        self.mgr.load_params(init)
        self.fx = ChunkFetcher(self.mgr, self.trace)
        self.opt = HybridAdam(self.mgr, **HP)
        self.fx.optimizer = self.opt
        self.K = len(self.access.coarse_ops)

    def names(self, i):
        return [f"b{i}.w1", f"b{i}.b1", f"b{i}.w2", f"b{i}.b2"]

    def step(self, x, y):
        fx, mgr, K = self.fx, self.mgr, self.K
        fx.begin_step(after=self.opt.done_event)
        acts, h = [], x
        with torch.no_grad():
            for i in range(K):
                fx.enter(i)
                acts.append(h)
                h = _block(h, *[mgr.param(p) for p in self.names(i)])
                fx.after_compute(i)
        grad, loss = None, None
        for j in range(K):
            i = K - 1 - j
            fx.enter(K + j)
            ps = [mgr.param(p).detach().requires_grad_(True) for p in self.names(i)]
            xin = acts[i].detach().requires_grad_(True)
            with torch.enable_grad():
                out = _block(xin, *ps)
                if i == K - 1:
                    loss = F.mse_loss(out.float(), y.float())
                    gs = torch.autograd.grad(loss, [xin] + ps)
                else:
                    gs = torch.autograd.grad(out, [xin] + ps, grad_outputs=grad)
            grad = gs[0]
            # the gradient overwrites the parameter data in the chunk
            by_chunk = {}
            for pid, g in zip(self.names(i), gs[1:]):
                c, off, _ = mgr.members[pid]
                by_chunk.setdefault(c, []).append((g.reshape(-1), off))
            for c, mem in by_chunk.items():
                st = mgr.storage(c)
                kernels.chunk_pack(st, mem, used_len=st.numel())
            fx.after_compute(K + j)
        self.opt.step(fx.finish())
        return loss.detach()


class OracleTrainer:
    """Standalone bf16 parameters, the same block function, the CPU oracle's
    release / clip / AdamW (oracle/arith.py)."""

    def __init__(self, init, members):
        self.members = members  # pid -> (chunk, offset, numel) of the layout the runtime uses
        self.p16 = {k: v.clone() for k, v in init.items()}
        self.master = {k: v.float().cpu().numpy().reshape(-1).copy() for k, v in init.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.master.items()}
        self.t = 0

    def step(self, x, y):
        names = [[f"b{i}.w1", f"b{i}.b1", f"b{i}.w2", f"b{i}.b2"] for i in range(BLOCKS)]
        acts, h = [], x
        with torch.no_grad():
            for i in range(BLOCKS):
                acts.append(h)
                h = _block(h, *[self.p16[p] for p in names[i]])
        grads, grad, loss = {}, None, None
        for i in reversed(range(BLOCKS)):
            ps = [self.p16[p].detach().requires_grad_(True) for p in names[i]]
            xin = acts[i].detach().requires_grad_(True)
            with torch.enable_grad():
                out = _block(xin, *ps)
                if i == BLOCKS - 1:
                    loss = F.mse_loss(out.float(), y.float())
                    gs = torch.autograd.grad(loss, [xin] + ps)
                else:
                    gs = torch.autograd.grad(out, [xin] + ps, grad_outputs=grad)
            grad = gs[0]
            grads.update({p: g for p, g in zip(names[i], gs[1:])})
        rel, bad = {}, False
        for p, g in grads.items():
            r, _, b = arith.release([g.detach().reshape(-1).cpu().view(torch.int16).numpy().view(np.uint16)], 1.0)
            rel[p], bad = r, bad or b
        # the chunk store's norm units: quads over each chunk from its offset 0 (oracle/arith.py sumsq_chunked)
        sq = arith.sumsq_chunked(rel, self.members)
        coef = arith.clip_coef(sq, HP["max_norm"])
        self.t += 0 if bad else 1
        for p in rel:
            mp, mm, vv, p16 = arith.adamw(self.master[p], self.m[p], self.v[p], rel[p], max(self.t, 1), HP["lr"],
                                          HP["betas"][0], HP["betas"][1], HP["eps"], HP["weight_decay"], coef, bad)
            self.master[p], self.m[p], self.v[p] = mp, mm, vv
            self.p16[p] = torch.from_numpy(p16.view(np.int16)).view(torch.bfloat16).view(self.p16[p].shape).to(x.device)
        return loss.detach()


@pytest.mark.parametrize("kind", ["all-gpu", "small-rcache", "half-offload"])
def test_generic_model_through_public_api(cuda, kind):
    profile, shapes = _profile()
    C = int(2.6 * 2 * D * D)  # chunks straddle block boundaries
    _, seq = partition_multiuse(profile)
    lay = pack_chunks(seq, C)
    tr = build_chunk_trace(coarsen_graph(profile), lay)
    n = lay.n_chunks
    ws = max(len(s) for s in tr.forward)
    plan = {"all-gpu": Plan(C, n, {c: "gpu" for c in range(n)}),
            "small-rcache": Plan(C, ws, {c: "gpu" for c in range(n)}),
            "half-offload": Plan(C, ws + 1, {c: ("cpu" if c % 2 else "gpu") for c in range(n)})}[kind]
    init = _init(shapes, cuda)
    ours = Trainer(profile, shapes, plan, init, cuda)
    ref = OracleTrainer(init, ours.mgr.members)
    for s in range(3):
        x, y = _data(cuda, s)
        lo = ours.step(x, y)
        lr_ = ref.step(x, y)
        assert lo.item() == lr_.item(), s
    ours.opt.synchronize()
    torch.cuda.synchronize()
    got = ours.mgr.master_params()
    for p, want in ref.master.items():
        if p in got:
            assert np.array_equal(got[p].float().cpu().numpy().reshape(-1), want), p
    assert set(got) == set(ref.master)
    # live counters == the oracle's schedule for the oracle's own packing of the same records
    _, where = L.pack([(p.id, p.numel) for p in seq], C)
    fwd, _, red = L.chunk_trace([set(s) for s in coarsen_graph(profile).coarse_ops], where)
    cpu = {c for c, d in plan.chunk_homes.items() if d.value == "cpu"}
    want, _ = L.simulate(fwd, plan.n_block, cpu, red)
    live = ours.fx.counters()
    for k in ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units"):
        assert live[k] == want[k], (k, live, want)
