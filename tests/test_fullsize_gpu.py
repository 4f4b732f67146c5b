"""Arithmetic parity at the BASELINE.json configurations themselves (not toy
sizes).

1. GPT-2 1.3B, plan plans/gpt2-1.3b_n1.json (configs[1] at N = 1): the real
   layout (12 chunks of 100 Mi elements, ragged last chunk) and the shared wte
   (102.9 M elements) in a ChunkManager; seeded gradients written into the
   chunks; the ChunkFetcher walks the real schedule (its releases fire at the
   real reduce positions, one K3 launch per position) and HybridAdam runs K4
   over the real 13-segment table in one launch. Checked against the C oracle
   (oracle/c/elx_oracle.c, OpenMP) on EVERY element: the sum of squares
   bit-exact in the kernels' fixed order, and p32 / m / v / the bf16 parameter
   bit-exact per segment (a stricter bar than north_star's 1e-6).
2. GPT-2 small, plan plans/gpt2-small_n1.json (configs[0]): two whole chunked
   training steps through ElixirGPT2 against the reference step (standalone
   tensors, same node functions, the numpy oracle's release + AdamW): losses
   and every fp32 master bit-identical, live counters equal to simulate.
"""

from __future__ import annotations

import ctypes
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from _refstep import ReferenceStep
from oracle import arith
from oracle import layout_ref as L
from paper_2212_05339_b200 import gpt2, kernels
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2
from paper_2212_05339_b200.layout import build_chunk_trace, pack_chunks
from paper_2212_05339_b200.profiles import coarsen_graph, partition_multiuse, synthesize_transformer_profile
from paper_2212_05339_b200.runtime import ChunkFetcher, ChunkManager, HybridAdam

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
HP = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, max_norm=1.0)


def _oracle_lib():
    lib = ctypes.CDLL(str(ROOT / "oracle" / "_build" / "liboracle.so"))
    lib.oracle_release_norm_bf16_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_bf16_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_float,
                                                     ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.oracle_adamw_bf16.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                                             ctypes.c_int, ctypes.c_int]
    return lib


def _threads() -> int:
    import os
    return max(1, len(os.sched_getaffinity(0)))


def _seeded(n: int, seed: int, dev):
    """The segment's inputs, regenerated identically on demand: p32, m, v
    (fp32) and the bf16 gradient."""
    g = torch.Generator(device=dev).manual_seed(seed)
    p = torch.randn(n, generator=g, device=dev) * 0.02
    m = torch.randn(n, generator=g, device=dev) * 1e-3
    v = torch.rand(n, generator=g, device=dev) * 1e-6
    gr = (torch.randn(n, generator=g, device=dev) * 1e-2).to(torch.bfloat16)
    return p, m, v, gr


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def test_gpt2_1p3b_release_and_adam_full_table_bit_exact(cuda):
    cfg = PRESETS["gpt2-1.3b"]
    plan = (ROOT / "plans" / "gpt2-1.3b_n1.json").read_text()
    prof = synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, cfg.vocab, cfg.seq_len, cfg.batch)
    _, seq = partition_multiuse(prof)
    layout = pack_chunks(seq, json.loads(plan)["chunk_length"])
    trace = build_chunk_trace(coarsen_graph(prof), layout)
    mgr = ChunkManager(prof, layout, plan, shapes=gpt2.param_shapes(cfg), device=cuda)
    assert mgr.world == 1 and len(mgr.gpu_ids) == layout.n_chunks == 12
    segs = [("chunk", c, mgr.valid(c)) for c in mgr.gpu_ids] + [("wte", "wte", mgr.shared["wte"].numel)]
    assert sum(n for *_, n in segs) == prof.total_elements == 1_313_626_112

    def views(kind, key):
        """(p32, m, v, bf16 gradient in, bf16 parameter out)"""
        if kind == "chunk":
            r = mgr.row[key]   # world 1: the gradient lives in the chunk and K4 overwrites it in place
            return mgr.p32[r], mgr.m[r], mgr.v[r], mgr.p16[r], mgr.p16[r]
        sp = mgr.shared[key]
        return sp.p32, sp.m, sp.v, sp.grad, sp.p16

    for i, (kind, key, n) in enumerate(segs):
        p, m, v, gr = _seeded(n, 100 + i, cuda)
        P, M, V, G, _ = views(kind, key)
        P[:n].copy_(p)
        M[:n].copy_(m)
        V[:n].copy_(v)
        G[:n].copy_(gr)
        del p, m, v, gr
    torch.cuda.synchronize()

    fx = ChunkFetcher(mgr, trace)
    opt = HybridAdam(mgr, lr=HP["lr"], betas=HP["betas"], eps=HP["eps"], weight_decay=HP["weight_decay"],
                     max_norm=HP["max_norm"])
    fx.optimizer = opt
    fx.time_release = True
    fx.begin_step()
    for pos in range(2 * fx.n_fwd):
        fx.enter(pos)
        fx.after_compute(pos)
    fx.release_shared(mgr.shared["wte"])
    stats = opt.step(fx.finish())
    opt.synchronize()
    torch.cuda.synchronize()
    sq_gpu, flag = stats.scalars()
    assert flag == 0.0
    assert fx.counters()["reduce_ops"] == 12

    # ---- the oracle: the same launches' fixed-order sums, in release order
    lib = _oracle_lib()
    thr = _threads()
    groups = [[c for c in fx.reduces[p] if mgr.valid(c) > 0] for p in range(len(fx.reduces))]
    groups = [g for g in groups if g] + [["wte"]]
    index = {key: i for i, (_, key, _) in enumerate(segs)}
    sq = 0.0
    for grp in groups:
        ns = [segs[index[k]][2] for k in grp]
        host = [_bits(_seeded(n, 100 + index[k], cuda)[3]) for k, n in zip(grp, ns)]
        ctas, tv = kernels.release_geometry(ns, 1)
        ptrs = (ctypes.c_void_p * len(host))(*[h.ctypes.data for h in host])
        nn = (ctypes.c_int64 * len(host))(*ns)
        sq = sq + lib.oracle_release_norm_bf16_ordered(ptrs, nn, len(host), ctypes.c_float(1.0), ctas, tv, thr)
        del host
    assert sq_gpu == sq, (sq_gpu, sq)

    coef = arith.clip_coef(sq, HP["max_norm"])
    k = arith.adam_consts(1, HP["lr"], HP["betas"][0], HP["betas"][1], HP["eps"], HP["weight_decay"])
    kv = np.array([k["decay"], k["omb1"], k["b2"], k["omb2"], k["bc2_sqrt"], k["neg_step"], k["eps"]], np.float32)
    mism = {}
    for i, (kind, key, n) in enumerate(segs):
        dp, dm, dv, dg = _seeded(n, 100 + i, cuda)
        p, m, v = dp.cpu().numpy(), dm.cpu().numpy(), dv.cpu().numpy()
        g32 = arith.bf16_bits_to_f32(_bits(dg))
        del dp, dm, dv, dg
        p16 = np.empty(n, np.uint16)
        lib.oracle_adamw_bf16(p.ctypes.data, m.ctypes.data, v.ctypes.data, g32.ctypes.data, p16.ctypes.data, n,
                              kv.ctypes.data, ctypes.c_float(coef), 0, thr)
        P, M, V, _, OUT = views(kind, key)
        bad = [name for name, got, want in (("p32", P[:n].cpu().numpy(), p), ("m", M[:n].cpu().numpy(), m),
                                            ("v", V[:n].cpu().numpy(), v), ("p16", _bits(OUT[:n]), p16))
               if not np.array_equal(got, want)]
        if bad:
            mism[key] = bad
    assert not mism, mism


@pytest.fixture
def deterministic_library():
    """cuDNN's attention backward accumulates dQ non-deterministically at full
    size, so two computations of the same gradient — the
    runtime's and the reference step's — differ in the last bits unless the
    library's deterministic algorithms are on. Our kernels are deterministic
    either way."""
    import os
    old_env = os.environ.get("CUBLAS_WORKSPACE_CONFIG")
    os.environ["CUBLAS_WORKSPACE_CONFIG"] = ":4096:8"
    old = (torch.backends.cudnn.deterministic, torch.are_deterministic_algorithms_enabled())
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
    yield
    torch.backends.cudnn.deterministic = old[0]
    torch.use_deterministic_algorithms(old[1])
    if old_env is None:
        os.environ.pop("CUBLAS_WORKSPACE_CONFIG", None)
    else:
        os.environ["CUBLAS_WORKSPACE_CONFIG"] = old_env


def test_gpt2_small_full_step_equals_reference(cuda, deterministic_library):
    cfg = PRESETS["gpt2-small"]
    plan = (ROOT / "plans" / "gpt2-small_n1.json").read_text()
    init = gpt2.init_params(cfg, cuda, seed=3)
    model = ElixirGPT2(cfg, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    ref = ReferenceStep(model, init, HP)
    for s in range(2):
        gen = torch.Generator(device=cuda).manual_seed(50 + s)
        t = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=gen, device=cuda)
        tok, tgt = t[:, :-1].contiguous(), t[:, 1:].contiguous()
        lo = model.train_step(tok, tgt)
        (lr_,), _ = ref.step([(tok, tgt)])
        torch.cuda.synchronize()
        assert lo.item() == lr_.item(), (s, lo.item(), lr_.item())
    model.synchronize()
    torch.cuda.synchronize()
    got = model.manager.master_params()
    sp = model.manager.shared["wte"]
    got["wte"] = sp.p32[:sp.numel].clone()
    for pid, want in ref.master.items():
        g = got[pid].float().cpu().numpy().reshape(-1)
        assert np.array_equal(g, want), (pid, float(np.abs(g - want).max()))
    pj = json.loads(plan)
    params, ops = L.gpt2_records(cfg.hidden, cfg.layers, cfg.vocab, cfg.seq_len)
    _, where = L.pack(L.partition(params, ops)[1], pj["chunk_length"])
    fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
    sim, _ = L.simulate(fwd, pj["n_block"], set(), red)
    live = model.fetcher.counters()
    for k in ("gather_ops", "replaced_ops", "reduce_ops"):
        assert live[k] == sim[k], (k, live, sim)


@pytest.mark.parametrize("graph", [False, True])
def test_gpt2_small_trainer_step_checked_by_oracle_parity(cuda, graph):
    """The bench's `parity` field on BASELINE configs[0] (GPT-2 small, plan
    gpt2-small_n1.json, the trainer's own state after real steps, eager or
    after CUDA-graph replays): one more step's K3 launches and K4 update
    recomputed by the C oracle from the update's own inputs — the sum of
    squares and every p32 / m / v / bf16 element bit-identical."""
    from oracle.parity import check_step
    cfg = PRESETS["gpt2-small"]
    plan = (ROOT / "plans" / "gpt2-small_n1.json").read_text()
    model = ElixirGPT2(cfg, plan, device=cuda, **HP)
    gen = torch.Generator(device=cuda).manual_seed(5)
    t = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=gen, device=cuda)
    tok, tgt = t[:, :-1].contiguous(), t[:, 1:].contiguous()
    model.train_step(tok, tgt)
    if graph:
        model.capture(tok, tgt, warmup=1)
        model.graph_step(tok, tgt)
        model._graph = None
    else:
        model.train_step(tok, tgt)
    rep = check_step(model, tok, tgt)
    assert rep["checked"] and rep["elements"] == 124_439_808
    assert rep["sumsq_bit_identical"], rep
    assert all(f == 1.0 for f in rep["bit_identical_frac"].values()), rep
    assert rep["within_tolerance"]


@pytest.mark.parametrize("cpu_update", ["host", "stream", "split"])
@pytest.mark.parametrize("plan_name", ["offload-half", "offload-all", "all-gpu-min", "offload-resident"])
def test_offloaded_trainer_step_checked_by_oracle_parity(cuda, plan_name, cpu_update):
    """The bench's `parity` check on plans with CPU-home chunks (configs[2]/[3]'s
    regime) and evictions: the CPU-home chunks' gradients are captured from
    their rCache blocks at release time, their fp32 state from pinned host
    memory, and the host-thread, GPU-streamed or split update is recomputed by
    the C oracle — every element bit-identical, the sum of squares too."""
    from oracle.parity import check_step
    from test_runtime_gpu import CFG as TOY, _batch, _plans
    plan = dict(_plans(TOY))[plan_name]
    model = ElixirGPT2(TOY, plan, device=cuda, cpu_update=cpu_update, **HP)
    if model.optimizer.stream_segs:
        model.optimizer._init_stream_update(1000)  # tiny tiles: several per chunk, both slots
    tok, tgt = _batch(TOY, cuda, 1)
    model.train_step(tok, tgt)
    rep = check_step(model, tok, tgt)
    assert rep["checked"] and rep["elements"] == rep["model_elements"], rep
    assert rep["cpu_home_chunks_checked"] == rep["cpu_home_chunks"] == len(model.manager.cpu_ids)
    assert rep["sumsq_bit_identical"], rep
    assert all(f == 1.0 for f in rep["bit_identical_frac"].values()), rep


def test_sweep_parity_check(cuda):
    """bench.py --sweep --sweep-check (configs[4]): every emulated world's K2/K3/K4 outputs equal the C oracle
    (the same checker that produced profiles/r02am_sweep_parity.jsonl at 4-256 MB), here at 8 and 32 MB."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "bench.py", "--sweep", "--sweep-check", "--sweep-sizes", "8,32",
                          "--steps", "2"], cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    recs = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    par = [r for r in recs if r.get("engine") == "parity"]
    assert len(par) == 8, par
    for r in par:
        assert r["k2_bytes_identical"] and r["k3_grad_bit_identical"] and r["k3_sumsq_bit_identical"], r
        assert r["k4_bit_identical"], r
