"""The N > 1 path in REAL separate processes (torch.distributed.run, one CUDA
context per rank, torch.distributed gloo collectives on CUDA tensors), all
ranks sharing the one GPU of the test box.

1. tests/mp_worker.py trains the tiny config for two steps per rank (over the
   gloo exchange path, or over the in-kernel P2P path with CUDA-IPC peer
   mappings and our device barrier); its
   losses, fp32 master shards and live counters must equal the thread
   loopback run of the same config (tests/test_multirank_gpu.py), which is
   itself checked bit for bit against the CPU oracle — so the multi-process
   path equals the oracle too.
2. bench.py --gpus 2 under torchrun (GPT-2 small, reference plans with
   rCache evictions and CPU-home chunks) prints one JSON line whose live
   counters equal the reference schedule (simulate) for that plan.
"""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from _refstep import run_ranks
from oracle import layout_ref as L
from paper_2212_05339_b200 import gpt2
from paper_2212_05339_b200.gpt2 import ElixirGPT2
from test_multirank_gpu import CFG, HP, _batches, _plan, _rank_masters

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(world: int, args: list[str], timeout: int = 600) -> subprocess.CompletedProcess:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    env = dict(os.environ, OMP_NUM_THREADS="4")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    if p.returncode != 0:  # the first failing rank's own lines, not just the launcher's tail
        r0 = [ln for ln in p.stderr.splitlines() if ln.startswith("[rank0]")]
        raise AssertionError("\n".join(r0[-60:]) + "\n----\n" + p.stdout[-2000:] + p.stderr[-3000:])
    return p


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("path", ["exchange-keep", "ipc-graph-keep"])
def test_multiprocess_keep_graph_equals_checkpointed_loopback(cuda, tmp_path, world, path):
    """The bench's N > 1 mode — every chunk resident (n_block = n_chunks), the
    forward graphs kept instead of recomputed, over the gloo exchange or the
    IPC P2P path with the second step replayed as a CUDA graph — in separate
    processes equals the checkpointed rank-thread run bit for bit (losses,
    masters) and its counters equal simulate."""
    _torchrun(world, ["tests/mp_worker.py", "rcache-max", str(tmp_path), path])
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    plan, fwd, red = _plan("rcache-max")
    init = gpt2.init_params(CFG, cuda, seed=11)

    def rank_fn(r, transport):
        model = ElixirGPT2(CFG, plan, device=cuda, transport=transport,
                           init={k: v.clone() for k, v in init.items()}, **HP)
        losses = []
        for s in range(2):
            tok, tgt = _batches(world, s, cuda)[r]
            losses.append(model.train_step(tok, tgt).item())
        model.synchronize()
        torch.cuda.synchronize()
        return losses, _rank_masters(model)

    want = run_ranks(world, rank_fn)
    sim, _ = L.simulate(fwd, plan.n_block, set(), red)
    for r in range(world):
        assert list(got[r]["losses"]) == want[r][0], r
        live = json.loads(str(got[r]["counters"]))
        for k in ("gather_ops", "replaced_ops", "reduce_ops"):
            assert live[k] == sim[k], (r, k)
        for pid, (off, ref_vals) in want[r][1].items():
            vals = got[r][f"val::{pid}"]
            if world == 2:
                assert np.array_equal(vals, ref_vals), (r, pid)
            else:  # gloo's fp64 all-reduce of the N sum-of-squares partials (see above)
                np.testing.assert_allclose(vals, ref_vals, rtol=1e-6, atol=0)


@pytest.mark.parametrize("path", ["exchange", "ipc", "ipc-ce", "ipc-graph"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["rcache-min", "offload"])
def test_multiprocess_gloo_equals_loopback(cuda, tmp_path, world, kind, path):
    """path "exchange": gloo all-gather / all-to-all + K3. path "ipc": the
    in-kernel P2P path across processes (CUDA-IPC peer mappings, our device
    barrier kernel), which symmetric memory cannot run on a shared GPU;
    "ipc-ce" with the fetch on the copy engines; "ipc-graph" with the second
    step captured and replayed as one CUDA graph per rank."""
    if path == "ipc-graph" and kind == "offload":
        pytest.skip("graph capture needs every chunk GPU-home")
    _torchrun(world, ["tests/mp_worker.py", kind, str(tmp_path), path])
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]

    plan, fwd, red = _plan(kind)
    init = gpt2.init_params(CFG, cuda, seed=11)

    def rank_fn(r, transport):
        model = ElixirGPT2(CFG, plan, device=cuda, transport=transport,
                           init={k: v.clone() for k, v in init.items()}, **HP)
        losses = []
        for s in range(2):
            tok, tgt = _batches(world, s, cuda)[r]
            losses.append(model.train_step(tok, tgt).item())
        model.synchronize()
        torch.cuda.synchronize()
        return losses, _rank_masters(model), model.fetcher.counters()

    want = run_ranks(world, rank_fn)
    cpu = {c for c, d in plan.chunk_homes.items() if d.value == "cpu"}
    sim, _ = L.simulate(fwd, plan.n_block, cpu, red)
    for r in range(world):
        assert list(got[r]["losses"]) == want[r][0], r
        live = json.loads(str(got[r]["counters"]))
        for k in ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units"):
            assert live[k] == want[r][2][k] == sim[k], (r, k)
        masters = {k[5:]: v for k, v in got[r].items() if k.startswith("val::")}
        assert set(masters) == set(want[r][1]), r
        for pid, vals in masters.items():
            off, ref_vals = want[r][1][pid]
            assert int(got[r][f"off::{pid}"]) == off
            # rank-ordered fp32 release and AdamW are bit-exact; the only order the
            # two transports may differ in is gloo's fp64 all-reduce of the N
            # sum-of-squares partials (exact for N = 2), which reaches the update
            # only through the fp32 clip coefficient
            if world == 2:
                assert np.array_equal(vals, ref_vals), (r, pid)
            else:
                np.testing.assert_allclose(vals, ref_vals, rtol=1e-6, atol=0)


@pytest.mark.parametrize("plan,transport", [("gpt2-small_n2.json", "nccl"), ("gpt2-small_rcache_n2.json", "nccl"),
                                            ("gpt2-small_rcache_n2.json", "ipc"), ("gpt2-small_n2.json", "ipc"),
                                            ("gpt2-small_n2.json", "ipc-ce")])
def test_bench_two_ranks_one_gpu(cuda, plan, transport):
    """transport "nccl" falls back to gloo on a shared GPU (same TorchDistTransport code)."""
    p = _torchrun(2, ["bench.py", "--gpus", "2", "--model", "gpt2-small", "--plan", plan, "--steps", "2",
                      "--warmup", "3", "--no-cpu", "--transport", transport], timeout=900)
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 16
    assert "oversubscribed" in line["config"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert np.isfinite(line["final_loss"])
    # live counters of rank 0 == the reference schedule for this plan
    pj = json.loads((ROOT / "plans" / plan).read_text())
    cfgm = gpt2.PRESETS["gpt2-small"]
    params, ops = L.gpt2_records(cfgm.hidden, cfgm.layers, cfgm.vocab, cfgm.seq_len)
    chunks, where = L.pack(L.partition(params, ops)[1], pj["chunk_length"])
    fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
    cpu = {int(c) for c, d in pj["chunk_homes"].items() if d == "cpu"}
    sim, _ = L.simulate(fwd, pj["n_block"], cpu, red)
    live = line["chunk_runtime"]["sim_counters"]
    for k in ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units"):
        assert live[k] == sim[k], (k, live, sim)
    if plan == "gpt2-small_rcache_n2.json":
        assert sim["replaced_ops"] > 0 and sim["c2g_units"] > 0
    # the IPC transport with every chunk GPU-home runs the step as CUDA graphs on both ranks
    assert line["config"]["cuda_graph"] == (transport in ("ipc", "ipc-ce") and plan == "gpt2-small_n2.json")
    # whole-step parity at N = 2 (oracle/parity.check_step_multirank): the reduced fp32 gradients, the sums
    # of squares and AdamW over both ranks' shards against the C oracle
    # (the rcache plan: evictions, re-gathers and 5 CPU-home chunks, their K3 into the fp32 staging shard and
    # their host-thread / streamed updates)
    par = line["parity"]
    assert par["checked"] and par["within_tolerance"], par
    assert par["reduced_grad_bit_identical_frac"] == 1.0 and par["sumsq_local_bit_identical"], par
    assert all(v == 1.0 for v in par["bit_identical_frac"].values()), par
    if transport == "ipc":
        assert par["sumsq_global_bit_identical"], par
    if plan == "gpt2-small_rcache_n2.json":
        assert sum(par["cpu_home_chunks_per_rank"]) > 0, par


@pytest.mark.parametrize("path", ["exchange-nosync", "ipc-nosync"])
def test_multiprocess_steps_without_host_sync(cuda, tmp_path, path):
    """Three steps with no host synchronisation between them (the
    next step's gathers must wait for the previous step's K4 through the
    runtime's stream ordering on every transport): losses and masters equal
    the host-synchronised rank-thread run bit for bit."""
    world = 2
    _torchrun(world, ["tests/mp_worker.py", "rcache-min", str(tmp_path), path])
    got = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]
    plan, _, _ = _plan("rcache-min")
    init = gpt2.init_params(CFG, cuda, seed=11)

    def rank_fn(r, transport):
        model = ElixirGPT2(CFG, plan, device=cuda, transport=transport,
                           init={k: v.clone() for k, v in init.items()}, **HP)
        losses = []
        for s in range(3):
            tok, tgt = _batches(world, s, cuda)[r]
            losses.append(model.train_step(tok, tgt).item())
        model.synchronize()
        torch.cuda.synchronize()
        return losses, _rank_masters(model)

    want = run_ranks(world, rank_fn)
    for r in range(world):
        assert list(got[r]["losses"]) == want[r][0], r
        for pid, (off, ref_vals) in want[r][1].items():
            assert np.array_equal(got[r][f"val::{pid}"], ref_vals), (r, pid)


@pytest.mark.parametrize("world", [2, 4])
def test_sweep_real_peer_pointers_oversubscribed(cuda, world):
    """bench.py --sweep under torchrun: every rank maps its peers' shards and
    blocks (our CUDA-IPC mappings) and K2 (SMs and copy engines), K3 and K4
    run on the real peer pointers between device barriers; one JSON line per
    (size, N, engine) with busBW; the NCCL bar lines say why they are absent
    when ranks share the GPU; each rank holds a context on its device only."""
    p = _torchrun(world, ["bench.py", "--sweep", "--gpus", str(world), "--sweep-sizes", "4,32", "--steps", "3",
                          "--sweep-check"], timeout=600)
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    # --sweep-check: K2's gathered bytes and K3 over the peers' blocks equal the C oracle on every rank
    par = [r for r in lines if r.get("engine") == "parity"]
    assert len(par) == 2 and all(r["k2_bytes_identical"] and r["k3_grad_bit_identical"] and
                                 r["k3_sumsq_bit_identical"] for r in par), par
    recs = [r for r in lines if r.get("sweep") == "chunk" and r.get("engine") != "parity"]
    got = {(r["chunk_mb"], r["engine"]) for r in recs}
    for mb in (4, 32):
        for eng in ("k2_fetch_sm", "k2_fetch_ce", "k3_release", "k4_adam", "nccl_all_gather",
                    "nccl_reduce_scatter_bf16", "nccl_reduce_scatter_f32"):
            assert (mb, eng) in got, (mb, eng)
    for r in recs:
        assert r["world"] == world and r["peers"] == "ipc" and "oversubscribed" in r
        if r["engine"].startswith("k2") or r["engine"].startswith("k3"):
            assert r["ms"] > 0 and r["bus_gbs"] > 0
        if r["engine"].startswith("nccl"):
            assert "unavailable" in r
    ctx = [r for r in lines if r.get("sweep") == "contexts"]
    assert ctx and ctx[0]["cuda_contexts_on_devices"] == [0]


def test_hardware_profiler_under_torchrun_oversubscribed(cuda, tmp_path):
    """scripts/profile_hw.py under torchrun (§8f row 2 at n > 1): every rank
    measures K6 / K4 / host Adam concurrently and K2's all-gather over real
    peer pointers; rank 0 prints the n = 2 row in the reference's format. With
    the ranks sharing a GPU the row is flagged oversubscribed and NOT written
    unless asked; written on request, it merges into the profile file with
    per-row provenance and derived rows for the rest, loadable by the
    reference's rate-table rules (every rate > 0; b_g2g > 0 for n > 1)."""
    out = tmp_path / "hw.json"
    p = _torchrun(2, ["scripts/profile_hw.py", "--out", str(out), "--gpus", "4"], timeout=600)
    rec = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")][0]
    assert rec["n"] == 2 and rec["oversubscribed"] and not out.exists()
    for k in ("b_c2g", "b_g2c", "v_g", "v_c", "b_g2g"):
        assert rec["row"][k] > 0, (k, rec)
    # n = 1 measured, then the n = 2 row merged on request
    subprocess.run([sys.executable, "scripts/profile_hw.py", "--out", str(out), "--gpus", "4"], cwd=ROOT,
                   check=True, capture_output=True, text=True, timeout=600)
    _torchrun(2, ["scripts/profile_hw.py", "--out", str(out), "--gpus", "4", "--write-oversubscribed"], timeout=600)
    doc = json.loads(out.read_text())
    assert sorted(doc["tables"], key=int) == ["1", "2", "3", "4"] and doc["gpu_count"] == 4
    rows = doc["meta"]["rows"]
    assert rows["1"]["measured"] and not rows["1"]["oversubscribed"]
    assert rows["2"]["measured"] and rows["2"]["oversubscribed"]
    assert not rows["3"]["measured"] and not rows["4"]["measured"]
    assert doc["tables"]["1"]["b_g2g"] is None
    for n in ("2", "3", "4"):
        t = doc["tables"][n]
        assert all(t[k] > 0 for k in ("b_c2g", "b_g2c", "v_g", "v_c", "b_g2g")), (n, t)
