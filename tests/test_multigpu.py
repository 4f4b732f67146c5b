"""The N > 1 path on DISTINCT GPUs (one process per GPU, the real layout):
skipped unless the node has at least two devices. On such a node these run
what the one-GPU box can only run oversubscribed:

1. tests/mp_worker.py on N = 4 GPUs (2 on a 2-3 GPU node) over the in-kernel P2P path
   (K2/K3 reading peers' HBM through our CUDA-IPC mappings with peer access
   enabled across devices; eager and CUDA-graph steps) and over NCCL: losses,
   fp32 master shards and live counters equal the rank-thread loopback run on
   one GPU (itself bit-exact to the CPU oracle).
2. bench.py --sweep under torchrun: K2 / K2-CE / K3 busBW on real NVLink peer
   pointers beside NCCL's all-gather / reduce-scatter on the same buffers, and
   every rank holding a CUDA context on its own device only.
3. bench.py --gpus N with no transport flag: the default is the P2P path with
   the step captured as a CUDA graph, counters equal to simulate, and the
   bench's whole-step parity check bit-identical on every rank.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

from _refstep import run_ranks
from oracle import layout_ref as L
from paper_2212_05339_b200 import gpt2
from paper_2212_05339_b200.gpt2 import ElixirGPT2
from test_multiprocess_gpu import _torchrun
from test_multirank_gpu import CFG, HP, _batches, _plan, _rank_masters

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two or more GPUs (one per rank)")]


def _world() -> int:
    return 4 if torch.cuda.device_count() >= 4 else 2


@pytest.mark.parametrize("path", ["ipc", "ipc-ce", "ipc-graph", "nccl"])
def test_distinct_gpus_equal_loopback(cuda, tmp_path, path):
    world = _world()
    kind = "rcache-min"
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
            if path.startswith("ipc") or world == 2:  # rank-ordered peer sums: bit-exact
                assert np.array_equal(vals, ref_vals), (r, pid)
            else:  # NCCL's all-reduce order of the N sum-of-squares partials
                np.testing.assert_allclose(vals, ref_vals, rtol=1e-6, atol=0)


def test_sweep_on_nvlink_peers_with_nccl_bar(cuda):
    world = _world()
    p = _torchrun(world, ["bench.py", "--sweep", "--gpus", str(world), "--sweep-sizes", "32", "--steps", "5"],
                  timeout=900)
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    recs = {r["engine"]: r for r in lines if r.get("sweep") == "chunk"}
    for eng in ("k2_fetch_sm", "k2_fetch_ce", "k3_release", "nccl_all_gather", "nccl_reduce_scatter_bf16",
                "nccl_reduce_scatter_f32"):
        assert eng in recs and recs[eng]["bus_gbs"] > 0 and "oversubscribed" not in recs[eng], eng
    ctx = [r for r in lines if r.get("sweep") == "contexts"]
    assert ctx and ctx[0]["cuda_contexts_on_devices"] == [0]


def test_bench_default_transport_is_p2p_graph(cuda):
    world = _world()
    p = _torchrun(world, ["bench.py", "--gpus", str(world), "--model", "gpt2-small", "--plan",
                          "gpt2-small_n{n}.json",
                          "--steps", "3", "--warmup", "3", "--no-cpu"], timeout=900)
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == world and "oversubscribed" not in line["config"]
    assert line["config"]["transport"] == "ipc" and line["config"]["cuda_graph"]
    assert line["config"]["cuda_contexts_on_devices"] == [0]
    assert line["kernels"]["fetch"]["bus_gbs"] > 0
    # whole-step parity on distinct GPUs: peers' gradients read over NVLink, every element vs the C oracle
    par = line["parity"]
    assert par["checked"] and par["within_tolerance"] and par["sumsq_global_bit_identical"], par
    assert par["reduced_grad_bit_identical_frac"] == 1.0, par
    assert all(v == 1.0 for v in par["bit_identical_frac"].values()), par
