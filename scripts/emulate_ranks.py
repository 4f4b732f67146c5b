"""The N > 1 runtime on a full-size plan, with N rank-threads sharing ONE GPU.

    python scripts/emulate_ranks.py [model] [world] [plan file] [--p2p] [--no-recompute] [--det] > gpurun_out/emulate.json

Each rank builds its chunk store from the reference planner's plan for N
GPUs (plans/<model>_n<N>.json, e.g. BASELINE config 2: GPT-2 1.3B at 8
ranks), holds 1/N of every chunk's shard state, and trains two steps through
the loopback transport of tests/_refstep.py (the bytes NCCL's all-gather /
all-to-all would move, or — with --p2p — the in-kernel peer-pointer path).
Per-rank micro-batch 1 (not 8) so eight ranks' activations fit one GPU; the
chunk plan does not depend on the batch. Checks every rank's live counters
against the oracle's simulate and that all ranks report finite losses.
"""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from _refstep import run_ranks  # noqa: E402
from oracle import layout_ref as L  # noqa: E402
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2, GPT2Config  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
model_name = args[0] if args else "gpt2-1.3b"
world = int(args[1]) if len(args) > 1 else 8
plan_file = args[2] if len(args) > 2 else f"{model_name}_n{world}.json"
p2p = "--p2p" in sys.argv
keep = "--no-recompute" in sys.argv  # the bench's mode when every chunk stays resident
base = PRESETS[model_name]
cfg = GPT2Config(base.hidden, base.layers, base.heads, base.vocab, base.seq_len, batch=1)
plan_text = (ROOT / "plans" / plan_file).read_text()
dev = torch.device("cuda:0")
if "--det" in sys.argv:  # deterministic library algorithms (cuDNN attention's deterministic backward)
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
if "--flash" in sys.argv:  # SDPA's flash backend instead of cuDNN (multi-thread determinism probe)
    torch.backends.cuda.enable_cudnn_sdp(False)
steps = 2


def rank_fn(r, transport):
    model = ElixirGPT2(cfg, plan_text, device=dev, transport=transport, seed=1234,
                       recompute=False if keep else True)
    g = torch.Generator(device=dev).manual_seed(1234 + r)
    ids = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=g, device=dev)
    losses, t0 = [], time.perf_counter()
    for _ in range(steps):
        losses.append(model.train_step(ids[:, :-1].contiguous(), ids[:, 1:].contiguous()).item())
    model.synchronize()
    torch.cuda.synchronize()
    return {"rank": r, "losses": losses, "seconds": time.perf_counter() - t0, "counters": model.fetcher.counters(),
            "shard_elements": model.manager.S, "chunks": model.layout.n_chunks,
            "gpu_state_bytes": model.manager.memory_report()}


t0 = time.perf_counter()
res = run_ranks(world, rank_fn, p2p=p2p)
wall = time.perf_counter() - t0
plan = json.loads(plan_text)
params, ops = L.gpt2_records(cfg.hidden, cfg.layers, cfg.vocab, cfg.seq_len)
chunks, where = L.pack(L.partition(params, ops)[1], plan["chunk_length"])
fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
cpu = {int(c) for c, d in plan["chunk_homes"].items() if d == "cpu"}
sim, _ = L.simulate(fwd, plan["n_block"], cpu, red)
keys = ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units")
ok = all(rr["counters"][k] == sim[k] for rr in res for k in keys)
finite = all(all(x == x and abs(x) < 1e6 for x in rr["losses"]) for rr in res)
print(json.dumps({"model": model_name, "world": world, "plan": plan_file, "transport": "p2p" if p2p else "exchange",
                  "recompute": not keep,
                  "per_rank_batch": cfg.batch, "steps": steps, "wall_s": round(wall, 2),
                  "counters_equal_simulate": ok, "losses_finite": finite, "simulate": {k: sim[k] for k in keys},
                  "ranks": res}, indent=1, default=str))
sys.exit(0 if ok and finite else 1)
