"""In-process A/B of GPT-2 step variants: each variant's whole step is
captured as its own CUDA graph on ONE model, then the graphs are replayed
alternately (ABAB...) and timed with CUDA events, so clock / power-cap drift
hits every variant alike (bench.py-to-bench.py differences on this
power-capped box are +-3%, larger than the effects measured here).

    python scripts/ab_step.py [model] [rounds] [--recompute | --lt]

Variants (monkeypatched, the product keeps the first):
  new         — as shipped
  sep_qkv     — q/k/v as three N = H GEMMs instead of one N = 3H GEMM
  unfused_res — residual gradient joined by autograd's add, not inside K11
  unfused_gc  — K12 backward then K7 instead of the fused gelu_bwd_colsum
"""
import json
import statistics
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200 import gpt2, kernels  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
model_name = args[0] if args else "gpt2-1.3b"
rounds = int(args[1]) if len(args) > 1 else 8
dev = torch.device("cuda:0")
cfg = gpt2.PRESETS[model_name]
plan = (ROOT / "plans" / f"{model_name}_n1.json").read_text()
model = gpt2.ElixirGPT2(cfg, plan, device=dev, seed=1234, recompute=True if "--recompute" in sys.argv else "auto")
g = torch.Generator(device=dev).manual_seed(1234)
ids = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=g, device=dev)
tok, tgt = ids[:, :-1].contiguous(), ids[:, 1:].contiguous()


def _sep_qkv(h, wq, wk, wv, bq, bk, bv):
    return F.linear(h, wq, bq), F.linear(h, wk, bk), F.linear(h, wv, bv)


def _unfused_res(x, w, b, w_target=None, b_target=None):
    return gpt2.layer_norm(x, w, b, w_target, b_target), x


def _unfused_gc(x, dy, db):
    d = kernels.gelu_bwd(x, dy)
    kernels.colsum(d, db)
    return d


VARIANTS = {"new": {}, "sep_qkv": {(gpt2, "_qkv_proj"): _sep_qkv},
            "unfused_res": {(gpt2, "layer_norm_residual"): _unfused_res},
            "unfused_gc": {(gpt2.kernels, "gelu_bwd_colsum"): _unfused_gc}}
if "--lt" in sys.argv:  # the tuned cuBLASLt algorithm table vs the heuristic's first choice
    VARIANTS = {"new": {}, "lt_first": {(kernels, "_lt_table"): lambda: {}}}
if "--recompute" in sys.argv:  # A/B activation checkpointing vs keeping the forward graphs
    VARIANTS = {"new": {}, "no_recompute": {(model, "keep_graph"): True}}
graphs = {}
for name, patches in VARIANTS.items():
    saved = {k: getattr(*k) for k in patches}
    for (mod, attr), fn in patches.items():
        setattr(mod, attr, fn)
    model.capture(tok, tgt, warmup=2)
    graphs[name] = model._graph
    for (mod, attr), fn in saved.items():
        setattr(mod, attr, fn)
    model._graph = None
times = {k: [] for k in graphs}
for r in range(rounds):
    for name, gr in graphs.items():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        if r > 0:
            times[name].append(a.elapsed_time(b))
med = {k: statistics.median(v) for k, v in times.items()}
# paired: each variant against the "new" replay of the same round (same clock state)
paired = {k: statistics.median([x - y for x, y in zip(v, times["new"])]) for k, v in times.items()}
print(json.dumps({"model": model_name, "rounds": rounds - 1,
                  "ms_per_step_median": {k: round(v, 3) for k, v in med.items()},
                  "paired_delta_vs_new_ms": {k: round(v, 3) for k, v in paired.items()}}))
