"""GPT-2 1.3B trained for a few hundred steps on a learnable synthetic stream
(token_{i+1} = (a * token_i + b) mod V, a random start per sequence), in the
bench's mode (forward graphs kept, the step replayed as one CUDA graph) and in
the reference's mode (per-layer checkpointing, eager), from the same init on
the same batches. Prints the loss every `every` steps for both and whether the
two sequences are bit-identical — the full-size counterpart of
tests/test_runtime_gpu.py::test_keep_graph_step_equals_recompute.

    python scripts/train_curve.py [steps] [every] > gpurun_out/train_curve.json
"""
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2, init_params  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steps = int(args[0]) if args else 200
every = int(args[1]) if len(args) > 1 else 10
dev = torch.device("cuda:0")
if "--det" in sys.argv:  # ask the libraries (cuDNN attention, cuBLAS) for deterministic algorithms
    torch.backends.cudnn.deterministic = True
    torch.use_deterministic_algorithms(True)
cfg = PRESETS["gpt2-1.3b"]
plan = (ROOT / "plans" / "gpt2-1.3b_n1.json").read_text()
V, B, T = cfg.vocab, cfg.batch, cfg.seq_len


def batch(step):
    g = torch.Generator(device=dev).manual_seed(10_000 + step)
    start = torch.randint(0, V, (B, 1), generator=g, device=dev)
    idx = torch.arange(T + 1, device=dev).view(1, -1)
    seq = (start * 1 + idx * 7919) % V  # an arithmetic progression mod V: the next token is predictable
    return seq[:, :-1].contiguous(), seq[:, 1:].contiguous()


def run(recompute, graph):
    init = init_params(cfg, dev, 1234, torch.bfloat16)
    model = ElixirGPT2(cfg, plan, device=dev, init=init, lr=3e-4, recompute=recompute)
    losses = []
    t0 = time.perf_counter()
    for s in range(steps):
        tok, tgt = batch(s)
        if graph and s == 3:
            model.capture(tok, tgt, warmup=0)
        lo = model.graph_step(tok, tgt) if graph and s >= 3 else model.train_step(tok, tgt)
        losses.append(float(lo))
    model.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    del model
    torch.cuda.empty_cache()
    return losses, wall


if "--repeat" in sys.argv:  # the checkpointed eager run twice: is the step itself run-to-run deterministic?
    keep, wk = run(True, graph=False)
else:
    keep, wk = run("auto", graph=True)
ac, wa = run(True, graph=False)
print(json.dumps({"model": "gpt2-1.3b", "steps": steps, "lr": 3e-4,
                  "data": "synthetic learnable stream: token_{i+1} = (token_i + 7919) mod V, random start",
                  "bench_mode": {"losses": keep[::every] + [keep[-1]], "wall_s": round(wk, 1)},
                  "checkpointed_eager": {"losses": ac[::every] + [ac[-1]], "wall_s": round(wa, 1)},
                  "bit_identical": keep == ac, "first_difference_step": next((i for i, (x, y) in
                                                                             enumerate(zip(keep, ac)) if x != y), None)}))
