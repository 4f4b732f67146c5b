"""A tiny chunked GPT-2 trained for three steps on the runtime paths that the
kernel-level sanitizer run (scripts/sanitize_kernels.py) does not reach: the
resident streamed update (K4 reading the gradient from and writing the
parameters into an rCache block), the copy-engine lanes, the CUDA-graph step.
For compute-sanitizer:

    compute-sanitizer --tool memcheck python scripts/sanitize_step.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from paper_2212_05339_b200 import kernels  # noqa: E402
from paper_2212_05339_b200.gpt2 import ElixirGPT2, GPT2Config  # noqa: E402
from paper_2212_05339_b200.schedule import Plan  # noqa: E402
from test_runtime_gpu import _plans  # noqa: E402

dev = torch.device("cuda:0")
cfg = GPT2Config(hidden=64, layers=2, heads=2, vocab=256, seq_len=32, batch=2)
plans = dict(_plans(cfg))
tok = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), device=dev)
x, y = tok[:, :-1].contiguous(), tok[:, 1:].contiguous()

# resident streamed update (world 1, never-evicting plan, half CPU-home)
m = ElixirGPT2(cfg, plans["offload-resident"], device=dev, cpu_update="stream")
assert m.optimizer.resident
m.optimizer._init_stream_update(1000)   # several tiles per chunk, both slots
losses = [float(m.train_step(x, y)) for _ in range(3)]
m.optimizer.host_params_current()

# the whole step as one CUDA graph (every chunk GPU-home)
g = ElixirGPT2(cfg, plans["all-gpu-max"], device=dev, recompute=False)
g.train_step(x, y)
g.capture(x, y, warmup=1)
losses += [float(g.graph_step(x, y)) for _ in range(2)]

# K2 on the copy-engine lanes
shards = [torch.randn(4096, device=dev).to(torch.bfloat16) for _ in range(8)]
block = torch.empty(8 * 4096, dtype=torch.bfloat16, device=dev)
kernels.fetch(block, [t.data_ptr() for t in shards], 4096, engine="ce", rank=3)
torch.cuda.synchronize()
assert torch.equal(block, torch.cat(shards))
print("sanitize step ok", [round(v, 4) for v in losses])
