"""K4 alone: eager launch vs the same launch as a one-node CUDA graph, zero vs
random state (why the sweep's graph-stream K4 line differs from the plain one).
    python scripts/k4_graph_probe.py
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda", 0)
hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
flush = torch.ones(64 * 2 ** 20, device=dev)
sink = torch.empty((), device=dev)
S = 64 * 2 ** 20


def time_fn(fn, reps=10):
    ts = []
    for i in range(reps + 2):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for init in ("zeros", "randn"):
    if init == "zeros":
        p32, m, v, g32 = (torch.zeros(S, device=dev) for _ in range(4))
    else:
        p32, m, v, g32 = (torch.randn(S, device=dev) * 0.01 for _ in range(4))
        v.abs_()
    p16 = torch.empty(S, dtype=torch.bfloat16, device=dev)
    for sc_kind in ("fresh",):
        sc = kernels.new_step_scalars(dev)
        tab = kernels.AdamTable([(p32, m, v, g32, p16, S)], dev)
        f = lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16)
        eager = time_fn(f)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            f()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        graph = time_fn(g.replay)
        eager2 = time_fn(f)
        print(json.dumps({"init": init, "S": S, "eager_ms": eager, "graph_ms": graph, "eager_after_ms": eager2,
                          "eager_frac": 30 * S / eager / 1e6 / 6460, "graph_frac": 30 * S / graph / 1e6 / 6460}))
