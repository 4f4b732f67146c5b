"""The GPT-2 1.3B step's GEMM shapes: torch (cuBLAS default) vs
elx_lt_matmul (cuBLASLt, heuristic top-1, or autotuned over the top 16 with
ELX_LT_AUTOTUNE=1). L2 flushed, median of 15.

    ELX_LT_AUTOTUNE=0 python scripts/gemm_probe.py; ELX_LT_AUTOTUNE=1 python scripts/gemm_probe.py
"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda:0")
bf = torch.bfloat16
T, H, Vp = 8192, 2048, 50304
flush = torch.ones(64 * 2 ** 20, device=dev)
sink = torch.empty((), device=dev)


def timed(fn, reps=15):
    ts = []
    for i in range(reps + 3):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def r(*s):
    return (torch.randn(*s, device=dev) * 0.05).to(bf)


cases = []
x, W3, b3 = r(T, H), r(3 * H, H), r(3 * H)
cases.append(("fwd qkv x.W3^T+b [8192x6144x2048]", lambda: F.linear(x, W3, b3),
              lambda: kernels.gemm(x, W3, tb=True, bias=b3), 2 * T * 3 * H * H))
g, Wq = r(T, H), r(H, H)
cases.append(("bwd dX g.W [8192x2048x2048]", lambda: torch.mm(g, Wq), lambda: kernels.gemm(g, Wq), 2 * T * H * H))
cases.append(("bwd dW g^T.x [2048x2048x8192]", lambda: torch.mm(g.t(), x), lambda: kernels.gemm(g, x, ta=True),
              2 * T * H * H))
d4, W4 = r(T, 4 * H), r(4 * H, H)
cases.append(("bwd fc dX d.Wfc [8192x2048x8192]", lambda: torch.mm(d4, W4), lambda: kernels.gemm(d4, W4),
              2 * T * 4 * H * H))
cases.append(("bwd fc dW d^T.x [8192x2048x8192]", lambda: torch.mm(d4.t(), x), lambda: kernels.gemm(d4, x, ta=True),
              2 * T * 4 * H * H))
Wm = r(H, 4 * H)
cases.append(("bwd mproj dX g.Wm [8192x8192x2048]", lambda: torch.mm(g, Wm), lambda: kernels.gemm(g, Wm),
              2 * T * 4 * H * H))
cases.append(("bwd mproj dW g^T.a [2048x8192x8192]", lambda: torch.mm(g.t(), d4), lambda: kernels.gemm(g, d4, ta=True),
              2 * T * 4 * H * H))
wte, lg = r(Vp, H), r(T, Vp)
cases.append(("head fwd x.wte^T [8192x50304x2048]", lambda: F.linear(x, wte), lambda: kernels.gemm(x, wte, tb=True),
              2 * T * Vp * H))
cases.append(("head dX dl.wte [8192x2048x50304]", lambda: torch.mm(lg, wte), lambda: kernels.gemm(lg, wte),
              2 * T * Vp * H))
cases.append(("head dW dl^T.x [50304x2048x8192]", lambda: torch.mm(lg.t(), x), lambda: kernels.gemm(lg, x, ta=True),
              2 * T * Vp * H))
tune = os.environ.get("ELX_LT_AUTOTUNE", "0")
for name, ft, fl, flop in cases:
    a, b = ft(), fl()
    err = ((a.float() - b.float()).abs().max() / a.float().abs().max()).item()
    mt, ml = timed(ft), timed(fl)
    print(json.dumps({"gemm": name, "autotune": tune, "torch_ms": round(mt, 4), "lt_ms": round(ml, 4),
                      "torch_tflops": round(flop / mt / 1e9, 1), "lt_tflops": round(flop / ml / 1e9, 1),
                      "rel_err": err}), flush=True)
