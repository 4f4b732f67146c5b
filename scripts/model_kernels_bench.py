"""Standalone timing of the GPT-2 step's own kernels (K7-K12) at the GPT-2
1.3B shapes (8192 tokens x 2048 hidden; the MLP's 8192 x 8192), L2 flushed
by a 256 MB read before each launch, median of 20. GB/s = algorithmic bytes
(each operand read once, each result written once) / time.

    python scripts/model_kernels_bench.py > gpurun_out/model_kernels.jsonl
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.ones(64 * 2 ** 20, device=dev)
sink = torch.empty((), device=dev)
peak = 6550.4


def timed(fn, reps=20):
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


def report(name, ms, nbytes):
    gbs = nbytes / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": name, "ms": round(ms, 5), "bytes": nbytes, "gbs": round(gbs, 1),
                      "frac": round(gbs / peak, 3)}), flush=True)


R, H = 8192, 2048
bf = torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(R, H, device=dev, generator=g).to(bf)
dy = torch.randn(R, H, device=dev, generator=g).to(bf)
w = torch.ones(H, device=dev, dtype=bf)
b = torch.zeros(H, device=dev, dtype=bf)
y, mean, rstd = kernels.layer_norm_fwd(x, w, b)
E = R * H * 2
report("K10 layer_norm_fwd 8192x2048", timed(lambda: kernels.layer_norm_fwd(x, w, b)), 2 * E + 8 * R)
report("K11 layer_norm_bwd_dx 8192x2048", timed(lambda: kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd)), 3 * E + 8 * R)
dres = torch.randn(R, H, device=dev, generator=g).to(bf)
report("K11 layer_norm_bwd_dx + dres 8192x2048 (fused)",
       timed(lambda: kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd, dres=dres)), 4 * E + 8 * R)
report("K11 layer_norm_bwd_dx then torch add 8192x2048",
       timed(lambda: kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd) + dres), 4 * E + 8 * R)
dg, db = torch.empty(H, device=dev, dtype=bf), torch.empty(H, device=dev, dtype=bf)
report("K9 ln_param_grad 8192x2048", timed(lambda: kernels.ln_param_grad(x, dy, mean.view(-1), rstd.view(-1), dg, db)),
       2 * E + 8 * R)
report("K7 colsum 8192x2048", timed(lambda: kernels.colsum(dy, db)), E)
xf = torch.randn(R, 4 * H, device=dev, generator=g).to(bf)
dyf = torch.randn(R, 4 * H, device=dev, generator=g).to(bf)
Ef = R * 4 * H * 2
report("K7 colsum 8192x8192", timed(lambda: kernels.colsum(dyf, torch.empty(4 * H, device=dev, dtype=bf))), Ef)
report("K12 gelu_fwd 8192x8192", timed(lambda: kernels.gelu_fwd(xf)), 2 * Ef)
report("K12 gelu_bwd 8192x8192", timed(lambda: kernels.gelu_bwd(xf, dyf)), 3 * Ef)
dbf4 = torch.empty(4 * H, device=dev, dtype=bf)
report("K12 gelu_bwd + K7 colsum 8192x8192 (unfused)",
       timed(lambda: kernels.colsum(kernels.gelu_bwd(xf, dyf), dbf4)), 3 * Ef)
report("K12+K7 gelu_bwd_colsum 8192x8192 (fused)", timed(lambda: kernels.gelu_bwd_colsum(xf, dyf, dbf4)), 3 * Ef)
report("torch gelu fwd (tanh) 8192x8192",
       timed(lambda: torch.nn.functional.gelu(xf, approximate="tanh")), 2 * Ef)
report("torch layer_norm fwd 8192x2048",
       timed(lambda: torch.nn.functional.layer_norm(x, (H,), w, b, 1e-5)), 2 * E)
V = 50304
logits = torch.randn(R, V, device=dev, generator=g).to(bf)
tgt = torch.randint(0, 50257, (R,), device=dev, generator=g)
lse = torch.empty(R, device=dev)
loss = torch.empty(R, device=dev)
from paper_2212_05339_b200 import _lib  # noqa: E402
lib = _lib.load()
report("K8 xent_fwd 8192x50304", timed(lambda: lib.elx_xent_fwd(logits.data_ptr(), _lib.BF16, R, V, 50257,
                                                                  tgt.data_ptr(), -100, lse.data_ptr(), loss.data_ptr(),
                                                                  torch.cuda.current_stream().cuda_stream)), R * V * 2)
scale = torch.ones(1, device=dev)
report("K8 xent_bwd 8192x50304", timed(lambda: lib.elx_xent_bwd(logits.data_ptr(), _lib.BF16, R, V, 50257,
                                                                  tgt.data_ptr(), -100, lse.data_ptr(), scale.data_ptr(),
                                                                  torch.cuda.current_stream().cuda_stream)), 2 * R * V * 2)

# cuBLASLt fused-epilogue GEMMs vs the unfused sequence they replace (GPT-2 1.3B MLP / attention shapes)
H4 = 4 * H
wfc = torch.randn(H4, H, device=dev, generator=g).to(bf)
bfc = torch.zeros(H4, device=dev, dtype=bf)
wmp = torch.randn(H, H4, device=dev, generator=g).to(bf)
pre = torch.randn(R, H4, device=dev, generator=g).to(bf)
dbf = torch.empty(H4, device=dev, dtype=bf)
gemm_fc = 2 * R * H * H4 / 1e12


def report_tf(name, ms, tflop):
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "tflops": round(tflop / (ms * 1e-3), 1)}), flush=True)


report_tf("lt fc fwd GELU_AUX_BIAS", timed(lambda: kernels.linear_gelu(x, wfc, bfc, True)), gemm_fc)
report_tf("lt fc fwd GELU_BIAS", timed(lambda: kernels.linear_gelu(x, wfc, bfc, False)), gemm_fc)
report_tf("torch linear + K12 gelu", timed(lambda: kernels.gelu_fwd(torch.nn.functional.linear(x, wfc, bfc))), gemm_fc)
report_tf("lt mproj dX DGELU_BGRAD", timed(lambda: kernels.linear_dgelu_bgrad(dy, wmp, pre, dbf)), gemm_fc)
report_tf("torch mm + K12 gelu_bwd + K7", timed(lambda: kernels.colsum(kernels.gelu_bwd(pre, dy @ wmp), dbf)), gemm_fc)
dw = torch.empty(H, H, device=dev, dtype=bf)
report_tf("lt wgrad BGRADB 2048x2048", timed(lambda: kernels.wgrad_bgrad(x, dy, dw, db)), 2 * R * H * H / 1e12)
report_tf("torch mm(out) + K7 2048x2048", timed(lambda: (torch.mm(dy.t(), x, out=dw), kernels.colsum(dy, db))),
          2 * R * H * H / 1e12)
