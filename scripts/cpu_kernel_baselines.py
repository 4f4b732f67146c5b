"""each hot-path kernel beside CPU implementations of
the same work at the same algorithmic bytes, on the B200 box's host cores —
a reported baseline (TEST INFRASTRUCTURE: the oracle is only timed here,
never used by the product path).

  K4 Adam     elx_adam (GPU) | oracle/c AdamW (C, all host threads) |
              torch.optim.AdamW CPU single-tensor (foreach=False) and fused
  K3 release  elx_release, world 4 (GPU) | oracle/c rank-ordered fp32 sum |
              torch CPU: sum of the float() of the 4 slices, * inv_scale
  K2 fetch    elx_fetch, world 8 (GPU) | torch.cat of the 8 shards (CPU)
  K1 pack     elx_chunk_pack (GPU) | torch.cat of the members + zero tail (CPU)

    python scripts/cpu_kernel_baselines.py [--elems 67108864]
One JSON line per (kernel, implementation): ms, G elements/s, GB/s at the
kernel's algorithmic bytes, threads.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import parity  # noqa: E402  (the C oracle's loader)
from paper_2212_05339_b200 import kernels  # noqa: E402


def host_time(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


def gpu_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=64 * 2 ** 20)
    args = ap.parse_args()
    n = args.elems
    threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    dev = torch.device("cuda", 0)
    lib = parity._lib()
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]

    def emit(kernel, impl, ms, elems, nbytes, th):
        print(json.dumps({"bench": "cpu_kernel_baselines", "kernel": kernel, "impl": impl, "ms": round(ms, 4),
                          "g_elems_per_s": elems / ms / 1e6, "gbs": nbytes / ms / 1e6, "threads": th,
                          "elements": elems, "algorithmic_bytes": nbytes}), flush=True)

    # ---------------------------------------------------------------- K4 Adam (30 B/element, fp32 gradient)
    g = torch.Generator().manual_seed(0)
    p, m, v, gr = (torch.randn(n, generator=g) * 0.02 for _ in range(4))
    v.abs_()
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
    dp, dm, dv, dg = (t.to(dev) for t in (p, m, v, gr))
    d16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
    tab = kernels.AdamTable([(dp, dm, dv, dg, d16, n)], dev)
    sc = kernels.new_step_scalars(dev)
    emit("k4_adam", "elx_adam (GPU)", gpu_time(lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16)), n, 30 * n, None)
    p16 = np.empty(n, np.uint16)
    kv = np.array([1 - 1e-5, 0.1, 0.999, 0.001, 0.0316, -0.01, 1e-8], np.float32)
    P, M, V, G = (t.numpy() for t in (p, m, v, gr))
    emit("k4_adam", "oracle C AdamW", host_time(lambda: lib.oracle_adamw_bf16(
        P.ctypes.data, M.ctypes.data, V.ctypes.data, G.ctypes.data, p16.ctypes.data, n, kv.ctypes.data,
        ctypes.c_float(1.0), 0, threads)), n, 30 * n, threads)
    for fused in (False, True):
        prm = torch.nn.Parameter(p.clone())
        prm.grad = gr.clone()
        try:
            opt = torch.optim.AdamW([prm], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                                    foreach=False, fused=fused)
            emit("k4_adam", f"torch.optim.AdamW CPU {'fused' if fused else 'single-tensor'}",
                 host_time(opt.step), n, 28 * n, threads)
        except (RuntimeError, TypeError) as exc:  # a torch without the CPU fused kernel
            print(json.dumps({"bench": "cpu_kernel_baselines", "kernel": "k4_adam", "impl": "torch fused",
                              "unavailable": str(exc)[:200]}))
    del dp, dm, dv, dg, d16, tab, P, M, V, G, p, m, v, gr

    # ---------------------------------------------------------------- K3 release, world 4 (2*4*S + 4*S bytes)
    w = 4
    S = n // w
    srcs = [(torch.randn(S, generator=g) * 3).to(torch.bfloat16) for _ in range(w)]
    dsrc = [s.to(dev) for s in srcs]
    out = torch.empty(S, device=dev)
    nb = 2 * w * S + 4 * S
    emit("k3_release_w4", "elx_release (GPU)", gpu_time(lambda: kernels.release(
        out, [t.data_ptr() for t in dsrc], S, torch.bfloat16, 0.5, sc)), S, nb, None)
    hs = [s.view(torch.int16).numpy() for s in srcs]
    ptrs = (ctypes.c_void_p * w)(*[h.ctypes.data for h in hs])
    ho = np.empty(S, np.float32)
    bad = ctypes.c_int(0)
    emit("k3_release_w4", "oracle C rank-ordered sum", host_time(lambda: lib.oracle_release_bf16(
        ho.ctypes.data, ptrs, w, S, ctypes.c_float(0.5), ctypes.byref(bad), threads)), S, nb, threads)

    def torch_rs():
        acc = srcs[0].float()
        for s in srcs[1:]:
            acc = acc + s.float()
        return acc * 0.5
    emit("k3_release_w4", "torch CPU float sum", host_time(torch_rs), S, nb, threads)
    del dsrc, out

    # ---------------------------------------------------------------- K2 fetch, world 8 (2 * 2 * P bytes)
    w = 8
    S = n // w
    shards = [torch.randn(S, generator=g).to(torch.bfloat16) for _ in range(w)]
    dsh = [s.to(dev) for s in shards]
    blk = torch.empty(w * S, dtype=torch.bfloat16, device=dev)
    emit("k2_fetch_w8", "elx_fetch (GPU, local shards)", gpu_time(lambda: kernels.fetch(
        blk, [t.data_ptr() for t in dsh], S)), w * S, 4 * w * S, None)
    hblk = torch.empty(w * S, dtype=torch.bfloat16)
    emit("k2_fetch_w8", "torch.cat CPU", host_time(lambda: torch.cat(shards, out=hblk)), w * S, 4 * w * S,
         threads)
    del dsh, blk

    # ---------------------------------------------------------------- K1 pack (2*sum(numel) + 2*C bytes)
    h = 2048
    layer = [h, h, 3 * h * h, 3 * h, h * h, h, h, h, 4 * h * h, 4 * h, 4 * h * h, h]
    members, off, i = [], 0, 0
    while off + layer[i % 12] <= n:
        members.append((torch.randn(layer[i % 12], generator=g).to(torch.bfloat16), off))
        off += layer[i % 12]
        i += 1
    dmem = [(t.to(dev), o) for t, o in members]
    chunk = torch.empty(n, dtype=torch.bfloat16, device=dev)
    emit("k1_pack", "elx_chunk_pack (GPU)", gpu_time(lambda: kernels.chunk_pack(chunk, dmem, used_len=off)),
         n, 2 * off + 2 * n, None)
    hch = torch.empty(n, dtype=torch.bfloat16)

    def torch_pack():
        torch.cat([t for t, _ in members], out=hch[:off])
        hch[off:].zero_()
    emit("k1_pack", "torch.cat CPU", host_time(torch_pack), n, 2 * off + 2 * n, threads)


if __name__ == "__main__":
    main()
