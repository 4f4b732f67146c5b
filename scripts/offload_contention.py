"""What bounds the CPU-home update (configs 3/4): the host threads' Adam
(elx_cpu_adam) and the copy engines' H2D/D2H both move the optimizer state
through host memory. Measured alone and at the same time:

  host   elx_cpu_adam over N elements (bf16 gradient), all host threads
  dma    pinned H2D and D2H of a 1 GiB buffer each, on two streams, looped
  both   the two concurrently (the split update's situation)

    python scripts/offload_contention.py [--elems 268435456]
One JSON line per mode: host G elements/s and GB/s (28 B/element), DMA GB/s
each way, and their sum of host-memory traffic.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=256 * 2 ** 20)
    args = ap.parse_args()
    n = args.elems
    threads = len(os.sched_getaffinity(0))
    dev = torch.device("cuda", 0)
    p32, m, v = (torch.randn(n) * 0.02 for _ in range(3))
    v.abs_()
    g16 = (torch.randn(n) * 1e-2).to(torch.bfloat16)
    p16 = torch.empty(n, dtype=torch.bfloat16)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)
    nb = 2 ** 30
    h_up = torch.empty(nb, dtype=torch.uint8).pin_memory()
    h_dn = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d_up = torch.empty(nb, dtype=torch.uint8, device=dev)
    d_dn = torch.empty(nb, dtype=torch.uint8, device=dev)
    s_up, s_dn = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def host_once():
        t0 = time.perf_counter()
        kernels.cpu_adam([(p32, m, v, g16, p16, n)], hp, 1, (0.5, 0.0), torch.bfloat16, threads)
        return time.perf_counter() - t0

    def dma(seconds, out):
        up = dn = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            with torch.cuda.stream(s_up):
                d_up.copy_(h_up, non_blocking=True)
            with torch.cuda.stream(s_dn):
                h_dn.copy_(d_dn, non_blocking=True)
            s_up.synchronize()
            s_dn.synchronize()
            up += nb
            dn += nb
        out["t"] = time.perf_counter() - t0
        out["up"], out["dn"] = up, dn

    host_once()
    th = [host_once() for _ in range(3)]
    t_host = sorted(th)[1]
    r = {}
    dma(2.0, r)
    alone = {"mode": "alone", "host_g_elems_s": n / t_host / 1e9, "host_gbs": 28 * n / t_host / 1e9,
             "dma_h2d_gbs": r["up"] / r["t"] / 1e9, "dma_d2h_gbs": r["dn"] / r["t"] / 1e9}
    print(json.dumps({"bench": "offload_contention", "threads": threads, **alone}), flush=True)
    r2: dict = {}
    ts = []
    worker = threading.Thread(target=dma, args=(3.0, r2))
    worker.start()
    time.sleep(0.2)
    for _ in range(3):
        ts.append(host_once())
    worker.join()
    t_host2 = sorted(ts)[1]
    both = {"mode": "concurrent", "host_g_elems_s": n / t_host2 / 1e9, "host_gbs": 28 * n / t_host2 / 1e9,
            "dma_h2d_gbs": r2["up"] / r2["t"] / 1e9, "dma_d2h_gbs": r2["dn"] / r2["t"] / 1e9}
    both["host_memory_gbs_total"] = both["host_gbs"] + both["dma_h2d_gbs"] + both["dma_d2h_gbs"]
    print(json.dumps({"bench": "offload_contention", "threads": threads, **both}), flush=True)


if __name__ == "__main__":
    main()
