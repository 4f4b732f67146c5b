"""B200 hardware profiler: measures the rates the reference planner consumes
(profiles.py:158-209 RateTable / HardwareProfile; benefit_J search.py:141-160;
simulate's update term rcache_sim.py:173-184) with THIS framework's kernels,
and writes them in the reference's hardware-profile JSON format
(profiles.py:342-378, GB/s decimal):

  b_c2g  pinned host -> HBM copy (K6, elx_copy_h2d), chunk-shard sized
  b_g2c  HBM -> pinned host copy (K6, elx_copy_d2h)
  v_g    GPU chunk Adam (K4) velocity in the reference's convention:
         bytes/s over 4-byte optimizer elements (search.py:18-22)
  v_c    host Adam (elx_cpu_adam) velocity, same convention, all host threads
  b_g2g  NCCL all-gather bus bandwidth when run under torchrun with N > 1;
         null at one process

    python scripts/profile_hw.py [--out plans/hardware_b200_measured.json]

Only the n = 1 row is measured on a one-GPU box; rows for n = 2..8 are
derived (per-GPU PCIe links and GPU updates scale with n, the host CPU does
not; b_g2g uses the pool's measured NVLink all-reduce bus bandwidth, 725 GB/s,
from B200_PROFILING.md) and marked as such in "meta".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200 import kernels  # noqa: E402

GB = 1e9


def _time(fn, reps=8, warm=3, stream=None):
    ts = []
    for i in range(warm + reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = stream or torch.cuda.current_stream()
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def measure(n_elems: int = 64 * 2 ** 20, cpu_elems: int = 32 * 2 ** 20):
    dev = torch.device("cuda:0")
    side = torch.cuda.Stream()
    # K6 copies: a bf16 shard of n_elems (128 MiB at the default)
    host = torch.randn(n_elems).to(torch.bfloat16).pin_memory()
    d = torch.empty(n_elems, dtype=torch.bfloat16, device=dev)
    nbytes = n_elems * 2
    t_h2d = _time(lambda: kernels.copy_h2d(d, host, stream=side), stream=side)
    t_d2h = _time(lambda: kernels.copy_d2h(host, d, stream=side), stream=side)
    # K4 Adam
    f = lambda: torch.randn(n_elems, device=dev) * 1e-3
    p32, m, v, g = f(), f(), f().abs(), f()
    tab = kernels.AdamTable([(p32, m, v, g, d, n_elems)], dev)
    sc = kernels.new_step_scalars(dev)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
    for _ in range(20):
        kernels.adam(tab, hp, 2, sc, torch.bfloat16)
    t_adam = _time(lambda: kernels.adam(tab, hp, 2, sc, torch.bfloat16))
    # host Adam
    threads = len(os.sched_getaffinity(0))
    hf = lambda: torch.randn(cpu_elems) * 1e-3
    hp32, hm, hv, hg = hf(), hf(), hf().abs(), hf()
    h16 = torch.empty(cpu_elems, dtype=torch.bfloat16)
    import time
    kernels.cpu_adam([(hp32, hm, hv, hg, h16, cpu_elems)], hp, 2, (0.0, 0.0), torch.bfloat16, threads)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        kernels.cpu_adam([(hp32, hm, hv, hg, h16, cpu_elems)], hp, 2, (0.0, 0.0), torch.bfloat16, threads)
        ts.append(time.perf_counter() - t0)
    t_cpu = statistics.median(ts)
    return {
        "b_c2g": nbytes / t_h2d / GB,
        "b_g2c": nbytes / t_d2h / GB,
        "v_g": 4 * n_elems / t_adam / GB,
        "v_c": 4 * cpu_elems / t_cpu / GB,
        "detail": {"copy_bytes": nbytes, "adam_elements": n_elems, "adam_hbm_gbs": 30 * n_elems / t_adam / GB,
                   "cpu_adam_elements": cpu_elems, "cpu_threads": threads,
                   "cpu_adam_gbs_algorithmic": 30 * cpu_elems / t_cpu / GB},
        "capacity_bytes": torch.cuda.get_device_properties(dev).total_memory,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "plans" / "hardware_b200_measured.json"))
    ap.add_argument("--gpus", type=int, default=8, help="gpu_count of the written profile")
    args = ap.parse_args()
    r = measure()
    tables = {}
    for n in range(1, args.gpus + 1):
        tables[str(n)] = {
            "b_g2g": None if n == 1 else 725.0,
            "b_c2g": r["b_c2g"] * n,
            "b_g2c": r["b_g2c"] * n,
            "v_g": r["v_g"] * n,
            "v_c": r["v_c"],
        }
    doc = {
        "format_version": 1,
        "gpu_count": args.gpus,
        "gpu_capacity_bytes": int(r["capacity_bytes"]),
        "tables": tables,
        "meta": {
            "generated_by": "scripts/profile_hw.py",
            "device": torch.cuda.get_device_name(0),
            "measured": "n=1 row (b_c2g, b_g2c via elx_copy_*; v_g via elx_adam; v_c via elx_cpu_adam)",
            "derived": "n>1 rows: b_c2g/b_g2c/v_g scale with n (one PCIe link and one GPU per process), "
                       "v_c is shared host CPU (not scaled), b_g2g = 725 GB/s NVLink bus (B200_PROFILING.md)",
            "detail": r["detail"],
        },
    }
    Path(args.out).write_text(json.dumps(doc, indent=2))
    print(json.dumps({k: v for k, v in r.items() if k != "detail"} | r["detail"]))


if __name__ == "__main__":
    main()
