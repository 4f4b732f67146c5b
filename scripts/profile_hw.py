"""B200 hardware profiler: measures the rates the reference planner consumes
(profiles.py:158-209 RateTable / HardwareProfile; benefit_J search.py:141-160;
simulate's update term rcache_sim.py:173-184) with THIS framework's kernels,
and writes them in the reference's hardware-profile JSON format
(profiles.py:342-378, GB/s decimal, per-process-count rows as in
pkg/hardware/dev_server_4gpu.json:6-8).

One process per GPU; run it once per process count n (torchrun for n > 1):

    python scripts/profile_hw.py                                  # row n = 1
    torchrun --nproc-per-node N scripts/profile_hw.py             # row n = N

Every rank measures AT THE SAME TIME (between barriers), so shared resources
(host memory bandwidth, the host CPU, PCIe switches) are contended exactly as
in a training step; the row is the aggregate over ranks (slowest rank's time
for the copies, sum for the updates):

  b_c2g  pinned host -> HBM copy (K6, elx_copy_h2d) of a chunk-shard-sized
         buffer on every rank concurrently: n * bytes / max time
  b_g2c  HBM -> pinned host copy (K6, elx_copy_d2h), same
  v_g    GPU chunk Adam (K4) velocity in the reference's convention (bytes/s
         over 4-byte optimizer elements, search.py:18-22), summed over ranks
  v_c    host Adam (elx_cpu_adam), every rank with its share of the host
         cores at once, summed (the host CPU is shared: it does not scale)
  b_g2g  chunk all-gather bus bandwidth (NCCL busBw convention
         (n-1)/n * bytes / t) of K2 over real peer pointers (our CUDA-IPC
         mappings, the runtime's default transport), max over ranks of the
         median time; NCCL all_gather_into_tensor on the same buffers is
         recorded beside it in meta

The row for n is merged into --out (default plans/hardware_b200_measured.json)
with its provenance in meta.rows[n]. Ranks sharing one GPU (the one-GPU
development box) measure the same code path but not NVLink: such a row is
flagged "oversubscribed" and written only with --write-oversubscribed (it is a
functional check, not a rate). Rows never measured are derived from the n = 1
row (per-GPU links and GPUs scale with n, the host CPU does not) with b_g2g the
900 GB/s per-direction NVLink 5 nominal, and say so in meta.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200 import kernels  # noqa: E402

GB = 1e9
NVLINK_NOMINAL_GBS = 900.0


def _world():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    torch.cuda.set_device(local % ndev)
    if world > 1:
        dist.init_process_group("gloo" if world > ndev else "nccl",
                                **({} if world > ndev else {"device_id": torch.device("cuda", local % ndev)}))
    return world, rank, world > ndev


def _barrier(world):
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()


def _max(x: float, world: int) -> float:
    if world == 1:
        return x
    out = [None] * world
    dist.all_gather_object(out, x)
    return max(out)


def _sum(x: float, world: int) -> float:
    if world == 1:
        return x
    out = [None] * world
    dist.all_gather_object(out, x)
    return sum(out)


def _time(fn, world, reps=8, warm=3, stream=None, pre=None):
    """Median over reps of one call, every rank starting together (`pre`, e.g.
    a device barrier, runs on the stream just before the timed region)."""
    ts = []
    for i in range(warm + reps):
        _barrier(world)
        s = stream or torch.cuda.current_stream()
        if pre is not None:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        if i >= warm:
            ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def measure(world, rank, oversub, n_elems=64 * 2 ** 20, cpu_elems=32 * 2 ** 20, fetch_mb=64):
    dev = torch.device("cuda", torch.cuda.current_device())
    side = torch.cuda.Stream()
    # ---- K6 copies: a bf16 shard of n_elems (128 MiB at the default) on every rank at once
    host = torch.randn(n_elems).to(torch.bfloat16).pin_memory()
    d = torch.empty(n_elems, dtype=torch.bfloat16, device=dev)
    nbytes = n_elems * 2
    t_h2d = _max(_time(lambda: kernels.copy_h2d(d, host, stream=side), world, stream=side), world)
    t_d2h = _max(_time(lambda: kernels.copy_d2h(host, d, stream=side), world, stream=side), world)
    # ---- K4 Adam on every rank at once
    f = lambda: torch.randn(n_elems, device=dev) * 1e-3
    p32, m, v, g = f(), f(), f().abs(), f()
    tab = kernels.AdamTable([(p32, m, v, g, d, n_elems)], dev)
    sc = kernels.new_step_scalars(dev)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
    t_adam = _time(lambda: kernels.adam(tab, hp, 2, sc, torch.bfloat16), world)
    v_g = _sum(4 * n_elems / t_adam, world)
    del p32, m, v, g, tab
    # ---- host Adam: the host cores split between the ranks, all at once
    threads = max(1, len(os.sched_getaffinity(0)) // world)
    hf = lambda: torch.randn(cpu_elems) * 1e-3
    hp32, hm, hv, hg = hf(), hf(), hf().abs(), hf()
    h16 = torch.empty(cpu_elems, dtype=torch.bfloat16)
    seg = [(hp32, hm, hv, hg, h16, cpu_elems)]
    kernels.cpu_adam(seg, hp, 2, (0.0, 0.0), torch.bfloat16, threads)
    ts = []
    for _ in range(3):
        _barrier(world)
        t0 = time.perf_counter()
        kernels.cpu_adam(seg, hp, 2, (0.0, 0.0), torch.bfloat16, threads)
        ts.append(time.perf_counter() - t0)
    v_c = _sum(4 * cpu_elems / statistics.median(ts), world)
    row = {"b_g2g": None, "b_c2g": world * nbytes / t_h2d / GB, "b_g2c": world * nbytes / t_d2h / GB,
           "v_g": v_g / GB, "v_c": v_c / GB}
    detail = {"copy_bytes_per_rank": nbytes, "adam_elements_per_rank": n_elems,
              "adam_hbm_gbs_per_rank": 30 * n_elems / t_adam / GB, "cpu_adam_elements_per_rank": cpu_elems,
              "cpu_threads_per_rank": threads}
    # ---- b_g2g: K2 all-gather of a fetch_mb chunk over real peer pointers
    if world > 1:
        from paper_2212_05339_b200.runtime import shard_length
        from paper_2212_05339_b200.transport import IpcTransport
        tr = IpcTransport()
        C = fetch_mb * 2 ** 20 // 2
        S = shard_length(C, world)
        shard = tr.alloc((S,), torch.bfloat16, dev)
        shard.normal_()
        block = tr.alloc((world * S,), torch.bfloat16, dev)
        ptrs = tr.peer_ptrs(shard)
        bus = (world - 1) / world * 2 * world * S
        # timed after a device barrier on the same stream: every rank's K2 starts together
        t_k2 = _max(_time(lambda: kernels.fetch(block, ptrs, S, rank=rank), world, pre=tr.device_barrier), world)
        row["b_g2g"] = bus / t_k2 / GB
        detail.update({"b_g2g_engine": "K2 (elx_fetch) over CUDA-IPC peer mappings", "fetch_chunk_mb": fetch_mb,
                       "k2_ms": t_k2 * 1e3})
        if not oversub and dist.get_backend() == "nccl":
            t_nccl = _max(_time(lambda: dist.all_gather_into_tensor(block, shard), world), world)
            detail["nccl_all_gather_bus_gbs"] = bus / t_nccl / GB
        _barrier(world)
        tr.close()
    return row, detail


def merge(out: Path, n: int, row: dict, detail: dict, oversub: bool, gpus: int) -> dict:
    doc = json.loads(out.read_text()) if out.exists() else {"format_version": 1, "tables": {}, "meta": {}}
    meta = doc.setdefault("meta", {})
    rows = meta.setdefault("rows", {})
    doc["tables"][str(n)] = row
    rows[str(n)] = {"measured": True, "oversubscribed": oversub, "device": torch.cuda.get_device_name(0),
                    "detail": detail, "generated_by": "scripts/profile_hw.py"}
    # rows never measured: derived from the measured n = 1 row, labelled as such
    base = doc["tables"].get("1")
    gpus = max(gpus, max(int(k) for k in doc["tables"]))
    if base is not None:
        for k in range(2, gpus + 1):
            if rows.get(str(k), {}).get("measured"):
                continue
            doc["tables"][str(k)] = {"b_g2g": NVLINK_NOMINAL_GBS, "b_c2g": base["b_c2g"] * k,
                                     "b_g2c": base["b_g2c"] * k, "v_g": base["v_g"] * k, "v_c": base["v_c"]}
            rows[str(k)] = {"measured": False,
                            "derived": "b_c2g/b_g2c/v_g = n x the measured n=1 row (one PCIe link and one GPU "
                                       "per process), v_c = the n=1 host rate (shared CPU), b_g2g = NVLink 5 "
                                       "nominal 900 GB/s per direction (unmeasured: run this script under "
                                       "torchrun on an n-GPU node)"}
    doc["gpu_count"] = gpus
    doc["gpu_capacity_bytes"] = int(torch.cuda.get_device_properties(0).total_memory)
    doc["tables"] = {k: doc["tables"][k] for k in sorted(doc["tables"], key=int)}
    meta["rows"] = {k: rows[k] for k in sorted(rows, key=int)}
    for stale in ("measured", "derived", "detail"):  # the single-row provenance of older files
        meta.pop(stale, None)
    meta["generated_by"] = "scripts/profile_hw.py"
    return doc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "plans" / "hardware_b200_measured.json"))
    ap.add_argument("--gpus", type=int, default=8, help="gpu_count of the written profile (rows 1..gpus)")
    ap.add_argument("--write-oversubscribed", action="store_true",
                    help="also write a row measured with ranks sharing a GPU (functional, not a rate)")
    ap.add_argument("--print-only", action="store_true")
    args = ap.parse_args()
    world, rank, oversub = _world()
    row, detail = measure(world, rank, oversub)
    if rank == 0:
        rec = {"n": world, "oversubscribed": oversub, "row": row, "detail": detail}
        print(json.dumps(rec), flush=True)
        if not args.print_only and (not oversub or args.write_oversubscribed):
            out = Path(args.out)
            out.write_text(json.dumps(merge(out, world, row, detail, oversub, args.gpus), indent=2) + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
