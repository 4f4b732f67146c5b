"""K3 release at BASELINE sizes, standalone (for ncu and A/B): world 1 norm
pass over the 1.3B plan's 12 x 100 Mi-element bf16 chunks as ONE batched
launch and as 12 launches, and world 2/4/8 reductions of a 32 MB chunk's
segment from local buffers standing in for peers.

    python scripts/k3_probe.py [--ncu]   (--ncu: a few launches, no timing)
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda", 0)
ncu = "--ncu" in sys.argv
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6550.4
sc = kernels.new_step_scalars(dev)


def timeit(fn, reps=10):
    if ncu:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    ts = []
    for i in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


C = 104_857_600
chunks = [torch.randn(C, device=dev).mul_(0.01).to(torch.bfloat16) for _ in range(12)]
segs = [(None, [c.data_ptr()], C) for c in chunks]
for scale in (1.0, 0.5):
    ms = timeit(lambda: kernels.release_batch(segs, torch.bfloat16, scale, sc))
    ms12 = timeit(lambda: [kernels.release_batch([s], torch.bfloat16, scale, sc) for s in segs])
    nbytes = 2 * C * 12
    print(json.dumps({"k3": "world1 norm", "inv_scale": scale, "elements": 12 * C,
                      "batched_ms": ms, "batched_gbs": nbytes / ms / 1e6, "batched_frac": nbytes / ms / 1e6 / peak,
                      "per_chunk_ms": ms12, "per_chunk_gbs": nbytes / ms12 / 1e6}), flush=True)
del chunks
for world in (2, 4, 8):
    S = 16 * 2 ** 20 // world
    srcs = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(world)]
    g = torch.empty(S, device=dev)
    ms = timeit(lambda: kernels.release(g, [s.data_ptr() for s in srcs], S, torch.bfloat16, 1.0, sc))
    nbytes = 2 * world * S + 4 * S
    print(json.dumps({"k3": f"world{world} reduce", "segment_elems": S, "ms": ms,
                      "local_hbm_gbs": nbytes / ms / 1e6}), flush=True)
# K2: the all-gather of one 32 MB chunk from world local shards (HBM stand-ins for peers), SMs vs copy engines
for world in (2, 4, 8):
    S = 16 * 2 ** 20 // world
    shards = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(world)]
    block = torch.empty(world * S, dtype=torch.bfloat16, device=dev)
    ptrs = [s.data_ptr() for s in shards]
    for engine in ("sm", "ce"):
        ms = timeit(lambda: kernels.fetch(block, ptrs, S, engine=engine))
        nbytes = 2 * 2 * world * S
        print(json.dumps({"k2": f"world{world} gather 32MB", "engine": engine, "ms": ms,
                          "local_hbm_gbs": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / peak}), flush=True)
