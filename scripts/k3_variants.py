"""A/B of the world-1 K3 (TMA-staged norm pass) shapes, under the same power
state the training step leaves the GPU in: each variant runs in its own
process (ELX_K3_TMA is read once per process), first heats the GPU with ~5 s
of bf16 GEMMs (the step's own regime: sw_power_cap, SM clock ~1.5-1.6 GHz),
then times the 1.3B plan's 12 x 100 Mi-element chunks in one launch and as
12 launches, sampling the SM clock around the timed region.

    python scripts/k3_variants.py [variants...]      (default: all)
"""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SHAPES = {0: "tile 32 KB, 4 stages (128 KB, 1 CTA/SM)", 1: "tile 16 KB, 4 stages (64 KB, 3 CTA/SM)",
          2: "tile 16 KB, 8 stages (128 KB, 1 CTA/SM)", 3: "tile 16 KB, 6 stages (96 KB, 2 CTA/SM)",
          4: "tile 8 KB, 8 stages (64 KB, 3 CTA/SM)", 5: "tile 32 KB, 3 stages (96 KB, 2 CTA/SM)"}


def child(variant: int) -> None:
    import torch
    sys.path.insert(0, str(ROOT))
    from paper_2212_05339_b200 import kernels
    dev = torch.device("cuda", 0)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6550.0
    sc = kernels.new_step_scalars(dev)
    C = 104_857_600
    chunks = [torch.randn(C, device=dev).mul_(0.01).to(torch.bfloat16) for _ in range(12)]
    segs = [(None, [c.data_ptr()], C) for c in chunks]
    a = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)

    def burn(seconds=5.0):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        while True:
            for _ in range(20):
                a @ a
            e1.record()
            e1.synchronize()
            if e0.elapsed_time(e1) > seconds * 1e3:
                return

    def clock():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True).stdout.strip()
        return float(out) if out else None

    def timeit(fn, reps=20):
        ts = []
        for i in range(reps + 3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    res = {"variant": variant, "shape": SHAPES.get(variant), "geometry": kernels.release_geometry([C] * 12, 1)}
    for state in ("cool", "hot"):
        if state == "hot":
            burn()
        clk0 = clock()
        ms = timeit(lambda: kernels.release_batch(segs, torch.bfloat16, 1.0, sc))
        ms12 = timeit(lambda: [kernels.release_batch([s], torch.bfloat16, 1.0, sc) for s in segs])
        clk1 = clock()
        nb = 2 * C * 12
        res[state] = {"sm_mhz": [clk0, clk1], "batched_ms": ms, "batched_frac": nb / ms / 1e6 / peak,
                      "per_chunk_ms": ms12, "per_chunk_frac": nb / ms12 / 1e6 / peak}
    print(json.dumps(res), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(int(sys.argv[2]))
        return
    variants = [int(x) for x in sys.argv[1:]] or sorted(SHAPES)
    for v in variants:
        env = dict(os.environ, ELX_K3_TMA=str(v))
        subprocess.run([sys.executable, __file__, "--child", str(v)], env=env, check=False)


if __name__ == "__main__":
    main()
