"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python scripts/ncu_summary.py <tag> [launches.csv] [report.ncu-rep ...]

Writes profiles/<tag>_launches.md (per-kernel share of one profiled step,
from the gpu__time_duration.sum launch list) and profiles/<tag>_<kernel>.json
(key metrics of each --set full capture: duration, DRAM bytes, throughput,
occupancy, registers) plus profiles/adam_ncu_traffic.json for bench.py's
roofline.traffic when an Adam capture is given.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "lts__t_bytes.sum", "dram__cycles_active.avg"]


def _to_ms(v: float, unit: str) -> float:
    return {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
            "second": 1e3}.get(unit, float("nan")) * v


def launches(tag: str, path: Path) -> None:
    rows = list(csv.reader(path.open()))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        ms = _to_ms(float(r[vi].replace(",", "")), r[ui])
        name = r[ki]
        short = name.split("(")[0][:110]
        tot[short] += ms
        cnt[short] += 1
    total = sum(tot.values())
    ours = {k: v for k, v in tot.items() if any(s in k for s in ("adam_kernel", "adam_tma_kernel", "adam_tma_st_kernel", "device_barrier", "release_kernel", "xent_fwd_kernel",
                                                                  "xent_bwd_kernel", "ln_param_grad_kernel", "ln_fwd_kernel", "ln_bwd_dx_kernel", "gelu_fwd_kernel", "gelu_bwd_kernel", "embedding_bwd_kernel", "release_norm_kernel", "::norm_kernel<",
                                                                  "pack_kernel", "fetch_kernel", "colsum_", "release_batch", "release_w1_tma", "release_tma", "fetch_tma", "peer_sum",
                                                                  "norm_finalize", "step_reset", "step_advance"))}
    lines = [f"# {tag}: kernel launch list of one training step (ncu gpu__time_duration.sum, cold, serialised)",
             "", f"Total device time {total:.3f} ms over {sum(cnt.values())} launches; "
             f"our kernels {sum(ours.values()):.3f} ms ({100 * sum(ours.values()) / total:.1f}%).", "",
             "| ms | share | launches | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:40]:
        mark = " **(ours)**" if k in ours else ""
        lines.append(f"| {v:.3f} | {100 * v / total:.1f}% | {cnt[k]} | `{k}`{mark} |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    print("wrote", PROF / f"{tag}_launches.md")


def report(tag: str, path: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120]}
        for k in KEYS:
            if k in d:
                try:
                    rec[k] = float(d[k].replace(",", ""))
                except ValueError:
                    rec[k] = d[k]
                rec[k + ".unit"] = units[h.index(k)]
        recs.append(rec)
    name = path.stem
    (PROF / f"{tag}_{name}.json").write_text(json.dumps(recs, indent=1))
    print("wrote", PROF / f"{tag}_{name}.json")
    return recs[0] if recs else {}


def _bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, float("nan"))


def main():
    tag = sys.argv[1]
    PROF.mkdir(exist_ok=True)
    for a in sys.argv[2:]:
        p = Path(a)
        if p.suffix == ".csv":
            launches(tag, p)
        elif p.suffix == ".ncu-rep":
            rec = report(tag, p)
            if "adam" in p.stem and "dram__bytes_read.sum" in rec:
                rd = _bytes(rec["dram__bytes_read.sum"], rec["dram__bytes_read.sum.unit"])
                wr = _bytes(rec["dram__bytes_write.sum"], rec["dram__bytes_write.sum.unit"])
                valid = int(sys.argv[sys.argv.index("--valid") + 1]) if "--valid" in sys.argv else None
                bpe = int(sys.argv[sys.argv.index("--bpe") + 1]) if "--bpe" in sys.argv else 30
                (PROF / "adam_ncu_traffic.json").write_text(json.dumps({
                    "source": f"profiles/{tag}_{p.stem}.json", "dram_bytes_per_launch": rd + wr,
                    "dram_read": rd, "dram_write": wr, "valid_elements": valid,
                    "bytes_per_element": bpe,
                    "algorithmic_bytes": None if valid is None else bpe * valid}, indent=1))


if __name__ == "__main__":
    main()
