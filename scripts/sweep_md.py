"""Format a `bench.py --sweep` JSONL (BASELINE.json configs[4]) as a markdown
table under profiles/.

    python scripts/sweep_md.py <sweep.jsonl> <profiles/out.md> [title]

N = 1 runs emulate the N ranks with local buffers (HBM-bound): K2 GB/s =
2*2*N*S (read + write), K3 = 2*N*S read + 4*S write (N > 1; N = 1 is the
runtime's norm pass, 2*S read), K4 = 30*S; fraction of the measured HBM copy
peak. Runs under torchrun on real peers report busBW instead.
"""
import json
import sys
from collections import defaultdict
from pathlib import Path


def main():
    src, out = Path(sys.argv[1]), Path(sys.argv[2])
    title = sys.argv[3] if len(sys.argv) > 3 else src.name
    recs = [json.loads(ln) for ln in src.read_text().splitlines() if ln.startswith("{")]
    recs = [r for r in recs if r.get("sweep") == "chunk"]
    if not recs:
        raise SystemExit("no sweep records")
    peak = recs[0].get("hbm_peak_gbs")
    table = defaultdict(dict)
    for r in recs:
        key = (r["chunk_mb"], r.get("emulated_world", r.get("world")))
        table[key][r["engine"]] = r
    engines = ["k1_pack", "k2_fetch_sm", "k2_fetch_ce", "k3_release", "k4_adam"]
    graph = any(r.get("mode") == "graph_stream" for r in recs)
    lines = [f"# {title}", "",
             f"`python bench.py --sweep`: standalone K2 (SM kernel / copy engines), K3 and K4 on one rank's share of "
             f"one chunk; N local HBM buffers stand in for the N ranks (one GPU). Median of the launches after "
             f"warm-up, L2 flushed (256 MB read) before each. GB/s = algorithmic bytes / time; fraction of the "
             f"measured {peak} GB/s copy peak (MEASURED_PEAKS.json; a read-only stream such as the N = 1 K3 norm "
             f"pass can exceed it). N = 1 K3 is the runtime's norm pass (2 B/element read, no fp32 output)."
             + (" GRAPH-STREAMED (`--sweep-graph`): K2/K3/K4 as R back-to-back launches on distinct buffers "
                "(R x bytes >= 512 MB) captured in one CUDA graph, ms per launch = replay time / R — the issue "
                "pattern of a step; K1 (run once per plan) stays a single launch." if graph else ""), "",
             "| chunk MB | N | shard elems | " + " | ".join(f"{e} ms | {e} GB/s | frac" for e in engines) + " |",
             "|---:|---:|---:|" + "---:|---:|---:|" * len(engines)]
    for (mb, n) in sorted(table):
        row = table[(mb, n)]
        s = next(iter(row.values()))["shard_elems"]
        cells = []
        for e in engines:
            r = row.get(e)
            if r is None or "ms" not in r:
                cells += ["", "", ""]
                continue
            gbs = r.get("hbm_gbs", r.get("bus_gbs"))
            frac = r.get("frac", r.get("frac_of_900"))
            cells += [f"{r['ms']:.4f}", f"{gbs:.0f}", f"{frac:.2f}"]
        lines.append(f"| {mb} | {n} | {s} | " + " | ".join(cells) + " |")
    out.write_text("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
