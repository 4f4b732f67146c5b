"""the host side of the path timed per BASELINE config —
pack_chunks + build_chunk_trace + simulate (the schedule the runtime replays)
— three ways on the same inputs:

  native     this package (elx_layout_pack / elx_schedule, C++ behind ctypes);
  reference  the reference's own offplan functions (live import of
             /root/reference, present only in the build container);
  oracle     oracle/layout_ref.py, the plain-loop restatement.

The three must agree (counters and layouts are compared on every row).

    python scripts/host_logic_bench.py [--reps 20]   -> one JSON line per (config, impl)

The sizes are the committed plans' (plans/*.json: model, chunk length, n_block,
homes). Runs on CPU only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = Path("/root/reference/pkg/src")

from oracle import layout_ref as L  # noqa: E402
from paper_2212_05339_b200 import layout, profiles, schedule  # noqa: E402
from paper_2212_05339_b200.gpt2 import PRESETS  # noqa: E402

PLANS = ["gpt2-small_n1.json", "gpt2-1.3b_n1.json", "gpt2-1.3b_32mb_n8.json", "gpt2-4b_offload_n1.json",
         "gpt2-10b_offload_n1.json", "gpt2-10b_offload_n8.json"]


def _time(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ref = None
    if REF.exists():
        sys.path.insert(0, str(REF))
        import offplan as ref  # noqa: F401
    host = {"cpus": len(os.sched_getaffinity(0)), "python": sys.version.split()[0]}
    for name in PLANS:
        doc = json.loads((ROOT / "plans" / name).read_text())
        plan = schedule.load_plan((ROOT / "plans" / name).read_text())
        cfg = PRESETS[doc["meta"]["model"]]
        gpus = doc["meta"]["gpu_count"]
        prof = profiles.synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, 50257, 1024, 8)
        _, seq = profiles.partition_multiuse(prof)
        coarse = profiles.coarsen_graph(prof)
        C, nb, homes = plan.chunk_length, plan.n_block, plan.chunk_homes

        def native():
            lay = layout.pack_chunks(seq, C)
            tr = layout.build_chunk_trace(coarse, lay)
            return schedule.simulate(tr, nb, C, homes, gpu_count=gpus)

        rows = {}
        rows["native"] = _time(native, args.reps)
        want = rows["native"][1]

        params, ops = L.gpt2_records(cfg.hidden, cfg.layers, cfg.vocab, cfg.seq_len)
        _, lseq = L.partition(params, ops)
        lcoarse = L.coarsen(params, ops)
        cpu = {c for c, d in homes.items() if str(getattr(d, "value", d)) == "cpu"}

        def oracle():
            chunks, where = L.pack(lseq, C)
            fwd, _, red = L.chunk_trace(lcoarse, where)
            return L.simulate(fwd, nb, cpu, red)[0]

        rows["oracle"] = _time(oracle, max(1, args.reps // 4))
        sim = rows["oracle"][1]
        assert sim["gather_ops"] == want.gather_ops, name
        assert sim["replaced_ops"] * C * 2 == want.replaced_bytes, name

        if ref is not None:
            rprof = ref.synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, 50257, 1024, 8)
            _, rseq = ref.partition_multiuse(rprof)
            rcoarse = ref.coarsen_graph(rprof)
            rhomes = {c: ref.Device(str(getattr(d, "value", d))) for c, d in homes.items()}

            def reference():
                lay = ref.pack_chunks(rseq, C)
                tr = ref.build_chunk_trace(rcoarse, lay)
                return ref.simulate(ref.CachePolicyInput(tr, nb, C, rhomes, ref.PrecisionSpec(), gpus))

            rows["reference"] = _time(reference, args.reps)
            got = rows["reference"][1]
            assert got.__dict__ == want.__dict__, name
        for impl, (ms, _) in rows.items():
            print(json.dumps({"bench": "host_logic", "plan": name, "impl": impl, "ms": round(ms, 4),
                              "n_chunks": len(homes), "n_block": nb, "gather_ops": want.gather_ops,
                              "speedup_vs_reference": (round(rows["reference"][0] / ms, 1)
                                                       if "reference" in rows else None),
                              "host": host}), flush=True)


if __name__ == "__main__":
    main()
