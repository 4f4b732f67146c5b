"""Where the GPU idles inside a training step: torch.profiler over two steps,
union of all kernel/memcpy intervals on the device vs the wall span, and the
largest idle gaps with the kernels on either side.

    python scripts/gap_profile.py [model] > gpurun_out/gaps.json
"""
import json
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt2-1.3b"
cfg = PRESETS[name]
dev = torch.device("cuda:0")
model = ElixirGPT2(cfg, (ROOT / "plans" / f"{name}_n1.json").read_text(), device=dev)
ids = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), device=dev)
tok, tgt = ids[:, :-1].contiguous(), ids[:, 1:].contiguous()
for _ in range(3):
    model.train_step(tok, tgt)
model.synchronize()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        model.train_step(tok, tgt)
    model.synchronize()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
busy, gaps = 0.0, []
cur_s, cur_e, last_name = iv[0][0], iv[0][1], iv[0][2]
for s, e, n in iv[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, last_name[:70], n[:70]))
        cur_s, cur_e = s, e
    elif e > cur_e:
        cur_e = e
    if e >= cur_e:
        last_name = n
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
gaps.sort(reverse=True)
out = {"model": name, "steps": 2, "span_ms": span / 1e3, "busy_ms": busy / 1e3, "idle_ms": (span - busy) / 1e3,
       "n_gaps": len(gaps), "gaps_over_20us_ms": sum(g for g, *_ in gaps if g > 20) / 1e3,
       "top_gaps_us": [{"us": round(g, 1), "after": a, "before": b} for g, a, b in gaps[:25]]}
print(json.dumps(out, indent=1))
