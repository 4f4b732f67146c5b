"""GPT-2 4B offload plan (configs[2]) trained for a few steps twice from the
same init on the same batches — with the resident streamed update (streamed
CPU-home chunks keep gradient and parameters in their rCache block) and with
the round-trip form (ELX_RESIDENT_STREAM=0) — under deterministic library
algorithms: the per-step losses and every fp32 master must be bit-identical.

    python scripts/offload_equivalence.py [steps] > gpurun_out/offload_equivalence.json
"""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2, init_params  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda:0")
torch.backends.cudnn.deterministic = True
torch.use_deterministic_algorithms(True)
cfg = PRESETS["gpt2-4b"]
plan = (ROOT / "plans" / "gpt2-4b_offload_n1.json").read_text()


def run(resident: bool):
    os.environ["ELX_RESIDENT_STREAM"] = "1" if resident else "0"
    model = ElixirGPT2(cfg, plan, device=dev, init=init_params(cfg, dev, 1234, torch.bfloat16), lr=3e-4)
    opt = model.optimizer
    info = {"resident": sorted(opt.resident), "streamed": sorted(opt.stream_segs), "host": sorted(opt.cpu_segs)}
    losses = []
    t0 = time.perf_counter()
    for s in range(steps):
        g = torch.Generator(device=dev).manual_seed(500 + s)
        ids = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=g, device=dev)
        losses.append(float(model.train_step(ids[:, :-1].contiguous(), ids[:, 1:].contiguous())))
    model.synchronize()
    torch.cuda.synchronize(dev)
    h = hashlib.sha256()
    for name, t in sorted(model.manager.master_params().items()):
        h.update(name.encode())
        h.update(t.float().cpu().numpy().tobytes())
    sp = model.manager.shared["wte"]
    h.update(sp.p32[:sp.numel].cpu().numpy().tobytes())
    info.update(losses=losses, masters_sha256=h.hexdigest(), seconds=round(time.perf_counter() - t0, 1))
    del model, opt
    torch.cuda.empty_cache()
    return info


a = run(True)
b = run(False)
print(json.dumps({"bench": "offload_equivalence", "model": "gpt2-4b", "plan": "gpt2-4b_offload_n1.json",
                  "steps": steps, "deterministic": True, "resident_run": a, "round_trip_run": b,
                  "losses_bit_identical": a["losses"] == b["losses"],
                  "masters_bit_identical": a["masters_sha256"] == b["masters_sha256"]}))
