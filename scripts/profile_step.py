"""One profiled training step for ncu (cudaProfilerStart/Stop around it).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:adam_kernel -c 1 -o gpurun_out/adam python scripts/profile_step.py
"""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05339_b200.gpt2 import PRESETS, ElixirGPT2  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
model_name = args[0] if args else "gpt2-1.3b"
cfg = PRESETS[model_name]
dev = torch.device("cuda:0")
# the bench's mode: forward graphs kept (no recompute) when the plan allows it; --recompute for checkpointing
model = ElixirGPT2(cfg, (ROOT / "plans" / f"{model_name}_n1.json").read_text(), device=dev,
                   recompute=True if "--recompute" in sys.argv else "auto")
ids = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), device=dev)
tok, tgt = ids[:, :-1].contiguous(), ids[:, 1:].contiguous()
for _ in range(2):
    model.train_step(tok, tgt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
model.train_step(tok, tgt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one step; valid adam elements", model.optimizer.gpu_elements)
