"""One launch each of K2 (fetch, world 8) and K3 (release, world 2/4/8, fp32
output) on a 128 MB chunk with local buffers standing in for the peers — the
target of the `ncu --set full` captures in profiles/ (r02n_*):
    ncu --set full -k regex:'release_tma|fetch_tma' python scripts/k2k3_ncu.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402
from paper_2212_05339_b200.runtime import shard_length  # noqa: E402

dev = torch.device("cuda", 0)
C = 128 * 2 ** 20 // 2
for w in (2, 4, 8):
    S = shard_length(C, w)
    shards = [torch.randn(S, device=dev).to(torch.bfloat16) for _ in range(w)]
    g32 = torch.empty(S, device=dev)
    sc = kernels.new_step_scalars(dev)
    kernels.release(g32, [s.data_ptr() for s in shards], S, torch.bfloat16, 1.0, sc)
    if w == 8:
        block = torch.empty(w * S, dtype=torch.bfloat16, device=dev)
        kernels.fetch(block, [s.data_ptr() for s in shards], S)
torch.cuda.synchronize()
print("ok")
