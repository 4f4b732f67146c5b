"""Probe: which multi-process primitives work with N ranks sharing ONE GPU.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/probe_multiproc.py

Prints one line per primitive (rank 0): gloo collectives on CUDA tensors, and
torch symmetric memory (peer pointers into another process's allocation on the
same device) read by our K2 fetch kernel.
"""
import os
import sys
import traceback
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
dist.init_process_group("gloo")
res = {}


def trial(name, fn):
    try:
        res[name] = fn()
    except Exception as exc:  # noqa: BLE001 - probe
        res[name] = f"FAIL {type(exc).__name__}: {str(exc)[:200]}"
        if rank == 0:
            traceback.print_exc()


def ag():
    s = torch.full((8,), rank, dtype=torch.bfloat16, device=dev)
    out = torch.empty(8 * world, dtype=torch.bfloat16, device=dev)
    dist.all_gather(list(out.chunk(world)), s)
    return out.float().tolist()[::8]


def a2a():
    s = torch.arange(4 * world, dtype=torch.float32, device=dev) + 100 * rank
    out = torch.empty_like(s)
    dist.all_to_all_single(out, s)
    return out.tolist()


def ar():
    t = torch.tensor([1.0 + rank], dtype=torch.float64, device=dev)
    dist.all_reduce(t)
    return t.item()


def symm():
    import torch.distributed._symmetric_memory as sm
    from paper_2212_05339_b200 import kernels
    try:
        sm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
    except Exception:
        pass
    t = sm.empty(1024, dtype=torch.bfloat16, device=dev)
    t.fill_(rank + 1)
    h = sm.rendezvous(t, dist.group.WORLD)
    torch.cuda.synchronize()
    h.barrier(channel=0)
    torch.cuda.synchronize()
    blk = torch.empty(1024 * world, dtype=torch.bfloat16, device=dev)
    kernels.fetch(blk, [int(p) for p in h.buffer_ptrs], 1024)
    torch.cuda.synchronize()
    return [blk[i * 1024].item() for i in range(world)]


trial("gloo_all_gather_cuda", ag)
trial("gloo_all_to_all_cuda", a2a)
trial("gloo_all_reduce_cuda", ar)
trial("symm_mem_same_gpu_fetch", symm)
dist.barrier()
if rank == 0:
    for k, v in res.items():
        print("PROBE", k, v, flush=True)
dist.destroy_process_group()
