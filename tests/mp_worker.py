"""One rank of a REAL multi-process run of the N > 1 runtime path (launched by
tests/test_multiprocess_gpu.py under torch.distributed.run; not a test file).

Every rank shares GPU 0 and talks over torch.distributed's gloo backend with
CUDA tensors: the same TorchDistTransport code the NCCL path runs (all-gather
fetch, all-to-all + K3 release, the shared wte exchange, the N-scalar
all-reduce), in separate processes with separate CUDA contexts. Trains the
tiny config of tests/test_multirank_gpu.py for two steps and saves this
rank's losses, fp32 master shards and live counters to <out>/rank<r>.npz.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mp_worker.py <plan kind> <out dir> [exchange|ipc|ipc-ce]

"ipc" runs the in-kernel P2P path instead: K2 reads the peers' shards and K3
the peers' rCache blocks through CUDA-IPC mappings of the other processes'
allocations, ordered by elx_device_barrier over IPC-mapped signal pads;
"ipc-ce" does the same with K2 on the copy engines (elx_fetch_ce); "ipc-graph"
captures the second step as one CUDA graph per rank (the ranks' graphs meet
at device-numbered barriers) and replays it. A "-keep" suffix runs the step
with the forward graphs kept instead of recomputed (recompute=False). A
"-nosync" suffix trains three steps with no host synchronisation between them
(losses kept on the device, read at the end): the comm stream's gathers of
step s+1 must be ordered after step s's optimizer update by the runtime's own
stream/event ordering, not by a host sync.
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE))

from paper_2212_05339_b200 import gpt2  # noqa: E402
from paper_2212_05339_b200.gpt2 import ElixirGPT2  # noqa: E402
from paper_2212_05339_b200.transport import IpcTransport, TorchDistTransport  # noqa: E402
from test_multirank_gpu import CFG, HP, _batches, _plan, _rank_masters  # noqa: E402


def main():
    kind, out = sys.argv[1], Path(sys.argv[2])
    path = sys.argv[3] if len(sys.argv) > 3 else "exchange"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # one GPU per rank when the node has them (tests/test_multigpu.py), else every rank on GPU 0
    ndev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", rank)) % ndev if ndev >= world else 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nccl = path.startswith("nccl")
    if nccl:  # the library exchange on distinct GPUs (NCCL refuses ranks that share one)
        path = "exchange" + path[len("nccl"):]
    dist.init_process_group("nccl" if nccl else "gloo", **({"device_id": dev} if nccl else {}))
    plan, _, _ = _plan(kind)
    init = gpt2.init_params(CFG, dev, seed=11)
    if path.startswith("ipc"):  # "ipc": K2 kernel, "ipc-ce": K2 on the copy engines, "ipc-graph": captured step
        transport = IpcTransport(fetch_engine="ce" if path == "ipc-ce" else "sm")
    else:
        transport = TorchDistTransport()
    nosync = path.endswith("-nosync")
    path = path.removesuffix("-nosync")
    keep = path.endswith("-keep")  # the bench's mode: forward graphs kept instead of recomputed
    path = path.removesuffix("-keep")
    model = ElixirGPT2(CFG, plan, device=dev, transport=transport, init=init, recompute=not keep, **HP)
    assert model.keep_graph == keep
    assert model.manager.p2p == path.startswith("ipc")
    losses = []
    for s in range(3 if nosync else 2):
        tok, tgt = _batches(world, s, dev)[rank]
        if path == "ipc-graph" and s == 1:  # step 1 replays a CUDA graph captured on every rank
            model.capture(tok, tgt, warmup=0)
            losses.append(model.graph_step(tok, tgt).clone())
        else:
            losses.append(model.train_step(tok, tgt).clone())
        if not nosync:
            losses[-1] = losses[-1].item()
    losses = [float(x) for x in losses]
    model.synchronize()
    torch.cuda.synchronize()
    rec = {"losses": np.array(losses, np.float64), "counters": np.array(json.dumps(model.fetcher.counters()))}
    for pid, (off, vals) in _rank_masters(model).items():
        rec[f"off::{pid}"] = np.array(off)
        rec[f"val::{pid}"] = vals
    out.mkdir(parents=True, exist_ok=True)
    np.savez(out / f"rank{rank}.npz", **rec)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
