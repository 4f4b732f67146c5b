"""Generate the committed golden fixtures and runtime plans FROM THE REFERENCE.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package (`/root/reference/pkg/src/offplan`) and
torch (CPU) and writes:

  tests/golden/layouts.json     pack_chunks / build_chunk_trace / simulate
                                outputs for the GPT-2 configs of BASELINE.json
                                and for seeded random chain profiles;
  tests/golden/adamw_golden.npz torch.optim.AdamW (single-tensor, CPU) +
                                unscale + clip_grad_norm_ trajectories;
  plans/*.json                  offplan.build_plan outputs used by bench.py /
                                tests (the runtime's input; BASELINE configs).

Nothing on the GPU box reads /root/reference; it reads these files.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
GOLDEN = ROOT / "tests" / "golden"
PLANS = ROOT / "plans"

GPT2 = {  # name: (hidden, layers, heads) — profiles.py:408, Table 7
    "gpt2-small": (768, 12, 12),
    "gpt2-1.3b": (2048, 24, 16),
    "gpt2-4b": (3072, 32, 24),
    "gpt2-10b": (4096, 48, 32),
}
MI = 2 ** 20


def b200_placeholder_hw(ref, n_max: int = 8):
    """Rate table used for planning until bench.py --profile-hw measures one.
    GB/s in the reference's conventions (profiles.py:158-178)."""
    tables = {}
    for n in range(1, n_max + 1):
        tables[n] = ref.RateTable(b_c2g=50e9 * n ** 0.5, b_g2c=45e9 * n ** 0.5, v_g=800e9 * n,
                                  v_c=10e9, b_g2g=None if n == 1 else 700e9)
    return ref.HardwareProfile(n_max, 180 * 10 ** 9, tables)


def layout_record(ref, profile, chunk_length, placements_rng):
    _, single = ref.partition_multiuse(profile)
    index = {p.id: i for i, p in enumerate(single)}
    try:
        layout = ref.pack_chunks(single, chunk_length)
    except ref.ChunkTooSmallError as exc:
        return {"chunk_length": chunk_length, "error": "chunk_too_small", "message": str(exc)}
    trace = ref.build_chunk_trace(ref.coarsen_graph(profile), layout)
    ws = ref.working_set_blocks(trace)
    sims = []
    nbs = sorted({ws, ws + 1, max(ws, layout.n_chunks // 2), layout.n_chunks})
    for nb in nbs:
        for mode in ("gpu", "cpu", "mixed"):
            if mode == "gpu":
                homes = {c: ref.Device.GPU for c in trace.chunk_ids}
            elif mode == "cpu":
                homes = {c: ref.Device.CPU for c in trace.chunk_ids}
            else:
                homes = {c: placements_rng.choice([ref.Device.GPU, ref.Device.CPU]) for c in trace.chunk_ids}
            try:
                rep = ref.simulate(ref.CachePolicyInput(trace, nb, chunk_length, homes,
                                                        ref.PrecisionSpec(), 4))
                sims.append({"n_block": nb, "cpu_home": sorted(c for c, d in homes.items()
                                                              if d is ref.Device.CPU),
                             "report": rep.__dict__})
            except ref.InfeasibleCacheError as exc:
                sims.append({"n_block": nb, "cpu_home": [], "error": "infeasible_cache",
                             "message": str(exc)})
    return {
        "chunk_length": chunk_length,
        "n_chunks": layout.n_chunks,
        "waste_rate": ref.waste_rate(layout),
        "total_elements": layout.total_elements,
        # per chunk: [sequence index, offset, numel]
        "chunks": [[[index[m.param_id], m.offset, m.numel] for m in c.members] for c in layout.chunks],
        "forward": [sorted(s) for s in trace.forward],
        "reduce_after": {str(k): v for k, v in sorted(trace.reduce_after.items())},
        "working_set": ws,
        "simulations": sims,
    }


def random_chain(ref, rng):
    n = rng.randint(1, 12)
    numels = [rng.randint(1, 64) for _ in range(n)]
    shared = {i for i in range(n) if rng.random() < 0.15}
    if len(shared) == n:
        shared.pop()
    params = tuple(ref.ParameterSpec(f"p{i}", x, shared=(i in shared)) for i, x in enumerate(numels))
    ops, pos, k = [], 0, 0
    while pos < n:
        size = rng.randint(1, min(3, n - pos))
        ids = tuple(f"p{i}" for i in range(pos, pos + size))
        group = rng.choice([None, None, k // 2])
        ops.append(ref.OperatorNode(f"op{k}", ids, group))
        pos += size
        k += 1
    # ops sharing a group must be contiguous for the profile to stay "common"
    return ref.ModelProfile("chain", params, tuple(ops), 0, 0)


def make_layouts(ref):
    out = {"gpt2": {}, "random": []}
    rng = random.Random(2212_05339)
    for name, (h, l, heads) in GPT2.items():
        prof = ref.synthesize_transformer_profile(h, l, heads, 50257, 1024, 8, name=name)
        _, single = ref.partition_multiuse(prof)
        biggest = max(p.numel for p in single)
        lengths = sorted({biggest, 16 * MI, 32 * MI, 100 * MI, 84182029, biggest + 12345})
        out["gpt2"][name] = {
            "hidden": h, "layers": l, "heads": heads,
            "sequence": [[p.id, p.numel] for p in single],
            "shared_elements": sum(p.numel for p in prof.parameters if p.shared),
            "coarse": [sorted(s) for s in ref.coarsen_graph(prof).coarse_ops],
            "layouts": [layout_record(ref, prof, L, rng) for L in lengths],
        }
    for case in range(150):
        prof = random_chain(ref, rng)
        try:
            trace_nodes = ref.coarsen_graph(prof)
        except ref.UncommonGraphError:
            continue
        shared_elems, single = ref.partition_multiuse(prof)
        if not single:
            continue
        L = max(p.numel for p in single) + rng.randint(0, 40)
        rec = layout_record(ref, prof, L, rng)
        rec["params"] = [[p.id, p.numel, p.shared] for p in prof.parameters]
        rec["ops"] = [[o.name, list(o.param_ids), o.ac_group] for o in prof.operators]
        rec["sequence"] = [[p.id, p.numel] for p in single]
        rec["shared_elements"] = shared_elems
        rec["coarse"] = [sorted(s) for s in trace_nodes.coarse_ops]
        out["random"].append(rec)
    # Memory contracts (cost_model.py:147-153, search.py:116-126)
    out["chunk_footprint"] = [[C, n, ref.chunk_footprint(C, n, ref.PrecisionSpec())]
                              for C in (1, 7, 16 * MI, 84182029) for n in (1, 2, 3, 4, 8)]
    out["shared_state_bytes"] = [[S, n, ref.shared_state_bytes(S, n)]
                                 for S in (0, 38597376, 102926336) for n in (1, 2, 4, 8)]
    (GOLDEN / "layouts.json").write_text(json.dumps(out, separators=(",", ":")))
    print("layouts.json:", (GOLDEN / "layouts.json").stat().st_size, "bytes")


def make_memory(ref):
    """The memory contracts (cost_model.py:147-167, search.py:116-126) at the
    BASELINE model sizes and edge cases, with default and custom widths."""
    sizes = [1, 7, 124439808, 1313626112, 3782697984, 9876287488]
    precs = [(2, 4, 3), (4, 4, 3), (2, 4, 2)]
    out = {"mixed_precision_states": [], "chunk_footprint": [], "shared_state_bytes": []}
    for lc, ob, of in precs:
        P = ref.PrecisionSpec(compute_bytes=lc, optimizer_bytes=ob, optimizer_factor=of)
        for M in sizes:
            out["mixed_precision_states"].append([M, [lc, ob, of], list(ref.mixed_precision_states(M, P))])
        for C in (1, 7, 16 * MI, 84182029, 100 * MI):
            for n in (1, 2, 3, 8):
                out["chunk_footprint"].append([C, n, [lc, ob, of], ref.chunk_footprint(C, n, P)])
        for S in (0, 38597376, 102926336):
            for n in (1, 2, 8):
                out["shared_state_bytes"].append([S, n, [lc, ob, of], ref.shared_state_bytes(S, n, P)])
    for bad in (0, -1):
        try:
            ref.mixed_precision_states(bad, ref.PrecisionSpec())
            raise SystemExit("expected ValidationError")
        except ref.ValidationError:
            out.setdefault("mixed_precision_states_invalid", []).append(bad)
    (GOLDEN / "memory.json").write_text(json.dumps(out, separators=(",", ":")))
    print("memory.json:", (GOLDEN / "memory.json").stat().st_size, "bytes")


def make_adamw():
    import torch

    torch.manual_seed(1234)
    sizes = [1000, 4099, 77, 8192]
    world = 3
    steps = 5
    hp = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    max_norm = 1.0
    inv_scale = 1.0 / 64.0
    params = [torch.nn.Parameter(torch.randn(n) * 0.02) for n in sizes]
    opt = torch.optim.AdamW(params, foreach=False, fused=False, **hp)
    rec = {f"p0_{i}": p.detach().numpy().copy() for i, p in enumerate(params)}
    for s in range(steps):
        # per-rank bf16 gradients (scaled by the loss scale 64)
        grads_r = [[(torch.randn(n) * 0.5 * (1 + s)).to(torch.bfloat16) for n in sizes] for _ in range(world)]
        if s == 3:
            grads_r[1][2][5] = float("inf")  # overflow step: GradScaler skips it
        for i in range(len(sizes)):
            for r in range(world):
                rec[f"g{s}_{i}_r{r}"] = grads_r[r][i].view(torch.int16).numpy().view(np.uint16).copy()
        reduced = []
        for i in range(len(sizes)):
            acc = grads_r[0][i].float()
            for r in range(1, world):
                acc = acc + grads_r[r][i].float()
            reduced.append(acc * inv_scale)
        found_inf = any(not torch.isfinite(g).all() for g in reduced)
        for p, g in zip(params, reduced):
            p.grad = g.clone()
        if not found_inf:
            norm = torch.nn.utils.clip_grad_norm_(params, max_norm)
            rec[f"norm{s}"] = np.float64(norm.item())
            opt.step()
        rec[f"skip{s}"] = np.int8(found_inf)
        opt.zero_grad(set_to_none=True)
        for i, p in enumerate(params):
            st = opt.state.get(p, {})
            rec[f"p{s + 1}_{i}"] = p.detach().numpy().copy()
            if st:
                rec[f"m{s + 1}_{i}"] = st["exp_avg"].numpy().copy()
                rec[f"v{s + 1}_{i}"] = st["exp_avg_sq"].numpy().copy()
    rec["meta"] = np.array(json.dumps(dict(sizes=sizes, world=world, steps=steps, max_norm=max_norm,
                                           inv_scale=inv_scale, lr=hp["lr"], betas=hp["betas"],
                                           eps=hp["eps"], weight_decay=hp["weight_decay"],
                                           torch=torch.__version__)))
    np.savez_compressed(GOLDEN / "adamw_golden.npz", **rec)
    print("adamw_golden.npz written")


def make_plans(ref):
    PLANS.mkdir(exist_ok=True)
    measured = PLANS / "hardware_b200_measured.json"
    if measured.exists():  # written by scripts/profile_hw.py on the B200 box (§8f row 2)
        hw = ref.load_hardware_profile(measured.read_text())
        print("planning with", measured.name)
    else:
        hw = b200_placeholder_hw(ref)
        (PLANS / "hardware_b200_placeholder.json").write_text(ref.serialize_hardware_profile(hw))

    def hw_n(n):
        return ref.HardwareProfile(n, hw.gpu_capacity_bytes, {k: hw.rates(k) for k in range(1, n + 1)})

    def emit(fname, name, n, **kw):
        h, l, heads = GPT2[name]
        prof = ref.synthesize_transformer_profile(h, l, heads, 50257, 1024, 8, name=name)
        plan = ref.build_plan(prof, hw_n(n), **kw)
        meta = {"model": name, "gpu_count": n,
                "overrides": {k: (v if not isinstance(v, list) else f"{len(v)} candidates")
                              for k, v in kw.items()}}
        (PLANS / fname).write_text(ref.serialize_plan(plan, meta=meta))
        print(fname, plan.chunk_length, plan.n_block, len(plan.chunk_homes), plan.gpu_home_chunks)

    mib_cands = lambda lo, hi, step: [k * MI for k in range(lo, hi + 1, step)]
    # C1: GPT-2 small, world 1, 32 MB chunks (16 Mi elements), all blocks.
    emit("gpt2-small_n1.json", "gpt2-small", 1, candidates=[16 * MI])
    # Multi-process runs of the N > 1 path (tests/test_multiprocess_gpu.py: N ranks on one GPU over
    # gloo): GPT-2 small at 2 and 4 ranks, all blocks, and with a tight budget (n_block 2 of 12: evictions, 5 chunks CPU-home).
    for n in (2, 4):
        emit(f"gpt2-small_n{n}.json", "gpt2-small", n, candidates=[16 * MI])
    emit("gpt2-small_rcache_n2.json", "gpt2-small", 2, candidates=[8 * MI], u_allowed=0.8e9)
    # C2: GPT-2 1.3B searched over Mi-multiple chunk lengths, 1/2/4/8 GPUs.
    for n in (1, 2, 4, 8):
        emit(f"gpt2-1.3b_n{n}.json", "gpt2-1.3b", n, candidates=mib_cands(16, 128, 2))
    emit("gpt2-1.3b_32mb_n8.json", "gpt2-1.3b", 8, candidates=[16 * MI])
    # C3: GPT-2 4B with partial offload (budget pinned so 0 < gpu_home < n_chunks).
    emit("gpt2-4b_offload_n1.json", "gpt2-4b", 1, u_allowed=30e9, candidates=mib_cands(36, 256, 4))
    emit("gpt2-4b_offload_n2.json", "gpt2-4b", 2, u_allowed=20e9, candidates=mib_cands(36, 256, 4))
    # C4: GPT-2 10B with cached chunks (working set < n_block < n_chunks) and cold chunks on CPU.
    # n=1: budget 100 GB -> 13 of 24 chunks GPU-home, 11 CPU-home (72 GB of pinned host shard state;
    # the B200 box has 196 GB of host RAM, which a 20 GB budget's all-CPU plan, ~158 GB pinned, would exhaust).
    for n, u in ((1, 100e9), (2, 12e9), (4, 8e9), (8, 8e9)):
        emit(f"gpt2-10b_offload_n{n}.json", "gpt2-10b", n, u_allowed=u, candidates=mib_cands(64, 512, 8))


def main():
    sys.path.insert(0, str(REF))
    import offplan as ref

    GOLDEN.mkdir(parents=True, exist_ok=True)
    make_layouts(ref)
    make_memory(ref)
    make_adamw()
    make_plans(ref)


if __name__ == "__main__":
    main()
