"""End-to-end runtime parity on a real GPU: a chunked GPT-2 step through
ChunkManager / ChunkFetcher / HybridAdam against
  * the oracle schedule (live fetch/release counters == simulate), and
  * a plain reference step — standalone parameter tensors, the same per-node
    recompute, and the CPU oracle's release + AdamW — bit-exact fp32 masters.
Covers GPU-only plans, partial CPU offload, small rCache (evictions and
re-gathers), fp16 with loss scaling and an injected overflow."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from _refstep import ReferenceStep
from oracle import layout_ref as L
from paper_2212_05339_b200 import gpt2
from paper_2212_05339_b200.gpt2 import ElixirGPT2, GPT2Config
from paper_2212_05339_b200.schedule import Plan

pytestmark = pytest.mark.gpu

CFG = GPT2Config(hidden=64, layers=4, heads=4, vocab=389, seq_len=32, batch=2)  # odd vocab: padded view
HP = dict(lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01, max_norm=1.0)


def _oracle_layout(cfg, C):
    params, ops = L.gpt2_records(cfg.hidden, cfg.layers, cfg.vocab, cfg.seq_len)
    _, seq = L.partition(params, ops)
    chunks, where = L.pack(seq, C)
    fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
    return chunks, where, fwd, red


def _plans(cfg):
    h = cfg.hidden
    C = 4 * h * h + 3 * h * h // 2  # forces layers to straddle chunks
    chunks, where, fwd, red = _oracle_layout(cfg, C)
    n = len(chunks)
    ws = max(len(s) for s in fwd)
    return [
        ("all-gpu-max", Plan(C, n, {c: "gpu" for c in range(n)})),
        ("all-gpu-min", Plan(C, ws, {c: "gpu" for c in range(n)})),
        ("offload-half", Plan(C, ws + 1, {c: ("cpu" if c % 2 else "gpu") for c in range(n)})),
        ("offload-all", Plan(C, ws, {c: "cpu" for c in range(n)})),
        # every chunk keeps a block (no eviction), half CPU-home: the resident streamed update
        ("offload-resident", Plan(C, n, {c: ("cpu" if c % 2 else "gpu") for c in range(n)})),
    ]


def _batch(cfg, dev, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    t = torch.randint(0, cfg.vocab, (cfg.batch, cfg.seq_len + 1), generator=g, device=dev)
    return t[:, :-1].contiguous(), t[:, 1:].contiguous()


def _masters(model):
    model.synchronize()
    torch.cuda.synchronize()
    out = model.manager.master_params()
    sp = model.manager.shared["wte"]
    out["wte"] = sp.p32[:sp.numel].clone()
    return {k: v.float().cpu().numpy().reshape(-1) for k, v in out.items()}


@pytest.mark.parametrize("plan_name", ["all-gpu-max", "all-gpu-min", "offload-half", "offload-all"])
def test_counters_equal_simulate(cuda, plan_name):
    plan = dict(_plans(CFG))[plan_name]
    model = ElixirGPT2(CFG, plan, device=cuda, **HP)
    tok, tgt = _batch(CFG, cuda, 0)
    model.train_step(tok, tgt)
    torch.cuda.synchronize()
    chunks, where, fwd, red = _oracle_layout(CFG, plan.chunk_length)
    cpu = {c for c, d in plan.chunk_homes.items() if d.value == "cpu"}
    want, _ = L.simulate(fwd, plan.n_block, cpu, red)
    live = model.fetcher.counters()
    for k in ("gather_ops", "replaced_ops", "reduce_ops", "c2g_units", "g2c_units"):
        assert live[k] == want[k], (k, live, want)
    assert live["peak_rcache_blocks"] == want["peak"]


@pytest.mark.parametrize("overlap", [True, False])
@pytest.mark.parametrize("plan_name", ["all-gpu-max", "all-gpu-min", "offload-half", "offload-all", "offload-resident"])
def test_step_parity_bit_exact(cuda, plan_name, overlap):
    plan = dict(_plans(CFG))[plan_name]
    init = gpt2.init_params(CFG, cuda, seed=5)
    model = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()},
                       overlap_update=overlap, **HP)
    ref = ReferenceStep(model, init, HP)
    for s in range(3):
        tok, tgt = _batch(CFG, cuda, s)
        lo = model.train_step(tok, tgt)
        (lr_,), _ = ref.step([(tok, tgt)])
        torch.cuda.synchronize()
        assert lo.item() == lr_.item(), (s, lo.item(), lr_.item())
        got = _masters(model)
        for pid, want in ref.master.items():
            assert np.array_equal(got[pid], want), (s, pid, np.abs(got[pid] - want).max())


@pytest.mark.parametrize("plan_name", ["offload-half", "offload-resident"])
def test_fp16_loss_scale_and_overflow_skip(cuda, plan_name):
    plan = dict(_plans(CFG))[plan_name]
    init = gpt2.init_params(CFG, cuda, seed=6, dtype=torch.float16)
    model = ElixirGPT2(CFG, plan, device=cuda, dtype=torch.float16, loss_scale=1024.0,
                       init={k: v.clone() for k, v in init.items()}, **HP)
    ref = ReferenceStep(model, init, HP)
    tok, tgt = _batch(CFG, cuda, 1)
    model.train_step(tok, tgt)
    ref.step([(tok, tgt)], scale=1024.0)
    # inject an overflow: an absurd loss scale makes the fp16 grads overflow
    model.scaler.scale = 2.0 ** 60
    before = _masters(model)
    model.train_step(tok, tgt)
    torch.cuda.synchronize()
    assert model.optimizer.last["found_inf"]
    after = _masters(model)
    for k in before:
        assert np.array_equal(before[k], after[k])
    # the compute copies were restored from the masters (grads overwrote them)
    model.scaler.scale = 1024.0
    lo = model.train_step(tok, tgt)
    (lr_,), _ = ref.step([(tok, tgt)], scale=1024.0)
    assert lo.item() == lr_.item()
    got = _masters(model)
    for pid, want in ref.master.items():
        assert np.array_equal(got[pid], want), pid


def test_loss_decreases_on_fixed_batch(cuda):
    plan = dict(_plans(CFG))["all-gpu-min"]
    model = ElixirGPT2(CFG, plan, device=cuda, **HP)
    tok, tgt = _batch(CFG, cuda, 3)
    losses = [model.train_step(tok, tgt).item() for _ in range(8)]
    assert losses[-1] < losses[0] - 0.05, losses


def test_checkpoint_round_trip(cuda):
    """state_dict / load_state_dict restore masters, moments, step and the
    compute copies: a restored trainer continues bit-identically."""
    plan = dict(_plans(CFG))["offload-half"]
    init = gpt2.init_params(CFG, cuda, seed=8)
    a = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    tok, tgt = _batch(CFG, cuda, 4)
    a.train_step(tok, tgt)
    a.train_step(tok, tgt)
    st = a.optimizer.state_dict()
    b = ElixirGPT2(CFG, plan, device=cuda, init=gpt2.init_params(CFG, cuda, seed=99), **HP)
    b.optimizer.load_state_dict(st)
    la = a.train_step(tok, tgt).item()
    lb = b.train_step(tok, tgt).item()
    assert la == lb
    ma, mb = _masters(a), _masters(b)
    for k in ma:
        assert np.array_equal(ma[k], mb[k]), k


@pytest.mark.parametrize("plan_name", ["offload-all", "offload-resident"])
@pytest.mark.parametrize("cpu_update", ["host", "stream", "split"])
def test_offloaded_update_modes_bit_exact(cuda, cpu_update, plan_name):
    """CPU-home chunks updated on host threads, by the GPU-streamed update
    (H2D -> K4 -> D2H in double-buffered tiles), or split between them: all
    bit-exact against the oracle; also across an fp16 overflow skip. On the
    never-evicting plan the streamed chunks are resident (gradient and
    parameters kept in their block between steps)."""
    plan = dict(_plans(CFG))[plan_name]
    init = gpt2.init_params(CFG, cuda, seed=12)
    model = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()},
                       cpu_update=cpu_update, **HP)
    opt = model.optimizer
    if cpu_update == "host":
        assert opt.cpu_segs and not opt.stream_segs
    elif cpu_update == "stream":
        assert opt.stream_segs and not opt.cpu_segs
    else:
        assert opt.cpu_segs and opt.stream_segs
    assert bool(opt.resident) == (plan_name == "offload-resident" and cpu_update != "host")
    opt._init_stream_update(1000) if opt.stream_segs else None  # tiny tiles: several per chunk, both slots
    ref = ReferenceStep(model, init, HP)
    for s in range(3):
        tok, tgt = _batch(CFG, cuda, 10 + s)
        lo = model.train_step(tok, tgt)
        (lr_,), _ = ref.step([(tok, tgt)])
        assert lo.item() == lr_.item(), s
        got = _masters(model)
        for pid, want in ref.master.items():
            assert np.array_equal(got[pid], want), (s, pid)


def test_resident_checkpoint_reload_into_trained_model(cuda):
    """A resident streamed chunk's current parameters live in its block; a checkpoint loaded into a model that
    has trained since must not be shadowed by them: the reloaded model continues exactly like a fresh one."""
    plan = dict(_plans(CFG))["offload-resident"]
    init = gpt2.init_params(CFG, cuda, seed=8)
    a = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, cpu_update="stream", **HP)
    assert a.optimizer.resident
    tok, tgt = _batch(CFG, cuda, 4)
    a.train_step(tok, tgt)
    st = a.optimizer.state_dict()
    a.train_step(tok, tgt)
    a.train_step(tok, tgt)
    assert a.manager.in_block
    a.optimizer.load_state_dict(st)
    b = ElixirGPT2(CFG, plan, device=cuda, init=gpt2.init_params(CFG, cuda, seed=99), cpu_update="stream", **HP)
    b.optimizer.load_state_dict(st)
    assert a.train_step(tok, tgt).item() == b.train_step(tok, tgt).item()
    ma, mb = _masters(a), _masters(b)
    for k in ma:
        assert np.array_equal(ma[k], mb[k]), k
    # the host copies written back on demand equal the parameters in the blocks
    a.optimizer.host_params_current()
    for c, blk in a.optimizer.resident.items():
        n = a.optimizer.stream_segs[c][5]
        assert torch.equal(a.optimizer.stream_segs[c][4][:n], blk[:n].cpu())


@pytest.mark.parametrize("plan_name", ["all-gpu-max", "all-gpu-min"])
def test_cuda_graph_step_equals_eager(cuda, plan_name):
    """The whole step captured as ONE CUDA graph (capture() + graph_step())
    trains exactly like the eager step: same losses, bit-identical fp32
    masters and compute copies after warm-up + replayed steps on new batches."""
    plan = dict(_plans(CFG))[plan_name]
    init = gpt2.init_params(CFG, cuda, seed=5)
    batches = [_batch(CFG, cuda, 100 + s) for s in range(6)]
    eager = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    graph = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    want = [eager.train_step(*batches[0]).item() for _ in range(3)]
    want += [eager.train_step(*b).item() for b in batches[1:]]
    graph.capture(*batches[0], warmup=3)  # the warm-up steps train on batches[0]
    got = [graph.graph_step(*b).item() for b in batches[1:]]
    assert got == want[3:]
    a, b = _masters(eager), _masters(graph)
    assert set(a) == set(b)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    # the compute copy (bf16 chunk) follows the masters too
    for c in eager.manager.gpu_ids:
        r = eager.manager.row[c]
        assert torch.equal(eager.manager.p16[r], graph.manager.p16[r])
    assert eager.optimizer.step_count == graph.optimizer.step_count == 8


@pytest.mark.parametrize("plan_name", ["all-gpu-max", "all-gpu-min"])
def test_keep_graph_step_equals_recompute(cuda, plan_name):
    """recompute=False (the forward keeps each node's autograd graph) trains
    bit-identically to activation checkpointing: same losses, same fp32
    masters — the recompute reproduces the forward exactly, so dropping it
    changes no result, only the work."""
    plan = dict(_plans(CFG))[plan_name]
    init = gpt2.init_params(CFG, cuda, seed=6)
    batches = [_batch(CFG, cuda, 200 + s) for s in range(3)]
    ac = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    kg = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, recompute=False, **HP)
    assert kg.keep_graph and not ac.keep_graph
    assert ElixirGPT2(CFG, plan, device=cuda, recompute="auto", **HP).keep_graph  # resident, small activations
    assert [ac.train_step(*b).item() for b in batches] == [kg.train_step(*b).item() for b in batches]
    a, b = _masters(ac), _masters(kg)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    kg.capture(*batches[0], warmup=1)  # and under graph capture
    kg.graph_step(*batches[1])


def test_keep_graph_refused_when_chunks_can_be_evicted(cuda):
    from paper_2212_05339_b200.errors import ValidationError
    plan = dict(_plans(CFG))["offload-all"]
    with pytest.raises(ValidationError):
        ElixirGPT2(CFG, plan, device=cuda, recompute=False, **HP)
    assert not ElixirGPT2(CFG, plan, device=cuda, recompute="auto", **HP).keep_graph


def test_cuda_graph_refuses_offloaded_plans(cuda):
    from paper_2212_05339_b200.errors import ValidationError
    plan = dict(_plans(CFG))["offload-half"]
    model = ElixirGPT2(CFG, plan, device=cuda, **HP)
    with pytest.raises(ValidationError):
        model.capture(*_batch(CFG, cuda, 1))


@pytest.mark.parametrize("world", [1, 2])
def test_memory_contract_chunk_footprint(cuda, world):
    """The runtime's per-rank allocation against the reference's memory
    contract: every GPU-home chunk holds exactly its shard of p16 + fp32
    p32/m/v (chunk_footprint, cost_model.py:147-153, up to the 8-element shard
    round-up); at N > 1 plus the documented 4 B/element fp32 gradient shard;
    at N = 1 no gradient shard and no rCache for GPU-home chunks (used in place).
    The shared wte holds shared_state_bytes (search.py:116-126) plus its
    vocab padding and, at N > 1, a replicated (not partitioned) gradient."""
    from _refstep import run_ranks
    from paper_2212_05339_b200.runtime import shard_length
    plan = dict(_plans(CFG))["all-gpu-max"]
    C = plan.chunk_length

    def rank_fn(r, transport):
        m = ElixirGPT2(CFG, plan, device=cuda, transport=transport, **HP).manager
        return m.memory_report(), len(m.gpu_ids), m.shared["wte"]

    res = [rank_fn(0, None)] if world == 1 else run_ranks(world, rank_fn)
    S = shard_length(C, world)
    for rep, n_gpu, sp in res:
        per_chunk = rep["gpu_chunk_state_bytes"] // n_gpu
        assert per_chunk == 14 * S
        assert 0 <= per_chunk - L.chunk_footprint(C, world) < 14 * 8
        assert rep["gpu_grad_shard_bytes"] == (0 if world == 1 else 4 * S * n_gpu)
        if world == 1:
            assert rep["rcache_bytes"] == 0
        # contract: replicated compute copy 2*S + partitioned ceil(14*S/N) (p16/gradient + 12 B state)
        contract = L.shared_state_bytes(sp.numel, world)
        vocab_pad = 2 * (sp.full.numel() - sp.numel)      # the lm_head's padded rows (compute view only)
        if world == 1:  # the shard IS the full copy; the gradient buffer is the contract's 2 B term
            ledger = vocab_pad + 2 * (sp.grad.numel() - sp.numel) + 12 * (sp.shard - sp.numel)
        else:           # replicated bf16 gradient buffer + fp32 gradient shard on top of the contract
            ledger = vocab_pad + 2 * sp.grad.numel() + (14 * sp.shard - -(-14 * sp.numel // world)) + 4 * sp.shard
        assert rep["shared_bytes"] - contract == ledger, (rep["shared_bytes"], contract, ledger)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_memory_ledger_partitions_mixed_precision_states(cuda, world):
    """Summed over ranks, the elements each rank owns give exactly the
    reference's whole-model states mixed_precision_states(M) =
    (2M, 2M, 12M) (cost_model.py:156-167): every parameter element is owned
    by one rank, with offloaded plans too."""
    from _refstep import run_ranks
    from paper_2212_05339_b200 import mixed_precision_states
    for name in ("all-gpu-max", "offload-half"):
        plan = dict(_plans(CFG))[name]

        def rank_fn(r, transport):
            model = ElixirGPT2(CFG, plan, device=cuda, transport=transport, **HP)
            return model.manager.memory_ledger(), model.profile.total_elements

        res = [rank_fn(0, None)] if world == 1 else run_ranks(world, rank_fn)
        total = res[0][1]  # M: every parameter element of the model, chunk members and the shared wte
        want = mixed_precision_states(total)
        got = [sum(led[k] for led, _ in res) for k in ("param_bytes", "grad_bytes", "optimizer_bytes")]
        assert tuple(got) == want, (name, got, want)
        assert all(led["reduced_grad_shard_bytes"] == (0 if world == 1 else 2 * led["grad_bytes"]) for led, _ in res)


def test_cuda_graph_checkpoint_round_trip(cuda):
    """A trainer stepping by graph replays checkpoints like an eager one: its
    state_dict (step count from the device counter) restores into a fresh
    eager trainer, and loading a checkpoint INTO the captured trainer (in
    place, same buffers) is picked up by the next replay."""
    plan = dict(_plans(CFG))["all-gpu-max"]
    init = gpt2.init_params(CFG, cuda, seed=12)
    tok, tgt = _batch(CFG, cuda, 6)
    g = ElixirGPT2(CFG, plan, device=cuda, init={k: v.clone() for k, v in init.items()}, **HP)
    g.capture(tok, tgt, warmup=2)
    g.graph_step(tok, tgt)
    g.graph_step(tok, tgt)
    st = g.optimizer.state_dict()
    assert st["step"] == 4
    e = ElixirGPT2(CFG, plan, device=cuda, init=gpt2.init_params(CFG, cuda, seed=99), **HP)
    e.optimizer.load_state_dict(st)
    le = e.train_step(tok, tgt).item()
    lg = g.graph_step(tok, tgt).item()
    assert le == lg
    me, mg = _masters(e), _masters(g)
    for k in me:
        assert np.array_equal(me[k], mg[k]), k
    # restore the step-4 state into the captured trainer and replay: equals the eager continuation
    g.optimizer.load_state_dict(st)
    assert g.graph_step(tok, tgt).item() == le
