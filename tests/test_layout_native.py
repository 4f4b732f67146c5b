"""The product's layout packer and schedule compiler (native, elx_layout_pack /
elx_schedule) against the reference's golden vectors, the oracle, and (in the
build container) the live reference. CPU only: host code in libelixir_b200."""

from __future__ import annotations

import random
import re

import pytest

from oracle import layout_ref as L
from paper_2212_05339_b200 import errors, layout, profiles, schedule
from paper_2212_05339_b200.schedule import Device


def _specs(seq):
    return tuple(profiles.ParameterSpec(pid, n) for pid, n in seq)


def _homes(n_chunks, cpu):
    return {c: (Device.CPU if c in cpu else Device.GPU) for c in range(n_chunks)}


def _check(rec, seq, coarse_nodes):
    specs = _specs(seq)
    if "error" in rec:
        with pytest.raises(errors.ChunkTooSmallError):
            layout.pack_chunks(specs, rec["chunk_length"])
        return
    lay = layout.pack_chunks(specs, rec["chunk_length"])
    index = {pid: i for i, (pid, _) in enumerate(seq)}
    assert [[[index[m.param_id], m.offset, m.numel] for m in c.members] for c in lay.chunks] == rec["chunks"]
    assert layout.waste_rate(lay) == rec["waste_rate"]
    tr = layout.build_chunk_trace(profiles.AccessTrace(tuple(frozenset(x) for x in coarse_nodes)), lay)
    assert [sorted(s) for s in tr.forward] == rec["forward"]
    assert {str(k): v for k, v in sorted(tr.reduce_after.items())} == rec["reduce_after"]
    assert layout.working_set_blocks(tr) == rec["working_set"]
    for sim in rec["simulations"]:
        homes = _homes(lay.n_chunks, set(sim["cpu_home"]))
        if "error" in sim:
            with pytest.raises(errors.InfeasibleCacheError):
                schedule.simulate(tr, sim["n_block"], rec["chunk_length"], homes, gpu_count=4)
            continue
        got = schedule.simulate(tr, sim["n_block"], rec["chunk_length"], homes, gpu_count=4)
        assert got.__dict__ == sim["report"]


@pytest.mark.parametrize("name", ["gpt2-small", "gpt2-1.3b", "gpt2-4b", "gpt2-10b"])
def test_gpt2_native_matches_golden(golden_layouts, name):
    g = golden_layouts["gpt2"][name]
    prof = profiles.synthesize_transformer_profile(g["hidden"], g["layers"], g["heads"], 50257, 1024, 8)
    shared, seq = profiles.partition_multiuse(prof)
    assert shared == g["shared_elements"]
    assert [[p.id, p.numel] for p in seq] == g["sequence"]
    assert [sorted(s) for s in profiles.coarsen_graph(prof).coarse_ops] == g["coarse"]
    for rec in g["layouts"]:
        _check(rec, [(p.id, p.numel) for p in seq], g["coarse"])


def test_random_native_matches_golden(golden_layouts):
    for rec in golden_layouts["random"]:
        prof = profiles.ModelProfile("chain", tuple(profiles.ParameterSpec(*p) for p in rec["params"]),
                                     tuple(profiles.OperatorNode(o[0], tuple(o[1]), o[2]) for o in rec["ops"]))
        shared, seq = profiles.partition_multiuse(prof)
        assert [[p.id, p.numel] for p in seq] == rec["sequence"]
        assert [sorted(s) for s in profiles.coarsen_graph(prof).coarse_ops] == rec["coarse"]
        _check(rec, rec["sequence"], rec["coarse"])


def test_native_events_match_oracle_events():
    """Beyond counters: the gather/evict/reduce event sequence is the oracle's."""
    rng = random.Random(3)
    for _ in range(300):
        n = rng.randint(1, 12)
        seq = [(f"p{i}", rng.randint(1, 40)) for i in range(n)]
        C = max(x for _, x in seq) + rng.randint(0, 40)
        chunks, where = L.pack(seq, C)
        nodes, pos = [], 0
        while pos < n:
            k = rng.randint(1, 3)
            nodes.append({p for p, _ in seq[pos:pos + k]})
            pos += k
        fwd, _, red = L.chunk_trace(nodes, where)
        lay = layout.pack_chunks(_specs(seq), C)
        tr = layout.build_chunk_trace(profiles.AccessTrace(tuple(frozenset(x) for x in nodes)), lay)
        for nb in range(max(len(s) for s in fwd), len(chunks) + 1):
            cpu = {c for c in range(len(chunks)) if rng.random() < 0.4}
            try:
                cnt, evs = L.simulate(fwd, nb, cpu, red)
            except L.OracleError:
                with pytest.raises(errors.InfeasibleCacheError):
                    schedule.compile_schedule(tr, nb, _homes(len(chunks), cpu))
                continue
            sch = schedule.compile_schedule(tr, nb, _homes(len(chunks), cpu))
            got = [("gather" if e["kind"] == 0 else "reduce", int(e["pos"]), int(e["chunk"]), int(e["victim"]))
                   for e in sch.events]
            assert got == evs
            assert sch.counters["peak_rcache_blocks"] == cnt["peak"]
            # block bookkeeping: a gather lands in its victim's block; blocks < n_block
            owner = {}
            for e in sch.events:
                assert 0 <= e["block"] < nb
                if e["kind"] == 0:
                    if e["victim"] >= 0:
                        assert owner[int(e["victim"])] == e["block"]
                        del owner[int(e["victim"])]
                    assert e["block"] not in owner.values()
                    owner[int(e["chunk"])] = int(e["block"])
                    assert 0 <= e["issue_pos"] <= e["pos"]


def _replay_check(walk, nf, red, events, n_block):
    """Replay a compiled program in HOST ISSUE ORDER (at each position: due
    gathers, then gathers issued early for later positions, then compute,
    then releases) and check the hazards the runtime relies on."""
    by_issue = {}
    for e in events:
        if e["kind"] == 0:
            key = int(e["issue_pos"])
            due = int(e["pos"]) == key
            by_issue.setdefault(key, []).append((0 if due else 1, int(e["pos"]), e))
    owner = {}                      # block -> chunk currently written there
    where = {}                      # chunk -> block
    pinned = set()
    for pos in range(len(walk)):
        for _, _, e in sorted(by_issue.get(pos, []), key=lambda t: (t[0], t[1])):
            b, c, v = int(e["block"]), int(e["chunk"]), int(e["victim"])
            assert 0 <= int(e["issue_pos"]) <= int(e["pos"])
            assert c not in where, "gather of a chunk that is still resident elsewhere"
            if v >= 0:
                assert owner.get(b) == v, "victim is not the block's occupant"
                assert v not in walk[pos], "block overwritten while its occupant is in use"
                assert v not in pinned, "block overwritten while its occupant holds unreleased grads"
                del where[v]
            else:
                assert b not in owner
            owner[b] = c
            where[c] = b
        for c in walk[pos]:
            assert c in where, f"chunk {c} needed at {pos} is not resident"
        if pos >= nf:
            pinned |= set(walk[pos])
            for c in walk[pos]:
                if red[c] == pos - nf:
                    pinned.discard(c)
    assert len(owner) <= n_block


def test_prefetch_never_overwrites_a_block_in_use():
    """The prefetch horizon (issue_pos) never lets a gather clobber a block whose
    chunk is in use or pinned, never double-maps a chunk, and every needed chunk
    is resident — checked by replaying the program in issue order."""
    rng = random.Random(11)
    checked = 0
    for _ in range(300):
        n = rng.randint(2, 14)
        seq = [(f"p{i}", rng.randint(1, 30)) for i in range(n)]
        C = max(x for _, x in seq) + rng.randint(0, 30)
        _, where = L.pack(seq, C)
        nodes, pos = [], 0
        while pos < n:
            k = rng.randint(1, 3)
            nodes.append({p for p, _ in seq[pos:pos + k]})
            pos += k
        fwd, bwd, red = L.chunk_trace(nodes, where)
        lay = layout.pack_chunks(_specs(seq), C)
        tr = layout.build_chunk_trace(profiles.AccessTrace(tuple(frozenset(x) for x in nodes)), lay)
        for nb in range(1, lay.n_chunks + 1):
            try:
                sch = schedule.compile_schedule(tr, nb, _homes(lay.n_chunks, set()))
            except errors.InfeasibleCacheError:
                continue
            _replay_check(fwd + bwd, len(fwd), red, sch.events, nb)
            checked += 1
    assert checked > 200


def test_prefetch_horizon_on_gpt2_plans():
    """Real plans: the replay check holds and gathers are issued ahead of time."""
    import json
    from pathlib import Path
    from paper_2212_05339_b200.gpt2 import PRESETS
    for f in ("gpt2-4b_offload_n1.json", "gpt2-10b_offload_n2.json", "gpt2-1.3b_32mb_n8.json"):
        path = Path(__file__).resolve().parents[1] / "plans" / f
        doc = json.loads(path.read_text())
        plan = schedule.load_plan(path.read_text())
        cfg = PRESETS[doc["meta"]["model"]]
        prof = profiles.synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, 50257, 1024, 8)
        _, seq = profiles.partition_multiuse(prof)
        lay = layout.pack_chunks(seq, plan.chunk_length)
        tr = layout.build_chunk_trace(profiles.coarsen_graph(prof), lay)
        sch = schedule.compile_schedule(tr, plan.n_block, plan.chunk_homes)
        walk = [set(x) for x in tr.forward] + [set(x) for x in tr.backward]
        _replay_check(walk, len(tr.forward), dict(tr.reduce_after), sch.events, plan.n_block)
        g = sch.events[sch.events["kind"] == 0]
        assert (g["pos"] - g["issue_pos"]).max() >= 2, f


def test_pack_errors_name_the_parameter():
    with pytest.raises(errors.ChunkTooSmallError, match="'p0'"):
        layout.pack_chunks(_specs([("p0", 5), ("p1", 3), ("p2", 4)]), 4)
    with pytest.raises(errors.ValidationError):
        layout.pack_chunks(_specs([("p0", 5)]), 0)
    assert layout.pack_chunks((), 8).n_chunks == 0


def test_schedule_validation_errors():
    tr = layout.ChunkTrace((frozenset({0, 1}),), (frozenset({0, 1}),), {0: 0, 1: 0})
    with pytest.raises(errors.InfeasibleCacheError, match="working set"):
        schedule.compile_schedule(tr, 1, {0: "gpu", 1: "gpu"})
    with pytest.raises(errors.ValidationError, match="placement"):
        schedule.compile_schedule(tr, 2, {0: "gpu"})
    with pytest.raises(errors.ValidationError):
        schedule.compile_schedule(tr, 0, {0: "gpu", 1: "gpu"})


def test_plan_files_load_and_match_layouts():
    """Every committed plan (made by offplan.build_plan) packs into the same chunk
    ids under the native packer (cli.py:255-259) and compiles."""
    import json
    from pathlib import Path
    from paper_2212_05339_b200.gpt2 import PRESETS
    plans = sorted((Path(__file__).resolve().parents[1] / "plans").glob("gpt2-*.json"))
    assert plans
    for f in plans:
        doc = json.loads(f.read_text())
        plan = schedule.load_plan(f.read_text())
        cfg = PRESETS[doc["meta"]["model"]]
        prof = profiles.synthesize_transformer_profile(cfg.hidden, cfg.layers, cfg.heads, 50257, 1024, 8)
        _, seq = profiles.partition_multiuse(prof)
        lay = layout.pack_chunks(seq, plan.chunk_length)
        assert set(plan.chunk_homes) == set(range(lay.n_chunks)), f.name
        tr = layout.build_chunk_trace(profiles.coarsen_graph(prof), lay)
        rep = schedule.simulate(tr, plan.n_block, plan.chunk_length, plan.chunk_homes,
                                gpu_count=doc["meta"]["gpu_count"])
        est = plan.estimates
        for k in ("gather_ops", "gather_bytes", "reduce_bytes", "g2c_bytes", "c2g_bytes", "replaced_bytes",
                  "peak_rcache_blocks"):
            assert getattr(rep, k) == getattr(est, k), (f.name, k)


@pytest.mark.ref
def test_native_vs_live_reference(offplan):
    ref = offplan
    rng = random.Random(5)
    for _ in range(100):
        n = rng.randint(1, 14)
        seq = [(f"p{i}", rng.randint(1, 60)) for i in range(n)]
        C = max(x for _, x in seq) + rng.randint(0, 50)
        lay_r = ref.pack_chunks(tuple(ref.ParameterSpec(p, x) for p, x in seq), C)
        lay_n = layout.pack_chunks(_specs(seq), C)
        assert [[(m.param_id, m.offset, m.numel) for m in c.members] for c in lay_r.chunks] == \
            [[(m.param_id, m.offset, m.numel) for m in c.members] for c in lay_n.chunks]
        nodes, pos = [], 0
        while pos < n:
            k = rng.randint(1, 4)
            nodes.append(frozenset(p for p, _ in seq[pos:pos + k]))
            pos += k
        tr_r = ref.build_chunk_trace(ref.AccessTrace(tuple(nodes)), lay_r)
        for nb in range(1, lay_r.n_chunks + 2):
            homes = {c: rng.choice([ref.Device.GPU, ref.Device.CPU]) for c in tr_r.chunk_ids}
            try:
                want = ref.simulate(ref.CachePolicyInput(tr_r, nb, C, homes, ref.PrecisionSpec(), 3))
            except ref.InfeasibleCacheError:
                with pytest.raises(errors.InfeasibleCacheError):
                    schedule.simulate(tr_r, nb, C, {c: d.value for c, d in homes.items()}, gpu_count=3)
                continue
            got = schedule.simulate(tr_r, nb, C, {c: d.value for c, d in homes.items()}, gpu_count=3)
            assert got.__dict__ == want.__dict__


from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=200, derandomize=True, deadline=None)
@given(st.lists(st.integers(1, 5000), min_size=1, max_size=40), st.integers(0, 3000))
def test_native_pack_property(numels, slack):
    """The reference's packing property (tests/test_chunking.py:97-116 of the
    reference, same hypothesis settings) on the native packer: in-order, no
    straddling, offsets contiguous from 0 inside each chunk, no chunk over C,
    a parameter opens a new chunk only when it would not fit — and equal to
    the oracle's packing."""
    C = max(numels) + slack
    seq = [(f"p{i}", n) for i, n in enumerate(numels)]
    lay = layout.pack_chunks(_specs(seq), C)
    flat = [m for c in lay.chunks for m in c.members]
    assert [m.param_id for m in flat] == [p for p, _ in seq]
    for ci, c in enumerate(lay.chunks):
        off = 0
        for m in c.members:
            assert m.offset == off
            off += m.numel
        assert off <= C
        if ci + 1 < len(lay.chunks):  # greedy: the next chunk's first member did not fit here
            assert off + lay.chunks[ci + 1].members[0].numel > C
    chunks, _ = L.pack(seq, C)
    assert [[(m.param_id, m.offset, m.numel) for m in c.members] for c in lay.chunks] == \
        [[(p, o, n) for p, o, n in ch] for ch in chunks]
