"""The layout/schedule oracle (oracle/layout_ref.py) pinned against the
reference: committed golden vectors made by the reference itself, the
reference's own known-answer tests, and (in the build container) the live
reference on seeded random inputs."""

from __future__ import annotations

import random

import pytest

from oracle import layout_ref as L


def _seq(rec):
    return [(pid, n) for pid, n in rec["sequence"]]


def _check_layout(seq, rec):
    if "error" in rec:
        with pytest.raises(L.OracleError):
            L.pack(seq, rec["chunk_length"])
        return None
    chunks, where = L.pack(seq, rec["chunk_length"])
    index = {pid: i for i, (pid, _) in enumerate(seq)}
    got = [[[index[pid], off, n] for pid, off, n in ch] for ch in chunks]
    assert got == rec["chunks"]
    total = sum(n for _, n in seq)
    assert L.waste(chunks, rec["chunk_length"], total) == pytest.approx(rec["waste_rate"], abs=0, rel=1e-15)
    return chunks, where


def _check_sims(forward, red, rec):
    for sim in rec["simulations"]:
        if "error" in sim:
            with pytest.raises(L.OracleError):
                L.simulate(forward, sim["n_block"], set(sim["cpu_home"]), red)
            continue
        cnt, _ = L.simulate(forward, sim["n_block"], set(sim["cpu_home"]), red)
        rep = sim["report"]
        C = rec["chunk_length"]
        assert cnt["gather_ops"] == rep["gather_ops"]
        assert cnt["gather_ops"] * 2 * C == rep["gather_bytes"]
        assert cnt["reduce_ops"] * 2 * C == rep["reduce_bytes"]
        assert cnt["replaced_ops"] * 2 * C == rep["replaced_bytes"]
        assert cnt["c2g_units"] * 2 * C == rep["c2g_bytes"]
        assert cnt["g2c_units"] * 2 * C == rep["g2c_bytes"]
        assert cnt["peak"] == rep["peak_rcache_blocks"]


@pytest.mark.parametrize("name", ["gpt2-small", "gpt2-1.3b", "gpt2-4b", "gpt2-10b"])
def test_gpt2_layouts_match_golden(golden_layouts, name):
    g = golden_layouts["gpt2"][name]
    params, ops = L.gpt2_records(g["hidden"], g["layers"], 50257, 1024)
    shared, single = L.partition(params, ops)
    assert shared == g["shared_elements"]
    assert [[p, n] for p, n in single] == g["sequence"]
    coarse = L.coarsen(params, ops)
    assert [sorted(s) for s in coarse] == g["coarse"]
    for rec in g["layouts"]:
        out = _check_layout(single, rec)
        if out is None:
            continue
        _, where = out
        fwd, bwd, red = L.chunk_trace(coarse, where)
        assert [sorted(s) for s in fwd] == rec["forward"]
        assert bwd == fwd[::-1]
        assert {str(k): v for k, v in sorted(red.items())} == rec["reduce_after"]
        assert max(len(s) for s in fwd) == rec["working_set"]
        _check_sims(fwd, red, rec)


def test_random_chains_match_golden(golden_layouts):
    recs = golden_layouts["random"]
    assert len(recs) > 100
    for rec in recs:
        params = [tuple(p) for p in rec["params"]]
        ops = [(o[0], o[1], o[2]) for o in rec["ops"]]
        shared, single = L.partition(params, ops)
        assert shared == rec["shared_elements"]
        assert [[p, n] for p, n in single] == rec["sequence"]
        out = _check_layout(single, rec)
        if out is None:
            continue
        _, where = out
        fwd, _, red = L.chunk_trace(L.coarsen(params, ops), where)
        assert [sorted(s) for s in fwd] == rec["forward"]
        _check_sims(fwd, red, rec)


def test_memory_contracts_match_golden(golden_layouts):
    for C, n, want in golden_layouts["chunk_footprint"]:
        assert L.chunk_footprint(C, n) == want
    for S, n, want in golden_layouts["shared_state_bytes"]:
        assert L.shared_state_bytes(S, n) == want


# ---- the reference's own known answers (pkg/tests/test_chunking.py, test_rcache_sim.py)

def test_pack_greedy_known_answer():
    # test_chunking.py:77-83
    chunks, where = L.pack([("p0", 5), ("p1", 3), ("p2", 4)], 8)
    assert [[n for _, _, n in c] for c in chunks] == [[5, 3], [4]]
    assert [o for _, o, _ in chunks[0]] == [0, 5]
    assert where == {"p0": 0, "p1": 0, "p2": 1}


def test_pack_too_small_known_answer():
    # test_chunking.py:86-88
    with pytest.raises(L.OracleError, match="p0"):
        L.pack([("p0", 5), ("p1", 3), ("p2", 4)], 4)


def test_waste_known_answers():
    # test_chunking.py:91-94
    ch, _ = L.pack([("a", 5), ("b", 3), ("c", 4)], 8)
    assert L.waste(ch, 8, 12) == pytest.approx(0.25)
    ch, _ = L.pack([("a", 4), ("b", 4)], 8)
    assert L.waste(ch, 8, 8) == 0.0
    assert L.waste([], 8, 0) == 0.0


def test_trace_reversal_known_answer():
    # test_chunking.py:147-162
    fwd, bwd, red = L.chunk_trace([{"a"}, {"b"}, {"c", "d"}], {"a": 0, "c": 0, "b": 1, "d": 1})
    assert fwd == [frozenset({0}), frozenset({1}), frozenset({0, 1})]
    assert bwd == [frozenset({0, 1}), frozenset({1}), frozenset({0})]
    assert red == {0: 2, 1: 1}


def _run_trace(runs):
    return [frozenset({c}) for c, k in enumerate(runs) for _ in range(k)]


def test_all_blocks_resident_known_answer():
    # test_rcache_sim.py:51-61: 4 chunks, n_block 4 -> 4 gathers, no replacement
    cnt, _ = L.simulate(_run_trace([1, 2, 1, 1]), 4, set())
    assert cnt["gather_ops"] == 4 and cnt["replaced_ops"] == 0 and cnt["reduce_ops"] == 4
    assert cnt["peak"] == 4


def test_pinning_infeasible_known_answer():
    # test_rcache_sim.py:162-172
    fwd = [frozenset({0}), frozenset({1}), frozenset({0})]
    with pytest.raises(L.OracleError, match="pinned"):
        L.simulate(fwd, 1, set(), {0: 2, 1: 1})
    cnt, _ = L.simulate(fwd, 2, set(), {0: 2, 1: 1})
    assert cnt["reduce_ops"] == 2


def test_cpu_home_charges_known_answer():
    # test_rcache_sim.py:204-222: one CPU-home chunk -> one c2g and one g2c unit
    cnt, _ = L.simulate(_run_trace([1]), 1, {0})
    assert cnt["c2g_units"] == 1 and cnt["g2c_units"] == 1


def test_belady_matches_exhaustive_oracle_on_random_runs():
    # test_rcache_sim.py:106-115: farthest-next-use equals the minimum-miss oracle
    rng = random.Random(20240601)
    for _ in range(100):
        runs, total = [], 0
        for _ in range(rng.randint(1, 8)):
            if total >= 8:
                break
            k = rng.randint(1, min(3, 8 - total))
            runs.append(k)
            total += k
        fwd = _run_trace(runs)
        walk = [c for s in fwd + fwd[::-1] for c in sorted(s)]
        for nb in range(1, len(set(walk)) + 2):
            cnt, _ = L.simulate(fwd, nb, set())
            assert cnt["gather_ops"] == _min_misses(walk, nb)


def _min_misses(seq, n_block):
    states = {frozenset(): 0}
    for item in seq:
        nxt = {}
        for st, miss in states.items():
            if item in st:
                cands = [(st, miss)]
            elif len(st) < n_block:
                cands = [(st | {item}, miss + 1)]
            else:
                cands = [((st - {v}) | {item}, miss + 1) for v in st]
            for s2, m2 in cands:
                if m2 < nxt.get(s2, 1 << 30):
                    nxt[s2] = m2
        states = nxt
    return min(states.values())


@pytest.mark.ref
def test_oracle_vs_live_reference_random(offplan):
    ref = offplan
    rng = random.Random(99)
    for _ in range(200):
        n = rng.randint(1, 14)
        seq = [(f"p{i}", rng.randint(1, 50)) for i in range(n)]
        C = max(x for _, x in seq) + rng.randint(0, 30)
        chunks, where = L.pack(seq, C)
        lay = ref.pack_chunks(tuple(ref.ParameterSpec(p, x) for p, x in seq), C)
        assert [[(m.param_id, m.offset, m.numel) for m in c.members] for c in lay.chunks] == \
            [[tuple(t) for t in c] for c in chunks]
        nodes, pos = [], 0
        while pos < n:
            k = rng.randint(1, 3)
            nodes.append({p for p, _ in seq[pos:pos + k]})
            pos += k
        fwd, _, red = L.chunk_trace(nodes, where)
        tr = ref.build_chunk_trace(ref.AccessTrace(tuple(frozenset(x) for x in nodes)), lay)
        ws = max(len(s) for s in fwd)
        for nb in range(ws, lay.n_chunks + 1):
            homes = {c: rng.choice([ref.Device.GPU, ref.Device.CPU]) for c in tr.chunk_ids}
            try:
                rep = ref.simulate(ref.CachePolicyInput(tr, nb, C, homes, ref.PrecisionSpec(), 2))
            except ref.InfeasibleCacheError:
                with pytest.raises(L.OracleError):
                    L.simulate(fwd, nb, {c for c, d in homes.items() if d is ref.Device.CPU}, red)
                continue
            cnt, _ = L.simulate(fwd, nb, {c for c, d in homes.items() if d is ref.Device.CPU}, red)
            assert cnt["gather_ops"] == rep.gather_ops
            assert cnt["replaced_ops"] * 2 * C == rep.replaced_bytes
            assert cnt["c2g_units"] * 2 * C == rep.c2g_bytes and cnt["g2c_units"] * 2 * C == rep.g2c_bytes
            assert cnt["peak"] == rep.peak_rcache_blocks
