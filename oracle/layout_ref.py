"""Pure-Python restatement of the reference's layout / trace / schedule path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Each function follows the
cited reference code statement by statement, in plain loops, so it can be
read side by side with it; it is the checker for the native packer and
schedule compiler (csrc/elx_schedule.cpp) on the GPU box, where the
reference package is not available.
"""

from __future__ import annotations

import math
from collections import deque


class OracleError(Exception):
    """kind in {"validation", "chunk_too_small", "infeasible_cache"}."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ---------------------------------------------------------------- profiles


def gpt2_records(hidden, layers, vocab, seq_len):
    """(params, ops) of offplan.synthesize_transformer_profile
    (profiles.py:438-470). params: [(id, numel, shared)], ops:
    [(name, [param ids], ac_group)]."""
    h = hidden
    params = [("wte", vocab * h, True), ("wpe", seq_len * h, False)]
    ops = [("embed", ["wte", "wpe"], None)]
    for i in range(layers):
        spec = [
            ("ln_1", [("ln_1.w", h), ("ln_1.b", h)]),
            ("attn.qkv", [("attn.qkv.w", 3 * h * h), ("attn.qkv.b", 3 * h)]),
            ("attn.proj", [("attn.proj.w", h * h), ("attn.proj.b", h)]),
            ("ln_2", [("ln_2.w", h), ("ln_2.b", h)]),
            ("mlp.fc", [("mlp.fc.w", 4 * h * h), ("mlp.fc.b", 4 * h)]),
            ("mlp.proj", [("mlp.proj.w", 4 * h * h), ("mlp.proj.b", h)]),
        ]
        for opname, tensors in spec:
            ids = []
            for suffix, n in tensors:
                params.append((f"h{i}.{suffix}", n, False))
                ids.append(f"h{i}.{suffix}")
            ops.append((f"h{i}.{opname}", ids, i))
    params += [("ln_f.w", h, False), ("ln_f.b", h, False)]
    ops += [("ln_f", ["ln_f.w", "ln_f.b"], None), ("lm_head", ["wte"], None)]
    return params, ops


def coarsen(params, ops):
    """profiles.py:490-521: merge AC groups, strip shared ids."""
    shared = {pid for pid, _, s in params if s}
    nodes = []
    group_index = {}
    for _, pids, group in ops:
        if group is None:
            nodes.append(set(pids))
            continue
        if group not in group_index:
            group_index[group] = len(nodes)
            nodes.append(set())
        nodes[group_index[group]].update(pids)
    owner = {}
    out = []
    for idx, node in enumerate(nodes):
        kept = node - shared
        for pid in sorted(kept):
            if pid in owner:
                raise OracleError("validation", f"parameter '{pid}' in two coarse nodes")
            owner[pid] = idx
        out.append(frozenset(kept))
    return out


def partition(params, ops):
    """chunking.py:82-99: shared element count; single-use params ordered by
    (first-use op, declaration index)."""
    first_use = {}
    for idx, (_, pids, _) in enumerate(ops):
        for pid in pids:
            first_use.setdefault(pid, idx)
    shared = sum(n for _, n, s in params if s)
    decl = {pid: i for i, (pid, _, _) in enumerate(params)}
    single = [(pid, n) for pid, n, s in params if not s]
    single.sort(key=lambda pn: (first_use[pn[0]], decl[pn[0]]))
    return shared, single


# ---------------------------------------------------------------- chunking


def pack(sequence, chunk_length):
    """chunking.py:102-138. sequence: [(id, numel)]. Returns
    (chunks = [[(id, offset, numel)]], param_to_chunk)."""
    if chunk_length < 1:
        raise OracleError("validation", "chunk_length must be >= 1")
    for pid, n in sequence:
        if n > chunk_length:
            raise OracleError("chunk_too_small",
                              f"chunk_length {chunk_length} cannot hold parameter '{pid}' with numel {n}")
    chunks, members, offset = [], [], 0
    where = {}
    for pid, n in sequence:
        if offset + n > chunk_length:
            if members:
                chunks.append(members)
            members, offset = [], 0
        where[pid] = len(chunks)
        members.append((pid, offset, n))
        offset += n
    if members:
        chunks.append(members)
    return chunks, where


def waste(chunks, chunk_length, total):
    """chunking.py:141-146."""
    agg = len(chunks) * chunk_length
    return 0.0 if agg == 0 else (agg - total) / agg


def chunk_trace(coarse_nodes, where):
    """chunking.py:149-170: (forward, backward, reduce_after)."""
    forward = []
    for node in coarse_nodes:
        ids = set()
        for pid in node:
            if pid not in where:
                raise OracleError("validation", f"parameter '{pid}' not mapped to any chunk")
            ids.add(where[pid])
        forward.append(frozenset(ids))
    backward = list(reversed(forward))
    reduce_after = {}
    for pos, ids in enumerate(backward):
        for cid in ids:
            reduce_after[cid] = pos
    return forward, backward, reduce_after


# ---------------------------------------------------------------- simulate


def simulate(forward, n_block, cpu_home, reduce_after=None):
    """rcache_sim.py:87-199 (unit counters). cpu_home: set of CPU-homed ids.
    Returns dict(gather_ops, replaced_ops, reduce_ops, c2g_units, g2c_units,
    peak) and the event list [(kind, pos, chunk, victim)]."""
    if n_block < 1:
        raise OracleError("validation", "n_block must be >= 1")
    backward = list(reversed(forward))
    if reduce_after is None:
        reduce_after = {}
        for pos, ids in enumerate(backward):
            for cid in ids:
                reduce_after[cid] = pos
    chunk_ids = set(reduce_after)
    working = max((len(ids) for ids in forward), default=0)
    if n_block < working:
        raise OracleError("infeasible_cache", f"n_block={n_block} below working set {working}")
    walk = list(forward) + backward
    nf = len(forward)
    occ = {c: deque() for c in chunk_ids}
    for pos, ids in enumerate(walk):
        for c in ids:
            occ[c].append(pos)
    resident, pinned, seen = set(), set(), set()
    cnt = dict(gather_ops=0, replaced_ops=0, reduce_ops=0, c2g_units=0, g2c_units=0, peak=0)
    events = []

    def next_use(c):
        return occ[c][0] if occ[c] else math.inf

    for pos, needed in enumerate(walk):
        bpos = pos - nf
        for c in needed:
            occ[c].popleft()
        for c in sorted(needed):
            if c in resident:
                continue
            victim = -1
            if len(resident) >= n_block:
                cands = [r for r in resident if r not in needed and r not in pinned]
                if not cands:
                    raise OracleError("infeasible_cache", f"pinned chunks fill all {n_block} blocks at {bpos}")
                victim = max(cands, key=lambda r: (next_use(r), -r))
                resident.discard(victim)
            resident.add(c)
            cnt["gather_ops"] += 1
            if c in seen:
                cnt["replaced_ops"] += 1
            seen.add(c)
            if c in cpu_home:
                cnt["c2g_units"] += 1
            events.append(("gather", pos, c, victim))
        cnt["peak"] = max(cnt["peak"], len(resident))
        if pos >= nf:
            pinned |= needed
            for c in sorted(needed):  # reference iterates the set; order within a position is immaterial
                if reduce_after[c] == bpos:
                    cnt["reduce_ops"] += 1
                    if c in cpu_home:
                        cnt["g2c_units"] += 1
                    pinned.discard(c)
                    events.append(("reduce", pos, c, -1))
    return cnt, events


# ---------------------------------------------------------------- memory


def chunk_footprint(chunk_length, gpus, compute_bytes=2, optimizer_state_bytes=12):
    """cost_model.py:147-153: ceil((Lc*C + Los*Fos*C) / N)."""
    return -(-(compute_bytes * chunk_length + optimizer_state_bytes * chunk_length) // gpus)


def mixed_precision_states(model_elements, compute_bytes=2, optimizer_state_bytes=12):
    """cost_model.py:156-167: (Lc*M, Lc*M, Los*Fos*M)."""
    return (compute_bytes * model_elements, compute_bytes * model_elements, optimizer_state_bytes * model_elements)


def shared_state_bytes(shared_elements, gpus, compute_bytes=2, optimizer_state_bytes=12):
    """search.py:116-126."""
    if shared_elements <= 0:
        return 0
    return compute_bytes * shared_elements + -(-((compute_bytes + optimizer_state_bytes) * shared_elements) // gpus)
