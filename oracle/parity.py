"""Whole-step arithmetic parity of a live trainer against the C oracle — TEST
INFRASTRUCTURE ONLY (the checker; bench.py's `parity` field and
tests/test_fullsize_gpu.py call it after their timed regions).

`check_step(model, tokens, targets)` runs ONE eager training step of an
ElixirGPT2 at world 1 — every BASELINE.json configuration that fits one GPU:
all chunks GPU-home (configs[0]/[1]) or partly CPU-home (configs[2]/[3],
updated on host threads or streamed through HBM) — with two observation hooks
and no change to what executes:
  * every K3 launch the step issues is logged in issue order, and the
    gradient segments it reads are copied on the launch's own stream right
    before it (the runtime calls `kernels.release_batch` / `kernels.release`;
    the wrapper forwards the call unchanged). A CPU-home chunk's gradient sits
    in an rCache block that a later gather may reuse, so it is captured there;
  * right before HybridAdam's update the update's other inputs are copied to
    host memory: the fp32 master / m / v of the GPU-home segments (device)
    and of the CPU-home chunks (pinned host), in update order up to
    `host_budget` bytes (the 10B configuration is checked on its first
    segments; the sum of squares always covers every element).
The oracle then recomputes, from those copies, (a) the sum of squares launch
by launch in each launch's fixed order (elx_release_geometry;
oracle/c/elx_oracle.c oracle_release_norm_bf16_ordered), added in issue order
as the kernels add them to step_scalars[0], and (b) AdamW with that norm's clip
coefficient over every checked element (oracle_adamw_bf16), and compares with
what the step produced: the sum of squares' bits, and per array the share of
bit-identical elements and the max relative error.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np
import torch

from . import arith

LIB = Path(__file__).resolve().parent / "_build" / "liboracle.so"


def _lib():
    lib = ctypes.CDLL(str(LIB))
    lib.oracle_release_norm_bf16_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_bf16_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_float,
                                                     ctypes.c_int, ctypes.c_int, ctypes.c_int]
    lib.oracle_adamw_bf16.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                                             ctypes.c_int, ctypes.c_int]
    return lib


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _compare(got: torch.Tensor, want: np.ndarray, bf16: bool = False) -> tuple[int, float]:
    """(bit-identical elements, max relative error) of an array (device or
    host) vs the oracle's, compared where `got` lives."""
    w = torch.from_numpy(want.view(np.int16) if bf16 else want).to(got.device)
    if bf16:
        same = int((got.view(torch.int16) == w).sum())
        a, b = got.float(), w.view(torch.bfloat16).float()
    else:
        same = int((got.view(torch.int32) == w.view(torch.int32)).sum())
        a, b = got, w
    den = b.abs().clamp_min(torch.finfo(torch.float32).tiny)
    rel = float(((a - b).abs() / den).max()) if a.numel() else 0.0
    return same, rel


def check_step(model, tokens: torch.Tensor, targets: torch.Tensor, threads: int | None = None,
               host_budget: float = 48e9, device_budget: float = 24e9) -> dict:
    from paper_2212_05339_b200 import kernels

    mgr, opt = model.manager, model.optimizer
    if mgr.world != 1:
        return {"checked": False, "reason": "the whole-step check runs at world 1 (the multi-rank parity tests "
                                            "cover N > 1)"}
    total = sum(mgr.valid(c) for c in range(mgr.n_chunks)) + sum(sp.numel for sp in mgr.shared.values())
    if 2 * total > device_budget:
        return {"checked": False, "reason": f"{2 * total / 1e9:.1f} GB of gradient copies exceed the "
                                            f"{device_budget / 1e9:.0f} GB device budget"}
    threads = threads or max(1, len(os.sched_getaffinity(0)))
    dev = mgr.device
    # every updated segment: GPU-home (the K4 table's order), then CPU-home chunks in forward order; the
    # Adam check covers them in that order up to `host_budget` bytes of host copies (12 B per element)
    host_all = sorted({**opt.cpu_segs, **opt.stream_segs}.items())
    updated = list(opt.gpu_segments) + host_all
    checked, budget = [], host_budget
    for key, seg in updated:
        if 12 * seg[5] > budget:
            break
        checked.append((key, seg))
        budget -= 12 * seg[5]
    launches: list = []
    grads: dict = {}
    snap: dict = {}
    real_batch, real_one, real_step = kernels.release_batch, kernels.release, opt.step

    def resolve():
        m = {st.data_ptr(): (c, st) for c, st in mgr._bound.items()}
        m.update({sp.grad.data_ptr(): (pid, sp.grad) for pid, sp in mgr.shared.items()})
        return m

    def log_batch(ss, dtype, inv_scale, step_scalars, stream=None):
        if step_scalars is mgr.step_scalars:
            where = resolve()
            grp = []
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream(dev)):
                for _, ptrs, n in ss:
                    if n <= 0:
                        continue
                    key, src = where[ptrs[0]]
                    grads[key] = src[:n].clone()   # on the release's stream: after the gradient, before reuse
                    grp.append((key, n))
            launches.append((grp, float(inv_scale)))
        return real_batch(ss, dtype, inv_scale, step_scalars, stream=stream)

    def log_one(g, ptrs, n, dtype, inv_scale, step_scalars, stream=None):
        return log_batch([(g, ptrs, n)], dtype, inv_scale, step_scalars, stream=stream)

    def snapshot_then_step(releases_done=None, grad_scale=1.0):
        cur = torch.cuda.current_stream(dev)
        if releases_done is not None:
            cur.wait_event(releases_done)
        for key, (p32, m, v, _, _, n) in checked:   # to host memory (K4 and the host update come after)
            snap[key] = tuple(t[:n].cpu() if t.is_cuda else t[:n].clone() for t in (p32, m, v))
        snap["__grad_scale__"] = float(grad_scale)
        return real_step(releases_done, grad_scale)

    model.synchronize()
    torch.cuda.synchronize(dev)
    completed = int(mgr.step_scalars[2].item())
    kernels.release_batch, kernels.release, opt.step = log_batch, log_one, snapshot_then_step
    try:
        model.train_step(tokens, targets)
    finally:
        kernels.release_batch, kernels.release = real_batch, real_one
        del opt.step                           # the bound method again
    model.synchronize()
    stats = opt.last_stats
    sq_gpu, flag = stats.scalars()
    torch.cuda.synchronize(dev)

    lib = _lib()
    released = sorted(str(k) for grp, _ in launches for k, _ in grp)
    want_keys = sorted(str(k) for k, _ in updated)
    assert released == want_keys, "every updated segment is released exactly once"
    gbits = {key: _bits(t) for key, t in grads.items()}
    grads.clear()
    sq = 0.0
    for grp, inv_scale in launches:
        ns = [n for _, n in grp]
        ctas, tv = kernels.release_geometry(ns, 1)
        ptrs = (ctypes.c_void_p * len(grp))(*[gbits[k].ctypes.data for k, _ in grp])
        nn = (ctypes.c_int64 * len(grp))(*ns)
        sq = sq + lib.oracle_release_norm_bf16_ordered(ptrs, nn, len(grp), ctypes.c_float(inv_scale), ctas, tv,
                                                      threads)

    hp = opt.hp
    skip = bool(flag) or not np.isfinite(sq)
    step = completed + (0 if skip else 1)
    coef = arith.clip_coef(sq, hp["max_norm"])
    k = arith.adam_consts(max(step, 1), hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"])
    kv = np.array([k["decay"], k["omb1"], k["b2"], k["omb2"], k["bc2_sqrt"], k["neg_step"], k["eps"]], np.float32)
    gs = np.float32(snap["__grad_scale__"])
    totals = {name: [0, 0.0] for name in ("p32", "m", "v", "p16")}
    elements = 0
    for key, (p32, m, v, _, p16, n) in checked:
        P, M, V = (t.numpy() for t in snap.pop(key))
        G = arith.bf16_bits_to_f32(gbits[key])
        if gs != np.float32(1.0):
            G = (G * gs).astype(np.float32)
        out16 = np.empty(n, np.uint16)
        lib.oracle_adamw_bf16(P.ctypes.data, M.ctypes.data, V.ctypes.data, G.ctypes.data, out16.ctypes.data, n,
                              kv.ctypes.data, ctypes.c_float(coef), int(skip), threads)
        # a resident streamed chunk's new parameters are in its rCache block (HybridAdam.attach_fetcher)
        p16_home = opt.resident[key] if key in getattr(opt, "resident", {}) else p16
        for name, got, want, bf in (("p32", p32[:n], P, False), ("m", m[:n], M, False), ("v", v[:n], V, False),
                                    ("p16", p16_home[:n], out16, True)):
            same, rel = _compare(got, want, bf)
            totals[name][0] += same
            totals[name][1] = max(totals[name][1], rel)
        elements += n
    torch.cuda.empty_cache()
    return {
        "checked": True,
        "elements": elements,
        "model_elements": total,
        "resident_streamed_chunks": len(getattr(opt, "resident", {})),
        "segments_checked": len(checked),
        "segments": len(updated),
        "cpu_home_chunks": len(host_all),
        "cpu_home_chunks_checked": sum(1 for key, _ in checked if key in dict(host_all)),
        "release_launches": len(launches),
        "sumsq_bit_identical": sq_gpu == sq,
        "sumsq_rel_err": abs(sq_gpu - sq) / sq if sq else 0.0,
        "bit_identical_frac": {name: t[0] / elements for name, t in totals.items()},
        "max_rel_err": {name: t[1] for name, t in totals.items()},
        "tolerance": "north_star: 1e-6 relative for fp32 Adam and reduced gradients; bit-exact for bytes",
        "within_tolerance": all(t[1] <= 1e-6 for t in totals.values()) and abs(sq_gpu - sq) <= 1e-6 * abs(sq),
        "oracle": "oracle/c/elx_oracle.c (ordered sum of squares per K3 launch, AdamW), "
                  f"{threads} host threads",
    }


def check_step_multirank(model, tokens: torch.Tensor, targets: torch.Tensor, threads: int | None = None) -> dict:
    """The whole-step check at N > 1 (every rank calls it; the ranks' results
    are merged and every rank gets the same dict). One eager step of the
    trainer, unchanged, observed at the same two points as `check_step`:
      * every K3 launch is logged in issue order and, on its own stream right
        before it (after the release's device barrier on the P2P path; after
        the exchange on the NCCL path), the N bf16 gradient slices it reads —
        segment `rank` of every rank's copy of the chunk, peers' through their
        mapped pointers — are copied to pinned host memory;
      * right before HybridAdam's update, the fp32 master / m / v of every
        GPU-home segment and this rank's local sum of squares (step_scalars[0]
        before the cross-rank reduction) are copied to the host.
    The oracle recomputes per rank (a) the reduced gradient of every segment,
    the rank-ordered fp32 sum times inv_scale (oracle_release_bf16), compared
    bit for bit with the fp32 shard K3 wrote; (b) the rank's sum of squares
    launch by launch in each launch's fixed order; (c) the global sum — the
    ranks' sums added in rank order from 0.0, as the P2P scalar reduction
    reads them (elx_peer_sum_f64; NCCL's all-reduce on the exchange path
    follows its own order, so there the global sum is compared to 1e-12) —
    and (d) AdamW with the resulting clip coefficient over every element of
    the rank's shards. CPU-home chunks are covered too: their K3 writes the
    shared fp32 staging shard (the chunk is identified through the release
    sources the fetcher computed for it), the reduced gradient is compared
    with the host shard it was copied to, and the host-thread or streamed
    update with the host state after the step."""
    import torch.distributed as dist

    from paper_2212_05339_b200 import _lib as elx_lib
    from paper_2212_05339_b200 import kernels

    mgr, opt = model.manager, model.optimizer
    world, rank = mgr.world, mgr.rank
    if world == 1:
        return check_step(model, tokens, targets, threads)
    threads = threads or max(1, len(os.sched_getaffinity(0)) // world)   # the ranks share the host's cores
    dev = mgr.device
    lib_elx = elx_lib.load()
    # GPU-home segments (K4's table order), then CPU-home chunks (host-thread or streamed update)
    host_all = sorted({**opt.cpu_segs, **opt.stream_segs}.items())
    segs = list(opt.gpu_segments) + host_all
    key_of = {seg[3].data_ptr(): key for key, seg in opt.gpu_segments}   # K4's gradient input = K3's output
    host = {key: torch.empty((world, seg[5]), dtype=torch.int16, pin_memory=True) for key, seg in segs}
    launches: list = []
    snap: dict = {}
    real_batch, real_one, real_step = kernels.release_batch, kernels.release, opt.step
    # a CPU-home chunk's K3 writes the shared fp32 staging shard (then D2H to its host gradient shard): the
    # chunk is the one whose release sources the fetcher computed last
    fetcher = model.fetcher
    real_srcs = fetcher._release_srcs
    last_chunk = [None]

    def srcs_noted(c):
        last_chunk[0] = c
        return real_srcs(c)

    def log_batch(ss, dtype, inv_scale, step_scalars, stream=None):
        if step_scalars is mgr.step_scalars:
            st = stream if stream is not None else torch.cuda.current_stream(dev)
            grp = []
            for g, ptrs, n in ss:
                if n <= 0:
                    continue
                key = key_of[g.data_ptr()] if g is not None and g.data_ptr() in key_of else last_chunk[0]
                for r in range(world):
                    rc = lib_elx.elx_copy_d2h(host[key][r].data_ptr(), int(ptrs[r]), 2 * n, st.cuda_stream, None)
                    elx_lib.check(rc, "parity copy of a K3 source")
                grp.append((key, n))
            launches.append((grp, float(inv_scale)))
        return real_batch(ss, dtype, inv_scale, step_scalars, stream=stream)

    def log_one(g, ptrs, n, dtype, inv_scale, step_scalars, stream=None):
        return log_batch([(g, ptrs, n)], dtype, inv_scale, step_scalars, stream=stream)

    def snapshot_then_step(releases_done=None, grad_scale=1.0):
        cur = torch.cuda.current_stream(dev)
        if releases_done is not None:
            cur.wait_event(releases_done)
        snap["__sq_local__"] = float(mgr.step_scalars[0].item())
        snap["__flag_local__"] = float(mgr.step_scalars[1].item())
        for key, (p32, m, v, _, _, n) in segs:   # (the host-home state: no update runs before real_step)
            snap[key] = tuple(t[:n].cpu() if t.is_cuda else t[:n].clone() for t in (p32, m, v))
        return real_step(releases_done, grad_scale)

    model.synchronize()
    torch.cuda.synchronize(dev)
    completed = int(mgr.step_scalars[2].item())
    kernels.release_batch, kernels.release, opt.step = log_batch, log_one, snapshot_then_step
    fetcher._release_srcs = srcs_noted
    try:
        model.train_step(tokens, targets)
    finally:
        kernels.release_batch, kernels.release = real_batch, real_one
        del opt.step
        del fetcher._release_srcs
    model.synchronize()
    sq_gpu, flag = opt.last_stats.scalars()
    torch.cuda.synchronize(dev)

    lib = _lib()
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
    lib.oracle_release_norm_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int]
    released = sorted(str(k) for grp, _ in launches for k, _ in grp)
    assert released == sorted(str(k) for k, _ in segs), "every updated segment is released exactly once"
    gref: dict = {}
    g_same = g_total = 0
    g_rel = 0.0
    sq_local = 0.0
    for grp, inv_scale in launches:
        for key, n in grp:
            src = host[key].numpy().view(np.uint16)
            ptrs = (ctypes.c_void_p * world)(*[src[r].ctypes.data for r in range(world)])
            out = np.empty(n, np.float32)
            bad = ctypes.c_int(0)
            lib.oracle_release_bf16(out.ctypes.data, ptrs, world, n, ctypes.c_float(inv_scale), ctypes.byref(bad),
                                    threads)
            gref[key] = out
            seg = dict(segs)[key]
            same, rel = _compare(seg[3][:n], out)
            g_same += same
            g_total += n
            g_rel = max(g_rel, rel)
        ns = [n for _, n in grp]
        ctas, tv = kernels.release_geometry(ns, world)
        gp = (ctypes.c_void_p * len(grp))(*[gref[k].ctypes.data for k, _ in grp])
        nn = (ctypes.c_int64 * len(grp))(*ns)
        sq_local = sq_local + lib.oracle_release_norm_ordered(gp, nn, len(grp), ctas, tv, threads)
    host.clear()
    everyone = [None] * world
    dist.all_gather_object(everyone, sq_local)
    sq = 0.0
    for s in everyone:
        sq = sq + s
    exact_order = bool(mgr.p2p)
    sq_ok = (sq_gpu == sq) if exact_order else abs(sq_gpu - sq) <= 1e-12 * abs(sq)
    # the exchange path's all-reduce adds in the library's order: once the global sum is within 1e-12, the
    # update is checked with the value the step used (its clip coefficient), so AdamW stays a bit-exact test
    sq_adam = sq if exact_order or not sq_ok else sq_gpu
    hp = opt.hp
    skip = bool(flag) or not np.isfinite(sq_adam)
    step = completed + (0 if skip else 1)
    coef = arith.clip_coef(sq_adam, hp["max_norm"])
    k = arith.adam_consts(max(step, 1), hp["lr"], hp["beta1"], hp["beta2"], hp["eps"], hp["weight_decay"])
    kv = np.array([k["decay"], k["omb1"], k["b2"], k["omb2"], k["bc2_sqrt"], k["neg_step"], k["eps"]], np.float32)
    totals = {name: [0, 0.0] for name in ("p32", "m", "v", "p16")}
    elements = 0
    for key, (p32, m, v, _, p16, n) in segs:
        P, M, V = (t.numpy() for t in snap.pop(key))
        out16 = np.empty(n, np.uint16)
        lib.oracle_adamw_bf16(P.ctypes.data, M.ctypes.data, V.ctypes.data, gref[key].ctypes.data,
                              out16.ctypes.data, n, kv.ctypes.data, ctypes.c_float(coef), int(skip), threads)
        for name, got, want, bf in (("p32", p32[:n], P, False), ("m", m[:n], M, False), ("v", v[:n], V, False),
                                    ("p16", p16[:n], out16, True)):
            same, rel = _compare(got, want, bf)
            totals[name][0] += same
            totals[name][1] = max(totals[name][1], rel)
        elements += n
    mine = {"elements": elements, "g_same": g_same, "g_total": g_total, "g_rel": g_rel, "cpu_home": len(host_all),
            "sq_local_gpu": snap["__sq_local__"], "sq_local_oracle": sq_local,
            "totals": totals, "launches": len(launches)}
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    torch.cuda.empty_cache()
    elements = sum(r["elements"] for r in allr)
    merged = {name: [sum(r["totals"][name][0] for r in allr), max(r["totals"][name][1] for r in allr)]
              for name in totals}
    g_total = sum(r["g_total"] for r in allr)
    return {
        "checked": True,
        "world": world,
        "transport": type(mgr.transport).__name__,
        "elements": elements,
        "cpu_home_chunks_per_rank": [r["cpu_home"] for r in allr],
        "release_launches_per_rank": [r["launches"] for r in allr],
        "reduced_grad_bit_identical_frac": sum(r["g_same"] for r in allr) / max(1, g_total),
        "reduced_grad_max_rel_err": max(r["g_rel"] for r in allr),
        "sumsq_local_bit_identical": all(r["sq_local_gpu"] == r["sq_local_oracle"] for r in allr),
        "sumsq_global_bit_identical" if exact_order else "sumsq_global_within_1e-12": sq_ok,
        "bit_identical_frac": {name: t[0] / elements for name, t in merged.items()},
        "max_rel_err": {name: t[1] for name, t in merged.items()},
        "tolerance": "north_star: 1e-6 relative for fp32 Adam and reduced gradients; bit-exact for bytes",
        "within_tolerance": all(t[1] <= 1e-6 for t in merged.values()) and max(r["g_rel"] for r in allr) <= 1e-6
                            and (sq_ok or abs(sq_gpu - sq) <= 1e-6 * abs(sq)),
        "oracle": "oracle/c/elx_oracle.c (rank-ordered release, ordered sum of squares per K3 launch, AdamW), "
                  f"{threads} host threads per rank",
    }
