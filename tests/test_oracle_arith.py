"""The arithmetic oracle (oracle/arith.py) pinned against torch (committed
golden trajectories of torch.optim.AdamW single-tensor + unscale + clip), the
plain-C oracle cross-checked against it, and the product's HOST Adam
(elx_cpu_adam, for CPU-home shards) checked bit-exact against it."""

from __future__ import annotations

import ctypes
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import arith

ROOT = Path(__file__).resolve().parents[1]


def _meta(g):
    return json.loads(str(g["meta"]))


def test_bf16_rounding_matches_torch():
    import torch
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100_000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 100_000),
                        np.array([0.0, -0.0, np.inf, -np.inf, 3.3895314e38, 1e-40, -1e-42], np.float32)])
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(arith.f32_to_bf16_bits(x), want)
    back = arith.bf16_bits_to_f32(want)
    assert np.array_equal(back, torch.from_numpy(want.view(np.int16)).view(torch.bfloat16).float().numpy())


def test_adamw_trajectory_matches_torch(adamw_golden):
    g = adamw_golden
    meta = _meta(g)
    sizes, world, steps = meta["sizes"], meta["world"], meta["steps"]
    hp = dict(lr=meta["lr"], beta1=meta["betas"][0], beta2=meta["betas"][1], eps=meta["eps"],
              wd=meta["weight_decay"], max_norm=meta["max_norm"])
    shards = [dict(p=g[f"p0_{i}"].astype(np.float32), m=np.zeros(n, np.float32), v=np.zeros(n, np.float32))
              for i, n in enumerate(sizes)]
    t = 0
    for s in range(steps):
        grads = [[g[f"g{s}_{i}_r{r}"] for r in range(world)] for i in range(len(sizes))]
        skip = bool(g[f"skip{s}"])
        t_next = t if skip else t + 1
        out, released, sq, bad = arith.hybrid_step(shards, grads, max(t_next, 1), hp, meta["inv_scale"])
        assert bad == skip
        if not skip:
            assert np.sqrt(sq) == pytest.approx(float(g[f"norm{s}"]), rel=1e-6)
        for i, (p, m, v, _) in enumerate(out):
            want_p = g[f"p{s + 1}_{i}"]
            # ~1 ulp: torch's vectorised lerp is fused (FMA); the oracle is not.
            np.testing.assert_allclose(p, want_p, rtol=1e-6, atol=1e-9)
            if f"m{s + 1}_{i}" in g:
                # moments: 1e-6 relative to the array scale (lerp cancellation
                # makes per-element relative error meaningless near zero)
                wm, wv = g[f"m{s + 1}_{i}"], g[f"v{s + 1}_{i}"]
                np.testing.assert_allclose(m, wm, rtol=1e-6, atol=1e-6 * float(np.abs(wm).max()))
                np.testing.assert_allclose(v, wv, rtol=1e-6, atol=1e-6 * float(np.abs(wv).max()))
            shards[i] = dict(p=p, m=m, v=v)
        t = t_next


def test_release_is_rank_ordered_fp32():
    rng = np.random.default_rng(1)
    srcs = [arith.f32_to_bf16_bits(rng.standard_normal(1001).astype(np.float32)) for _ in range(5)]
    g, sq, bad = arith.release(srcs, 0.25)
    acc = arith.bf16_bits_to_f32(srcs[0])
    for s in srcs[1:]:
        acc = (acc + arith.bf16_bits_to_f32(s)).astype(np.float32)
    assert np.array_equal(g, (acc * np.float32(0.25)).astype(np.float32))
    assert sq == pytest.approx(arith.sumsq(g), rel=1e-12)
    # the quad-fp32 units keep the sum of squares within the 1e-6 bar of the exact fp64 sum
    assert sq == pytest.approx(float(np.sum(g.astype(np.float64) ** 2)), rel=1e-6)
    assert not bad
    srcs[2][7] = 0x7F80  # +inf in bf16
    _, _, bad = arith.release(srcs, 0.25)
    assert bad


def test_clip_coef_convention():
    assert arith.clip_coef(4.0, 1.0) == np.float32(1.0 / (2.0 + 1e-6))
    assert arith.clip_coef(0.25, 1.0) == np.float32(1.0)
    assert arith.clip_coef(4.0, 0.0) == np.float32(1.0)


def _c_oracle():
    lib_path = ROOT / "oracle" / "_build" / "liboracle.so"
    if not lib_path.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=True)
    lib = ctypes.CDLL(str(lib_path))
    lib.oracle_release_bf16.restype = ctypes.c_double
    lib.oracle_release_bf16.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
    lib.oracle_adamw_bf16.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                                             ctypes.c_int, ctypes.c_int]
    return lib


def test_c_oracle_matches_numpy_oracle():
    lib = _c_oracle()
    rng = np.random.default_rng(2)
    n, world = 50_003, 3
    srcs = [arith.f32_to_bf16_bits(rng.standard_normal(n).astype(np.float32)) for _ in range(world)]
    ptrs = (ctypes.c_void_p * world)(*[s.ctypes.data for s in srcs])
    g = np.zeros(n, np.float32)
    bad = ctypes.c_int(0)
    sq = lib.oracle_release_bf16(g.ctypes.data, ptrs, world, n, ctypes.c_float(0.5), ctypes.byref(bad), 4)
    wg, wsq, wbad = arith.release(srcs, 0.5)
    assert np.array_equal(g, wg) and bad.value == int(wbad)
    assert sq == pytest.approx(wsq, rel=1e-12)
    p = (rng.standard_normal(n) * 0.02).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = (rng.random(n) * 1e-6).astype(np.float32)
    k = arith.adam_consts(3, 1e-3, 0.9, 0.999, 1e-8, 0.01)
    kv = np.array([k[x] for x in ("decay", "omb1", "b2", "omb2", "bc2_sqrt", "neg_step", "eps")], np.float32)
    coef = arith.clip_coef(wsq, 1.0)
    P, M, V, P16 = p.copy(), m.copy(), v.copy(), np.zeros(n, np.uint16)
    lib.oracle_adamw_bf16(P.ctypes.data, M.ctypes.data, V.ctypes.data, wg.ctypes.data, P16.ctypes.data, n,
                          kv.ctypes.data, ctypes.c_float(coef), 0, 4)
    rp, rm, rv, r16 = arith.adamw(p, m, v, wg, 3, 1e-3, 0.9, 0.999, 1e-8, 0.01, coef)
    assert np.array_equal(P, rp) and np.array_equal(M, rm) and np.array_equal(V, rv)
    assert np.array_equal(P16, r16)


def _c_oracle_norm():
    import ctypes
    from pathlib import Path
    lib_path = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "liboracle.so"
    if not lib_path.exists():
        pytest.skip("C oracle not built")
    lib = ctypes.CDLL(str(lib_path))
    lib.oracle_release_norm_ordered.restype = ctypes.c_double
    lib.oracle_release_norm_ordered.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int]
    return lib


@pytest.mark.parametrize("ctas,tile_vecs", [(1, 256), (3, 512), (148 * 6, 1024), (2040, 256), (7, 1024)])
def test_release_norm_order_c_equals_numpy(ctas, tile_vecs):
    """The K3 fixed-order sum of squares restated twice (numpy vectorised and
    plain C) gives the same bits on ragged multi-segment inputs."""
    import ctypes
    lib = _c_oracle_norm()
    rng = np.random.default_rng(ctas + tile_vecs)
    gs = [(rng.standard_normal(int(n)) * rng.uniform(0.1, 10)).astype(np.float32)
          for n in rng.integers(1, 200_000, 5)]
    gs.append(np.zeros(0, np.float32))
    want = arith.release_norm_ordered(gs, ctas, tile_vecs)
    ptrs = (ctypes.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    ns = (ctypes.c_int64 * len(gs))(*[g.size for g in gs])
    got = lib.oracle_release_norm_ordered(ptrs, ns, len(gs), ctas, tile_vecs, 4)
    assert got == want
    # and it is the sum of the same quad partials (only the fp64 order differs) ...
    assert want == pytest.approx(sum(arith.sumsq(g) for g in gs), rel=1e-12)
    # ... within the 1e-6 bar of the exact float64 sum of squares
    tot = sum(float(np.dot(g.astype(np.float64), g)) for g in gs)
    assert want == pytest.approx(tot, rel=1e-6)
