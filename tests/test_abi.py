"""The C-ABI library loads and exports every symbol include/elixir_b200.h
declares; host-side entry points (no GPU needed) behave per the header."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import arith
from paper_2212_05339_b200 import _lib, errors, kernels

HEADER = Path(__file__).resolve().parents[1] / "include" / "elixir_b200.h"


def _declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(elx_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)


def test_struct_layouts_match_header():
    lib = _lib.load()
    for i, st in enumerate((_lib.Event, _lib.SimCounters, _lib.Member, _lib.AdamSeg, _lib.AdamHP, _lib.CpuSeg)):
        assert lib.elx_sizeof(i) == ctypes.sizeof(st), st.__name__
    assert lib.elx_sizeof(99) == -1


def test_abi_version_and_errors():
    lib = _lib.load()
    assert lib.elx_abi_version() == 1
    rc = lib.elx_layout_pack(None, 0, 0, None, None, None)
    assert rc == _lib.ERR_VALIDATION
    assert b"chunk_length" in lib.elx_last_error()
    with pytest.raises(errors.ValidationError):
        _lib.check(rc)


def test_gpu_entry_points_validate_before_launch():
    """Argument validation happens on the host; no GPU is touched."""
    lib = _lib.load()
    assert lib.elx_fetch(None, None, 8, 0, _lib.BF16, None) == _lib.ERR_VALIDATION
    assert lib.elx_fetch(None, None, 7, 1, _lib.BF16, None) == _lib.ERR_VALIDATION
    assert lib.elx_fetch_ranked(None, None, 8, 2, 2, _lib.BF16, 0, None) == _lib.ERR_VALIDATION  # rank >= world
    assert lib.elx_fetch_ranked(None, None, 8, 0, 2, _lib.BF16, 7, None) == _lib.ERR_VALIDATION  # bad engine
    assert lib.elx_release(None, None, 8, 1, _lib.BF16, ctypes.c_float(1.0), None, None) == _lib.ERR_VALIDATION
    assert lib.elx_adam(None, 1, 1, None, 1, None, None) == _lib.ERR_VALIDATION
    hp = _lib.AdamHP(1e-3, 0.9, 0.999, 1e-8, 0.0, 0.0, 1.0, _lib.BF16, 0)
    sc = (ctypes.c_double * 2)()
    assert lib.elx_adam(None, 1, 1, ctypes.byref(hp), 0, ctypes.addressof(sc), None) == _lib.ERR_VALIDATION


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("skip", [False, True])
def test_host_adam_bit_exact_vs_oracle(dtype, skip):
    """elx_cpu_adam (the CPU-home optimizer of the hybrid Adam) == oracle, bit for bit."""
    rng = np.random.default_rng(3)
    sizes = [1, 7, 4096, 100_003]
    segs, refs = [], []
    sq = 0.0
    for n in sizes:
        p = (rng.standard_normal(n) * 0.02).astype(np.float32)
        m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        v = (rng.random(n) * 1e-6).astype(np.float32)
        g = (rng.standard_normal(n) * 0.3).astype(np.float32)
        sq += float(np.dot(g.astype(np.float64), g))
        T = [torch.from_numpy(a.copy()) for a in (p, m, v, g)]
        p16 = torch.zeros(n, dtype=dtype)
        segs.append((T[0], T[1], T[2], T[3], p16, n))
        refs.append((p, m, v, g))
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)
    kernels.cpu_adam(segs, hp, 4, (sq, 1.0 if skip else 0.0), dtype, threads=4)
    coef = arith.clip_coef(sq, 1.0)
    name = "bf16" if dtype == torch.bfloat16 else "f16"
    for (P, M, V, G, P16, n), (p, m, v, g) in zip(segs, refs):
        rp, rm, rv, r16 = arith.adamw(p, m, v, g, 4, 1e-3, 0.9, 0.999, 1e-8, 0.01, coef, skip, name)
        assert np.array_equal(P.numpy(), rp)
        assert np.array_equal(M.numpy(), rm)
        assert np.array_equal(V.numpy(), rv)
        assert np.array_equal(P16.view(torch.int16).numpy().view(np.uint16), r16)


def test_host_f16_rounding_edge_cases():
    """elx_cpu_adam's float->half conversion equals numpy's (IEEE RNE), incl.
    subnormals and overflow (exercised through the skip path, which only
    converts the master)."""
    vals = np.array([0.0, -0.0, 1.0, 65504.0, 65519.0, 65520.0, 1e6, -1e6, 6.1e-5, 6.0e-8, 5.96e-8, 2.98e-8,
                     2.9e-8, 1e-10, 3.0e-5, -4.5e-6, np.inf, -np.inf], np.float32)
    n = vals.size
    P = torch.from_numpy(vals.copy())
    z = torch.zeros(n)
    p16 = torch.zeros(n, dtype=torch.float16)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, max_norm=0.0)
    kernels.cpu_adam([(P, z.clone(), z.clone(), z.clone(), p16, n)], hp, 1, (0.0, 1.0), torch.float16, 1)
    assert np.array_equal(p16.numpy().view(np.uint16), vals.astype(np.float16).view(np.uint16))


def test_host_adam_compute_dtype_grads():
    """elx_cpu_adam reading a bf16 gradient (world-1 CPU-home path) == released fp32 path."""
    rng = np.random.default_rng(8)
    n = 70_001
    p = (rng.standard_normal(n) * 0.02).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = (rng.random(n) * 1e-6).astype(np.float32)
    gbits = arith.f32_to_bf16_bits((rng.standard_normal(n) * 10).astype(np.float32))
    g, sq, _ = arith.release([gbits], 1.0 / 64)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)
    T = [torch.from_numpy(a.copy()) for a in (p, m, v)]
    g16 = torch.from_numpy(gbits.view(np.int16).copy()).view(torch.bfloat16)
    p16 = torch.zeros(n, dtype=torch.bfloat16)
    kernels.cpu_adam([(T[0], T[1], T[2], g16, p16, n)], hp, 3, (sq, 0.0), torch.bfloat16, 4, grad_scale=1.0 / 64)
    rp, rm, rv, r16 = arith.adamw(p, m, v, g, 3, 1e-3, 0.9, 0.999, 1e-8, 0.01, arith.clip_coef(sq, 1.0))
    assert np.array_equal(T[0].numpy(), rp) and np.array_equal(T[1].numpy(), rm) and np.array_equal(T[2].numpy(), rv)
    assert np.array_equal(p16.view(torch.int16).numpy().view(np.uint16), r16)


def test_missing_extension_fails_loudly(tmp_path):
    """No CPU fallback: without libelixir_b200.so every hot-path entry raises."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "from paper_2212_05339_b200 import errors, layout, profiles\n"
        "try:\n"
        "    layout.pack_chunks((profiles.ParameterSpec('a', 4),), 8)\n"
        "except errors.ExtensionMissingError as e:\n"
        "    print('raised', e)\n"
    ) % str(HEADER.parents[1])
    env = {"ELX_LIB": str(tmp_path / "missing.so"), "PATH": "/usr/bin:/bin"}
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=120)
    assert "raised" in out.stdout, out.stderr


def test_device_step_bias_tables_equal_oracle_constants():
    """K4's device-step tables hold exactly the oracle's per-step constants
    (float64 bias corrections; the same float32 casts)."""
    for b1, b2, lr in ((0.9, 0.999, 1e-3), (0.8, 0.95, 3e-4)):
        tab = kernels.BiasTables(b1, b2, "cpu", length=20_001)
        bc1, bc2s = tab.bc1.numpy(), tab.bc2s.numpy()
        for t in list(range(1, 300)) + list(range(300, 20_001, 97)):
            k = arith.adam_consts(t, lr, b1, b2, 1e-8, 0.0)
            assert np.float32(-(lr / bc1[t])) == k["neg_step"], t
            assert bc2s[t] == k["bc2_sqrt"], t
        tab.ensure(50_000)
        assert tab.bc1.numel() >= 50_002


def test_lt_algorithm_table_well_formed():
    """plans/lt_algos_b200.json (scripts/tune_lt.py): one entry per GEMM key
    of the step, heuristic-candidate indices in range, loaded by kernels."""
    import json
    from pathlib import Path
    from paper_2212_05339_b200 import kernels
    d = json.loads((Path(__file__).resolve().parents[1] / "plans" / "lt_algos_b200.json").read_text())
    keys = [tuple(c["key"]) for c in d["choices"]]
    assert len(keys) == len(set(keys)) > 0
    for c in d["choices"]:
        assert len(c["key"]) == 12 and all(isinstance(v, int) for v in c["key"])
        assert 0 <= c["index"] < 16 and str(c["index"]) in c["ms"]
    table = kernels._lt_table()
    assert all(table[k] == c["index"] for k, c in zip(keys, d["choices"]))
