"""Parity of the sm_100a kernels (K1-K6), called through the C-ABI, against the
CPU oracle on the same seeded inputs. Integer/byte work is bit-exact; the
fp32 release and Adam are also bit-exact (the kernels apply the oracle's
IEEE operations in the oracle's order), which is stricter than the 1e-6
relative bar of BASELINE.json."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import arith
from paper_2212_05339_b200 import _lib, errors, kernels

pytestmark = pytest.mark.gpu

HP = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def _name(dt):
    return "bf16" if dt == torch.bfloat16 else "f16"


# ------------------------------------------------------------------ K1 pack

@pytest.mark.parametrize("chunk_dtype", [torch.bfloat16, torch.float32, torch.float16])
def test_pack_unpack_members_and_padding(cuda, chunk_dtype):
    g = torch.Generator().manual_seed(0)
    sizes = [5, 3, 4096, 17, 40000, 1, 8]
    offs, o = [], 3  # start at an odd offset: exercises the unaligned path too
    for n in sizes:
        offs.append(o)
        o += n
    used, phys = o, o + 101
    srcs = [torch.randn(n, generator=g).to(torch.bfloat16) for n in sizes]
    chunk = torch.full((phys,), 7.0, dtype=chunk_dtype, device=cuda)
    kernels.chunk_pack(chunk, [(s.to(cuda), off) for s, off in zip(srcs, offs)], used_len=used)
    ref = np.full(phys, 7.0, np.float32)
    for s, off in zip(srcs, offs):
        ref[off:off + s.numel()] = s.float().numpy()
    ref[used:] = 0.0
    want = torch.from_numpy(ref).to(chunk_dtype).float().numpy()  # RNE, as the kernel converts
    assert np.array_equal(chunk.float().cpu().numpy(), want)
    # unpack back into fresh tensors of the source dtype
    outs = [torch.empty(n, dtype=torch.bfloat16, device=cuda) for n in sizes]
    kernels.chunk_unpack(chunk, list(zip(outs, offs)))
    torch.cuda.synchronize()
    for s, t in zip(srcs, outs):
        assert torch.equal(t.cpu(), s.to(chunk_dtype).to(torch.bfloat16))


def test_pack_is_bit_exact_gpt2_layout(cuda):
    """Pack a real layout (GPT-2 tiny) and compare with the oracle's byte image."""
    from oracle import layout_ref as L
    params, ops = L.gpt2_records(64, 3, 128, 16)
    _, seq = L.partition(params, ops)
    C = 4 * 64 * 64 + 999
    chunks, _ = L.pack(seq, C)
    g = torch.Generator().manual_seed(1)
    vals = {pid: torch.randn(n, generator=g).to(torch.bfloat16) for pid, n in seq}
    for ch in chunks:
        phys = C + 5
        buf = torch.empty(phys, dtype=torch.bfloat16, device=cuda)
        kernels.chunk_pack(buf, [(vals[p].to(cuda), off) for p, off, _ in ch], used_len=sum(n for *_, n in ch))
        want = arith.pack(phys, [(_bits(vals[p]), off) for p, off, _ in ch])
        assert np.array_equal(_bits(buf), want)


def test_pack_validation(cuda):
    buf = torch.zeros(10, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(errors.ValidationError):
        kernels.chunk_pack(buf, [(torch.zeros(8, dtype=torch.bfloat16, device=cuda), 5)])


# ------------------------------------------------------------------ K2 fetch

@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("shard", [8, 4096, 16_384, 1_000_008, 3_000_000])
def test_fetch_gathers_shards_in_rank_order(cuda, world, shard):
    g = torch.Generator().manual_seed(world * 7 + shard)
    shards = [torch.randint(-32768, 32767, (shard,), generator=g, dtype=torch.int16).view(torch.bfloat16).to(cuda)
              for _ in range(world)]
    block = torch.zeros(world * shard, dtype=torch.bfloat16, device=cuda)
    kernels.fetch(block, [s.data_ptr() for s in shards], shard)
    want = arith.gather([_bits(s) for s in shards])
    assert np.array_equal(_bits(block), want)


@pytest.mark.parametrize("world", [1, 2, 8])
def test_fetch_copy_engine_equals_kernel(cuda, world):
    """K2 on the copy engines (elx_fetch_ce) gathers the same bytes as the kernel."""
    g = torch.Generator().manual_seed(world)
    shard = 1_000_008
    shards = [torch.randint(-32768, 32767, (shard,), generator=g, dtype=torch.int16).view(torch.bfloat16).to(cuda)
              for _ in range(world)]
    block = torch.zeros(world * shard, dtype=torch.bfloat16, device=cuda)
    kernels.fetch(block, [s.data_ptr() for s in shards], shard, engine="ce")
    torch.cuda.synchronize()
    assert np.array_equal(_bits(block), arith.gather([_bits(s) for s in shards]))
    with pytest.raises(errors.ValidationError):
        kernels.fetch(block, [s.data_ptr() + 2 for s in shards], 8, engine="ce")


_K2K3_VARIANT_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from paper_2212_05339_b200 import kernels
from oracle import arith
dev = torch.device("cuda", 0)
bits = lambda t: t.cpu().view(torch.int16).numpy().view(np.uint16)
for world in (1, 2, 3, 4, 8):
    for n in (8, 4104, 1_000_008, 2_500_000):
        g = torch.Generator().manual_seed(n + world)
        srcs = [(torch.randn(n, generator=g) * 3.0).to(torch.bfloat16) for _ in range(world)]
        dsrc = [s.to(dev) for s in srcs]
        block = torch.zeros(world * n, dtype=torch.bfloat16, device=dev)
        kernels.fetch(block, [t.data_ptr() for t in dsrc], n)
        torch.cuda.synchronize()
        assert np.array_equal(bits(block), arith.gather([bits(s) for s in srcs])), (world, n)
        for scale in (1.0, 1.0 / 64):
            out = torch.full((n,), -1.0, device=dev)
            sc = kernels.new_step_scalars(dev)
            kernels.release(out, [t.data_ptr() for t in dsrc], n, torch.bfloat16, scale, sc)
            torch.cuda.synchronize()
            wg, wsq, wbad = arith.release([bits(s) for s in srcs], scale, "bf16")
            assert np.array_equal(out.cpu().numpy(), wg), (world, n, scale)
            ctas, tv = kernels.release_geometry([n], world)
            assert sc[0].item() == arith.release_norm_ordered([wg], ctas, tv), (world, n, scale, ctas, tv)
print("ok")
"""


@pytest.mark.parametrize("env", [{"ELX_K2_TMA": "-1", "ELX_K3_PEER_TMA": "0"}, {"ELX_K2_TMA": "1", "ELX_K3_TMA": "1"},
                                 {"ELX_K2_TMA": "2"}, {"ELX_K2_TMA": "3"}])
def test_fetch_release_variants_bit_exact(cuda, env):
    """Every K2 shape (register copy, TMA tiles x stages) gathers the oracle's bytes, and K3 at world 1-8 with
    the TMA stages off (register-staged peer loads) or in their other shape equals the oracle: the reduced
    fp32 bits, and the sum of squares in the order elx_release_geometry reports."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    out = subprocess.run([sys.executable, "-c", _K2K3_VARIANT_SCRIPT, root], env=dict(os.environ, **env),
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


@pytest.mark.parametrize("engine", ["sm", "ce"])
@pytest.mark.parametrize("world,rank", [(2, 1), (4, 3), (8, 0), (8, 5), (3, 2)])
def test_fetch_rank_rotation_gathers_the_same_bytes(cuda, engine, world, rank):
    """elx_fetch_ranked: the peer reads start at rank+1 (tiles interleaved over the ranks / copy-engine order
    rotated), the gathered block is the same rank-ordered concatenation."""
    g = torch.Generator().manual_seed(world * 31 + rank)
    shard = 600_008
    shards = [torch.randint(-32768, 32767, (shard,), generator=g, dtype=torch.int16).view(torch.bfloat16).to(cuda)
              for _ in range(world)]
    block = torch.zeros(world * shard, dtype=torch.bfloat16, device=cuda)
    kernels.fetch(block, [s.data_ptr() for s in shards], shard, engine=engine, rank=rank)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(block), arith.gather([_bits(s) for s in shards]))


def test_fetch_rejects_unaligned(cuda):
    block = torch.zeros(64, dtype=torch.bfloat16, device=cuda)
    s = torch.zeros(16, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(errors.ValidationError):
        kernels.fetch(block, [s.data_ptr()], 7)
    with pytest.raises(errors.ValidationError):
        kernels.fetch(block, [s.data_ptr() + 2], 8)


# ------------------------------------------------------------------ K3 release

@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [1, 7, 8, 4103, 1_048_579])
def test_release_bit_exact(cuda, dtype, world, n):
    g = torch.Generator().manual_seed(n + world)
    srcs = [(torch.randn(n, generator=g) * 3.0).to(dtype) for _ in range(world)]
    dsrc = [s.to(cuda) for s in srcs]
    out = torch.full((n,), -1.0, device=cuda)
    sc = kernels.new_step_scalars(cuda)
    kernels.release(out, [t.data_ptr() for t in dsrc], n, dtype, 1.0 / 128, sc)
    torch.cuda.synchronize()
    wg, wsq, wbad = arith.release([_bits(s) for s in srcs], 1.0 / 128, _name(dtype))
    assert np.array_equal(out.cpu().numpy(), wg)
    assert sc[0].item() == pytest.approx(wsq, rel=1e-12)
    # the sum of squares in the kernel's fixed order (no atomics) is bit-exact to the oracle's restatement
    ctas, tv = kernels.release_geometry([n], world, dtype)
    assert sc[0].item() == arith.release_norm_ordered([wg], ctas, tv)
    assert sc[1].item() == 0.0 and not wbad


def test_release_unaligned_sources_use_scalar_path(cuda):
    n, world = 10_001, 3
    g = torch.Generator().manual_seed(5)
    base = [torch.randn(n + 1, generator=g).to(torch.bfloat16).to(cuda) for _ in range(world)]
    out = torch.zeros(n, device=cuda)
    sc = kernels.new_step_scalars(cuda)
    kernels.release(out, [b.data_ptr() + 2 for b in base], n, torch.bfloat16, 1.0, sc)
    wg, wsq, _ = arith.release([_bits(b)[1:] for b in base], 1.0)
    assert np.array_equal(out.cpu().numpy(), wg)
    assert sc[0].item() == pytest.approx(wsq, rel=1e-12)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("inv_scale", [1.0, 1.0 / 65536])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 4103, 1_048_583])
@pytest.mark.parametrize("bad", [None, "inf", "nan", "-inf"])
def test_release_norm_only_world1(cuda, dtype, inv_scale, n, bad):
    """World-1 release with no gradient output (the dedicated norm kernel:
    16-byte loads, scalar tail, flag derived from the fp64 sum): sum of squares
    within 1e-12 of the oracle and the overflow flag exact, including a
    non-finite element in the vector body or the tail."""
    g = torch.Generator().manual_seed(n)
    src = (torch.randn(n, generator=g) * 3.0).to(dtype)
    if bad is not None:
        src[(n * 7) // 11] = float(bad)
    d = src.to(cuda)
    sc = kernels.new_step_scalars(cuda)
    kernels.release(None, [d.data_ptr()], n, dtype, inv_scale, sc)
    torch.cuda.synchronize()
    wg, wsq, wbad = arith.release([_bits(src)], inv_scale, _name(dtype))
    assert sc[1].item() == (1.0 if wbad else 0.0)
    assert wbad == (bad is not None)
    if not wbad:
        assert sc[0].item() == pytest.approx(wsq, rel=1e-12)
        ctas, tv = kernels.release_geometry([n], 1, dtype)
        assert sc[0].item() == arith.release_norm_ordered([wg], ctas, tv)
    # 8-byte aligned but not 16: same answer through the general path
    if n > 8 and bad is None:
        buf = torch.zeros(n + 4, dtype=dtype, device=cuda)
        buf[4:] = d
        sc2 = kernels.new_step_scalars(cuda)
        kernels.release(None, [buf.data_ptr() + 8], n, dtype, inv_scale, sc2)
        torch.cuda.synchronize()
        assert sc2[0].item() == pytest.approx(wsq, rel=1e-12) and sc2[1].item() == 0.0


@pytest.mark.parametrize("where", ["even", "odd", "both", "zeros"])
def test_release_norm_subnormal_and_zero_elements_exact(cuda, where):
    """The world-1 bf16 norm pass (TMA-staged) squares in fp32: a subnormal
    element's square underflows to a subnormal or zero, -0.0 squares to +0.0,
    with IEEE gradual underflow on both sides (no flush-to-zero in the kernel
    or the oracle). The sum stays bit-exact to the oracle's fixed order
    whatever the element classes and positions."""
    n = 3 * 2 ** 20 + 5
    rng = np.random.default_rng(11)
    x = arith.f32_to_bf16_bits((rng.standard_normal(n) * 1e-3).astype(np.float32))
    idx = rng.integers(0, n, 4000)
    if where in ("even", "both"):
        x[idx[idx % 2 == 0]] = rng.integers(1, 0x80, (idx % 2 == 0).sum()).astype(np.uint16)   # subnormals
    if where in ("odd", "both"):
        x[idx[idx % 2 == 1]] = (rng.integers(1, 0x80, (idx % 2 == 1).sum()) | 0x8000).astype(np.uint16)
    if where == "zeros":
        x[: n // 2] = 0
        x[idx] = 0x8000  # -0.0
    d = torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).to(cuda)
    sc = kernels.new_step_scalars(cuda)
    kernels.release(None, [d.data_ptr()], n, torch.bfloat16, 1.0, sc)
    torch.cuda.synchronize()
    wg, _, wbad = arith.release([x], 1.0)
    ctas, tv = kernels.release_geometry([n], 1)
    assert not wbad and sc[1].item() == 0.0
    assert sc[0].item() == arith.release_norm_ordered([wg], ctas, tv)


@pytest.mark.parametrize("world", [1, 2, 4, 8, 3])
def test_release_batch_one_launch_bit_exact(cuda, world):
    """Every chunk due at one reduce position in ONE K3 launch: ragged segment
    lengths (tails of 1..7 elements, an empty one), fp32 outputs or none (the
    world-1 norm pass), 20 segments (two launches of 16 + 4): released values
    bit-exact, the sum of squares bit-exact to the oracle's fixed-order
    restatement per launch, and identical on a second run (deterministic)."""
    rng = np.random.default_rng(world)
    lens = [int(x) for x in rng.integers(1, 300_000, 20)]
    lens[3], lens[7], lens[11] = 0, 5, 8 * 4096 + 3
    srcs, outs, segs, want = [], [], [], []
    for i, n in enumerate(lens):
        hs = [arith.f32_to_bf16_bits((rng.standard_normal(n) * 2).astype(np.float32)) for _ in range(world)]
        ds = [torch.from_numpy(h.view(np.int16).copy()).view(torch.bfloat16).to(cuda) for h in hs]
        srcs.append(ds)
        o = None if (world == 1 and i % 2) else torch.full((max(n, 1),), -1.0, device=cuda)
        outs.append(o)
        segs.append((o, [d.data_ptr() for d in ds], n))
        want.append(arith.release(hs, 0.25)[0])
    sc = kernels.new_step_scalars(cuda)
    kernels.release_batch(segs, torch.bfloat16, 0.25, sc)
    torch.cuda.synchronize()
    nz = [i for i, n in enumerate(lens) if n > 0]
    total = 0.0
    for part in (nz[:16], nz[16:]):
        ctas, tv = kernels.release_geometry([lens[i] for i in part], world)
        total = total + arith.release_norm_ordered([want[i] for i in part], ctas, tv)
    assert sc[0].item() == total
    for o, w, n in zip(outs, want, lens):
        if o is not None and n > 0:
            assert np.array_equal(o[:n].cpu().numpy(), w)
    sc2 = kernels.new_step_scalars(cuda)
    kernels.release_batch(segs, torch.bfloat16, 0.25, sc2)
    torch.cuda.synchronize()
    assert sc2[0].item() == sc[0].item() and sc2[1].item() == 0.0


def test_release_accumulates_norm_and_flags_overflow(cuda):
    n = 50_000
    g = torch.Generator().manual_seed(9)
    a = torch.randn(n, generator=g).to(torch.bfloat16)
    b = torch.randn(n, generator=g).to(torch.bfloat16)
    b[12345] = float("inf")
    sc = kernels.new_step_scalars(cuda)
    out = torch.zeros(n, device=cuda)
    kernels.release(out, [a.to(cuda).data_ptr()], n, torch.bfloat16, 1.0, sc)
    first = sc[0].item()
    bb = b.to(cuda)
    kernels.release(out, [bb.data_ptr()], n, torch.bfloat16, 1.0, sc)
    torch.cuda.synchronize()
    assert sc[1].item() == 1.0
    assert first == pytest.approx(arith.sumsq(a.float().numpy()), rel=1e-12)
    kernels.step_reset(sc)
    torch.cuda.synchronize()
    assert sc[0].item() == 0.0 and sc[1].item() == 0.0


# ------------------------------------------------------------------ K4 Adam

def _segments(cuda, sizes, seed, misalign=False):
    rng = np.random.default_rng(seed)
    host, dev = [], []
    for n in sizes:
        p = (rng.standard_normal(n) * 0.02).astype(np.float32)
        m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        v = (rng.random(n) * 1e-6).astype(np.float32)
        gg = (rng.standard_normal(n) * 0.05).astype(np.float32)
        host.append([p, m, v, gg])
        off = 1 if misalign else 0
        ts = []
        for a in (p, m, v, gg):
            t = torch.zeros(n + off, device=cuda)
            t[off:] = torch.from_numpy(a)
            ts.append(t[off:])
        p16 = torch.zeros(n + off, dtype=torch.bfloat16, device=cuda)[off:]
        dev.append((*ts, p16, n))
    return host, dev


@pytest.mark.parametrize("misalign", [False, True])
def test_adam_bit_exact_multi_segment_multi_step(cuda, misalign):
    sizes = [1, 3, 4096, 4097, 12_288, 1_000_003]
    host, dev = _segments(cuda, sizes, 11, misalign)
    table = kernels.AdamTable(dev, cuda)
    sc = kernels.new_step_scalars(cuda)
    for step in range(1, 4):
        sq = float(sum(np.dot(h[3].astype(np.float64), h[3]) for h in host))
        sc[0] = sq
        sc[1] = 0.0
        kernels.adam(table, HP, step, sc, torch.bfloat16)
        torch.cuda.synchronize()
        coef = arith.clip_coef(sq, HP["max_norm"])
        for h, d in zip(host, dev):
            rp, rm, rv, r16 = arith.adamw(h[0], h[1], h[2], h[3], step, HP["lr"], HP["beta1"], HP["beta2"],
                                          HP["eps"], HP["weight_decay"], coef)
            assert np.array_equal(d[0].cpu().numpy(), rp)
            assert np.array_equal(d[1].cpu().numpy(), rm)
            assert np.array_equal(d[2].cpu().numpy(), rv)
            assert np.array_equal(_bits(d[4]), r16)
            h[0], h[1], h[2] = rp, rm, rv


def test_adam_zero_state_and_zero_gradients_bit_exact(cuda):
    """K4 routes exact zeros around the slow sqrt/div paths (a never-seen embedding row: m = v = 0, g = 0);
    the bits equal the oracle's for zero state, zero gradients, signed zeros, and mixed elements, across
    steps, in every K4 variant family reached by the default launch."""
    rng = np.random.default_rng(5)
    n = 200_003
    p = (rng.standard_normal(n) * 0.02).astype(np.float32)
    p[::7] = 0.0
    p[1::7] = -0.0
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    g[: n // 2] = 0.0                 # half the elements never get a gradient
    g[n // 2::5] = -0.0
    host = [p, m, v, g]
    ts = [torch.from_numpy(a.copy()).to(cuda) for a in host]
    p16 = torch.zeros(n, dtype=torch.bfloat16, device=cuda)
    table = kernels.AdamTable([(*ts, p16, n)], cuda)
    sc = kernels.new_step_scalars(cuda)
    for step in range(1, 4):
        sq = float(np.dot(host[3].astype(np.float64), host[3]))
        sc[0] = sq
        sc[1] = 0.0
        kernels.adam(table, HP, step, sc, torch.bfloat16)
        torch.cuda.synchronize()
        coef = arith.clip_coef(sq, HP["max_norm"])
        rp, rm, rv, r16 = arith.adamw(host[0], host[1], host[2], host[3], step, HP["lr"], HP["beta1"],
                                      HP["beta2"], HP["eps"], HP["weight_decay"], coef)
        for got, want in ((ts[0], rp), (ts[1], rm), (ts[2], rv)):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32))
        assert np.array_equal(_bits(p16), r16)
        host[0], host[1], host[2] = rp, rm, rv


def test_adam_skips_on_overflow_and_restores_compute_copy(cuda):
    host, dev = _segments(cuda, [5000, 77], 12)
    for d in dev:
        d[4].fill_(3.0)  # stale grads in the compute copy
    table = kernels.AdamTable(dev, cuda)
    sc = torch.tensor([1.0, 1.0, 0, 0], dtype=torch.float64, device=cuda)
    kernels.adam(table, HP, 1, sc, torch.bfloat16)
    torch.cuda.synchronize()
    for h, d in zip(host, dev):
        assert np.array_equal(d[0].cpu().numpy(), h[0])
        assert np.array_equal(d[1].cpu().numpy(), h[1])
        assert np.array_equal(d[2].cpu().numpy(), h[2])
        assert np.array_equal(_bits(d[4]), arith.f32_to_bf16_bits(h[0]))


def test_adam_f16_output(cuda):
    host, dev = _segments(cuda, [9999], 13)
    p16 = torch.zeros(9999, dtype=torch.float16, device=cuda)
    dev = [(d[0], d[1], d[2], d[3], p16, d[5]) for d in dev]
    table = kernels.AdamTable(dev, cuda)
    sc = kernels.new_step_scalars(cuda)
    hp = dict(HP, max_norm=0.0)
    kernels.adam(table, hp, 2, sc, torch.float16)
    h = host[0]
    rp, _, _, r16 = arith.adamw(h[0], h[1], h[2], h[3], 2, HP["lr"], HP["beta1"], HP["beta2"], HP["eps"],
                                HP["weight_decay"], np.float32(1.0), False, "f16")
    assert np.array_equal(dev[0][0].cpu().numpy(), rp)
    assert np.array_equal(p16.cpu().numpy().view(np.uint16), r16)


def test_norm_finalize(cuda):
    sc = torch.tensor([16.0, 0.0, 0, 0], dtype=torch.float64, device=cuda)
    out = torch.zeros(3, dtype=torch.float64, device=cuda)
    kernels.norm_finalize(sc, 1.0, out)
    o = out.cpu().tolist()
    assert o[0] == 4.0
    assert o[1] == float(np.float32(1.0 / (4.0 + 1e-6)))
    assert o[2] == 0.0


# ------------------------------------------------------------------ K6 copies

def test_offload_copies_round_trip(cuda):
    n = 3_000_001
    src = torch.randn(n).to(torch.bfloat16).pin_memory()
    dev = torch.zeros(n, dtype=torch.bfloat16, device=cuda)
    back = torch.zeros(n, dtype=torch.bfloat16).pin_memory()
    side = torch.cuda.Stream()
    kernels.copy_h2d(dev, src, stream=side)
    kernels.copy_d2h(back, dev, stream=side)
    side.synchronize()
    assert torch.equal(back, src)


def test_launch_counter_counts_kernels(cuda):
    before = _lib.launch_count()
    sc = kernels.new_step_scalars(cuda)
    kernels.step_reset(sc)
    kernels.step_reset(sc)
    assert _lib.launch_count() - before == 2


_VARIANT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import arith
from paper_2212_05339_b200 import kernels
dev = torch.device('cuda:0')
rng = np.random.default_rng(21)
sizes = [1, 3, 2048, 4096, 4097, 6143, 12288, 300_001]
host, segs = [], []
for n in sizes:
    arrs = [(rng.standard_normal(n) * s).astype(np.float32) for s in (0.02, 1e-3, 1e-3, 0.05)]
    arrs[2] = np.abs(arrs[2]) * 1e-3
    host.append(arrs)
    off = 1 if n == 4097 else 0   # one misaligned segment -> global-memory tile path
    ts = []
    for a in arrs:
        t = torch.zeros(n + off, device=dev); t[off:] = torch.from_numpy(a); ts.append(t[off:])
    segs.append((*ts, torch.zeros(n, dtype=torch.bfloat16, device=dev), n))
# one segment whose gradient is bf16 in place (world-1 fused path), scale 1/8
nb = 10_240
gb = arith.f32_to_bf16_bits((rng.standard_normal(nb) * 0.4).astype(np.float32))
hb = [(rng.standard_normal(nb) * 0.02).astype(np.float32), (rng.standard_normal(nb) * 1e-3).astype(np.float32),
      (rng.random(nb) * 1e-6).astype(np.float32), arith.release([gb], 0.125)[0]]
host.append(hb)
tb = [torch.from_numpy(a.copy()).to(dev) for a in hb[:3]]
pb16 = torch.from_numpy(gb.view(np.int16).copy()).view(torch.bfloat16).to(dev)
segs.append((tb[0], tb[1], tb[2], pb16, pb16, nb))
tab = kernels.AdamTable(segs, dev)
hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)
sc = kernels.new_step_scalars(dev)
for step in (1,):
    sq = float(sum(np.dot(h[3].astype(np.float64), h[3]) for h in host))
    sc[0] = sq
    kernels.adam(tab, hp, step, sc, torch.bfloat16, grad_scale=0.125)
    torch.cuda.synchronize()
    coef = arith.clip_coef(sq, 1.0)
    for h, d in zip(host, segs):
        rp, rm, rv, r16 = arith.adamw(h[0], h[1], h[2], h[3], step, 1e-3, 0.9, 0.999, 1e-8, 0.01, coef)
        assert np.array_equal(d[0].cpu().numpy(), rp) and np.array_equal(d[1].cpu().numpy(), rm)
        assert np.array_equal(d[2].cpu().numpy(), rv)
        assert np.array_equal(d[4].cpu().view(torch.int16).numpy().view(np.uint16), r16)
        h[0], h[1], h[2] = rp, rm, rv
sc[1] = 1.0
kernels.adam(tab, hp, 3, sc, torch.bfloat16, grad_scale=0.125)
torch.cuda.synchronize()
for h, d in zip(host, segs):
    assert np.array_equal(d[0].cpu().numpy(), h[0])
print("ok")
"""


@pytest.mark.parametrize("variant", [0, 1, 3, 5, 6, 7, 8, 9, 10, 11, 12, 14, 15])
def test_adam_variants_bit_exact(cuda, variant):
    """Every K4 variant (register-staged, TMA-staged, TMA in + TMA bulk-store out) is bit-exact vs the oracle."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ, ELX_ADAM_VARIANT=str(variant))
    out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_adam_compute_dtype_grads_equal_released_path(cuda):
    """World-1 fused path: K4 reading the bf16 gradient in place (unscaled
    in-register) == K3 release to fp32 + K4, bit for bit; mixed segment kinds."""
    rng = np.random.default_rng(31)
    inv_scale = 1.0 / 256
    sizes = [5, 4096, 9000, 300_000]
    segs, host = [], []
    sq = 0.0
    for j, n in enumerate(sizes):
        p = (rng.standard_normal(n) * 0.02).astype(np.float32)
        m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        v = (rng.random(n) * 1e-6).astype(np.float32)
        gbits = arith.f32_to_bf16_bits((rng.standard_normal(n) * 40).astype(np.float32))
        g, s, _ = arith.release([gbits], inv_scale)
        sq += s
        host.append((p, m, v, g))
        P, M, V = (torch.from_numpy(a.copy()).to(cuda) for a in (p, m, v))
        p16 = torch.from_numpy(gbits.view(np.int16).copy()).view(torch.bfloat16).to(cuda)
        if j % 2 == 0:  # in place: gradient read from, and parameter written to, the same bf16 buffer
            segs.append((P, M, V, p16, p16, n))
        else:           # released fp32 gradient
            segs.append((P, M, V, torch.from_numpy(g).to(cuda), torch.empty_like(p16), n))
    sc = torch.tensor([sq, 0, 0, 0], dtype=torch.float64, device=cuda)
    # the norm-only release accumulates the same sum of squares
    sc2 = kernels.new_step_scalars(cuda)
    for j, ((P, M, V, g, p16, n), (p, m, v, gg)) in enumerate(zip(segs, host)):
        if j % 2 == 0:
            kernels.release(None, [g.data_ptr()], n, torch.bfloat16, inv_scale, sc2)
    torch.cuda.synchronize()
    want_even = sum(arith.sumsq(h[3]) for j, h in enumerate(host) if j % 2 == 0)
    assert sc2[0].item() == pytest.approx(want_even, rel=1e-12)
    tab = kernels.AdamTable(segs, cuda)
    kernels.adam(tab, HP, 2, sc, torch.bfloat16, grad_scale=inv_scale)
    torch.cuda.synchronize()
    coef = arith.clip_coef(sq, HP["max_norm"])
    for (P, M, V, g, p16, n), (p, m, v, gg) in zip(segs, host):
        rp, rm, rv, r16 = arith.adamw(p, m, v, gg, 2, HP["lr"], HP["beta1"], HP["beta2"], HP["eps"],
                                      HP["weight_decay"], coef)
        assert np.array_equal(P.cpu().numpy(), rp)
        assert np.array_equal(M.cpu().numpy(), rm)
        assert np.array_equal(V.cpu().numpy(), rv)
        assert np.array_equal(_bits(p16), r16)


def test_adam_device_step_equals_host_step(cuda):
    """K4 device-step mode (step number from step_scalars[2], bias corrections
    from host-computed device tables) == host-step mode, bit for bit; and
    elx_step_advance counts only non-overflow steps."""
    host, dev = _segments(cuda, [4096 * 3 + 5, 77], 41)
    host2, dev2 = _segments(cuda, [4096 * 3 + 5, 77], 41)
    ta, tb = kernels.AdamTable(dev, cuda), kernels.AdamTable(dev2, cuda)
    tabs = kernels.BiasTables(HP["beta1"], HP["beta2"], cuda, length=16)
    sq = 3.0
    for t in (1, 2, 3, 7):
        sa = torch.tensor([sq, 0, 0, 0], dtype=torch.float64, device=cuda)
        sb = torch.tensor([sq, 0, float(t - 1), 0], dtype=torch.float64, device=cuda)
        kernels.adam(ta, HP, t, sa, torch.bfloat16)
        kernels.adam(tb, HP, 0, sb, torch.bfloat16, bias_tables=tabs)
        torch.cuda.synchronize()
        for a, b in zip(dev, dev2):
            for x, y in zip(a[:3], b[:3]):
                assert torch.equal(x, y), t
            assert torch.equal(a[4], b[4])
    sc = torch.tensor([1.0, 0.0, 5.0, 0.0], dtype=torch.float64, device=cuda)
    kernels.step_advance(sc)
    torch.cuda.synchronize()
    assert sc.tolist()[:3] == [0.0, 0.0, 6.0]
    sc[1] = 1.0
    kernels.step_advance(sc)
    torch.cuda.synchronize()
    assert sc.tolist()[:3] == [0.0, 0.0, 6.0]


@pytest.mark.parametrize("rows,cols", [(1, 8), (7, 24), (8192, 2048), (1000, 8200), (4096, 6144), (300, 768)])
def test_colsum_deterministic_and_exact(cuda, rows, cols):
    """K7 bias-gradient column sum: fp32 accumulation in the library's fixed
    order (rows within a sub-slice, sub-slices within a slice, slices) —
    reproduced exactly by the oracle."""
    rng = np.random.default_rng(rows + cols)
    bits = arith.f32_to_bf16_bits((rng.standard_normal((rows, cols)) * 0.1).astype(np.float32))
    x = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).to(cuda)
    out = torch.empty(cols, dtype=torch.bfloat16, device=cuda)
    kernels.colsum(x, out)
    out2 = torch.empty(cols, dtype=torch.float32, device=cuda)
    kernels.colsum(x, out2)
    slices, groups = kernels.colsum_geometry(rows, cols)
    xf = arith.bf16_bits_to_f32(bits).reshape(rows, cols)
    tot = arith.colsum_ordered(xf, slices, groups)
    assert np.array_equal(out2.cpu().numpy(), tot)
    assert np.array_equal(_bits(out), arith.f32_to_bf16_bits(tot))


_SYMM_SCRIPT = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", sys.argv[2])
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_2212_05339_b200 import kernels
from paper_2212_05339_b200.transport import SymmMemTransport
t = SymmMemTransport()
shard = t.alloc((4096,), torch.bfloat16, torch.device("cuda", 0))
block = t.alloc((4096,), torch.bfloat16, torch.device("cuda", 0))
shard.copy_(torch.arange(4096, device="cuda").to(torch.bfloat16))
ps, pb = t.peer_ptrs(shard), t.peer_ptrs(block)
assert len(ps) == 1 and ps[0] == shard.data_ptr() and pb[0] == block.data_ptr()
t.device_barrier()
kernels.fetch(block, ps, 4096)
t.device_barrier()
sc = kernels.new_step_scalars("cuda")
g = torch.empty(4096, device="cuda")
kernels.release(g, pb, 4096, torch.bfloat16, 1.0, sc)
torch.cuda.synchronize()
assert torch.equal(block, shard) and torch.equal(g, shard.float())
dist.destroy_process_group()
print("ok")
"""


def test_symmetric_memory_transport_api(cuda):
    """The P2P transport's torch symmetric-memory calls (alloc, rendezvous peer
    pointers, device barrier) work on the real box (one rank), and K2/K3 run on
    the mapped pointers."""
    import os
    import socket
    import subprocess
    import sys
    from pathlib import Path

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    root = str(Path(__file__).resolve().parents[1])
    out = subprocess.run([sys.executable, "-c", _SYMM_SCRIPT, root, port], capture_output=True, text=True,
                         timeout=300, env=dict(os.environ))
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


# ------------------------------------------------------------------ K8 lm_head cross-entropy

@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("rows,vocab,ld", [(1, 8, 8), (7, 389, 448), (64, 50257, 50304), (300, 1000, 1000)])
def test_lm_head_cross_entropy_matches_torch(cuda, rows, vocab, ld, dtype):
    """K8 vs torch F.cross_entropy on the fp32 copy of the unpadded bf16 logits:
    loss within 2e-6 relative, gradient within bf16 rounding (the kernel writes
    the bf16 gradient in place over the logits); pad columns get 0; an
    ignore_index row contributes nothing."""
    g = torch.Generator(device=cuda).manual_seed(rows + vocab)
    logits = (torch.randn(rows, ld, device=cuda, generator=g) * 3).to(dtype)
    tgt = torch.randint(0, vocab, (rows,), device=cuda, generator=g)
    if rows > 2:
        tgt[1] = -100
    ref_in = logits[:, :vocab].float().clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(ref_in, tgt)
    ref.backward(torch.tensor(3.0, device=cuda))
    x = logits.clone().requires_grad_(True)
    loss = kernels.lm_head_cross_entropy(x, tgt, vocab)
    (gx,) = torch.autograd.grad(loss, [x], torch.tensor(3.0, device=cuda))
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) <= 2e-6 * abs(ref.item())
    want = ref_in.grad
    got = gx[:, :vocab].float()
    # f16 flushes gradients below its subnormal step (6e-8) to zero; bf16 keeps fp32's range
    atol = 1e-6 * float(want.abs().max()) + (6e-8 if dtype == torch.float16 else 0.0)
    assert torch.allclose(got, want, rtol=1e-2, atol=atol)
    assert torch.equal(gx[:, vocab:].float(), torch.zeros_like(gx[:, vocab:].float()))
    if rows > 2:
        assert torch.count_nonzero(gx[1]) == 0


def test_lm_head_cross_entropy_deterministic(cuda):
    g = torch.Generator(device=cuda).manual_seed(5)
    logits = torch.randn(512, 50304, device=cuda, generator=g).to(torch.bfloat16)
    tgt = torch.randint(0, 50257, (512,), device=cuda, generator=g)
    outs = []
    for _ in range(2):
        x = logits.clone().requires_grad_(True)
        loss = kernels.lm_head_cross_entropy(x, tgt, 50257)
        (gx,) = torch.autograd.grad(loss, [x])
        outs.append((loss.item(), gx.clone()))
    assert outs[0][0] == outs[1][0] and torch.equal(outs[0][1], outs[1][1])


# ------------------------------------------------------------------ K9 LayerNorm parameter gradients

@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("rows,cols", [(1, 4), (7, 132), (8192, 2048), (1000, 3072), (4096, 4096)])
def test_ln_param_grad_matches_float64(cuda, dtype, rows, cols):
    """K9 vs a float64 reduction of the same inputs (dgamma = sum dy*(x-mean)*rstd,
    dbeta = sum dy) within the output dtype's rounding; deterministic."""
    g = torch.Generator(device=cuda).manual_seed(rows * 3 + cols)
    x = (torch.randn(rows, cols, device=cuda, generator=g) * 2 + 0.5).to(dtype)
    w = torch.randn(cols, device=cuda, generator=g).to(dtype)
    b = torch.randn(cols, device=cuda, generator=g).to(dtype)
    _, mean, rstd = torch.native_layer_norm(x, (cols,), w, b, 1e-5)
    dy = torch.randn(rows, cols, device=cuda, generator=g).to(dtype)
    dg = torch.empty(cols, dtype=dtype, device=cuda)
    db = torch.empty(cols, dtype=dtype, device=cuda)
    kernels.ln_param_grad(x, dy, mean.reshape(-1), rstd.reshape(-1), dg, db)
    xhat = (x.double() - mean.double().reshape(-1, 1)) * rstd.double().reshape(-1, 1)
    want_g = (dy.double() * xhat).sum(0)
    want_b = dy.double().sum(0)
    tol = 2 ** -7 if dtype == torch.bfloat16 else 2 ** -10
    for got, want in ((dg, want_g), (db, want_b)):
        err = (got.double() - want).abs()
        assert bool((err <= tol * want.abs() + 1e-4 * (rows ** 0.5)).all()), float(err.max())
    dg2, db2 = torch.empty_like(dg), torch.empty_like(db)
    kernels.ln_param_grad(x, dy, mean.reshape(-1), rstd.reshape(-1), dg2, db2)
    assert torch.equal(dg, dg2) and torch.equal(db, db2)


# ------------------------------------------------------------------ K10-K12 LayerNorm / GELU

@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("rows,cols", [(1, 8), (5, 64), (300, 768), (8192, 2048), (64, 3072), (33, 4096),
                                       (17, 6144), (3, 20480)])
def test_layer_norm_matches_torch(cuda, dtype, rows, cols):
    """K10/K11 vs torch's LayerNorm (fp32 math on the same inputs): y and dx
    within the output dtype's rounding, mean/rstd within 1e-5."""
    g = torch.Generator(device=cuda).manual_seed(rows + cols)
    x = (torch.randn(rows, cols, device=cuda, generator=g) * 1.5 + 0.3).to(dtype)
    w = (torch.randn(cols, device=cuda, generator=g) * 0.5 + 1).to(dtype)
    b = (torch.randn(cols, device=cuda, generator=g) * 0.1).to(dtype)
    dy = torch.randn(rows, cols, device=cuda, generator=g).to(dtype)
    y, mean, rstd = kernels.layer_norm_fwd(x, w, b)
    xf = x.float().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xf, (cols,), w.float(), b.float(), 1e-5)
    (gref,) = torch.autograd.grad(ref, [xf], dy.float())
    eps = 2 ** -7 if dtype == torch.bfloat16 else 2 ** -10
    assert torch.allclose(y.float(), ref, rtol=eps, atol=eps)
    m_ref = x.float().mean(-1)
    r_ref = torch.rsqrt(x.float().var(-1, unbiased=False) + 1e-5)
    assert torch.allclose(mean, m_ref, rtol=1e-5, atol=1e-5) and torch.allclose(rstd, r_ref, rtol=1e-5)
    dx = kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd)
    scale = float(gref.abs().max())
    assert torch.allclose(dx.float(), gref, rtol=2 * eps, atol=2 * eps * scale)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_gelu_matches_torch(cuda, dtype):
    g = torch.Generator(device=cuda).manual_seed(3)
    x = (torch.randn(8192 * 8 + 8, device=cuda, generator=g) * 3).to(dtype)
    dy = torch.randn(x.shape, device=cuda, generator=g).to(dtype)
    y = kernels.gelu_fwd(x)
    xf = x.float().requires_grad_(True)
    ref = torch.nn.functional.gelu(xf, approximate="tanh")
    (gref,) = torch.autograd.grad(ref, [xf], dy.float())
    eps = 2 ** -7 if dtype == torch.bfloat16 else 2 ** -9
    assert torch.allclose(y.float(), ref, rtol=eps, atol=1e-3)
    dx = kernels.gelu_bwd(x, dy)
    assert torch.allclose(dx.float(), gref, rtol=2 * eps, atol=2e-3)


def test_gpt2_layer_on_our_kernels_matches_stock_torch(cuda):
    """The product's GPT-2 layer (K10/K11/K9 LayerNorm, K12 GELU, K7 bias sums,
    overwrite-linear) vs the stock-torch layer of the CPU baseline
    (oracle/gpt2_ref.py) on the same bf16 inputs: output and input gradient
    agree to bf16 accuracy."""
    from oracle.gpt2_ref import block as ref_block
    from paper_2212_05339_b200 import gpt2
    H, heads, B, T = 256, 4, 2, 64
    g = torch.Generator(device=cuda).manual_seed(0)
    pieces = [(pid, off, shape) for pid, off, shape in gpt2.layer_pieces(0, H)]
    ps = []
    for pid, _, shape in pieces:
        if pid.endswith(".b"):
            ps.append((torch.randn(shape, device=cuda, generator=g) * 0.02).to(torch.bfloat16))
        elif "ln_" in pid:
            ps.append((1 + torch.randn(shape, device=cuda, generator=g) * 0.1).to(torch.bfloat16))
        else:
            ps.append((torch.randn(shape, device=cuda, generator=g) * 0.05).to(torch.bfloat16))
    x = torch.randn(B, T, H, device=cuda, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, T, H, device=cuda, generator=g).to(torch.bfloat16)
    outs = []
    for fn, tgt in ((ref_block, None), (gpt2._block, True)):
        xi = x.clone().requires_grad_(True)
        q = [p.clone().requires_grad_(True) for p in ps]
        targets = [torch.empty_like(p) for p in ps] if tgt else None
        out = fn(xi, q, heads) if targets is None else fn(xi, q, heads, targets)
        (gx,) = torch.autograd.grad(out, [xi], dy, allow_unused=True)
        outs.append((out.float(), gx.float()))
    (o_ref, g_ref), (o, gxx) = outs
    assert (o - o_ref).abs().max() <= 0.05 * o_ref.abs().max()
    assert (gxx - g_ref).abs().max() <= 0.05 * g_ref.abs().max()


# ------------------------------------------------------------------ cuBLASLt fused-epilogue GEMMs

def _gelu_ref(x):
    return torch.nn.functional.gelu(x, approximate="tanh")


@pytest.mark.parametrize("T,I,O", [(256, 64, 256), (8192, 2048, 8192), (512, 768, 3072)])
def test_lt_linear_gelu_and_dgelu_bgrad(cuda, T, I, O):
    """GELU_AUX_BIAS forward and DGELU_BGRAD backward vs fp32 torch: outputs
    within bf16 rounding, the bias gradient too; repeated calls bit-identical."""
    g = torch.Generator(device=cuda).manual_seed(T + O)
    x = (torch.randn(T, I, device=cuda, generator=g)).to(torch.bfloat16)
    w = (torch.randn(O, I, device=cuda, generator=g) * I ** -0.5).to(torch.bfloat16)
    b = (torch.randn(O, device=cuda, generator=g) * 0.1).to(torch.bfloat16)
    y, pre = kernels.linear_gelu(x, w, b, keep_aux=True)
    y2, none = kernels.linear_gelu(x, w, b, keep_aux=False)
    pre_ref = x.float() @ w.float().t() + b.float()
    assert none is None and torch.equal(y, y2)
    assert torch.allclose(pre.float(), pre_ref, rtol=2 ** -7, atol=2e-2)
    assert torch.allclose(y.float(), _gelu_ref(pre_ref), rtol=2 ** -7, atol=2e-2)
    # backward of out = gelu(pre) Wp^T + c through DGELU_BGRAD
    wp = (torch.randn(I, O, device=cuda, generator=g) * O ** -0.5).to(torch.bfloat16)
    dy = torch.randn(T, I, device=cuda, generator=g).to(torch.bfloat16)
    db = torch.empty(O, dtype=torch.bfloat16, device=cuda)
    d = kernels.linear_dgelu_bgrad(dy, wp, pre, db)
    pf = pre.float().requires_grad_(True)
    (want,) = torch.autograd.grad(_gelu_ref(pf) @ wp.float().t(), [pf], dy.float())
    scale = float(want.abs().max())
    assert torch.allclose(d.float(), want, rtol=2 ** -6, atol=2 ** -6 * scale)
    db_want = d.float().sum(0)
    assert torch.allclose(db.float(), db_want, rtol=2 ** -6, atol=2 ** -6 * float(db_want.abs().max()))
    db2 = torch.empty_like(db)
    d2 = kernels.linear_dgelu_bgrad(dy, wp, pre, db2)
    assert torch.equal(d, d2) and torch.equal(db, db2)


@pytest.mark.parametrize("T,I,O", [(256, 64, 128), (8192, 2048, 2048), (8192, 8192, 2048), (8192, 2048, 8192)])
def test_lt_wgrad_bgrad(cuda, T, I, O):
    """Weight gradient with the bias gradient from the same GEMM's epilogue
    (BGRADB) vs fp32 torch; deterministic."""
    g = torch.Generator(device=cuda).manual_seed(T * 3 + I)
    x = torch.randn(T, I, device=cuda, generator=g).to(torch.bfloat16)
    dy = torch.randn(T, O, device=cuda, generator=g).to(torch.bfloat16)
    dw = torch.empty(O, I, dtype=torch.bfloat16, device=cuda)
    db = torch.empty(O, dtype=torch.bfloat16, device=cuda)
    kernels.wgrad_bgrad(x, dy, dw, db)
    want_w = dy.float().t() @ x.float()
    want_b = dy.float().sum(0)
    assert torch.allclose(dw.float(), want_w, rtol=2 ** -7, atol=2 ** -7 * float(want_w.abs().max()))
    assert torch.allclose(db.float(), want_b, rtol=2 ** -7, atol=2 ** -7 * float(want_b.abs().max()))
    dw2, db2 = torch.empty_like(dw), torch.empty_like(db)
    kernels.wgrad_bgrad(x, dy, dw2, db2)
    assert torch.equal(dw, dw2) and torch.equal(db, db2)


def test_lt_linear_residual(cuda):
    """res + x W^T + b from one GEMM (C operand + bias epilogue) vs fp32 torch."""
    g = torch.Generator(device=cuda).manual_seed(1)
    x = torch.randn(4096, 2048, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(1024, 2048, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    b = torch.randn(1024, device=cuda, generator=g).to(torch.bfloat16)
    r = torch.randn(4096, 1024, device=cuda, generator=g).to(torch.bfloat16)
    y = kernels.linear_residual(x, w, b, r)
    want = r.float() + x.float() @ w.float().t() + b.float()
    assert torch.allclose(y.float(), want, rtol=2 ** -7, atol=2 ** -6 * float(want.abs().max()))


def test_colsum_batched_equals_single(cuda):
    """K7 over 3 same-shape inputs in one launch == three single launches, bit for bit."""
    g = torch.Generator(device=cuda).manual_seed(8)
    xs = [torch.randn(8192, 2048, device=cuda, generator=g).to(torch.bfloat16) for _ in range(3)]
    outs = [torch.empty(2048, dtype=torch.bfloat16, device=cuda) for _ in range(3)]
    kernels.colsum_batched(xs, outs)
    for x, o in zip(xs, outs):
        single = torch.empty_like(o)
        kernels.colsum(x, single)
        assert torch.equal(o, single)


@pytest.mark.parametrize("rows,cols", [(8192, 8192), (1000, 3072), (7, 264)])
def test_gelu_bwd_colsum_equals_unfused(cuda, rows, cols):
    """The fused GELU-backward + bias column sum is bit-identical to K12's
    backward followed by K7 (same rounding, same fp32 summation order)."""
    g = torch.Generator(device=cuda).manual_seed(rows + cols)
    x = (torch.randn(rows, cols, device=cuda, generator=g) * 2).to(torch.bfloat16)
    dy = torch.randn(rows, cols, device=cuda, generator=g).to(torch.bfloat16)
    db = torch.empty(cols, dtype=torch.bfloat16, device=cuda)
    dx = kernels.gelu_bwd_colsum(x, dy, db)
    dx2 = kernels.gelu_bwd(x, dy)
    db2 = torch.empty_like(db)
    kernels.colsum(dx2, db2)
    assert torch.equal(dx, dx2) and torch.equal(db, db2)


@pytest.mark.parametrize("rows,cols", [(8192, 2048), (33, 264), (5, 6144)])
def test_layer_norm_bwd_dx_residual_equals_separate_add(cuda, rows, cols):
    """K11 with the residual gradient folded in == K11 then a bf16 add."""
    g = torch.Generator(device=cuda).manual_seed(rows)
    x = torch.randn(rows, cols, device=cuda, generator=g).to(torch.bfloat16)
    dy = torch.randn(rows, cols, device=cuda, generator=g).to(torch.bfloat16)
    dres = torch.randn(rows, cols, device=cuda, generator=g).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(cols, device=cuda, generator=g)).to(torch.bfloat16)
    b = torch.zeros(cols, device=cuda, dtype=torch.bfloat16)
    _, mean, rstd = kernels.layer_norm_fwd(x, w, b)
    fused = kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd, dres=dres)
    sep = kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd) + dres
    assert torch.equal(fused, sep)


@pytest.mark.parametrize("ta,tb,M,N,K", [(False, False, 256, 384, 128), (True, False, 128, 256, 512),
                                         (False, True, 512, 768, 256), (False, False, 8192, 2048, 2048)])
def test_gemm_matches_torch(cuda, ta, tb, M, N, K):
    """kernels.gemm (elx_lt_matmul_ex, row-major op(a) @ op(b) [+ c] [+ bias])
    vs torch.mm in fp32 on the same bf16 operands."""
    g = torch.Generator(device=cuda).manual_seed(M + N + K)
    a = (torch.randn((K, M) if ta else (M, K), device=cuda, generator=g) * 0.1).to(torch.bfloat16)
    b = (torch.randn((N, K) if tb else (K, N), device=cuda, generator=g) * 0.1).to(torch.bfloat16)
    bias = torch.randn(N, device=cuda, generator=g).to(torch.bfloat16)
    c = torch.randn(M, N, device=cuda, generator=g).to(torch.bfloat16)
    A = a.float().t() if ta else a.float()
    B = b.float().t() if tb else b.float()
    for kw, want in (({}, A @ B), ({"bias": bias}, A @ B + bias.float()), ({"c": c}, A @ B + c.float())):
        got = kernels.gemm(a, b, ta=ta, tb=tb, **kw).float()
        assert (got - want).abs().max() <= 1e-2 * want.abs().max() + 1e-2, kw
    out = c.clone()
    kernels.gemm(a, b, ta=ta, tb=tb, out=out, c=out)  # in place: out += op(a) op(b)
    assert (out.float() - (A @ B + c.float())).abs().max() <= 1e-2 * (A @ B).abs().max() + 2e-2


def test_lt_table_choices_compute_the_same_gemm(cuda):
    """Every tuned entry of plans/lt_algos_b200.json, run through
    elx_lt_matmul_ex with its index, equals the heuristic's first candidate to
    bf16 accumulation-order accuracy (the table only changes the algorithm)."""
    from paper_2212_05339_b200 import _lib
    lib = _lib.load()
    ws = kernels._lt_workspace(cuda)
    g = torch.Generator(device=cuda).manual_seed(7)
    for key, idx in kernels._lt_table().items():
        epi, dt, ta, tb, m, n, k, lda, ldb, ldd, ldaux, has_c = key
        if m * n * k > 2 ** 34 or idx == 0:
            continue
        tdt = torch.bfloat16 if dt == _lib.BF16 else torch.float16
        A = (torch.randn(lda * (m if ta else k), device=cuda, generator=g) * 0.1).to(tdt)
        B = (torch.randn(ldb * (k if tb else n), device=cuda, generator=g) * 0.1).to(tdt)
        C = torch.randn(ldd * n, device=cuda, generator=g).to(tdt) if has_c else None
        bias = torch.randn(max(m, n), device=cuda, generator=g).to(tdt) if epi else None
        aux = torch.randn(max(ldaux, 1) * n, device=cuda, generator=g).to(tdt) if ldaux else None
        outs = []
        for i in (0, idx):
            D = torch.zeros(ldd * n, dtype=tdt, device=cuda)
            bb = None if bias is None else bias.clone()
            rc = lib.elx_lt_matmul_ex(epi, dt, ta, tb, m, n, k, A.data_ptr(), lda, B.data_ptr(), ldb,
                                      None if C is None else C.data_ptr(), D.data_ptr(), ldd,
                                      None if bb is None else bb.data_ptr(), None if aux is None else aux.data_ptr(),
                                      ldaux, ws, kernels._LT_WS_BYTES, i, torch.cuda.current_stream().cuda_stream)
            _lib.check(rc, "elx_lt_matmul_ex")
            outs.append(D.float())
        ref = outs[0]
        assert (outs[1] - ref).abs().max() <= 2e-2 * ref.abs().max() + 1e-2, key


@pytest.mark.parametrize("n,H,V,repeat", [(8192, 2048, 50304, False), (300, 64, 17, True), (1, 8, 4, False)])
def test_embedding_bwd_k13(cuda, n, H, V, repeat):
    """K13 accumulates the embedding gradient into grad_w in place: equal to
    round(grad_w + round(fp32 per-token sums in position order)); the sums
    match torch's embedding backward to fp32 accuracy; rows of absent tokens
    are untouched."""
    g = torch.Generator(device=cuda).manual_seed(n + H)
    hi = 3 if repeat else V
    tok = torch.randint(0, hi, (n,), device=cuda, generator=g)
    dy = torch.randn(n, H, device=cuda, generator=g).to(torch.bfloat16)
    base = torch.randn(V, H, device=cuda, generator=g).to(torch.bfloat16)
    got = base.clone()
    kernels.embedding_bwd(got, tok, dy)
    # reference: per-token fp32 sums in position order
    want = base.clone()
    S = torch.zeros(V, H, dtype=torch.float64, device=cuda).index_add_(0, tok, dy.double())
    present = torch.zeros(V, dtype=torch.bool, device=cuda)
    present[tok] = True
    want[present] = (base.float()[present] + S[present].float().to(torch.bfloat16).float()).to(torch.bfloat16)
    assert torch.equal(got[~present], base[~present])
    err = (got.float() - want.float()).abs()
    assert float(err.max()) <= 2 ** -7 * float(want.float().abs().max()) + 1e-3
    again = base.clone()
    kernels.embedding_bwd(again, tok, dy)
    assert torch.equal(got, again)
    # strided grad rows (a [V, H] view of a wider buffer)
    wide = torch.zeros(V, H + 8, dtype=torch.bfloat16, device=cuda)
    kernels.embedding_bwd(wide[:, :H], tok, dy)
    assert torch.equal(wide[:, H:], torch.zeros_like(wide[:, H:]))
