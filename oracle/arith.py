"""numpy restatement of the hot path's byte and floating-point semantics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference contains no implementation of any function here (SURVEY.md
§0.5, §8c): the semantics come from the paper (PAPER.md:107-113 mixed
precision, :170-181 chunks/rCache, :221-238 gradient overwrite + reduce +
paired optimizer chunk) and the concrete arithmetic is torch's:
  * AdamW, single-tensor path (torch/optim/adam.py:347-547 of torch 2.11):
    decoupled decay (:419), m.lerp_(g, 1-b1) (:457),
    v.mul_(b2).addcmul_(g, g, value=1-b2) (:476),
    denom = v.sqrt()/sqrt(bc2) + eps (:545), p.addcdiv_(m, denom, -lr/bc1) (:547);
  * unscale then clip: GradScaler unscale (g * inv_scale) followed by
    clip_grad_norm_ (coef = max_norm / (norm + 1e-6), clamped to 1);
  * overflow: any non-finite reduced gradient skips the step (no state change).

Every elementwise operation is one float32 IEEE rounding, in the order
written (numpy ufuncs never fuse), which is exactly the order the CUDA kernels
use with explicit _rn intrinsics — GPU vs this oracle is bit-exact. Versus
torch CPU (whose vectorised lerp uses an FMA) it agrees to ~1 ulp; that
agreement is pinned by tests/golden/adamw_golden.npz.
"""

from __future__ import annotations

import numpy as np

F32 = np.float32


# ------------------------------------------------------------ bf16 / f16

def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit pattern (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = ((u & 0x7F800000) == 0x7F800000) & ((u & 0x007FFFFF) != 0)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    r = np.where(nan, (u >> 16) | 0x40, r)
    return (r & 0xFFFF).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def to_f32(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Compute-precision payload (uint16 bits for bf16, float16 for f16) -> f32."""
    if dtype == "bf16":
        return bf16_bits_to_f32(bits)
    if dtype == "f16":
        return np.asarray(bits).view(np.float16).astype(np.float32)
    raise ValueError(dtype)


def from_f32(x: np.ndarray, dtype: str) -> np.ndarray:
    """float32 -> compute-precision payload (uint16 bit patterns)."""
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    if dtype == "f16":
        return np.asarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)
    raise ValueError(dtype)


# ------------------------------------------------------------ K1 pack

def pack(phys_len: int, members, fill_dtype=np.uint16) -> np.ndarray:
    """Chunk buffer with members copied at their offsets, zeros elsewhere
    (chunking.py:113-131 offsets; padding per chunking.py:141-146).
    members: [(array, offset)] in the chunk's element type."""
    out = np.zeros(phys_len, dtype=fill_dtype)
    for arr, off in members:
        a = np.asarray(arr).reshape(-1)
        out[off:off + a.size] = a
    return out


def unpack(chunk: np.ndarray, offset: int, numel: int) -> np.ndarray:
    return chunk[offset:offset + numel].copy()


# ------------------------------------------------------------ K2 fetch

def gather(shards) -> np.ndarray:
    """All-gather: block = shard_0 || shard_1 || ... (rank order)."""
    return np.concatenate([np.asarray(s).reshape(-1) for s in shards])


def shard_len(chunk_length: int, world: int, align: int = 8) -> int:
    """Per-rank shard: ceil(C/N) rounded up to `align` elements (16 bytes)."""
    s = -(-chunk_length // world)
    return -(-s // align) * align


# ------------------------------------------------------------ K3 release

def release(srcs, inv_scale: float, dtype: str = "bf16"):
    """Rank-ordered fp32 reduction of this rank's segment from every rank,
    times inv_scale; plus float64 sum of squares and the overflow flag."""
    acc = None
    for s in srcs:
        x = to_f32(np.asarray(s).reshape(-1), dtype)
        acc = x.copy() if acc is None else (acc + x).astype(np.float32)
    g = (acc * F32(inv_scale)).astype(np.float32)
    return g, sumsq(g), bool(not np.isfinite(g).all())


def quad_sq(a: np.ndarray) -> np.ndarray:
    """The release kernel's sum-of-squares unit over the last axis (length 4):
    q = ((a0*a0 + a1*a1) + a2*a2) + a3*a3 in float32, every multiply and add
    separately rounded (include/elixir_b200.h, K3). Exact for bf16 values'
    squares; <= ~4 * 2^-24 relative error otherwise."""
    a = np.asarray(a, np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        q = a[..., 0] * a[..., 0]
        for e in (1, 2, 3):
            q = (q + a[..., e] * a[..., e]).astype(np.float32)
    return q


def sumsq(g) -> float:
    """Sum of squares of one released segment in K3's units: quads of
    consecutive elements from element 0 (zero-padded), each an fp32 partial
    (quad_sq), added in float64 (the order of the fp64 additions is the
    kernel's launch geometry: release_norm_ordered; here numpy's)."""
    g = np.asarray(g, np.float32).reshape(-1)
    pad = np.zeros(-(-g.size // 4) * 4, np.float32)
    pad[:g.size] = g
    with np.errstate(over="ignore", invalid="ignore"):
        return float(np.sum(quad_sq(pad.reshape(-1, 4)).astype(np.float64)))


def sumsq_chunked(rel: dict, members: dict) -> float:
    """Sum of squares of a whole step's released gradients as K3 forms it: the
    quad units run over each CHUNK's elements from the chunk's offset 0 (the
    members packed at their layout offsets, pack_chunks' contiguous order,
    chunking.py:113-131), and over each parameter outside the chunks (the
    shared wte) from its own element 0. rel: pid -> released fp32 gradient;
    members: pid -> (chunk id, offset, numel) for chunk members."""
    chunks: dict = {}
    sq = 0.0
    for pid, g in rel.items():
        if pid in members:
            c, off, n = members[pid]
            chunks.setdefault(c, []).append((off, np.asarray(g, np.float32).reshape(-1)))
        else:
            sq += sumsq(g)
    for c in sorted(chunks):
        parts = sorted(chunks[c], key=lambda t: t[0])
        flat = np.zeros(max(o + a.size for o, a in parts), np.float32)
        for o, a in parts:
            flat[o:o + a.size] = a
        sq += sumsq(flat)
    return sq


def _block_sum_fixed(x: np.ndarray) -> np.ndarray:
    """The release kernel's fixed CTA reduction over the last axis (256 fp64
    values): a butterfly (xor 16, 8, 4, 2, 1) inside each warp of 32, then the
    same butterfly over the 8 warp sums padded with zeros; lane 0's value."""
    lanes = np.arange(32)
    w = x.reshape(x.shape[:-1] + (8, 32))
    for o in (16, 8, 4, 2, 1):
        w = w + w[..., lanes ^ o]
    y = np.zeros(x.shape[:-1] + (32,), np.float64)
    y[..., :8] = w[..., 0]
    for o in (16, 8, 4, 2, 1):
        y = y + y[..., lanes ^ o]
    return y[..., 0]


def release_norm_ordered(gs, ctas: int, tile_vecs: int) -> float:
    """Sum of squares of one K3 launch (elx_release_batch) in the kernel's
    exact fp64 order (include/elixir_b200.h, K3; elx_release_geometry gives
    ctas/tile_vecs): the segments' tiles of `tile_vecs` 8-element vectors
    concatenated, tile k to CTA k % ctas, thread t of 256 taking vectors t,
    t+256, ... of a tile; per thread a sequential fp64 sum of its vectors' two
    fp32 quad partials (quad_sq; np.cumsum is sequential), elements past a
    segment's end +0.0; per CTA the fixed block
    reduction; the partials summed per thread in slot order, then reduced the
    same way. Vectorised over CTAs and threads."""
    T = 256
    U = tile_vecs // T
    tiles = []
    for g in gs:
        g = np.asarray(g, np.float32).reshape(-1)
        te = tile_vecs * 8
        nt = -(-g.size // te)
        pad = np.zeros(nt * te, np.float32)
        pad[:g.size] = g
        tiles.append(pad.reshape(nt, U, T, 8))
    if not tiles or sum(t.shape[0] for t in tiles) == 0 or ctas <= 0:
        return 0.0
    allt = np.concatenate(tiles)                    # [tiles, U, T, 8]
    nt = allt.shape[0]
    k = -(-nt // ctas)
    full = np.zeros((k * ctas, U, T, 8), np.float32)
    full[:nt] = allt
    q = quad_sq(full.reshape(k * ctas, U, T, 2, 4)).astype(np.float64)   # [tiles, U, T, 2]
    # [k, ctas, U, T, 2] -> per (cta, thread): sequence over (k, U, 2)
    seq = q.reshape(k, ctas, U, T, 2).transpose(1, 3, 0, 2, 4).reshape(ctas, T, -1)
    with np.errstate(over="ignore", invalid="ignore"):
        sq = np.cumsum(seq, axis=-1)[..., -1]        # [ctas, T]
    part = _block_sum_fixed(sq)                       # [ctas]
    rows = -(-ctas // T)
    slots = np.zeros(rows * T, np.float64)
    slots[:ctas] = part
    per_thread = np.cumsum(slots.reshape(rows, T), axis=0)[-1]   # thread t: slots t, t+256, ... in order
    return float(_block_sum_fixed(per_thread))


def colsum_ordered(x: np.ndarray, slices: int, groups: int) -> np.ndarray:
    """Bias-gradient column sum (K7) in its fixed fp32 order: rows cut into
    `slices` contiguous slices of ceil(rows/slices) rows, each slice into
    `groups` contiguous sub-slices of ceil(slice/groups); a sub-slice is
    summed from 0 in row order, sub-slices in order, then slices in order.
    (The bias gradient of y = x W^T + b is the column sum of dy; torch's
    reference computes it as dy.sum(0) with an unspecified order.)"""
    rows, cols = x.shape
    per = -(-rows // slices)
    sub = -(-per // groups)
    tot = np.zeros(cols, np.float32)
    for s in range(slices):
        end = min(rows, (s + 1) * per)
        cta = np.zeros(cols, np.float32)
        for w in range(groups):
            r0 = s * per + w * sub
            acc = np.zeros(cols, np.float32)
            for r in range(r0, min(end, r0 + sub)):
                acc = (acc + x[r]).astype(np.float32)
            cta = (cta + acc).astype(np.float32)
        tot = (tot + cta).astype(np.float32)
    return tot


def clip_coef(sq: float, max_norm: float) -> np.float32:
    """clip_grad_norm_ convention: min(1, max_norm / (norm + 1e-6)) (float64 -> float32)."""
    if not max_norm > 0:
        return F32(1.0)
    c = max_norm / (np.sqrt(sq) + 1e-6)
    return F32(c) if c < 1.0 else F32(1.0)


# ------------------------------------------------------------ K4 AdamW

def adam_consts(step: int, lr: float, beta1: float, beta2: float, eps: float, wd: float):
    """Host scalars in float64, each cast once to float32 (torch passes
    Python floats; the kernels cast them to the tensor dtype)."""
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    return dict(decay=F32(1.0 - lr * wd), omb1=F32(1.0 - beta1), b2=F32(beta2),
                omb2=F32(1.0 - beta2), bc2_sqrt=F32(bc2 ** 0.5), neg_step=F32(-(lr / bc1)),
                eps=F32(eps))


def adamw(p, m, v, g, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0,
          coef=F32(1.0), skip=False, p16_dtype="bf16"):
    """One AdamW step on float32 arrays (returns new p, m, v, p16 bits)."""
    p = np.asarray(p, np.float32)
    m = np.asarray(m, np.float32)
    v = np.asarray(v, np.float32)
    if skip:
        return p.copy(), m.copy(), v.copy(), from_f32(p, p16_dtype)
    k = adam_consts(step, lr, beta1, beta2, eps, wd)
    g = np.asarray(g, np.float32) * F32(coef)
    p = p * k["decay"]
    m = m + k["omb1"] * (g - m)
    v = v * k["b2"] + (k["omb2"] * g) * g
    denom = np.sqrt(v) / k["bc2_sqrt"] + k["eps"]
    p = p + (k["neg_step"] * m) / denom
    p, m, v = (a.astype(np.float32) for a in (p, m, v))
    return p, m, v, from_f32(p, p16_dtype)


def hybrid_step(shards, grads_by_rank, step, hp, inv_scale=1.0, dtype="bf16"):
    """Whole optimizer step over several shards of one rank: release every
    shard, combine the norm/overflow across them, then AdamW each shard.
    shards: [dict(p, m, v)], grads_by_rank: per shard, list over ranks of
    this rank's segment (compute dtype payloads)."""
    released, sq, bad = [], 0.0, False
    for srcs in grads_by_rank:
        g, s, b = release(srcs, inv_scale, dtype)
        released.append(g)
        sq += s
        bad |= b
    coef = clip_coef(sq, hp.get("max_norm", 0.0))
    out = []
    for sh, g in zip(shards, released):
        out.append(adamw(sh["p"], sh["m"], sh["v"], g, step, hp["lr"], hp["beta1"], hp["beta2"],
                         hp["eps"], hp["wd"], coef, bad, dtype))
    return out, released, sq, bad
