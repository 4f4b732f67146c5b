"""Run every kernel of the library once, at small but non-trivial sizes (tails,
misaligned segments, multi-strip clusters), for compute-sanitizer:

    compute-sanitizer --tool memcheck  python scripts/sanitize_kernels.py
    compute-sanitizer --tool racecheck python scripts/sanitize_kernels.py
    compute-sanitizer --tool synccheck python scripts/sanitize_kernels.py

Each kernel's result is also checked against the CPU oracle, so a run under a
tool that perturbs scheduling still proves the outputs.
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import arith  # noqa: E402
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
bf = torch.bfloat16


def bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


# K1 pack / unpack (aligned + misaligned members, zero tail)
chunk = torch.full((20_011,), 3.0, dtype=bf, device=dev)
members = [(torch.randn(n, device=dev, generator=g).to(bf), off) for n, off in ((4096, 0), (17, 4096), (9000, 4113))]
kernels.chunk_pack(chunk, members, used_len=13_113)
outs = [torch.empty_like(t) for t, _ in members]
kernels.chunk_unpack(chunk, [(o, off) for o, (_, off) in zip(outs, members)])
torch.cuda.synchronize()
assert all(torch.equal(o, t) for o, (t, _) in zip(outs, members))
assert torch.count_nonzero(chunk[13_113:]) == 0

# K2 fetch (SM kernel and copy engines)
shards = [torch.randn(40_000, device=dev, generator=g).to(bf) for _ in range(4)]
block = torch.empty(160_000, dtype=bf, device=dev)
for engine in ("sm", "ce"):
    kernels.fetch(block, [s.data_ptr() for s in shards], 40_000, engine=engine)
    torch.cuda.synchronize()
    assert np.array_equal(bits(block), arith.gather([bits(s) for s in shards]))

# K3 release (world 4 with output; world 1 norm-only incl. tail)
sc = kernels.new_step_scalars(dev)
out = torch.empty(40_000, device=dev)
kernels.release(out, [s.data_ptr() for s in shards], 39_997, bf, 0.5, sc)
kernels.release(None, [shards[0].data_ptr()], 39_999, bf, 1.0, sc)
torch.cuda.synchronize()
want, _, _ = arith.release([bits(s)[:39_997] for s in shards], 0.5)
assert np.array_equal(out[:39_997].cpu().numpy(), want)

# K3 at world 2 and 8 over several tiles per CTA (TMA stages wrap, the two fp32 output stages alternate
# with their bulk stores) plus a partial tile; K2 over several tiles per CTA (stages reused)
for w, n in ((2, 1_300_003), (8, 700_005)):
    big = [torch.randn(n + 5, device=dev, generator=g).to(bf) for _ in range(w)]
    outw = torch.empty(n, device=dev)
    kernels.release(outw, [t.data_ptr() for t in big], n, bf, 1.0, sc)
    torch.cuda.synchronize()
    want, _, _ = arith.release([bits(t)[:n] for t in big], 1.0)
    assert np.array_equal(outw.cpu().numpy(), want)
    L = (n + 5) // 8 * 8
    blk = torch.empty(w * L, dtype=bf, device=dev)
    kernels.fetch(blk, [t.data_ptr() for t in big], L)
    torch.cuda.synchronize()
    assert np.array_equal(bits(blk), arith.gather([bits(t)[:L] for t in big]))

# K4 Adam: every variant family (TMA in/out default, TMA in, register-staged) over a tail + misaligned segment
sizes = [4096 * 3 + 5, 2048, 777]
segs = []
for n in sizes:
    p, m, v = (torch.randn(n + 1, device=dev, generator=g)[1:] * 0.02 for _ in range(3))
    v = v.abs()
    gg = torch.randn(n, device=dev, generator=g).to(bf)
    segs.append((p.contiguous(), m.contiguous(), v.contiguous(), gg, torch.empty(n, dtype=bf, device=dev), n))
segs.append((*(torch.randn(1000, device=dev)[1:] for _ in range(3)), torch.randn(999, device=dev),
             torch.empty(999, dtype=bf, device=dev), 999))  # misaligned fp32 segment
tab = kernels.AdamTable(segs, dev)
sc.zero_()
sc[0] = 1.0
kernels.adam(tab, dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0), 1, sc, bf)
torch.cuda.synchronize()

# K7 / K9 / K10-K12 / K8
x = torch.randn(1000, 3072, device=dev, generator=g).to(bf)
dy = torch.randn(1000, 3072, device=dev, generator=g).to(bf)
w, b = torch.ones(3072, dtype=bf, device=dev), torch.zeros(3072, dtype=bf, device=dev)
cs = torch.empty(3072, device=dev)
kernels.colsum(dy, cs)
y, mean, rstd = kernels.layer_norm_fwd(x, w, b)
dx = kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd)
dg, db = torch.empty_like(w), torch.empty_like(b)
kernels.ln_param_grad(x, dy, mean.view(-1), rstd.view(-1), dg, db)
gy = kernels.gelu_fwd(x)
gx = kernels.gelu_bwd(x, dy)
dres = torch.randn(1000, 3072, device=dev, generator=g).to(bf)
dxr = kernels.layer_norm_bwd_dx(x, dy, w, mean, rstd, dres=dres)  # K11 + residual gradient
x2, dy2, dres2 = x[:, :2048].contiguous(), dy[:, :2048].contiguous(), dres[:, :2048].contiguous()
y2, mean2, rstd2 = kernels.layer_norm_fwd(x2, w[:2048], b[:2048])
dxr2 = kernels.layer_norm_bwd_dx(x2, dy2, w[:2048], mean2, rstd2, dres=dres2)  # warp-per-row variant
dbg = torch.empty(3072, dtype=bf, device=dev)
gxc = kernels.gelu_bwd_colsum(x, dy, dbg)  # K12 backward + K7
wg = torch.randn(500, 3072, device=dev, generator=g).to(bf)
tok = torch.randint(0, 500, (1000,), device=dev, generator=g)
kernels.embedding_bwd(wg, tok, dy)  # K13
a_ = torch.randn(256, 384, device=dev, generator=g).to(bf)
b_ = torch.randn(384, 512, device=dev, generator=g).to(bf)
cg = kernels.gemm(a_, b_)  # elx_lt_matmul_ex
kernels.gemm(a_, b_, out=cg, c=cg)
logits = torch.randn(64, 1032, device=dev, generator=g).to(bf).requires_grad_(True)
tgt = torch.randint(0, 1000, (64,), device=dev, generator=g)
loss = kernels.lm_head_cross_entropy(logits, tgt, 1000)
(gl,) = torch.autograd.grad(loss, [logits])
torch.cuda.synchronize()
unit, group = kernels.colsum_geometry(1000, 3072)
want = arith.colsum_ordered(dy.float().cpu().numpy(), unit, group)
assert np.array_equal(cs.cpu().numpy(), want)
print("sanitize run ok")
