"""Plain-torch GPT-2 layer — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The CPU baseline (bench.py --impl reference and the bench line's
cpu_baseline) times the training step's math with this restatement on host
cores. It is the same layer the product computes (paper_2212_05339_b200/
gpt2.py `_block`: pre-LN attention + MLP, q/k/v as three row blocks of
attn.qkv, causal SDPA, tanh-GELU, parameter order of profiles.py:451-456)
written with stock torch ops only, so it runs on any device and never touches
the product's CUDA kernels.
"""

from __future__ import annotations

import torch.nn.functional as F


def block(x, p, heads):
    """One GPT-2 layer on its 16 pieces (gpt2.layer_pieces order)."""
    B, T, H = x.shape
    ln1w, ln1b, qw, kw, vw, qb, kb, vb, projw, projb, ln2w, ln2b, fcw, fcb, mpw, mpb = p
    hd = H // heads
    h = F.layer_norm(x, (H,), ln1w, ln1b, 1e-5)
    q, k, v = (F.linear(h, w, b).view(B, T, heads, hd).transpose(1, 2) for w, b in ((qw, qb), (kw, kb), (vw, vb)))
    a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    x = x + F.linear(a.transpose(1, 2).reshape(B, T, H), projw, projb)
    h = F.layer_norm(x, (H,), ln2w, ln2b, 1e-5)
    return x + F.linear(F.gelu(F.linear(h, fcw, fcb), approximate="tanh"), mpw, mpb)
