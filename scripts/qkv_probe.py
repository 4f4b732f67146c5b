"""Probe: q/k/v as strided views of ONE [B, T, 3H] projection output — does
SDPA (cuDNN) accept them without a copy, do its gradients come back packed,
and what does one N=3H GEMM save over three N=H ones (GPT-2 1.3B shapes)?

    python scripts/qkv_probe.py
"""
import json
import statistics

import torch
import torch.nn.functional as F

dev = torch.device("cuda:0")
B, T, H, heads = 8, 1024, 2048, 16
hd = H // heads
bf = torch.bfloat16
g = torch.Generator(device=dev).manual_seed(0)
h = torch.randn(B, T, H, device=dev, generator=g).to(bf)
W = (torch.randn(3 * H, H, device=dev, generator=g) * 0.02).to(bf)
bias = torch.zeros(3 * H, device=dev, dtype=bf)
flush = torch.ones(64 * 2 ** 20, device=dev)
sink = torch.empty((), device=dev)


def timed(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        torch.sum(flush, dim=0, out=sink)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def sep():
    return [F.linear(h, W[j * H:(j + 1) * H], bias[j * H:(j + 1) * H]) for j in range(3)]


def packed():
    return F.linear(h, W, bias)


out = {"gemm_3x_N2048_ms": timed(sep), "gemm_1x_N6144_ms": timed(packed)}


def attn_sep():
    q, k, v = (t.view(B, T, heads, hd).transpose(1, 2) for t in sep())
    return q, k, v


def attn_packed():
    qkv = packed().view(B, T, 3, heads, hd)
    q, k, v = (qkv[:, :, j].transpose(1, 2) for j in range(3))
    return q, k, v


for name, mk in (("sep", attn_sep), ("packed", attn_packed)):
    q, k, v = (t.detach().requires_grad_(True) for t in mk())
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    go = torch.randn_like(o)
    dq, dk, dv = torch.autograd.grad(o, (q, k, v), go)
    out[name + "_fwd_ms"] = timed(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))
    out[name + "_fwdbwd_ms"] = timed(
        lambda: torch.autograd.grad(F.scaled_dot_product_attention(q, k, v, is_causal=True), (q, k, v), go))
    out[name + "_grad_strides"] = [list(dq.stride()), list(dk.stride())]
    out[name + "_grads_one_storage"] = dq.untyped_storage().data_ptr() == dk.untyped_storage().data_ptr()
    out[name + "_q_strides"] = list(q.stride())
    if name == "sep":
        ref = (o, dq, dk, dv)
    else:
        out["packed_equals_sep_bitwise"] = all(torch.equal(a, b) for a, b in zip(ref, (o, dq, dk, dv)))
print(json.dumps(out))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    q, k, v = (t.detach().requires_grad_(True) for t in attn_packed())
    o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    torch.autograd.grad(o, (q, k, v), torch.randn_like(o))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
