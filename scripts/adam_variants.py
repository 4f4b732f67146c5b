"""Time the K4 variant (ELX_ADAM_VARIANT) and K3 variant (ELX_REL_VARIANT) on
bench-sized shards, after ~1 s of warm-up work so clocks are ramped."""
import os, statistics, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2212_05339_b200 import kernels  # noqa: E402

dev = torch.device("cuda:0")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_313_626_112
segs_n = 12
per = -(-n // segs_n)
per = -(-per // 8) * 8
g0 = torch.Generator(device=dev).manual_seed(0)
f = lambda s: (torch.randn(segs_n, per, device=dev, generator=g0) * s)
p32, m, v, g = f(0.02), f(1e-3), f(1e-3).abs() * 1e-3, f(0.05)
p16 = torch.zeros(segs_n, per, dtype=torch.bfloat16, device=dev)
# argv[2] == "bf16": the world-1 fused layout of the training step — the gradient is the bf16
# chunk itself (read in place, overwritten by the new parameter): 28 B/element instead of 30
fused = len(sys.argv) > 2 and sys.argv[2] == "bf16"
if fused:
    p16.copy_(g)
tab = kernels.AdamTable([(p32[i], m[i], v[i], p16[i] if fused else g[i], p16[i], per) for i in range(segs_n)], dev)
bpe = 28 if fused else 30
sc = kernels.new_step_scalars(dev)
hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)


def timed(fn, reps=10, warm=40):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


t = timed(lambda: kernels.adam(tab, hp, 3, sc, torch.bfloat16), warm=60)
print(f"adam variant {os.environ.get('ELX_ADAM_VARIANT', '0')} ({bpe} B/elem): {t:.3f} ms  "
      f"{bpe * segs_n * per / t / 1e6:.1f} GB/s")
src = p16.view(-1)[: segs_n * per]
out = g.view(-1)
tot = segs_n * per
t = timed(lambda: kernels.release(out, [src.data_ptr()], tot, torch.bfloat16, 1.0, sc), warm=200)
print(f"release variant {os.environ.get('ELX_REL_VARIANT', '0')} world1 {tot} elems: {t:.3f} ms  {6 * tot / t / 1e6:.1f} GB/s")
