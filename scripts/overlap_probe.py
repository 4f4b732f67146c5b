"""Concurrency probe: 24 fc-forward GEMMs (GPT-2 1.3B shapes) on one stream while K4 over
the full 1.3B shard set runs capped at N CTAs on another; vs each alone."""
import statistics, sys, torch
sys.path.insert(0, '.')
from paper_2212_05339_b200 import kernels
dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(0)
n = 1313626112; segs_n = 12; per = -(-n // segs_n); per = -(-per // 8) * 8
p32 = torch.randn(segs_n, per, device=dev, generator=g) * 0.02
m = torch.zeros_like(p32); v = torch.zeros_like(p32)
p16 = p32.to(torch.bfloat16)
tab = kernels.AdamTable([(p32[i], m[i], v[i], p16[i], p16[i], per) for i in range(segs_n)], dev)
sc = kernels.new_step_scalars(dev)
hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=0.0)
x = torch.randn(8192, 2048, device=dev, generator=g).to(torch.bfloat16)
w = torch.randn(8192, 2048, device=dev, generator=g).to(torch.bfloat16)
b = torch.zeros(8192, device=dev, dtype=torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def gemms():
    for _ in range(60):
        torch.nn.functional.linear(x, w, b)
def timed(fn):
    ts = []
    for i in range(5):
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); e.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(a.elapsed_time(e))
    return statistics.median(ts)
print('gemms alone ms', round(timed(gemms), 3))
print('adam alone ms', round(timed(lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16)), 3))
for cap in (8, 16, 32, 64, 0):
    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s2):
            kernels.adam(tab, hp, 1, sc, torch.bfloat16, stream=s2, max_ctas=cap)
        with torch.cuda.stream(s1):
            gemms()
        cur.wait_stream(s1); cur.wait_stream(s2)
    t_adam_cap = timed(lambda: kernels.adam(tab, hp, 1, sc, torch.bfloat16, max_ctas=cap))
    print('cap', cap, 'adam capped alone', round(t_adam_cap, 3), 'both concurrent', round(timed(both), 3))
