"""Host AdamW (elx_cpu_adam) throughput on the CPU-home path: 128 Mi bf16-gradient elements, median of 6.
    python scripts/cpu_adam_probe.py [threads]     (ELX_LIB=<other .so> for an A/B)
"""
import time, torch, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2212_05339_b200 import kernels
n = 128 * 2**20
th = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p32 = torch.randn(n) * 0.02; m = torch.randn(n) * 1e-3; v = torch.rand(n) * 1e-6
g16 = (torch.randn(n) * 1e-2).to(torch.bfloat16); p16 = torch.empty(n, dtype=torch.bfloat16)
hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, max_norm=1.0)
segs = [(p32, m, v, g16, p16, n)]
ts = []
for i in range(6):
    t0 = time.perf_counter()
    kernels.cpu_adam(segs, hp, 1, [0.5, 0.0], torch.bfloat16, th)
    ts.append(time.perf_counter() - t0)
t = sorted(ts)[len(ts)//2]
print(f"threads {th}: {t*1e3:.1f} ms, {n/t/1e9:.2f} G elem/s, {30*n/t/1e9:.1f} GB/s (30 B/elem incl RFO)")
