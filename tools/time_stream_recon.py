"""Time l1f_reconstruct for small k at cfg4's shape: python tools/time_stream_recon.py [m n k]"""
import sys
import torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import engine
m, n, k = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (76800, 10000, 10)
mt = torch.randn(m, n, device="cuda")
af = torch.randn(m, k, device="cuda"); bf = torch.randn(n, k, device="cuda")
l = torch.empty_like(mt); s = torch.empty_like(mt)
for _ in range(3): engine.reconstruct(mt, af, bf, l, s)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): _, _, rs = engine.reconstruct(mt, af, bf, l, s)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"m={m} n={n} k={k}: {ms:.3f} ms  {12*m*n/ms/1e6:.0f} GB/s  check {(l - af @ bf.T).abs().max().item():.2e} {(s - (mt - l)).abs().max().item():.1e} m2 {rs[1].item():.6e} vs {(mt.double()**2).sum().item():.6e}")
