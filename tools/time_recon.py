"""Kernel time of l1f_reconstruct with CUDA events (m n k reps)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _device as dv, _lib
m, n, k = map(int, sys.argv[1:4])
af = torch.randn(m, k, device='cuda'); bf = torch.randn(n, k, device='cuda')
M = torch.randn(m, n, device='cuda'); L = torch.empty_like(M); S = torch.empty_like(M)
rs = torch.zeros(2, dtype=torch.float64, device='cuda')
def run():
    _lib.call("l1f_reconstruct", _lib.F32, m, n, k, dv.ptr(af), k, dv.ptr(bf), k, dv.ptr(M), n, dv.ptr(L), n, dv.ptr(S), n, dv.ptr(rs), dv.stream())
for _ in range(3): run()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(5): run()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"m={m} n={n} k={k} mask={__import__('os').environ.get('L1F_RECON_TC_MASK','0')}: {ms:.3f} ms/call, {12*m*n/ms/1e6:.0f} GB/s (12 B/entry)")
