"""Check l1f_reconstruct (tcgen05 path for k > 16) against an FP64 reference: m n k [M]."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _device as dv, _lib
m, n, k = map(int, sys.argv[1:4])
g = torch.Generator(device='cuda').manual_seed(0)
af = torch.randn(m, k, device='cuda', generator=g)
bf = torch.randn(n, k, device='cuda', generator=g)
M = torch.randn(m, n, device='cuda', generator=g) * 10
L = torch.empty_like(M); S = torch.empty_like(M)
rs = torch.zeros(2, dtype=torch.float64, device='cuda')
for it in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    _lib.call("l1f_reconstruct", _lib.F32, m, n, k, dv.ptr(af), k, dv.ptr(bf), k, dv.ptr(M), n, dv.ptr(L), n, dv.ptr(S), n, dv.ptr(rs), dv.stream())
    torch.cuda.synchronize(); dt = time.time() - t0
ref = af.double() @ bf.double().T
err_l = ((L.double() - ref).norm() / ref.norm()).item()
err_s = ((S.double() - (M.double() - ref)).norm() / (M.double() - ref).norm()).item()
print(f"m={m} n={n} k={k}: {dt*1e3:.3f} ms, {12*m*n/dt/1e9:.0f} GB/s, rel L {err_l:.2e}, rel S {err_s:.2e}, resid {rs.tolist()}, M2 {float((M.double()**2).sum()):.6e}")
