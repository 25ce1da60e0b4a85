"""Per-pass cost of the TC filter vs cluster size: python tools/tc_pass_scan.py (run with L1F_TC_PROF=1)"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200.l1reg import filter_units
k, n = int(os.environ.get("K", 100)), int(os.environ.get("N", 20000))
for s in (250, 500, 1000, 2000):
    rng = np.random.default_rng(s)
    a, _ = np.linalg.qr(rng.standard_normal((s, k)))
    at = torch.from_numpy(a.astype(np.float32)).cuda()
    x = at @ torch.randn(k, n, device="cuda") * 5
    x = x + (torch.rand_like(x) < 0.05) * (torch.rand_like(x) * 1000 - 500)
    xt = x.T.contiguous()
    filter_units(xt, at, l1pcp.AdmConfig(tol=1e-7), want_e=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z, e, it, res, st = filter_units(xt, at, l1pcp.AdmConfig(tol=1e-7), want_e=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"s={s} k={k} n={n}: {dt*1e3:.2f} ms  iters {it.float().mean().item():.2f}  unit-iter/us {n*it.float().mean().item()/dt/1e6:.1f}", flush=True)
