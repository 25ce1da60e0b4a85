"""Run one filter case (dtype, s, k, n) and compare with the oracle; used under `timeout`."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200.l1reg import filter_units
from oracle import adm_filter
dt = torch.float32 if sys.argv[1] == 'f32' else torch.float64
s, k, n = map(int, sys.argv[2:5])
rng = np.random.default_rng(s * 1000 + k)
a, _ = np.linalg.qr(rng.standard_normal((s, k)))
x = a @ rng.standard_normal((k, n)) * 5.0
mask = rng.random(x.shape) < 0.08
x[mask] += rng.uniform(-200, 200, mask.sum())
x[:, 0] = 0.0
tol = 1e-7 if dt == torch.float32 else 1e-9
ndt = np.float32 if dt == torch.float32 else np.float64
xt = torch.from_numpy(np.ascontiguousarray(x.T.astype(ndt))).cuda()
at = torch.from_numpy(a.astype(ndt)).cuda()
t0 = time.time()
z, e, it, res, st = filter_units(xt, at, l1pcp.AdmConfig(tol=tol))
torch.cuda.synchronize()
zr, er, itr, rr, sr = adm_filter.solve_units(x, a, tol)
lc = a @ z.double().cpu().numpy().T; lr = a @ zr
print(sys.argv[1:], 'time', round(time.time() - t0, 3), 'err', np.linalg.norm(lc - lr) / np.linalg.norm(lr), 'iters', it.float().mean().item(), itr.mean(), 'status', np.bincount(st.cpu().numpy(), minlength=4))
