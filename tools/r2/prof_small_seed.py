"""Per-phase cycles of the one-CTA Gram ALM kernel (build with -DL1F_SEED_PROF)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import pcp_adm
rng = np.random.default_rng(0)
for (m, n, r) in [(100, 100, 10), (113, 113, 11)]:
    L0 = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    M = torch.from_numpy(L0 + np.where(rng.random((m, n)) < 0.1, rng.uniform(-50, 50, (m, n)), 0.0)).cuda()
    pcp_adm.solve_pcp_device(M, pcp_adm.AdmConfig(tol=1e-7)); torch.cuda.synchronize()
