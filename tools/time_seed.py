"""Seed PCP timing + agreement between the SVD and Gram SVT paths: python tools/time_seed.py s r rho"""
import os, sys, time, subprocess
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
s, r, rho = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
mt, _, _, _ = engine.generate_matrix(s, s, r, rho, 500.0, seed=0)
block = mt.double()
torch.cuda.synchronize(); t0 = time.time()
u, sg, v, seed_l, it = engine.recover_seed_device(block, l1pcp.AdmConfig(tol=1e-7))
torch.cuda.synchronize(); dt = time.time() - t0
print(f"s={s} r={r}: mode={os.environ.get('L1F_SEED_SVT','gram')} t={dt:.3f}s iters={it} r'={sg.shape[0]} sigma0={sg[0].item():.6e} sigma_last={sg[-1].item():.6e}")
np.save(f"gpurun_out/seed_l_{os.environ.get('L1F_SEED_SVT','gram')}_{s}.npy", seed_l.cpu().numpy())
