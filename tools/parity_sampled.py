"""Sampled-oracle parity of the full device solve at a BASELINE config (SURVEY 8(c')), at the
sample size the SURVEY names for config 5 (1000 rows x 1000 columns by default).  The oracle
(test infrastructure) solves the seed in FP64 with the reference's index draw and filters only
the sampled non-seed rows/columns, which gives L and S exactly on the sampled sub-block.

    python tools/parity_sampled.py <config> [rows] [cols]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import test_gpu_configs as tg  # noqa: E402
from oracle import philox_gen  # noqa: E402
from oracle import pipeline as opipe  # noqa: E402

c = int(sys.argv[1])
n_rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
n_cols = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
t0 = time.time()
cfg, mt, seed, out = tg._device_solve(c)
m, n, r = cfg["m"], cfg["n"], cfg["r"]
x, y = philox_gen.factors(0, cfg["kind"], m, n, r)


def block(rows, cols):
    return philox_gen.block(0, cfg["kind"], m, n, r, cfg["rho_s"], cfg["magnitude"], rows, cols, x=x,
                            y=y).astype(np.float64)


rng = np.random.default_rng(123)
rows = np.union1d(np.sort(rng.choice(m, n_rows, replace=False)), seed.row_idx[:5])
cols = np.union1d(np.sort(rng.choice(n, n_cols, replace=False)), seed.col_idx[:5])
t1 = time.time()
ref = opipe.sampled_blocks(m, n, block, r, rows, cols, 0, tol=tg.TOL)
t2 = time.time()
assert ref["kind"] == "seed" and ref["r_prime"] == seed.r_prime
ri = torch.as_tensor(rows, device="cuda")
ci = torch.as_tensor(cols, device="cuda")
l = out["l"][ri][:, ci].double().cpu().numpy()
s = out["s"][ri][:, ci].double().cpu().numpy()
same_m = np.array_equal(mt[ri][:, ci].cpu().numpy(), block(rows, cols).astype(np.float32))
print(f"config {c} ({m}x{n}, r={r}): sampled {rows.size} rows x {cols.size} cols "
      f"(incl. 5 seed rows / 5 seed cols); rel_F(L) {tg._rel(l, ref['l']):.3e}, rel_F(S) {tg._rel(s, ref['s']):.3e} "
      f"(gate 1e-4); device M bit-identical to the oracle regeneration: {same_m}; r' {seed.r_prime}; "
      f"device solve {t1 - t0:.1f} s, oracle {t2 - t1:.1f} s")
