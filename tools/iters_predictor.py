"""Can a unit's ADM iteration count be predicted before the solve?  For the cfg3 column units:
device iteration counts vs cheap features of x and its projection residual r0 = x - A A^T x.
(diagnostic)"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm, want_e=False)
f = engine.filter_stage(plan, mt)
it = f["iters_c"].cpu().numpy()
ri = torch.as_tensor(seed.row_idx, device="cuda")
x = mt[ri][:, torch.as_tensor(plan.comp_cols, device="cuda")].double()   # s x N
u = plan.u.double()
r0 = x - u @ (u.T @ x)
xinf = x.abs().max(0).values
feats = {
    "max|r0|/|x|inf": (r0.abs().max(0).values / xinf),
    "|r0|_2/|x|_2": (r0.norm(dim=0) / x.norm(dim=0)),
    "#(|r0| > 0.1|x|inf)": (r0.abs() > 0.1 * xinf).sum(0).double(),
    "#(|r0| > 0.01|x|inf)": (r0.abs() > 0.01 * xinf).sum(0).double(),
    "|x|inf": xinf,
    "|x|_1/|x|inf": x.abs().sum(0) / xinf,
    "|r0|_1/|r0|inf": r0.abs().sum(0) / r0.abs().max(0).values,
}
long = it >= 33
print(f"units {it.size}, long (>= 33 iterations) {long.mean():.3f}, mean iters {it.mean():.2f}")
for name, v in feats.items():
    v = v.cpu().numpy()
    cc = np.corrcoef(v, it)[0, 1]
    # how well does ranking by the feature put long units first?  fraction of long units in the top 'long' share
    order = np.argsort(-v)
    top = order[: long.sum()]
    order2 = np.argsort(v)
    top2 = order2[: long.sum()]
    print(f"{name:24s} corr {cc:+.3f}  long-unit precision in top (desc) {long[top].mean():.3f}  (asc) {long[top2].mean():.3f}")
