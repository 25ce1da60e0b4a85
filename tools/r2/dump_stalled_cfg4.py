"""Dump the cfg4 row units the FP64 small-k kernel marks stalled (x, V) and the device's per-
iteration residual trajectory (max_iter sweep) for offline analysis."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.l1reg import filter_units
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
cfg = BENCHMARK_CONFIGS[4]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
out = engine.solve_from_seed(mt, plan)
st = out["status_r"].cpu().numpy()
bad = np.flatnonzero(st != 0)
rows = plan.comp_rows[bad]
x = engine.gather(mt, rows, seed.col_idx, out_dtype=torch.float64)
v = seed.v.contiguous()
traj = []
for t in range(1, 80):
    _, _, it, res, stt = filter_units(x, v, l1pcp.AdmConfig(tol=1e-7, max_iter=t), want_e=False)
    traj.append(res.cpu().numpy())
np.savez("gpurun_out/stalled_cfg4.npz", x=x.cpu().numpy(), v=v.cpu().numpy(), rows=rows,
         iters=out["iters_r"].cpu().numpy()[bad], traj=np.array(traj))
print(len(bad), out["iters_r"].cpu().numpy()[bad])
