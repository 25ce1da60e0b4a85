"""Per-unit iteration counts of the device filter vs the oracle replayed in FP64 and FP32 on the
same sampled units of one config (diagnostic; the oracle is test infrastructure).

    python tools/iters_vs_oracle.py <config> [units]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from oracle import adm_filter
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS

cfg = BENCHMARK_CONFIGS[int(sys.argv[1])]
nu = int(sys.argv[2]) if len(sys.argv) > 2 else 256
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm, want_e=False)
f = engine.filter_stage(plan, mt)
torch.cuda.synchronize()
it_dev = f["iters_c"].cpu().numpy()
st_dev = f["status_c"].cpu().numpy()
rng = np.random.default_rng(0)
pick = np.sort(rng.choice(len(plan.comp_cols), size=min(nu, len(plan.comp_cols)), replace=False))
cols = np.asarray(plan.comp_cols)[pick]
x = mt[torch.as_tensor(np.asarray(seed.row_idx), device="cuda")][:, torch.as_tensor(cols, device="cuda")]
x = x.double().cpu().numpy()
u = plan.u.double().cpu().numpy() if hasattr(plan.u, "cpu") else np.asarray(plan.u, dtype=np.float64)
for name, dt in (("fp64", np.float64), ("fp32", np.float32)):
    _, _, it, res, st = adm_filter.solve_units(x, u, 1e-7, dtype=dt)
    d = it_dev[pick].astype(np.int64) - it
    print(f"{name}: oracle mean {it.mean():.2f} p50 {np.median(it)} max {it.max()} status {np.bincount(st, minlength=4)}"
          f" | device mean {it_dev[pick].mean():.2f} max {it_dev[pick].max()} status {np.bincount(st_dev[pick], minlength=4)}"
          f" | device - oracle: mean {d.mean():.2f} min {d.min()} max {d.max()}")
    print(f"  oracle iteration histogram {np.bincount(it, minlength=41)[10:41]}")
print(f"  device iteration histogram {np.bincount(it_dev[pick], minlength=41)[10:41]}")
print(f"  device (all column units) mean {it_dev.mean():.2f}, histogram {np.bincount(it_dev, minlength=41)[10:41]}")
