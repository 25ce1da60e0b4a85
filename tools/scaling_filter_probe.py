"""Strong-scaling probe of the filter stage on one GPU: the per-rank unit counts of an N-GPU run of
a config (19000/N column + 19000/N row units at cfg3) timed with the paired call in each mode
(0: library choice, 1: one grid, 2: two grids).  Prints the per-rank filter time and the
filter-stage speed-up over N = 1 (ideal N).

    python tools/scaling_filter_probe.py [config]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.l1reg import filter_units_pair
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm, want_e=False)
ri = torch.as_tensor(seed.row_idx, device="cuda")
ci = torch.as_tensor(seed.col_idx, device="cuda")
xc_all = mt[ri][:, torch.as_tensor(plan.comp_cols, device="cuda")].T.contiguous()
xr_all = mt[torch.as_tensor(plan.comp_rows, device="cuda")][:, ci].contiguous()
u, v = plan.u, plan.v
base = {}
for n_gpus in (1, 2, 4, 8):
    nc, nr = xc_all.shape[0] // n_gpus, xr_all.shape[0] // n_gpus
    xc, xr = xc_all[:nc].contiguous(), xr_all[:nr].contiguous()
    line = f"N={n_gpus}: {nc} + {nr} units per rank;"
    for mode in (0, 1, 2):
        for _ in range(2):
            filter_units_pair(xc, u, xr, v, fcfg.adm, mode=mode)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            filter_units_pair(xc, u, xr, v, fcfg.adm, mode=mode)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        base.setdefault(mode, ms if n_gpus == 1 else base.get(mode))
        line += f"  mode {mode}: {ms:.3f} ms (x{base[mode] / ms:.2f})"
    print(line)
