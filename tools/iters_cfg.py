"""Per-filter iteration statistics of one config's device solve: python tools/iters_cfg.py <config>"""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
cfg = BENCHMARK_CONFIGS[int(sys.argv[1])]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm, want_e=False)
f = engine.filter_stage(plan, mt)
torch.cuda.synchronize()
tag = os.environ.get("L1F_FILTER_TC", "tc")
sig = seed.sigma.cpu().numpy()
print(f"[{tag}] sigma range {sig.min():.3g}..{sig.max():.3g}")
for side in ("c", "r"):
    it = f["iters_" + side].cpu().numpy(); st = f["status_" + side].cpu().numpy()
    print(f"[{tag}] {side}: mean {it.mean():.2f} max {it.max()} status {np.bincount(st, minlength=4)} p50 {np.median(it)}")
for side, x in (("c", None), ("r", None)):
    st = f["status_" + side].cpu().numpy()
    bad = np.flatnonzero((st == 1) | (st == 2))
    if bad.size:
        res = f["res_" + side].cpu().numpy()
        it = f["iters_" + side].cpu().numpy()
        print(f"[{tag}] {side}: failed units {bad[:10]} status {st[bad[:10]]} iters {it[bad[:10]]} res {res[bad[:10]]}")
