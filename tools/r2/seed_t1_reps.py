"""Steady-state t1 (seed stage) per config: five solves after one warm-up, median reported."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
for c in [int(x) for x in sys.argv[1].split(',')]:
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    engine.seed_stage(mt, fcfg)
    ts = [engine.seed_stage(mt, fcfg)[3] for _ in range(5)]
    print(f"cfg{c}: t1 median {np.median(ts):.4f} s, runs {[round(t, 4) for t in ts]}", flush=True)
    del mt; torch.cuda.empty_cache()
