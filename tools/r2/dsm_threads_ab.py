import sys, time, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
for c in (2, 3, 5):
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    res = {}
    for mode in (1,):
        with _lib.options(seed_eig_dsm=mode):
            kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
        res.setdefault(mode, []).append(t1)
        print(f"cfg{c} dsm={mode} ({"256" if mode == 1 else "512"} threads): t1 {t1:.4f} s iters {seed.pcp_iterations} r' {seed.r_prime}", flush=True)
    del mt; torch.cuda.empty_cache()
