"""Seed-stage budget per config: t1, ALM iterations, r', and syevd time at the Gram sizes."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
for p in [100, 500, 1000, 2000]:
    g = torch.randn(p, p, dtype=torch.float64, device="cuda"); g = g @ g.T
    for _ in range(2): torch.linalg.eigh(g)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): torch.linalg.eigh(g)
    torch.cuda.synchronize(); print(f"eigh p={p}: {(time.perf_counter()-t0)/5*1e3:.2f} ms", flush=True)
for c in [int(x) for x in sys.argv[1].split(',')]:
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
        torch.cuda.synchronize(); el = time.perf_counter() - t0
        print(f"cfg{c} rep{rep}: t1={t1:.4f}s wall={el:.4f}s iters={seed.pcp_iterations} r'={seed.r_prime} attempts={att}", flush=True)
    del mt
    torch.cuda.empty_cache()
