"""A/B of the small-block ALM SVT: Gram + shared-memory tridiagonal (seed_small_svt=1) vs one-sided
Jacobi (0): L/S agreement, ALM iterations, rank, time; and the FP64 oracle on small shapes."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _lib, engine, pcp_adm
import paper_1108_5359_b200 as l1pcp
sys.path.insert(0, 'oracle')
rng = np.random.default_rng(0)
def case(m, n, r, rho=0.1):
    L0 = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    S0 = np.where(rng.random((m, n)) < rho, rng.uniform(-50, 50, (m, n)), 0.0)
    return L0 + S0
shapes = [(5, 3, 1), (3, 5, 1), (20, 20, 2), (40, 100, 4), (100, 40, 4), (100, 100, 10), (110, 110, 11), (113, 113, 11), (64, 200, 5)]
for (m, n, r) in shapes:
    M = torch.from_numpy(case(m, n, r)).cuda()
    cfg = pcp_adm.AdmConfig(tol=1e-7)
    out = {}
    for mode in (0, 1):
        with _lib.options(seed_small_svt=mode):
            l, s, info = pcp_adm.solve_pcp_device(M, cfg)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for _ in range(3): l, s, info = pcp_adm.solve_pcp_device(M, cfg)
            torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
        out[mode] = (l.cpu().numpy(), s.cpu().numpy(), info, dt)
    (l0, s0, i0, t0_), (l1, s1, i1, t1_) = out[0], out[1]
    dl = np.linalg.norm(l1 - l0) / max(np.linalg.norm(l0), 1e-300)
    print(f"{m}x{n} r{r}: jacobi it={i0['iterations']} rank={i0.get('rank')} {t0_*1e3:.2f} ms | gram it={i1['iterations']} rank={i1.get('rank')} {t1_*1e3:.2f} ms | relL {dl:.2e} maxS {np.abs(s1-s0).max():.2e}", flush=True)
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
for c in (1, 4):
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    for mode in (0, 1):
        with _lib.options(seed_small_svt=mode):
            for rep in range(2):
                torch.cuda.synchronize()
                kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
            print(f"cfg{c} mode{mode}: t1 {t1:.4f} s, iters {seed.pcp_iterations}, r' {seed.r_prime}, attempts {att}", flush=True)
