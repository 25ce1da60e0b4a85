"""Large-seed Gram eigensolver A/B: cuSOLVER syevd (seed_eig=1) vs the hand-written solver with the
L2-resident (seed_eig_dsm=0) or shared-memory-resident (1) tridiagonalisation: seed stage t1,
ALM iterations, r' and the seed L difference; eigensolver time alone."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
torch.manual_seed(0)
for p in ():
    a = torch.randn(p, 100, dtype=torch.float64, device="cuda") @ torch.randn(100, p, dtype=torch.float64, device="cuda")
    a += 0.0
    res = {}
    for mode in ((1, 1), (0, 0), (0, 1)):
        with _lib.options(seed_eig=mode[0], seed_eig_dsm=mode[1]):
            engine.svd_device(a, gram=True)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for _ in range(3): u, s, v = engine.svd_device(a, gram=True)
            torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
        res[mode] = (s[:110].cpu().numpy(), dt, (u[:, :100] * s[:100]) @ v[:, :100].T)
    ref = res[(1, 1)]
    for mode, (sg, dt, rec) in res.items():
        print(f"svd_gram p={p} mode={mode}: {dt*1e3:.2f} ms, sigma diff {np.abs(sg - ref[0]).max()/ref[0][0]:.2e}, rank-100 recon diff {float((rec-ref[2]).norm()/ref[2].norm()):.2e}", flush=True)
for c in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3,5").split(",")]:
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    out = {}
    for mode in ((1, 1), (0, 0), (0, 1)):
        with _lib.options(seed_eig=mode[0], seed_eig_dsm=mode[1]):
            for rep in range(2):
                kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
        out[mode] = seed
        print(f"cfg{c} mode={mode}: t1 {t1:.4f} s, iters {seed.pcp_iterations}, r' {seed.r_prime}", flush=True)
    base = out[(1, 1)]
    for mode, sd in out.items():
        lb, ls = base.seed_l, sd.seed_l
        try:
            print(f"   mode={mode} seed L rel diff {float((ls - lb).norm() / lb.norm()):.2e}", flush=True)
        except Exception as ex:
            print("   (no l_seed attr)", ex, flush=True)
    del mt
    torch.cuda.empty_cache()
