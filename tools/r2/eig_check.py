"""Hand-written Gram eigensolver (eig_sym.cu) vs cuSOLVER syevd: l1f_svd_gram_f64 on low-rank +
noise matrices, and the seed stage (t1, iterations, r', seed L) of configs 2, 3, 5 with both."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
torch.manual_seed(0)
for (m, n, r) in [(600, 500, 20), (1200, 1000, 100)]:
    a = torch.randn(m, r, dtype=torch.float64, device="cuda") @ torch.randn(r, n, dtype=torch.float64, device="cuda")
    a += 1e-3 * torch.randn(m, n, dtype=torch.float64, device="cuda")
    out = {}
    for opt in (1, 0):
        with _lib.options(seed_eig=opt):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            u, s, v = engine.svd_device(a, gram=True)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        out[opt] = (u, s, v, dt)
    ref = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    for opt in (1, 0):
        u, s, v, dt = out[opt]
        k = r + 5
        sk = s[:k].cpu().numpy()
        rec = (u[:, :r] * s[:r]) @ v[:, :r].T
        lr = (torch.linalg.svd(a)[0][:, :r] * torch.linalg.svd(a)[1][:r]) @ torch.linalg.svd(a)[2][:r]
        print(f"{m}x{n} r={r} seed_eig={opt}: {dt*1e3:.1f} ms, max rel sigma err (top {k}) "
              f"{np.abs(sk - ref[:k]).max() / ref[0]:.2e}, rank-{r} recon vs exact {float((rec - lr).norm() / lr.norm()):.2e}, "
              f"U orth {float((u[:, :r].T @ u[:, :r] - torch.eye(r, device='cuda', dtype=torch.float64)).abs().max()):.1e}", flush=True)
for c in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3").split(",")]:
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    res = {}
    for opt in (1, 0, 0):
        with _lib.options(seed_eig=opt):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
            torch.cuda.synchronize()
        res[opt] = seed
        print(f"cfg{c} seed_eig={opt}: t1 {t1:.3f} s, iterations {seed.pcp_iterations}, r' {seed.r_prime}, attempts {att}", flush=True)
    d = float((res[0].seed_l - res[1].seed_l).norm() / res[1].seed_l.norm())
    print(f"cfg{c}: seed L rel diff hand-written vs syevd {d:.2e}", flush=True)
    del mt
    torch.cuda.empty_cache()
