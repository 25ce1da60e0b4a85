"""Probe the small-block seed kernels: time of one Jacobi SVD (cold) and the ALM sweeps."""
import sys, time, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _lib, engine
from paper_1108_5359_b200 import _device as dv
lib = _lib.load()
for s in (60, 100, 200, 256):
    a = torch.randn(s, s, dtype=torch.float64, device="cuda")
    u, sg, v = engine.svd_device(a)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3):
        u, sg, v = engine.svd_device(a)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
    ref = np.linalg.svd(a.cpu().numpy(), compute_uv=False)
    print(f"svd {s}x{s}: {dt*1e3:.2f} ms, max rel sigma err {np.abs(sg.cpu().numpy()-ref).max()/ref[0]:.2e}", flush=True)
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
import paper_1108_5359_b200 as l1pcp
for c in (1, 4):
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
    print(f"cfg{c}: t1 {t1:.3f} s, iters {seed.pcp_iterations}, sweeps {lib.l1f_diag_seed_small_sweeps()}", flush=True)
