"""Where the time of the numpy float64 public call goes (cfg3)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
cfg = BENCHMARK_CONFIGS[3]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0)
m_np = mt.double().cpu().numpy(); del mt; torch.cuda.empty_cache()
T = {}
t = time.perf_counter(); ok = np.isfinite(m_np).all(); T['isfinite'] = time.perf_counter() - t
t = time.perf_counter(); d = torch.from_numpy(m_np).cuda(); torch.cuda.synchronize(); T['h2d_pageable'] = time.perf_counter() - t
t = time.perf_counter(); h = d.cpu(); T['d2h_pageable_new'] = time.perf_counter() - t
t = time.perf_counter(); h2 = d.cpu(); T['d2h_pageable_new2'] = time.perf_counter() - t
out = np.empty_like(m_np)
t = time.perf_counter(); torch.from_numpy(out).copy_(d); T['d2h_into_numpy_fresh'] = time.perf_counter() - t
t = time.perf_counter(); torch.from_numpy(out).copy_(d); T['d2h_into_numpy_touched'] = time.perf_counter() - t
cfgf = l1pcp.FilterConfig(rank_hint=100, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
l1pcp.estimate_rank_and_solve(m_np[:2000, :2000], cfgf)
t = time.perf_counter(); sol = l1pcp.estimate_rank_and_solve(m_np, cfgf); T['public_call'] = time.perf_counter() - t
print({k: round(v, 3) for k, v in T.items()}, sol.stats)
