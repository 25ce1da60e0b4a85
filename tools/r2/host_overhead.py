"""Host enqueue time vs device time of one solve_step (small configs are launch-bound)."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
l, s = torch.empty_like(mt), torch.empty_like(mt)
for _ in range(5): engine.solve_step(plan, mt, l, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50): engine.solve_step(plan, mt, l, s)
t_host = (time.perf_counter() - t0) / 50
torch.cuda.synchronize()
t_all = (time.perf_counter() - t0) / 50
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
print(f"cfg{c}: host enqueue {t_host*1e3:.3f} ms/step, wall {t_all*1e3:.3f} ms/step, s={len(seed.row_idx)}")
