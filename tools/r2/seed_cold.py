"""t1 of the first seed stage in a fresh process (as bench.py measures it) and of a second call."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1])
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
torch.cuda.synchronize()
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
out = []
for rep in range(2):
    kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
    out.append(t1)
print(f"cfg{c}: t1 cold {out[0]:.4f} s, warm {out[1]:.4f} s, iters {seed.pcp_iterations}, r' {seed.r_prime}", flush=True)
