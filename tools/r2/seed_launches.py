"""One seed stage (hand-written eigensolver) of a config, for an ncu launch list."""
import sys, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
if len(sys.argv) > 2: _lib.load(sys.argv[2])
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1])
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
torch.cuda.synchronize()
with _lib.options(seed_eig=0, seed_eig_dsm=1):
    kind, seed, att, t1 = engine.seed_stage(mt, fcfg)
torch.cuda.synchronize()
print("t1", t1)
