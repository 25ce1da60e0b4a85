import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, pcp_adm
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
cfg = BENCHMARK_CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
r = cfg["r"]
ri, ci = engine.sample_indices(cfg["m"], cfg["n"], 10 * r, 10 * r, np.random.SeedSequence(0).spawn(1)[0])
for rep in range(3):
    T = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    block = engine.gather(mt, ri, ci, out_dtype=torch.float64); torch.cuda.synchronize(); T['gather'] = time.perf_counter() - t0
    c2 = pcp_adm.AdmConfig(lam=pcp_adm.default_lambda(*block.shape), tol=1e-7)
    t0 = time.perf_counter(); l, s, info = pcp_adm.solve_pcp_device(block, c2); torch.cuda.synchronize(); T['pcp'] = time.perf_counter() - t0
    t0 = time.perf_counter(); u, sg, v = engine.svd_device(l, gram=True); torch.cuda.synchronize(); T['svd'] = time.perf_counter() - t0
    t0 = time.perf_counter(); out = engine.recover_seed_device(block, l1pcp.AdmConfig(tol=1e-7)); torch.cuda.synchronize(); T['recover'] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in T.items()}, info['iterations'], flush=True)
