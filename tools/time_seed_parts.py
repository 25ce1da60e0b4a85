"""Break the seed stage time into PCP loop / final SVD / rest: python tools/time_seed_parts.py <config>"""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.pcp_adm import solve_pcp_device, default_lambda, AdmConfig
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
cfg = BENCHMARK_CONFIGS[int(sys.argv[1])]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
s_r = 10 * cfg["r"]
ri, ci = engine.sample_indices(cfg["m"], cfg["n"], s_r, s_r, np.random.SeedSequence(0).spawn(1)[0])
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    block = engine.gather(mt, ri, ci, out_dtype=torch.float64)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    lam = default_lambda(*block.shape)
    l, _, info = solve_pcp_device(block, AdmConfig(lam=lam, tol=1e-7))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    u, s, v = engine.svd_device(l)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"rep {rep}: gather {1e3*(t1-t0):.1f} ms  pcp {1e3*(t2-t1):.1f} ms ({info['iterations']} it, {1e3*(t2-t1)/info['iterations']:.1f} ms/it)  svd {1e3*(t3-t2):.1f} ms")
