# debug: dump the m=500 acceptance instances and the drop-in's recovery error per seed
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
out = {}
for seed in range(5):
    spec = l1pcp.SynthSpec(m=500, n=500, rho_r=0.01, rho_s=0.01, rng_seed=seed)
    gt = l1pcp.generate(spec)
    sol = l1pcp.estimate_rank_and_solve(gt.m_obs, l1pcp.FilterConfig(rank_hint=5, rng_seed=seed))
    err = l1pcp.rel_err(sol.l, gt.l0)
    print(seed, err, sol.rank_of_l, sol.stats)
    out[f"m{seed}"] = gt.m_obs; out[f"l0{seed}"] = gt.l0; out[f"l{seed}"] = sol.l
np.savez_compressed("gpurun_out/m500.npz", **out)
