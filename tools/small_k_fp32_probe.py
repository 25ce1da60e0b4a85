"""cfg4 / cfg1 (k <= 16): the small-k filter in FP32 instead of FP64 — time of the step and
agreement of L with the FP64 filter's L (relative Frobenius), iteration counts, failed units.

    python tools/small_k_fp32_probe.py [config]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1108_5359_b200 as l1pcp  # noqa: E402
from paper_1108_5359_b200 import engine  # noqa: E402
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = BENCHMARK_CONFIGS[c]
m, n, r = cfg["m"], cfg["n"], cfg["r"]
mt, _, _, _ = engine.generate_matrix(m, n, r, cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
out = {}
for thr in (16, 0):
    engine.SMALL_K_FP64 = thr
    plan = engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)
    l_out, s_out = torch.empty_like(mt), torch.empty_like(mt)
    for _ in range(3):
        f = engine.solve_step(plan, mt, l_out, s_out)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(10)]
    for e in evs:
        f = engine.solve_step(plan, mt, l_out, s_out, e)
    torch.cuda.synchronize()
    step = sum(e[0].elapsed_time(e[4]) for e in evs) / 10
    filt = sum(e[1].elapsed_time(e[2]) for e in evs) / 10
    it = (f["iters_c"].double().sum() + f["iters_r"].double().sum()).item() / (f["iters_c"].numel() + f["iters_r"].numel())
    failed = int(((f["status_c"] == 1) | (f["status_c"] == 2)).sum() + ((f["status_r"] == 1) | (f["status_r"] == 2)).sum())
    name = "fp64" if thr else "fp32"
    out[name] = l_out.clone()
    print(f"cfg{c} filter {name} ({plan.filter_dtype}): step {step:.3f} ms, filters {filt:.3f} ms, mean iters {it:.2f}, "
          f"max {max(int(f['iters_c'].max()), int(f['iters_r'].max()))}, failed {failed}", flush=True)
d = torch.linalg.norm((out["fp32"] - out["fp64"]).double()) / torch.linalg.norm(out["fp64"].double())
print(f"rel_F(L_fp32 - L_fp64) = {d.item():.3e}")
