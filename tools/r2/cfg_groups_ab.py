"""tcgen05 filter: three vs two slot groups per CTA on a config's timed step (CUDA-graph replay)."""
import sys, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
l, s = torch.empty_like(mt), torch.empty_like(mt)
for groups in (0, 2, 0, 2):
    with _lib.options(tc_groups=groups):
        g = engine.CapturedStep(plan, mt, l, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): g.replay()
        b.record(); torch.cuda.synchronize()
        print(f"cfg{c} tc_groups={groups}: {a.elapsed_time(b)/20:.3f} ms/step", flush=True)
        del g
