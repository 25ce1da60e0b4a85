"""Potential of running the row filter concurrently with the column filter (two streams: the row
filter's clusters start as the column filter's clusters exit) against the two launches in series.
cfg3 panels, FP32 tensor-core filter, no reconstruction."""
import sys, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.l1reg import filter_units
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
xc = engine.gather(mt, seed.row_idx, plan.comp_cols, out_dtype=torch.float32, transpose=True)
xr = engine.gather(mt, plan.comp_rows, seed.col_idx, out_dtype=torch.float32)
u, v = plan.u, plan.v
ws2 = torch.empty_like(plan.workspace) if plan.workspace is not None else None
s2 = torch.cuda.Stream()
def serial():
    filter_units(xc, u, fcfg.adm, want_e=False, workspace=plan.workspace)
    filter_units(xr, v, fcfg.adm, want_e=False, workspace=ws2)
def concurrent():
    filter_units(xc, u, fcfg.adm, want_e=False, workspace=plan.workspace)
    s2.wait_stream(torch.cuda.current_stream()) if False else None
    with torch.cuda.stream(s2):
        filter_units(xr, v, fcfg.adm, want_e=False, workspace=ws2)
    torch.cuda.current_stream().wait_stream(s2)
for name, fn in (("serial", serial), ("concurrent", concurrent), ("serial", serial), ("concurrent", concurrent)):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): fn()
    b.record(); torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 5:.3f} ms", flush=True)
