"""A/B of the k <= 10 FP64 filter variants on the cfg4 panels (column + row units)."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
if len(sys.argv) > 3: _lib.load(sys.argv[3])
from paper_1108_5359_b200.l1reg import filter_units
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = BENCHMARK_CONFIGS[c]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
xc = engine.gather(mt, seed.row_idx, plan.comp_cols, out_dtype=torch.float64, transpose=True)
xr = engine.gather(mt, plan.comp_rows, seed.col_idx, out_dtype=torch.float64)
u, v = plan.u, plan.v
ref = None
for lanes in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,16,32").split(",")]:
    with _lib.options(small_lanes=lanes):
        for _ in range(2):
            out_c = filter_units(xc, u, fcfg.adm, want_e=False)
            out_r = filter_units(xr, v, fcfg.adm, want_e=False)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            out_c = filter_units(xc, u, fcfg.adm, want_e=False)
            out_r = filter_units(xr, v, fcfg.adm, want_e=False)
        b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    its = (out_c[2].double().sum() + out_r[2].double().sum()).item()
    flops = its * 100 * (4 * seed.r_prime + 12)
    same = None
    if ref is None:
        ref = (out_c[0].clone(), out_r[0].clone(), out_c[2].clone(), out_r[2].clone())
    else:
        same = bool(torch.equal(ref[2], out_c[2]) and torch.equal(ref[3], out_r[2]))
        zdiff = max((ref[0] - out_c[0]).abs().max().item(), (ref[1] - out_r[0]).abs().max().item())
    print(f"lanes={lanes}: {ms:.3f} ms (cols+rows), {flops/ms/1e9:.2f} TFLOP/s algorithmic, same iters {same}" + ("" if same is None else f", max |dz| {zdiff:.2e}"), flush=True)
