"""Per-unit filter parity on the benchmark configs: device (pipeline) vs the FP64 oracle on the
same panels and the same (device) seed factors.  Prints status agreement, iteration deltas,
per-unit relative L error and the FP64-recomputed residual of the device's own (z, e)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.l1reg import filter_units
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
from oracle import adm_filter

TOL = 1e-7
cfgs = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [2, 3, 4]
nsample = int(sys.argv[2]) if len(sys.argv) > 2 else 0
summary = {}
for c in cfgs:
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=TOL))
    kind, seed, _, _ = engine.seed_stage(mt, fcfg)
    plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
    out = engine.solve_from_seed(mt, plan)
    torch.cuda.synchronize()
    fdt = plan.filter_dtype
    res = {}
    for side in ("c", "r"):
        if side == "c":
            units = plan.comp_cols
            xd = engine.gather(mt, seed.row_idx, units, out_dtype=fdt, transpose=True)   # (N, s)
            A = seed.u
        else:
            units = plan.comp_rows
            xd = engine.gather(mt, units, seed.col_idx, out_dtype=fdt)                 # (N, s)
            A = seed.v
        it_d = out["iters_" + side].cpu().numpy(); st_d = out["status_" + side].cpu().numpy()
        z_pipe = out["z" + side].double().cpu().numpy()
        # e from a want_e call on the same panel (per-unit arithmetic is call-independent)
        ze, ee, it_e, _, st_e = filter_units(xd, A.to(fdt).contiguous(), fcfg.adm, want_e=True)
        z_e = ze.double().cpu().numpy(); e_e = ee.double().cpu().numpy()
        N = len(units)
        sel = np.arange(N)
        if nsample and N > nsample:
            rng = np.random.default_rng(1)
            flagged = np.flatnonzero(st_d != 0)
            sel = np.union1d(np.sort(rng.choice(N, nsample, replace=False)), flagged)
        x64 = xd.double().cpu().numpy()[sel]                                        # (n, s)
        a64 = A.double().cpu().numpy()
        t0 = time.time()
        zo, eo, ito, reso, sto = adm_filter.solve_units(x64.T, a64, TOL)
        t_or = time.time() - t0
        zo = zo.T; eo = eo.T
        scale = np.abs(x64).max(axis=1)
        lc_d = z_pipe[sel] @ a64.T; lc_o = zo @ a64.T
        rel_l = np.linalg.norm(lc_d - lc_o, axis=1) / np.maximum(np.linalg.norm(lc_o, axis=1), 1e-300)
        r64 = x64 - z_e[sel] @ a64.T - e_e[sel]
        resid_ratio = np.abs(r64).max(axis=1) / np.maximum(TOL * scale, 1e-300)
        dit = it_d[sel] - ito
        ok = (st_d[sel] == 0)
        bitwise_e = bool(np.array_equal(z_e, z_pipe)) and bool(np.array_equal(it_e.cpu().numpy(), it_d))
        r = dict(N=int(N), checked=int(sel.size), oracle_s=round(t_or, 1),
                 status_dev=np.bincount(st_d[sel], minlength=4).tolist(), status_or=np.bincount(sto, minlength=4).tolist(),
                 status_mismatch=int((st_d[sel] != sto).sum()),
                 dit_min=int(dit.min()), dit_max=int(dit.max()), dit_mean=float(dit.mean()),
                 dit_hist={int(k): int(v) for k, v in zip(*np.unique(np.clip(dit, -20, 20), return_counts=True))},
                 rel_l_max=float(rel_l.max()), rel_l_max_ok=float(rel_l[ok].max() if ok.any() else 0),
                 rel_l_p99=float(np.quantile(rel_l, 0.99)),
                 resid_ratio_max_ok=float(resid_ratio[ok].max() if ok.any() else 0),
                 resid_ratio_p99_ok=float(np.quantile(resid_ratio[ok], 0.99) if ok.any() else 0),
                 n_resid_over_1001=int((resid_ratio[ok] > 1.001).sum()),
                 pipeline_eq_want_e=bitwise_e,
                 worst_units=[int(u) for u in sel[np.argsort(-np.abs(dit))[:10]]])
        res[side] = r
        print(f"cfg{c} {side}: {json.dumps(r)}", flush=True)
    summary[f"cfg{c}"] = res
    del mt, out
    torch.cuda.empty_cache()
json.dump(summary, open(f"gpurun_out/unit_parity_{'_'.join(map(str, cfgs))}.json", "w"), indent=1)
