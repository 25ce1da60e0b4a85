"""Filter a subset of a config's real column-panel units with the TC and SIMT kernels (iteration check).
    python tools/debug_cfg_units.py <config> [n_units ...]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200 import _device as dv
from paper_1108_5359_b200.l1reg import filter_units
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS
from oracle import adm_filter
cfg = BENCHMARK_CONFIGS[int(sys.argv[1])]
mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0, kind=cfg["kind"])
fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
kind, seed, _, _ = engine.seed_stage(mt, fcfg)
plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm, want_e=False)
N = 4000
xc = torch.empty((N, len(plan.seed.row_idx)), dtype=torch.float32, device="cuda")
_lib.call("l1f_gather", dv.dtype_code(mt), dv.ptr(mt), mt.stride(0), dv.ptr(plan.d_row_idx), len(plan.seed.row_idx),
          dv.ptr(plan.d_comp_cols), N, _lib.F32, dv.ptr(xc), xc.stride(0), 1, dv.stream())
u = plan.u
print("dictionary", tuple(u.shape), u.dtype, "x absmax", xc.abs().max().item(), "x std", xc.std().item())
for n in [int(a) for a in sys.argv[2:]] or [200, 4000]:
    for mode in ("tc", "0"):
        os.environ["L1F_FILTER_TC"] = mode
        for scale in (1.0, 0.01):
            z, e, it, res, st = filter_units((xc[:n] * scale).contiguous(), u, plcfg := fcfg.adm) if False else filter_units((xc[:n] * scale).contiguous(), u, fcfg.adm)
            torch.cuda.synchronize()
            print(f"n={n} mode={mode} scale={scale}: iters mean {it.float().mean().item():.2f} max {it.max().item()} status {np.bincount(st.cpu().numpy(), minlength=4)}")
# oracle on 100 units
x64 = xc[:100].double().cpu().numpy().T
zr, er, itr, rr, sr = adm_filter.solve_units(x64, u.double().cpu().numpy(), 1e-7)
print("oracle 100 units: iters mean", itr.mean(), "max", itr.max())
# ---- swap ingredients
rng = np.random.default_rng(7)
q, _ = np.linalg.qr(rng.standard_normal((u.shape[0], u.shape[1])))
qs = torch.from_numpy(q.astype(np.float32)).cuda()
ureal = u.contiguous()
xs = (qs @ torch.randn(u.shape[1], 200, device="cuda") * 5).T.contiguous()
mask = torch.rand_like(xs) < 0.08
xs = xs + mask * (torch.rand_like(xs) * 400 - 200)
xr_real_u = (ureal @ torch.randn(u.shape[1], 200, device="cuda") * 5).T.contiguous() + mask * (torch.rand_like(xs) * 400 - 200)
for name, xx, aa in (("real x, synthetic Q", xc[:200].contiguous(), qs), ("synthetic x, synthetic Q", xs, qs),
                     ("synthetic x in span(U), real U", xr_real_u, ureal), ("real x, real U", xc[:200].contiguous(), ureal)):
    for mode in ("tc", "0"):
        os.environ["L1F_FILTER_TC"] = mode
        z, e, it, res, st = filter_units(xx, aa, fcfg.adm)
        torch.cuda.synchronize()
        print(f"{name:32s} mode={mode}: iters mean {it.float().mean().item():.2f}")
G = (ureal.T @ ureal).double()
print("U^T U - I max", (G - torch.eye(G.shape[0], device='cuda', dtype=G.dtype)).abs().max().item(), "U absmax", ureal.abs().max().item(),
      "stride", ureal.stride(), u.stride(), u.is_contiguous())
