"""Generate golden fixtures by running the REFERENCE implementation (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the unmodified reference package ``l1pcp`` from /root/reference/pkg/src, runs it
on small seeded inputs covering the hot path (l1reg._solve_block / solve_l1reg /
solve_l1reg_columnwise, recover_seed / solve_pcp, Nystrom completion + assemble,
estimate_rank_and_solve) and stores inputs and outputs as compressed .npz files next to
this script.  /root/reference does not exist on the GPU box; the fixtures travel instead.
"""

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import l1pcp  # noqa: E402  (the reference)
from l1pcp import l1reg, synth  # noqa: E402
from l1pcp.l1filter import (FilterConfig, FilterResult, SeedRecovery, assemble,  # noqa: E402
                            estimate_rank_and_solve, filter_columns, filter_rows, nystrom_complete,
                            recover_seed, sample_submatrix)
from l1pcp.matcore import svd  # noqa: E402
from l1pcp.pcp_adm import AdmConfig, solve_pcp, spectral_norm_estimate  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def orthonormal(rng, rows, cols):
    q, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
    return q


def cfg_dict(cfg):
    return dict(tol=cfg.tol, rho=cfg.rho, beta0=cfg.beta0, beta_max=cfg.beta_max, max_iter=cfg.max_iter)


def save(name, meta, **arrays):
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def l1reg_case(name, x, a, cfg, columnwise=False):
    sol = (l1reg.solve_l1reg_columnwise(x, a, cfg, parallelism=3) if columnwise
           else l1reg.solve_l1reg(x, a, cfg))
    # per-unit bookkeeping from the reference's own block solver
    z, e, iters, res, failed = l1reg._solve_block(np.ascontiguousarray(x, dtype=float), a, cfg)
    save(name, dict(cfg=cfg_dict(cfg), iterations=sol.iterations, final_residual=sol.final_residual,
                    converged=sol.converged, failed=sol.failed_columns, columnwise=columnwise),
         x=x, a=a, z=sol.z, e=sol.e, unit_iters=iters, unit_res=res)


def main():
    print("reference l1pcp", l1pcp.__version__, "numpy", np.__version__)
    # ---- l1 regression (l1reg.py) ------------------------------------------------
    rng = np.random.default_rng(0)
    a = orthonormal(rng, 50, 4)
    l1reg_case("l1reg_exact_fit", a @ rng.standard_normal((4, 7)), a, AdmConfig())

    rng = np.random.default_rng(1)
    a = orthonormal(rng, 200, 5)
    x = a @ rng.standard_normal((5, 30))
    idx = rng.choice(200 * 30, size=300, replace=False)
    x.flat[idx] += rng.uniform(-100, 100, size=300)
    l1reg_case("l1reg_spiked", x, a, AdmConfig(tol=1e-9))

    a = np.zeros((8, 1)); a[0, 0] = 1.0
    x = np.zeros((8, 1)); x[0, 0] = 10.0; x[1, 0] = 3.0
    l1reg_case("l1reg_hand", x, a, AdmConfig(tol=1e-10))

    rng = np.random.default_rng(2)
    a = orthonormal(rng, 120, 6)
    x = a @ rng.standard_normal((6, 90))
    x.flat[rng.choice(x.size, 200, replace=False)] += rng.uniform(-50, 50, 200)
    l1reg_case("l1reg_columnwise", x, a, AdmConfig(), columnwise=True)

    rng = np.random.default_rng(8)
    a = orthonormal(rng, 40, 3)
    x = a @ rng.standard_normal((3, 6))
    x.flat[rng.choice(x.size, 20, replace=False)] += rng.uniform(-5, 5, 20)
    l1reg_case("l1reg_failed", x, a, AdmConfig(tol=1e-12, max_iter=2))

    # a config-1-shaped panel: s = 100, k = 10, 10% corruption of magnitude 500, zero units
    rng = np.random.default_rng(11)
    a = orthonormal(rng, 100, 10)
    x = a @ (rng.standard_normal((10, 160)) * 10.0)
    mask = rng.random(x.shape) < 0.10
    x[mask] += rng.uniform(-500, 500, size=mask.sum())
    x[:, [7, 71]] = 0.0
    l1reg_case("l1reg_cfg1_panel", x, a, AdmConfig(tol=1e-7))

    # ---- seed PCP (pcp_adm.py, recover_seed) -------------------------------------
    rng = np.random.default_rng(2)
    block = rng.standard_normal((60, 2)) @ rng.standard_normal((60, 2)).T
    seed = recover_seed(block, AdmConfig(tol=1e-9))
    save("seed_clean_rank2", dict(r_prime=seed.r_prime, pcp_iterations=seed.pcp_iterations, tol=1e-9),
         block=block, seed_l=seed.seed_l, sigma=seed.seed_svd.sigma)

    gt = synth.generate(synth.SynthSpec(m=100, n=100, rho_r=0.05, rho_s=0.05, rng_seed=4))
    seed = recover_seed(gt.m_obs, AdmConfig(tol=1e-9))
    save("seed_corrupt_rank5", dict(r_prime=seed.r_prime, pcp_iterations=seed.pcp_iterations, tol=1e-9),
         block=gt.m_obs, seed_l=seed.seed_l, sigma=seed.seed_svd.sigma, l0=gt.l0)

    gt = synth.generate(synth.SynthSpec(m=80, n=60, rho_r=0.05, rho_s=0.03, rng_seed=1))
    sol = solve_pcp(gt.m_obs)
    save("pcp_rect", dict(iterations=sol.iterations, final_residual=sol.final_residual, rank=sol.rank_of_l,
                          converged=sol.converged, spectral=spectral_norm_estimate(gt.m_obs)),
         m=gt.m_obs, l=sol.l, s=sol.s)

    # ---- Nystrom completion + assembly (l1filter.py:137-167) ----------------------
    rng = np.random.default_rng(6)
    l0 = rng.standard_normal((80, 3)) @ rng.standard_normal((70, 3)).T
    ri, ci, blk = sample_submatrix(l0, 30, 30, rng)
    f = svd(blk)
    seed = SeedRecovery(row_idx=ri, col_idx=ci, seed_svd=f, seed_l=f.reconstruct(), seed_s=blk - f.reconstruct(),
                        r_prime=f.rank)
    comp_r = np.setdiff1d(np.arange(80), ri)
    comp_c = np.setdiff1d(np.arange(70), ci)
    q, s_c, _ = filter_columns(l0[np.ix_(ri, comp_c)], f.u, AdmConfig(tol=1e-10))
    p, s_r, _ = filter_rows(l0[np.ix_(comp_r, ci)], f.v, AdmConfig(tol=1e-10))
    fr = FilterResult(q_tilde=q, p_tilde=p, s_col=s_c, s_row=s_r)
    comp = nystrom_complete(seed, fr)
    l_hat = assemble(seed, fr, comp, 80, 70)
    save("nystrom_exact", dict(r_prime=f.rank), l0=l0, row_idx=ri, col_idx=ci, u=f.u, sigma=f.sigma, v=f.v,
         q=q, p=p, completion=comp, l_hat=l_hat)

    # ---- full pipeline (estimate_rank_and_solve) ----------------------------------
    # inputs are regenerated by oracle/ref_synth.py (a restatement of synth.generate) and
    # pinned by their sha256; only the reference's outputs are stored
    for name, spec, cfg in (
        ("pipeline_hint", synth.SynthSpec(m=300, n=300, rho_r=0.01, rho_s=0.01, rng_seed=0),
         FilterConfig(rank_hint=3, rng_seed=0)),
        ("pipeline_rect_norank", synth.SynthSpec(m=240, n=200, rho_r=0.01, rho_s=0.02, rng_seed=5),
         FilterConfig(rng_seed=3)),
        ("pipeline_tol7", synth.SynthSpec(m=300, n=300, rho_r=0.01, rho_s=0.05, rng_seed=7),
         FilterConfig(rank_hint=3, rng_seed=1, adm=AdmConfig(tol=1e-7))),
    ):
        gt = synth.generate(spec)
        sol = estimate_rank_and_solve(gt.m_obs, cfg)
        st = {k: (v if not isinstance(v, tuple) else list(v)) for k, v in sol.stats.items()
              if not k.startswith("t")}
        save(name, dict(method=sol.method, rank=sol.rank_of_l, iterations=sol.iterations,
                        final_residual=sol.final_residual, stats=st, rank_hint=cfg.rank_hint, rng_seed=cfg.rng_seed,
                        tol=cfg.adm.tol, rel_err=synth.rel_err(sol.l, gt.l0),
                        spec=dict(m=spec.m, n=spec.n, rho_r=spec.rho_r, rho_s=spec.rho_s, magnitude=spec.magnitude,
                                  sigma_scale=spec.sigma_scale, rng_seed=spec.rng_seed),
                        m_sha256=hashlib.sha256(np.ascontiguousarray(gt.m_obs).tobytes()).hexdigest(),
                        l0_sha256=hashlib.sha256(np.ascontiguousarray(gt.l0).tobytes()).hexdigest()),
             l=sol.l)

    sol = estimate_rank_and_solve(np.zeros((50, 50)), FilterConfig(rng_seed=0))
    save("pipeline_zero", dict(method=sol.method, rank=sol.rank_of_l, iterations=sol.iterations), m=np.zeros((50, 50)))


if __name__ == "__main__":
    main()
