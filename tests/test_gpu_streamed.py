"""GPU: the overlapped row filter + reconstruction (l1f_rowfilter_reconstruct_f32) equals the
separate calls bitwise.

engine.solve_step runs the column filter, builds Bf, then the row filter with the
reconstruction of each 128-row strip streamed beside it (work items claimed at run time, the
strip's Af rows built and split by the CTA that claims its first item).  The per-unit filter
arithmetic and the per-entry reconstruction are those of l1f_filter_f32 + l1f_build_factors +
l1f_reconstruct, so Zr, the unit statistics, L and S must be identical — with the concurrent
launch on, off (all strips after the filter), ragged strips, dead (all-zero) row units and the
large-k (TA filter, 4-stage reconstruction) variant.
"""

import os

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import _lib, engine

pytestmark = pytest.mark.gpu


def _solve(mt, plan, streamed, concurrent=True):
    old = engine._streamed_ok
    try:
        engine._streamed_ok = (lambda p, t: True) if streamed else (lambda p, t: False)
        with _lib.options(recon_concurrent=1 if concurrent else 0):
            f = engine.solve_step(plan, mt)
            torch.cuda.synchronize()
    finally:
        engine._streamed_ok = old
    assert f["streamed"] == streamed
    return f


def _plan(mt, r, zero_rows=0):
    m, n = mt.shape
    fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    kind, seed, _, _ = engine.seed_stage(mt, fcfg)
    assert kind == "seed"
    if zero_rows:  # after the seed: rows whose seed-column entries are all zero -> dead row units
        comp = np.setdiff1d(np.arange(m), seed.row_idx)[:zero_rows]
        ci = torch.as_tensor(seed.col_idx, device="cuda")
        for i in comp:
            mt[int(i), ci] = 0.0
    return engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)


@pytest.mark.parametrize("m,n,r,concurrent,zero_rows", [
    (6000, 5000, 40, True, 0),
    (6000, 5000, 40, False, 0),
    (4133, 3004, 30, True, 7),     # ragged strips and column tiles, dead row units
    (5200, 4700, 100, True, 0),    # three slot groups at k = 100, the cfg3 shape class
])
def test_streamed_matches_separate_calls(m, n, r, concurrent, zero_rows):
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=11)
    plan = _plan(mt, r, zero_rows)
    ref = _solve(mt, plan, streamed=False)
    for _ in range(2):  # repeated calls reuse the side stream and its events
        got = _solve(mt, plan, streamed=True, concurrent=concurrent)
        assert torch.equal(got["zr"], ref["zr"])
        assert torch.equal(got["iters_r"], ref["iters_r"])
        assert torch.equal(got["status_r"], ref["status_r"])
        assert torch.equal(got["zc"], ref["zc"])
        assert torch.equal(got["l"], ref["l"])
        assert torch.equal(got["s"], ref["s"])
        r_ref = ref["resid_sq"].cpu().numpy()
        np.testing.assert_allclose(got["resid_sq"].cpu().numpy(), r_ref, rtol=1e-12, atol=1e-12 * r_ref[1])
    if zero_rows:
        assert int((got["status_r"] == 3).sum().item()) >= zero_rows


def test_streamed_large_k():
    """k = 200: the TA filter variant (clusters of 16) and the 4-stage reconstruction (KJ = 7)."""
    m, n, r = 4400, 4000, 200
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=5)
    plan = _plan(mt, r)
    ref = _solve(mt, plan, streamed=False)
    got = _solve(mt, plan, streamed=True)
    assert torch.equal(got["zr"], ref["zr"])
    assert torch.equal(got["l"], ref["l"])
    assert torch.equal(got["s"], ref["s"])


def test_streamed_policy_and_public_api():
    """The public estimate_rank_and_solve (whichever path the library's pass model picks)
    reports t2 / t_assemble and matches the separate calls."""
    m = n = 12000
    r = 60
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=2)
    plan = _plan(mt, r)
    ref = _solve(mt, plan, streamed=False)
    sol = l1pcp.estimate_rank_and_solve(mt, l1pcp.FilterConfig(rank_hint=r, rng_seed=0,
                                                                adm=l1pcp.AdmConfig(tol=1e-7)))
    assert torch.equal(sol.l, ref["l"])
    assert torch.equal(sol.s, ref["s"])
    assert sol.stats["t2"] > 0 and sol.stats["t_assemble"] >= 0


@pytest.mark.parametrize("m,n,r", [
    (600, 520, 17),     # five strips (the last partial), one column-tile item per strip
    (1200, 1000, 30),   # s_r = 300 of 1200 rows: strips with more than 32 seed rows (the scan path)
    (4200, 4000, 130),  # k = 130: one slot group (KP 160), 4-stage reconstruction (KJ2 = 3)
])
def test_streamed_shapes(m, n, r):
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=9)
    plan = _plan(mt, r)
    ref = _solve(mt, plan, streamed=False)
    got = _solve(mt, plan, streamed=True)
    assert torch.equal(got["zr"], ref["zr"])
    assert torch.equal(got["l"], ref["l"])
    assert torch.equal(got["s"], ref["s"])


def test_streamed_library_refusal_falls_back(monkeypatch):
    """If the library declines the overlapped calls (here: the recon_stream / gather_overlap options
    switched off underneath a forced streamed plan) solve_step falls back to the separate calls."""
    m, n, r = 3000, 2800, 40
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=12)
    plan = _plan(mt, r)
    ref = _solve(mt, plan, streamed=False)
    with _lib.options(recon_stream=0, gather_overlap=0):
        got = _solve(mt, plan, streamed=True)
    assert torch.equal(got["l"], ref["l"]) and torch.equal(got["s"], ref["s"])


def _solve_small(mt, plan, streamed, concurrent=True):
    old = engine._streamed_small_ok
    try:
        engine._streamed_small_ok = (lambda p, t: True) if streamed else (lambda p, t: False)
        with _lib.options(recon_concurrent=1 if concurrent else 0):
            f = engine.solve_step(plan, mt)
            torch.cuda.synchronize()
    finally:
        engine._streamed_small_ok = old
    return f


@pytest.mark.parametrize("m,n,r,concurrent,kind", [
    (6000, 3000, 10, True, 0),
    (6000, 3000, 10, False, 0),
    (4100, 2050, 3, True, 0),     # ragged strips and 512-column chunks, KM = 4
    (5000, 2600, 16, True, 0),
    (7680, 1000, 10, True, 1),    # video kind (moving boxes), the cfg4 statistics
])
def test_streamed_small_k_matches_separate_calls(m, n, r, concurrent, kind):
    """k <= 16: the FP64 small-k filter with the SIMT reconstruction beside it
    (l1f_rowfilter_reconstruct_small) equals the separate calls bitwise."""
    from paper_1108_5359_b200 import _lib
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 255.0 if kind else 500.0, seed=13,
                                         kind=_lib.GEN_VIDEO if kind else _lib.GEN_GAUSSIAN)
    plan = _plan(mt, r)
    assert plan.filter_dtype == torch.float64
    ref = _solve_small(mt, plan, streamed=False)
    for _ in range(2):
        got = _solve_small(mt, plan, streamed=True, concurrent=concurrent)
        assert got.get("streamed")
        assert torch.equal(got["zr"], ref["zr"])
        assert torch.equal(got["iters_r"], ref["iters_r"])
        assert torch.equal(got["l"], ref["l"])
        assert torch.equal(got["s"], ref["s"])
        r_ref = ref["resid_sq"].cpu().numpy()  # sum(M^2): fp32 partials grouped differently
        np.testing.assert_allclose(got["resid_sq"].cpu().numpy(), r_ref, rtol=1e-6, atol=1e-6 * r_ref[1])


@pytest.mark.parametrize("max_iter,beta0,beta_max", [(3, None, None), (25, 0.05, 50.0)])
def test_streamed_iteration_limits_and_explicit_beta(max_iter, beta0, beta_max):
    """Units that stop at max_iter and explicit beta0 / beta_max: the overlapped path counts every
    finished unit the same way (status MAXITER included) and matches the separate calls."""
    m, n, r = 3000, 2800, 40
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=21)
    plan = _plan(mt, r)
    plan.adm = l1pcp.AdmConfig(tol=1e-7, max_iter=max_iter, beta0=beta0, beta_max=beta_max)
    ref = _solve(mt, plan, streamed=False)
    got = _solve(mt, plan, streamed=True)
    assert torch.equal(got["iters_r"], ref["iters_r"])
    assert torch.equal(got["status_r"], ref["status_r"])
    assert torch.equal(got["l"], ref["l"]) and torch.equal(got["s"], ref["s"])
    if max_iter == 3:
        assert int((got["status_r"] == 2).sum().item()) > 0


def test_wait_timeout_recomputes_step():
    """A timed-out device wait of the overlapped row filter + reconstruction (forced here with a
    zero bound, so every wait that is not already satisfied gives up) leaves a NaN residual; the
    public call recomputes the step with the separate calls and returns the same L and S (ADVICE r1:
    recon_tc.cu wait_geq)."""
    m, n, r = 6000, 5000, 60
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=21)
    cfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    old = engine._streamed_ok
    try:
        engine._streamed_ok = lambda p, t: True
        ref = l1pcp.estimate_rank_and_solve(mt, cfg)
        assert "overlap_retry" not in ref.stats
        with _lib.options(wait_timeout_ms=0):
            got = l1pcp.estimate_rank_and_solve(mt, cfg)
    finally:
        engine._streamed_ok = old
    assert got.stats.get("overlap_retry") is True
    assert torch.equal(got.l, ref.l) and torch.equal(got.s, ref.s)
    assert got.final_residual == ref.final_residual
