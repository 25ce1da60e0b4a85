"""GPU: parity of the full FP32 device solve with the CPU oracle at BASELINE.json's five configs.

Inputs are the device Philox matrices (bit-identical to the oracle's host regeneration).
Configs 1 and 2 are compared in full; configs 3, 4 and 5 through the sampled oracle of SURVEY
8(c'): the oracle solves the seed (FP64, the reference's index draw) and filters only the sampled
non-seed rows/columns, which yields L and S exactly on the sampled sub-block.  Gate: relative
Frobenius difference <= 1e-4 for L and S (north_star FP32 tolerance).  Config 5 (120 GB of
device memory for M, L, S, a 2000^2 numpy seed solve and 1000 + 1000 sampled FP64 filter units,
~40 s) can be skipped with
L1F_SKIP_CFG5=1.
"""

import os

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from oracle import philox_gen
from oracle import pipeline as opipe
from paper_1108_5359_b200 import engine
from paper_1108_5359_b200.synth import BENCHMARK_CONFIGS

pytestmark = pytest.mark.gpu
TOL = 1e-7


def _device_solve(c):
    cfg = BENCHMARK_CONFIGS[c]
    mt, _, _, _ = engine.generate_matrix(cfg["m"], cfg["n"], cfg["r"], cfg["rho_s"], cfg["magnitude"], seed=0,
                                         kind=cfg["kind"])
    fcfg = l1pcp.FilterConfig(rank_hint=cfg["r"], rng_seed=0, adm=l1pcp.AdmConfig(tol=TOL))
    kind, seed, _, _ = engine.seed_stage(mt, fcfg)
    assert kind == "seed"
    plan = engine.FilterPlan(cfg["m"], cfg["n"], seed, mt.dtype, fcfg.adm)
    out = engine.solve_from_seed(mt, plan)
    torch.cuda.synchronize()
    return cfg, mt, seed, out


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("c", [1, 2])
def test_config_full_parity(c):
    cfg, mt, seed, out = _device_solve(c)
    m_host = mt.double().cpu().numpy()
    ref = opipe.solve(m_host, cfg["r"], 0, tol=TOL)
    assert seed.r_prime == ref["r_prime"]
    np.testing.assert_array_equal(seed.row_idx, ref["row_idx"])
    l = out["l"].double().cpu().numpy()
    s = out["s"].double().cpu().numpy()
    print(f"config {c}: full, rel L {_rel(l, ref['l']):.2e}, rel S {_rel(s, ref['s']):.2e}")
    assert _rel(l, ref["l"]) <= 1e-4
    assert _rel(s, ref["s"]) <= 1e-4


def _sampled(c, n_rows, n_cols):
    cfg, mt, seed, out = _device_solve(c)
    m, n, r = cfg["m"], cfg["n"], cfg["r"]
    x, y = philox_gen.factors(0, cfg["kind"], m, n, r)

    def block(rows, cols):
        return philox_gen.block(0, cfg["kind"], m, n, r, cfg["rho_s"], cfg["magnitude"], rows, cols, x=x,
                                y=y).astype(np.float64)

    rng = np.random.default_rng(123)
    rows = np.sort(rng.choice(m, n_rows, replace=False))
    cols = np.sort(rng.choice(n, n_cols, replace=False))
    # include a few seed rows / columns so every block type of the assembly is checked
    rows = np.union1d(rows, seed.row_idx[:5])
    cols = np.union1d(cols, seed.col_idx[:5])
    ref = opipe.sampled_blocks(m, n, block, r, rows, cols, 0, tol=TOL)
    assert ref["kind"] == "seed" and ref["r_prime"] == seed.r_prime
    np.testing.assert_array_equal(ref["row_idx"], seed.row_idx)
    ri = torch.as_tensor(rows, device="cuda")
    ci = torch.as_tensor(cols, device="cuda")
    l = out["l"][ri][:, ci].double().cpu().numpy()
    s = out["s"][ri][:, ci].double().cpu().numpy()
    print(f"config {c}: sampled {rows.size}x{cols.size}, rel L {_rel(l, ref['l']):.2e}, rel S {_rel(s, ref['s']):.2e}")
    assert _rel(l, ref["l"]) <= 1e-4
    assert _rel(s, ref["s"]) <= 1e-4
    # the device matrix is the generator's (regenerated here bit for bit)
    np.testing.assert_array_equal(mt[ri][:, ci].cpu().numpy(), block(rows, cols).astype(np.float32))


def test_config3_sampled_parity():
    _sampled(3, 1000, 1000)


def test_config4_sampled_parity():
    _sampled(4, 1000, 1000)


@pytest.mark.skipif(os.environ.get("L1F_SKIP_CFG5") == "1", reason="L1F_SKIP_CFG5=1")
def test_config5_sampled_parity():
    _sampled(5, 1000, 1000)  # BASELINE.json: "Oracle check on 1000 sampled columns and rows"


# ---------------------------------------------------------------------------------------------
# Per-unit parity on the benchmark data (l1reg.py:59-137 per unit; reference guard
# test_l1reg.py:99-108).  The device pipeline's own per-unit outputs (status, iterations, z) are
# compared with the FP64 oracle run on the same panels against the same (device) seed factors:
#  * every unit for configs 2-4, 1000 sampled + every flagged unit per side for config 5;
#  * status: identical, except units in the exact-arithmetic stall class (below);
#  * per-unit L (A z) relative error <= 1e-5 (FP32 path) / 1e-7 (FP64 path);
#  * the device's own (z, e) recomputed in FP64: max|x - A z - e| <= tol*||x||_inf * (1 + 1e-3)
#    on the FP64 path; on the FP32 path the bound is 1.5x — an fp32 x, z and e carry ~2^-24*||x||
#    rounding, ~30% of tol*||x||_inf at tol = 1e-7, so no FP32 solver can certify the FP64
#    residual to 1e-3 (profiles/r2_unit_parity.json: max 1.40);
#  * iteration counts: mostly equal (>= 93% within +-1); the rest sit on the bimodal threshold
#    (stop at ~20 vs at beta saturation ~38), where the last-bit difference of the residual
#    decides, so |delta| <= 25.
# Exact-arithmetic stall class: while the support of e is fixed and e = 0, z = A^T x exactly
# (A^T y = 0) and max|r| is constant, so the reference's 20-iteration stagnation rule
# (l1reg.py:102-108) fires in exact arithmetic; numpy's BLAS rounding jitter (~1e-9 relative)
# resets the counter and the oracle runs on to beta saturation.  A status mismatch is accepted
# only where the oracle's own residual trajectory over the 20 iterations before the device's
# stall moved by < 1e-8 relative (rounding noise of a constant), and its L matches.
# ---------------------------------------------------------------------------------------------

from oracle import adm_filter  # noqa: E402
from paper_1108_5359_b200.l1reg import filter_units  # noqa: E402


def _oracle_traj(x, a, n_it):
    """max|r| per iteration of the reference recurrence (FP64), first n_it iterations."""
    sc = np.abs(x).max(axis=0)
    b = 1.0 / sc
    bmax = 1e7 * b
    z = np.zeros((a.shape[1], x.shape[1]))
    y = np.zeros_like(x)
    out = []
    for _ in range(n_it):
        w = x - a @ z + y / b
        e = np.sign(w) * np.maximum(np.abs(w) - 1 / b, 0)
        z = a.T @ (x - e + y / b)
        r = x - a @ z - e
        out.append(np.abs(r).max(axis=0))
        y = y + b * r
        b = np.minimum(1.5 * b, bmax)
    return np.array(out)


def _unit_parity(c, n_sample=0):
    cfg, mt, seed, out = _device_solve(c)
    plan_dtype = torch.float64 if seed.r_prime <= engine.SMALL_K_FP64 else torch.float32
    fp64 = plan_dtype == torch.float64
    report = {}
    for side in ("c", "r"):
        comp = np.setdiff1d(np.arange(cfg["n"] if side == "c" else cfg["m"]),
                            seed.col_idx if side == "c" else seed.row_idx)
        if side == "c":
            xd = engine.gather(mt, seed.row_idx, comp, out_dtype=plan_dtype, transpose=True)
            a = seed.u
        else:
            xd = engine.gather(mt, comp, seed.col_idx, out_dtype=plan_dtype)
            a = seed.v
        st_d = out["status_" + side].cpu().numpy()
        it_d = out["iters_" + side].cpu().numpy()
        z_d = out["z" + side].double().cpu().numpy()
        # the device's e for the same units (a want_e call; per-unit arithmetic is call-independent)
        ze, ee, it_e, _, _ = filter_units(xd, a.to(plan_dtype).contiguous(), l1pcp.AdmConfig(tol=TOL), want_e=True)
        assert np.array_equal(it_e.cpu().numpy(), it_d)
        sel = np.arange(len(comp))
        if n_sample and len(comp) > n_sample:
            rng = np.random.default_rng(7)
            sel = np.union1d(rng.choice(len(comp), n_sample, replace=False), np.flatnonzero(st_d != 0))
        x64 = xd.double().cpu().numpy()[sel]
        a64 = a.double().cpu().numpy()
        zo, _, ito, _, sto = adm_filter.solve_units(x64.T, a64, TOL)
        lo = zo.T @ a64.T
        ld = z_d[sel] @ a64.T
        rel_l = np.linalg.norm(ld - lo, axis=1) / np.linalg.norm(lo, axis=1)
        assert rel_l.max() <= (1e-7 if fp64 else 1e-5), (side, rel_l.max())
        # status: equal, or the exact-arithmetic stall class
        mism = np.flatnonzero(st_d[sel] != sto)
        for j in mism:
            assert st_d[sel][j] == adm_filter.STALLED and sto[j] == adm_filter.OK, (side, j)
            n_it = int(it_d[sel][j])
            traj = _oracle_traj(x64[j][:, None], a64, n_it)[:, 0]
            window = traj[n_it - 20:n_it]
            assert np.abs(np.diff(window)).max() / window.max() < 1e-8, (side, j, window)
        # feasibility of the device's own (z, e), recomputed in FP64 (test_l1reg.py:99-108)
        e64 = ee.double().cpu().numpy()[sel]
        r64 = np.abs(x64 - ze.double().cpu().numpy()[sel] @ a64.T - e64).max(axis=1)
        thr = TOL * np.abs(x64).max(axis=1)
        okd = st_d[sel] == adm_filter.OK
        bound = (1 + 1e-3) if fp64 else 1.5
        assert (r64[okd] <= thr[okd] * bound).all(), (side, float((r64[okd] / thr[okd]).max()))
        dit = it_d[sel] - ito
        assert (np.abs(dit) <= 1).mean() >= 0.93 and np.abs(dit).max() <= 25, (side, np.abs(dit).max())
        report[side] = dict(units=int(sel.size), status_mismatch=int(mism.size), rel_l_max=float(rel_l.max()),
                            resid_ratio_max=float((r64[okd] / thr[okd]).max()), dit_max=int(np.abs(dit).max()))
    print(f"config {c} per-unit: {report}")


@pytest.mark.parametrize("c", [2, 3, 4])
def test_config_unit_parity(c):
    _unit_parity(c)


@pytest.mark.skipif(os.environ.get("L1F_SKIP_CFG5") == "1", reason="L1F_SKIP_CFG5=1")
def test_config5_unit_parity():
    _unit_parity(5, n_sample=1000)
