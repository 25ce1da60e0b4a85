"""GPU: the tensor-core ADM filter (csrc/filter_tc.cu) against the FP64 oracle and the SIMT kernel.

Covers the variants (three slot groups for k <= 112, two with the tc_groups=2 option; one group with two phase-c M tiles
for 112 < k <= 160; one group with the phase-a dictionary in TMEM and the residual-form z step
for 160 < k <= 224), cluster sizes 1..16, slot refills (many more units than slots) with dead units
in between, the e output, max_iter status codes, and bitwise independence of unit order.
Reference semantics: _solve_block, pkg/src/l1pcp/l1reg.py:59-137.  Gate (north_star, FP32):
relative Frobenius difference of A z <= 1e-4; iteration counts within +-1 of the oracle for
most units (FP32 vs FP64 arithmetic can move the stopping iteration by one).
"""

import os

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from oracle import adm_filter
from paper_1108_5359_b200 import _lib
from paper_1108_5359_b200.l1reg import filter_units

pytestmark = pytest.mark.gpu


def _units(rng, s, k, n, mag=200.0, frac=0.08, scale=5.0):
    a, _ = np.linalg.qr(rng.standard_normal((s, k)))
    x = a @ rng.standard_normal((k, n)) * scale
    mask = rng.random(x.shape) < frac
    x[mask] += rng.uniform(-mag, mag, mask.sum())
    return a, x


def _run(x, a, tol=1e-7, max_iter=1000, want_e=False, tc=True):
    with _lib.options(filter_tc=1 if tc else 0):
        xt = torch.from_numpy(np.ascontiguousarray(x.T, dtype=np.float32)).cuda()
        at = torch.from_numpy(a.astype(np.float32)).cuda()
        out = filter_units(xt, at, l1pcp.AdmConfig(tol=tol, max_iter=max_iter), want_e=want_e)
        torch.cuda.synchronize()
        return [o.cpu() if o is not None else None for o in out]


@pytest.mark.parametrize("s,k,n", [(100, 20, 50), (500, 48, 700), (1000, 100, 2500), (1000, 112, 400),
                                   (2000, 100, 300), (1000, 128, 300), (1500, 150, 200), (777, 37, 900),
                                   (2000, 200, 700), (1800, 176, 300), (2048, 224, 100)])
def test_tc_filter_matches_oracle(s, k, n):
    rng = np.random.default_rng(s + 7 * k + n)
    a, x = _units(rng, s, k, n)
    x[:, 5] = 0.0     # dead units in the middle of the stream
    x[:, n // 2] = 0.0
    zr, er, itr, rr, sr = adm_filter.solve_units(x, a, 1e-7)
    z, e, it, res, st = _run(x, a)
    lc = a @ z.double().numpy().T
    lr = a @ zr
    err = np.linalg.norm(lc - lr) / np.linalg.norm(lr)
    print(f"s={s} k={k} n={n}: rel {err:.2e} iters {it.float().mean():.2f} vs {itr.mean():.2f}")
    assert err <= 1e-4
    st = st.numpy()
    assert st[5] == _lib.UNIT_ZERO and st[n // 2] == _lib.UNIT_ZERO
    assert it.numpy()[5] == 0
    live = sr != adm_filter.ZERO
    assert (st[live] == _lib.UNIT_OK).all()
    d_it = np.abs(it.numpy()[live].astype(int) - itr[live].astype(int))
    assert (d_it <= 1).mean() >= 0.97 and d_it.max() <= 3


def test_tc_filter_e_output_and_statuses():
    rng = np.random.default_rng(11)
    a, x = _units(rng, 1000, 100, 200)
    zr, er, itr, rr, sr = adm_filter.solve_units(x, a, 1e-7)
    z, e, it, res, st = _run(x, a, want_e=True)
    e_ref = np.ascontiguousarray(er.T)
    assert np.linalg.norm(e.double().numpy() - e_ref) <= 1e-4 * np.linalg.norm(e_ref)
    # residuals reported are the stopping values: max|r| <= tol * ||x||_inf for OK units
    scale = np.abs(x).max(axis=0)
    assert (res.numpy() <= 1e-7 * scale * (1 + 1e-5)).all()
    # max_iter cap: every unit stops at max_iter with MAXITER
    z2, e2, it2, res2, st2 = _run(x, a, max_iter=5)
    assert (it2.numpy() == 5).all() and (st2.numpy() == _lib.UNIT_MAXITER).all()
    zr5, _, itr5, _, sr5 = adm_filter.solve_units(x, a, 1e-7, max_iter=5)
    assert (sr5 == adm_filter.MAXITER).all()
    assert np.linalg.norm(a @ z2.double().numpy().T - a @ zr5) <= 1e-4 * np.linalg.norm(a @ zr5)


def test_tc_agrees_with_simt_kernel():
    rng = np.random.default_rng(5)
    a, x = _units(rng, 1000, 100, 600)
    z_tc, _, it_tc, _, st_tc = _run(x, a, tc=True)
    z_si, _, it_si, _, st_si = _run(x, a, tc=False)
    lc, ls = a @ z_tc.double().numpy().T, a @ z_si.double().numpy().T
    assert np.linalg.norm(lc - ls) <= 1e-5 * np.linalg.norm(ls)
    assert (np.abs(it_tc.numpy().astype(int) - it_si.numpy().astype(int)) <= 1).mean() >= 0.97


@pytest.mark.parametrize("k", [64, 150, 200])
def test_tc_results_independent_of_unit_order(k):
    rng = np.random.default_rng(k)
    a, x = _units(rng, 640, k, 700)
    full = _run(x, a)
    perm = np.random.default_rng(1).permutation(700)
    part = _run(x[:, perm], a)
    for f, p in zip(full[:4], part[:4]):
        if f is not None:
            assert torch.equal(f[torch.from_numpy(perm)], p)
    sub = _run(x[:, 100:140], a)
    assert torch.equal(sub[0], full[0][100:140])


@pytest.mark.parametrize("s,k,n,want_e", [(1000, 100, 1500, False), (300, 40, 800, True), (2000, 112, 400, False)])
def test_tc_three_and_two_slot_groups_bitwise_equal(s, k, n, want_e):
    # k <= 112 runs three slot groups per CTA (x in TMEM, 8-slot blocks); option tc_groups=2 forces the
    # two-group layout.  A unit's arithmetic does not depend on its group or slot.
    rng = np.random.default_rng(s + k)
    a, x = _units(rng, s, k, n)
    three = _run(x, a, want_e=want_e)
    with _lib.options(tc_groups=2):
        two = _run(x, a, want_e=want_e)
    for f, p in zip(three, two):
        if f is not None:
            assert torch.equal(f, p)


def test_tc_filter_few_units_many_slots():
    # C = 8 CTAs, 2 groups x 32 slots, only 3 units: nearly every slot of both groups is empty
    rng = np.random.default_rng(21)
    a, x = _units(rng, 1000, 100, 3)
    zr, er, itr, rr, sr = adm_filter.solve_units(x, a, 1e-7)
    z, e, it, res, st = _run(x, a)
    assert np.linalg.norm(a @ z.double().numpy().T - a @ zr) <= 1e-4 * np.linalg.norm(a @ zr)
    assert (np.abs(it.numpy().astype(int) - itr.astype(int)) <= 1).all()


@pytest.mark.parametrize("k", [100, 200])
def test_tc_filter_explicit_beta_and_rho(k):
    rng = np.random.default_rng(k + 1)
    a, x = _units(rng, 2 * k if k > 100 else 1000, k, 150)
    cfg = dict(tol=1e-7, rho=1.3, beta0=0.01, beta_max=500.0)
    zr, er, itr, rr, sr = adm_filter.solve_units(x, a, cfg["tol"], rho=cfg["rho"], beta0=cfg["beta0"],
                                                 beta_max=cfg["beta_max"])
    xt = torch.from_numpy(np.ascontiguousarray(x.T, dtype=np.float32)).cuda()
    at = torch.from_numpy(a.astype(np.float32)).cuda()
    z, e, it, res, st = filter_units(xt, at, l1pcp.AdmConfig(**cfg), want_e=False)
    lc, lr = a @ z.double().cpu().numpy().T, a @ zr
    assert np.linalg.norm(lc - lr) <= 1e-4 * np.linalg.norm(lr)
    assert (np.abs(it.cpu().numpy().astype(int) - itr.astype(int)) <= 1).mean() >= 0.95


def test_tc_filter_strided_abi():
    # leading dimensions larger than the logical widths (X, A and Z with padding)
    import ctypes
    from paper_1108_5359_b200 import _device as dv
    rng = np.random.default_rng(9)
    s, k, n = 1000, 100, 120
    a, x = _units(rng, s, k, n)
    xp = torch.zeros((n, s + 7), dtype=torch.float32, device="cuda")
    xp[:, :s] = torch.from_numpy(x.T.astype(np.float32)).cuda()
    ap = torch.zeros((s, k + 5), dtype=torch.float32, device="cuda")
    ap[:, :k] = torch.from_numpy(a.astype(np.float32)).cuda()
    zp = torch.full((n, k + 3), 7.0, dtype=torch.float32, device="cuda")
    iters = torch.empty(n, dtype=torch.int32, device="cuda")
    res = torch.empty(n, dtype=torch.float32, device="cuda")
    status = torch.empty(n, dtype=torch.uint8, device="cuda")
    _lib.call("l1f_filter_f32", dv.ptr(xp), xp.stride(0), s, n, dv.ptr(ap), ap.stride(0), k, 1e-7, 1.5, 0.0, 0.0,
              1000, dv.ptr(zp), zp.stride(0), None, s, dv.ptr(iters), dv.ptr(res), dv.ptr(status), None, 0,
              dv.stream())
    torch.cuda.synchronize()
    zr, er, itr, rr, sr = adm_filter.solve_units(x, a, 1e-7)
    z = zp[:, :k].double().cpu().numpy()
    assert np.linalg.norm(a @ z.T - a @ zr) <= 1e-4 * np.linalg.norm(a @ zr)
    assert (zp[:, k:] == 7.0).all()  # padding untouched
