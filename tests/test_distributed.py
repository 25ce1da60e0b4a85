"""CPU: the row-sharded multi-process solve (paper_1108_5359_b200/distributed.py) over gloo
with world_size 1 and 2.  The compute backend is the numpy oracle (tests only); the shard
plan, the collectives and the assembly are the product's.  Sharded L/S must equal the
unsharded solve and the oracle's full pipeline."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_1108_5359_b200 import distributed as pdist  # noqa: E402
from paper_1108_5359_b200.pcp_adm import AdmConfig  # noqa: E402


class OracleBackend:
    """CPU stand-in for CudaBackend built on the numpy oracle."""

    def empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype)

    def seed(self, block, adm, rank_tol):
        from oracle import seed_pcp
        u, s, v, _, it = seed_pcp.recover(block.double().numpy(), tol=adm.tol, rank_tol=rank_tol)
        return torch.from_numpy(np.ascontiguousarray(u)), torch.from_numpy(s.copy()), \
            torch.from_numpy(np.ascontiguousarray(v)), it

    def column_panel(self, seed_rows, cols):
        return seed_rows[:, torch.as_tensor(cols)].t().contiguous()

    def panel_t(self, m_local, local_rows, cols, out=None):
        t = m_local[torch.as_tensor(local_rows, dtype=torch.int64)][:, torch.as_tensor(cols)].t().contiguous()
        if out is not None:
            out.copy_(t)
            return out
        return t

    def row_panel(self, m_local, local_rows, cols):
        return m_local[torch.as_tensor(local_rows)][:, torch.as_tensor(cols)].contiguous()

    def filter(self, x_um, a64, adm):
        from oracle import adm_filter
        z, _, it, _, st = adm_filter.solve_units(x_um.double().numpy().T, a64.double().numpy(), adm.tol)
        return torch.from_numpy(np.ascontiguousarray(z.T)), torch.from_numpy(it), torch.from_numpy(st)

    def reconstruct(self, m_local, plan, u, sig, v, zc_all, zr):
        u, sig, v = u.numpy(), sig.numpy(), v.numpy()
        rows = np.arange(plan.r0, plan.r1)
        seed_pos = {int(r): p for p, r in enumerate(plan.row_idx)}
        col_pos = {int(c): q for q, c in enumerate(plan.col_idx)}
        zr = zr.numpy()
        ri = 0
        a = np.empty((rows.size, sig.size))
        for i, r in enumerate(rows):
            if int(r) in seed_pos:
                a[i] = u[seed_pos[int(r)]]
            else:
                a[i] = zr[ri] / sig
                ri += 1
        zc = zc_all.numpy()
        b = np.empty((plan.n, sig.size))
        ci = 0
        for j in range(plan.n):
            if j in col_pos:
                b[j] = sig * v[col_pos[j]]
            else:
                b[j] = zc[ci]
                ci += 1
        l = a @ b.T
        return torch.from_numpy(l), m_local.double() - torch.from_numpy(l)


def _instance(m=120, n=100, r=2, seed=3):
    from oracle import ref_synth
    mm, l0, _ = ref_synth.generate(m, n, r / m, 0.05, rng_seed=seed)
    return mm, l0


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mm, _ = _instance()
        m, n = mm.shape
        from paper_1108_5359_b200 import engine
        ri, ci = engine.sample_indices(m, n, 20, 20, np.random.SeedSequence(0).spawn(1)[0])
        plan = pdist.ShardPlan(m, n, rank, world, ri, ci)
        m_local = torch.from_numpy(mm[plan.r0:plan.r1].copy())
        l, s, info = pdist.solve_sharded(m_local, plan, OracleBackend(), AdmConfig(tol=1e-9))
        out_q.put((rank, plan.r0, l.numpy(), s.numpy(), info["k"], info["units"]))
    finally:
        dist.destroy_process_group()


def _run(world):
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(g, world, port, q)) for g in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    return np.concatenate([t[2] for t in res]), np.concatenate([t[3] for t in res]), res


def test_shard_plan_partitions_units():
    ri = np.array([3, 10, 57, 99])
    ci = np.array([1, 2, 50])
    units_c, units_r = [], []
    for g in range(3):
        p = pdist.ShardPlan(100, 80, g, 3, ri, ci)
        units_c.extend(p.my_cols.tolist())
        units_r.extend(p.my_rows.tolist())
        assert np.all((p.my_rows >= p.r0) & (p.my_rows < p.r1))
    assert sorted(units_c) == np.setdiff1d(np.arange(80), ci).tolist()
    assert sorted(units_r) == np.setdiff1d(np.arange(100), ri).tolist()
    assert pdist.row_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]


@pytest.mark.timeout(900)
def test_sharded_solve_matches_single_process_and_oracle():
    l1, s1, r1 = _run(1)
    l2, s2, r2 = _run(2)
    l3, s3, r3 = _run(3)  # uneven seed-row and column-unit counts in the all-to-all
    np.testing.assert_allclose(l3, l1, rtol=0, atol=1e-10 * np.abs(l1).max())
    np.testing.assert_allclose(s3, s1, rtol=0, atol=1e-10 * np.abs(s1).max())
    assert r2[0][4] == r1[0][4]                 # same seed rank
    assert r2[0][5] == r1[0][5]                 # all units accounted for
    np.testing.assert_allclose(l2, l1, rtol=0, atol=1e-10 * np.abs(l1).max())
    np.testing.assert_allclose(s2, s1, rtol=0, atol=1e-10 * np.abs(s1).max())
    from oracle import pipeline
    mm, l0 = _instance()
    ref = pipeline.solve(mm, 2, 0, tol=1e-9)
    assert np.linalg.norm(l2 - ref["l"]) <= 1e-8 * np.linalg.norm(ref["l"])
    assert np.linalg.norm(l2 - l0) <= 1e-5 * np.linalg.norm(l0)


def _exchange_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        m, n = 50, 37
        mm = rng.standard_normal((m, n))
        ri = np.arange(0, 9)                   # every seed row in rank 0's block: others send nothing
        ci = np.array([0, 5, 11, 20, 36])
        plan = pdist.ShardPlan(m, n, rank, world, ri, ci)
        m_local = torch.from_numpy(mm[plan.r0:plan.r1].copy())
        xc = pdist.exchange_column_panel(m_local, plan, OracleBackend())
        out_q.put((rank, bool(np.array_equal(xc.numpy(), mm[np.ix_(ri, plan.my_cols)].T))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_column_panel_all_to_all_exchange():
    """Exchange 1 (all-to-all of M[row_idx, C_h]) equals the direct gather, with ranks that own
    no seed rows and uneven column-unit counts."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    procs = [ctx.Process(target=_exchange_worker, args=(g, world, port, q)) for g in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)
