"""GPU: the pipelined host-buffer solve (engine.HostPipeline) equals the device-resident solve.

M, L and S live in pinned host memory; the column panel is gathered zero-copy, M moves in row
chunks and L, S come back per chunk.  Per-unit filter results and the per-entry reconstruction
do not depend on the chunking, so L and S must be bitwise identical to solve_from_seed's.
"""

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,r,chunks", [(2000, 1500, 20, 8), (1200, 1700, 8, 3), (3000, 3000, 30, 1)])
def test_host_pipeline_matches_device_solve(m, n, r, chunks):
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.1, 500.0, seed=3)
    fcfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    kind, seed, _, _ = engine.seed_stage(mt, fcfg)
    assert kind == "seed"
    plan = engine.FilterPlan(m, n, seed, mt.dtype, fcfg.adm, want_e=False)
    ref = engine.solve_from_seed(mt, plan)
    m_host = mt.cpu().pin_memory()
    l_host = torch.empty((m, n), dtype=mt.dtype).pin_memory()
    s_host = torch.empty((m, n), dtype=mt.dtype).pin_memory()
    pipe = engine.HostPipeline(plan, n_chunks=chunks)
    for _ in range(2):  # reuse of the pipeline buffers
        l_host.zero_()
        s_host.zero_()
        stats, rs = pipe.solve(m_host, l_host, s_host)
        torch.cuda.synchronize()
        assert torch.equal(l_host, ref["l"].cpu())
        assert torch.equal(s_host, ref["s"].cpu())
    assert torch.equal(stats["iters_c"], ref["iters_c"])
    assert torch.equal(stats["iters_r"], ref["iters_r"])
    r_ref = ref["resid_sq"].cpu().numpy()
    np.testing.assert_allclose(rs.cpu().numpy(), r_ref, rtol=1e-9, atol=1e-9 * r_ref[1])


@pytest.mark.parametrize("pinned,r", [(True, 25), (False, 25), (True, 8)])
def test_public_api_host_tensor_path(pinned, r):
    """estimate_rank_and_solve on a float32 HOST tensor (the end-to-end call of bench.py's e2e):
    L, S come back as host tensors, bitwise equal to the device-resident public call; the seed
    block and the column panel are read zero-copy from host memory."""
    m, n = 2500, 2200  # r = 8: the FP64 small-k filter inside the pipeline
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=4)
    cfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    dev = l1pcp.estimate_rank_and_solve(mt, cfg)
    m_host = mt.cpu()
    if pinned:
        m_host = m_host.pin_memory()
    sol = l1pcp.estimate_rank_and_solve(m_host, cfg)
    assert sol.stats.get("path") == "host-pipeline"
    assert not sol.l.is_cuda and sol.l.is_pinned() and sol.l.dtype == torch.float32
    assert torch.equal(sol.l, dev.l.cpu()) and torch.equal(sol.s, dev.s.cpu())
    assert sol.rank_of_l == dev.rank_of_l == r
    assert sol.iterations == dev.iterations
    assert sol.stats["seed_iterations"] == dev.stats["seed_iterations"]


def test_public_api_host_tensor_rejects_non_finite():
    m_host = torch.ones((600, 500), dtype=torch.float32)
    m_host[3, 4] = float("nan")
    with pytest.raises(ValueError):
        l1pcp.estimate_rank_and_solve(m_host, l1pcp.FilterConfig(rank_hint=20))
