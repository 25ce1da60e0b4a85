"""CUDA-graph replay of the timed step (engine.CapturedStep) equals the eager step bitwise, on the
small-k FP64 path (config-1-like, non-streamed), the streamed small-k path, the tcgen05 streamed
path and the paired-filter path."""

import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200 import engine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,r", [(1000, 1000, 10), (4500, 4200, 10), (3000, 2800, 40), (2500, 2500, 50)])
def test_captured_step_matches_eager(m, n, r):
    mt, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=5)
    cfg = l1pcp.FilterConfig(rank_hint=r, rng_seed=0, adm=l1pcp.AdmConfig(tol=1e-7))
    kind, seed, _, _ = engine.seed_stage(mt, cfg)
    plan = engine.FilterPlan(m, n, seed, mt.dtype, cfg.adm)
    ref = engine.solve_step(plan, mt)
    torch.cuda.synchronize()
    l_out, s_out = torch.empty_like(mt), torch.empty_like(mt)
    step = engine.CapturedStep(plan, mt, l_out, s_out)
    for _ in range(3):
        l_out.zero_()
        s_out.zero_()
        out = step.replay()
        torch.cuda.synchronize()
        assert torch.equal(l_out, ref["l"]) and torch.equal(s_out, ref["s"])
        assert torch.equal(out["iters_c"], ref["iters_c"]) and torch.equal(out["iters_r"], ref["iters_r"])
    # a new M in the same buffer: the replay follows the data
    mt2, _, _, _ = engine.generate_matrix(m, n, r, 0.05, 500.0, seed=5)
    mt.copy_(mt2 * 1.0)
    out = step.replay()
    torch.cuda.synchronize()
    assert torch.equal(l_out, ref["l"])
