"""GPU: the reconstruction kernels (l1f_reconstruct) against an FP64 product.

L = Af Bf^T and S = M - L (reference: nystrom_complete + assemble + s = m - l,
pkg/src/l1pcp/l1filter.py:137-167,253).  k > 16 runs the tcgen05 kernel (recon_tc.cu, two-piece
FP16 split with power-of-two row scales), k <= 16 the streaming kernel (dense.cu).  Every entry of
L must sit within 2^-18 of sum_t |a_t b_t| of the exact product (FP32 accumulation of 22-bit
operand pieces), S must equal the FP32 difference M - L bit for bit, and the residual partials
are sum((M - L) - S)^2 = 0 and sum(M^2).  Shapes cover ragged tiles, one-row/one-column edges,
K chunk padding, strided operands and factor rows whose magnitudes span 40 decades.
"""

import numpy as np
import pytest
import torch

from paper_1108_5359_b200 import engine

pytestmark = pytest.mark.gpu


def _factors(rows, k, gen, spread):
    x = torch.randn(rows, k, generator=gen, dtype=torch.float64)
    if spread:
        x *= torch.pow(10.0, (torch.rand(rows, 1, generator=gen, dtype=torch.float64) * 2 - 1) * spread)
    return x


def _check(m, n, k, spread_a=0.0, spread_b=0.0, zero_rows=False, pad=0, seed=0):
    gen = torch.Generator().manual_seed(seed)
    a64 = _factors(m, k, gen, spread_a)
    b64 = _factors(n, k, gen, spread_b)
    if zero_rows and m > 2 and n > 2:
        a64[1] = 0.0
        b64[2] = 0.0
    a_full = torch.zeros(m, k + pad, dtype=torch.float32)
    b_full = torch.zeros(n, k + pad, dtype=torch.float32)
    a_full[:, :k] = a64.float()
    b_full[:, :k] = b64.float()
    af = a_full.cuda()[:, :k]
    bf = b_full.cuda()[:, :k]
    a64 = a_full[:, :k].double()
    b64 = b_full[:, :k].double()
    mt = (torch.randn(m, n, generator=gen) * 10).cuda()
    l, s, rs = engine.reconstruct(mt, af, bf)
    torch.cuda.synchronize()
    ref = a64 @ b64.T
    bound = (a64.abs() @ b64.abs().T) * 2.0 ** -18 + 1e-38
    err = (l.cpu().double() - ref).abs()
    assert bool((err <= bound).all()), f"max err/bound {(err / bound).max().item():.3g}"
    assert torch.equal(s, mt - l)
    r = rs.cpu().numpy()
    assert r[0] == 0.0
    m2 = float((mt.double() ** 2).sum())
    assert abs(r[1] - m2) <= 1e-5 * m2


@pytest.mark.parametrize("m,n,k", [
    (1, 1, 17), (1, 300, 40), (300, 1, 40), (129, 257, 17), (300, 200, 100), (1000, 777, 200),
    (513, 1030, 224), (640, 384, 32), (2048, 2048, 250), (333, 4100, 64),
])
def test_reconstruct_tc_shapes(m, n, k):
    _check(m, n, k, seed=m + n + k)


@pytest.mark.parametrize("k", [24, 100, 208])
def test_reconstruct_tc_wide_dynamic_range(k):
    _check(700, 900, k, spread_a=20.0, spread_b=5.0, zero_rows=True, seed=k)


def test_reconstruct_tc_strided_factors():
    _check(500, 600, 100, pad=12, seed=7)


@pytest.mark.parametrize("m,n,k", [(100, 100, 5), (1000, 2100, 16), (37, 5000, 1)])
def test_reconstruct_stream_small_k(m, n, k):
    _check(m, n, k, seed=k)
