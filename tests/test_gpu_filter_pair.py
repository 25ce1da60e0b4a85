"""GPU: l1f_filter_pair_f32 (column and row filters in one call) against two l1f_filter_f32 calls.

The paired grid splits the tensor-core kernel's clusters between the two unit sets; a unit's
arithmetic does not depend on its cluster, group or slot, so z, iterations, residuals and
statuses must be bitwise those of the separate calls, whichever mode (library choice, one grid,
two grids) runs.  Reference semantics: filter_columns / filter_rows, pkg/src/l1pcp/l1filter.py:116-134.
"""

import numpy as np
import pytest
import torch

import paper_1108_5359_b200 as l1pcp
from paper_1108_5359_b200.l1reg import filter_units, filter_units_pair

pytestmark = pytest.mark.gpu


def _units(rng, s, k, n, mag=200.0, frac=0.08, scale=5.0):
    a, _ = np.linalg.qr(rng.standard_normal((s, k)))
    x = a @ rng.standard_normal((k, n)) * scale
    mask = rng.random(x.shape) < frac
    x[mask] += rng.uniform(-mag, mag, mask.sum())
    return (torch.from_numpy(np.ascontiguousarray(x.T, dtype=np.float32)).cuda(),
            torch.from_numpy(a.astype(np.float32)).cuda())


@pytest.mark.parametrize("s,k,n1,n2", [(1000, 100, 3000, 2500), (500, 48, 900, 60), (300, 40, 7, 1500),
                                       (2000, 200, 400, 350), (1000, 112, 0, 500), (1500, 150, 300, 200)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_pair_equals_two_calls(s, k, n1, n2, mode):
    rng = np.random.default_rng(s + k + n1 + mode)
    x1, a1 = _units(rng, s, k, n1)
    x2, a2 = _units(rng, s, k, n2)
    if n1 > 3:
        x1[3] = 0.0  # a dead unit
    cfg = l1pcp.AdmConfig(tol=1e-7)
    one = filter_units(x1, a1, cfg, want_e=False)
    two = filter_units(x2, a2, cfg, want_e=False)
    p1, p2 = filter_units_pair(x1, a1, x2, a2, cfg, mode=mode)
    torch.cuda.synchronize()
    for ref, got in ((one, p1), (two, p2)):
        z, _, it, res, st = ref
        for a, b in zip((z, it, res, st), got):
            assert torch.equal(a, b)
