"""Oracle: the reference's PCG64 instance generator (TEST INFRASTRUCTURE ONLY).

Restates synth.generate (/root/reference/pkg/src/l1pcp/synth.py:43-64): two child streams
of SeedSequence(rng_seed) — one for the Gaussian factors (L0 = A B^T), one for the exact
support (choice without replacement over m*n) and its U[-magnitude, magnitude] values —
and M = L0 + sigma_scale * S0.  Used to regenerate the inputs of the golden pipeline
fixtures (pinned there by sha256) instead of storing them.
"""

import numpy as np


def generate(m, n, rho_r, rho_s, magnitude=500.0, sigma_scale=1.0, rng_seed=0):
    rank = int(round(rho_r * m))
    count = int(round(rho_s * m * n))
    factor_stream, support_stream = np.random.SeedSequence(rng_seed).spawn(2)
    g = np.random.default_rng(factor_stream)
    if rank:
        left = g.standard_normal((m, rank))
        right = g.standard_normal((n, rank))
        l0 = left @ right.T
    else:
        l0 = np.zeros((m, n))
    g = np.random.default_rng(support_stream)
    flat = np.zeros(m * n)
    if count:
        where = g.choice(m * n, size=count, replace=False)
        flat[where] = g.uniform(-magnitude, magnitude, size=count)
    s0 = flat.reshape(m, n)
    return l0 + sigma_scale * s0, l0, s0
