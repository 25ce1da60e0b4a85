"""Oracle: per-unit ADM for min ||e||_1 s.t. x = A z + e (TEST INFRASTRUCTURE ONLY).

Restates the column-separable solver of /root/reference/pkg/src/l1pcp/l1reg.py:59-137
(_solve_block) with its per-unit penalty start (:77-84), stopping threshold (:65-66),
stagnation rule (:33-34,102-108) and max_iter exit (:130-135).  Units are held in a dense
active set that shrinks as they finish; ``dtype=np.float32`` replays the recurrence in
single precision (the GPU benchmark path's arithmetic, up to summation order).

Status codes match include/l1pcp_b200.h: 0 ok, 1 stalled (failed), 2 max_iter (failed),
3 zero unit.
"""

import numpy as np

STALL_EPS = 1e-12   # l1reg.py:33
STALL_ITERS = 20    # l1reg.py:34

OK, STALLED, MAXITER, ZERO = 0, 1, 2, 3


def solve_units(x, a, tol, rho=1.5, beta0=None, beta_max=None, max_iter=1000, dtype=np.float64):
    """x: (s, N) units as columns; a: (s, k).  Returns (z (k,N), e (s,N), iters, res, status)."""
    x = np.asarray(x, dtype=dtype)
    a = np.asarray(a, dtype=dtype)
    s, n = x.shape
    k = a.shape[1]
    one = dtype(1)
    scale = np.abs(x).max(axis=0) if s else np.zeros(n, dtype)
    thresh = dtype(tol) * scale

    z_out = np.zeros((k, n), dtype)
    e_out = np.zeros((s, n), dtype)
    iters = np.zeros(n, dtype=np.int64)
    res_out = np.zeros(n, dtype)
    status = np.full(n, OK, dtype=np.uint8)
    status[~(scale > 0)] = ZERO

    cols = np.flatnonzero(scale > 0)
    if max_iter <= 0:
        iters[cols] = max_iter
        res_out[cols] = np.inf
        status[cols] = MAXITER
        return z_out, e_out, iters, res_out, status

    b = np.full(cols.size, dtype(beta0), dtype) if beta0 is not None else one / scale[cols]
    bmax = np.full(cols.size, dtype(beta_max), dtype) if beta_max is not None else dtype(1e7) * b
    X = x[:, cols]
    Z = np.zeros((k, cols.size), dtype)
    AZ = np.zeros((s, cols.size), dtype)
    E = np.zeros_like(X)
    Y = np.zeros_like(X)
    prev = np.full(cols.size, np.inf, dtype)
    stall = np.zeros(cols.size, dtype=np.int64)
    tiny = np.finfo(dtype).tiny
    last_res = prev.copy()

    for it in range(1, max_iter + 1):
        if cols.size == 0:
            break
        yb = Y / b
        W = (X - AZ) + yb
        E = np.sign(W) * np.maximum(np.abs(W) - one / b, dtype(0))
        Z = a.T @ ((X - E) + yb)
        AZ = a @ Z
        R = (X - AZ) - E
        res = np.abs(R).max(axis=0) if s else np.zeros(cols.size, dtype)

        rel = np.abs(res - prev) / np.maximum(res, tiny)
        stall = np.where(rel < STALL_EPS, stall + 1, 0)
        prev = res
        last_res = res

        ok = res <= thresh[cols]
        done = ok | (stall >= STALL_ITERS)
        if done.any():
            fin = cols[done]
            z_out[:, fin] = Z[:, done]
            e_out[:, fin] = E[:, done]
            iters[fin] = it
            res_out[fin] = res[done]
            status[fin] = np.where(ok[done], OK, STALLED)
            keep = ~done
            cols, X, Z, AZ, E, Y, R = cols[keep], X[:, keep], Z[:, keep], AZ[:, keep], E[:, keep], Y[:, keep], R[:, keep]
            b, bmax, prev, stall, last_res = b[keep], bmax[keep], prev[keep], stall[keep], last_res[keep]
            if cols.size == 0:
                break
        Y = Y + b * R
        b = np.minimum(dtype(rho) * b, bmax)

    if cols.size:
        z_out[:, cols] = Z
        e_out[:, cols] = E
        iters[cols] = max_iter
        res_out[cols] = last_res
        status[cols] = MAXITER
    return z_out, e_out, iters, res_out, status


def summarize(x, iters, res, status):
    """solve_l1reg's aggregation (l1reg.py:155-160): (iterations, final_residual, failed)."""
    scale = float(np.abs(x).max()) if np.asarray(x).size else 0.0
    failed = [int(c) for c in np.flatnonzero((status == STALLED) | (status == MAXITER))]
    return int(iters.max(initial=0)), (float(res.max(initial=0.0)) / scale if scale else 0.0), failed
