"""Oracle: small-PCP seed recovery (TEST INFRASTRUCTURE ONLY).

Restates /root/reference/pkg/src/l1pcp/pcp_adm.py:62-140 (default_lambda,
spectral_norm_estimate, solve_pcp) and matcore.py:66-105 (soft_threshold, svd rank cut,
svt_with_rank) plus recover_seed (l1filter.py:90-113) in numpy float64 / LAPACK.
"""

import math

import numpy as np


def default_lambda(m, n):
    return 1.0 / math.sqrt(max(m, n))


def spectral_norm(m, iters=25):
    """25-step power iteration from the all-ones vector (pcp_adm.py:69-87)."""
    m = np.asarray(m, dtype=np.float64)
    v = np.full(m.shape[1], 1.0 / math.sqrt(m.shape[1]))
    sigma = 0.0
    for _ in range(iters):
        w = m @ v
        nw = np.linalg.norm(w)
        if nw == 0:
            return 0.0
        v = m.T @ (w / nw)
        sigma = np.linalg.norm(v)
        if sigma == 0:
            return 0.0
        v = v / sigma
    return float(sigma)


def shrink(w, eta):
    return np.sign(w) * np.maximum(np.abs(w) - eta, 0.0)


def svd_cut(m, rank_tol):
    """Thin SVD keeping sigma > rank_tol * sigma_max (matcore.py:73-88)."""
    u, s, vt = np.linalg.svd(np.asarray(m, dtype=np.float64), full_matrices=False)
    keep = int((s > rank_tol * (s[0] if s.size else 0.0)).sum())
    return u[:, :keep], s[:keep], vt[:keep].T


def svt(w, eta):
    """(U max(S - eta, 0) V^T, rank) (matcore.py:96-105)."""
    u, s, v = svd_cut(w, 0.0)
    d = s - eta
    k = int((d > 0).sum())
    if k == 0:
        return np.zeros_like(w), 0
    return (u[:, :k] * d[:k]) @ v[:, :k].T, k


def pcp(m, lam=None, tol=1e-7, beta0=None, rho=1.5, beta_max=None, max_iter=1000):
    """Inexact-ALM PCP (pcp_adm.py:90-140).  Returns (L, S, iterations, residual, rank, converged)."""
    m = np.asarray(m, dtype=np.float64)
    norm_m = np.linalg.norm(m)
    if norm_m == 0.0:
        return np.zeros_like(m), np.zeros_like(m), 1, 0.0, 0, True
    lam = lam if lam is not None else default_lambda(*m.shape)
    beta = beta0 if beta0 is not None else 1.25 / max(spectral_norm(m), np.finfo(float).tiny)
    bmax = beta_max if beta_max is not None else 1e7 * beta
    l = np.zeros_like(m)
    s = np.zeros_like(m)
    y = np.zeros_like(m)
    rank = 0
    residual = 1.0
    it = 0
    for it in range(1, max_iter + 1):
        s = shrink((m - l) + y / beta, lam / beta)
        l, rank = svt((m - s) + y / beta, 1.0 / beta)
        r = (m - l) - s
        residual = np.linalg.norm(r) / norm_m
        if not np.isfinite(residual):
            raise FloatingPointError(f"non-finite residual at iteration {it}")
        y = y + beta * r
        if residual <= tol:
            return l, s, it, residual, rank, True
        beta = min(rho * beta, bmax)
    return l, s, it, residual, rank, False


def recover(block, tol=1e-9, rank_tol=1e-6, rho=1.5, max_iter=1000):
    """recover_seed (l1filter.py:90-113): forced lam = 1/sqrt(max dims).
    Returns (u, sigma, v, seed_l, pcp_iterations) or None for a zero seed."""
    block = np.asarray(block, dtype=np.float64)
    l, _, it, _, _, _ = pcp(block, lam=default_lambda(*block.shape), tol=tol, rho=rho, max_iter=max_iter)
    u, s, v = svd_cut(l, rank_tol)
    if s.size == 0:
        return None
    return u, s, v, (u * s) @ v.T, it
