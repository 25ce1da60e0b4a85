"""Inexact-ALM PCP solver on the device (mirrors pkg/src/l1pcp/pcp_adm.py).

    min ||L||_* + lambda * ||S||_l1   s.t.   M = L + S

Used by l1 filtering as the FP64 seed solver (recover_seed, l1filter.py:90-113) and by the
full-matrix fallback.  The loop (shrink -> SVT -> residual -> dual/penalty update) runs in
the C-ABI library (l1f_pcp_f64); only the per-iteration stopping decision crosses to the
host, as a scalar.
"""

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as dv
from . import _lib
from .matcore import as_dense


class PcpDivergenceError(RuntimeError):
    """The iteration produced non-finite values (pcp_adm.py:19-20)."""


@dataclass
class AdmConfig:
    """Hyperparameters for the ADM solvers (pcp_adm.py:23-46).

    lam=None picks 1/sqrt(max(m, n)); beta0=None picks 1.25 over a power-iteration estimate
    of the spectral norm; beta_max=None picks 1e7 * beta0.
    """

    lam: float | None = None
    tol: float = 1e-7
    beta0: float | None = None
    rho: float = 1.5
    beta_max: float | None = None
    max_iter: int = 1000

    def __post_init__(self):
        if self.rho <= 1:
            raise ValueError("rho must be > 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.beta0 is not None and self.beta_max is not None:
            if self.beta0 >= self.beta_max:
                raise ValueError("beta0 must be < beta_max")


@dataclass
class PcpSolution:
    l: object
    s: object
    iterations: int
    final_residual: float
    rank_of_l: int
    elapsed: float
    converged: bool
    method: str = "adm"
    stats: dict = field(default_factory=dict)


def default_lambda(m_rows, m_cols):
    """The exact-recovery weight 1/sqrt(max(m, n)) (pcp_adm.py:62-66)."""
    if m_rows < 1 or m_cols < 1:
        raise ValueError("matrix dimensions must be >= 1")
    return 1.0 / math.sqrt(max(m_rows, m_cols))


def spectral_norm_estimate(m, iters=25):
    """Power-iteration estimate of the largest singular value, from the all-ones vector
    (pcp_adm.py:69-87)."""
    t, _ = dv.as_device(m, keep_f32=False)
    if t.dim() != 2:
        t = t.reshape(t.shape[0], -1)
    out = ctypes.c_double(0.0)
    _lib.call("l1f_spectral_norm_f64", dv.ptr(t), t.shape[0], t.shape[1], int(iters), ctypes.addressof(out),
              dv.stream())
    return float(out.value)


def solve_pcp_device(t, cfg):
    """Run the ALM loop on a float64 CUDA matrix; returns (L, S, info dict)."""
    m, n = t.shape
    lam = cfg.lam if cfg.lam is not None else default_lambda(m, n)
    l = dv.empty((m, n))
    s = dv.empty((m, n))
    iters, rank, conv = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    resid, beta_final = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _lib.call("l1f_pcp_f64", dv.ptr(t), m, n, float(lam), float(cfg.tol),
              float(cfg.beta0) if cfg.beta0 is not None else 0.0, float(cfg.rho),
              float(cfg.beta_max) if cfg.beta_max is not None else 0.0, int(cfg.max_iter),
              dv.ptr(l), dv.ptr(s), ctypes.addressof(iters), ctypes.addressof(resid), ctypes.addressof(rank),
              ctypes.addressof(conv), ctypes.addressof(beta_final), dv.stream())
    info = dict(iterations=int(iters.value), final_residual=float(resid.value), rank=int(rank.value),
                converged=bool(conv.value), beta_final=float(beta_final.value), lam=lam)
    return l, s, info


def solve_pcp(m, cfg=None):
    """Solve PCP by ADM (pcp_adm.py:90-140). Returns a PcpSolution; converged=False flags
    max_iter exhaustion with final_residual above tol."""
    t0 = time.perf_counter()
    m = as_dense(m)
    host = isinstance(m, np.ndarray)
    if (m.size if host else m.numel()) == 0:
        raise ValueError("matrix must be nonempty")
    cfg = cfg or AdmConfig()
    t, _ = dv.as_device(m, keep_f32=False)
    l, s, info = solve_pcp_device(t, cfg)
    # the zero-matrix early exit carries no stats (pcp_adm.py:100-105)
    stats = {"beta_final": info["beta_final"], "lambda": info["lam"]} if info["beta_final"] else {}
    return PcpSolution(
        l=dv.to_host_if(l, host), s=dv.to_host_if(s, host), iterations=info["iterations"],
        final_residual=info["final_residual"], rank_of_l=info["rank"], elapsed=time.perf_counter() - t0,
        converged=info["converged"], stats=stats,
    )
