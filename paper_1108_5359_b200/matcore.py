"""Dense primitives of the reference API on the device (mirrors pkg/src/l1pcp/matcore.py).

Norms, shrinkage, thin SVD, SVT and pseudo-inverse application, each executed by the
C-ABI library (include/l1pcp_b200.h).  numpy inputs return numpy float64 results like the
reference; CUDA tensors stay on the device.
"""

from dataclasses import dataclass

import numpy as np

from . import _device as dv
from . import _lib


class SvdConvergenceError(RuntimeError):
    """The underlying SVD factorization failed to converge (matcore.py:9-10)."""


def as_dense(a):
    """Coerce *a* to a 2-D matrix, rejecting NaN/Inf entries (matcore.py:13-20).

    Array-likes become C-contiguous float64 numpy arrays exactly as in the reference;
    torch tensors become contiguous CUDA tensors (float32 kept) validated on the device.
    """
    if dv.is_tensor(a):
        if a.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got ndim={a.dim()}")
        t, _ = dv.as_device(a)
        if t.numel() and dv.norms(t)[4] > 0:
            raise ValueError("matrix contains non-finite entries")
        return t
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={arr.ndim}")
    arr = np.ascontiguousarray(arr)
    if arr.size >= dv.BIG_HOST:  # the same check on all host cores (torch's parallel CPU kernels)
        finite = bool(dv.torch.isfinite(dv.torch.from_numpy(arr)).all())
    else:
        finite = bool(np.isfinite(arr).all())
    if not finite:
        raise ValueError("matrix contains non-finite entries")
    return arr


@dataclass(frozen=True)
class SkinnySvd:
    """Skinny SVD: u (m x k) and v (n x k) with orthonormal columns, sigma strictly positive
    and nonincreasing (matcore.py:23-38)."""

    u: object
    sigma: object
    v: object

    @property
    def rank(self):
        return int(self.sigma.shape[0])

    def reconstruct(self):
        """Return u @ diag(sigma) @ v.T (rank-k product on the device)."""
        host = not dv.is_tensor(self.u)
        u, _ = dv.as_device(self.u, keep_f32=False)
        v, _ = dv.as_device(self.v, keep_f32=False)
        s, _ = dv.as_device(np.asarray(self.sigma) if host else self.sigma, keep_f32=False)
        m, n, k = u.shape[0], v.shape[0], self.rank
        if k == 0:
            out = dv.zeros((m, n))
        else:
            us = u * s.reshape(1, -1)
            out = dv.gemm_nt(us.contiguous(), v.contiguous(), k=k)
        return dv.to_host_if(out, host)


def _scalar_norms(m, thr=0.0):
    if dv.is_tensor(m):
        t, _ = dv.as_device(m)
    else:
        arr = np.asarray(m, dtype=np.float64)
        if arr.size == 0:
            return [0.0, 0.0, 0.0, 0.0, 0.0]
        t, _ = dv.as_device(np.atleast_2d(arr))
    if t.numel() == 0:
        return [0.0, 0.0, 0.0, 0.0, 0.0]
    return dv.norms(t.reshape(t.shape[0], -1) if t.dim() >= 2 else t.reshape(1, -1), thr)


def frobenius_norm(m):
    return float(np.sqrt(_scalar_norms(m)[2]))


def l1_norm(m):
    return float(_scalar_norms(m)[0])


def linf_norm(m):
    return float(_scalar_norms(m)[1])


def l0_count(m, threshold=None):
    """Count entries with |x| > threshold; default 1e-6 * ||m||_inf (matcore.py:53-63)."""
    if threshold is None:
        threshold = 1e-6 * linf_norm(m)
    if threshold < 0:
        raise ValueError("threshold must be nonnegative")
    return int(_scalar_norms(m, threshold)[3])


def soft_threshold(m, eta):
    """Elementwise soft shrinkage sgn(x) * max(|x| - eta, 0) (matcore.py:66-70)."""
    if eta < 0:
        raise ValueError("eta must be nonnegative")
    t, host = dv.as_device(m)
    out = dv.empty(t.shape, like=t)
    _lib.call("l1f_soft_threshold", dv.dtype_code(t), dv.ptr(t), dv.ptr(out), t.numel(), float(eta), dv.stream())
    return dv.to_host_if(out, host)


def _svd_full(t):
    """Thin SVD of a float64 CUDA matrix: (u m x p, sigma p, v n x p), sigma descending."""
    m, n = t.shape
    p = min(m, n)
    u = dv.empty((m, p))
    s = dv.empty((p,))
    v = dv.empty((n, p))
    _lib.call("l1f_svd_f64", dv.ptr(t), m, n, t.stride(0), dv.ptr(u), dv.ptr(s), dv.ptr(v), dv.stream(),
              what=f"SVD failed on {tuple(t.shape)} matrix")
    return u, s, v


def svd(m, rank_tol=1e-8):
    """Skinny SVD of *m*, dropping singular values <= rank_tol * sigma_max (matcore.py:73-88).

    Exact zeros are always dropped, so the result has strictly positive singular values
    even at rank_tol=0.
    """
    if rank_tol < 0:
        raise ValueError("rank_tol must be nonnegative")
    t, host = dv.as_device(m, keep_f32=False)
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={t.dim()}")
    if t.numel() == 0:
        z = dv.empty((t.shape[0], 0)), dv.empty((0,)), dv.empty((t.shape[1], 0))
        return SkinnySvd(*(dv.to_host_if(a, host) for a in z))
    u, s, v = _svd_full(t)
    sh = s.cpu().numpy()
    cutoff = rank_tol * (sh[0] if sh.size else 0.0)
    k = int((sh > cutoff).sum())
    u, s, v = u[:, :k].contiguous(), s[:k].contiguous(), v[:, :k].contiguous()
    return SkinnySvd(u=dv.to_host_if(u, host), sigma=dv.to_host_if(s, host), v=dv.to_host_if(v, host))


def nuclear_norm(m):
    """Sum of singular values."""
    t, _ = dv.as_device(m, keep_f32=False)
    if t.numel() == 0:
        return 0.0
    _, s, _ = _svd_full(t)
    return float(s.sum().item())


def svt_with_rank(w, eta):
    """Singular value thresholding, returning (matrix, retained_rank) (matcore.py:96-105)."""
    if eta < 0:
        raise ValueError("eta must be nonnegative")
    t, host = dv.as_device(w, keep_f32=False)
    m, n = t.shape
    out = dv.empty((m, n))
    rank = _lib._i32(0)
    import ctypes
    _lib.call("l1f_svt_f64", dv.ptr(t), m, n, float(eta), dv.ptr(out), ctypes.addressof(rank), dv.stream())
    return dv.to_host_if(out, host), int(rank.value)


def svt(w, eta):
    """Singular value thresholding: U S_eta(Sigma) V^T (matcore.py:108-113)."""
    return svt_with_rank(w, eta)[0]


def pseudo_inverse_apply(f, rhs):
    """Apply V Sigma^{-1} U^T to *rhs* using the retained singular values (matcore.py:116-123)."""
    host = not dv.is_tensor(rhs)
    r, _ = dv.as_device(np.asarray(rhs, dtype=np.float64) if host else rhs, keep_f32=False)
    if r.dim() == 1:
        r = r.reshape(-1, 1)
    u, _ = dv.as_device(f.u, keep_f32=False)
    v, _ = dv.as_device(f.v, keep_f32=False)
    s, _ = dv.as_device(np.asarray(f.sigma) if not dv.is_tensor(f.sigma) else f.sigma, keep_f32=False)
    if u.shape[0] != r.shape[0]:
        raise ValueError(f"dimension mismatch: factor has {u.shape[0]} rows, rhs has {r.shape[0]}")
    k = int(s.shape[0])
    # (U^T rhs) = (rhs^T U)^T ; then / sigma ; then V (.)
    ut_r = dv.gemm_nt(dv.transpose(u), dv.transpose(r)) if k else dv.zeros((0, r.shape[1]))
    scaled = (ut_r / s.reshape(-1, 1)).contiguous()
    out = dv.gemm_nt(v, dv.transpose(scaled), k=k) if k else dv.zeros((v.shape[0], r.shape[1]))
    return dv.to_host_if(out, host)
