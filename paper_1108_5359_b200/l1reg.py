"""Column-separable l1 regression by ADM on the device (mirrors pkg/src/l1pcp/l1reg.py).

    min ||E||_l1   s.t.   X = A Z + E,   A with orthonormal columns

Every column ("unit") carries its own penalty schedule and stopping threshold derived from
its linf norm (l1reg.py:59-137); all units are solved by one persistent CUDA kernel
(csrc/filter.cu) whose per-unit results do not depend on how units are grouped, so
``solve_l1reg`` and ``solve_l1reg_columnwise`` return identical results for any
``parallelism`` (the reference's bitwise contract, l1reg.py:183-186).
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _device as dv
from . import _lib
from .matcore import as_dense
from .pcp_adm import AdmConfig

STAGNATION_EPS = 1e-12
STAGNATION_ITERS = 20
CHUNK_COLS = 64

# ||A^T A - I||_inf tolerance of _check_dictionary (l1reg.py:52) for float64 dictionaries.
# A float32 dictionary (the FP32 benchmark path) is checked at its own precision.
ORTHO_TOL = {np.dtype("float64"): 1e-8, np.dtype("float32"): 1e-5}


@dataclass
class L1RegSolution:
    z: object
    e: object
    iterations: int
    final_residual: float
    converged: bool
    failed_columns: list = field(default_factory=list)


def _check_dictionary(a):
    """Reject dictionaries whose columns are not orthonormal (l1reg.py:48-56)."""
    a = as_dense(a)
    t, _ = dv.as_device(a)
    k = t.shape[1]
    t64 = t.to(dv.torch.float64) if t.dtype != dv.torch.float64 else t
    gram = dv.gemm_nt(dv.transpose(t64), dv.transpose(t64))  # A^T A, k x k
    gram -= dv.torch.eye(k, dtype=dv.torch.float64, device="cuda")
    dev = dv.norms(gram)[1] if k else 0.0
    tol = 1e-8 if t.dtype == dv.torch.float64 else 1e-5
    if dev > tol:
        raise ValueError(f"dictionary columns are not orthonormal (||A^T A - I||_inf = {dev:.3g})")
    return a


def filter_units(x_um, a, cfg, want_e=True, workspace=None):
    """Run the ADM kernel on a unit-major CUDA panel.

    x_um: (n_units, s) tensor, one unit per row; a: (s, k) tensor of the same dtype.
    Returns (z_um (n_units, k), e_um (n_units, s) or None, iters int32, res, status uint8).
    """
    n_units, s = x_um.shape
    k = a.shape[1]
    torch = dv.torch
    z = dv.empty((n_units, k), like=x_um)
    e = dv.empty((n_units, s), like=x_um) if want_e else None
    iters = torch.empty(n_units, dtype=torch.int32, device="cuda")
    res = dv.empty((n_units,), like=x_um)
    status = torch.empty(n_units, dtype=torch.uint8, device="cuda")
    if n_units == 0:
        return z, e, iters, res, status
    fn = "l1f_filter_f32" if x_um.dtype == torch.float32 else "l1f_filter_f64"
    beta0 = float(cfg.beta0) if cfg.beta0 is not None else 0.0
    beta_max = float(cfg.beta_max) if cfg.beta_max is not None else 0.0
    ws_ptr, ws_bytes = (None, 0) if workspace is None else (workspace.data_ptr(), workspace.numel())
    _lib.call(fn, dv.ptr(x_um), x_um.stride(0), s, n_units, dv.ptr(a), a.stride(0), k, float(cfg.tol),
              float(cfg.rho), beta0, beta_max, int(cfg.max_iter), dv.ptr(z), z.stride(0), dv.ptr(e),
              e.stride(0) if e is not None else s, dv.ptr(iters), dv.ptr(res), dv.ptr(status), ws_ptr, ws_bytes,
              dv.stream())
    return z, e, iters, res, status


def filter_units_pair(x1, a1, x2, a2, cfg, mode=0):
    """Two unit-major fp32 panels of the same width against their dictionaries in one call
    (l1f_filter_pair_f32): the column and row filters of the pipeline.  Returns
    ((z1, iters1, res1, status1), (z2, iters2, res2, status2)); no e output."""
    torch = dv.torch
    outs = []
    for x, a in ((x1, a1), (x2, a2)):
        n_units = x.shape[0]
        outs.append((dv.empty((n_units, a.shape[1]), like=x), torch.empty(n_units, dtype=torch.int32, device="cuda"),
                     dv.empty((n_units,), like=x), torch.empty(n_units, dtype=torch.uint8, device="cuda")))
    s, k = x1.shape[1], a1.shape[1]
    if x2.shape[1] != s or a2.shape[1] != k:
        raise ValueError("filter_units_pair: the two panels need the same s and k")
    beta0 = float(cfg.beta0) if cfg.beta0 is not None else 0.0
    beta_max = float(cfg.beta_max) if cfg.beta_max is not None else 0.0
    (z1, i1, r1, s1), (z2, i2, r2, s2) = outs
    _lib.call("l1f_filter_pair_f32", dv.ptr(x1), max(x1.stride(0), s), x1.shape[0], dv.ptr(a1), a1.stride(0),
              dv.ptr(z1), max(z1.stride(0), k), dv.ptr(i1), dv.ptr(r1), dv.ptr(s1), dv.ptr(x2), max(x2.stride(0), s),
              x2.shape[0], dv.ptr(a2), a2.stride(0), dv.ptr(z2), max(z2.stride(0), k), dv.ptr(i2), dv.ptr(r2),
              dv.ptr(s2), s, k, float(cfg.tol),
              float(cfg.rho), beta0, beta_max, int(cfg.max_iter), int(mode), dv.stream())
    return outs[0], outs[1]


def workspace_bytes(dtype_code, s, k, n_units):
    return int(_lib.load().l1f_filter_workspace_bytes(dtype_code, s, k, n_units))


def _solve(x, a, cfg):
    """Shared body of solve_l1reg / solve_l1reg_columnwise."""
    x = as_dense(x)
    a = _check_dictionary(a)
    host = isinstance(x, np.ndarray)
    if x.shape[0] != a.shape[0]:
        raise ValueError(f"row mismatch: X has {x.shape[0]}, A has {a.shape[0]}")
    cfg = cfg or AdmConfig()
    s, n_cols = x.shape
    k = a.shape[1]
    xt, _ = dv.as_device(x)
    at, _ = dv.as_device(a)
    if at.dtype != xt.dtype:
        at = at.to(xt.dtype)
    scale = dv.norms(xt)[1] if xt.numel() else 0.0
    if n_cols == 0 or scale == 0.0:
        z = dv.zeros((k, n_cols), like=xt)
        e = dv.zeros((s, n_cols), like=xt)
        return L1RegSolution(z=dv.to_host_if(z, host), e=dv.to_host_if(e, host), iterations=0,
                             final_residual=0.0, converged=True)
    x_um = dv.transpose(xt)  # (n_cols, s): unit-major panel
    z_um, e_um, iters, res, status = filter_units(x_um, at.contiguous(), cfg)
    z = dv.transpose(z_um)
    e = dv.transpose(e_um)
    it_h = iters.cpu().numpy()
    st_h = status.cpu().numpy()
    res_h = res.cpu().numpy().astype(np.float64)
    failed = np.flatnonzero((st_h == _lib.UNIT_STALLED) | (st_h == _lib.UNIT_MAXITER))
    return L1RegSolution(
        z=dv.to_host_if(z, host), e=dv.to_host_if(e, host), iterations=int(it_h.max(initial=0)),
        final_residual=float(res_h.max(initial=0.0)) / scale, converged=failed.size == 0,
        failed_columns=[int(c) for c in failed],
    )


def solve_l1reg(x, a, cfg=None):
    """Solve min ||E||_l1 s.t. X = A Z + E for orthonormal-column A (l1reg.py:140-160)."""
    return _solve(x, a, cfg)


def solve_l1reg_columnwise(x, a, cfg=None, parallelism=0):
    """Column-parallel variant of solve_l1reg with identical results (l1reg.py:163-214).

    ``parallelism`` is accepted for API compatibility; the device kernel's results are
    independent of any grouping of the columns.
    """
    return _solve(x, a, cfg)
