"""ctypes binding of the C-ABI library ``libl1pcp_b200.so`` (declared in include/l1pcp_b200.h).

The library is built in-tree (``paper_1108_5359_b200/_lib/``) by ``__graft_entry__.build()``
or ``make -C paper_1108_5359_b200/csrc``.  There is no fallback: if the library or a CUDA
device is missing, every compute entry point raises :class:`NativeUnavailable`.
"""

import ctypes
import glob
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libl1pcp_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "l1pcp_b200.h")

L1F_OK = 0
L1F_ERR_ARG = -1
L1F_ERR_CUDA = -2
L1F_ERR_SVD = -3
L1F_ERR_DIVERGED = -4
L1F_ERR_UNSUPPORTED = -5

F32 = 0
F64 = 1

UNIT_OK, UNIT_STALLED, UNIT_MAXITER, UNIT_ZERO = 0, 1, 2, 3
GEN_GAUSSIAN, GEN_VIDEO = 0, 1


class NativeUnavailable(RuntimeError):
    """The CUDA extension (or a CUDA device) is not available; there is no CPU fallback."""


class NativeError(RuntimeError):
    """A C-ABI call returned an error status."""

    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f32 = ctypes.c_float
_f64 = ctypes.c_double
_sz = ctypes.c_size_t
_int = ctypes.c_int

# name -> (restype, argtypes); mirrors include/l1pcp_b200.h
SIGNATURES = {
    "l1f_last_error": (ctypes.c_char_p, []),
    "l1f_set_option": (_int, [_int, _i64]),
    "l1f_get_option": (_int, [_int, _vp]),
    "l1f_version": (_int, []),
    "l1f_init": (_int, [_vp]),
    "l1f_sm_count": (_int, [_vp]),
    "l1f_filter_workspace_bytes": (_sz, [_int, _i32, _i32, _i64]),
    "l1f_filter_f32": (_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _f32, _f32, _f32, _f32, _i32,
                              _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1f_filter_f64": (_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _f64, _f64, _f64, _f64, _i32,
                              _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "l1f_filter_pair_f32": (_int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp,
                                   _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp,
                                   _i32, _i32, _f32, _f32, _f32, _f32, _i32, _i32, _vp]),
    "l1f_filter_pair_plan_f32": (_int, [_i32, _i32, _i64, _i64, _vp]),
    "l1f_gather": (_int, [_int, _vp, _i64, _vp, _i64, _vp, _i64, _int, _vp, _i64, _i32, _vp]),
    "l1f_build_factors": (_int, [_int, _i64, _i64, _i32, _vp, _i64, _vp, _i64, _vp, _vp, _vp,
                                 _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "l1f_reconstruct": (_int, [_int, _i64, _i64, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                               _vp, _i64, _vp, _vp]),
    "l1f_rowfilter_reconstruct_f32": (_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _f32, _f32, _f32, _f32, _i32,
                                             _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                                             _vp, _i64,
                                             _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "l1f_rowfilter_reconstruct_small": (_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _f64, _f64, _f64, _f64, _i32,
                                               _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                                               _vp, _i64,
                                               _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp]),
    "l1f_filter_with_gather_f32": (_int, [_vp, _i64, _i32, _i64, _vp, _i64, _i32, _f32, _f32, _f32, _f32, _i32,
                                          _vp, _i64, _vp, _vp, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _i64,
                                          _vp, _i64, _i32, _vp]),
    "l1f_gemm_nt": (_int, [_int, _i64, _i64, _i64, _f64, _vp, _i64, _vp, _i64, _f64, _vp, _i64, _vp]),
    "l1f_generate_factors_f32": (_int, [_u64, _i32, _i64, _i64, _i32, _vp, _vp, _vp]),
    "l1f_generate_f32": (_int, [_u64, _i32, _i64, _i64, _i32, _f32, _f32, _vp, _vp, _i64, _i64,
                                _vp, _i64, _vp, _i64, _vp]),
    "l1f_generate_sparse_exact": (_int, [_int, _u64, _i64, _i64, _i64, _f64, _vp, _vp]),
    "l1f_norms": (_int, [_int, _vp, _i64, _i64, _i64, _f64, _vp, _vp]),
    "l1f_diff_norms": (_int, [_int, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _vp]),
    "l1f_soft_threshold": (_int, [_int, _vp, _vp, _i64, _f64, _vp]),
    "l1f_svd_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "l1f_svd_gram_f64": (_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "l1f_spectral_norm_f64": (_int, [_vp, _i64, _i64, _i32, _vp, _vp]),
    "l1f_svt_f64": (_int, [_vp, _i64, _i64, _f64, _vp, _vp, _vp]),
    "l1f_pcp_f64": (_int, [_vp, _i64, _i64, _f64, _f64, _f64, _f64, _f64, _i32, _vp, _vp, _vp, _vp,
                           _vp, _vp, _vp, _vp]),
    "l1f_fma_peak_probe": (_int, [_i32, _vp, _vp, _vp]),
    "l1f_fma_peak_probe_f64": (_int, [_i32, _vp, _vp, _vp]),
}

# library options (include/l1pcp_b200.h L1F_OPT_*): explicit process-wide switches of the kernel
# selection; the defaults are the production choices
C_OPTIONS = {"filter_streaming": 1, "filter_tc": 2, "tc_groups": 3, "recon_tc": 4, "recon_stream": 5,
             "recon_concurrent": 6, "gather_overlap": 7, "wait_timeout_ms": 8, "small_lanes": 9, "seed_eig": 10,
             "seed_small_svt": 11, "seed_eig_dsm": 12}
# host-side choices of the Python engine: the paired column+row filter call, the streamed form of
# the sharded step (None = the library's pass model), the rank up to which the filter runs in FP64
PY_OPTIONS = {"filter_pair": True, "sharded_stream": None, "small_k_fp64": 16}


_c_option_cache = {}  # last value set through this module (the library's options change only via set_option)


def set_option(name, value):
    """Set one option (C_OPTIONS: in the library; PY_OPTIONS: in the engine)."""
    if name in C_OPTIONS:
        call("l1f_set_option", C_OPTIONS[name], int(value))
        _c_option_cache[name] = int(value)
    elif name in PY_OPTIONS:
        PY_OPTIONS[name] = value
    else:
        raise ValueError(f"unknown option {name!r}")


def get_option(name):
    if name in _c_option_cache:  # hot path (engine checks per step): no ctypes round trip
        return _c_option_cache[name]
    if name in C_OPTIONS:
        v = ctypes.c_int64(0)
        call("l1f_get_option", C_OPTIONS[name], ctypes.addressof(v))
        _c_option_cache[name] = int(v.value)
        return int(v.value)
    if name in PY_OPTIONS:
        return PY_OPTIONS[name]
    raise ValueError(f"unknown option {name!r}")


class options:
    """Context manager: ``with _lib.options(recon_concurrent=0): ...`` sets options and restores
    the previous values on exit (tests and A/B comparisons)."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


_lock = threading.Lock()
_lib = None


def _preload_cuda_libraries():
    """Make the CUDA math libraries resolve to the copies torch already uses.

    torch ships its own cuBLAS/cuSOLVER; loading those (RTLD_GLOBAL) before our library
    keeps one consistent set in the process.  Outside a torch environment the library's
    RPATH (/usr/local/cuda/lib64) is used instead.
    """
    try:
        import nvidia  # noqa: F401  (namespace package of the CUDA wheels)
    except ImportError:
        return
    roots = [os.path.dirname(p) for p in getattr(__import__("nvidia"), "__path__", [])]
    for sub, names in (("cublas", ("libcublasLt.so.*", "libcublas.so.*")),
                       ("cusolver", ("libcusolver.so.*",))):
        for root in roots:
            for pat in names:
                for path in sorted(glob.glob(os.path.join(root, "nvidia", sub, "lib", pat))):
                    try:
                        ctypes.CDLL(path, mode=ctypes.RTLD_GLOBAL)
                    except OSError:
                        pass


def load(path=None):
    """Load (once) and return the ctypes handle of the C-ABI library."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeUnavailable(
                f"{p} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_1108_5359_b200/csrc`")
        try:
            import torch  # noqa: F401  (loads torch's CUDA libraries first)
        except ImportError:
            pass
        _preload_cuda_libraries()
        lib = ctypes.CDLL(p, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        _init_device(lib)
        return lib


def _init_device(lib):
    """One-time device initialisation (l1f_init: cuBLAS handle and first GEMMs, eigensolver kernels)
    when a GPU is present, so that it is not charged to the first solve."""
    try:
        import torch
        if not torch.cuda.is_available():
            return
    except ImportError:
        return
    code = lib.l1f_init(None)
    if code != 0:
        raise NativeError(f"l1f_init failed ({code}): {lib.l1f_last_error().decode(errors='replace')}")


def last_error():
    return load().l1f_last_error().decode(errors="replace")


def check(code, what=""):
    """Raise the reference's exception type for a non-zero status."""
    if code == L1F_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if code == L1F_ERR_ARG:
        raise ValueError(msg)
    if code == L1F_ERR_SVD:
        from .matcore import SvdConvergenceError
        raise SvdConvergenceError(msg)
    if code == L1F_ERR_DIVERGED:
        from .pcp_adm import PcpDivergenceError
        raise PcpDivergenceError(msg)
    raise NativeError(code, msg)


def call(name, *args, what=None):
    code = getattr(load(), name)(*args)
    check(code, what or name)
    return code
