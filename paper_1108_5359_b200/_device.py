"""Device plumbing: torch tensors for memory and streams, the C-ABI for all compute.

Type policy of the drop-in API (mirrors the reference's numpy-in/numpy-out contract):
  * numpy / array-like inputs are coerced like ``as_dense`` (float64) and the results come
    back as new float64 numpy arrays;
  * torch CUDA tensors stay on the device (float32 is kept as float32 — the benchmark
    path — anything else becomes float64) and results are torch tensors.
"""

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


def require_cuda():
    """Fail loudly when there is no GPU or no native library; there is no CPU fallback."""
    if torch is None or not torch.cuda.is_available():
        raise _lib.NativeUnavailable("a CUDA device is required: l1pcp_b200 has no CPU path")
    _lib.load()


def is_tensor(a):
    return torch is not None and isinstance(a, torch.Tensor)


def stream():
    return torch.cuda.current_stream().cuda_stream


def dtype_code(t):
    return _lib.F32 if t.dtype == torch.float32 else _lib.F64


def ptr(t):
    return None if t is None else t.data_ptr()


def as_device(a, keep_f32=True):
    """Return (contiguous CUDA tensor, came_from_host)."""
    require_cuda()
    if is_tensor(a):
        t = a
        if t.dtype not in (torch.float32, torch.float64) or (t.dtype == torch.float32 and not keep_f32):
            t = t.to(torch.float64)
        if not t.is_cuda:
            t = t.cuda()
        return t.contiguous(), False
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if not arr.flags.writeable:  # e.g. np.frombuffer from a file read: torch needs a writable array
        arr = arr.copy()
    if arr.size >= BIG_HOST:
        return _staged_h2d(arr), True
    return torch.from_numpy(arr).cuda(), True


_STAGE = {}


def _staged_h2d(arr, chunk_bytes=64 << 20):
    """Large host array -> device through two reusable pinned chunks: the (multi-threaded) host
    copy of chunk i + 1 overlaps the DMA of chunk i; ~3x the pageable copy rate."""
    out = torch.empty(arr.shape, dtype=torch.float64, device="cuda")
    flat_src = torch.from_numpy(arr).reshape(-1)
    flat_dst = out.reshape(-1)
    n = flat_src.numel()
    per = chunk_bytes // 8
    if "bufs" not in _STAGE:
        _STAGE["bufs"] = [torch.empty(per, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        _STAGE["events"] = [torch.cuda.Event(), torch.cuda.Event()]
        _STAGE["stream"] = torch.cuda.Stream()
    bufs, evs, st = _STAGE["bufs"], _STAGE["events"], _STAGE["stream"]
    st.wait_stream(torch.cuda.current_stream())
    for i, off in enumerate(range(0, n, per)):
        b = i & 1
        m = min(per, n - off)
        evs[b].synchronize()  # the DMA that last read this buffer is done
        bufs[b][:m].copy_(flat_src[off:off + m])
        with torch.cuda.stream(st):
            flat_dst[off:off + m].copy_(bufs[b][:m], non_blocking=True)
            evs[b].record(st)
    torch.cuda.current_stream().wait_stream(st)
    out.record_stream(st)
    return out


# host arrays at least this large (elements) take the parallel host paths below
BIG_HOST = 1 << 22


def to_host_if(t, host):
    """A new float64 numpy array for host callers (the reference returns fresh numpy arrays).
    Large results are copied into a numpy buffer whose pages were first touched on all host cores
    (first-touch page faults of a fresh multi-GB allocation otherwise cost more than the copy)."""
    if not host:
        return t
    t = t.detach()
    if t.numel() < BIG_HOST:
        return t.to("cpu", torch.float64).numpy()
    out = np.empty(tuple(t.shape), dtype=np.float64)
    ho = torch.from_numpy(out)
    ho.zero_()  # parallel first touch
    ho.copy_(t if t.dtype == torch.float64 else t.to(torch.float64))
    return out


def empty(shape, dtype=None, like=None):
    dt = dtype if dtype is not None else (like.dtype if like is not None else torch.float64)
    return torch.empty(shape, dtype=dt, device="cuda")


def zeros(shape, dtype=None, like=None):
    dt = dtype if dtype is not None else (like.dtype if like is not None else torch.float64)
    return torch.zeros(shape, dtype=dt, device="cuda")


def transpose(t):
    """Materialised transpose through the C-ABI gather kernel (out[c][r] = t[r][c])."""
    r, c = t.shape
    out = empty((c, r), like=t)
    code = dtype_code(t)
    _lib.call("l1f_gather", code, ptr(t), t.stride(0), None, r, None, c, code, ptr(out), r, 1, stream())
    return out


def norms(t, thr=0.0):
    """(sum|x|, max|x|, sum x^2, count(|x|>thr), count(non-finite)) on the device."""
    t = t.contiguous()
    out = zeros(5, dtype=torch.float64)
    rows = t.shape[0] if t.dim() == 2 else 1
    cols = t.shape[1] if t.dim() == 2 else t.numel()
    _lib.call("l1f_norms", dtype_code(t), ptr(t), rows, cols, cols, float(thr), ptr(out), stream())
    return out.cpu().tolist()


def gemm_nt(a, b, alpha=1.0, k=None, out=None, beta=0.0):
    """alpha * a[:, :k] @ b[:, :k].T (+ beta * out) with the C-ABI tile GEMM."""
    m, n = a.shape[0], b.shape[0]
    kk = a.shape[1] if k is None else k
    if out is None:
        out = empty((m, n), like=a)
        beta = 0.0
    _lib.call("l1f_gemm_nt", dtype_code(a), m, n, kk, float(alpha), ptr(a), a.stride(0), ptr(b), b.stride(0),
              float(beta), ptr(out), out.stride(0), stream())
    return out
