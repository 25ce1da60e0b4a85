"""Matrix files: the reference's CSV and DMAT formats, plus device readers and
writers that stream the float64 payload between the file and HBM.

Formats (pkg/src/l1pcp/matio.py:1-17):
  * CSV: one matrix row per line, comma separated.
  * DMAT: 16-byte header (magic b"DMAT", u32 rows, u32 cols, little endian, 4 pad bytes) then
    rows * cols little-endian float64 values, row major.

Host functions keep the reference's names, validation and errors (ValueError on a short header,
bad magic or wrong payload size; `as_dense` on every matrix).  The device functions move a DMAT
payload through two pinned float64 staging buffers: the file read of chunk i+1 overlaps the
host->device copy of chunk i, and the dtype conversion runs on the GPU (l1f_gather with no index
lists), so a float64 file lands as a float32 (or float64) CUDA tensor without a host-side
conversion pass.
"""

import os
import struct

import numpy as np

from .matcore import as_dense

MAGIC = b"DMAT"
_HEADER = struct.Struct("<4sII4x")
_CHUNK_BYTES = 64 << 20  # staging chunk for the device paths


# ------------------------------------------------------------------ host (reference semantics)
def write_csv(path, m):
    m = as_dense(m)
    np.savetxt(path, m, delimiter=",", fmt="%.17g")


def read_csv(path):
    m = np.loadtxt(path, delimiter=",", ndmin=2)
    return as_dense(m)


def _read_header(fh, path):
    header = fh.read(_HEADER.size)
    if len(header) < _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, rows, cols = _HEADER.unpack(header)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    return rows, cols


def write_dmat(path, m):
    m = as_dense(m)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, m.shape[0], m.shape[1]))
        fh.write(m.astype("<f8").tobytes(order="C"))


def read_dmat(path):
    with open(path, "rb") as fh:
        rows, cols = _read_header(fh, path)
        data = np.frombuffer(fh.read(), dtype="<f8")
    if data.size != rows * cols:
        raise ValueError(f"{path}: expected {rows * cols} values, got {data.size}")
    return as_dense(data.reshape(rows, cols))


def read_matrix(path):
    """Read a matrix, picking the format from the extension (.csv) or the DMAT magic."""
    path = str(path)
    if path.endswith(".csv"):
        return read_csv(path)
    with open(path, "rb") as fh:
        head = fh.read(4)
    if head == MAGIC:
        return read_dmat(path)
    return read_csv(path)


def write_matrix(path, m):
    """Write a matrix; a .csv extension selects CSV, anything else DMAT."""
    if str(path).endswith(".csv"):
        write_csv(path, m)
    else:
        write_dmat(path, m)


# ------------------------------------------------------------------ device paths
def _convert(src, dst):
    """dst[:] = src with a dtype change, on the device (l1f_gather without index lists)."""
    from . import _device as dv
    from . import _lib
    rows, cols = src.shape
    _lib.call("l1f_gather", dv.dtype_code(src), dv.ptr(src), src.stride(0), None, rows, None, cols,
              dv.dtype_code(dst), dv.ptr(dst), dst.stride(0), 0, dv.stream())


def read_dmat_device(path, dtype=None):
    """DMAT file -> CUDA tensor (float32 by default).  Streams the payload in row chunks through
    two pinned float64 buffers; the conversion runs on the GPU.  Same errors as read_dmat."""
    from . import _device as dv
    torch = dv.torch
    dv.require_cuda()
    dtype = dtype or torch.float32
    path = str(path)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        rows, cols = _read_header(fh, path)
        if size - _HEADER.size != 8 * rows * cols:
            raise ValueError(f"{path}: expected {rows * cols} values, got {(size - _HEADER.size) // 8}")
        out = torch.empty((rows, cols), dtype=dtype, device="cuda")
        if rows == 0 or cols == 0:
            return out
        crow = max(1, min(rows, _CHUNK_BYTES // (8 * cols)))
        stage = [torch.empty((crow, cols), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        dbuf = [torch.empty((crow, cols), dtype=torch.float64, device="cuda") for _ in range(2)]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        copy = torch.cuda.Stream()
        comp = torch.cuda.current_stream()
        for i, r0 in enumerate(range(0, rows, crow)):
            b = i & 1
            nr = min(crow, rows - r0)
            done[b].synchronize()  # staging buffer b is free again (its previous copy finished)
            view = stage[b][:nr].numpy().reshape(-1)
            got = fh.readinto(memoryview(view).cast("B"))
            if got != 8 * nr * cols:
                raise ValueError(f"{path}: truncated payload")
            if not np.little_endian:
                view.byteswap(inplace=True)
            with torch.cuda.stream(copy):
                copy.wait_stream(comp)
                dbuf[b][:nr].copy_(stage[b][:nr], non_blocking=True)
                _convert(dbuf[b][:nr], out[r0:r0 + nr])
                done[b].record(copy)
        comp.wait_stream(copy)
    return out


def write_dmat_device(path, t):
    """CUDA tensor -> DMAT file (float64 payload).  Converts on the GPU and streams row chunks
    through two pinned buffers; the file write of chunk i overlaps the copy of chunk i+1."""
    from . import _device as dv
    torch = dv.torch
    if t.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    rows, cols = t.shape
    t = t.contiguous()
    with open(str(path), "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, rows, cols))
        if rows == 0 or cols == 0:
            return
        crow = max(1, min(rows, _CHUNK_BYTES // (8 * cols)))
        stage = [torch.empty((crow, cols), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        dbuf = [torch.empty((crow, cols), dtype=torch.float64, device="cuda") for _ in range(2)]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        copy = torch.cuda.Stream()
        copy.wait_stream(torch.cuda.current_stream())
        chunks = list(range(0, rows, crow))

        def launch(i):
            b = i & 1
            r0 = chunks[i]
            nr = min(crow, rows - r0)
            with torch.cuda.stream(copy):
                if t.dtype == torch.float64:
                    stage[b][:nr].copy_(t[r0:r0 + nr], non_blocking=True)
                else:
                    _convert(t[r0:r0 + nr], dbuf[b][:nr])
                    stage[b][:nr].copy_(dbuf[b][:nr], non_blocking=True)
                ready[b].record(copy)

        launch(0)
        for i in range(len(chunks)):
            if i + 1 < len(chunks):
                launch(i + 1)  # its buffer held chunk i - 1, written out in the previous iteration
            b = i & 1
            nr = min(crow, rows - chunks[i])
            ready[b].synchronize()
            arr = stage[b][:nr].numpy()
            if not np.little_endian:
                arr = arr.byteswap()
            fh.write(memoryview(np.ascontiguousarray(arr)).cast("B"))


def read_matrix_device(path, dtype=None):
    """read_matrix onto the device: DMAT files stream straight to HBM, CSV goes through numpy."""
    from . import _device as dv
    torch = dv.torch
    path = str(path)
    if not path.endswith(".csv"):
        with open(path, "rb") as fh:
            head = fh.read(4)
        if head == MAGIC:
            return read_dmat_device(path, dtype)
    return torch.as_tensor(read_csv(path)).to(device="cuda", dtype=dtype or torch.float32)


def write_matrix_device(path, t):
    """write_matrix from the device: .csv through numpy, anything else DMAT streamed from HBM."""
    if str(path).endswith(".csv"):
        write_csv(path, t.double().cpu().numpy())
    else:
        write_dmat_device(path, t)
