"""Zero-copy column-panel gather from pinned host M (HostPipeline's first step): time and PCIe GB/s."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import _device as dv, _lib
m = n = 20000
s = 1000
mh = torch.randn(m, n).pin_memory()
rng = np.random.default_rng(0)
rows = np.sort(rng.choice(m, s, replace=False)); cols = np.setdiff1d(np.arange(n), np.sort(rng.choice(n, s, replace=False)))
dr = torch.as_tensor(rows, device='cuda'); dc = torch.as_tensor(cols, device='cuda')
xc = torch.empty((len(cols), s), device='cuda')
def run():
    _lib.call("l1f_gather", _lib.F32, mh.data_ptr(), mh.stride(0), dv.ptr(dr), s, dv.ptr(dc), len(cols), _lib.F32,
              dv.ptr(xc), xc.stride(0), 1, dv.stream())
run(); torch.cuda.synchronize()
assert torch.equal(xc.cpu(), mh[rows][:, cols].T.contiguous())
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): run()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print(f"zero-copy gather {s}x{len(cols)}: {ms:.3f} ms, {s * len(cols) * 4 / ms / 1e6:.1f} GB/s")
