import sys; sys.path.insert(0, '.')
import torch, numpy as np
from paper_1108_5359_b200 import engine, _lib
from paper_1108_5359_b200 import _device as dv
h = torch.arange(64 * 100, dtype=torch.float32).reshape(64, 100).pin_memory()
rows = np.array([3, 7, 60]); cols = np.array([1, 50, 99])
out = torch.empty((3, 3), dtype=torch.float32, device="cuda")
rt, ct = engine.index_tensor(rows), engine.index_tensor(cols)
_lib.call("l1f_gather", _lib.F32, h.data_ptr(), h.stride(0), dv.ptr(rt), 3, dv.ptr(ct), 3, _lib.F32, dv.ptr(out), 3, 0, dv.stream())
torch.cuda.synchronize()
print(out.cpu().numpy(), h[rows][:, cols].numpy(), torch.cuda.cudart().cudaHostGetDevicePointer if hasattr(torch.cuda.cudart(),'cudaHostGetDevicePointer') else '')
