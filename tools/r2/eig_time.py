import sys, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import engine, _lib
p = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
r = int(sys.argv[2]) if len(sys.argv) > 2 else 100
torch.manual_seed(0)
a = torch.randn(p, r, dtype=torch.float64, device="cuda") @ torch.randn(r, p, dtype=torch.float64, device="cuda")
with _lib.options(seed_eig=0):
    for _ in range(2):
        engine.svd_device(a, gram=True)
torch.cuda.synchronize()
