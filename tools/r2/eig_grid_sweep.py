import sys, time, torch
sys.path.insert(0, '.')
from paper_1108_5359_b200 import engine, _lib
torch.manual_seed(0)
for p, r in ((1000, 100), (2000, 200)):
    a = torch.randn(p, r, dtype=torch.float64, device="cuda") @ torch.randn(r, p, dtype=torch.float64, device="cuda")
    for g in (0,):
        with _lib.options(seed_eig=0):
            engine.svd_device(a, gram=True); torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3): engine.svd_device(a, gram=True)
            torch.cuda.synchronize()
        print(f"p={p} grid={g}: {(time.perf_counter()-t0)/3*1e3:.1f} ms", flush=True)
    with _lib.options(seed_eig=1):
        engine.svd_device(a, gram=True); torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3): engine.svd_device(a, gram=True)
        torch.cuda.synchronize()
    print(f"p={p} syevd: {(time.perf_counter()-t0)/3*1e3:.1f} ms", flush=True)
