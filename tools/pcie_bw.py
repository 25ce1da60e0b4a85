"""PCIe copy bandwidth with 1..4 streams (pinned host), H2D and D2H, plus both directions at once."""
import torch, time
n = 3_200_000_000 // 4
dev = torch.empty(n, dtype=torch.float32, device="cuda")
host = torch.empty(n, dtype=torch.float32, pin_memory=True)
host2 = torch.empty(n // 2, dtype=torch.float32, pin_memory=True)
dev2 = torch.empty(n // 2, dtype=torch.float32, device="cuda")
def run(kind, ns):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            sl = slice(i * chunk, (i + 1) * chunk)
            if kind == "d2h": host[sl].copy_(dev[sl], non_blocking=True)
            else: dev[sl].copy_(host[sl], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{kind} streams={ns}: {n*4/dt/1e9:.1f} GB/s")
for kind in ("h2d", "d2h"):
    for ns in (1, 2, 4):
        run(kind, ns)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): host.copy_(dev, non_blocking=True)
with torch.cuda.stream(s2): dev2.copy_(host2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"duplex: d2h 3.2 GB + h2d 1.6 GB in {dt*1e3:.1f} ms")
