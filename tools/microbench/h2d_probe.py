"""PCIe copy probe: pinned H2D bandwidth with 1 and 3 streams, and H2D with a
concurrent D2H (what bounds bench.py's e2e number).  Measured on B200: 55.5 GB/s H2D,
46.5 GB/s H2D + 15.5 GB/s D2H concurrently."""
import torch, time
dev = torch.device("cuda:0")
n = 256 * 1024 * 1024 // 4  # 256 MB of f32
h = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in range(3)]
d = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
ho = torch.empty(n, dtype=torch.float32).pin_memory()
for streams in (1, 3):
    ss = [torch.cuda.Stream(dev) for _ in range(streams)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        for i in range(3):
            with torch.cuda.stream(ss[i % streams]):
                d[i].copy_(h[i], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.time() - t0
        print(f"H2D {streams} streams: {3*n*4/dt/1e9:.1f} GB/s")
# bidirectional
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
torch.cuda.synchronize(); t0 = time.time()
with torch.cuda.stream(s1):
    for i in range(3): d[i].copy_(h[i], non_blocking=True)
with torch.cuda.stream(s2):
    ho.copy_(d[0], non_blocking=True)
torch.cuda.synchronize(); dt = time.time() - t0
print(f"bidir: {3*n*4/dt/1e9:.1f} GB/s H2D with 1 GB D2H concurrently... total {(4*n*4)/dt/1e9:.1f}")
