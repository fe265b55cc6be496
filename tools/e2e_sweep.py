"""e2e through ifa_int_flash_fwd_host at C2 for several pipeline chunk sizes
(IFA_B200_HOST_CHUNK), plus the raw pinned H2D / D2H / bidirectional rates."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
from paper_2409_16997_b200.runtime import AttentionPlan  # noqa: E402

dev = torch.device("cuda", 0)
slices, N, d = 128, 4096, 128
plan = AttentionPlan(slices, N, d, bc=128, fast=True, device=dev)
q, k, v = (torch.randn(slices, N, d, device=dev) for _ in range(3))
plan.forward(q, k, v)
torch.cuda.synchronize()
ops = slices * bench.attn_ops(N, d, False)
# raw copy rates
hb = torch.empty(268435456, dtype=torch.uint8).pin_memory()
db = torch.empty(268435456, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: db.copy_(hb, non_blocking=True)),
                 ("d2h", lambda: hb.copy_(db, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{name}: {hb.numel() / dt / 1e9:.1f} GB/s")
hb2 = torch.empty_like(hb).pin_memory(); db2 = torch.empty_like(db)
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): db.copy_(hb, non_blocking=True)
with torch.cuda.stream(s2): hb2.copy_(db2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"bidirectional: {2 * hb.numel() / dt / 1e9:.1f} GB/s total")
for c in ("0", "4", "8", "16", "32", "64"):
    os.environ["IFA_B200_HOST_CHUNK"] = c
    r = bench.e2e_plugin_run(torch, plan, slices, N, d, 128, False, True, dev, ops, 5)
    print(f"chunk {c:>3}: {r['ms_per_step']:.3f} ms  {r['value']:.1f} TOPS")
