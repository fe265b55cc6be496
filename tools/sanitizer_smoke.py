"""compute-sanitizer smoke: a few small calls of every kernel family (two-Q-tile
fast/causal, exact, half-INT8, FP8).  Run as
  compute-sanitizer --tool memcheck python tools/sanitizer_smoke.py"""
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2409_16997_b200 as ifa
from oracle_bindings import Oracle
o = Oracle()
for (n, d, fast, causal) in [(200, 100, True, False), (384, 128, True, True), (130, 64, False, False)]:
    q, k, v = [np.stack([x]) for x in o.slice_inputs("normal", n, d, seed=1)]
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inp = ifa.QuantizedAttentionInputs(ifa.quantize_per_row(dev(q)), ifa.quantize_per_row(dev(k)),
                                       ifa.quantize_per_tensor(dev(v)))
    out = ifa.int_flash_attention(inp, ifa.AttentionConfig(ifa.BlockSpec(64, 128), causal=causal, fast=fast))
    torch.cuda.synchronize()
    print(n, d, fast, causal, float(out.abs().sum()))
x = torch.randn(2, 256, 128, device="cuda")
ifa.half_int8_attention(ifa.quantize_per_row(x), ifa.quantize_per_row(x), x)
ifa.fp8_emulated_attention(x, x, x)
torch.cuda.synchronize()
print("done")
