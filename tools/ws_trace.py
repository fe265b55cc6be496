"""Pipeline timeline of the attn_ws.cu kernel (CTA 0), from a build with
-DIFA_WS_TRACE=1:

  tools/build_variant.sh trace -DIFA_WS_TRACE=1
  IFA_B200_LIB=build/trace/libifa_b200.so python tools/ws_trace.py [slices n]

Prints, per tile of each group, the clock64 stamps (relative to the first
event) of: softmax S-ready / alpha posted / P buffer free / P published; MMA
S(next) issued / P ready / O ready / P.V issued; correction message / P.V(j-1)
done / o_ready.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2409_16997_b200 as ifa  # noqa: E402
from paper_2409_16997_b200 import _lib  # noqa: E402


def main():
    slices = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    d = 128
    from paper_2409_16997_b200.runtime import AttentionPlan
    plan = AttentionPlan(slices, n, d, fast=True)
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(slices, n, d, device="cuda", generator=g) for _ in range(3))
    plan.quantize(q, k, v)
    for _ in range(3):
        plan.attention()
    torch.cuda.synchronize()
    lib = _lib.load()
    fn = lib.ifa_ws_trace_read
    fn.argtypes = [C.c_void_p, C.c_int64]
    buf = np.zeros(49152, dtype=np.uint64)
    assert fn(buf.ctypes.data, buf.size) == 0
    t = buf.reshape(3, 2, 1024, 8).astype(np.int64)
    valid = t[t > 0]
    t0 = valid.min()
    names = ["softmax", "mma", "corr"]
    evs = [["S", "alpha", "Pfree", "Pfull"], ["Snext", "Pok", "Ook", "PV"], ["msg", "PVprev", "oready"]]
    for tile in range(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
        cells = []
        for gr in range(2):
            for r in range(3):
                row = t[r, gr, tile]
                cells.append(" ".join(f"{(x - t0) if x > 0 else -1:7d}" for x in row[: len(evs[r])]))
        print(f"{tile:3d} | " + " | ".join(cells))
    # per-tile period and phase lengths (group 0, softmax), skipping the first item
    s = t[0, 0]
    ok = (s[:, 0] > 0) & (s[:, 3] > 0)
    idx = np.nonzero(ok)[0]
    if len(idx) > 4:
        per = np.diff(s[idx, 0])
        print("softmax g0 period median", np.median(per), "A (S->alpha)", np.median(s[idx, 1] - s[idx, 0]),
              "wait Pfree", np.median(s[idx, 2] - s[idx, 1]), "B (Pfree->Pfull)", np.median(s[idx, 3] - s[idx, 2]),
              "S wait", np.median(s[idx[1:], 0] - s[idx[:-1], 3]))
        print("  A split: S->ld done", np.median(s[idx, 4] - s[idx, 0]), "ld->kfull", np.median(s[idx, 7] - s[idx, 4]), "kfull->u", np.median(s[idx, 5] - s[idx, 7]),
              "u->max", np.median(s[idx, 6] - s[idx, 5]), "max->alpha posted", np.median(s[idx, 1] - s[idx, 6]))
        s1 = t[0, 1]
        print("  group offset (g1 S - g0 S)", np.median(s1[idx, 0] - s[idx, 0]))


if __name__ == "__main__":
    main()
