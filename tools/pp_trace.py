"""Pipeline timeline of the two-Q-tile kernel (attn_pp.cu), CTA 0, from a
build with -DIFA_PP_TRACE=1:

  tools/build_variant.sh pptrace -DIFA_PP_TRACE=1
  IFA_B200_LIB=build/pptrace/libifa_b200.so python tools/pp_trace.py [slices n]

Math warp 4 + 8g (group g), per tile: wait-for-S start (W), S ready (S), S
loaded (L), row max done (M), P buffer free (F), codes + P stored (C), P
published after the O rescale (P).  MMA issuer g: S(next) issued, P ready,
P.V issued.  Prints per-tile stamps and the median phase lengths."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2409_16997_b200 import _lib  # noqa: E402
from paper_2409_16997_b200.runtime import AttentionPlan  # noqa: E402


def main():
    slices = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    plan = AttentionPlan(slices, n, 128, fast=True)
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(slices, n, 128, device="cuda", generator=g) for _ in range(3))
    plan.quantize(q, k, v)
    for _ in range(3):
        plan.attention()
    torch.cuda.synchronize()
    fn = _lib.load().ifa_pp_trace_read
    fn.argtypes = [C.c_void_p, C.c_int64]
    buf = np.zeros(2 * 2 * 1024 * 8, dtype=np.uint64)
    assert fn(buf.ctypes.data, buf.size) == 0
    t = buf.reshape(2, 2, 1024, 8).astype(np.int64)
    t0 = t[t > 0].min()
    rel = np.where(t > 0, t - t0, -1)
    print("tile | g0: W S L M F C P | mma0: Sn Pok PV | g1: W S L M F C P | mma1: Sn Pok PV")
    for tile in [int(x) for x in os.environ.get("PP_TRACE_TILES", "28,29,30,31,32,33,34,35,60,61,62,63,64,65").split(",")]:
        cells = []
        for gr in range(2):
            m = rel[0, gr, tile]
            cells.append(" ".join(f"{x:8d}" for x in (m[7], m[0], m[1], m[2], m[3], m[4], m[5])))
            mm = rel[1, gr, tile]
            cells.append(" ".join(f"{x:8d}" for x in mm[:3]))
        print(f"{tile:4d} | " + " | ".join(cells))
    for gr in range(2):
        mm = rel[1, gr]
        ends = [i for i in range(1024) if mm[i, 5] > 0]
        for i in ends[:4]:
            nxt = rel[0, gr, i + 1, 7] if i + 1 < 1024 else -1
            print(f"group {gr} item end at tile {i}: P published {rel[0, gr, i, 5]}, epilogue start "
                  f"{mm[i, 5]}, o_full {mm[i, 6]}, epilogue done {mm[i, 7]}, next tile wait {nxt}")
    for gr in range(2):
        m = t[0, gr]
        ok = np.all(m[:, [7, 0, 1, 2, 3, 4, 5]] > 0, axis=1)
        idx = np.nonzero(ok)[0][5:]
        if len(idx) < 4:
            continue
        d = lambda a, b: float(np.median(m[idx, b] - m[idx, a]))
        per = float(np.median(np.diff(m[idx, 0])))
        print(f"group {gr}: period {per:.0f}  waitS {d(7, 0):.0f}  loadS {d(0, 1):.0f}  "
              f"dequant+max {d(1, 2):.0f}  waitPfree {d(2, 3):.0f}  codes {d(3, 4):.0f}  "
              f"rescale+publish {d(4, 5):.0f}  tail->next {float(np.median(m[idx[1:], 7] - m[idx[:-1], 5])):.0f}")
        mm = t[1, gr]
        okm = np.all(mm[:, :3] > 0, axis=1)
        im = np.nonzero(okm)[0][5:]
        if len(im) > 4:
            print(f"  mma {gr}: P ready -> PV issued {float(np.median(mm[im, 2] - mm[im, 1])):.0f}, "
                  f"S(next) issued -> P ready {float(np.median(mm[im, 1] - mm[im, 0])):.0f}")


if __name__ == "__main__":
    main()
