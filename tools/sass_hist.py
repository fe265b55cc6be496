#!/usr/bin/env python
"""Per-opcode histogram of executed warp instructions and stall samples from
an ncu source-page export (`ncu -i rep --page source --csv --print-source sass`).

  python tools/sass_hist.py src.csv [--per N]   # N = normaliser (e.g. tiles)
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    ss = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    ops = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    lines = []
    for r in rows[2:]:
        if len(r) <= ia:
            continue
        try:
            n = int(r[ia] or 0)
            s = int(r[ss] or 0)
        except ValueError:
            continue
        text = r[src].strip()
        op = text.split()[0] if text else "?"
        if op.startswith("@"):
            op = text.split()[1]
        op = op.split(".")[0]
        ops[op][0] += n
        ops[op][1] += s
        tot_i += n
        tot_s += s
        lines.append((n, s, r[0], text))
    print(f"total warp instructions {tot_i} ({tot_i / per:.0f} per unit), stall samples {tot_s}")
    print(f"{'opcode':12s} {'inst/unit':>12s} {'inst%':>7s} {'stall%':>7s}")
    for op, (n, s) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:40]:
        print(f"{op:12s} {n / per:12.1f} {100 * n / tot_i:6.1f}% {100 * s / max(tot_s, 1):6.1f}%")
    print("\ntop stalled instructions:")
    for n, s, addr, text in sorted(lines, key=lambda x: -x[1])[:25]:
        print(f"  {100 * s / max(tot_s, 1):5.1f}%  {n / per:9.1f}  {text[:90]}")


if __name__ == "__main__":
    main()
