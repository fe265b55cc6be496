"""Stall-reason breakdown per code region of an ncu source-page export
(`ncu -i rep --page source --csv --print-source sass > src.csv`).

  python tools/stall_regions.py src.csv [--per UNITS]

Regions are cut at the softmax landmarks of attn_ws.cu: the first LDTM of the
S load (A phase: load, dequantize, max) and the first / last MUFU.EX2 of the
code loop (B phase); everything else is reported as "other".
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
    hdr = rows[1]
    ia = hdr.index("Instructions Executed")
    src = hdr.index("Source")
    reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    lines = []
    for r in rows[2:]:
        try:
            n = int(r[ia] or 0)
            st = [int(r[i] or 0) for i in reasons]
        except ValueError:
            continue
        lines.append((n, st, r[src]))
    hot = [i for i, l in enumerate(lines) if l[0] > 0]
    ldtm = [i for i, l in enumerate(lines) if "LDTM" in l[2]]
    mufu = [i for i, l in enumerate(lines) if "MUFU.EX2" in l[2] and not l[2].lstrip().startswith("@")]
    a0 = ldtm[0] - 10 if ldtm else 0
    b0, b1 = (mufu[0] - 30, mufu[-1] + 60) if mufu else (0, 0)
    regions = {"A (S load, dequant, max)": range(a0, b0), "B (codes, P stores)": range(b0, b1)}
    inside = set()
    for rg in regions.values():
        inside.update(rg)
    regions["other"] = [i for i in range(len(lines)) if i not in inside]
    total = sum(sum(l[1]) for l in lines)
    for name, rg in regions.items():
        agg = defaultdict(int)
        ins = 0
        for i in rg:
            n, st, _ = lines[i]
            ins += n
            for k, v in zip(reasons, st):
                agg[hdr[k]] += v
        tot = sum(agg.values())
        top = sorted(agg.items(), key=lambda kv: -kv[1])[:7]
        print(f"{name}: {ins / per:.0f} warp-instr/unit, {100 * tot / max(total, 1):.1f}% of samples: " +
              ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.0f}%" for k, v in top))


if __name__ == "__main__":
    main()
