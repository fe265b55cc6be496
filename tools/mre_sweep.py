#!/usr/bin/env python
"""C4 accuracy sweep on the GPU: MRE of the full-INT8 forward (exact and
tolerance mode) and of the half-INT8 forward against the
fp64 reference attention, N = 1k..16k, d = 128, normal and uniform
activations, with and without outlier tokens (BASELINE.json configs[3]).

Inputs are the reference harness's own (the oracle restatement of
generate() + stream_seed(), eval.cpp:36-51 / 169-180), so the exact-mode
numbers are directly comparable with SURVEY.md Appendix B (computed with the
reference library on the same inputs).  The INT8 path is the product's
(quantize kernels + attention kernel through the public API); the fp64
ground truth and the normalized-L1 accumulation are
paper_2409_16997_b200.evaluation.

    python tools/mre_sweep.py [--quick] [--out profiles/r1_c4_mre_sweep]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2409_16997_b200 as ifa  # noqa: E402
from paper_2409_16997_b200.evaluation import ErrorAccum, inject_outliers, reference_attention  # noqa: E402
from oracle_bindings import Oracle  # noqa: E402

# reference full-INT8 MRE vs fp64, d=128, Br=Bc=128, seed 0.
APPENDIX_B = {
    "normal": {1024: 2.68, 2048: 2.93, 4096: 3.06, 8192: 3.15, 16384: 3.19},
    "uniform": {1024: 1.83, 2048: 2.11, 4096: 2.57, 8192: 3.04, 16384: 3.45},
}
# reference half-INT8 MRE vs fp64 (same inputs).
APPENDIX_B_HALF = {
    "normal": {1024: 2.01, 2048: 2.30, 4096: 2.41, 8192: 2.52, 16384: 2.56},
    "uniform": {1024: 0.496, 2048: 0.498, 4096: 0.514, 8192: 0.523, 16384: 0.514},
}
# reference fp8_emulated_attention MRE vs fp64.
APPENDIX_B_FP8 = {
    "normal": {1024: 9.49, 2048: 10.5, 4096: 11.2, 8192: 11.5, 16384: 11.8},
    "uniform": {1024: 4.17, 2048: 4.13, 4096: 4.22, 8192: 4.34, 16384: 4.25},
}
# Paper tables (RTX 4090, Triton; shape details unstated): PAPER.md:163-187.
PAPER = {
    "normal": {1024: 4.05, 2048: 4.18, 4096: 4.21, 8192: 4.38, 16384: 4.52},
    "uniform": {1024: 1.69, 2048: 1.62, 4096: 1.65, 8192: 1.85, 16384: 1.82},
}


def int8_forward(q, k, v, bc, fast):
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    qq = ifa.quantize_per_row(dev(q))
    kq = ifa.quantize_per_row(dev(k))
    vq = ifa.quantize_per_tensor(dev(v))
    cfg = ifa.AttentionConfig(ifa.BlockSpec(128, bc), fast=fast)
    return ifa.int_flash_attention(ifa.QuantizedAttentionInputs(qq, kq, vq), cfg)


def half_forward(q, k, v):
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    qq = ifa.quantize_per_row(dev(q))
    kq = ifa.quantize_per_row(dev(k))
    return ifa.half_int8_attention(qq, kq, dev(v), ifa.AttentionConfig(ifa.BlockSpec(128, 128)))


def run_case(o, dist, n, d, seed_idx, outlier=None):
    q, k, v = o.slice_inputs(dist, n, d, seed=0, seed_idx=seed_idx)
    if outlier is not None:
        factor, roles = outlier
        mats = [q, k, v]
        for r in roles:
            mats[r] = inject_outliers(mats[r], 0.01, factor, seed=1000 * seed_idx + r)
        q, k, v = mats
    ref = reference_attention(*(torch.from_numpy(a).cuda() for a in (q, k, v)))
    res = {}
    for mode in ("exact", "fast"):
        out = int8_forward(q, k, v, 128, mode == "fast")
        acc = ErrorAccum()
        acc.add(ref, out)
        res[mode] = acc
    acc = ErrorAccum()
    acc.add(ref, half_forward(q, k, v))
    res["half"] = acc
    acc = ErrorAccum()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    acc.add(ref, ifa.fp8_emulated_attention(dev(q), dev(k), dev(v),
                                            ifa.AttentionConfig(ifa.BlockSpec(128, 128))))
    res["fp8"] = acc
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="N <= 4096 only")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_c4_mre_sweep"))
    args = ap.parse_args()
    o = Oracle()
    d = 128
    ns = [1024, 2048, 4096] if args.quick else [1024, 2048, 4096, 8192, 16384]
    rows = []
    t0 = time.time()
    for dist in ("normal", "uniform"):
        for n in ns:
            r = run_case(o, dist, n, d, seed_idx=0)
            rows.append({"dist": dist, "n": n, "outliers": "none",
                         "mre_exact_pct": 100 * r["exact"].ratio(),
                         "mre_fast_pct": 100 * r["fast"].ratio(),
                         "mre_half_pct": 100 * r["half"].ratio(),
                         "mre_fp8_pct": 100 * r["fp8"].ratio(),
                         "appendix_b_pct": APPENDIX_B[dist][n], "paper_pct": PAPER[dist][n],
                         "appendix_b_half_pct": APPENDIX_B_HALF[dist][n],
                         "appendix_b_fp8_pct": APPENDIX_B_FP8[dist][n]})
    settings = [("x10 in Q,K,V", (10.0, (0, 1, 2))), ("x100 in Q,K,V", (100.0, (0, 1, 2))),
                ("x10 in Q,K only", (10.0, (0, 1))), ("x10 in V only", (10.0, (2,)))]
    for dist in ("normal", "uniform"):
        for label, spec in settings:
            per_seed = {"exact": [], "fast": [], "half": [], "fp8": []}
            for seed_idx in (21, 22, 23):
                r = run_case(o, dist, 1024, d, seed_idx, outlier=spec)
                for m in per_seed:
                    per_seed[m].append(r[m].ratio())
            rows.append({"dist": dist, "n": 1024, "outliers": label,
                         "mre_exact_pct": 100 * float(np.mean(per_seed["exact"])),
                         "mre_fast_pct": 100 * float(np.mean(per_seed["fast"])),
                         "mre_half_pct": 100 * float(np.mean(per_seed["half"])),
                         "mre_fp8_pct": 100 * float(np.mean(per_seed["fp8"]))})
    wall = time.time() - t0
    with open(args.out + ".json", "w") as f:
        json.dump({"rows": rows, "wall_s": wall, "d": d, "bc": 128,
                   "inputs": "reference generator + stream_seed(0, seed_idx, role, 0, 0)",
                   "outlier_definition": "paper_2409_16997_b200.evaluation.inject_outliers "
                                         "(1% of rows, PCG64 partial Fisher-Yates)"}, f,
                  indent=1)
    lines = ["| dist | N | outliers | full-INT8 exact (%) | full-INT8 fast (%) | "
             "reference full-INT8, App. B (%) | paper full-INT8, RTX 4090 (%) | half-INT8 (%) | "
             "reference half-INT8, App. B (%) | FP8 e4m3 (%) | reference FP8, App. B (%) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['dist']} | {r['n']} | {r['outliers']} | {r['mre_exact_pct']:.3f} | "
                     f"{r['mre_fast_pct']:.3f} | {r.get('appendix_b_pct', '')} | "
                     f"{r.get('paper_pct', '')} | {r['mre_half_pct']:.3f} | "
                     f"{r.get('appendix_b_half_pct', '')} | {r['mre_fp8_pct']:.3f} | "
                     f"{r.get('appendix_b_fp8_pct', '')} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + f"\n\nwall {wall:.1f} s on one B200\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
