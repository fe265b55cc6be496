#!/usr/bin/env python
"""Per-kernel Blackwell instruction evidence of the built library.

Disassembles paper_2409_16997_b200/lib/libifa_b200.so (cuobjdump -sass) and
counts, per shipped kernel, the SASS mnemonics that prove the sm_100a
execution model is used:

  UTCIMMA  tcgen05.mma kind::i8         (int8 x int8 -> int32 in TMEM)
  UTCHMMA  tcgen05.mma kind::f16        (fp16 x fp16 -> f32 in TMEM)
  UTCQMMA  tcgen05.mma kind::f8f6f4     (e4m3 x e4m3 -> f32 in TMEM)
  UTMALDG  cp.async.bulk.tensor (TMA load)
  LDTM / STTM  tcgen05.ld / tcgen05.st  (TMEM <-> registers)
  UTCBAR   tcgen05.commit (MMA completion -> mbarrier)
  MUFU     ex2 (softmax), I2FP, FMNMX3, FFMA2 for reference

  python tools/sass_evidence.py [--md profiles/<name>.md] [--json out.json]

tests/test_sass_evidence.py checks the same counts on every CPU test run,
so a build that loses any of them fails.
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2409_16997_b200", "lib", "libifa_b200.so")
MNEMONICS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTMALDG", "LDTM", "STTM", "UTCBAR",
             "MUFU", "FFMA2", "FMNMX3", "I2FP"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.splitlines()
    return out if len(out) == len(names) else names


def kernels(lib=LIB):
    """{demangled kernel name: (counts dict, first tcgen05/TMA lines)}."""
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                          text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : (\S+)\n", sass)
    names = blocks[1::2]
    bodies = blocks[2::2]
    out = {}
    for name, body in zip(demangle(names), bodies):
        counts = {m: 0 for m in MNEMONICS}
        excerpt, seen = [], set()
        for line in body.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
            if not m:
                continue
            op = m.group(2)
            if op in counts:
                counts[op] += 1
                if (op.startswith("UTC") or op in ("UTMALDG", "LDTM", "STTM")) and op not in seen:
                    seen.add(op)
                    text = re.sub(r"/\*[0-9a-f]+\*/", "", line.split(";")[0])
                    excerpt.append(re.sub(r"\s+", " ", text).strip())
        out[name.replace("(anonymous namespace)::", "anon::")] = (counts, excerpt)
    return out


def family(name):
    if "int_flash_pp_kernel" in name:
        mode = re.search(r"<\d+, \w+, (\d), \w+(, \w+)*>", name)
        return {"0": "pp full-INT8 (tolerance, bench default)", "1": "pp half-INT8",
                "2": "pp FP8"}[mode.group(1)] if mode else "pp"
    if "int_flash_ws_kernel" in name:
        return "ws full-INT8 (one thread per row)"
    if "int_flash_fwd_kernel" in name:
        return "exact / quad full-INT8"
    if "half_int8_fwd_kernel" in name:
        return "half-INT8 / FP8 16-warp"
    return "quantize / conversion"


def main():
    md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    js = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    ks = kernels()
    lines = ["# SASS evidence: Blackwell instructions per shipped kernel",
             "", f"`cuobjdump -sass {os.path.relpath(LIB, ROOT)}` "
             "(regenerate: `python tools/sass_evidence.py --md <this file>`; "
             "checked by `tests/test_sass_evidence.py`).", "",
             "| kernel | family | " + " | ".join(MNEMONICS) + " |",
             "|---|---|" + "---|" * len(MNEMONICS)]
    for name, (c, _) in ks.items():
        short = re.sub(r"\(CUtensorMap_st.*", "", name).replace("void ", "")
        short = re.sub(r"\(.*", "", short)
        lines.append(f"| `{short}` | {family(name)} | " +
                     " | ".join(str(c[m]) for m in MNEMONICS) + " |")
    lines += ["", "## Excerpts (first tcgen05 / TMA instruction of each kind)", ""]
    for name, (c, ex) in ks.items():
        if not ex:
            continue
        short = re.sub(r"\(.*", "", name.replace("void ", ""))
        lines.append(f"`{short}`:")
        lines.append("```")
        lines += ex
        lines.append("```")
    text = "\n".join(lines) + "\n"
    if md:
        open(md, "w").write(text)
    else:
        print(text)
    if js:
        json.dump({k: v[0] for k, v in ks.items()}, open(js, "w"), indent=1)


if __name__ == "__main__":
    main()
