"""Summarise tools/gpu_runs/ab.sh output: attention ms per (workload, lib)."""
import collections, glob, json, os, sys

d = sys.argv[1]
acc = collections.defaultdict(list)
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        j = json.load(open(f))
    except Exception:
        continue
    w, rest = os.path.basename(f)[:-5].split("_", 1)
    lib = rest.rsplit("_", 1)[0]
    acc[(w, lib)].append(j["breakdown_ms"]["attention"])
for (w, lib), v in sorted(acc.items()):
    print(f"{w:4s} {lib:20s} " + " ".join(f"{x:.4f}" for x in v) + f"   min {min(v):.4f}")
