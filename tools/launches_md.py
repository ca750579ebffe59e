"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel:
    python tools/launches_md.py gpurun_out/launches.csv "python bench.py --steps 2 ..." > profiles/rNN_launches.md"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki][:70]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print(f"# ncu launch list: `{sys.argv[2] if len(sys.argv) > 2 else ''}`\n")
print("Serialised, cold-cache per-launch times (`--metrics gpu__time_duration.sum --clock-control none`);")
print("compare shares, not absolutes. Includes setup (mesh upload, grid build), warm-up, timed and e2e steps.\n")
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| `{k}` | {cnt[k]} | {tot[k]:.3f} | {100 * tot[k] / T:.1f}% |")
