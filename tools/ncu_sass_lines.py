"""Per-source-line executed instructions and stall samples of one kernel, by
joining ncu's SASS source page (CSV, --print-source sass) with the line table
of `nvdisasm -g` (ncu's CUDA-source view needs the sources at the box's path).

usage: ncu_sass_lines.py SASS_CSV NVDISASM_TXT KERNEL_MANGLED [steps] [top]
"""
import collections
import csv
import re
import sys

csvf, dis, fn = sys.argv[1:4]
steps = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 60

rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
sass = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        sass.append((int(r[ix["Address"]], 16), int(r[ix["Instructions Executed"]] or 0),
                     int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]].strip()))
    except ValueError:
        continue
base = sass[0][0]

lines = {}
inside, cur = False, "?"
for ln in open(dis):
    if ln.startswith("//----") and ".text." in ln:
        inside = ln.strip().split(".text.")[1].split()[0] == fn
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        lines[int(m.group(1), 16)] = cur

agg = collections.defaultdict(lambda: [0, 0])
for a, ex, s, _ in sass:
    k = lines.get(a - base, "?")
    agg[k][0] += ex
    agg[k][1] += s
tot_ex = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total {tot_ex / steps:.1f} instructions per step, {tot_s} samples")
for k, (ex, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{ex / steps:8.1f}/step {100 * s / tot_s:6.2f}% samples  {k}")
