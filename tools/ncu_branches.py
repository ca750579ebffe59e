"""Branch instructions (BRA / BSSY / BSYNC) of one kernel per source line, from
ncu's SASS source page joined with `nvdisasm -g` (as tools/ncu_sass_lines.py),
and the instruction mix per step.

usage: ncu_branches.py SASS_CSV NVDISASM_TXT KERNEL_MANGLED STEPS [top]
"""
import collections
import csv
import re
import sys

csvf, dis, fn, steps = sys.argv[1:5]
steps = float(steps)
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
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
lines, inside, cur = {}, False, "?"
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


def opcode(src):
    toks = [t for t in src.split() if not t.startswith("@")]
    return toks[0].split(".")[0] if toks else ""


mix = collections.Counter()
br = collections.defaultdict(lambda: [0, 0])
tot_s = sum(x[2] for x in sass)
for a, ex, s, src in sass:
    op = opcode(src)
    mix[op] += ex
    if op in ("BRA", "BSSY", "BSYNC"):
        k = lines.get(a - base, "?")
        br[k][0] += ex
        br[k][1] += s
print("instruction mix per step:")
for op, c in mix.most_common(12):
    print(f"  {op:8s} {c / steps:6.1f}")
print("branch instructions by source line (per step, share of stall samples):")
for k, (e, s) in sorted(br.items(), key=lambda x: -x[1][1])[:top]:
    print(f"  {k:24s} {e / steps:5.1f}  {100 * s / tot_s:5.2f}%")
