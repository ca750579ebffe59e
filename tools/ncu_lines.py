"""Top source lines of an ncu --print-source cuda,sass CSV export by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, hdr, res = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr[4:], r[4:]))
        try:
            smp = int(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        st = {k[6:]: int(d[k]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k
              and d.get(k, "0").isdigit() and int(d[k]) > 0}
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        res.append((smp, cur, r[0], r[1].strip()[:80], d.get("Instructions Executed", ""), top))
res.sort(key=lambda x: -x[0])
tot = sum(x[0] for x in res)
print("total samples", tot)
for x in res[:n]:
    print(f"{x[0]:7d} {100*x[0]/tot:5.1f}% {x[1]}:{x[2]} inst={x[4]} {x[5]} | {x[3]}")
