"""Write profiles/walk_dram_traffic.json (read by bench.py's roofline.traffic)
from an ncu --set full report of one walk launch:
    python tools/ncu_traffic.py gpurun_out/walk.ncu-rep profiles/r01_ncu_walk_f32.json"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main(rep, source_note):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(name):
        i = h.index(name)
        return float(v[i]) * scale[u[i]]
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {"kernel": v[h.index("Kernel Name")], "dram_read_bytes": rd, "dram_write_bytes": wr,
           "bytes_per_launch": rd + wr, "source": source_note,
           "note": "dram__bytes_read.sum + dram__bytes_write.sum of one walk launch "
                   "(bench workload, ncu --set full --clock-control none)"}
    (ROOT / "profiles" / "walk_dram_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
