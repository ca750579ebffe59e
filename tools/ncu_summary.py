"""Summarise an ncu --set full report of the walk kernel into profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "warp_instructions",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}


def main(rep, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for k, un, val in zip(h, u, v):
        if k in KEYS:
            res[KEYS[k]] = {"value": val, "unit": un}
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                if float(val) > 0:
                    res.setdefault("stall_samples", {})[k.split("stalled_")[1]] = int(float(val))
            except ValueError:
                pass
    json.dump(res, open(out_json, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
