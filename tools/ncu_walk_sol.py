"""Speed-of-light figures of one walk launch, per tet-crossing, from an ncu
--set full report of the bench's walk kernel -> profiles/walk_sol.json (read
by bench.py to build its `roofline` block from the live kernel time).

    python tools/ncu_walk_sol.py gpurun_out/walk_full.ncu-rep CROSSINGS_PER_LAUNCH [NOTE] [OUT]

OUT (default walk_sol.json) names the file under profiles/; the transport
kernel's capture goes to transport_sol.json (CROSSINGS = the batch's events).

CROSSINGS_PER_LAUNCH is the TraceSummary.events of the captured move (the
bench move: 569,602,285 on C2 with 1e7 particles, sigma_t = 2).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "": 1,
         "inst": 1, "sector": 1, "cycle": 1, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "%": 1, "warp": 1, "ms": 1e-3, "us": 1e-6,
         "ns": 1e-9, "s": 1, "Ghz": 1e9, "Mhz": 1e6, "Khz": 1e3, "hz": 1}


def main(rep, crossings, note="", out_name="walk_sol.json"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        i = h.index(name)
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
    x = float(crossings)

    def lsu_wavefronts():
        """LSU data-pipe wavefronts of the launch (1 per SM-cycle peak)."""
        sms = get("device__attribute_multiprocessor_count")
        try:
            return get("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg") * sms
        except ValueError:  # not collected in this capture: from its % of peak
            pct = get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")
            return pct / 100.0 * get("sm__cycles_elapsed.avg") * sms
    dur = get("gpu__time_duration.sum")
    out = {
        "kernel": v[h.index("Kernel Name")],
        "source": note or rep,
        "crossings_per_launch": x,
        "duration_s": dur,
        "sm_clock_hz": get("sm__cycles_elapsed.avg.per_second"),
        "per_crossing": {
            "warp_instructions": get("smsp__inst_executed.sum") / x,
            "lsu_wavefronts": lsu_wavefronts() / x,
            "l2_bytes": 32 * get("lts__t_sectors.sum") / x,
            "dram_bytes": (get("dram__bytes_read.sum") + get("dram__bytes_write.sum")) / x,
        },
        "per_launch": {
            "warp_instructions": get("smsp__inst_executed.sum"),
            "dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
            "l2_bytes": 32 * get("lts__t_sectors.sum"),
        },
        "ncu_pct_of_peak": {
            "issue_active": get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
            "l1tex_lsu_wavefronts": get(
                "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            "l1tex_throughput": get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_throughput": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_throughput": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        },
        "occupancy_warps_per_sm": get("sm__warps_active.avg.per_cycle_active"),
        "registers": get("launch__registers_per_thread"),
    }
    (ROOT / "profiles" / out_name).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
