"""Transport bench line: the device transport on the
paper's verification physics (1 cm cube n = 10, 6,000 tets,
Sigma_t = Sigma_s = 100 /cm, source in 1/8 of the domain, vacuum boundary),
one JSON line in bench.py's vocabulary:

  value      tet-crossings/s (scored track-length events) over the device time
             of the transport launches (localization excluded, as in the
             reference's t_batch);
  roofline   the kernel's demands per crossing from the committed ncu capture
             (profiles/transport_sol.json) x the live crossings / live time,
             against the same peaks bench.py uses;
  reference  the stock reference's transport.run (baseline/_ref, numba,
             threads = all host cores) on a bounded sample, same physics.

    python tools/transport_line.py [--particles 1000000] [--batches 2]
                                   [--ref-particles 20000] [--no-reference]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def sol(events, seconds):
    p = ROOT / "profiles" / "transport_sol.json"
    if not p.exists():
        return None
    s = json.loads(p.read_text())
    pk = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (
        ROOT / "MEASURED_PEAKS.json").exists() else {}
    clk = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    l2 = json.loads((ROOT / "profiles" / "r02_l2_peak.json").read_text())
    l2_peak = float(l2.get("l2_gather32_v8_gbs", 9150.3))
    hbm = float(pk.get("hbm_gbs", 6554.6))
    per = s["per_crossing"]
    rate = events / seconds
    units = {
        "issue": (per["warp_instructions"] * rate, 4 * 148 * clk, "warp-inst/s"),
        "l1tex_lsu": (per["lsu_wavefronts"] * rate, 148 * clk, "wavefronts/s"),
        "l2": (per["l2_bytes"] * rate / 1e9, l2_peak, "GB/s"),
        "hbm": (per["dram_bytes"] * rate / 1e9, hbm, "GB/s"),
    }
    fr = {k: a / b for k, (a, b, _) in units.items()}
    bound = max(fr, key=fr.get)
    return {"kernel": s["kernel"], "bound": bound, "frac": fr[bound], "fracs": fr,
            "units": {k: {"achieved": a, "peak": b, "unit": u} for k, (a, b, u) in units.items()},
            "sol_source": "profiles/transport_sol.json (ncu --set full of one transport_kernel "
                          "launch, tools/gpu_prof_tr.sh) per-crossing demands x live rate",
            "ncu_pct_of_peak": s.get("ncu_pct_of_peak"),
            "warp_instructions_per_crossing": per["warp_instructions"]}


def reference(k, threads):
    ref = ROOT / "baseline" / "_ref"
    if not ref.exists():
        return {"unavailable": "baseline/_ref not installed"}
    sys.path.insert(0, str(ref))
    try:
        import numba
        from meshtally import transport as RT
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"stock reference does not import: {e}"}
    numba.set_num_threads(threads)
    RT.run(RT.RunConfig(mesh_n=10, num_particles=64, num_batches=1, threads=threads))  # JIT
    t = time.perf_counter()
    r = RT.run(RT.RunConfig(mesh_n=10, num_particles=k, num_batches=1, threads=threads))
    wall = time.perf_counter() - t
    return {"value": r.events / r.t_batch, "unit": "crossings/s", "cores": threads,
            "kind": "reference", "collisions_per_s": r.collisions / r.t_batch,
            "histories_per_s": k / r.t_batch, "events": r.events, "collisions": r.collisions,
            "t_batch_s": r.t_batch, "wall_s": wall,
            "sample": f"{k} histories x 1 batch, stock meshtally.transport.run(threads={threads}) "
                      "from baseline/_ref (numba)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--particles", type=int, default=1_000_000)
    ap.add_argument("--batches", type=int, default=2)
    ap.add_argument("--ref-particles", type=int, default=200_000)
    ap.add_argument("--no-reference", action="store_true")
    a = ap.parse_args()
    from paper_2504_19048_b200 import build_cube_mesh
    from paper_2504_19048_b200 import transport as T
    mesh = build_cube_mesh(10)
    T.run(T.RunConfig(mesh_n=10, num_particles=20_000, num_batches=1), mesh)  # warm-up
    cfg = T.RunConfig(mesh_n=10, num_particles=a.particles, num_batches=a.batches, seed=42)
    t = time.perf_counter()
    r = T.run(cfg, mesh)
    wall = time.perf_counter() - t
    out = {"metric": "tet-crossings/s (device transport, track-length + collision estimators)",
           "value": r.events / r.t_batch, "unit": "crossings/s",
           "collisions_per_s": r.collisions / r.t_batch,
           "histories_per_s": a.particles * a.batches / r.t_batch,
           "events": r.events, "collisions": r.collisions, "sweeps": r.sweeps,
           "t_transport_s": r.t_batch, "t_localization_s": r.t_localization, "wall_s": wall,
           "higher_is_better": True, "dtype": "f64", "data": "synthetic (philox source, seed 42)",
           "config": {"workload": "paper verification physics (PAPER.md:279): cube n=10 "
                                  "(6,000 tets), 1 group, sigma_t = sigma_s = 100/cm, source box "
                                  "[0,0.5]^3, isotropic", "histories_per_batch": a.particles,
                      "batches": a.batches},
           "roofline": sol(r.events, r.t_batch)}
    if not a.no_reference:
        out["reference"] = reference(a.ref_particles, os.cpu_count() or 1)
        if "value" in out["reference"]:
            out["vs_reference"] = out["value"] / out["reference"]["value"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
