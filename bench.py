"""Benchmark of the tet-walk track-length tally (BASELINE.json metric:
tet-crossings/s and particle-moves/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) there is one rank per GPU; every rank owns a shard of
particles (weak scaling: the per-GPU particle count is fixed), a replica of
the mesh and a private tally; once per batch the tallies are summed with one
NCCL all-reduce before the on-device finalize.

A step is one batch of the hot path over the whole synthetic workload:
restore the localized start state (device-to-device), one
move_to_next_location of every particle, tally reduce (N > 1), finalize.
`e2e` repeats the batch through the public API with pinned HOST buffers:
initialize_particle_location + move_to_next_location + finalize, H2D of the
inputs and D2H of the TraceSummary inside the timed region.

The CPU baseline is the oracle port of the reference's algorithm
(oracle/walk_oracle.c, OpenMP, all host threads) timed on a bounded sample
of the same workload on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

B_CROSSING = 133  # algorithmic bytes per tet-crossing
B_MOVE = 100      # algorithmic bytes per particle-move


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=55, help="cube subdivisions (55 -> 998,250 tets)")
    p.add_argument("--particles", type=int, default=10_000_000, help="particles per GPU")
    p.add_argument("--sigma-t", type=float, default=2.0)
    p.add_argument("--cpu-seconds", type=float, default=10.0,
                   help="target CPU work for the bounded baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-transport", action="store_true",
                   help="skip the device-transport line (SURVEY §8f row 1) added on rank 0")
    p.add_argument("--sort", type=int, default=0)
    p.add_argument("--warp-agg", type=int, default=-1,
                   help="tally atomics: -1 adaptive aggregation (default), 0 never, 1 always")
    p.add_argument("--blocks-per-sm", type=int, default=0)
    p.add_argument("--staged", type=int, default=-1,
                   help="refill: -1 library default, 0 v1, 1 stage kernel, 2 direct")
    p.add_argument("--no-stream-move", action="store_true",
                   help="e2e: one walk launch per input chunk instead of one streamed launch")
    return p.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload(n_particles, sigma_t, rank):
    from paper_2504_19048_b200 import synth
    gen = synth.rng(synth.SEED + 1000 * rank)
    pos = synth.uniform_box(gen, n_particles)
    dest = synth.flight_destinations(gen, pos, sigma_t)
    return pos, dest


def config(args, world, ne):
    return {
        "workload": (f"north-star point of configs[1]/[2]: unit cube n={args.n} "
                     f"({ne:,} tets), {args.particles:,} particles per GPU uniform in "
                     f"[0.05,0.95]^3, isotropic flights -ln(u)/{args.sigma_t} cm, weight 1, "
                     "1 group, one move per batch"),
        "mesh_elements": ne,
        "particles_per_gpu": args.particles,
        "global_particles": args.particles * world,
        "sigma_t": args.sigma_t,
        "parallelism": f"dp{world} (particle shards, mesh replicated, tally all-reduce)",
        "l2": "particle state ~1 GB/GPU streamed per step (> 126 MB L2, no flush needed); "
              "mesh 38 MB stays L2-resident by design",
        "options": {"sort": bool(args.sort),
                    "warp_agg": ("adaptive" if args.warp_agg < 0 else bool(args.warp_agg)),
                    "staged": "default" if args.staged < 0 else args.staged,
                    "blocks_per_sm": args.blocks_per_sm or "default",
                    "stream_move": not args.no_stream_move},
    }


# ---------------------------------------------------------------------------
# clocks sampling during the timed region

class Clocks:
    """SM clock and clock-event reasons sampled every 5 ms by NVML (a
    background thread) for the duration of the timed region; nvidia-smi in
    loop mode if NVML is unavailable."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, dev):
        self.dev = dev
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self._p = None

    def _nvml_loop(self, nv, h):
        while not self._stop.is_set():  # every 5 ms
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis else self.dev
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 2.0:  # sampler running first
                time.sleep(0.002)
            self.samples.clear()  # keep only samples taken inside the region
            return self
        except Exception:
            pass
        cmd = ["nvidia-smi", "-i", str(self.dev), "-lms", "50",
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
               "--format=csv,noheader,nounits"]
        try:
            self._p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                       text=True)
        except OSError:
            return self

        def read():
            for line in self._p.stdout:
                try:
                    a = [x.strip() for x in line.strip().split(",")]
                    self.max_mhz = float(a[1])
                    self.samples.append((float(a[0]), int(a[2], 16)))
                except (ValueError, IndexError):
                    pass
        self._t = threading.Thread(target=read, daemon=True)
        self._t.start()
        t0 = time.time()
        while not self.samples and time.time() - t0 < 5.0:  # first sample before the region
            time.sleep(0.01)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._p.kill()
        if self._t is not None:
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        busy = [s for s in self.samples if not s[1] & 0x1] or self.samples
        bits = 0
        for _, b in busy:
            bits |= b
        return {"sm_mhz": statistics.median(s[0] for s in busy),
                "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.NAMES.items() if bits & k and k != 0x1],
                "samples": len(self.samples), "samples_under_load": len(busy)}


# ---------------------------------------------------------------------------
# CPU baseline: oracle port, bounded sample

def cpu_sample_rate(mesh, pos, dest, target_s, threads=None):
    """Time the oracle's trace_and_score restatement on a sample sized for
    ~target_s seconds; returns (crossings/s, moves/s, detail)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    threads = threads or orc.max_threads()

    def run(k):
        t = orc.OracleTally(mesh, k, threads=threads)
        t.initialize_particle_location(pos[:k])
        fly = np.ones(k, np.int8)
        w = np.ones(k)
        t0 = time.perf_counter()
        s = t.move_to_next_location(dest[:k], fly, w)
        dt = time.perf_counter() - t0
        return s, dt

    k = min(20_000, pos.shape[0])
    s, dt = run(k)
    if dt < target_s / 4 and k < pos.shape[0]:
        k = int(min(pos.shape[0], k * target_s / max(dt, 1e-3)))
        s, dt = run(k)
    detail = {"sample": f"first {k:,} particles of rank 0's workload, one move "
                        f"({s.events:,} crossings), localization untimed",
              "cores": threads, "seconds": round(dt, 3), "particles": k}
    return s.events / dt, k / dt, detail, s, dt


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------

def _import_stock_reference():
    """The unmodified reference package installed in baseline/_ref (numba);
    None when it is not importable on this host."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "meshtally").is_dir():
        return None
    sys.path.insert(0, str(ref))
    try:
        import meshtally  # noqa: F401
        import numba  # noqa: F401
    except Exception:
        sys.path.remove(str(ref))
        return None
    return meshtally


def run_reference_stock(args, mt_mod):
    """The reference's own CPU path (baseline/_ref, numba, unmodified) through
    its public MeshTally API: per step, the localized start state is restored
    and one move_to_next_location (load_step + trace_and_score,
    search.py:492-517) + finalize_batch runs over a bounded sample of the same
    workload, on every host core (numba.set_num_threads(T) with T tally slabs,
    the configuration in which the reference's threads > 1 path is correct,
    SURVEY.md §8b)."""
    import numba
    T = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    T = max(1, min(T, numba.config.NUMBA_NUM_THREADS))
    numba.set_num_threads(T)
    t_build = time.perf_counter()
    mesh = mt_mod.build_cube_mesh(args.n)
    t_build = time.perf_counter() - t_build
    pos, dest = workload(args.particles, args.sigma_t, 0)
    per_step = float(os.environ.get("BENCH_REF_STEP_S", "2.0"))

    def make(k):
        t = mt_mod.MeshTally(mesh, k, threads=T)
        t.initialize_particle_location(pos[:k])
        b, ws = t._batch, t._ws
        snap = [(a, a[:k].copy()) for a in (b.position, b.element, b.alive, ws.entry_face,
                                             ws.stuck, ws.outcome, ws.seg_total)]
        return t, snap

    fly_all = np.ones(args.particles, np.int8)
    w_all = np.ones(args.particles)

    def step(t, snap, k):
        for a, v in snap:
            a[:k] = v
        s = t.move_to_next_location(dest[:k], fly_all[:k], w_all[:k])
        t.finalize_batch()
        return s

    # JIT warm-up and sizing on a small sample, then the bounded sample
    k = min(50_000, args.particles)
    t, snap = make(k)
    step(t, snap, k)
    t0 = time.perf_counter()
    s = step(t, snap, k)
    dt = time.perf_counter() - t0
    k = int(min(args.particles, max(k, k * per_step / max(dt, 1e-3))))
    t, snap = make(k)
    for _ in range(args.warmup):
        step(t, snap, k)
    ev = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ev += step(t, snap, k).events
    dt = time.perf_counter() - t0
    val = ev / dt
    rank, world, _ = env_rank()
    sample = (f"first {k:,} of the {args.particles:,} particles per step (same workload); "
              "stock reference from baseline/_ref (meshtally 0.1.0, numba "
              f"{numba.__version__}): MeshTally(threads={T}).move_to_next_location + "
              "finalize_batch, localized start state restored per step (untimed "
              "localization)")
    out = {
        "impl": "reference",
        "metric": "tet-crossings/s", "value": val, "unit": "crossings/s",
        "particle_moves_per_s": k * args.steps / dt,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(args, 1, mesh.num_elements),
        "cpu_baseline": {"value": val, "unit": "crossings/s", "cores": T, "kind": "reference",
                         "sample": sample, "cpu": cpu_model(),
                         "mesh_build_s": round(t_build, 3)},
        "e2e": {"value": val, "unit": "crossings/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def run_reference(args):
    rank, world, local = env_rank()
    if rank != 0:
        return
    mt_mod = None if os.environ.get("BENCH_REF_PORT") else _import_stock_reference()
    if mt_mod is not None:
        return run_reference_stock(args, mt_mod)
    from paper_2504_19048_b200 import build_cube_mesh
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    mesh = build_cube_mesh(args.n)
    pos, dest = workload(args.particles, args.sigma_t, 0)
    threads = orc.max_threads()
    # size one step at ~2 s of CPU work so the whole run stays within minutes
    per_step = float(os.environ.get("BENCH_REF_STEP_S", "2.0"))
    _, _, detail, _, _ = cpu_sample_rate(mesh, pos, dest, per_step, threads)
    k = detail["particles"]
    t = orc.OracleTally(mesh, k, threads=threads)
    t.initialize_particle_location(pos[:k])
    snap = {f: getattr(t, f).copy() for f in ("position", "element", "alive", "entry_face",
                                              "stuck", "outcome", "seg_total")}
    fly = np.ones(k, np.int8)
    w = np.ones(k)

    def step():
        for f, v in snap.items():
            getattr(t, f)[:] = v
        s = t.move_to_next_location(dest[:k], fly, w)
        t.finalize_batch()
        return s

    for _ in range(args.warmup):
        step()
    ev = moves = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s = step()
        ev += s.events
        moves += k
    dt = time.perf_counter() - t0
    val = ev / dt
    out = {
        "impl": "reference",
        "metric": "tet-crossings/s", "value": val, "unit": "crossings/s",
        "particle_moves_per_s": moves / dt,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(args, 1, mesh.num_elements),
        "cpu_baseline": {"value": val, "unit": "crossings/s", "cores": threads, "kind": "port",
                         "sample": f"first {k:,} of the {args.particles:,} particles per "
                                   "step (same workload), oracle/walk_oracle.c (C "
                                   "restatement of search.py:169-275, OpenMP)",
                         "cpu": cpu_model()},
        "e2e": {"value": val, "unit": "crossings/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def roofline(stats, steps, walk_s, alg_gbps, hbm_peak, peak_src, clk):
    """The walk kernel against each resource it can be bound by, from the live
    kernel time and the per-crossing demands of the committed ncu capture of
    the same kernel (profiles/walk_sol.json, tools/ncu_walk_sol.py): warp
    instruction issue (4 per SM per cycle at the measured SM clock), the
    L1TEX LSU data pipe (1 wavefront per SM per cycle), L2 (the measured
    random 32-byte-sector gather rate, profiles/r02_l2_peak.json), DRAM (the
    measured HBM copy rate).  `bound` is the resource with the highest
    fraction; SURVEY §8d's algorithmic-byte figure against HBM stays as
    `alg_frac` (the walk's gathers are served by L1/L2, not HBM)."""
    ev = stats["events"] / steps  # crossings per launch
    t = walk_s / steps
    sol_p, l2_p = ROOT / "profiles" / "walk_sol.json", ROOT / "profiles" / "r02_l2_peak.json"
    out = {"kernel": "walk_staged_kernel<192,2,0,1>", "kernel_ms_per_step": 1e3 * t,
           "alg_gbps": alg_gbps, "alg_frac": alg_gbps / hbm_peak,
           "algorithmic_bytes": "133 B/crossing + 100 B/move (SURVEY.md §8d) vs HBM",
           "hbm_peak_source": peak_src}
    try:
        sol = json.loads(sol_p.read_text())
        l2 = json.loads(l2_p.read_text())
    except (OSError, ValueError):
        out.update({"bound": "hbm", "achieved": alg_gbps, "peak": hbm_peak, "unit": "GB/s",
                    "frac": alg_gbps / hbm_peak, "traffic": None})
        return out
    pc = sol["per_crossing"]
    sms = int(l2.get("sms", 148))
    mhz = clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0
    hz = float(mhz) * 1e6
    units = {
        "issue": (pc["warp_instructions"] * ev / t, 4 * sms * hz, "warp-inst/s"),
        "l1tex_lsu": (pc["lsu_wavefronts"] * ev / t, sms * hz, "wavefronts/s"),
        "l2": (pc["l2_bytes"] * ev / t / 1e9,
               float(l2.get("l2_gather32_v8_gbs") or l2["l2_gather32_gbs"]), "GB/s"),
        "hbm": (pc["dram_bytes"] * ev / t / 1e9, hbm_peak, "GB/s"),
    }
    fr = {k: a / p for k, (a, p, _) in units.items()}
    bound = max(fr, key=fr.get)
    a, p, unit = units[bound]
    out.update({"bound": bound, "achieved": a, "peak": p, "unit": unit, "frac": fr[bound],
                "traffic": sol["per_launch"]["dram_bytes"],
                "traffic_source": f"dram__bytes_read+write.sum of one launch, {sol['source']}",
                "fracs": fr,
                "units": {k: {"achieved": a, "peak": p, "unit": u}
                          for k, (a, p, u) in units.items()},
                "sol_source": "profiles/walk_sol.json per-crossing demands x live crossings "
                              "/ live kernel time; peaks: 4 warp-inst and 1 LSU wavefront per "
                              f"SM-cycle at {mhz} MHz x {sms} SMs, L2 = measured 32-B sector "
                              "gather rate (profiles/r02_l2_peak.json), HBM = " + peak_src})
    return out


def run_ours(args):
    import torch
    rank, world, local = env_rank()
    # BENCH_SHARE_GPU=1: every rank on cuda:0 over gloo -- a smoke test of the
    # N > 1 path on a one-GPU box (tests/test_gpu_bench_dist.py); NCCL refuses
    # two ranks on one GPU
    share = os.environ.get("BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from paper_2504_19048_b200 import MeshTally, build_cube_mesh
    from paper_2504_19048_b200 import _lib

    mesh = build_cube_mesh(args.n)
    P = args.particles
    pos, dest = workload(P, args.sigma_t, rank)

    mt = MeshTally(mesh, P, device=local, sort=bool(args.sort),
                   warp_aggregate=None if args.warp_agg < 0 else bool(args.warp_agg),
                   staged=True if args.staged < 0 else args.staged,
                   stream_move=not args.no_stream_move)
    if args.blocks_per_sm:
        mt.set_option(_lib.BT_OPT_BLOCKS_PER_SM, args.blocks_per_sm)
    d_pos = torch.from_numpy(pos).to(dev)
    d_dest = torch.from_numpy(dest).to(dev)
    d_fly = torch.ones(P, dtype=torch.int8, device=dev)
    d_w = torch.ones(P, dtype=torch.float64, device=dev)
    mt.initialize_particle_location(d_pos)
    st = mt.read_particles(P)
    lost = int((st.element < 0).sum())
    mt.save_state()

    nb = mesh.num_elements
    tally_t = None
    if dist is not None:
        class _CAI:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                                 "data": (ptr, False), "version": 3,
                                                 "strides": None}
        tally_t = torch.as_tensor(_CAI(mt.tally_device_ptr(), nb), device=dev)

    stats = {"events": 0, "moves": 0, "walk_ms": 0.0, "kernels": 0}

    def step(record):
        mt.restore_state()
        s = mt.move_to_next_location(d_dest, d_fly, d_w)
        wk, _, kern = mt.last_timing()
        if dist is not None:
            dist.all_reduce(tally_t)
            w = torch.tensor([mt.source_weight], dtype=torch.float64, device=dev)
            dist.all_reduce(w)
            mt.finalize_batch(float(w.item()))
        else:
            mt.finalize_batch()
        if record:
            stats["events"] += s.events
            stats["moves"] += P - lost
            stats["walk_ms"] += wk
            stats["kernels"] += kern + 1
        return s

    for _ in range(args.warmup):
        step(False)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with clocks:
        e0.record()
        for _ in range(args.steps):
            step(True)
        e1.record()
        barrier()
    ms = e0.elapsed_time(e1)
    tot = torch.tensor([stats["events"], stats["moves"]], dtype=torch.float64, device=dev)
    msmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(tot)
        dist.all_reduce(msmax, op=dist.ReduceOp.MAX)
    ms_total = float(msmax.item())
    events_all, moves_all = float(tot[0].item()), float(tot[1].item())
    value = events_all / (ms_total / 1e3)
    moves_per_s = moves_all / (ms_total / 1e3)

    # roofline of the walk kernel (rank-local, CUDA events on the library stream)
    walk_s = stats["walk_ms"] / 1e3
    alg_bytes = B_CROSSING * stats["events"] + B_MOVE * stats["moves"]
    alg_gbps = alg_bytes / walk_s / 1e9
    hbm_peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    try:
        hbm_peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, ValueError, KeyError, TypeError):
        pass

    # e2e through the public API with host buffers: pinned (the contract's
    # case) and ordinary pageable numpy arrays (what a drop-in user passes)
    def e2e_run(h_pos, h_dest, h_fly, h_w):
        ev_e2e = 0

        def e2e_step():
            mt.initialize_particle_location(h_pos)
            s = mt.move_to_next_location(h_dest, h_fly, h_w)
            if dist is not None:
                dist.all_reduce(tally_t)
                w = torch.tensor([mt.source_weight], dtype=torch.float64, device=dev)
                dist.all_reduce(w)
                mt.finalize_batch(float(w.item()))
            else:
                mt.finalize_batch()
            return s
        e2e_step()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(args.steps):
            ev_e2e += e2e_step().events
        f1.record()
        barrier()
        ms2 = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        ev2 = torch.tensor([float(ev_e2e)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
            dist.all_reduce(ev2)
        return {"value": float(ev2.item()) / (float(ms2.item()) / 1e3), "unit": "crossings/s",
                "h2d_bytes_per_step": int(h_pos.nbytes + h_dest.nbytes + h_fly.nbytes
                                          + h_w.nbytes) * world,
                "d2h_bytes_per_step": 48 * world,
                "ms_per_step": float(ms2.item()) / args.steps}

    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(torch.from_numpy(pos).pin_memory().numpy(),
                      torch.from_numpy(dest).pin_memory().numpy(),
                      torch.ones(P, dtype=torch.int8).pin_memory().numpy(),
                      torch.ones(P, dtype=torch.float64).pin_memory().numpy())
        e2e["host_memory"] = "pinned"
        pg = e2e_run(pos, dest, np.ones(P, np.int8), np.ones(P))
        e2e["pageable"] = {"value": pg["value"], "ms_per_step": pg["ms_per_step"],
                           "host_memory": "pageable numpy (library-staged through a pinned "
                                          "ring by host threads)"}

    cpu = None
    # SURVEY §8f row 1 beside the headline: the device transport on the
    # paper's verification physics, device time of the
    # transport launches (tools/transport_line.py has the reference arm)
    transport = None
    if rank == 0 and not args.no_transport:
        from paper_2504_19048_b200 import transport as T
        tm = build_cube_mesh(10)
        T.run(T.RunConfig(mesh_n=10, num_particles=20_000, num_batches=1), tm, device=local)
        tr = T.run(T.RunConfig(mesh_n=10, num_particles=1_000_000, num_batches=2, seed=42), tm,
                   device=local)
        x = np.array([0.5])
        exact = _lib.load().bt_glibc_math(x.ctypes.data, 1, 0, local, x.ctypes.data) == 0
        transport = {"metric": "tet-crossings/s", "value": tr.events / tr.t_batch,
                     "unit": "crossings/s", "collisions_per_s": tr.collisions / tr.t_batch,
                     "histories_per_s": 2_000_000 / tr.t_batch, "events": tr.events,
                     "collisions": tr.collisions, "t_transport_s": tr.t_batch,
                     "bit_exact_histories": bool(exact),
                     "config": "paper verification physics: cube n=10 (6,000 tets), sigma_t = "
                               "sigma_s = 100/cm, 1e6 histories x 2 batches, seed 42"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, mrate, detail, _, _ = cpu_sample_rate(mesh, pos, dest, args.cpu_seconds)
        cpu = {"value": rate, "unit": "crossings/s", "cores": detail["cores"], "kind": "port",
               "sample": detail["sample"], "particle_moves_per_s": mrate,
               "seconds": detail["seconds"], "cpu": cpu_model()}

    if rank == 0:
        out = {
            "metric": "tet-crossings/s", "value": value, "unit": "crossings/s",
            "particle_moves_per_s": moves_per_s,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded numpy: uniform starts, isotropic exponential flights)",
            "config": config(args, world, mesh.num_elements),
            "crossings_per_move": events_all / max(moves_all, 1.0),
            "e2e": e2e,
            "roofline": roofline(stats, args.steps, walk_s, alg_gbps, hbm_peak, peak_src,
                                 clocks.summary()),
            "cpu_baseline": cpu,
            "transport": transport,
            "clocks": clocks.summary(),
            "gpu_launches": stats["kernels"],
            "lost_at_localization": lost,
        }
        print(json.dumps(out), flush=True)
    mt.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
