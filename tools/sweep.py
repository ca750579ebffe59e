"""Configuration sweeps of BASELINE.json configs[2..4] on one GPU (SURVEY.md
§8d C3, C4, C5).  Prints one JSON line per point; `--out` collects them.

  C3  particle-count sweep 1e5..1e8 on the 998,250-tet cube (n=55)
  C4  element-count sweep n in {12, 26, 55, 95, 119} with 1e7 particles
  C5  toroidal shell 8x256x408 (5,013,504 tets), fixed source in a sector,
      multi-move batches chained on the device (dest = pos + l*dir, flying = alive)

Timing: CUDA events around each move on the library stream (walk kernel) and
around the whole batch (localization + moves + finalize) on the torch stream;
inputs device-resident and generated before the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def iso_dirs_torch(torch, n, gen, dev):
    mu = 2.0 * torch.rand(n, generator=gen, device=dev, dtype=torch.float64) - 1.0
    phi = 2.0 * math.pi * torch.rand(n, generator=gen, device=dev, dtype=torch.float64)
    s = torch.sqrt(torch.clamp(1.0 - mu * mu, min=0.0))
    return torch.stack([s * torch.cos(phi), s * torch.sin(phi), mu], dim=1)


def flights_torch(torch, n, gen, dev, sigma_t):
    u = 1.0 - torch.rand(n, generator=gen, device=dev, dtype=torch.float64)
    return -torch.log(u) / sigma_t


def run_point(mesh, positions, sigma_t, moves, label, warm=1, chain=False, **mt_kw):
    """positions: device tensor (N,3).  One batch = init + `moves` moves.  The
    moves' destinations are generated before the timed region (a chained
    move continues from the previous destination, which is where a particle
    that reached it stands, bit for bit; `flying` = the library's alive flags),
    so the batch time is the library's alone."""
    import torch
    from paper_2504_19048_b200 import MeshTally
    dev = positions.device
    n = positions.shape[0]
    mt = MeshTally(mesh, n, device=dev.index or 0, **mt_kw)
    gen = torch.Generator(device=dev)
    gen.manual_seed(20261017)
    fly = torch.ones(n, dtype=torch.int8, device=dev)
    w = torch.ones(n, dtype=torch.float64, device=dev)
    dests = []
    cur = positions
    for k in range(moves):
        d = (cur + flights_torch(torch, n, gen, dev, sigma_t)[:, None] *
             iso_dirs_torch(torch, n, gen, dev)).contiguous()
        dests.append(d)
        if chain:
            cur = d

    def batch():
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record()
        mt.initialize_particle_location(positions)
        alive_t = mt.particle_tensors()[2] if chain else None  # (a host sync: chains only)
        ev = mv = 0
        walk = 0.0
        for k in range(moves):
            f = alive_t.clone() if chain else fly
            s = mt.move_to_next_location(dests[k], f, w)
            ev += s.events
            mv += s.reached + s.boundary_exits + s.stuck_terminations  # the flying count
            walk += mt.last_timing()[0]
        mt.finalize_batch()
        t1.record()
        torch.cuda.synchronize()
        return ev, mv, walk, t0.elapsed_time(t1)

    for _ in range(warm):
        batch()
    ev, mv, walk_ms, batch_ms = batch()
    out = {"point": label, "elements": mesh.num_elements, "particles": n, "moves": moves,
           "sigma_t": sigma_t, "crossings": ev, "particle_moves": mv,
           "crossings_per_move": ev / max(mv, 1),
           "walk_ms": walk_ms, "batch_ms": batch_ms,
           "crossings_per_s_walk": ev / (walk_ms / 1e3),
           "crossings_per_s_batch": ev / (batch_ms / 1e3),
           "moves_per_s_batch": mv / (batch_ms / 1e3),
           "gbps_walk": (133 * ev + 100 * mv) / (walk_ms / 1e3) / 1e9}
    mt.close()
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="c3,c4,c5,tr")
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-particles", type=float, default=1e8)
    args = ap.parse_args()
    import torch
    from paper_2504_19048_b200 import build_cube_mesh, build_torus_shell_mesh, synth
    dev = torch.device("cuda", 0)
    res = []
    which = set(args.which.split(","))
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)

    def box(n):
        return 0.05 + 0.9 * torch.rand(n, 3, generator=gen, device=dev, dtype=torch.float64)

    if "c3" in which:
        m = build_cube_mesh(55)
        for n in (1e5, 1e6, 1e7, 1e8):
            if n > args.max_particles:
                continue
            res.append(run_point(m, box(int(n)), 2.0, 1, f"C3 n=55 N={int(n):.0e}"))
        del m
    if "c4" in which:
        for nc in (12, 26, 55, 95, 119):
            t = time.time()
            m = build_cube_mesh(nc)
            build_s = time.time() - t
            r = run_point(m, box(10_000_000), 2.0, 1, f"C4 n={nc}")
            r["mesh_build_s"] = build_s
            res.append(r)
            del m
    if "c5" in which:
        t = time.time()
        m = build_torus_shell_mesh(8, 256, 408, R=300.0, a_in=100.0, a_out=120.0)
        build_s = time.time() - t
        # fixed source in a shell sector: theta index < 32, phi index < 51
        g = np.random.default_rng(5)
        i = g.integers(0, 8, 10_000_000)
        j = g.integers(0, 32, 10_000_000)
        k = g.integers(0, 51, 10_000_000)
        cells = (i * 256 + j) * 408 + k
        elems = cells * 6 + g.integers(0, 6, cells.size)
        pts = synth.points_in_elements(g, m.vertices, m.elements, elems)
        r = run_point(m, torch.from_numpy(pts).to(dev), 1.0 / 30.0, 10, "C5 torus 5.0M tets",
                      chain=True)
        r["mesh_build_s"] = build_s
        res.append(r)
    if "tr" in which:
        # paper verification physics: 1 cm cube (n=10), source in
        # 1/8 of the domain, sigma_t = sigma_s = 100 /cm, vacuum boundary
        from paper_2504_19048_b200 import transport as T
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle as orc
        m = build_cube_mesh(10)
        for n in (10_000, 1_000_000):
            cfg = T.RunConfig(mesh_n=10, num_particles=n, num_batches=2, seed=42)
            T.run(T.RunConfig(mesh_n=10, num_particles=min(n, 10000), num_batches=1), m)
            t = time.time()
            r = T.run(cfg, m)
            wall = time.time() - t
            out = {"point": f"transport paper physics N={n}", "elements": m.num_elements,
                   "particles": n, "batches": 2, "events": r.events,
                   "collisions": r.collisions, "t_transport_s": r.t_batch,
                   "t_localization_s": r.t_localization, "wall_s": wall,
                   "events_per_s": r.events / r.t_batch,
                   "collisions_per_s": r.collisions / r.t_batch,
                   "histories_per_s": 2 * n / r.t_batch}
            print(json.dumps(out), flush=True)
            res.append(out)
        # CPU: the oracle restatement of transport.run (serial, the reference's order)
        k = 2000
        t = time.time()
        o = orc.transport_run(m, [100.0], [[100.0]], k, 1, 42, ((0, 0, 0), (0.5, 0.5, 0.5)))
        dt = time.time() - t
        out = {"point": f"transport paper physics CPU oracle (1 thread) N={k}",
               "events": o["events"], "collisions": o["collisions"], "wall_s": dt,
               "events_per_s": o["events"] / dt, "collisions_per_s": o["collisions"] / dt}
        print(json.dumps(out), flush=True)
        res.append(out)
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(r) for r in res) + "\n")


if __name__ == "__main__":
    main()
