"""Fixed per-call cost of short moves: batches of
device-resident, pre-generated inputs (no caller work inside the timed
region), timed on the device around the whole batch (initialize + moves +
finalize) against the library's own walk-kernel time.  One JSON line per
point.
    python tools/short_moves.py"""
import json
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402


def dests(gen, pos, sigma_t):
    n = pos.shape[0]
    dev = pos.device
    mu = 2.0 * torch.rand(n, generator=gen, device=dev, dtype=torch.float64) - 1.0
    phi = 2.0 * math.pi * torch.rand(n, generator=gen, device=dev, dtype=torch.float64)
    s = torch.sqrt(torch.clamp(1.0 - mu * mu, min=0.0))
    d = torch.stack([s * torch.cos(phi), s * torch.sin(phi), mu], dim=1)
    u = 1.0 - torch.rand(n, generator=gen, device=dev, dtype=torch.float64)
    return (pos + (-torch.log(u) / sigma_t)[:, None] * d).contiguous()


def point(mesh, n, sigma_t, moves, label, reps=5):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(11)
    pos = 0.05 + 0.9 * torch.rand(n, 3, generator=gen, device=dev, dtype=torch.float64)
    # a chain of moves: each destination continues from the previous one
    chain = [pos]
    for _ in range(moves):
        chain.append(dests(gen, chain[-1], sigma_t))
    fly = torch.ones(n, dtype=torch.int8, device=dev)
    w = torch.ones(n, dtype=torch.float64, device=dev)
    mt = MeshTally(mesh, n)
    best = None
    for r in range(reps + 1):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        mt.initialize_particle_location(pos)
        walk = 0.0
        ev = 0
        for k in range(moves):
            s = mt.move_to_next_location(chain[k + 1], fly, w)
            walk += mt.last_timing()[0]
            ev += s.events
        mt.finalize_batch()
        e1.record()
        torch.cuda.synchronize()
        batch = e0.elapsed_time(e1)
        if r and (best is None or batch < best[0]):
            best = (batch, walk, ev)
    mt.close()
    batch, walk, ev = best
    out = {"point": label, "elements": mesh.num_elements, "particles": n, "moves": moves,
           "sigma_t": sigma_t, "crossings": ev, "crossings_per_move": ev / (n * moves),
           "batch_ms": batch, "walk_ms": walk, "walk_over_batch": walk / batch,
           "per_move_overhead_ms": (batch - walk) / moves,
           "crossings_per_s_batch": ev / batch * 1e3, "crossings_per_s_walk": ev / walk * 1e3}
    print(json.dumps(out), flush=True)


def main():
    m55 = build_cube_mesh(55)
    for n in (100_000, 1_000_000, 10_000_000):
        point(m55, n, 2.0, 1, f"C3 N={n:.0e} sigma_t=2, one move")
    for n in (1_000_000, 10_000_000):
        point(m55, n, 100.0, 1, f"paper physics N={n:.0e} sigma_t=100, one move")
        point(m55, n, 100.0, 10, f"paper physics N={n:.0e} sigma_t=100, 10 chained moves")


if __name__ == "__main__":
    main()
