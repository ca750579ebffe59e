"""C5 (torus shell, 5M tets, 1e7 particles, 10 chained moves) per refill mode:
per-move walk kernel time and whole-call time (diagnostics for the refill choice)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path[:0] = [str(Path(__file__).resolve().parent), str(Path(__file__).resolve().parent.parent)]
from sweep import flights_torch, iso_dirs_torch  # noqa: E402

from paper_2504_19048_b200 import MeshTally, build_torus_shell_mesh, synth  # noqa: E402

m = build_torus_shell_mesh(8, 256, 408, R=300.0, a_in=100.0, a_out=120.0)
g = np.random.default_rng(5)
n = 10_000_000
i = g.integers(0, 8, n)
j = g.integers(0, 32, n)
k = g.integers(0, 51, n)
elems = ((i * 256 + j) * 408 + k) * 6 + g.integers(0, 6, n)
pts = torch.from_numpy(synth.points_in_elements(g, m.vertices, m.elements, elems)).cuda()
dev = pts.device
for st in [int(a) for a in (sys.argv[1:] or ["1", "2"])]:
    mt = MeshTally(m, n, staged=st)
    gen = torch.Generator(device=dev)
    gen.manual_seed(20261017)
    w = torch.ones(n, dtype=torch.float64, device=dev)
    for rep in range(2):
        torch.cuda.synchronize()
        tb0 = time.perf_counter()
        mt.initialize_particle_location(pts)
        torch.cuda.synchronize()
        tinit = time.perf_counter() - tb0
        pos_t, _, alive_t = mt.particle_tensors()
        rows = []
        for mv in range(10):
            dest = (pos_t + flights_torch(torch, n, gen, dev, 1.0 / 30.0)[:, None] *
                    iso_dirs_torch(torch, n, gen, dev)).contiguous()
            f = alive_t.clone()
            nf = int(f.sum().item())
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mt.move_to_next_location(dest, f, w)
            t1 = time.perf_counter()
            wk, call, kern = mt.last_timing()
            rows.append((nf, round(wk, 3), round(call, 3), round(1e3 * (t1 - t0), 3), kern))
        mt.finalize_batch()
        torch.cuda.synchronize()
        tbatch = time.perf_counter() - tb0
        if rep == 1:
            print(f"staged={st} init {1e3 * tinit:.2f} ms batch {1e3 * tbatch:.2f} ms moves "
                  f"{sum(r[3] for r in rows):.2f} ms", rows, flush=True)
    mt.close()
