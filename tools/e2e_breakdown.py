"""Host-side breakdown of the e2e step (bench.py's e2e loop): wall time of
initialize_particle_location (host positions), move_to_next_location (host
inputs) and finalize, plus the library's own event timings."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402

P = 10_000_000
m = build_cube_mesh(55)
pos, dest = workload(P, 2.0, 0)
h_pos = torch.from_numpy(pos).pin_memory().numpy()
h_dest = torch.from_numpy(dest).pin_memory().numpy()
h_fly = torch.ones(P, dtype=torch.int8).pin_memory().numpy()
h_w = torch.ones(P, dtype=torch.float64).pin_memory().numpy()
mt = MeshTally(m, P, move_chunks=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mt.initialize_particle_location(h_pos)
    t1 = time.perf_counter()
    mt.move_to_next_location(h_dest, h_fly, h_w)
    t2 = time.perf_counter()
    walk_ms, call_ms, k = mt.last_timing()
    mt.finalize_batch()
    t3 = time.perf_counter()
    print(f"iter {it}: init {1e3*(t1-t0):.2f} ms, move {1e3*(t2-t1):.2f} ms "
          f"(walk kernels {walk_ms:.2f}, move call events {call_ms:.2f}), "
          f"finalize {1e3*(t3-t2):.2f} ms, total {1e3*(t3-t0):.2f} ms", flush=True)
