"""Device-input bench step breakdown (bench.py's timed step): wall time of
restore_state, move_to_next_location and finalize_batch, plus the library's
own kernel timing, to locate the step's non-kernel time."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402

P = 10_000_000
m = build_cube_mesh(55)
pos, dest = workload(P, 2.0, 0)
dev = torch.device("cuda", 0)
d_pos, d_dest = torch.from_numpy(pos).to(dev), torch.from_numpy(dest).to(dev)
d_fly = torch.ones(P, dtype=torch.int8, device=dev)
d_w = torch.ones(P, dtype=torch.float64, device=dev)
mt = MeshTally(m, P)
mt.initialize_particle_location(d_pos)
mt.save_state()
for it in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mt.restore_state()
    t1 = time.perf_counter()
    mt.move_to_next_location(d_dest, d_fly, d_w)
    t2 = time.perf_counter()
    walk_ms, call_ms, k = mt.last_timing()
    mt.finalize_batch()
    t3 = time.perf_counter()
    print(f"iter {it}: restore {1e3*(t1-t0):.3f} ms, move {1e3*(t2-t1):.3f} ms (walk {walk_ms:.3f}, "
          f"call events {call_ms:.3f}), finalize {1e3*(t3-t2):.3f} ms, total {1e3*(t3-t0):.3f}",
          flush=True)
