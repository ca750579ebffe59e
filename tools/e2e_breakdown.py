"""Host-side breakdown of the e2e step (bench.py's e2e loop): wall time of
initialize_particle_location (host positions), move_to_next_location (host
inputs) and finalize, plus the library's own event timings, for pinned and
pageable inputs with and without the deferred initialize (BT_OPT_DEFER_INIT).

    python tools/e2e_breakdown.py [move_chunks] [stream_move 0/1] [particles]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import workload  # noqa: E402
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh  # noqa: E402

P = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000_000
m = build_cube_mesh(55)
pos, dest = workload(P, 2.0, 0)
pinned = (torch.from_numpy(pos).pin_memory().numpy(), torch.from_numpy(dest).pin_memory().numpy(),
          torch.ones(P, dtype=torch.int8).pin_memory().numpy(),
          torch.ones(P, dtype=torch.float64).pin_memory().numpy())
pageable = (pos, dest, np.ones(P, np.int8), np.ones(P))
SM = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mt = MeshTally(m, P, move_chunks=int(sys.argv[1]) if len(sys.argv) > 1 else 0, stream_move=bool(SM))
import os
for label, (h_pos, h_dest, h_fly, h_w) in (("pinned", pinned), ("pageable", pageable)):
    for defer in (1, 0):
        mt.set_option(_lib.BT_OPT_DEFER_INIT, defer)
        tot = []
        for it in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mt.initialize_particle_location(h_pos)
            t1 = time.perf_counter()
            mt.move_to_next_location(h_dest, h_fly, h_w)
            t2 = time.perf_counter()
            walk_ms, call_ms, k = mt.last_timing()
            mt.finalize_batch()
            t3 = time.perf_counter()
            if it:
                tot.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), walk_ms, 1e3 * (t3 - t2),
                            1e3 * (t3 - t0)))
        a = np.mean(tot, axis=0)
        print(f"P={P} {label:8s} stream_move={SM} defer={defer} init_chunks={os.environ.get('B200TALLY_INIT_CHUNKS', 4)}: init {a[0]:.2f} ms, move {a[1]:.2f} ms (walk kernels "
              f"{a[2]:.2f}), finalize {a[3]:.2f} ms, total {a[4]:.2f} ms", flush=True)
