"""Grid localization throughput per lane-group width (BT_OPT_LOCATE_LANES) on the
bench workload (C2 mesh, 1e7 uniform points, device inputs); checks that every
width returns the same elements."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 55
P = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
m = build_cube_mesh(n)
pos = torch.from_numpy(synth.uniform_box(synth.rng(), P)).cuda()
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
mt = MeshTally(m, P)
mt.initialize_particle_location(pos[:1])  # builds the grid
torch.cuda.synchronize()
print(json.dumps({"mesh_elements": m.num_elements, "create_and_grid_build_s": time.perf_counter() - t0}),
      flush=True)
ref = None
for g in (1, 2, 4, 8, 16, 32):
    mt.set_option(_lib.BT_OPT_LOCATE_LANES, g)
    mt.initialize_particle_location(pos)
    ms = []
    for _ in range(3):
        mt.initialize_particle_location(pos)
        ms.append(mt.last_timing()[1])
    el = mt.read_particles(P).element
    same = True if ref is None else bool(np.array_equal(el, ref))
    ref = el if ref is None else ref
    print(json.dumps({"lanes": g, "ms": min(ms), "points_per_s": P / (min(ms) / 1e3),
                      "same_elements": same, "mesh_elements": m.num_elements}), flush=True)
