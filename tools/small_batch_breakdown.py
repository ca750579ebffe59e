"""Where a small batch's time goes (C3 1e5 point: C2 mesh, 1e5 particles,
one Sigma_t = 2 move, device inputs): host wall time of each API call and
the device time between CUDA events recorded around them, best of 20."""
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(5)
pos = 0.05 + 0.9 * torch.rand(n, 3, generator=g, device=dev, dtype=torch.float64)
mu = 2 * torch.rand(n, generator=g, device=dev, dtype=torch.float64) - 1
phi = 2 * math.pi * torch.rand(n, generator=g, device=dev, dtype=torch.float64)
s = torch.sqrt(1 - mu * mu)
d = torch.stack([s * torch.cos(phi), s * torch.sin(phi), mu], 1)
dest = (pos - torch.log(torch.rand(n, generator=g, device=dev, dtype=torch.float64))[:, None] / 2.0 * d).contiguous()
fly = torch.ones(n, dtype=torch.int8, device=dev)
w = torch.ones(n, dtype=torch.float64, device=dev)
mt = MeshTally(build_cube_mesh(55), n)
best = None
for it in range(21):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record()
    mt.initialize_particle_location(pos)
    t1 = time.perf_counter()
    ev[1].record()
    mt.move_to_next_location(dest, fly, w)
    t2 = time.perf_counter()
    walk = mt.last_timing()[0]
    ev[2].record()
    mt.finalize_batch()
    t3 = time.perf_counter()
    ev[3].record()
    torch.cuda.synchronize()
    row = (1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), ev[0].elapsed_time(ev[1]),
           ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), walk, ev[0].elapsed_time(ev[3]))
    if it and (best is None or row[-1] < best[-1]):
        best = row
print("host ms: init %.3f move %.3f finalize %.3f | device ms: init %.3f move %.3f finalize %.3f "
      "| walk kernel %.3f | batch %.3f" % best)
