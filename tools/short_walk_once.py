"""One paper-physics move (C2 mesh, 1e7 particles, sigma_t = 100, device
inputs) after a warm-up move: the capture target of tools/gpu_prof_short.sh."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
sig = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(3)
pos = 0.05 + 0.9 * torch.rand(n, 3, generator=g, device=dev, dtype=torch.float64)
mu = 2 * torch.rand(n, generator=g, device=dev, dtype=torch.float64) - 1
phi = 2 * math.pi * torch.rand(n, generator=g, device=dev, dtype=torch.float64)
s = torch.sqrt(1 - mu * mu)
d = torch.stack([s * torch.cos(phi), s * torch.sin(phi), mu], 1)
dest = (pos - torch.log(torch.rand(n, generator=g, device=dev, dtype=torch.float64))[:, None] / sig * d).contiguous()
fly = torch.ones(n, dtype=torch.int8, device=dev)
w = torch.ones(n, dtype=torch.float64, device=dev)
mt = MeshTally(build_cube_mesh(55), n)
for _ in range(3):
    mt.initialize_particle_location(pos)
    r = mt.move_to_next_location(dest, fly, w)
    print(r.events, mt.last_timing()[0], flush=True)
