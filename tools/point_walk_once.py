"""Walk time of one move of 1e7 particles from the point source (SURVEY §8d
S) on the C2 mesh, Sigma_t given (the contended-tally case of the adaptive
warp aggregation): prints crossings and walk-kernel ms of the last of 3 moves."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, build_cube_mesh, synth  # noqa: E402

sig = float(sys.argv[1]) if len(sys.argv) > 1 else 100.0
n = 10_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(9)
pos = torch.tensor(synth.POINT_SOURCE, dtype=torch.float64, device=dev).repeat(n, 1)
mu = 2 * torch.rand(n, generator=g, device=dev, dtype=torch.float64) - 1
phi = 2 * math.pi * torch.rand(n, generator=g, device=dev, dtype=torch.float64)
s = torch.sqrt(1 - mu * mu)
d = torch.stack([s * torch.cos(phi), s * torch.sin(phi), mu], 1)
dest = (pos - torch.log(torch.rand(n, generator=g, device=dev, dtype=torch.float64))[:, None] / sig * d).contiguous()
fly = torch.ones(n, dtype=torch.int8, device=dev)
w = torch.ones(n, dtype=torch.float64, device=dev)
wa = int(sys.argv[2]) if len(sys.argv) > 2 else -1  # -1 adaptive, 0 never, 1 always
mt = MeshTally(build_cube_mesh(55), n, warp_aggregate=None if wa < 0 else bool(wa))
for _ in range(3):
    mt.initialize_particle_location(pos)
    r = mt.move_to_next_location(dest, fly, w)
print('point', sig, 'wagg', wa, r.events, round(mt.last_timing()[0], 3))
