"""Locality probe: walk throughput on a mesh whose elements and vertices are
renumbered along a Morton curve, against the original numbering (same
geometry, same particles).  Used to size the renumbering idea."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from sweep import run_point  # noqa: E402

from paper_2504_19048_b200 import TetMesh, build_cube_mesh  # noqa: E402


def morton3(p, bits=10):
    q = np.clip((p * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    code = np.zeros(len(p), np.int64)
    for b in range(bits):
        for ax in range(3):
            code |= ((q[:, ax] >> b) & 1) << (3 * b + ax)
    return code


n = int(sys.argv[1]) if len(sys.argv) > 1 else 119
m = build_cube_mesh(n)
lo, hi = m.vertices.min(0), m.vertices.max(0)
vperm = np.argsort(morton3((m.vertices - lo) / (hi - lo)), kind="stable")
vinv = np.empty_like(vperm)
vinv[vperm] = np.arange(len(vperm))
el = vinv[m.elements]
cent = (m.vertices[m.elements].mean(1) - lo) / (hi - lo)
eperm = np.argsort(morton3(cent), kind="stable")
t = time.time()
m2 = TetMesh.from_arrays(m.vertices[vperm], el[eperm])
print("renumbered in", round(time.time() - t, 1), "s", flush=True)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
box = 0.05 + 0.9 * torch.rand(10_000_000, 3, generator=gen, device=dev, dtype=torch.float64)
for name, mesh in (("original", m), ("morton", m2)):
    r = run_point(mesh, box, 2.0, 1, f"n={n} {name}")
