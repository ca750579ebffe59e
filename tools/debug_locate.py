"""Debug: grid localization vs the exhaustive oracle on boundary points."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402
from paper_2504_19048_b200 import MeshTally, build_cube_mesh  # noqa: E402

gen = np.random.default_rng(17)
m = build_cube_mesh(7)
V, E = m.vertices, m.elements
k = 6000
el = gen.integers(0, E.shape[0], k)
bc = gen.dirichlet(np.ones(4), k)
kind = gen.integers(0, 4, k)
bc[kind == 0] = np.eye(4)[gen.integers(0, 4, (kind == 0).sum())]
for sel, nz in ((kind == 1, 2), (kind == 2, 3)):
    for i in np.where(sel)[0]:
        keep = gen.choice(4, nz, replace=False)
        b = np.zeros(4)
        b[keep] = gen.dirichlet(np.ones(nz))
        bc[i] = b
pts = np.einsum("ij,ijk->ik", bc, V[E[el]])
near = gen.random(k) < 0.3
pts[near] += gen.normal(size=(near.sum(), 3)) * 1e-11
mt = MeshTally(m, k)
mt.initialize_particle_location(pts)
st = mt.read_particles()
ex = orc.locate_exhaustive(m, pts)
bad = np.where(st.element != ex)[0]
print("mismatches", len(bad), "of", k)
for i in bad[:10]:
    print(i, kind[i], near[i], repr(pts[i].tolist()), "ours", st.element[i], "oracle", ex[i])
