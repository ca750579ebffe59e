"""Golden VTK / CSV outputs of the REFERENCE's writers (meshtally.tally.write_vtk,
write_flux_csv; tally.py:155-200) for a 2-group flux on a small cube mesh,
written to tests/golden/writers_ref.npz (run in the build container, where
/root/reference is importable):

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_writers_golden.py
"""
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
import meshtally as mt  # noqa: E402
from meshtally import tally as rt  # noqa: E402

mesh = mt.build_cube_mesh(2)
gen = np.random.default_rng(31)
mean = gen.random((mesh.num_elements, 2)) * 10.0 ** gen.integers(-12, 3, (mesh.num_elements, 2))
mean[0, 0] = 0.0
rel = gen.random((mesh.num_elements, 2))
res = rt.FluxResult(mean=mean, rel_error=rel)
with tempfile.TemporaryDirectory() as d:
    rt.write_vtk(mesh, res, Path(d) / "f.vtk")
    rt.write_flux_csv(res, Path(d) / "f.csv")
    vtk = (Path(d) / "f.vtk").read_text()
    csv = (Path(d) / "f.csv").read_text()
np.savez_compressed(ROOT / "tests" / "golden" / "writers_ref.npz", mean=mean, rel_error=rel,
                    vtk=np.array(vtk), csv=np.array(csv))
print("wrote writers_ref.npz", len(vtk), len(csv))
