"""VTK and CSV writers byte-identical to the reference's (tally.py:155-200),
pinned by tests/golden/writers_ref.npz (oracle/gen_writers_golden.py ran the
reference's own writers)."""
import numpy as np

from golden_cases import GOLDEN
from paper_2504_19048_b200 import build_cube_mesh
from paper_2504_19048_b200.tally import FluxResult, write_flux_csv, write_vtk


def test_writers_match_reference(tmp_path):
    g = np.load(GOLDEN / "writers_ref.npz")
    res = FluxResult(mean=g["mean"], rel_error=g["rel_error"])
    write_vtk(build_cube_mesh(2), res, tmp_path / "f.vtk")
    write_flux_csv(res, tmp_path / "f.csv")
    assert (tmp_path / "f.vtk").read_text() == str(g["vtk"])
    assert (tmp_path / "f.csv").read_text() == str(g["csv"])
