"""Host mesh builder vs the reference's meshes (tests/golden/mesh_ref.npz)
and the reference's own mesh test cases (pkg/tests/test_mesh.py)."""

import numpy as np
import pytest

from golden_cases import GOLDEN
from paper_2504_19048_b200 import mesh as M

FIELDS = ("vertices", "elements", "adj_elem", "adj_face", "volumes", "centroids",
          "bounding_box")


# device: None = the host numpy builder; "auto" = the library's native ingest
# (bt_mesh_from_arrays; host adjacency without a GPU, GPU adjacency with one)
DEVICES = [None, "auto"]


@pytest.mark.parametrize("device", DEVICES)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 10])
def test_cube_matches_reference(n, device):
    d = np.load(GOLDEN / "mesh_ref.npz")
    m = M.build_cube_mesh(n, device=device)
    for f in FIELDS:
        ref = d[f"cube{n}_{f}"]
        got = getattr(m, f)
        assert got.dtype == ref.dtype and np.array_equal(got, ref), f


@pytest.mark.parametrize("device", DEVICES)
def test_torus_matches_reference(device):
    d = np.load(GOLDEN / "mesh_ref.npz")
    m = M.TetMesh.from_arrays(d["torus_raw_vertices"], d["torus_raw_elements"], device=device)
    for f in FIELDS:
        assert np.array_equal(getattr(m, f), d[f"torus_{f}"]), f
    assert M.validate(m) == []


@pytest.mark.parametrize("n", [1, 2, 4])
def test_cube_counts(n):
    m = M.build_cube_mesh(n)
    assert m.num_elements == 6 * n ** 3
    assert m.num_vertices == (n + 1) ** 3
    assert int((m.adj_elem < 0).sum()) == 12 * n * n
    assert abs(m.volumes.sum() - 1.0) < 1e-12
    assert (m.volumes > 0).all()
    assert M.validate(m) == []


def test_bad_params():
    with pytest.raises(ValueError):
        M.build_cube_mesh(0)
    with pytest.raises(ValueError):
        M.build_cube_mesh(2, edge_length=-1.0)


@pytest.mark.parametrize("device", DEVICES)
def test_adjacency_two_tets_and_errors(device):
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 1]], float)
    e = np.array([[0, 1, 2, 3], [1, 2, 3, 4]])
    m = M.TetMesh.from_arrays(v, e, device=device)
    assert (m.adj_elem >= 0).sum() == 2
    assert M.validate(m) == []
    with pytest.raises(M.MalformedMeshError):   # three tets on one face
        M.build_adjacency(np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]]), 6)
    with pytest.raises(M.MalformedMeshError):   # duplicated element (reference misses it)
        M.build_adjacency(np.array([[0, 1, 2, 3], [0, 1, 2, 3]]), 4)
    with pytest.raises(M.MalformedMeshError):   # degenerate
        M.TetMesh.from_arrays(np.zeros((4, 3)), [[0, 1, 2, 3]], device=device)
    with pytest.raises(M.MalformedMeshError):
        M.TetMesh.from_arrays(v, [[0, 1, 2, 9]], device=device)


@pytest.mark.parametrize("device", DEVICES)
def test_orientation_fixed(device):
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    m = M.TetMesh.from_arrays(v, [[0, 1, 3, 2]], device=device)
    assert m.elements.tolist() == [[0, 1, 2, 3]]
    assert m.volumes[0] == pytest.approx(1 / 6)


@pytest.mark.parametrize("device", DEVICES)
def test_text_roundtrip(tmp_path, device):
    m = M.build_cube_mesh(3)
    p = tmp_path / "m.tet"
    M.write_tetmesh(m, p)
    r = M.read_tetmesh(p, device=device)
    for f in FIELDS:
        if f == "volumes":   # recomputed from re-oriented rows: equal to rounding
            assert np.allclose(r.volumes, m.volumes, rtol=1e-14, atol=0)
        else:
            assert np.array_equal(getattr(r, f), getattr(m, f)), f
    bad = tmp_path / "bad.tet"
    bad.write_text("tetmesh 4 1\n0 0 0\n1 0 0\n0 1 0\n")
    with pytest.raises(M.MalformedMeshError):
        M.read_tetmesh(bad, device=device)
    bad.write_text("mesh 4 1\n")
    with pytest.raises(M.MalformedMeshError):
        M.read_tetmesh(bad, device=device)
    bad.write_text("tetmesh 4 1\n0 0 0\n1 0 x\n0 1 0\n0 0 1\n0 1 2 3\n")
    with pytest.raises(M.MalformedMeshError):
        M.read_tetmesh(bad, device=device)
