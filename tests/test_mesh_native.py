"""The library's native mesh ingest (bt_mesh_read / bt_mesh_from_arrays,
csrc/mesh_io.cuh) against the host numpy path, which is itself pinned to the
reference's meshes (tests/test_mesh.py): bit-identical arrays and the same
MalformedMeshError messages; and the writers' float format against Python's
repr.  Host-only code paths: these run without a GPU."""

import struct

import numpy as np
import pytest

from paper_2504_19048_b200 import _lib
from paper_2504_19048_b200 import mesh as M

FIELDS = ("vertices", "elements", "adj_elem", "adj_face", "volumes", "centroids",
          "bounding_box")


def _same(a, b):
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype and np.array_equal(x, y), f


def _bt_repr(x: float) -> str:
    import ctypes as C
    buf = C.create_string_buffer(48)
    _lib.check(_lib.load().bt_format_double(float(x), buf, 48))
    return buf.value.decode()


def test_float_format_is_python_repr():
    gen = np.random.default_rng(3)
    vals = [0.0, -0.0, 1.0, -1.0, 0.1, 1e-4, 1e-5, 1.5e-5, 9.999e-5, 123.0, 1e15, 1e16,
            1.2345e16, 1e17, 1e22, 1e-300, 5e-324, 1.7976931348623157e308, 2.0 ** 53,
            float("inf"), float("-inf"), 0.8999999999999999, 1 / 3, 2 / 3, 4678.448070712665]
    bits = gen.integers(0, 2 ** 63, 20000, dtype=np.int64)
    vals += [struct.unpack("<d", struct.pack("<q", int(b)))[0] for b in bits]
    vals += list(gen.random(5000) * 10.0 ** gen.integers(-20, 20, 5000))
    vals += list(np.round(gen.random(2000) * 1000, 3))
    for v in vals:
        if v != v:
            continue
        assert _bt_repr(v) == repr(float(v)), v


@pytest.mark.parametrize("n", [1, 2, 7, 16])
def test_native_cube_equals_numpy(n):
    _same(M.build_cube_mesh(n, device=None), M.build_cube_mesh(n, device=-1))


def test_native_torus_permuted_scaled_equals_numpy():
    v, e = M.torus_shell_arrays(3, 16, 24)
    gen = np.random.default_rng(1)
    for _ in range(4):
        perm = np.argsort(gen.random((e.shape[0], 4)), axis=1)
        els = np.take_along_axis(e, perm, axis=1)[gen.permutation(e.shape[0])]
        vv = v * gen.uniform(1e-3, 1e3) + gen.normal(size=3) * 100.0
        _same(M.TetMesh.from_arrays(vv, els, device=None), M.TetMesh.from_arrays(vv, els, device=-1))


def test_native_errors_match_numpy():
    v = np.random.default_rng(0).random((6, 3))
    cases = [np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]]),
             np.array([[0, 1, 2, 3], [0, 1, 2, 3]]),
             np.array([[0, 1, 1, 3]]),
             np.array([[0, 1, 2, 6]]),
             np.array([[0, 1, 2, -1]])]
    for els in cases:
        msgs = []
        for dev in (None, -1):
            with pytest.raises(M.MalformedMeshError) as ei:
                M.TetMesh.from_arrays(v, els, device=dev)
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1]


def test_native_reader_roundtrip_and_errors(tmp_path):
    gen = np.random.default_rng(8)
    v, e = M.torus_shell_arrays(2, 8, 12)
    m = M.TetMesh.from_arrays(v * 1.37 + 0.1, e, device=None)
    p = tmp_path / "t.tet"
    M.write_tetmesh(m, p)
    _same(M.read_tetmesh(p, device=None), M.read_tetmesh(p, device=-1))
    # CRLF line ends, trailing blank lines, '+' signs: what float()/int() accept
    text = p.read_text().replace("\n", "\r\n") + "\r\n\r\n"
    q = tmp_path / "crlf.tet"
    q.write_text(text)
    _same(M.read_tetmesh(p, device=None), M.read_tetmesh(q, device=-1))
    for body in ("tetmesh 4\n", "tetmesh a b\n", "mesh 4 1\n", "tetmesh 4 1\n0 0 0\n",
                 "tetmesh 4 1\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n0 1 2\n",
                 "tetmesh 4 1\n0 0 0\n1 0 0\n0 1 0\n0 0 1 5\n0 1 2 3\n",
                 "tetmesh 4 1\n0 0 0\n1 0 0\n0 1 0\n0 0 z\n0 1 2 3\n"):
        bad = tmp_path / "bad.tet"
        bad.write_text(body)
        for dev in (None, -1):
            with pytest.raises(M.MalformedMeshError):
                M.read_tetmesh(bad, device=dev)
    del gen
