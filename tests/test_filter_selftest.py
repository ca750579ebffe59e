"""CPU self-test of the filtered exit search against the reference's literal
arithmetic (tests/native/filter_selftest.cu), step by step along walks, on
random and adversarial (grid-plane, vertex-aligned, long/short) segments."""

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2504_19048_b200 import build_cube_mesh, build_torus_shell_mesh, synth

HERE = Path(__file__).resolve().parent
SRC = HERE / "native" / "filter_selftest.cu"
LIB = HERE / "native" / "libfilter_selftest.so"


@pytest.fixture(scope="module")
def lib():
    deps = [SRC, HERE.parent / "paper_2504_19048_b200" / "csrc" / "geometry.cuh"]
    if not LIB.exists() or LIB.stat().st_mtime < max(d.stat().st_mtime for d in deps):
        subprocess.run(["nvcc", "-O2", "-std=c++17", "-x", "cu", "-Xcompiler",
                        "-fPIC,-ffp-contract=off", "-shared", "-o", str(LIB), str(SRC)],
                       check=True)
    L = C.CDLL(str(LIB))
    L.bt_filter_selftest.argtypes = [C.c_void_p] * 7 + [C.c_int64, C.c_int64, C.c_void_p]
    return L


def run(L, mesh, elem, pos, dest, max_steps=100000):
    pos = np.ascontiguousarray(pos, dtype=np.float64)
    dest = np.ascontiguousarray(dest, dtype=np.float64)
    elem = np.ascontiguousarray(elem, dtype=np.int32)
    st = np.zeros(5, np.int64)
    L.bt_filter_selftest(mesh.vertices.ctypes.data, mesh.elements.ctypes.data,
                         mesh.adj_elem.ctypes.data, mesh.adj_face.ctypes.data,
                         elem.ctypes.data, pos.ctypes.data, dest.ctypes.data,
                         pos.shape[0], max_steps, st.ctypes.data)
    return dict(zip(("steps", "mismatches", "fallbacks", "stuck", "undecided32"), st.tolist()))


def _locate(mesh, pts):
    import sys
    sys.path.insert(0, str(HERE.parent / "oracle"))
    import oracle as orc
    return orc.locate_exhaustive(mesh, pts)


def test_random_walks_cube(lib):
    m = build_cube_mesh(12)
    gen = np.random.default_rng(1)
    pos = synth.uniform_box(gen, 20000)
    dest = pos + gen.normal(size=pos.shape) * 0.6
    r = run(lib, m, _locate(m, pos), pos, dest)
    assert r["steps"] > 100000
    assert r["mismatches"] == 0, r
    assert r["fallbacks"] < 1e-3 * r["steps"], r
    # the fp32 pre-filter decides almost every generic step
    assert r["undecided32"] < 5e-3 * r["steps"], r


def test_adversarial_grid_planes(lib):
    m = build_cube_mesh(10)
    gen = np.random.default_rng(2)
    k = 20000
    grid = m.vertices[:11, 2]           # exact vertex coordinates k*h
    pos = synth.uniform_box(gen, k, 0.06, 0.94)
    dest = synth.uniform_box(gen, k, -0.2, 1.2)
    # snap one or two coordinates of start / destination onto grid planes
    for arr in (pos, dest):
        for ax in range(3):
            sel = gen.random(k) < 0.35
            arr[sel, ax] = grid[gen.integers(1, 10, sel.sum())]
    # and some exactly diagonal directions (Kuhn face planes)
    d = gen.random(k) < 0.2
    dest[d] = pos[d] + (gen.random((d.sum(), 1)) - 0.5) * np.array([1.0, 1.0, 1.0])
    r = run(lib, m, _locate(m, pos), pos, dest)
    assert r["mismatches"] == 0, r
    assert r["fallbacks"] > 0  # the adversarial set does reach the exact path


def test_short_and_vertex_segments(lib):
    m = build_cube_mesh(7)
    gen = np.random.default_rng(3)
    k = 20000
    pos = synth.uniform_box(gen, k)
    scale = 10.0 ** gen.uniform(-13, 0, (k, 1))
    dest = pos + gen.normal(size=(k, 3)) * scale
    inner = m.vertices[(m.vertices > 0.1).all(1) & (m.vertices < 0.9).all(1)]
    vd = gen.random(k) < 0.2
    dest[vd] = inner[gen.integers(0, len(inner), vd.sum())]
    r = run(lib, m, _locate(m, pos), pos, dest)
    assert r["mismatches"] == 0, r


def test_torus_walks(lib):
    m = build_torus_shell_mesh(3, 16, 24)
    gen = np.random.default_rng(4)
    k = 5000
    cells = gen.integers(0, m.num_elements, k)
    pos = synth.points_in_elements(gen, m.vertices, m.elements, cells)
    dest = pos + gen.normal(size=pos.shape) * 60.0
    r = run(lib, m, cells, pos, dest)
    assert r["steps"] > 10000
    assert r["mismatches"] == 0, r


@pytest.mark.parametrize("tol", [1e-10, 1e-9])
def test_contains_fast_matches_exact(lib, tol):
    m = build_cube_mesh(4)
    gen = np.random.default_rng(5)
    k = 6000
    pts = gen.uniform(-0.05, 1.05, (k, 3))
    grid = m.vertices[:5, 2]
    for ax in range(3):  # points on grid planes, edges and vertices
        sel = gen.random(k) < 0.4
        pts[sel, ax] = grid[gen.integers(0, 5, sel.sum())]
    # points within ~tol of faces: nudge vertices/face points by tiny offsets
    near = gen.random(k) < 0.2
    pts[near] += gen.normal(size=(near.sum(), 3)) * 1e-11
    L = lib
    L.bt_contains_selftest.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_double, C.c_void_p]
    L.bt_contains_selftest.restype = C.c_int64
    fb = np.zeros(1, np.int64)
    pts = np.ascontiguousarray(pts)
    mism = L.bt_contains_selftest(m.vertices.ctypes.data, m.elements.ctypes.data,
                                  m.num_elements, pts.ctypes.data, k, tol, fb.ctypes.data)
    assert mism == 0


@pytest.mark.parametrize("scale,offset", [(1e-2, 1e4), (1e3, -5e5), (1e9, 0.0), (1e11, 3e12)])
def test_scaled_translated_meshes(lib, scale, offset):
    """The fp32 pre-filter's bounds are scale-free inside its range guard and
    hand everything outside it (tiny or huge meshes) to the fp64 filter."""
    from paper_2504_19048_b200 import TetMesh
    m0 = build_cube_mesh(6)
    m = TetMesh.from_arrays(m0.vertices * scale + offset, m0.elements)
    gen = np.random.default_rng(6)
    k = 4000
    pos = synth.uniform_box(gen, k) * scale + offset
    dest = pos + gen.normal(size=pos.shape) * 0.4 * scale
    r = run(lib, m, _locate(m, pos), pos, dest)
    assert r["steps"] > 4000
    assert r["mismatches"] == 0, r
