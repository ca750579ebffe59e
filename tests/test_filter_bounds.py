"""The fp32 pre-filter's error bounds (csrc/geometry.cuh, "Single-precision
pre-filter") checked against EXACT rational arithmetic: for tets and segments
drawn from walks on cube, torus, sliver and scaled meshes, every determinant
the filter evaluates in fp32 is compared with the exact determinant of the
reference's own fp64 difference vectors (Fraction), and the observed error is
required to stay inside the bound the margins are built on.

Claims checked (u = 2^-24, P32 = Nx^2 (S + Nx), Pc = Nx^2 (S + 2 Nx)):
  face D, NT, NU, NW:           |err| <= 14.1 u P32
  containment t_k = b.n_k (= D_k - NT_k) and y0 = |Dc|-t1-t2-t3 (= sign(Dc) (NT0 - D0)):
                                |err| <= 29.3 u P32 <= 37 u Pc  (the margin is 48 u Pc)
"""
import ctypes as C
from fractions import Fraction as Fr

import numpy as np
import pytest

from test_filter_selftest import LIB, lib as _lib_fixture  # noqa: F401  (builds the shim)
from paper_2504_19048_b200 import TetMesh, build_cube_mesh, build_torus_shell_mesh, synth

U = 2.0 ** -24
FV = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))


def det(a, b, c):
    return (a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0])
            + a[2] * (b[0] * c[1] - b[1] * c[0]))


def sub(p, q):  # the reference's fp64 difference, then exact
    return [Fr(float(np.float64(p[k]) - np.float64(q[k]))) for k in range(3)]


def cases(gen, mesh, k, scale):
    el = gen.integers(0, mesh.num_elements, k)
    V = mesh.vertices[mesh.elements[el]]                       # (k, 4, 3)
    bc = gen.dirichlet(np.ones(4), k)
    o = np.einsum("ij,ijk->ik", bc, V)
    onface = gen.random(k) < 0.5                                  # origins on a face (walk steps)
    bc2 = bc.copy()
    bc2[onface, gen.integers(0, 4, onface.sum())] = 0.0
    bc2 /= bc2.sum(1, keepdims=True)
    o[onface] = np.einsum("ij,ijk->ik", bc2[onface], V[onface])
    d = o + gen.normal(size=o.shape) * scale * 10.0 ** gen.uniform(-3, 1, (k, 1))
    return V, o, d


def check(L, V, o, d):
    k = V.shape[0]
    tets = np.ascontiguousarray(np.concatenate([V[:, :, 0], V[:, :, 1], V[:, :, 2]], axis=1))
    od = np.ascontiguousarray(np.concatenate([o, d], axis=1))
    out = np.zeros((k, 27), np.float32)
    pm = np.zeros(1, np.int64)
    L.bt_f32_probe(tets.ctypes.data, od.ctypes.data, k, out.ctypes.data, pm.ctypes.data)
    # the packed (FFMA2) filter's intermediates equal the scalar formulation's
    assert pm[0] == 0, pm
    worst = {"face": 0.0, "y0": 0.0, "cont32": 0.0}
    for i in range(k):
        p = out[i]
        if p[0] < 1:
            continue
        v = [V[i, j] for j in range(4)]
        a = [sub(v[j], v[0]) for j in (1, 2, 3)]
        b = sub(d[i], v[0])
        Dc = det(a[0], a[1], a[2])
        N = [det(b, a[1], a[2]), det(a[0], b, a[2]), det(a[0], a[1], b)]
        sg = 1 if Dc >= 0 else -1
        y0 = sg * (Dc - N[0] - N[1] - N[2])
        Pc, P32 = float(p[9]), float(p[10])
        worst["y0"] = max(worst["y0"], abs(float(Fr(float(p[8])) - y0)) / (U * Pc))
        for got, e in zip((p[5], p[6], p[7], p[8]), (sg * N[0], sg * N[1], sg * N[2], y0)):
            worst["cont32"] = max(worst["cont32"], abs(float(Fr(float(got)) - e)) / (U * P32))
        if p[0] < 2:
            continue
        s = sub(d[i], o[i])
        for f, (ia, ib, ic) in enumerate(FV):
            e1, e2, r = sub(v[ia], v[ib]), sub(v[ia], v[ic]), sub(v[ia], o[i])
            exact = (det(s, e1, e2), det(r, e1, e2), det(s, r, e2), det(s, e1, r))
            got = (p[11 + f], p[15 + f], p[19 + f], p[23 + f])
            for g, e in zip(got, exact):
                worst["face"] = max(worst["face"], abs(float(Fr(float(g)) - e)) / (U * P32))
    return worst


@pytest.mark.parametrize("name", ["cube", "torus", "sliver", "scaled"])
def test_fp32_filter_error_bounds(_lib_fixture, name):
    L = _lib_fixture
    L.bt_f32_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    gen = np.random.default_rng(123)
    if name == "cube":
        m, scale = build_cube_mesh(20), 0.05
    elif name == "torus":
        m, scale = build_torus_shell_mesh(3, 16, 24), 5.0
    elif name == "sliver":  # a strongly anisotropic cube: flat, elongated tets
        m0 = build_cube_mesh(6)
        m, scale = TetMesh.from_arrays(m0.vertices * np.array([1.0, 1e-3, 30.0]), m0.elements), 1.0
    else:
        m0 = build_cube_mesh(8)
        m, scale = TetMesh.from_arrays(m0.vertices * 1e3 - 5e5, m0.elements), 100.0
    V, o, d = cases(gen, m, 400, scale)
    w = check(L, V, o, d)
    assert w["face"] <= 14.1, w
    assert w["y0"] <= 37.0, w
    assert w["cont32"] <= 29.3, w
