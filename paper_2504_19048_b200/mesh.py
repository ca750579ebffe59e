"""Host-side tetrahedral mesh: load, orientation fix, face adjacency.

Mirrors the reference's mesh-load API (``meshtally/mesh.py``) so a
``MeshTally`` user can switch packages without touching mesh code:

* ``TetMesh`` (mesh.py:73-107) with the same arrays and dtypes
  (``vertices (V,3) f64``, ``elements (E,4) i32``, ``adj_elem (E,4) i32``,
  ``adj_face (E,4) i8``, ``volumes``, ``centroids``, ``bounding_box``);
* ``TetMesh.from_arrays`` (mesh.py:109-148): positive orientation by swapping
  local vertices 2<->3, degeneracy rejection at ``vol6 <= 1e-12*max(span,1)^3``;
* ``build_cube_mesh`` (mesh.py:159-185): the Kuhn 6-tet split, element id
  ``6*cell + t`` with ``cell = (i*n + j)*n + k``;
* ``build_adjacency`` (mesh.py:188-235): face i is opposite local vertex i;
* ``read_tetmesh``/``write_tetmesh`` (mesh.py:302-331) text format.

Element ids and local vertex order decide ties in the walk, so they must be
exactly the reference's.  Adjacency of a conforming mesh is unique, so any
correct builder reproduces it; this one sorts one packed 64-bit key per face
(or a lexsort when the vertex count is too large to pack).

Deliberate deviation: a duplicated element (same 4 vertex ids twice) is
rejected, as the reference's docstring and its own test
(test_mesh.py:104-107) require; the reference's builder misses this case
because the two copies share every face exactly twice.

The device copy of the mesh (packed element records, padded vertices) is
built by the C-ABI library from these arrays; see DESIGN.md "Data layout".
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from pathlib import Path

import numpy as np


class MalformedMeshError(ValueError):
    """The element/vertex data does not describe a conforming tet mesh."""


# local face f (opposite local vertex f) -> the three local vertices spanning it
FACE_VERTICES = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]], dtype=np.int64)

_DEGENERATE_REL = 1e-12


def _kuhn_tets() -> np.ndarray:
    """The 6 monotone corner paths 0 -> 7 of a hex (corner bits x=4, y=2, z=1),
    one per axis order, in lexicographic order of (x, y, z) permutations.
    Every tet holds the main diagonal 0-7, so neighbouring cells split their
    shared faces the same way and the tessellation conforms."""
    out = []
    for order in itertools.permutations((4, 2, 1)):
        c, path = 0, [0]
        for bit in order:
            c |= bit
            path.append(c)
        out.append(path)
    return np.array(out, dtype=np.int64)


KUHN_TETS = _kuhn_tets()


@dataclass(frozen=True)
class TetMesh:
    """Immutable tet mesh with adjacency, volumes, centroids and bbox."""

    vertices: np.ndarray       # (V, 3) float64
    elements: np.ndarray       # (E, 4) int32
    adj_elem: np.ndarray       # (E, 4) int32, -1 on the boundary
    adj_face: np.ndarray       # (E, 4) int8, -1 on the boundary
    volumes: np.ndarray        # (E,) float64
    centroids: np.ndarray      # (E, 3) float64
    bounding_box: np.ndarray   # (2, 3) float64

    @property
    def num_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def num_elements(self) -> int:
        return int(self.elements.shape[0])

    @property
    def face_adjacency(self) -> np.ndarray:
        return np.stack([self.adj_elem, self.adj_face.astype(np.int32)], axis=2)

    @classmethod
    def from_arrays(cls, vertices, elements, device: int | str | None = "auto") -> "TetMesh":
        """Orientation fix, degeneracy check, adjacency.

        ``device="auto"`` (default): the library's native ingest
        (bt_mesh_from_arrays: all host threads, adjacency on GPU 0 when one is
        visible, else a host sort); an int: the same on that GPU; ``None``:
        the host numpy path.  All three give bit-identical arrays."""
        if device is not None:
            return _native_from_arrays(vertices, elements, device)
        return cls._from_arrays_numpy(vertices, elements)

    @classmethod
    def _from_arrays_numpy(cls, vertices, elements) -> "TetMesh":
        vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        elements = np.array(elements, dtype=np.int32, copy=True, order="C")
        if vertices.ndim != 2 or vertices.shape[1] != 3:
            raise MalformedMeshError("vertices must be (V, 3)")
        if elements.ndim != 2 or elements.shape[1] != 4:
            raise MalformedMeshError("elements must be (E, 4)")
        nv = vertices.shape[0]
        if elements.size and (int(elements.min()) < 0 or int(elements.max()) >= nv):
            raise MalformedMeshError("element vertex id out of range")

        vol6 = signed_volumes6(vertices, elements)
        flip = vol6 < 0.0
        if flip.any():
            elements[flip, 2:4] = elements[flip, 3:1:-1]
            vol6 = np.abs(vol6)
        if vertices.size:
            span = float((vertices.max(axis=0) - vertices.min(axis=0)).max())
        else:
            span = 1.0
        limit = _DEGENERATE_REL * max(span, 1.0) ** 3
        if elements.shape[0] and (vol6 <= limit).any():
            bad = int(np.argmin(vol6))
            raise MalformedMeshError(
                f"element {bad} is degenerate (volume {vol6[bad] / 6.0:g})")

        adj_elem, adj_face = build_adjacency(elements, nv)
        centroids = vertices[elements].mean(axis=1)
        if vertices.size:
            bbox = np.stack([vertices.min(axis=0), vertices.max(axis=0)])
        else:
            bbox = np.zeros((2, 3))
        return cls(vertices, elements, adj_elem, adj_face,
                   np.ascontiguousarray(vol6 / 6.0),
                   np.ascontiguousarray(centroids),
                   np.ascontiguousarray(bbox))


def _native_device(device) -> int:
    from . import _lib
    if device == "auto":
        return 0 if _lib.device_count() > 0 else -1
    return int(device)


def _native_mesh(h, L) -> TetMesh:
    """Copy a bt_mesh's arrays into a TetMesh and release it."""
    import ctypes as C
    from . import _lib
    try:
        nv, ne = C.c_int64(), C.c_int64()
        _lib.check(L.bt_mesh_info(h, C.byref(nv), C.byref(ne)))
        nv, ne = int(nv.value), int(ne.value)
        v = np.empty((nv, 3))
        e = np.empty((ne, 4), np.int32)
        ae = np.empty((ne, 4), np.int32)
        af = np.empty((ne, 4), np.int8)
        vol = np.empty(ne)
        cen = np.empty((ne, 3))
        bbox = np.empty((2, 3))
        _lib.check(L.bt_mesh_arrays(h, v.ctypes.data, e.ctypes.data, ae.ctypes.data,
                                    af.ctypes.data, vol.ctypes.data, cen.ctypes.data,
                                    bbox.ctypes.data))
    finally:
        L.bt_mesh_destroy(h)
    return TetMesh(v, e, ae, af, vol, cen, bbox)


def _native_call(fn, *args) -> TetMesh:
    import ctypes as C
    from . import _lib
    L = _lib.load()
    h = C.c_void_p()
    st = getattr(L, fn)(*args, C.byref(h))
    if st == _lib.BT_EINVAL:
        raise MalformedMeshError(L.bt_last_error().decode())
    _lib.check(st)
    return _native_mesh(h, L)


def _native_from_arrays(vertices, elements, device) -> TetMesh:
    vertices = np.ascontiguousarray(vertices, dtype=np.float64)
    elements = np.ascontiguousarray(elements, dtype=np.int32)
    if vertices.ndim != 2 or vertices.shape[1] != 3:
        raise MalformedMeshError("vertices must be (V, 3)")
    if elements.ndim != 2 or elements.shape[1] != 4:
        raise MalformedMeshError("elements must be (E, 4)")
    return _native_call("bt_mesh_from_arrays", vertices.ctypes.data, vertices.shape[0],
                        elements.ctypes.data, elements.shape[0], _native_device(device))


def signed_volumes6(vertices: np.ndarray, elements: np.ndarray) -> np.ndarray:
    """6x signed volume: (v1-v0) x (v2-v0) . (v3-v0)."""
    p = vertices[elements]                      # (E, 4, 3)
    a = p[:, 1] - p[:, 0]
    b = p[:, 2] - p[:, 0]
    c = p[:, 3] - p[:, 0]
    return np.einsum("ij,ij->i", np.cross(a, b), c)


def build_cube_mesh(n: int, edge_length: float = 1.0, device: int | str | None = "auto") -> TetMesh:
    """[0, edge_length]^3 split into n^3 hex cells of 6 Kuhn tets each."""
    if not isinstance(n, (int, np.integer)) or isinstance(n, bool) or n < 1:
        raise ValueError(f"subdivisions must be a positive integer, got {n!r}")
    if not edge_length > 0.0:
        raise ValueError(f"edge_length must be positive, got {edge_length!r}")
    n = int(n)
    nv = n + 1
    h = edge_length / n
    coord = np.arange(nv, dtype=np.float64) * h
    coord[-1] = edge_length  # far face exactly on edge_length
    # vertex (i, j, k) -> id (i*nv + j)*nv + k at (coord[i], coord[j], coord[k])
    vid = np.arange(nv ** 3, dtype=np.int64)
    vi, vj, vk = vid // (nv * nv), (vid // nv) % nv, vid % nv
    vertices = np.stack([coord[vi], coord[vj], coord[vk]], axis=1)

    cell = np.arange(n ** 3, dtype=np.int64)
    ci, cj, ck = cell // (n * n), (cell // n) % n, cell % n
    base = (ci * nv + cj) * nv + ck
    # corner bit b = (x<<2)|(y<<1)|z -> vertex id offset
    offs = np.array([((b >> 2) & 1) * nv * nv + ((b >> 1) & 1) * nv + (b & 1)
                     for b in range(8)], dtype=np.int64)
    elements = base[:, None, None] + offs[KUHN_TETS][None, :, :]   # (cells, 6, 4)
    return TetMesh.from_arrays(vertices, elements.reshape(-1, 4), device=device)


def build_torus_shell_mesh(nr: int, ntheta: int, nphi: int, R: float = 300.0,
                           a_in: float = 100.0, a_out: float = 120.0,
                           device: int | str | None = "auto") -> TetMesh:
    """Toroidal-shell mesh; see torus_shell_arrays."""
    return TetMesh.from_arrays(*torus_shell_arrays(nr, ntheta, nphi, R, a_in, a_out),
                               device=device)


def torus_shell_arrays(nr: int, ntheta: int, nphi: int, R: float = 300.0,
                       a_in: float = 100.0, a_out: float = 120.0):
    """Raw (vertices, elements) of a structured (r, theta, phi) toroidal shell, Kuhn-split in index space
    with periodic wrap in theta and phi.

    Corner b of cell (i, j, k) is vertex
    ``(i+b2)*nth*nph + ((j+b1) mod nth)*nph + ((k+b0) mod nph)``.
    """
    for name, v in (("nr", nr), ("ntheta", ntheta), ("nphi", nphi)):
        if int(v) < 1:
            raise ValueError(f"{name} must be positive")
    if ntheta < 3 or nphi < 3:
        raise ValueError("ntheta and nphi must be >= 3 for a conforming wrap")
    nr1 = nr + 1
    r = a_in + (a_out - a_in) * np.arange(nr1, dtype=np.float64) / nr
    th = 2.0 * np.pi * np.arange(ntheta, dtype=np.float64) / ntheta
    ph = 2.0 * np.pi * np.arange(nphi, dtype=np.float64) / nphi
    ri, tj, pk = np.meshgrid(r, th, ph, indexing="ij")
    rr = R + ri * np.cos(tj)
    vertices = np.stack([(rr * np.cos(pk)).ravel(), (rr * np.sin(pk)).ravel(),
                         (ri * np.sin(tj)).ravel()], axis=1)
    cell = np.arange(nr * ntheta * nphi, dtype=np.int64)
    ci, cj, ck = cell // (ntheta * nphi), (cell // nphi) % ntheta, cell % nphi
    corners = np.empty((cell.size, 8), dtype=np.int64)
    for b in range(8):
        corners[:, b] = ((ci + ((b >> 2) & 1)) * ntheta * nphi
                         + ((cj + ((b >> 1) & 1)) % ntheta) * nphi
                         + ((ck + (b & 1)) % nphi))
    elements = corners[:, KUHN_TETS].reshape(-1, 4)
    return vertices, elements


def _face_keys(elements: np.ndarray, nv: int):
    """Sorted vertex triple of every (element, local face), row = 4*e + f."""
    tri = elements[:, FACE_VERTICES].astype(np.int64)   # (E, 4, 3)
    tri.sort(axis=2)
    return tri.reshape(-1, 3)


def build_adjacency(elements, vertex_count: int, device: int | None = None):
    """(adj_elem, adj_face), both (E, 4), -1 on the boundary.

    Raises MalformedMeshError for a face shared by 3+ elements, an element
    listing one face twice, or a duplicated element.  With `device`, the
    sort runs on that GPU (bt_build_adjacency); the result is identical
    (adjacency of a conforming mesh is unique).
    """
    elements = np.ascontiguousarray(elements, dtype=np.int32)
    ne = elements.shape[0]
    adj_elem = np.full((ne, 4), -1, dtype=np.int32)
    adj_face = np.full((ne, 4), -1, dtype=np.int8)
    if ne == 0:
        return adj_elem, adj_face
    if device is not None:
        from . import _lib
        L = _lib.load()
        st = L.bt_build_adjacency(elements.ctypes.data, ne, int(vertex_count), int(device),
                                  adj_elem.ctypes.data, adj_face.ctypes.data)
        if st == _lib.BT_EINVAL:
            raise MalformedMeshError(L.bt_last_error().decode())
        _lib.check(st)
        return adj_elem, adj_face
    if int(elements.min()) < 0 or int(elements.max()) >= vertex_count:
        raise MalformedMeshError("element vertex id out of range")

    tri = _face_keys(elements, vertex_count)
    nv = max(int(vertex_count), 1)
    if nv < (1 << 21):
        key = (tri[:, 0] << 42) | (tri[:, 1] << 21) | tri[:, 2]
        order = np.argsort(key, kind="stable")
        ks = key[order]
        same = ks[1:] == ks[:-1]
    else:
        order = np.lexsort((tri[:, 2], tri[:, 1], tri[:, 0]))
        ts = tri[order]
        same = (ts[1:] == ts[:-1]).all(axis=1)

    if (same[1:] & same[:-1]).any():
        i = int(np.nonzero(same[1:] & same[:-1])[0][0])
        key3 = tuple(int(v) for v in tri[order[i]])
        raise MalformedMeshError(
            f"face with vertices {key3} is shared by more than two elements "
            "(duplicate or non-manifold mesh)")

    first = order[:-1][same]
    second = order[1:][same]
    e1, f1 = first // 4, first % 4
    e2, f2 = second // 4, second % 4
    if (e1 == e2).any():
        bad = int(e1[np.nonzero(e1 == e2)[0][0]])
        raise MalformedMeshError(
            f"element {bad} lists the same face twice (repeated vertex id)")
    adj_elem[e1, f1] = e2
    adj_face[e1, f1] = f2
    adj_elem[e2, f2] = e1
    adj_face[e2, f2] = f1

    # duplicated element: all four faces shared with one and the same element
    full = (adj_elem >= 0).all(axis=1)
    if full.any():
        rows = adj_elem[full]
        dup = (rows == rows[:, :1]).all(axis=1)
        if dup.any():
            bad = int(np.nonzero(full)[0][np.nonzero(dup)[0][0]])
            raise MalformedMeshError(
                f"element {bad} duplicates element {int(adj_elem[bad, 0])}")
    return adj_elem, adj_face


def element_volume(mesh: TetMesh, elem: int) -> float:
    if not 0 <= elem < mesh.num_elements:
        raise IndexError(f"element id {elem} out of range [0, {mesh.num_elements})")
    v = mesh.vertices[mesh.elements[elem]]
    return abs(float(np.linalg.det(v[1:] - v[0]))) / 6.0


def validate(mesh: TetMesh) -> list[str]:
    """Diagnostics for the mesh invariants; empty iff valid."""
    report: list[str] = []
    vol6 = signed_volumes6(mesh.vertices, mesh.elements)
    for e in np.nonzero(vol6 <= 0.0)[0][:10]:
        report.append(f"element {int(e)}: non-positive volume {vol6[e] / 6.0:g}")
    ne = mesh.num_elements
    ae, af = mesh.adj_elem, mesh.adj_face
    e_idx, f_idx = np.nonzero(ae >= 0)
    nb = ae[e_idx, f_idx].astype(np.int64)
    nf = af[e_idx, f_idx].astype(np.int64)
    bad_nb = (nb < 0) | (nb >= ne)
    bad_nf = (nf < 0) | (nf >= 4)
    for k in np.nonzero(bad_nb)[0][:10]:
        report.append(f"element {int(e_idx[k])} face {int(f_idx[k])}: neighbor id "
                      f"{int(nb[k])} out of range")
    for k in np.nonzero(bad_nf & ~bad_nb)[0][:10]:
        report.append(f"element {int(e_idx[k])} face {int(f_idx[k])}: neighbor face "
                      f"id {int(nf[k])} out of range")
    ok = ~(bad_nb | bad_nf)
    e_idx, f_idx, nb, nf = e_idx[ok], f_idx[ok], nb[ok], nf[ok]
    back_e = ae[nb, nf]
    back_f = af[nb, nf]
    asym = (back_e != e_idx) | (back_f != f_idx)
    for k in np.nonzero(asym)[0][:10]:
        report.append(f"element {int(e_idx[k])} face {int(f_idx[k])}: asymmetric "
                      f"adjacency (neighbor {int(nb[k])} face {int(nf[k])})")
    mine = np.sort(mesh.elements[e_idx[:, None], FACE_VERTICES[f_idx]], axis=1)
    theirs = np.sort(mesh.elements[nb[:, None], FACE_VERTICES[nf]], axis=1)
    mism = (mine != theirs).any(axis=1)
    for k in np.nonzero(mism)[0][:10]:
        report.append(f"element {int(e_idx[k])} face {int(f_idx[k])}: adjacency "
                      f"pairs mismatched vertex sets")
    try:
        ref_e, ref_f = build_adjacency(mesh.elements, mesh.num_vertices)
    except MalformedMeshError as err:
        report.append(str(err))
    else:
        if not (np.array_equal(ref_e, ae) and np.array_equal(ref_f, af)):
            bad = np.argwhere(ref_e != ae)
            if bad.size:
                e, f = (int(x) for x in bad[0])
                report.append(f"element {e} face {f}: stored adjacency disagrees "
                              f"with connectivity (stored {ae[e, f]}, derived "
                              f"{ref_e[e, f]})")
    return report


def write_tetmesh(mesh: TetMesh, path) -> None:
    """Text format: ``tetmesh <nv> <ne>``, nv vertex lines, ne element lines."""
    with open(path, "w") as fh:
        fh.write(f"tetmesh {mesh.num_vertices} {mesh.num_elements}\n")
        for x, y, z in mesh.vertices.tolist():
            fh.write(f"{x!r} {y!r} {z!r}\n")
        for a, b, c, d in mesh.elements.tolist():
            fh.write(f"{a} {b} {c} {d}\n")


def read_tetmesh(path, device: int | str | None = "auto") -> TetMesh:
    """read_tetmesh (mesh.py:312-331).  ``device`` as in
    ``TetMesh.from_arrays``: the native reader (bt_mesh_read, parsed on all
    host threads) unless ``None`` (the host Python parser + numpy path)."""
    if device is not None:
        return _native_call("bt_mesh_read", str(path).encode(), _native_device(device))
    path = Path(path)
    with open(path) as fh:
        header = fh.readline().split()
        if len(header) != 3 or header[0] != "tetmesh":
            raise MalformedMeshError(
                f"{path}: expected header 'tetmesh <nverts> <nelems>'")
        try:
            nv, ne = int(header[1]), int(header[2])
        except ValueError as err:
            raise MalformedMeshError(f"{path}: bad header counts") from err
        if nv < 0 or ne < 0:
            raise MalformedMeshError(f"{path}: bad header counts")
        try:
            vlines = [fh.readline() for _ in range(nv)]
            elines = [fh.readline() for _ in range(ne)]
            vertices = np.array([[float(t) for t in ln.split()] for ln in vlines],
                                dtype=np.float64).reshape(nv, -1) if nv else np.zeros((0, 3))
            elements = np.array([[int(t) for t in ln.split()] for ln in elines],
                                dtype=np.int64).reshape(ne, -1) if ne else np.zeros((0, 4), np.int64)
        except ValueError as err:
            raise MalformedMeshError(f"{path}: {err}") from err
    if vertices.shape != (nv, 3) or elements.shape != (ne, 4):
        raise MalformedMeshError(f"{path}: body does not match header counts")
    return TetMesh.from_arrays(vertices, elements, device=None)
