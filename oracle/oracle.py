"""ctypes front end of the CPU oracle (oracle/walk_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs import this module.

``OracleTally`` restates the reference's ``MeshTally`` facade
(tally.py:203-286) over the C restatement: ``initialize_particle_location``
(search.py:557-601), ``move_to_next_location`` (tally.py:247-271 with
particles.py:57-89 ``load_step``), ``finalize_batch`` (tally.py:83-112) and
``flux`` (tally.py:123-152).  It also returns per-particle sequence digests
and event counts for the current move (see oracle/gen_golden.py for the
digest definition).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from collections import namedtuple
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "lib" / "libwalk_oracle.so"
DIGEST_INIT = np.uint64(0xCBF29CE484222325)

Summary = namedtuple("Summary", "sweeps events reached boundary_exits "
                     "stuck_recoveries stuck_terminations")

_P = C.c_void_p


class _Particles(C.Structure):
    _fields_ = [(n, _P) for n in ("position", "destination", "weight", "group", "element",
                                  "flying", "alive", "entry_face", "stuck", "outcome",
                                  "seg_total", "digest", "count")]


def build() -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = HERE / "walk_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        L.om_bary.restype = C.c_double
        L.om_face_hit.restype = C.c_double
        L.om_trace.restype = C.c_int
        L.om_initialize.restype = C.c_int
        L.om_trace.argtypes = [_P, _P, _P, _P, C.c_int64, C.POINTER(_Particles), C.c_int64,
                               _P, C.c_int64, C.c_int32, C.c_int, C.c_int, C.c_int64, _P]
        L.om_initialize.argtypes = [_P, _P, _P, _P, C.c_int64, _P, _P,
                                    C.POINTER(_Particles), C.c_int64, C.c_int64, C.c_int, _P]
        L.om_locate_exhaustive.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, _P, C.c_int]
        L.om_finalize.argtypes = [_P, C.c_int64, C.c_int64, C.c_double, _P, _P]
        L.om_max_threads.restype = C.c_int
        L.om_philox.argtypes = [_P, _P, _P]
        L.om_uniform_block.argtypes = [C.c_uint64] * 4 + [_P]
        L.om_transport_run.restype = C.c_int
        L.om_transport_run.argtypes = (
            [_P, _P, _P, _P, C.c_int64, _P, C.c_int64, _P, _P, _P, C.c_int64, C.c_int64,
             C.c_uint64, _P, C.c_int, _P] + [_P] * 7 + [C.POINTER(_Particles), _P, _P, _P])
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def max_threads() -> int:
    return int(lib().om_max_threads())


# ----------------------------------------------------------------------------
# scalar cores (geometry KATs)

def bary(tet, p):
    tet = np.ascontiguousarray(tet, dtype=np.float64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.zeros(4)
    d = lib().om_bary(_ptr(tet), _ptr(p), _ptr(out))
    return out, d


def face_hit(face, o, s):
    face = np.ascontiguousarray(face, dtype=np.float64)
    o = np.ascontiguousarray(o, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    return lib().om_face_hit(_ptr(face), _ptr(o), _ptr(s))


def exit_search(mesh, e, o, d, entry):
    o = np.ascontiguousarray(o, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    face = C.c_int(0)
    t = C.c_double(0)
    k = lib().om_exit_search(_ptr(mesh.vertices), _ptr(mesh.elements), C.c_int64(int(e)),
                             _ptr(o), _ptr(d), C.c_int(int(entry)), C.byref(face), C.byref(t))
    return k, face.value, t.value


def locate_exhaustive(mesh, pts, threads=None):
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.empty(pts.shape[0], dtype=np.int32)
    lib().om_locate_exhaustive(_ptr(mesh.vertices), _ptr(mesh.elements),
                               C.c_int64(mesh.num_elements), _ptr(pts),
                               C.c_int64(pts.shape[0]), _ptr(out),
                               C.c_int(threads or max_threads()))
    return out


# ----------------------------------------------------------------------------

class OracleTally:
    """CPU restatement of ``MeshTally`` (tally.py:203-286)."""

    def __init__(self, mesh, num_particles: int, num_groups: int = 1, threads: int = 1):
        if num_particles <= 0:
            raise ValueError("num_particles must be positive")
        self.mesh = mesh
        self.threads = max(1, int(threads))
        n = int(num_particles)
        self.capacity = n
        self.num_groups = int(num_groups)
        self.position = np.zeros((n, 3))
        self.destination = np.zeros((n, 3))
        self.weight = np.zeros(n)
        self.group = np.zeros(n, np.int32)
        self.element = np.full(n, -1, np.int32)
        self.flying = np.zeros(n, np.int8)
        self.alive = np.zeros(n, np.int8)
        self.entry_face = np.full(n, -1, np.int8)
        self.stuck = np.zeros(n, np.int8)
        self.outcome = np.zeros(n, np.int8)
        self.seg_total = np.zeros(n)
        self.digest = np.full(n, DIGEST_INIT, np.uint64)
        self.count = np.zeros(n, np.int64)
        nb = mesh.num_elements * self.num_groups
        self.partials = np.zeros((self.threads, nb))
        self.sum = np.zeros(nb)
        self.sum_sq = np.zeros(nb)
        self.batches_completed = 0
        self.source_weight = 0.0
        self._mesh_arrays = tuple(np.ascontiguousarray(a) for a in (
            mesh.vertices, mesh.elements, mesh.adj_elem, mesh.adj_face))
        self._c0 = np.ascontiguousarray(mesh.centroids[0], dtype=np.float64)
        self._bbox = np.ascontiguousarray(mesh.bounding_box, dtype=np.float64)

    def _particles(self):
        p = _Particles()
        for name, _ in _Particles._fields_:
            setattr(p, name, getattr(self, name).ctypes.data)
        return p

    def initialize_particle_location(self, positions, threads=None):
        pos = np.asarray(positions, dtype=np.float64).reshape(-1)
        count = pos.size // 3
        if count > self.capacity:
            raise ValueError(f"count {count} exceeds capacity {self.capacity}")
        if pos.size != 3 * count:
            raise ValueError("positions must hold 3*count floats")
        self.destination[:count] = pos.reshape(count, 3)
        s = np.zeros(6, np.int64)
        v, e, ae, af = self._mesh_arrays
        P = self._particles()
        rc = lib().om_initialize(_ptr(v), _ptr(e), _ptr(ae), _ptr(af),
                                 C.c_int64(self.mesh.num_elements), _ptr(self._c0),
                                 _ptr(self._bbox), C.byref(P), C.c_int64(count),
                                 C.c_int64(self.capacity), C.c_int(threads or self.threads),
                                 _ptr(s))
        if rc != 0:
            raise RuntimeError("localization did not terminate")
        self.source_weight = 0.0
        return Summary(*s.tolist())

    def load_step(self, destinations, flying, weights):
        """particles.py:57-89 (direction is not used by the walk; skipped)."""
        fly = np.asarray(flying).reshape(-1).astype(np.int8)
        count = fly.size
        dest = np.asarray(destinations, dtype=np.float64).reshape(-1)
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        if dest.size != 3 * count or w.size != count or count > self.capacity:
            raise ValueError("array sizes do not match count")
        if count == 0:
            return 0
        self.flying[count:] = 0
        self.destination[:count] = dest.reshape(count, 3)
        self.flying[:count] = fly
        self.weight[:count] = w
        self.alive[:count] |= fly
        return count

    def move_to_next_location(self, destinations, flying, weights, groups=None,
                              max_sweeps=-1):
        count = self.load_step(destinations, flying, weights)
        if count == 0:
            return None
        if groups is not None:
            g = np.asarray(groups, dtype=np.int32).reshape(-1)
            if g.size != count:
                raise ValueError("groups size mismatch")
            self.group[:count] = g
        if self.source_weight == 0.0:
            self.source_weight = float(self.weight[:count][self.flying[:count] != 0].sum())
        return self.trace(max_sweeps=max_sweeps)

    def trace(self, score=True, max_sweeps=-1):
        self.digest[:] = DIGEST_INIT
        self.count[:] = 0
        s = np.zeros(6, np.int64)
        v, e, ae, af = self._mesh_arrays
        P = self._particles()
        rc = lib().om_trace(_ptr(v), _ptr(e), _ptr(ae), _ptr(af),
                            C.c_int64(self.mesh.num_elements), C.byref(P),
                            C.c_int64(self.capacity), _ptr(self.partials),
                            C.c_int64(self.partials.shape[0]), C.c_int32(self.num_groups),
                            C.c_int(1 if score else 0), C.c_int(self.threads),
                            C.c_int64(max_sweeps), _ptr(s))
        if rc != 0:
            raise RuntimeError("trace did not terminate within the sweep guard")
        return Summary(*s.tolist())

    def batch_totals(self):
        return self.partials.sum(axis=0)

    def finalize_batch(self, source_weight=None):
        w = self.source_weight if source_weight is None else source_weight
        if not w or w <= 0.0:
            raise RuntimeError("no source weight recorded for this batch; pass source_weight")
        lib().om_finalize(_ptr(self.partials), C.c_int64(self.partials.shape[0]),
                          C.c_int64(self.partials.shape[1]), C.c_double(w),
                          _ptr(self.sum), _ptr(self.sum_sq))
        self.batches_completed += 1
        self.source_weight = 0.0

    def flux(self):
        """tally.py:123-152."""
        n = self.batches_completed
        if n == 0:
            raise RuntimeError("no batches completed; nothing to normalize")
        shape = (self.mesh.num_elements, self.num_groups)
        s = self.sum.reshape(shape)
        sq = self.sum_sq.reshape(shape)
        bm = s / n
        mean = bm / self.mesh.volumes[:, None]
        rel = np.zeros(shape)
        if n >= 2:
            var = (sq - s * s / n) / (n - 1)
            np.clip(var, 0.0, None, out=var)
            se = np.sqrt(var / n)
            nz = bm > 0.0
            rel[nz] = se[nz] / bm[nz]
        return mean, rel


if os.environ.get("ORACLE_BUILD_ON_IMPORT"):
    build()


# ----------------------------------------------------------------------------
# transport: restatement of transport.run, serial

def philox(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    out = np.zeros(4, np.uint64)
    lib().om_philox(_ptr(c), _ptr(k), _ptr(out))
    return out


def uniform_block(seed, batch, particle, block):
    u = np.zeros(4)
    lib().om_uniform_block(C.c_uint64(seed), C.c_uint64(batch), C.c_uint64(particle),
                           C.c_uint64(block), _ptr(u))
    return u


def xs_kernel_data(sigma_t, sigma_s):
    """XSData (transport.py:83-99): scatter probability and group CDF."""
    st = np.ascontiguousarray(np.atleast_1d(sigma_t), dtype=np.float64)
    ss = np.ascontiguousarray(np.atleast_2d(sigma_s), dtype=np.float64)
    g = st.shape[0]
    rows = ss.sum(axis=1)
    prob = rows / st
    cdf = np.zeros((g, g))
    for i in range(g):
        if rows[i] > 0.0:
            cdf[i] = np.cumsum(ss[i]) / rows[i]
        cdf[i, g - 1] = 1.0
    return st, np.ascontiguousarray(prob), np.ascontiguousarray(cdf)


def transport_run(mesh, sigma_t, sigma_s, num_particles, num_batches, seed, box,
                  direction=None):
    """Returns dict with totals, flux moments and final particle state."""
    L = lib()
    st, prob, cdf = xs_kernel_data(sigma_t, sigma_s)
    ng = st.shape[0]
    n = int(num_particles)
    nb = mesh.num_elements * ng
    t = OracleTally(mesh, n, ng, threads=1)
    direction_arr = np.zeros((n, 3))
    rngb = np.zeros(n, np.uint64)
    grp = np.zeros(n, np.int32)
    tp, ts, tsq = np.zeros(nb), np.zeros(nb), np.zeros(nb)
    cp, cs, csq = np.zeros(nb), np.zeros(nb), np.zeros(nb)
    totals = np.zeros(8)
    box = np.ascontiguousarray(np.asarray(box, dtype=np.float64).reshape(6))
    fd = np.zeros(3) if direction is None else np.ascontiguousarray(direction, dtype=np.float64)
    v, e, ae, af = t._mesh_arrays
    P = t._particles()
    rc = L.om_transport_run(
        _ptr(v), _ptr(e), _ptr(ae), _ptr(af), C.c_int64(mesh.num_elements), _ptr(t._c0),
        C.c_int64(ng), _ptr(st), _ptr(prob), _ptr(cdf), C.c_int64(n), C.c_int64(num_batches),
        C.c_uint64(seed), _ptr(box), C.c_int(0 if direction is None else 1), _ptr(fd),
        _ptr(tp), _ptr(ts), _ptr(tsq), _ptr(cp), _ptr(cs), _ptr(csq), _ptr(totals),
        C.byref(P), _ptr(direction_arr), _ptr(grp), _ptr(rngb))
    if rc != 0:
        raise RuntimeError("oracle transport did not terminate")
    keys = ("source_weight", "leaked_weight", "absorbed_weight", "stuck_weight",
            "collisions", "events", "sweeps", "track_length_total")
    out = dict(zip(keys, totals.tolist()))
    out.update(track_sum=ts, track_sum_sq=tsq, col_sum=cs, col_sum_sq=csq,
               position=t.position.copy(), direction=direction_arr, element=t.element.copy(),
               group=grp, alive=t.alive.copy(), outcome=t.outcome.copy(), rng_block=rngb,
               seg_total=t.seg_total.copy())
    return out


def flux_from_moments(s, sq, n, volumes, ng):
    shape = (volumes.shape[0], ng)
    s = s.reshape(shape)
    sq = sq.reshape(shape)
    bm = s / n
    mean = bm / volumes[:, None]
    rel = np.zeros(shape)
    if n >= 2:
        var = (sq - s * s / n) / (n - 1)
        np.clip(var, 0.0, None, out=var)
        se = np.sqrt(var / n)
        nz = bm > 0.0
        rel[nz] = se[nz] / bm[nz]
    return mean, rel
