"""Drop-in ``MeshTally`` facade over the CUDA library (C ABI, ctypes).

Mirrors the reference's tally API (meshtally/tally.py):

* ``MeshTally(mesh, num_particles, num_groups=1, threads=1)`` -- tally.py:211-229
* ``.initialize_particle_location(positions)``                 -- tally.py:239-245
* ``.move_to_next_location(destinations, flying, weights, groups=None)``
  -> ``TraceSummary | None``                                    -- tally.py:247-271
* ``.finalize_batch(source_weight=None)``                       -- tally.py:273-279
* ``.flux() -> FluxResult``, ``.write(filename)``, ``.mesh``, ``.grid``
* module functions ``batch_totals``, ``finalize_batch``, ``flux`` over a grid
  view (tally.py:101-152) and the VTK/CSV writers (tally.py:159-200).

Arguments accept host arrays (anything ``numpy.asarray`` takes, converted
exactly as the reference converts them) or CUDA tensors that expose
``data_ptr()`` and live on the handle's GPU (zero-copy).

Documented deviations from the reference:

* ``threads`` is accepted and ignored (there are no CPU slabs; the
  reference's slab/thread mismatch bug, cannot occur).
* ``groups`` values outside ``[0, num_groups)`` raise ``IndexError`` instead
  of silently scoring into another element's bin (tally.py:262-266).
* A flying particle with ``element == -1`` is not moved and the call raises
  ``ValueError`` after moving the others (the reference's fused path reads
  element -1 with numba wraparound; its callback path raises up front).
* Localization defaults to the grid search (``localize="grid"``): it returns
  the lowest-id element containing the point (pkg/tests/oracles.py:36-57),
  which equals the reference's centroid-0 walk + tie-break on every generic
  point and also finds the points that walk loses.
  ``localize="walk"`` reproduces the reference bit for bit, losses included.
"""

from __future__ import annotations

import atexit
import ctypes as C
import weakref
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .mesh import TetMesh, read_tetmesh

OUTCOME_NONE, OUTCOME_REACHED, OUTCOME_LEAKED, OUTCOME_STUCK_KILLED = 0, 1, 2, 3


@dataclass(frozen=True)
class TraceSummary:
    """search.py:150-157."""

    sweeps: int
    events: int
    reached: int
    boundary_exits: int
    stuck_recoveries: int
    stuck_terminations: int

    @classmethod
    def _from(cls, s: _lib.Summary) -> "TraceSummary":
        return cls(int(s.sweeps), int(s.events), int(s.reached), int(s.boundary_exits),
                   int(s.stuck_recoveries), int(s.stuck_terminations))


@dataclass(frozen=True)
class FluxResult:
    """tally.py:115-120."""

    mean: np.ndarray       # (E, G)
    rel_error: np.ndarray  # (E, G)


@dataclass(frozen=True)
class ParticleState:
    position: np.ndarray
    element: np.ndarray
    alive: np.ndarray
    entry_face: np.ndarray
    stuck: np.ndarray
    outcome: np.ndarray
    seg_total: np.ndarray


def _is_device(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


def _producer_sync(t) -> None:
    """The library runs on its own stream: wait for the producer stream of a
    CUDA tensor argument (torch's current stream on its device) first."""
    import torch
    torch.cuda.current_stream(t.device).synchronize()


class _LiveArray:
    """A device tally array seen from the host: every read returns the current
    device contents (``np.asarray(a)``, ``a[i]``, ``a.sum()`` ...), every item
    assignment writes through (``a[i] = x``, ``a[:] = 0``) -- the live,
    writable arrays of the reference's jitclass grid (tally.py:21-44)."""

    def __init__(self, grid: "TallyGrid", which: int, shape):
        self._grid = grid
        self._which = which
        self.shape = tuple(shape)
        self.dtype = np.dtype(np.float64)
        self.ndim = len(self.shape)
        self.size = int(np.prod(self.shape))

    def _read(self) -> np.ndarray:
        return self._grid._read(self._which).reshape(self.shape)

    def __array__(self, dtype=None, copy=None):
        a = self._read()
        return a if dtype is None else a.astype(dtype)

    def __len__(self) -> int:
        return self.shape[0]

    def __getitem__(self, idx):
        return self._read()[idx]

    def __setitem__(self, idx, value):
        a = self._read()
        a[idx] = value
        self._grid._write(self._which, a.reshape(-1))

    def __iter__(self):
        return iter(self._read())

    def __getattr__(self, name):  # sum, max, reshape, copy, tolist, ...
        return getattr(self._read(), name)

    def __repr__(self) -> str:
        return f"_LiveArray({self._read()!r})"


class TallyGrid:
    """The device tally of a MeshTally (or of ``create_grid``) with the
    reference grid's fields (tally.py:21-44): ``partials`` (1, E*G) -- the
    unfinalized batch, one slab --, ``batch_accum`` (vestigial in the
    reference too: always zero), ``sum``, ``sum_sq``, ``batches_completed``.
    The arrays are live views of the device memory (read on access, written
    through on assignment)."""

    def __init__(self, owner):
        self._owner = owner
        self.num_elements = owner.num_elements
        self.num_groups = owner.num_groups
        nb = self.num_elements * self.num_groups
        self._partials = _LiveArray(self, _lib.BT_TALLY_BATCH, (1, nb))
        self._sum = _LiveArray(self, _lib.BT_TALLY_SUM, (nb,))
        self._sum_sq = _LiveArray(self, _lib.BT_TALLY_SUM_SQ, (nb,))

    def _read(self, which):
        return self._owner._read_tally(which)

    def _write(self, which, a):
        self._owner._write_tally(which, a)

    @property
    def partials(self) -> _LiveArray:
        return self._partials

    @property
    def batch_accum(self) -> np.ndarray:
        return np.zeros(self.num_elements * self.num_groups)

    @property
    def sum(self) -> _LiveArray:
        return self._sum

    @sum.setter
    def sum(self, v):
        self._sum[:] = v

    @property
    def sum_sq(self) -> _LiveArray:
        return self._sum_sq

    @sum_sq.setter
    def sum_sq(self, v):
        self._sum_sq[:] = v

    @property
    def batches_completed(self) -> int:
        return self._owner.batches_completed

    @batches_completed.setter
    def batches_completed(self, n: int) -> None:
        _lib.check(self._owner._L.bt_set_batches_completed(self._owner._h, int(n)))


class _GridHandle:
    """A tally-only device handle (bt_create_grid) behind ``create_grid``."""

    def __init__(self, num_elements: int, num_groups: int, device: int):
        self._L = _lib.load()
        self.num_elements = int(num_elements)
        self.num_groups = int(num_groups)
        self._h = C.c_void_p()
        _lib.check(self._L.bt_create_grid(self.num_elements, self.num_groups, int(device),
                                          C.byref(self._h)))
        _LIVE.add(self)

    @property
    def batches_completed(self) -> int:
        n = C.c_int64()
        _lib.check(self._L.bt_batches_completed(self._h, C.byref(n)))
        return int(n.value)

    def finalize_batch(self, w: float) -> None:
        _lib.check(self._L.bt_finalize_batch(self._h, float(w)))

    def _read_tally(self, which) -> np.ndarray:
        n = self.num_elements * self.num_groups
        out = np.empty(n)
        _lib.check(self._L.bt_read_tally(self._h, which, out.ctypes.data, n))
        return out

    def _write_tally(self, which, a) -> None:
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        _lib.check(self._L.bt_write_tally(self._h, which, a.ctypes.data, a.size))

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.bt_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def create_grid(num_elements: int, num_groups: int, max_threads: int = 1, *,
                device: int = 0) -> TallyGrid:
    """tally.py:47-55: a zeroed element x group grid, allocated once (on the
    GPU; ``max_threads`` is accepted -- one device tally replaces the
    per-thread slabs)."""
    if num_elements <= 0 or num_groups <= 0:
        raise ValueError(f"grid sizes must be positive, got ({num_elements}, {num_groups})")
    if max_threads < 1:
        raise ValueError(f"max_threads must be >= 1, got {max_threads}")
    return TallyGrid(_GridHandle(num_elements, num_groups, device))


def _score(grid: TallyGrid, kind: int, element, group, weight, value) -> None:
    e = np.ascontiguousarray(np.atleast_1d(element), dtype=np.int64)
    g = np.ascontiguousarray(np.atleast_1d(group), dtype=np.int64)
    w = np.ascontiguousarray(np.atleast_1d(weight), dtype=np.float64)
    x = np.ascontiguousarray(np.atleast_1d(value), dtype=np.float64)
    e, g, w, x = np.broadcast_arrays(e, g, w, x)
    # _check_bin (tally.py:58-64) / the sigma_t check, before anything lands
    if kind == 1 and not (x > 0.0).all():
        raise ValueError(f"sigma_t must be positive, got {float(x[~(x > 0.0)][0])!r}")
    bad = (e < 0) | (e >= grid.num_elements)
    if bad.any():
        raise IndexError(f"element {int(e[bad][0])} out of range [0, {grid.num_elements})")
    bad = (g < 0) | (g >= grid.num_groups)
    if bad.any():
        raise IndexError(f"group {int(g[bad][0])} out of range [0, {grid.num_groups})")
    e32 = np.ascontiguousarray(e, dtype=np.int32)
    g32 = np.ascontiguousarray(g, dtype=np.int32)
    w = np.ascontiguousarray(w)
    x = np.ascontiguousarray(x)
    o = grid._owner
    _lib.check(o._L.bt_score(o._h, kind, e32.ctypes.data, g32.ctypes.data, w.ctypes.data,
                             x.ctypes.data, e32.size, _lib.BT_MEM_HOST))


def score_track_length(grid: TallyGrid, element, group, weight, length) -> None:
    """tally.py:67-71: batch tally[element, group] += weight * length
    (scalars as the reference, or equal-length arrays of events)."""
    _score(grid, 0, element, group, weight, length)


def score_collision(grid: TallyGrid, element, group, weight, sigma_t) -> None:
    """tally.py:74-80: batch tally[element, group] += weight / sigma_t."""
    _score(grid, 1, element, group, weight, sigma_t)


def batch_totals(grid: TallyGrid) -> np.ndarray:
    """tally.py:101-104."""
    return grid.partials.sum(axis=0).reshape(grid.num_elements, grid.num_groups)


def finalize_batch(grid: TallyGrid, batch_source_weight: float) -> None:
    """tally.py:107-112."""
    if not batch_source_weight > 0.0:
        raise ValueError(
            f"batch_source_weight must be positive, got {batch_source_weight!r}")
    grid._owner.finalize_batch(float(batch_source_weight))


def flux(grid: TallyGrid, volumes) -> FluxResult:
    """tally.py:123-152 (same formula, evaluated on the read-back moments)."""
    n = grid.batches_completed
    if n == 0:
        raise RuntimeError("no batches completed; nothing to normalize")
    volumes = np.asarray(volumes, dtype=np.float64)
    if volumes.shape != (grid.num_elements,):
        raise ValueError(f"volumes must be ({grid.num_elements},), got {volumes.shape}")
    if not (volumes > 0.0).all():
        raise ValueError("volumes must be positive")
    shape = (grid.num_elements, grid.num_groups)
    s = grid.sum.reshape(shape)
    sq = grid.sum_sq.reshape(shape)
    batch_mean = s / n
    mean = batch_mean / volumes[:, None]
    rel = np.zeros(shape)
    if n >= 2:
        var = (sq - s * s / n) / (n - 1)
        np.clip(var, 0.0, None, out=var)
        se = np.sqrt(var / n)
        nz = batch_mean > 0.0
        rel[nz] = se[nz] / batch_mean[nz]
    return FluxResult(mean=mean, rel_error=rel)


def _fmt(v: float) -> str:
    return repr(float(v))


def write_vtk(mesh, flux_result: FluxResult, filename) -> None:
    """Legacy ASCII VTK unstructured grid, one flux and one rel_error cell
    field per group (tally.py:159-189 file layout)."""
    mean = np.atleast_2d(flux_result.mean)
    rel = np.atleast_2d(flux_result.rel_error)
    if mean.shape[0] != mesh.num_elements:
        raise ValueError(f"flux has {mean.shape[0]} elements, mesh has {mesh.num_elements}")
    ne, nv = mesh.num_elements, mesh.num_vertices
    with open(filename, "w") as fh:
        fh.write("# vtk DataFile Version 3.0\ntetrahedral mesh flux tally\nASCII\n"
                 "DATASET UNSTRUCTURED_GRID\n")
        fh.write(f"POINTS {nv} double\n")
        fh.writelines(f"{_fmt(x)} {_fmt(y)} {_fmt(z)}\n" for x, y, z in mesh.vertices.tolist())
        fh.write(f"CELLS {ne} {5 * ne}\n")
        fh.writelines(f"4 {a} {b} {c} {d}\n" for a, b, c, d in mesh.elements.tolist())
        fh.write(f"CELL_TYPES {ne}\n")
        fh.write("10\n" * ne)
        fh.write(f"CELL_DATA {ne}\n")
        for g in range(mean.shape[1]):
            fh.write(f"SCALARS flux_g{g} double 1\nLOOKUP_TABLE default\n")
            fh.writelines(_fmt(x) + "\n" for x in mean[:, g].tolist())
            fh.write(f"SCALARS rel_error_g{g} double 1\nLOOKUP_TABLE default\n")
            fh.writelines(_fmt(x) + "\n" for x in rel[:, g].tolist())


def write_flux_csv(flux_result: FluxResult, filename) -> None:
    """tally.py:192-200 row layout."""
    mean = np.atleast_2d(flux_result.mean)
    rel = np.atleast_2d(flux_result.rel_error)
    with open(filename, "w") as fh:
        fh.write("element,group,mean,rel_error\n")
        for e in range(mean.shape[0]):
            for g in range(mean.shape[1]):
                fh.write(f"{e},{g},{_fmt(mean[e, g])},{_fmt(rel[e, g])}\n")


_LIVE = weakref.WeakSet()


@atexit.register
def _close_all() -> None:
    """Release device memory of handles still alive at interpreter exit."""
    for mt in list(_LIVE):
        mt.close()


class MeshTally:
    """Batched track-length tally on a tet mesh, computed on one B200."""

    def __init__(self, mesh, num_particles: int, num_groups: int = 1, threads: int = 1, *,
                 device: int = 0, devices=None, localize: str = "grid", digest: bool = False,
                 sort: bool = False, warp_aggregate: bool | None = None, staged: bool | int = True,
                 move_chunks: int = 0, stream_move: bool = True):
        if isinstance(mesh, (str, Path)):
            mesh = read_tetmesh(mesh)
        if not all(hasattr(mesh, a) for a in ("vertices", "elements", "adj_elem", "adj_face",
                                              "volumes", "centroids", "bounding_box")):
            raise TypeError("mesh must be a TetMesh or a path to one")
        if int(num_particles) <= 0:
            raise ValueError("num_particles must be positive")
        if int(num_groups) <= 0:
            raise ValueError(f"grid sizes must be positive, got ({mesh.num_elements}, "
                             f"{num_groups})")
        if localize not in ("grid", "walk"):
            raise ValueError("localize must be 'grid' or 'walk'")
        self._mesh = mesh
        self.threads = max(1, int(threads))  # accepted for API compatibility
        self.num_groups = int(num_groups)
        self.capacity = int(num_particles)
        # devices=[d0, d1, ...]: one handle over several GPUs of this process
        # (bt_create_multi: contiguous particle shards, replicated mesh, one
        # NCCL all-reduce of the tallies per batch)
        self.devices = None if devices is None else [int(d) for d in devices]
        if self.devices is not None and not self.devices:
            raise ValueError("devices must name at least one GPU")
        self.device = self.devices[0] if self.devices else int(device)
        self.localize = localize
        self._count = 0
        L = _lib.load()
        v = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        e = np.ascontiguousarray(mesh.elements, dtype=np.int32)
        ae = np.ascontiguousarray(mesh.adj_elem, dtype=np.int32)
        af = np.ascontiguousarray(mesh.adj_face, dtype=np.int8)
        bbox = np.ascontiguousarray(mesh.bounding_box, dtype=np.float64)
        c0 = np.ascontiguousarray(mesh.centroids[0], dtype=np.float64)
        h = C.c_void_p()
        if self.devices is None:
            _lib.check(L.bt_create(v.ctypes.data, v.shape[0], e.ctypes.data, ae.ctypes.data,
                                   af.ctypes.data, e.shape[0], bbox.ctypes.data, c0.ctypes.data,
                                   self.capacity, self.num_groups, self.device, C.byref(h)))
        else:
            dv = np.ascontiguousarray(self.devices, dtype=np.int32)
            _lib.check(L.bt_create_multi(v.ctypes.data, v.shape[0], e.ctypes.data,
                                         ae.ctypes.data, af.ctypes.data, e.shape[0],
                                         bbox.ctypes.data, c0.ctypes.data, self.capacity,
                                         self.num_groups, dv.ctypes.data, dv.size, C.byref(h)))
        self._h = h
        self._L = L
        _LIVE.add(self)
        self.set_option(_lib.BT_OPT_DIGEST, int(digest))
        self.set_option(_lib.BT_OPT_SORT, int(sort))
        # None: adaptive (aggregate while a warp's lanes score the same bins)
        self.set_option(_lib.BT_OPT_WARP_AGG,
                        0 if warp_aggregate is None else (1 if warp_aggregate else 2))
        # staged: True -> the library's default refill, False -> v1, 1 / 2 -> stage
        # kernel / direct refill explicitly
        if staged is not True:
            self.set_option(_lib.BT_OPT_STAGED, int(staged))
        self.set_option(_lib.BT_OPT_MOVE_CHUNKS, int(move_chunks))
        self.set_option(_lib.BT_OPT_STREAM_MOVE, int(stream_move))
        self._grid = TallyGrid(self)

    # ------------------------------------------------------------------ props
    @property
    def mesh(self) -> TetMesh:
        return self._mesh

    @property
    def grid(self) -> TallyGrid:
        return self._grid

    @property
    def batches_completed(self) -> int:
        n = C.c_int64()
        _lib.check(self._L.bt_batches_completed(self._h, C.byref(n)))
        return int(n.value)

    @property
    def source_weight(self) -> float:
        w = C.c_double()
        _lib.check(self._L.bt_get_source_weight(self._h, C.byref(w)))
        return float(w.value)

    @source_weight.setter
    def source_weight(self, w: float) -> None:
        _lib.check(self._L.bt_set_source_weight(self._h, float(w)))

    @property
    def num_shards(self) -> int:
        n = C.c_int32()
        _lib.check(self._L.bt_num_shards(self._h, C.byref(n)))
        return int(n.value)

    def shard_bounds(self, index: int) -> tuple[int, int]:
        """Particle range [lo, hi) of GPU shard `index`."""
        lo, hi = C.c_int64(), C.c_int64()
        _lib.check(self._L.bt_shard(self._h, int(index), None, C.byref(lo), C.byref(hi)))
        return int(lo.value), int(hi.value)

    def set_option(self, key: int, value: int) -> None:
        _lib.check(self._L.bt_set_option(self._h, int(key), int(value)))

    # ------------------------------------------------------------------ API
    def initialize_particle_location(self, positions, *, mode: str | None = None) -> None:
        """tally.py:239-245; `mode` overrides the constructor's `localize`."""
        mode = self.localize if mode is None else mode
        m = _lib.BT_LOCATE_WALK if mode == "walk" else _lib.BT_LOCATE_GRID
        s = _lib.Summary()
        if _is_device(positions):
            self._check_tensor(positions, 8)
            _producer_sync(positions)
            size = positions.numel()
            _lib.check(self._L.bt_initialize_particle_location(
                self._h, positions.data_ptr(), size, _lib.BT_MEM_DEVICE, m, C.byref(s)))
        else:
            pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1))
            size = pos.size
            count = size // 3
            if count > self.capacity:
                raise ValueError(f"count {count} exceeds capacity {self.capacity}")
            if size != 3 * count:
                raise ValueError(f"positions must hold 3*count = {3 * count} floats, "
                                 f"got {size}")
            _lib.check(self._L.bt_initialize_particle_location(
                self._h, pos.ctypes.data, size, _lib.BT_MEM_HOST, m, C.byref(s)))
        self._count = size // 3
        self.last_init_summary = TraceSummary._from(s)

    def move_to_next_location(self, destinations, flying, weights, groups=None):
        """tally.py:247-271. Returns TraceSummary, or None when count == 0."""
        s = _lib.Summary()
        if _is_device(flying):
            count = flying.numel()
            for t, isz in ((destinations, 8), (flying, 1), (weights, 8)):
                self._check_tensor(t, isz)
            if destinations.numel() != 3 * count or weights.numel() != count:
                raise ValueError(
                    f"array sizes ({destinations.numel()}, {count}, {weights.numel()}) do not "
                    f"match count {count} (need 3*count, count, count)")
            if count > self.capacity:
                raise ValueError(f"count {count} outside [0, {self.capacity}]")
            gp = None
            if groups is not None:
                self._check_tensor(groups, 4)
                if groups.numel() != count:
                    raise ValueError("groups size mismatch")
                gp = groups.data_ptr()
            if count == 0:
                return None
            _producer_sync(flying)
            _lib.check(self._L.bt_move_to_next_location(
                self._h, destinations.data_ptr(), flying.data_ptr(), weights.data_ptr(), gp,
                count, _lib.BT_MEM_DEVICE, C.byref(s)))
            return TraceSummary._from(s)
        fly = np.ascontiguousarray(np.asarray(flying).reshape(-1).astype(np.int8, copy=False))
        count = fly.size
        dest = np.ascontiguousarray(np.asarray(destinations, dtype=np.float64).reshape(-1))
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
        if count > self.capacity:
            raise ValueError(f"count {count} outside [0, {self.capacity}]")
        if dest.size != 3 * count or w.size != count:
            raise ValueError(
                f"array sizes ({dest.size}, {fly.size}, {w.size}) do not match "
                f"count {count} (need 3*count, count, count)")
        if count == 0:
            return None
        gp = None
        if groups is not None:
            g = np.ascontiguousarray(np.asarray(groups, dtype=np.int32).reshape(-1))
            if g.size != count:
                raise ValueError("groups size mismatch")
            gp = g.ctypes.data
        _lib.check(self._L.bt_move_to_next_location(
            self._h, dest.ctypes.data, fly.ctypes.data, w.ctypes.data, gp, count,
            _lib.BT_MEM_HOST, C.byref(s)))
        return TraceSummary._from(s)

    def finalize_batch(self, source_weight: float | None = None) -> None:
        """tally.py:273-279."""
        w = self.source_weight if source_weight is None else source_weight
        if not w or w <= 0.0:
            raise RuntimeError("no source weight recorded for this batch; pass source_weight")
        _lib.check(self._L.bt_finalize_batch(self._h, float(w)))

    def flux(self) -> FluxResult:
        return flux(self._grid, self._mesh.volumes)

    def flux_device(self, estimator: str = "track") -> FluxResult:
        """flux() evaluated on the GPU (bt_flux); estimator 'track' or 'collision'."""
        ne, ng = self._mesh.num_elements, self.num_groups
        vol = np.ascontiguousarray(self._mesh.volumes, dtype=np.float64)
        mean = np.empty((ne, ng))
        rel = np.empty((ne, ng))
        _lib.check(self._L.bt_flux(self._h, 0 if estimator == "track" else 1, vol.ctypes.data,
                                   mean.ctypes.data, rel.ctypes.data))
        return FluxResult(mean=mean, rel_error=rel)

    def write(self, filename) -> None:
        write_vtk(self._mesh, self.flux(), filename)

    # ------------------------------------------------------- callback path
    def load_step(self, destinations, flying, weights, groups=None) -> int:
        """load_step (particles.py:57-89): load a step for ``trace_batch``."""
        return _mt_load_step(self, destinations, flying, weights, groups)

    def trace_batch(self, callback=None, *, score: bool = True, max_sweeps: int | None = None,
                    device_events: bool = False) -> TraceSummary:
        """trace_batch (search.py:453-489): lockstep sweeps over the loaded step
        with ``callback(SweepEvents)`` between each proposal and commit."""
        return _mt_trace_batch(self, callback, score=score, max_sweeps=max_sweeps,
                               device_events=device_events)

    # ------------------------------------------------------------------ extras
    # dtypes a CUDA tensor argument must have: the library reads its bits as
    # float64 / int8 / int32 (the reference converts host arrays with
    # np.asarray(dtype=...); a device buffer is never converted silently)
    _DEVICE_DTYPES = {8: ("float64",), 1: ("int8", "uint8", "bool"), 4: ("int32",)}

    def _check_tensor(self, t, itemsize):
        if not t.is_contiguous():
            raise ValueError("device arrays must be contiguous")
        dt = str(t.dtype).replace("torch.", "")
        if dt not in self._DEVICE_DTYPES[itemsize]:
            raise TypeError(f"device array has dtype {dt}, expected "
                            f"{' or '.join(self._DEVICE_DTYPES[itemsize])}")
        if t.device.index is not None and t.device.index != self.device:
            raise ValueError(f"tensor on cuda:{t.device.index}, handle on cuda:{self.device}")

    @property
    def num_elements(self) -> int:
        return self._mesh.num_elements

    def _write_tally(self, which, a) -> None:
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
        _lib.check(self._L.bt_write_tally(self._h, which, a.ctypes.data, a.size))

    def _read_tally(self, which) -> np.ndarray:
        n = self._mesh.num_elements * self.num_groups
        out = np.empty(n)
        _lib.check(self._L.bt_read_tally(self._h, which, out.ctypes.data, n))
        return out

    def batch_totals(self) -> np.ndarray:
        return batch_totals(self._grid)

    def tally_device_ptr(self, which=_lib.BT_TALLY_BATCH) -> int:
        p = C.c_void_p()
        _lib.check(self._L.bt_tally_device_ptr(self._h, which, C.byref(p)))
        return int(p.value)

    def read_particles(self, count: int | None = None) -> ParticleState:
        n = self._count if count is None else int(count)
        pos = np.empty((n, 3))
        el = np.empty(n, np.int32)
        al = np.empty(n, np.int8)
        ef = np.empty(n, np.int8)
        st = np.empty(n, np.int8)
        oc = np.empty(n, np.int8)
        sg = np.empty(n)
        _lib.check(self._L.bt_read_particles(self._h, n, pos.ctypes.data, el.ctypes.data,
                                             al.ctypes.data, ef.ctypes.data, st.ctypes.data,
                                             oc.ctypes.data, sg.ctypes.data))
        return ParticleState(pos, el, al, ef, st, oc, sg)

    def read_digest(self, count: int | None = None):
        n = self._count if count is None else int(count)
        d = np.empty(n, np.uint64)
        c = np.empty(n, np.int64)
        _lib.check(self._L.bt_read_digest(self._h, n, d.ctypes.data, c.ctypes.data))
        return d, c

    def last_timing(self):
        """(walk kernel ms, whole call ms, kernels launched) of the last call."""
        w = C.c_float()
        c = C.c_float()
        k = C.c_int64()
        _lib.check(self._L.bt_last_timing(self._h, C.byref(w), C.byref(c), C.byref(k)))
        return float(w.value), float(c.value), int(k.value)

    def particle_tensors(self):
        """Zero-copy torch views (position (N,3) f64, element i32, alive i8) of
        the device particle state, for device-side drivers."""
        import torch
        from .distributed import _CudaArray
        p, e, a = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.check(self._L.bt_particle_device_ptrs(self._h, C.byref(p), C.byref(e), C.byref(a)))
        dev = torch.device("cuda", self.device)
        n = self.capacity
        pos = torch.as_tensor(_CudaArray(p.value, 3 * n, "<f8"), device=dev).view(n, 3)
        el = torch.as_tensor(_CudaArray(e.value, n, "<i4"), device=dev)
        al = torch.as_tensor(_CudaArray(a.value, n, "|i1"), device=dev)
        return pos, el, al

    def save_state(self) -> None:
        _lib.check(self._L.bt_save_state(self._h))

    def restore_state(self) -> None:
        _lib.check(self._L.bt_restore_state(self._h))

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.bt_destroy(h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---------------------------------------------------------------------------
# Listing-1 callback path (search.py:95-147, 453-489)

@dataclass(frozen=True)
class InterfaceEvent:
    """One element-interface crossing of one particle (search.py:95-105)."""

    particle: int
    element: int
    exit_face: int
    boundary: bool
    segment_start: np.ndarray
    segment_end: np.ndarray
    segment_length: float


class SweepEvents:
    """Batched view of one sweep's events (search.py:108-147).

    Read-only: particle, element, exit_face, boundary, segment_start,
    segment_end, segment_length.  Writable decisions: next_element and
    particle_done.  Host numpy copies by default; with
    ``trace_batch(..., device_events=True)`` the arrays are zero-copy torch
    CUDA tensors of the library's event buffers.
    """

    def __init__(self, arrays: dict, count: int):
        self.count = count
        for k, v in arrays.items():
            setattr(self, k, v)

    @property
    def boundary(self):
        return (self.next_proposed < 0) & (self.exit_face >= 0)

    def __len__(self) -> int:
        return self.count

    def event(self, k: int) -> InterfaceEvent:
        if not 0 <= k < self.count:
            raise IndexError(k)
        return InterfaceEvent(
            particle=int(self.particle[k]), element=int(self.element[k]),
            exit_face=int(self.exit_face[k]), boundary=bool(self.boundary[k]),
            segment_start=np.array(self.segment_start[k].tolist()),
            segment_end=np.array(self.segment_end[k].tolist()),
            segment_length=float(self.segment_length[k]))


_EV_FIELDS = (("particle", np.int64, 1), ("element", np.int32, 1), ("exit_face", np.int8, 1),
              ("segment_start", np.float64, 3), ("segment_end", np.float64, 3),
              ("segment_length", np.float64, 1), ("next_element", np.int32, 1),
              ("particle_done", np.int8, 1), ("next_proposed", np.int32, 1))


def _mt_load_step(self, destinations, flying, weights, groups=None) -> int:
    """load_step (particles.py:57-89) for the callback path."""
    fly = np.ascontiguousarray(np.asarray(flying).reshape(-1).astype(np.int8, copy=False))
    count = fly.size
    dest = np.ascontiguousarray(np.asarray(destinations, dtype=np.float64).reshape(-1))
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64).reshape(-1))
    if count > self.capacity:
        raise ValueError(f"count {count} outside [0, {self.capacity}]")
    if dest.size != 3 * count or w.size != count:
        raise ValueError(f"array sizes ({dest.size}, {fly.size}, {w.size}) do not match "
                         f"count {count} (need 3*count, count, count)")
    gp = None
    if groups is not None:
        g = np.ascontiguousarray(np.asarray(groups, dtype=np.int32).reshape(-1))
        if g.size != count:
            raise ValueError("groups size mismatch")
        gp = g.ctypes.data
    _lib.check(self._L.bt_load_step(self._h, dest.ctypes.data, fly.ctypes.data, w.ctypes.data,
                                    gp, count, _lib.BT_MEM_HOST))
    self._count = max(self._count, count)
    return count


def _mt_trace_batch(self, callback=None, *, score: bool = True, max_sweeps: int | None = None,
                    device_events: bool = False) -> TraceSummary:
    """trace_batch (search.py:453-489) on the loaded step: one lockstep sweep
    at a time, ``callback(SweepEvents)`` between proposal and commit."""
    L = self._L
    _lib.check(L.bt_trace_begin(self._h, int(bool(score)),
                                -1 if max_sweeps is None else int(max_sweeps)))
    ev = _lib.SweepEventsC()
    flying = C.c_int64()
    while True:
        _lib.check(L.bt_trace_propose(self._h, C.byref(ev), C.byref(flying)))
        if flying.value == 0:
            break
        n = int(ev.count)
        if callback is not None and n > 0:
            if device_events:
                import torch
                from .distributed import _CudaArray
                dev = torch.device("cuda", self.device)
                arrays = {}
                for name, dt, k in _EV_FIELDS:
                    t = torch.as_tensor(_CudaArray(getattr(ev, name), n * k,
                                                   np.dtype(dt).str), device=dev)
                    arrays[name] = t.view(n, 3) if k == 3 else t
                view = SweepEvents(arrays, n)
                callback(view)
                torch.cuda.current_stream(dev).synchronize()
            else:
                arrays = {}
                for name, dt, k in _EV_FIELDS:
                    a = np.empty(n * k, dtype=dt)
                    _lib.check(_copy_d2h(a, getattr(ev, name)))
                    arrays[name] = a.reshape(n, 3) if k == 3 else a
                view = SweepEvents(arrays, n)
                callback(view)
                _lib.check(_copy_h2d(getattr(ev, "next_element"),
                                     np.ascontiguousarray(view.next_element, dtype=np.int32)))
                _lib.check(_copy_h2d(getattr(ev, "particle_done"),
                                     np.ascontiguousarray(view.particle_done, dtype=np.int8)))
        _lib.check(L.bt_trace_commit(self._h))
    s = _lib.Summary()
    _lib.check(L.bt_trace_end(self._h, C.byref(s)))
    return TraceSummary._from(s)


def _copy_d2h(host: np.ndarray, dptr: int) -> int:
    return _lib.load().bt_memcpy(host.ctypes.data, dptr, host.nbytes, 0)


def _copy_h2d(dptr: int, host: np.ndarray) -> int:
    return _lib.load().bt_memcpy(dptr, host.ctypes.data, host.nbytes, 1)

