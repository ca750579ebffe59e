"""Fixed-source analog multigroup transport on the GPU,
a drop-in for the reference's driver API (meshtally/transport.py):

* ``CrossSections`` (transport.py:50-99) with the same validation and the same
  derived scatter probability / group CDF (``XSData``),
* ``RunConfig`` (transport.py:102-147) and ``RunResult`` (transport.py:422-442),
* ``run(config, mesh=None)`` (transport.py:445-549).

The reference alternates flight / walk / collide events over all particles.
Here one lane runs each particle's whole history on the device
(``bt_transport_run``); the per-particle random draws are the reference's
philox4x64-10 stream keyed (seed, batch, particle, block), so histories are
the same sequence of operations.  They match the reference bit for bit as
long as CUDA's ``log``/``sin``/``cos`` round like the host C library; a
differing last bit sends a history elsewhere, so parity is statistical
(tests/test_transport_gpu.py measures both).  Localization uses the grid
search (lowest-id containing element) instead of the centroid-0 walk; for
source points in the interior of the mesh the element is the same.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .mesh import TetMesh, build_cube_mesh
from .tally import FluxResult, MeshTally, flux as _flux


@dataclass(frozen=True)
class CrossSections:
    """Multigroup total and scattering data; absorption is the difference."""

    sigma_t: np.ndarray
    sigma_s: np.ndarray

    def __post_init__(self):
        st = np.ascontiguousarray(np.atleast_1d(self.sigma_t), dtype=np.float64)
        ss = np.ascontiguousarray(np.atleast_2d(self.sigma_s), dtype=np.float64)
        object.__setattr__(self, "sigma_t", st)
        object.__setattr__(self, "sigma_s", ss)
        g = st.shape[0]
        if ss.shape != (g, g):
            raise ValueError(f"sigma_s must be ({g}, {g}), got {ss.shape}")
        if not (st > 0.0).all():
            raise ValueError("sigma_t must be positive in every group")
        if (ss < 0.0).any():
            raise ValueError("sigma_s entries must be non-negative")
        rows = ss.sum(axis=1)
        if (rows > st * (1.0 + 1e-12)).any():
            bad = int(np.argmax(rows - st))
            raise ValueError(f"scattering row sum {rows[bad]:g} exceeds sigma_t "
                             f"{st[bad]:g} in group {bad}")

    @property
    def num_groups(self) -> int:
        return int(self.sigma_t.shape[0])

    @classmethod
    def one_group(cls, sigma_t: float, sigma_s: float) -> "CrossSections":
        return cls(np.array([sigma_t]), np.array([[sigma_s]]))

    def kernel_data(self):
        """(sigma_t, scatter_prob, group_cdf) exactly as XSData (transport.py:83-99)."""
        g = self.num_groups
        rows = self.sigma_s.sum(axis=1)
        prob = rows / self.sigma_t
        cdf = np.zeros((g, g))
        for i in range(g):
            if rows[i] > 0.0:
                cdf[i] = np.cumsum(self.sigma_s[i]) / rows[i]
            cdf[i, g - 1] = 1.0
        return (np.ascontiguousarray(self.sigma_t), np.ascontiguousarray(prob),
                np.ascontiguousarray(cdf))


@dataclass(frozen=True)
class RunConfig:
    mesh_n: int = 10
    edge_length: float = 1.0
    num_particles: int = 10_000
    num_batches: int = 5
    cross_sections: CrossSections = field(
        default_factory=lambda: CrossSections.one_group(100.0, 100.0))
    source_box: tuple = ((0.0, 0.0, 0.0), (0.5, 0.5, 0.5))
    seed: int = 42
    backend: str = "adjacency"
    threads: int = 1
    vtk_path: str | None = None
    csv_path: str | None = None
    source_direction: tuple | None = None

    def __post_init__(self):
        if self.mesh_n < 1:
            raise ValueError("mesh_n must be >= 1")
        if self.edge_length <= 0.0:
            raise ValueError("edge_length must be positive")
        if self.num_particles <= 0:
            raise ValueError("num_particles must be positive")
        if self.num_batches <= 0:
            raise ValueError("num_batches must be positive")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.backend not in ("adjacency", "baseline"):
            raise ValueError(f"unknown backend {self.backend!r} "
                             "(expected 'adjacency' or 'baseline')")
        if self.backend == "baseline":
            raise ValueError("the KD-tree baseline backend is not part of this package "
                             "(SURVEY.md §2: out of scope)")
        box = np.asarray(self.source_box, dtype=np.float64).reshape(2, 3)
        if (box[1] < box[0]).any():
            raise ValueError("source_box max corner below min corner")
        if (box[0] < 0.0).any() or (box[1] > self.edge_length).any():
            raise ValueError("source_box must lie inside the mesh domain")
        object.__setattr__(self, "source_box", (tuple(box[0]), tuple(box[1])))
        if self.source_direction is not None:
            d = np.asarray(self.source_direction, dtype=np.float64).reshape(3)
            n = float(np.sqrt(d @ d))
            if n == 0.0:
                raise ValueError("source_direction must be non-zero")
            object.__setattr__(self, "source_direction", tuple(d / n))


@dataclass
class RunResult:
    config: RunConfig
    mesh: TetMesh
    flux_track: FluxResult
    flux_collision: FluxResult
    track_grid: object
    collision_grid: object
    t_init: float
    t_localization: float
    t_batch: float
    t_output: float
    source_weight: float
    leaked_weight: float
    absorbed_weight: float
    stuck_weight: float
    collisions: int
    events: int
    sweeps: int
    track_length_total: float
    threads_used: int
    final_state: dict = field(default_factory=dict, repr=False)


class _CollisionGrid:
    """Grid view of the collision estimator (same fields as TallyGrid)."""

    def __init__(self, mt: MeshTally):
        self._mt = mt
        self.num_elements = mt.mesh.num_elements
        self.num_groups = mt.num_groups

    @property
    def sum(self):
        return self._mt._read_tally(_lib.BT_TALLY_COL_SUM)

    @property
    def sum_sq(self):
        return self._mt._read_tally(_lib.BT_TALLY_COL_SUM_SQ)

    @property
    def partials(self):
        return self._mt._read_tally(_lib.BT_TALLY_COL_BATCH)[None, :]

    @property
    def batches_completed(self):
        return self._mt.batches_completed


def run(config: RunConfig, mesh: TetMesh | None = None, *, device: int = 0,
        tally: MeshTally | None = None) -> RunResult:
    """transport.run on the GPU: flux results for both estimators, balance
    totals and phase timings (device-measured)."""
    t0 = time.perf_counter()
    if mesh is None:
        mesh = build_cube_mesh(config.mesh_n, config.edge_length)
    xs = config.cross_sections
    mt = tally if tally is not None else MeshTally(mesh, config.num_particles, xs.num_groups,
                                                   device=device)
    st, prob, cdf = xs.kernel_data()
    box = np.ascontiguousarray(np.asarray(config.source_box, dtype=np.float64).reshape(6))
    fd = (None if config.source_direction is None
          else np.ascontiguousarray(config.source_direction, dtype=np.float64))
    t_init = time.perf_counter() - t0
    tot = _lib.TransportTotals()
    _lib.check(mt._L.bt_transport_run(
        mt._h, st.ctypes.data, prob.ctypes.data, cdf.ctypes.data, xs.num_groups,
        config.num_particles, config.num_batches, int(config.seed) & (2**64 - 1),
        box.ctypes.data, None if fd is None else fd.ctypes.data, C.byref(tot)))
    n = config.num_particles
    flux_track = _flux(mt.grid, mesh.volumes)
    cgrid = _CollisionGrid(mt)
    flux_col = _flux(cgrid, mesh.volumes)
    ps = mt.read_particles(n)
    d = np.empty((n, 3))
    g = np.empty(n, np.int32)
    rb = np.empty(n, np.uint32)
    _lib.check(mt._L.bt_read_transport_state(mt._h, n, d.ctypes.data, g.ctypes.data,
                                             rb.ctypes.data))
    final = dict(position=ps.position, element=ps.element, alive=ps.alive, outcome=ps.outcome,
                 seg_total=ps.seg_total, direction=d, group=g, rng_block=rb.astype(np.uint64))
    res = RunResult(
        config=config, mesh=mesh, flux_track=flux_track, flux_collision=flux_col,
        track_grid=mt.grid, collision_grid=cgrid, t_init=t_init,
        t_localization=tot.ms_localization / 1e3, t_batch=tot.ms_transport / 1e3,
        t_output=0.0, source_weight=tot.source_weight, leaked_weight=tot.leaked_weight,
        absorbed_weight=tot.absorbed_weight, stuck_weight=tot.stuck_weight,
        collisions=int(tot.collisions), events=int(tot.events), sweeps=int(tot.sweeps),
        track_length_total=tot.track_length_total, threads_used=1, final_state=final)
    if config.vtk_path:
        from .tally import write_vtk
        write_vtk(mesh, flux_track, config.vtk_path)
    if config.csv_path:
        from .tally import write_flux_csv
        write_flux_csv(flux_track, config.csv_path)
    res._tally = mt
    return res


def uniform_blocks(keys, device: int = 0) -> np.ndarray:
    """Device philox uniform_block for rows (seed, batch, particle, block)."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, 4))
    out = np.empty((k.shape[0], 4))
    L = _lib.load()
    _lib.check(L.bt_uniform_blocks(k.ctypes.data, k.shape[0], device, out.ctypes.data))
    return out
