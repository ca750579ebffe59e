"""B200-native PUMI-Tally hot path (arXiv 2504.19048): tet-mesh adjacency walk
with per-element track-length tallies, as a drop-in for the reference
package's tally API (``meshtally``: mesh load, ``MeshTally``, batch
finalize, flux readout).

The walk, localization and tally kernels are hand-written sm_100a CUDA in
``csrc/`` behind the C ABI of ``include/b200tally.h``; this package is the
Python host side (ctypes).  There is no CPU fallback.
"""

from .mesh import (
    FACE_VERTICES,
    MalformedMeshError,
    TetMesh,
    build_adjacency,
    build_cube_mesh,
    build_torus_shell_mesh,
    element_volume,
    read_tetmesh,
    validate,
    write_tetmesh,
)
from .tally import (
    OUTCOME_LEAKED,
    OUTCOME_NONE,
    OUTCOME_REACHED,
    OUTCOME_STUCK_KILLED,
    FluxResult,
    MeshTally,
    ParticleState,
    TallyGrid,
    TraceSummary,
    batch_totals,
    create_grid,
    finalize_batch,
    flux,
    score_collision,
    score_track_length,
    write_flux_csv,
    write_vtk,
)
from .transport import CrossSections, RunConfig, RunResult, run

__all__ = [
    "FACE_VERTICES", "MalformedMeshError", "TetMesh", "build_adjacency", "build_cube_mesh",
    "build_torus_shell_mesh", "element_volume", "read_tetmesh", "validate", "write_tetmesh",
    "OUTCOME_LEAKED", "OUTCOME_NONE", "OUTCOME_REACHED", "OUTCOME_STUCK_KILLED",
    "FluxResult", "MeshTally", "ParticleState", "TallyGrid", "TraceSummary", "batch_totals",
    "create_grid", "finalize_batch", "flux", "score_collision", "score_track_length",
    "write_flux_csv", "write_vtk",
    "CrossSections", "RunConfig", "RunResult", "run",
]
