"""ctypes binding of libb200tally.so (the C ABI in include/b200tally.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is visible, handle creation raises.  Status codes map onto
the reference's exception classes (tally.py:219-222, particles.py:65-73,
search.py:513-516, tally.py:275-277).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# BT_LIB_PATH: an alternative build of the same library (tools/build_variant.sh
# experiments); there is no non-native path either way
LIB_PATH = Path(os.environ.get("BT_LIB_PATH") or PKG / "libb200tally.so")

BT_OK, BT_EINVAL, BT_ERUNTIME, BT_ECUDA, BT_EINDEX, BT_ENOMEM = range(6)
BT_MEM_HOST, BT_MEM_DEVICE = 0, 1
BT_LOCATE_GRID, BT_LOCATE_WALK = 0, 1
(BT_TALLY_BATCH, BT_TALLY_SUM, BT_TALLY_SUM_SQ, BT_TALLY_COL_BATCH, BT_TALLY_COL_SUM,
 BT_TALLY_COL_SUM_SQ) = range(6)
(BT_OPT_MAX_SWEEPS, BT_OPT_DIGEST, BT_OPT_SORT, BT_OPT_WARP_AGG,
 BT_OPT_BLOCKS_PER_SM, BT_OPT_STAGED, BT_OPT_MOVE_CHUNKS, BT_OPT_LOCATE_LANES,
 BT_OPT_EXACT_ONLY, BT_OPT_DEFER_INIT, BT_OPT_STREAM_MOVE) = range(11)

# every symbol declared in include/b200tally.h (checked by tests/test_abi.py)
EXPORTS = (
    "bt_create", "bt_create_multi", "bt_num_shards", "bt_shard", "bt_destroy",
    "bt_initialize_particle_location",
    "bt_move_to_next_location", "bt_finalize_batch", "bt_read_tally",
    "bt_tally_device_ptr", "bt_get_source_weight", "bt_set_source_weight",
    "bt_batches_completed", "bt_read_particles", "bt_read_digest", "bt_set_option",
    "bt_last_timing", "bt_particle_device_ptrs", "bt_save_state", "bt_restore_state",
    "bt_info", "bt_build_adjacency", "bt_transport_run", "bt_read_transport_state",
    "bt_uniform_blocks", "bt_glibc_math", "bt_load_step", "bt_trace_begin", "bt_trace_propose",
    "bt_trace_commit", "bt_trace_end", "bt_memcpy", "bt_flux",
    "bt_create_grid", "bt_score", "bt_write_tally", "bt_set_batches_completed",
    "bt_mesh_read", "bt_mesh_from_arrays", "bt_mesh_info", "bt_mesh_arrays", "bt_mesh_destroy",
    "bt_create_from_mesh", "bt_create_from_file", "bt_write_vtk", "bt_write_flux_csv",
    "bt_device_count", "bt_format_double",
    "bt_last_error", "bt_version",
)


class TransportTotals(C.Structure):
    _fields_ = [("source_weight", C.c_double), ("leaked_weight", C.c_double),
                ("absorbed_weight", C.c_double), ("stuck_weight", C.c_double),
                ("track_length_total", C.c_double), ("collisions", C.c_int64),
                ("events", C.c_int64), ("sweeps", C.c_int64),
                ("ms_localization", C.c_float), ("ms_transport", C.c_float)]


class SweepEventsC(C.Structure):
    """bt_sweep_events (device pointers)."""
    _fields_ = [("count", C.c_int64)] + [(n, C.c_void_p) for n in (
        "particle", "element", "exit_face", "segment_start", "segment_end", "segment_length",
        "next_element", "particle_done", "next_proposed")]


class Summary(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("events", C.c_int64), ("reached", C.c_int64),
                ("boundary_exits", C.c_int64), ("stuck_recoveries", C.c_int64),
                ("stuck_terminations", C.c_int64)]


_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

_SIGS = {
    "bt_create": [_P, _I64, _P, _P, _P, _I64, _P, _P, _I64, _I32, _I32, C.POINTER(_P)],
    "bt_create_multi": [_P, _I64, _P, _P, _P, _I64, _P, _P, _I64, _I32, _P, _I32, C.POINTER(_P)],
    "bt_num_shards": [_P, C.POINTER(_I32)],
    "bt_shard": [_P, _I32, C.POINTER(_P), C.POINTER(_I64), C.POINTER(_I64)],
    "bt_destroy": [_P],
    "bt_initialize_particle_location": [_P, _P, _I64, _I32, _I32, C.POINTER(Summary)],
    "bt_move_to_next_location": [_P, _P, _P, _P, _P, _I64, _I32, C.POINTER(Summary)],
    "bt_finalize_batch": [_P, C.c_double],
    "bt_read_tally": [_P, _I32, _P, _I64],
    "bt_tally_device_ptr": [_P, _I32, C.POINTER(_P)],
    "bt_get_source_weight": [_P, C.POINTER(C.c_double)],
    "bt_set_source_weight": [_P, C.c_double],
    "bt_batches_completed": [_P, C.POINTER(_I64)],
    "bt_read_particles": [_P, _I64, _P, _P, _P, _P, _P, _P, _P],
    "bt_read_digest": [_P, _I64, _P, _P],
    "bt_set_option": [_P, _I32, _I64],
    "bt_last_timing": [_P, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(_I64)],
    "bt_particle_device_ptrs": [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)],
    "bt_save_state": [_P],
    "bt_restore_state": [_P],
    "bt_info": [_P, C.POINTER(_I32), C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I32)],
    "bt_build_adjacency": [_P, _I64, _I64, _I32, _P, _P],
    "bt_transport_run": [_P, _P, _P, _P, _I32, _I64, _I64, C.c_uint64, _P, _P,
                         C.POINTER(TransportTotals)],
    "bt_read_transport_state": [_P, _I64, _P, _P, _P],
    "bt_uniform_blocks": [_P, _I64, _I32, _P],
    "bt_glibc_math": [_P, _I64, _I32, _I32, _P],
    "bt_load_step": [_P, _P, _P, _P, _P, _I64, _I32],
    "bt_trace_begin": [_P, _I32, _I64],
    "bt_trace_propose": [_P, C.POINTER(SweepEventsC), C.POINTER(_I64)],
    "bt_trace_commit": [_P],
    "bt_trace_end": [_P, C.POINTER(Summary)],
    "bt_memcpy": [_P, _P, _I64, _I32],
    "bt_flux": [_P, _I32, _P, _P, _P],
    "bt_create_grid": [_I64, _I32, _I32, C.POINTER(_P)],
    "bt_score": [_P, _I32, _P, _P, _P, _P, _I64, _I32],
    "bt_write_tally": [_P, _I32, _P, _I64],
    "bt_set_batches_completed": [_P, _I64],
    "bt_mesh_read": [C.c_char_p, _I32, C.POINTER(_P)],
    "bt_mesh_from_arrays": [_P, _I64, _P, _I64, _I32, C.POINTER(_P)],
    "bt_mesh_info": [_P, C.POINTER(_I64), C.POINTER(_I64)],
    "bt_mesh_arrays": [_P, _P, _P, _P, _P, _P, _P, _P],
    "bt_mesh_destroy": [_P],
    "bt_create_from_mesh": [_P, _I64, _I32, _I32, C.POINTER(_P)],
    "bt_create_from_file": [C.c_char_p, _I64, _I32, _I32, C.POINTER(_P)],
    "bt_write_vtk": [_P, C.c_char_p, _P],
    "bt_write_flux_csv": [_P, C.c_char_p, _P],
    "bt_device_count": [C.POINTER(_I32)],
    "bt_format_double": [C.c_double, C.c_char_p, _I32],
    "bt_last_error": [],
    "bt_version": [],
}

_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load(build_if_missing: bool = True):
    """Load (building first if needed) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and build_if_missing:
        from . import build as _build
        _build.build()
    if not LIB_PATH.exists():
        raise ExtensionMissing(
            f"{LIB_PATH} is missing: run `python -m paper_2504_19048_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_char_p if name in ("bt_last_error", "bt_version") else C.c_int
    _lib = L
    return L


def device_count() -> int:
    """Visible CUDA devices (0 on a host without a GPU)."""
    n = C.c_int32()
    check(load().bt_device_count(C.byref(n)))
    return int(n.value)


def check(status: int) -> None:
    if status == BT_OK:
        return
    msg = load().bt_last_error().decode(errors="replace")
    if status == BT_EINVAL:
        raise ValueError(msg)
    if status == BT_EINDEX:
        raise IndexError(msg)
    if status == BT_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
