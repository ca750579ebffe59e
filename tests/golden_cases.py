"""Loader for the reference-generated golden fixtures (tests/golden/*.npz,
written by oracle/gen_golden.py from the reference package itself)."""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from paper_2504_19048_b200 import mesh as mymesh

GOLDEN = Path(__file__).resolve().parent / "golden"
WALK_CASES = ["c1_point_s2", "c1_point_s100", "n6_uniform_g3", "straight_ray",
              "grid_plane_ladder", "torus_small"]
STATE_KEYS = ("position", "element", "alive", "flying", "entry_face", "stuck", "outcome")


@dataclass
class Move:
    dest: np.ndarray
    flying: np.ndarray
    weights: np.ndarray
    groups: np.ndarray | None
    expect: dict = field(default_factory=dict)


@dataclass
class Batch:
    init_positions: np.ndarray
    init_element: np.ndarray
    init_alive: np.ndarray
    moves: list
    source_weight: float
    sum: np.ndarray
    sum_sq: np.ndarray


@dataclass
class WalkCase:
    name: str
    mesh: object
    num_groups: int
    capacity: int
    batches: list
    flux_mean: np.ndarray
    flux_rel: np.ndarray


_MESH_CACHE = {}


def case_mesh(d):
    kind = str(d["mesh_kind"])
    if kind == "cube":
        key = ("cube", int(d["mesh_n"]))
        if key not in _MESH_CACHE:
            _MESH_CACHE[key] = mymesh.build_cube_mesh(int(d["mesh_n"]))
    else:
        params = dict(nr=int(d["mesh_nr"]), ntheta=int(d["mesh_ntheta"]),
                      nphi=int(d["mesh_nphi"]), R=float(d["mesh_R"]),
                      a_in=float(d["mesh_a_in"]), a_out=float(d["mesh_a_out"]))
        key = ("torus",) + tuple(params.values())
        if key not in _MESH_CACHE:
            _MESH_CACHE[key] = mymesh.build_torus_shell_mesh(**params)
    return _MESH_CACHE[key]


def load_walk_case(name: str) -> WalkCase:
    d = np.load(GOLDEN / f"walk_{name}.npz")
    batches = []
    for bi in range(int(d["num_batches"])):
        pre = f"b{bi}_"
        moves = []
        for mi in range(int(d[pre + "num_moves"])):
            pm = f"{pre}m{mi}_"
            g = d[pm + "groups"] if (pm + "groups") in d.files else None
            exp = {k: d[pm + k] for k in STATE_KEYS + ("seg_delta", "count", "digest",
                                                      "summary", "tally")}
            if (pm + "seq_codes") in d.files:
                exp["seq_codes"] = d[pm + "seq_codes"]
            moves.append(Move(d[pm + "dest"], d[pm + "flying_in"], d[pm + "weights"], g, exp))
        batches.append(Batch(d[pre + "init_positions"], d[pre + "init_element"],
                             d[pre + "init_alive"], moves, float(d[pre + "source_weight"]),
                             d[pre + "sum"], d[pre + "sum_sq"]))
    return WalkCase(name, case_mesh(d), int(d["num_groups"]), int(d["capacity"]), batches,
                    d["flux_mean"], d["flux_rel"])


def rel_close(a, b, tol):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.abs(a), np.abs(b))
    diff = np.abs(a - b)
    ok = (diff <= tol * den) | (diff == 0)
    return bool(ok.all()), float((diff / np.where(den > 0, den, 1)).max(initial=0.0))
