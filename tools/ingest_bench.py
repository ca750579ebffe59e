"""Mesh ingest at the sizes that motivate it (reference
mesh.py:109-148, 188-235, 302-331): text read + orientation + adjacency of
the C4 cubes (n = 95: 5,144,250 tets; n = 119: 10,110,954) and the C5 torus
shell (5,013,504 tets).  Times the native ingest (bt_mesh_read /
bt_mesh_from_arrays: all host threads, adjacency on the GPU), the host numpy
builder, and -- when baseline/_ref imports -- the reference's own
read_tetmesh / from_arrays.  One JSON line per measurement.

    python tools/ingest_bench.py [--out profiles/r02_ingest.jsonl] [--reference]
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def cube_arrays(n):
    from paper_2504_19048_b200 import mesh as M
    nv = n + 1
    coord = np.arange(nv, dtype=np.float64) * (1.0 / n)
    coord[-1] = 1.0
    vid = np.arange(nv ** 3, dtype=np.int64)
    v = np.stack([coord[vid // (nv * nv)], coord[(vid // nv) % nv], coord[vid % nv]], axis=1)
    cell = np.arange(n ** 3, dtype=np.int64)
    base = ((cell // (n * n)) * nv + (cell // n) % n) * nv + cell % n
    offs = np.array([((b >> 2) & 1) * nv * nv + ((b >> 1) & 1) * nv + (b & 1) for b in range(8)])
    e = (base[:, None, None] + offs[M.KUHN_TETS][None, :, :]).reshape(-1, 4)
    return v, e


def write_text(path, v, e):
    """write_tetmesh's format (mesh.py:302-309), vectorised."""
    with open(path, "w") as fh:
        fh.write(f"tetmesh {v.shape[0]} {e.shape[0]}\n")
        fh.write("\n".join(f"{x!r} {y!r} {z!r}" for x, y, z in v.tolist()))
        fh.write("\n")
        np.savetxt(fh, e, fmt="%d")


def timed(fn):
    t = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reference", action="store_true")
    ap.add_argument("--sizes", default="95,119,torus")
    args = ap.parse_args()
    from paper_2504_19048_b200 import mesh as M
    ref = None
    if args.reference:
        sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
        try:
            import meshtally as ref
        except Exception as err:  # noqa: BLE001
            print(json.dumps({"reference": f"unavailable: {err}"}))
    res = []
    tmp = Path(tempfile.mkdtemp())
    M.build_cube_mesh(2)  # library load + CUDA context outside the timings
    for size in args.sizes.split(","):
        if size == "torus":
            v, e = M.torus_shell_arrays(8, 256, 408)
            label = "C5 torus 8x256x408"
        else:
            v, e = cube_arrays(int(size))
            label = f"C4 cube n={size}"
        path = tmp / f"{size}.tet"
        write_text(path, v, e)
        mb = path.stat().st_size / 1e6
        rows = []
        m, t = timed(lambda: M.read_tetmesh(path))
        rows.append(("read_tetmesh", "native (bt_mesh_read, GPU adjacency)", t))
        _, t2 = timed(lambda: M.TetMesh.from_arrays(v, e))
        rows.append(("from_arrays", "native (bt_mesh_from_arrays, GPU adjacency)", t2))
        m2, t3 = timed(lambda: M.TetMesh.from_arrays(v, e, device=None))
        rows.append(("from_arrays", "host numpy (this package)", t3))
        same = all(np.array_equal(getattr(m, f), getattr(m2, f))
                   for f in ("elements", "adj_elem", "adj_face", "volumes", "centroids"))
        if ref is not None:
            r, t4 = timed(lambda: ref.read_tetmesh(path))
            rows.append(("read_tetmesh", "reference (baseline/_ref, numpy)", t4))
            same = same and all(np.array_equal(getattr(m, f), getattr(r, f))
                                for f in ("elements", "adj_elem", "adj_face", "volumes",
                                          "centroids"))
            del r
        for op, impl, t in rows:
            d = {"mesh": label, "tets": int(e.shape[0]), "vertices": int(v.shape[0]),
                 "file_mb": round(mb, 1), "op": op, "impl": impl, "seconds": round(t, 3),
                 "identical_arrays": bool(same)}
            print(json.dumps(d), flush=True)
            res.append(d)
        path.unlink()
        del m, m2
    if args.out:
        Path(args.out).write_text("".join(json.dumps(d) + "\n" for d in res))


if __name__ == "__main__":
    main()
