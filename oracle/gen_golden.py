"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the reference
package is importable from /root/reference/pkg/src (numba 0.65.0,
numpy 2.3.5).  /root/reference does not exist on the GPU box:
the fixtures are committed so that tests there never need it.

Every walk case is driven through the reference's own drop-in API
(``meshtally.MeshTally``, tally.py:203-286) for states, tallies and
``TraceSummary``; a second pass through ``trace_batch(callback=...)``
(search.py:453-489) on identical inputs records the per-particle
(element, exit_face) sequences, and the script asserts that both passes end in
bitwise-identical states and tallies before writing anything.

Sequence digest (shared with the C oracle and the CUDA kernel):
  h = 0xcbf29ce484222325; for each scored event:
      h = (h ^ (element*8 + exit_face + 1)) * 0x100000001b3   (mod 2^64)
with exit_face = -1 for the final in-element segment.

Usage:  python oracle/gen_golden.py        (writes tests/golden/*.npz)
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import meshtally as mt                                   # noqa: E402
from meshtally import search as mts                      # noqa: E402
from meshtally import particles as mtp                   # noqa: E402
from meshtally import tally as mtt                       # noqa: E402
from meshtally import geometry as mtg                    # noqa: E402

from paper_2504_19048_b200 import synth                 # noqa: E402
from paper_2504_19048_b200 import mesh as mymesh         # noqa: E402

OUT = REPO / "tests" / "golden"
H0 = np.uint64(0xCBF29CE484222325)
HP = np.uint64(0x100000001B3)


# ----------------------------------------------------------------------------
# meshes

def ref_mesh(kind: str, params: dict):
    if kind == "cube":
        return mt.build_cube_mesh(int(params["n"]))
    if kind == "torus":
        v, e = mymesh.torus_shell_arrays(**params)
        return mt.TetMesh.from_arrays(v, e)
    raise ValueError(kind)


# ----------------------------------------------------------------------------
# recording pass (trace_batch + callback)

class Recorder:
    def __init__(self, n):
        self.h = np.full(n, H0, dtype=np.uint64)
        self.count = np.zeros(n, dtype=np.int64)
        self.seq = None

    def keep_sequences(self, n):
        self.seq = [[] for _ in range(n)]

    def __call__(self, ev):
        p = np.asarray(ev.particle, dtype=np.int64)
        code = (np.asarray(ev.element, dtype=np.int64) * 8
                + np.asarray(ev.exit_face, dtype=np.int64) + 1).astype(np.uint64)
        with np.errstate(over="ignore"):
            self.h[p] = (self.h[p] ^ code) * HP
        self.count[p] += 1
        if self.seq is not None:
            for pi, c in zip(p.tolist(), code.tolist()):
                self.seq[pi].append(c)


def state_of(batch, ws, count):
    return dict(
        position=np.array(batch.position[:count]),
        element=np.array(batch.element[:count]),
        alive=np.array(batch.alive[:count]),
        flying=np.array(batch.flying[:count]),
        entry_face=np.array(ws.entry_face[:count]),
        stuck=np.array(ws.stuck[:count]),
        outcome=np.array(ws.outcome[:count]),
        seg_total=np.array(ws.seg_total[:count]),
    )


def summary_tuple(s):
    return np.array([s.sweeps, s.events, s.reached, s.boundary_exits,
                     s.stuck_recoveries, s.stuck_terminations], dtype=np.int64)


# ----------------------------------------------------------------------------
# one walk case

def run_case(name, kind, params, num_groups, batches, keep_seq=False):
    """batches: list of dicts {init: (n,3), moves: [callable(state)->(dest, fly, w, groups)]}"""
    mesh = ref_mesh(kind, params)
    n = max(b["init"].shape[0] for b in batches)
    tal = mt.MeshTally(mesh, n, num_groups=num_groups, threads=1)
    # recording twin (same reference code, callback path)
    batch2 = mtp.create_batch(n)
    ws2 = mts.create_workspace(n)
    grid2 = mtt.create_grid(mesh.num_elements, num_groups, 1)

    out = {"mesh_kind": np.array(kind), "num_groups": np.array(num_groups),
           "capacity": np.array(n), "num_batches": np.array(len(batches))}
    for k, v in params.items():
        out[f"mesh_{k}"] = np.array(v)
    for bi, b in enumerate(batches):
        init = np.ascontiguousarray(b["init"], dtype=np.float64)
        cnt = init.shape[0]
        tal.initialize_particle_location(init.reshape(-1))
        mts.initialize_locations(mesh, batch2, init.reshape(-1), cnt, ws2)
        st = state_of(tal._batch, tal._ws, cnt)
        st2 = state_of(batch2, ws2, cnt)
        for key in st:
            assert np.array_equal(st[key], st2[key], equal_nan=True), (name, key)
        pre = f"b{bi}_"
        out[pre + "init_positions"] = init
        out[pre + "init_element"] = st["element"]
        out[pre + "init_alive"] = st["alive"]
        out[pre + "num_moves"] = np.array(len(b["moves"]))
        for mi, mover in enumerate(b["moves"]):
            dest, fly, w, groups = mover(st)
            dest = np.ascontiguousarray(dest, dtype=np.float64)
            fly = np.ascontiguousarray(fly, dtype=np.int8)
            w = np.ascontiguousarray(w, dtype=np.float64)
            seg_before = st["seg_total"].copy()
            summ = tal.move_to_next_location(dest.reshape(-1), fly, w, groups)
            # twin: load_step + groups + trace_batch(callback, grid)
            mtp.load_step(batch2, dest.reshape(-1), fly, w, fly.size)
            if groups is not None:
                batch2.group[:fly.size] = np.asarray(groups, dtype=np.int32)
            rec = Recorder(n)
            if keep_seq:
                rec.keep_sequences(n)
            summ2 = mts.trace_batch(mesh, batch2, callback=rec, workspace=ws2, grid=grid2)
            st = state_of(tal._batch, tal._ws, cnt)
            st2 = state_of(batch2, ws2, cnt)
            for key in st:
                assert np.array_equal(st[key], st2[key], equal_nan=True), (name, bi, mi, key)
            tot = mtt.batch_totals(tal.grid).reshape(-1)
            tot2 = mtt.batch_totals(grid2).reshape(-1)
            assert np.array_equal(tot, tot2), (name, bi, mi, "tally")
            s1 = summary_tuple(summ)
            s2 = summary_tuple(summ2)
            # trace_batch recompacts every sweep; sweeps/events/reached/... agree
            assert np.array_equal(s1, s2), (name, s1, s2)
            pm = f"{pre}m{mi}_"
            out[pm + "dest"] = dest
            out[pm + "flying_in"] = fly
            out[pm + "weights"] = w
            if groups is not None:
                out[pm + "groups"] = np.asarray(groups, dtype=np.int32)
            for key in ("position", "element", "alive", "flying", "entry_face",
                        "stuck", "outcome"):
                out[pm + key] = st[key]
            out[pm + "seg_delta"] = st["seg_total"] - seg_before
            out[pm + "count"] = rec.count[:cnt]
            out[pm + "digest"] = rec.h[:cnt]
            out[pm + "summary"] = s1
            print(f"  {name} b{bi} m{mi}: summary {s1.tolist()}")
            out[pm + "tally"] = tot
            if keep_seq:
                flat = np.concatenate([np.asarray(s, dtype=np.uint64) for s in rec.seq[:cnt]]
                                      ) if rec.count[:cnt].sum() else np.zeros(0, np.uint64)
                out[pm + "seq_codes"] = flat
        sw = b.get("source_weight")
        mtt.finalize_batch(grid2, sw if sw is not None else tal._batch_source_weight)
        out[pre + "source_weight"] = np.array(tal._batch_source_weight)
        tal.finalize_batch(sw)
        out[pre + "sum"] = np.array(tal.grid.sum)
        out[pre + "sum_sq"] = np.array(tal.grid.sum_sq)
    fl = tal.flux()
    out["flux_mean"] = fl.mean
    out["flux_rel"] = fl.rel_error
    path = OUT / f"walk_{name}.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}  ({path.stat().st_size/1e3:.0f} kB)")


def chain_mover(gen, sigma_t, weights="ones", groups=None, all_fly=False):
    def mover(st):
        pos = st["position"]
        n = pos.shape[0]
        dest = synth.flight_destinations(gen, pos, sigma_t)
        fly = np.ones(n, np.int8) if all_fly else st["alive"].astype(np.int8)
        if weights == "ones":
            w = np.ones(n)
        else:
            w = 0.5 + gen.random(n)
        g = None if groups is None else gen.integers(0, groups, n).astype(np.int32)
        return dest, fly, w, g
    return mover


# ----------------------------------------------------------------------------

def geometry_kats():
    """Bit-exact scalar KATs from the reference's own numba cores."""
    gen = np.random.default_rng(7)
    out = {}
    # SPEC examples
    ref = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    out["spec_bary"] = mt.barycentric_coords(ref, [0.1, 0.2, 0.3])
    # random tets (perturbed reference tet) and points
    n = 2000
    tets = ref[None] + 0.3 * gen.standard_normal((n, 4, 3))
    pts = 0.25 + 0.4 * gen.standard_normal((n, 3))
    bary = np.array([mtg._bary_arr(tets[i], pts[i]) for i in range(n)])
    out["bary_tets"], out["bary_pts"], out["bary_out"] = tets, pts, bary
    faces = tets[:, :3]
    orig = pts
    seg = gen.standard_normal((n, 3))
    fh = np.array([mtg._face_hit_arr(faces[i], orig[i], seg[i]) for i in range(n)])
    out["fh_faces"], out["fh_orig"], out["fh_seg"], out["fh_t"] = faces, orig, seg, fh
    # find_exit_face on cube(3) elements
    m = mt.build_cube_mesh(3)
    ne = m.num_elements
    elem = gen.integers(0, ne, n)
    o = m.centroids[elem]
    d = o + 0.6 * gen.standard_normal((n, 3))
    ent = gen.integers(-1, 4, n)
    res = np.array([mtg.exit_search_core(m.kernel_data(), int(elem[i]), *o[i], *d[i], int(ent[i]))
                    for i in range(n)], dtype=np.float64)
    out["xs_elem"], out["xs_orig"], out["xs_dest"], out["xs_entry"] = elem, o, d, ent
    out["xs_out"] = res
    path = OUT / "geometry_kat.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


def mesh_fixtures():
    out = {}
    for n in (1, 2, 3, 4, 10):
        m = mt.build_cube_mesh(n)
        for f in ("vertices", "elements", "adj_elem", "adj_face", "volumes",
                  "centroids", "bounding_box"):
            out[f"cube{n}_{f}"] = getattr(m, f)
    v, e = mymesh.torus_shell_arrays(2, 8, 12)
    m = mt.TetMesh.from_arrays(v, e)
    out["torus_raw_vertices"], out["torus_raw_elements"] = v, e
    for f in ("vertices", "elements", "adj_elem", "adj_face", "volumes",
              "centroids", "bounding_box"):
        out[f"torus_{f}"] = getattr(m, f)
    path = OUT / "mesh_ref.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path}")


def localization_fixture():
    """Reference localization on pathological points (it loses some)."""
    m = mt.build_cube_mesh(10)
    gen = np.random.default_rng(11)
    n = 600
    # 1) generic points, 2) points on x - 2y + z = 0, 3) interior vertices,
    # 4) grid-plane points, 5) outside the bbox
    gpts = synth.uniform_box(gen, n)
    x = gen.uniform(0.1, 0.9, n)
    z = gen.uniform(0.1, 0.9, n)
    plane = np.stack([x, (x + z) / 2.0, z], axis=1)
    verts = m.vertices[(m.vertices > 0).all(1) & (m.vertices < 1).all(1)][:n]
    gp = synth.uniform_box(gen, n)
    gp[:, 1] = m.vertices[gen.integers(0, 11, n) * 11, 1]  # exact grid-plane y
    outside = synth.uniform_box(gen, n, -0.5, 1.5)
    outside[:, 0] = np.where(outside[:, 0] < 0.5, -0.25, 1.25)
    pts = np.concatenate([gpts, plane, verts, gp, outside])
    tal = mt.MeshTally(m, pts.shape[0])
    tal.initialize_particle_location(pts.reshape(-1))
    st = state_of(tal._batch, tal._ws, pts.shape[0])
    path = OUT / "localize_ref.npz"
    np.savez_compressed(path, points=pts, element=st["element"], alive=st["alive"],
                        position=st["position"], outcome=st["outcome"],
                        groups=np.array([n, n, verts.shape[0], n, n]))
    print(f"wrote {path}")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    mesh_fixtures()
    geometry_kats()
    localization_fixture()

    S = synth.POINT_SOURCE
    gen = synth.rng()
    # C1: n=10, 1e4 particles, point source, sigma_t=2, 3-move chain, 2 batches
    run_case("c1_point_s2", "cube", {"n": 10}, 1, [
        {"init": synth.point_source(10000, S),
         "moves": [chain_mover(gen, 2.0) for _ in range(3)]},
        {"init": synth.point_source(10000, S),
         "moves": [chain_mover(gen, 2.0) for _ in range(2)]},
    ])
    # C1 paper physics: sigma_t = 100, 10 moves, random weights, 2 batches
    gen = synth.rng(synth.SEED + 1)
    run_case("c1_point_s100", "cube", {"n": 10}, 1, [
        {"init": synth.point_source(4000, S),
         "moves": [chain_mover(gen, 100.0, weights="rand") for _ in range(5)]},
        {"init": synth.point_source(4000, S),
         "moves": [chain_mover(gen, 100.0, weights="rand") for _ in range(5)]},
    ])
    # random starts, 3 energy groups, n=6; full sequences kept
    gen = synth.rng(synth.SEED + 2)
    run_case("n6_uniform_g3", "cube", {"n": 6}, 3, [
        {"init": synth.uniform_box(gen, 3000),
         "moves": [chain_mover(gen, 2.0, weights="rand", groups=3) for _ in range(2)]},
        {"init": synth.uniform_box(gen, 2500),
         "moves": [chain_mover(gen, 2.0, weights="rand", groups=3, all_fly=True)
                   for _ in range(2)]},
    ], keep_seq=True)

    # SPEC.md:235 straight ray through Kuhn face planes (exercises the stuck ladder)
    def ray_mover(st):
        return np.array([[0.95, 0.05, 0.05]]), np.ones(1, np.int8), np.ones(1), None
    run_case("straight_ray", "cube", {"n": 10}, 1, [
        {"init": np.array([[0.05, 0.05, 0.05]]), "moves": [ray_mover]}], keep_seq=True)

    # in-plane moves on an exact grid plane: many stuck-ladder events
    gen = synth.rng(synth.SEED + 3)
    m10 = mt.build_cube_mesh(10)
    zplane = m10.vertices[3, 2]     # exact vertex coordinate 3*h

    def plane_pts(k):
        p = synth.uniform_box(gen, k, 0.08, 0.92)
        p[:, 2] = zplane
        return p

    def plane_mover(st):
        k = st["position"].shape[0]
        d = plane_pts(k)
        return d, st["alive"].astype(np.int8), np.ones(k), None
    run_case("grid_plane_ladder", "cube", {"n": 10}, 1, [
        {"init": plane_pts(2000), "moves": [plane_mover, plane_mover]}], keep_seq=True)

    # non-convex toroidal shell: leaks into the hole, long walks
    gen = synth.rng(synth.SEED + 4)
    tp = dict(nr=2, ntheta=8, nphi=12, R=300.0, a_in=100.0, a_out=120.0)
    tm = mymesh.build_torus_shell_mesh(**tp)
    # fixed source in one shell sector: cells with theta index 0, phi index < 2
    cells = np.array([(i * 8 + 0) * 12 + k for i in range(2) for k in range(2)])
    sector = (cells[:, None] * 6 + np.arange(6)[None]).ravel()
    src_elems = sector[gen.integers(0, sector.size, 3000)]
    run_case("torus_small", "torus", tp, 2, [
        {"init": synth.points_in_elements(gen, tm.vertices, tm.elements, src_elems),
         "moves": [chain_mover(gen, 0.02, weights="rand", groups=2) for _ in range(3)]},
    ])


if __name__ == "__main__" and not {"--transport", "--callback"} & set(sys.argv):
    main()


# ----------------------------------------------------------------------------
# transport: philox KATs and small reference runs

def transport_fixtures():
    from meshtally import rng as mtr
    from meshtally import transport as mtt2
    out = {}
    # raw philox4x64-10 words (rng.py:38-49) and (0,1] uniforms (rng.py:52-64)
    ctrs = [(0, 0, 0, 0), (1, 2, 3, 4), (2**63 - 1, 5, 7, 0), (123456789, 42, 3, 0)]
    keys = [(0, 0), (42, 2**62 + 5), (2**62, 99), (7, 7)]  # raw_block rejects words >= 2^63
    raw = np.array([mtr.raw_block(c, k) for c in ctrs for k in keys], dtype=np.uint64)
    out["philox_ctr"] = np.array([c for c in ctrs for _ in keys], dtype=np.uint64)
    out["philox_key"] = np.array([k for _ in ctrs for k in keys], dtype=np.uint64)
    out["philox_out"] = raw
    gen = np.random.default_rng(3)
    q = gen.integers(0, 2**31, (500, 4))
    out["uni_key"] = q.astype(np.int64)
    out["uni_out"] = np.array([mtr._uniform_block_arr(int(a), int(b), int(c), int(d))
                               for a, b, c, d in q])
    cases = {
        "t1g": mtt2.RunConfig(mesh_n=4, num_particles=3000, num_batches=3,
                              cross_sections=mtt2.CrossSections.one_group(10.0, 8.0),
                              seed=42),
        "t2g": mtt2.RunConfig(mesh_n=5, num_particles=2000, num_batches=2,
                              cross_sections=mtt2.CrossSections(
                                  np.array([5.0, 8.0]), np.array([[2.0, 2.5], [0.5, 6.0]])),
                              seed=7, source_box=((0.1, 0.2, 0.3), (0.6, 0.5, 0.9))),
        "tdir": mtt2.RunConfig(mesh_n=3, num_particles=1500, num_batches=2,
                               cross_sections=mtt2.CrossSections.one_group(3.0, 2.0),
                               seed=11, source_direction=(1.0, 0.5, 0.25)),
    }
    for name, cfg in cases.items():
        mesh = mt.build_cube_mesh(cfg.mesh_n, cfg.edge_length)
        eng = mtt2.build_engine(cfg, mesh)
        res = mtt2.run(cfg, engine=eng)
        n = cfg.num_particles
        pre = f"{name}_"
        xs = cfg.cross_sections
        out[pre + "cfg"] = np.array([cfg.mesh_n, cfg.num_particles, cfg.num_batches, cfg.seed],
                                    dtype=np.int64)
        out[pre + "sigma_t"] = xs.sigma_t
        out[pre + "sigma_s"] = xs.sigma_s
        out[pre + "box"] = np.array(cfg.source_box, dtype=np.float64)
        out[pre + "dir"] = (np.array(cfg.source_direction) if cfg.source_direction is not None
                            else np.zeros(0))
        for key in ("source_weight", "leaked_weight", "absorbed_weight", "stuck_weight",
                    "collisions", "events", "sweeps", "track_length_total"):
            out[pre + key] = np.array(getattr(res, key))
        out[pre + "flux_track_mean"] = res.flux_track.mean
        out[pre + "flux_track_rel"] = res.flux_track.rel_error
        out[pre + "flux_col_mean"] = res.flux_collision.mean
        out[pre + "flux_col_rel"] = res.flux_collision.rel_error
        b, ws = eng.batch, eng.workspace
        out[pre + "final_position"] = np.array(b.position[:n])
        out[pre + "final_direction"] = np.array(b.direction[:n])
        out[pre + "final_element"] = np.array(b.element[:n])
        out[pre + "final_group"] = np.array(b.group[:n])
        out[pre + "final_alive"] = np.array(b.alive[:n])
        out[pre + "final_outcome"] = np.array(ws.outcome[:n])
        out[pre + "final_rng_block"] = np.array(ws.rng_block[:n])
        out[pre + "final_seg_total"] = np.array(ws.seg_total[:n])
        print(f"  transport {name}: collisions {res.collisions} events {res.events} "
              f"leaked {res.leaked_weight} absorbed {res.absorbed_weight} stuck {res.stuck_weight}")
    path = OUT / "transport_ref.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size/1e3:.0f} kB)")


if __name__ == "__main__" and "--transport" in sys.argv:
    OUT.mkdir(parents=True, exist_ok=True)
    transport_fixtures()


# ----------------------------------------------------------------------------
# Listing-1 callback path: trace_batch with a callback that
# records every event and modifies decisions deterministically

def callback_decisions(sweep, particle, element, exit_face, next_element, particle_done):
    """Deterministic redirect / kill / resurrect rule applied in place
    (shared verbatim by the GPU parity test)."""
    pid = np.asarray(particle, dtype=np.int64)
    face = np.asarray(exit_face)
    interior = (face >= 0) & (np.asarray(next_element) >= 0)
    kill = interior & ((pid + sweep) % 13 == 0)
    particle_done[kill] = 1
    stay = interior & ~kill & (pid % 17 == 3) & (sweep % 3 == 1)
    next_element[stay] = -1
    boundary = (face >= 0) & (np.asarray(next_element) < 0) & (np.asarray(particle_done) != 0)
    revive = boundary & (pid % 5 == 0) & (sweep == 2)
    particle_done[revive] = 0
    jump = interior & ~kill & ~stay & (pid % 23 == 7)
    next_element[jump] = np.asarray(element)[jump]   # "redirect" into the same element


def callback_fixtures():
    out = {}
    cases = [("cb_n6", 6, 2500, 11, True), ("cb_plane", 10, 1500, 12, False)]
    for name, n, k, seed, modify in cases:
        mesh = mt.build_cube_mesh(n)
        gen = np.random.default_rng(seed)
        if name == "cb_plane":
            z = mesh.vertices[3, 2]
            pos = synth.uniform_box(gen, k, 0.08, 0.92)
            pos[:, 2] = z
            dest = synth.uniform_box(gen, k, 0.08, 0.92)
            dest[:, 2] = z
        else:
            pos = synth.uniform_box(gen, k)
            dest = synth.flight_destinations(gen, pos, 2.0)
        w = 0.5 + gen.random(k)
        groups = gen.integers(0, 2, k).astype(np.int32)
        fly = (gen.random(k) < 0.9).astype(np.int8)
        batch = mtp.create_batch(k)
        ws = mts.create_workspace(k)
        grid = mtt.create_grid(mesh.num_elements, 2, 1)
        mts.initialize_locations(mesh, batch, pos.reshape(-1), k, ws)
        mtp.load_step(batch, dest.reshape(-1), fly, w, k)
        batch.group[:k] = groups
        h = np.full(k, H0, dtype=np.uint64)
        cnt = np.zeros(k, np.int64)
        counts = []
        state = {"sweep": 0}

        def cb(ev):
            p = np.asarray(ev.particle, dtype=np.int64)
            code = (np.asarray(ev.element, dtype=np.int64) * 8
                    + np.asarray(ev.exit_face, dtype=np.int64) + 1).astype(np.uint64)
            with np.errstate(over="ignore"):
                h[p] = (h[p] ^ code) * HP
            cnt[p] += 1
            counts.append(len(ev))
            if modify:
                callback_decisions(state["sweep"], ev.particle, ev.element, ev.exit_face,
                                   ev.next_element, ev.particle_done)
            state["sweep"] += 1
        s = mts.trace_batch(mesh, batch, callback=cb, workspace=ws, grid=grid)
        pre = name + "_"
        out[pre + "mesh_n"] = np.array(n)
        out[pre + "modify"] = np.array(modify)
        out[pre + "pos"], out[pre + "dest"], out[pre + "w"] = pos, dest, w
        out[pre + "groups"], out[pre + "fly"] = groups, fly
        out[pre + "summary"] = summary_tuple(s)
        out[pre + "sweep_counts"] = np.array(counts, np.int64)
        out[pre + "digest"], out[pre + "count"] = h, cnt
        st = state_of(batch, ws, k)
        for key in ("position", "element", "alive", "flying", "entry_face", "stuck", "outcome",
                    "seg_total"):
            out[pre + key] = st[key]
        out[pre + "tally"] = mtt.batch_totals(grid).reshape(-1)
        print(f"  callback {name}: summary {out[pre + 'summary'].tolist()} sweeps {len(counts)}")
    path = OUT / "callback_ref.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size/1e3:.0f} kB)")


if __name__ == "__main__" and "--callback" in sys.argv:
    OUT.mkdir(parents=True, exist_ok=True)
    callback_fixtures()
