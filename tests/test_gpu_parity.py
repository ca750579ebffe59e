"""CUDA path (libb200tally.so through the MeshTally facade / C ABI) vs the
reference's golden outputs and the CPU oracle.

Bars (BASELINE.json north_star): element sequences, exit faces, positions,
outcomes, flags and event counts BIT-EXACT; per-bin tallies within 1e-9
relative (fp64 atomics reorder the sums).
"""

import numpy as np
import pytest

import oracle as orc
from golden_cases import GOLDEN, STATE_KEYS, WALK_CASES, load_walk_case, rel_close
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh, synth

pytestmark = pytest.mark.gpu

TALLY_RTOL = 1e-9


def _run(case, localize, **kw):
    mt = MeshTally(case.mesh, case.capacity, case.num_groups, localize=localize,
                   digest=True, **kw)
    for b in case.batches:
        mt.initialize_particle_location(b.init_positions)
        n = b.init_positions.shape[0]
        st = mt.read_particles(n)
        yield "init", mt, b, None, None, st
        for mv in b.moves:
            seg0 = st.seg_total.copy()
            s = mt.move_to_next_location(mv.dest, mv.flying, mv.weights, mv.groups)
            st = mt.read_particles(n)
            yield "move", mt, b, mv, s, (st, st.seg_total - seg0)
        yield "finalize", mt, b, None, None, None
        mt.finalize_batch()


def _check_case(case, localize, **kw):
    for kind, mt, b, mv, s, st in _run(case, localize, **kw):
        if kind == "init":
            if localize == "walk" or case.name != "torus_small":
                assert np.array_equal(st.element, b.init_element)
                assert np.array_equal(st.alive, b.init_alive)
        elif kind == "move":
            st, seg = st
            e = mv.expect
            got = np.array([s.sweeps, s.events, s.reached, s.boundary_exits,
                            s.stuck_recoveries, s.stuck_terminations])
            assert np.array_equal(got, e["summary"]), (got, e["summary"])
            for k in STATE_KEYS:
                if k == "flying":
                    assert not e[k].any()
                    continue
                assert np.array_equal(getattr(st, k), e[k]), k
            d, c = mt.read_digest(len(st.element))
            assert np.array_equal(c, e["count"])
            assert np.array_equal(d, e["digest"])
            if localize == "walk":
                assert np.array_equal(seg, e["seg_delta"])
            else:
                # the reference's seg_total also holds the centroid-0 trial walk
                # length L0, so its per-move delta carries the rounding of sums
                # at L0's magnitude: compare absolutely (cm)
                assert np.abs(seg - e["seg_delta"]).max() <= 1e-12
            ok, worst = rel_close(mt.batch_totals().reshape(-1), e["tally"], TALLY_RTOL)
            assert ok, worst
        else:
            pass
    assert rel_close(mt.grid.sum, case.batches[-1].sum, TALLY_RTOL)[0]
    assert rel_close(mt.grid.sum_sq, case.batches[-1].sum_sq, TALLY_RTOL)[0]
    fl = mt.flux()
    assert rel_close(fl.mean, case.flux_mean, TALLY_RTOL)[0]
    fd = mt.flux_device()
    assert rel_close(fd.mean, fl.mean, 1e-15)[0]
    assert np.abs(fd.rel_error - fl.rel_error).max() < 1e-12
    # rel_error cancels catastrophically between near-equal batches; see
    # tests/test_oracle_golden.py
    assert np.abs(fl.rel_error - case.flux_rel).max() < 1e-5
    mt.close()


@pytest.mark.parametrize("name", WALK_CASES)
def test_walk_matches_reference_walk_localize(name):
    _check_case(load_walk_case(name), "walk")


@pytest.mark.parametrize("name", [c for c in WALK_CASES if c != "torus_small"])
def test_walk_matches_reference_grid_localize(name):
    _check_case(load_walk_case(name), "grid")


@pytest.mark.parametrize("name", ["c1_point_s2", "torus_small"])
def test_wide_crossing_records_keep_parity(name, monkeypatch):
    # meshes of >= 2^24 vertices keep the crossing records' vertex-order
    # selectors in a separate array (layout.cuh XRec); force that layout
    monkeypatch.setenv("B200TALLY_WIDE_XREC", "1")
    _check_case(load_walk_case(name), "walk")


@pytest.mark.parametrize("opts", [dict(sort=True), dict(warp_aggregate=True),
                                  dict(staged=False), dict(staged=False, sort=True,
                                                           warp_aggregate=True),
                                  dict(move_chunks=3), dict(move_chunks=16, warp_aggregate=True),
                                  dict(warp_aggregate=False), dict(staged=1), dict(staged=2),
                                  dict(staged=2, sort=True), dict(staged=2, move_chunks=5),
                                  dict(move_chunks=5, stream_move=False)])
def test_walk_options_keep_parity(opts):
    _check_case(load_walk_case("c1_point_s2"), "grid", **opts)
    _check_case(load_walk_case("n6_uniform_g3"), "grid", **opts)


@pytest.mark.parametrize("lanes", [0, 1, 2, 4, 8, 16, 32])
def test_localize_pathologies(lanes):
    d = np.load(GOLDEN / "localize_ref.npz")
    m = build_cube_mesh(10)
    pts = d["points"]
    mt = MeshTally(m, pts.shape[0], localize="walk")
    mt.initialize_particle_location(pts)
    st = mt.read_particles()
    # walk mode reproduces the reference bit for bit, lost points included
    assert np.array_equal(st.element, d["element"])
    assert np.array_equal(st.alive, d["alive"])
    assert np.array_equal(st.outcome, d["outcome"])
    assert np.array_equal(st.position, d["position"])
    # grid mode: lowest-id containing element everywhere (finds what the walk loses),
    # for every lane-group width of the warp-parallel search
    mt.set_option(_lib.BT_OPT_LOCATE_LANES, lanes)
    mt.initialize_particle_location(pts, mode="grid")
    st = mt.read_particles()
    low = orc.locate_exhaustive(m, pts)
    assert np.array_equal(st.element, low)
    assert np.array_equal(st.alive, (low >= 0).astype(np.int8))
    found = low >= 0
    assert np.array_equal(st.position[found], pts[found])


@pytest.mark.parametrize("lanes", [1, 4, 8, 32])
def test_grid_localize_random_meshes(lanes):
    gen = np.random.default_rng(5)
    for n in (1, 3, 7, 16):
        m = build_cube_mesh(n)
        pts = gen.uniform(-0.1, 1.1, (5003, 3))
        mt = MeshTally(m, pts.shape[0])
        mt.set_option(_lib.BT_OPT_LOCATE_LANES, lanes)
        mt.initialize_particle_location(pts)
        st = mt.read_particles()
        assert np.array_equal(st.element, orc.locate_exhaustive(m, pts))
        found = st.element >= 0
        assert np.array_equal(st.position[found], pts[found])
    with pytest.raises(ValueError):
        mt.set_option(_lib.BT_OPT_LOCATE_LANES, 3)


@pytest.mark.parametrize("scale,offset", [(1.0, 0.0), (1e-2, 1e4), (1e3, -5e5)])
def test_grid_localize_boundary_points(scale, offset):
    """Points on mesh vertices, edges, faces and within 1e-11 (relative) of
    them, on scaled/translated cubes and the torus shell: the fp32 barycentric
    pre-filter must hand every borderline candidate to the exact test."""
    from paper_2504_19048_b200 import TetMesh, build_torus_shell_mesh
    gen = np.random.default_rng(17)
    m0 = build_cube_mesh(7)
    meshes = [TetMesh.from_arrays(m0.vertices * scale + offset, m0.elements)]
    if scale == 1.0:
        meshes.append(build_torus_shell_mesh(2, 8, 12))
    for m in meshes:
        V, E = m.vertices, m.elements
        k = 6000
        el = gen.integers(0, E.shape[0], k)
        bc = gen.dirichlet(np.ones(4), k)
        kind = gen.integers(0, 4, k)          # 0 vertex, 1 edge, 2 face, 3 interior
        bc[kind == 0] = np.eye(4)[gen.integers(0, 4, (kind == 0).sum())]
        for sel, nz in ((kind == 1, 2), (kind == 2, 3)):
            idx = np.where(sel)[0]
            for i in idx:
                keep = gen.choice(4, nz, replace=False)
                b = np.zeros(4)
                b[keep] = gen.dirichlet(np.ones(nz))
                bc[i] = b
        pts = np.einsum("ij,ijk->ik", bc, V[E[el]])
        near = gen.random(k) < 0.3
        span = np.ptp(V, axis=0).max()
        pts[near] += gen.normal(size=(near.sum(), 3)) * 1e-11 * span
        mt = MeshTally(m, k)
        mt.initialize_particle_location(pts)
        st = mt.read_particles()
        # points outside the (inclusive) bounding box are not searched by the
        # reference (search.py:574-583), even when within EPS_BARY of a face
        bb = m.bounding_box
        inside = ((pts >= bb[0]) & (pts <= bb[1])).all(axis=1)
        assert (~inside).any()  # the set does probe that rule
        expect = np.where(inside, orc.locate_exhaustive(m, pts), -1)
        assert np.array_equal(st.element, expect)
        mt.close()


@pytest.mark.parametrize("sigma_t", [2.0, 100.0])
def test_full_size_c2_against_oracle(sigma_t):
    """C2 mesh (998,250 tets); 2e5 particles checked exhaustively against the
    multi-threaded oracle: digests, states bit-exact; tallies <= 1e-9."""
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 10)
    n = 200_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, sigma_t)
    w = 0.5 + gen.random(n)
    fly = np.ones(n, np.int8)
    mt = MeshTally(m, n, digest=True, sort=True)
    mt.initialize_particle_location(pos)
    st0 = mt.read_particles()
    s = mt.move_to_next_location(dest, fly, w)
    st = mt.read_particles()
    ref = orc.OracleTally(m, n, threads=orc.max_threads())
    ref.initialize_particle_location(pos)
    assert np.array_equal(st0.element, ref.element)
    ref.seg_total[:] = 0.0  # grid localization has no trial-walk length
    r = ref.move_to_next_location(dest, fly, w)
    assert tuple(r) == (s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                        s.stuck_terminations)
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st, k), getattr(ref, k)[:n]), k
    d, c = mt.read_digest()
    assert np.array_equal(d, ref.digest) and np.array_equal(c, ref.count)
    ok, worst = rel_close(mt.batch_totals().reshape(-1), ref.batch_totals(), TALLY_RTOL)
    assert ok, worst
    # size-independent property: path-length conservation
    tot = mt.batch_totals().sum()
    assert abs(tot - float((w * st.seg_total).sum())) <= 1e-9 * tot


@pytest.mark.parametrize("digest", [True, False])
@pytest.mark.parametrize("sigma_t", [2.0, 100.0])
def test_point_source_c2_against_oracle(sigma_t, digest):
    """C2 mesh, 2e5 particles from one point (SURVEY §8d's clean source S):
    every lane starts in the same element, so the tally atomics collide and
    the adaptive warp aggregation (walk.cuh flush_pending) takes over -- at
    Σt = 100 for most of the walk.  States and digests bit-exact against the
    oracle, tally within 1e-9."""
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 47)
    n = 200_000
    pos = synth.point_source(n)
    dest = synth.flight_destinations(gen, pos, sigma_t)
    w = 0.5 + gen.random(n)
    fly = np.ones(n, np.int8)
    mt = MeshTally(m, n, digest=digest)
    mt.initialize_particle_location(pos)
    s = mt.move_to_next_location(dest, fly, w)
    st = mt.read_particles()
    ref = orc.OracleTally(m, n, threads=orc.max_threads())
    ref.initialize_particle_location(pos)
    ref.seg_total[:] = 0.0
    r = ref.move_to_next_location(dest, fly, w)
    assert tuple(r) == (s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                        s.stuck_terminations)
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st, k), getattr(ref, k)[:n]), k
    if digest:
        d, c = mt.read_digest()
        assert np.array_equal(d, ref.digest) and np.array_equal(c, ref.count)
    ok, worst = rel_close(mt.batch_totals().reshape(-1), ref.batch_totals(), TALLY_RTOL)
    assert ok, worst
    mt.close()


@pytest.mark.parametrize("inputs", ["host", "device"])
def test_multigroup_chained_moves_c2_against_oracle(inputs):
    """C2 mesh, 3 energy groups, 1.5e5 particles with random groups and
    U[0.5, 1.5] weights, two chained moves (the second from where the first
    left every particle, flying = alive, new groups), through the benchmarked
    digest-free kernel: every particle's state bit-exact against the oracle
    and the whole (element, group) tally within 1e-9 -- the bin index
    e*G + g, the group change between moves and the chained start state at
    scale."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 31)
    n, G = 150_000, 3
    pos = synth.uniform_box(gen, n)
    mt = MeshTally(m, n, G)
    ref = orc.OracleTally(m, n, G, threads=orc.max_threads())
    dev = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()) if inputs == "device" \
        else (lambda a: a)
    mt.initialize_particle_location(dev(pos))
    ref.initialize_particle_location(pos)
    ref.seg_total[:] = 0.0
    fly = np.ones(n, np.int8)
    cur = pos
    for k in range(2):
        dest = synth.flight_destinations(gen, cur, 3.0)
        w = 0.5 + gen.random(n)
        g = gen.integers(0, G, n).astype(np.int32)
        s = mt.move_to_next_location(dev(dest), dev(fly), dev(w), dev(g))
        r = ref.move_to_next_location(dest, fly, w, g)
        assert tuple(r) == (s.sweeps, s.events, s.reached, s.boundary_exits,
                            s.stuck_recoveries, s.stuck_terminations), k
        st = mt.read_particles()
        for key in ("position", "element", "alive", "entry_face", "stuck", "outcome",
                    "seg_total"):
            assert np.array_equal(getattr(st, key), getattr(ref, key)[:n]), (k, key)
        cur = st.position.copy()
        fly = st.alive.astype(np.int8)
    ok, worst = rel_close(mt.batch_totals().reshape(-1), ref.batch_totals(), TALLY_RTOL)
    assert ok, worst
    mt.close()


@pytest.mark.parametrize("opts", [{}, dict(sort=True), dict(staged=False),
                                  dict(warp_aggregate=True), dict(warp_aggregate=False),
                                  dict(staged=1), dict(staged=2), dict(staged=2, sort=True)])
def test_device_pointer_path_equals_host_path(opts):
    torch = pytest.importorskip("torch")
    case = load_walk_case("n6_uniform_g3")
    b = case.batches[0]
    mv = b.moves[0]
    host = MeshTally(case.mesh, case.capacity, case.num_groups, digest=True, **opts)
    dev = MeshTally(case.mesh, case.capacity, case.num_groups, digest=True, **opts)
    host.initialize_particle_location(b.init_positions)
    dev.initialize_particle_location(torch.from_numpy(b.init_positions).cuda())
    s1 = host.move_to_next_location(mv.dest, mv.flying, mv.weights, mv.groups)
    s2 = dev.move_to_next_location(torch.from_numpy(mv.dest).cuda(),
                                   torch.from_numpy(mv.flying).cuda(),
                                   torch.from_numpy(mv.weights).cuda(),
                                   torch.from_numpy(mv.groups).cuda())
    assert s1 == s2
    a, c = host.read_particles(), dev.read_particles()
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome"):
        assert np.array_equal(getattr(a, k), getattr(c, k))
    assert rel_close(host.batch_totals(), dev.batch_totals(), TALLY_RTOL)[0]
    assert host.source_weight == pytest.approx(dev.source_weight, rel=1e-14)
    assert dev.source_weight > 0.0  # recorded on every device-input path
    host.finalize_batch()
    dev.finalize_batch()
    assert rel_close(host.grid.sum, dev.grid.sum, TALLY_RTOL)[0]


def test_error_behaviour():
    m = build_cube_mesh(4)
    mt = MeshTally(m, 10)
    with pytest.raises(ValueError):
        mt.initialize_particle_location(np.zeros(33))      # count 11 > capacity
    with pytest.raises(ValueError):
        mt.initialize_particle_location(np.zeros(7))       # not 3*count
    pos = np.full((4, 3), 0.3123)
    mt.initialize_particle_location(pos)
    with pytest.raises(ValueError):
        mt.move_to_next_location(np.zeros(11), np.ones(4), np.ones(4))
    with pytest.raises(IndexError):
        mt.move_to_next_location(pos + 0.1, np.ones(4), np.ones(4), groups=[0, 0, 0, 5])
    assert mt.move_to_next_location(np.zeros(0), np.zeros(0, np.int8), np.zeros(0)) is None
    with pytest.raises(RuntimeError):
        mt.flux()
    with pytest.raises(RuntimeError):
        mt.finalize_batch()
    # unlocalized flying particle: not moved, reported after the move
    mt2 = MeshTally(m, 4)
    mt2.initialize_particle_location(np.array([[0.31, 0.32, 0.33], [2.0, 0, 0]]))
    with pytest.raises(ValueError):
        mt2.move_to_next_location([[0.4, 0.4, 0.4], [0.5, 0.5, 0.5]], [1, 1], [1.0, 1.0])
    st = mt2.read_particles(2)
    assert st.element[1] == -1 and np.array_equal(st.position[0], [0.4, 0.4, 0.4])
    # sweep guard
    mt.set_option(0, 1)
    mt.initialize_particle_location(np.array([[0.05, 0.05, 0.05]]))
    with pytest.raises(RuntimeError):
        mt.move_to_next_location([0.95, 0.95, 0.9], [1], [1.0])
    with pytest.raises(TypeError):
        MeshTally(object(), 4)
    with pytest.raises(ValueError):
        MeshTally(m, 0)


def test_gpu_adjacency_matches_host():
    from paper_2504_19048_b200 import mesh as M
    gen = np.random.default_rng(9)
    for n in (1, 2, 5, 13):
        h = M.build_cube_mesh(n)
        g = M.build_cube_mesh(n, device=0)
        assert np.array_equal(h.adj_elem, g.adj_elem) and np.array_equal(h.adj_face, g.adj_face)
    v, e = M.torus_shell_arrays(3, 16, 24)
    perm = gen.permutation(e.shape[0])
    for els in (e, e[perm]):
        a = M.TetMesh.from_arrays(v, els)
        b = M.TetMesh.from_arrays(v, els, device=0)
        assert np.array_equal(a.adj_elem, b.adj_elem) and np.array_equal(a.adj_face, b.adj_face)
    bad = [np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]]),   # 3 tets on one face
           np.array([[0, 1, 2, 3], [0, 1, 2, 3]]),                 # duplicated element
           np.array([[0, 1, 1, 3]])]                               # repeated vertex id
    for els in bad:
        with pytest.raises(M.MalformedMeshError):
            M.build_adjacency(els, 6, device=0)
        with pytest.raises(M.MalformedMeshError):
            M.build_adjacency(els, 6)


@pytest.mark.parametrize("frac_flying", [1.0, 0.83])
def test_recorded_source_weight_is_numpy_sum(frac_flying):
    """The recorded source weight of a host-input move equals the reference's
    weights[flying].sum() (numpy pairwise order) bit for bit, also when the
    selection and the summation tree run on several host threads."""
    m = build_cube_mesh(6)
    gen = np.random.default_rng(11)
    n = 700_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 20.0)
    fly = (gen.random(n) < frac_flying).astype(np.int8)
    w = 0.5 + gen.random(n)
    mt = MeshTally(m, n)
    mt.initialize_particle_location(pos)
    mt.move_to_next_location(dest, fly, w)
    assert mt.source_weight == w[fly != 0].sum()
    mt.close()


@pytest.mark.parametrize("n,stream_move,pinned", [(5_000_000, True, False), (5_000_000, True, True),
                                                   (5_000_000, False, False), (300_001, True, True)])
def test_pipelined_host_inputs_match_device_inputs(n, stream_move, pinned):
    """Host positions are copied and localized in chunks (>= 4M particles),
    host move inputs are copied in chunks (from 2^18 particles when streamed)
    and walked either by ONE launch that
    waits for each chunk (stream_move, the default, with pinned inputs) or by
    one launch per chunk on two streams (pageable inputs, or stream_move off)
    -- the result must equal the single-launch device-input path bit for
    bit."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(12)
    gen = np.random.default_rng(21)
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 5.0)
    fly = (gen.random(n) < 0.9).astype(np.int8)
    w = 0.5 + gen.random(n)
    host = MeshTally(m, n, stream_move=stream_move)
    dev = MeshTally(m, n)

    def h(x):  # pageable numpy, or a numpy view of pinned host memory
        return torch.from_numpy(x).pin_memory().numpy() if pinned else x
    host.initialize_particle_location(pos)
    dev.initialize_particle_location(torch.from_numpy(pos).cuda())
    # two chained moves: the second one's input buffers on the device still
    # hold the first move's values, so a walk chunk that started before its
    # own inputs landed would show up as a mismatch
    for move in range(2):
        s1 = host.move_to_next_location(h(dest), h(fly), h(w))
        s2 = dev.move_to_next_location(torch.from_numpy(dest).cuda(),
                                       torch.from_numpy(fly).cuda(), torch.from_numpy(w).cuda())
        assert s1 == s2
        a, b = host.read_particles(), dev.read_particles()
        for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (move, k)
        assert rel_close(host.batch_totals(), dev.batch_totals(), TALLY_RTOL)[0]
        assert host.source_weight == w[fly != 0].sum()
        if move == 0:
            dest = synth.flight_destinations(gen, a.position, 5.0)
            fly = a.alive.astype(np.int8)
            w = 0.5 + gen.random(n)
            host.source_weight = dev.source_weight = 0.0  # record the second move too
    host.close()
    dev.close()


@pytest.mark.parametrize("source,sigma_t", [("uniform", 2.0), ("point", 100.0)])
def test_bench_size_sampled_parity(source, sigma_t):
    """The bench workload at full size (C2, 1e7 particles, device inputs): a
    random 20,000-particle sample is replayed on the oracle and must match bit
    for bit (walks are independent per particle), and the size-independent
    properties hold for all 1e7: path-length conservation, reached particles
    sit exactly on their destinations, counters add up."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 77)
    n = 10_000_000
    pos = synth.uniform_box(gen, n) if source == "uniform" else synth.point_source(n)
    dest = synth.flight_destinations(gen, pos, sigma_t)
    w = 0.5 + gen.random(n)
    mt = MeshTally(m, n, digest=True)
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    s = mt.move_to_next_location(torch.from_numpy(dest).cuda(),
                                 torch.ones(n, dtype=torch.int8, device="cuda"),
                                 torch.from_numpy(w).cuda())
    st = mt.read_particles()
    d, c = mt.read_digest()
    assert s.events == int(c.sum())
    assert s.reached + s.boundary_exits + s.stuck_terminations == n
    reached = st.outcome == 1
    assert int(reached.sum()) == s.reached
    assert np.array_equal(st.position[reached], dest[reached])
    tot = mt.batch_totals().sum()
    assert abs(tot - float((w * st.seg_total).sum())) <= 1e-9 * tot
    idx = np.sort(gen.choice(n, 20_000, replace=False))
    ref = orc.OracleTally(m, idx.size, threads=orc.max_threads())
    ref.initialize_particle_location(pos[idx])
    ref.seg_total[:] = 0.0
    ref.move_to_next_location(dest[idx], np.ones(idx.size, np.int8), w[idx])
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st, k)[idx], getattr(ref, k)[:idx.size]), k
    assert np.array_equal(d[idx], ref.digest) and np.array_equal(c[idx], ref.count)
    mt.close()


def test_torus_chained_moves_sampled_parity():
    """Non-convex toroidal shell (C5 family, 8x64x102 cells = 313,344 tets),
    1e6 particles from a shell sector, three chained moves (flying = alive,
    leaked particles stop): a 10,000-particle sample replayed on the oracle
    matches bit for bit after every move."""
    from paper_2504_19048_b200 import build_torus_shell_mesh
    m = build_torus_shell_mesh(8, 64, 102)
    gen = synth.rng(synth.SEED + 5)
    n = 1_000_000
    i = gen.integers(0, 8, n)
    j = gen.integers(0, 8, n)
    k = gen.integers(0, 12, n)
    el = ((i * 64 + j) * 102 + k) * 6 + gen.integers(0, 6, n)
    pos = synth.points_in_elements(gen, m.vertices, m.elements, el)
    idx = np.sort(gen.choice(n, 10_000, replace=False))
    mt = MeshTally(m, n, digest=True)
    mt.initialize_particle_location(pos)
    ref = orc.OracleTally(m, idx.size, threads=orc.max_threads())
    ref.initialize_particle_location(pos[idx])
    st = mt.read_particles()
    found = ref.element[:idx.size] >= 0  # the reference's walk loses points behind the hole
    assert np.array_equal(st.element[idx][found], ref.element[:idx.size][found])
    ref.element[:idx.size] = st.element[idx]  # continue both from the grid's placement
    ref.alive[:idx.size] = st.alive[idx]
    ref.position[:idx.size] = st.position[idx]
    ref.outcome[:idx.size] = st.outcome[idx]
    ref.entry_face[:idx.size] = st.entry_face[idx]  # a lost trial walk leaves its last face
    ref.stuck[:idx.size] = st.stuck[idx]
    ref.seg_total[:] = 0.0
    cur = pos.copy()
    for move in range(3):
        dest = synth.flight_destinations(gen, cur, 1.0 / 30.0)
        fly = st.alive.astype(np.int8)
        w = 0.5 + gen.random(n)
        mt.move_to_next_location(dest, fly, w)
        ref.move_to_next_location(dest[idx], fly[idx], w[idx])
        st = mt.read_particles()
        for key in ("position", "element", "alive", "entry_face", "stuck", "outcome"):
            assert np.array_equal(getattr(st, key)[idx], getattr(ref, key)[:idx.size]), (move, key)
        d, c = mt.read_digest()
        assert np.array_equal(d[idx], ref.digest) and np.array_equal(c[idx], ref.count), move
        cur = st.position
    mt.close()


@pytest.mark.parametrize("mesh_kind", ["cube", "torus"])
def test_filters_equal_literal_arithmetic_at_scale(mesh_kind):
    """The walk with its fp32/fp64 filters against the same walk with every exit
    search in the reference's literal arithmetic (BT_OPT_EXACT_ONLY), on the
    device, for every particle of a bench-size move: ~5.7e8 (cube) exit searches
    must take identical decisions -- digests, positions and flags bit-exact."""
    torch = pytest.importorskip("torch")
    if mesh_kind == "cube":
        m = build_cube_mesh(55)
        gen = synth.rng(synth.SEED + 91)
        n = 10_000_000
        pos = synth.uniform_box(gen, n)
        dest = synth.flight_destinations(gen, pos, 2.0)
    else:
        from paper_2504_19048_b200 import build_torus_shell_mesh
        m = build_torus_shell_mesh(8, 64, 102)
        gen = synth.rng(synth.SEED + 92)
        n = 2_000_000
        el = gen.integers(0, m.num_elements, n)
        pos = synth.points_in_elements(gen, m.vertices, m.elements, el)
        dest = synth.flight_destinations(gen, pos, 1.0 / 30.0)
    res = []
    for exact in (0, 1):
        mt = MeshTally(m, n, digest=True)
        mt.set_option(_lib.BT_OPT_EXACT_ONLY, exact)
        mt.initialize_particle_location(torch.from_numpy(pos).cuda())
        s = mt.move_to_next_location(torch.from_numpy(dest).cuda(),
                                     torch.ones(n, dtype=torch.int8, device="cuda"),
                                     torch.ones(n, dtype=torch.float64, device="cuda"))
        res.append((s, mt.read_particles(), mt.read_digest(), mt.batch_totals()))
        mt.close()
    (s0, st0, (d0, c0), t0), (s1, st1, (d1, c1), t1) = res
    assert s0 == s1
    assert s0.events > 10 * n
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st0, k), getattr(st1, k)), k
    assert np.array_equal(d0, d1) and np.array_equal(c0, c1)
    assert rel_close(t0.reshape(-1), t1.reshape(-1), TALLY_RTOL)[0]


def test_localization_prefilter_equals_exact_at_scale():
    """Grid localization with the fp32 barycentric pre-filter against the same
    search with every candidate tested exactly (BT_OPT_EXACT_ONLY): identical
    elements for 1e7 points on C2, a third of them on grid planes, edges and
    vertices or within 1e-12 of them."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 93)
    n = 10_000_000
    pts = gen.uniform(0.0, 1.0, (n, 3))
    grid = np.arange(56) / 55.0
    for ax in range(3):
        sel = gen.random(n) < 0.2
        pts[sel, ax] = grid[gen.integers(0, 56, sel.sum())]
    near = gen.random(n) < 0.1
    pts[near] += gen.normal(size=(near.sum(), 3)) * 1e-12
    out = []
    for exact in (0, 1):
        mt = MeshTally(m, n)
        mt.set_option(_lib.BT_OPT_EXACT_ONLY, exact)
        mt.initialize_particle_location(torch.from_numpy(pts).cuda())
        out.append(mt.read_particles().element)
        mt.close()
    assert np.array_equal(out[0], out[1])
    assert (out[0] >= 0).mean() > 0.9


@pytest.mark.parametrize("mesh_kind", ["cube", "torus"])
def test_grid_pruning_equals_box_lists_at_scale(mesh_kind, monkeypatch):
    """The localization grid lists an element only in the cells its
    tolerance-expanded barycentric half-spaces reach (csrc/locate.cuh
    elem_cell_overlap).  Against the bounding-box lists
    (B200TALLY_GRID_PRUNE=0): identical elements for every point, a third of
    the cube's points on grid planes, edges and vertices or within 1e-12 of
    them, and the torus's points in curved shell elements."""
    torch = pytest.importorskip("torch")
    gen = synth.rng(synth.SEED + 94)
    if mesh_kind == "cube":
        m = build_cube_mesh(55)
        n = 10_000_000
        pts = gen.uniform(0.0, 1.0, (n, 3))
        grid = np.arange(56) / 55.0
        for ax in range(3):
            sel = gen.random(n) < 0.2
            pts[sel, ax] = grid[gen.integers(0, 56, sel.sum())]
        near = gen.random(n) < 0.1
        pts[near] += gen.normal(size=(near.sum(), 3)) * 1e-12
    else:
        from paper_2504_19048_b200 import build_torus_shell_mesh
        m = build_torus_shell_mesh(4, 64, 96, R=300.0, a_in=100.0, a_out=120.0)
        n = 2_000_000
        elems = gen.integers(0, m.num_elements, n)
        pts = synth.points_in_elements(gen, m.vertices, m.elements, elems)
        onv = gen.random(n) < 0.05  # on mesh vertices
        pts[onv] = m.vertices[m.elements[elems[onv], 0]]
    out = []
    for prune in ("1", "0"):
        monkeypatch.setenv("B200TALLY_GRID_PRUNE", prune)
        mt = MeshTally(m, n)
        mt.initialize_particle_location(torch.from_numpy(pts).cuda())
        out.append(mt.read_particles().element)
        mt.close()
    assert np.array_equal(out[0], out[1])
    assert (out[0] >= 0).mean() > 0.9


def test_permuted_vertex_orders_sampled_parity():
    """The walk keeps a lane's element vertices in shared-memory slots and
    re-maps them through each crossing record's vertex-order selector
    (csrc/layout.cuh XRec).  A mesh whose elements list their vertices in
    random local orders (orientation fixed by from_arrays) exercises every
    selector: the walk must still match the oracle bit for bit."""
    torch = pytest.importorskip("torch")
    from paper_2504_19048_b200 import TetMesh
    base = build_cube_mesh(20)
    gen = np.random.default_rng(4242)
    perm = np.argsort(gen.random((base.num_elements, 4)), axis=1)
    m = TetMesh.from_arrays(base.vertices, np.take_along_axis(base.elements, perm, axis=1))
    n = 400_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 2.0)
    w = 0.5 + gen.random(n)
    mt = MeshTally(m, n, digest=True)
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    s = mt.move_to_next_location(torch.from_numpy(dest).cuda(),
                                 torch.ones(n, dtype=torch.int8, device="cuda"),
                                 torch.from_numpy(w).cuda())
    st = mt.read_particles()
    d, c = mt.read_digest()
    assert s.events == int(c.sum())
    idx = np.sort(gen.choice(n, 20_000, replace=False))
    ref = orc.OracleTally(m, idx.size, threads=orc.max_threads())
    ref.initialize_particle_location(pos[idx])
    ref.seg_total[:] = 0.0
    ref.move_to_next_location(dest[idx], np.ones(idx.size, np.int8), w[idx])
    for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st, k)[idx], getattr(ref, k)[:idx.size]), k
    assert np.array_equal(d[idx], ref.digest) and np.array_equal(c[idx], ref.count)
    mt.close()


@pytest.mark.parametrize("localize", ["grid", "walk"])
def test_ragged_moves_and_edge_inputs(localize):
    """Edge inputs the reference's facade accepts, each move checked against
    the oracle bit for bit: initialization below capacity with points outside
    the mesh (lost, element -1), a move over fewer particles than were
    initialized (ragged count: the rest stay put), mixed flying flags (only
    localized particles fly), an empty move (None), a move where almost
    nothing flies, and a zero-weight particle."""
    m = build_cube_mesh(8)
    gen = np.random.default_rng(99)
    cap, n0 = 1000, 700
    pos = synth.uniform_box(gen, n0)
    pos[650:] = [1.5, 0.5, 0.5] + 0.1 * gen.random((50, 3))  # outside the bbox: lost
    mt = MeshTally(m, cap, digest=True, localize=localize)
    ref = orc.OracleTally(m, cap)
    mt.initialize_particle_location(pos)
    ref.initialize_particle_location(pos)
    st = mt.read_particles(n0)
    assert np.array_equal(st.element, ref.element[:n0])
    assert (st.element[650:] == -1).all()
    ref.seg_total[:] = 0.0

    def check(count, fly, w):
        dest = synth.flight_destinations(gen, ref.position[:count].copy(), 2.0)
        s = mt.move_to_next_location(dest, fly, w)
        e = ref.move_to_next_location(dest, fly, w)
        if count == 0:
            assert s is None and e is None
            return
        assert (s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                s.stuck_terminations) == tuple(e)
        got = mt.read_particles(n0)
        for k in ("position", "element", "alive", "entry_face", "stuck", "outcome"):
            assert np.array_equal(getattr(got, k), getattr(ref, k)[:n0]), k
        d, c = mt.read_digest(n0)
        assert np.array_equal(d[:count], ref.digest[:count])
        assert np.array_equal(c[:count], ref.count[:count])
        ok, worst = rel_close(mt.batch_totals().reshape(-1), ref.batch_totals(), TALLY_RTOL)
        assert ok, worst

    loc = ref.element[:n0] >= 0
    fly = ((gen.random(500) < 0.7) & loc[:500]).astype(np.int8)
    w = 0.5 + gen.random(500)
    w[3] = 0.0
    check(500, fly, w)
    check(0, np.zeros(0, np.int8), np.zeros(0))
    fly = np.zeros(n0, np.int8)
    fly[[5, 17, 400]] = 1
    fly &= loc.astype(np.int8)
    check(n0, fly, np.ones(n0))
    mt.finalize_batch()
    ref.finalize_batch()
    assert rel_close(mt.grid.sum, ref.sum, TALLY_RTOL)[0]
    mt.close()
