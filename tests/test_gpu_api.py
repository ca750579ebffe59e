"""Facade / C-ABI behaviour on the GPU: the recorded source weight of
device-input moves (numpy's pairwise sum, deterministic), argument dtype
checks, the sweep guard's boundary, and the device-side refill choice."""

import numpy as np
import pytest

import oracle as orc
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,frac", [(1, 1.0), (5, 1.0), (7, 0.6), (100, 0.9), (129, 1.0),
                                    (1000, 0.5), (70_001, 0.97), (3_000_000, 0.8),
                                    (3_000_000, 0.0)])
def test_device_source_weight_is_numpy_pairwise_sum(n, frac):
    """tally.py:267-269 records weight[:count][fly.astype(bool)].sum(): the
    device-input path compacts the flying weights and evaluates numpy's
    pairwise summation tree on the device -- the same bits as numpy and as
    the host-input path, on every run."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(6)
    gen = np.random.default_rng(n)
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 50.0)
    fly = (gen.random(n) < frac).astype(np.int8)
    w = gen.random(n) * 10.0 ** gen.integers(-3, 4, n)  # magnitudes that expose the order
    want = w[fly != 0].sum()
    got = []
    for rep in range(2):
        mt = MeshTally(m, n)
        mt.initialize_particle_location(torch.from_numpy(pos).cuda())
        mt.move_to_next_location(torch.from_numpy(dest).cuda(), torch.from_numpy(fly).cuda(),
                                 torch.from_numpy(w).cuda())
        got.append(mt.source_weight)
        mt.close()
    host = MeshTally(m, n)
    host.initialize_particle_location(pos)
    host.move_to_next_location(dest, fly, w)
    assert got[0] == got[1] == host.source_weight == want or (want == 0.0 and got[0] == 0.0)
    host.close()


def test_device_arguments_must_have_the_reference_dtypes():
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(4)
    mt = MeshTally(m, 8)
    pos = torch.full((8, 3), 0.3123, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        mt.initialize_particle_location(pos.to(torch.int64))
    mt.initialize_particle_location(pos)
    d = pos + 0.1
    fly = torch.ones(8, dtype=torch.int8, device="cuda")
    w = torch.ones(8, dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        mt.move_to_next_location(d.to(torch.int64), fly, w)
    with pytest.raises(TypeError):
        mt.move_to_next_location(d, fly, w.to(torch.int64))
    with pytest.raises(TypeError):
        mt.move_to_next_location(d, fly, w, torch.zeros(8, dtype=torch.float32, device="cuda"))
    s = mt.move_to_next_location(d, fly.to(torch.bool), w)
    assert s.reached == 8


@pytest.mark.parametrize("opts", [{}, dict(digest=True), dict(staged=False), dict(staged=1)])
def test_sweep_guard_boundary_matches_reference(opts):
    """search.py:510-516 raises once the sweep count exceeds the limit, even if
    the last particle finished in that sweep: with the limit one below the
    walk's sweep count the move raises, at the sweep count it does not."""
    m = build_cube_mesh(10)
    gen = np.random.default_rng(5)
    n = 2000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 2.0)
    fly = np.ones(n, np.int8)
    w = np.ones(n)
    ref = orc.OracleTally(m, n)
    ref.initialize_particle_location(pos)
    sweeps = ref.move_to_next_location(dest, fly, w).sweeps
    ref2 = orc.OracleTally(m, n)
    ref2.initialize_particle_location(pos)
    with pytest.raises(RuntimeError):
        ref2.move_to_next_location(dest, fly, w, max_sweeps=sweeps - 1)
    for limit, raises in ((sweeps - 1, True), (sweeps, False)):
        mt = MeshTally(m, n, **opts)
        mt.set_option(_lib.BT_OPT_MAX_SWEEPS, limit)
        mt.initialize_particle_location(pos)
        if raises:
            with pytest.raises(RuntimeError):
                mt.move_to_next_location(dest, fly, w)
        else:
            assert mt.move_to_next_location(dest, fly, w).sweeps == sweeps
        mt.close()


def test_device_refill_choice_keeps_parity():
    """Device-input moves choose the refill on the device (direct when at least
    half the slots walk, stage kernel otherwise): a chained move where most
    particles have leaked runs the stage-kernel path, a full move the direct
    one -- both equal the oracle, with one host synchronisation per move."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(12)
    gen = np.random.default_rng(77)
    n = 200_000
    pos = synth.uniform_box(gen, n)
    mt = MeshTally(m, n, digest=True)
    ref = orc.OracleTally(m, n, threads=orc.max_threads())
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    ref.initialize_particle_location(pos)
    ref.seg_total[:] = 0.0
    for frac in (1.0, 0.2, 0.7):
        cur = ref.position[:n].copy()
        dest = synth.flight_destinations(gen, cur, 3.0)
        fly = ((gen.random(n) < frac) & (ref.alive[:n] != 0)).astype(np.int8)
        w = 0.5 + gen.random(n)
        s = mt.move_to_next_location(torch.from_numpy(dest).cuda(),
                                     torch.from_numpy(fly).cuda(), torch.from_numpy(w).cuda())
        r = ref.move_to_next_location(dest, fly, w)
        assert (s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                s.stuck_terminations) == tuple(r)
        st = mt.read_particles()
        for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
            assert np.array_equal(getattr(st, k), getattr(ref, k)[:n]), (frac, k)
        d, c = mt.read_digest()
        assert np.array_equal(d, ref.digest) and np.array_equal(c, ref.count)
    mt.close()


def test_device_group_error_leaves_tally_untouched():
    """A group id out of range on a device-input move raises IndexError before
    any particle moves (the walk launches are gated on the device)."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(6)
    gen = np.random.default_rng(3)
    n = 100_000
    pos = synth.uniform_box(gen, n)
    mt = MeshTally(m, n, num_groups=2)
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    before = mt.read_particles()
    dest = torch.from_numpy(synth.flight_destinations(gen, pos, 5.0)).cuda()
    g = torch.zeros(n, dtype=torch.int32, device="cuda")
    g[n // 2] = 2
    with pytest.raises(IndexError):
        mt.move_to_next_location(dest, torch.ones(n, dtype=torch.int8, device="cuda"),
                                 torch.ones(n, dtype=torch.float64, device="cuda"), g)
    after = mt.read_particles()
    assert np.array_equal(before.position, after.position)
    assert not mt.batch_totals().any()
    assert mt.source_weight == 0.0
    mt.close()


def test_paper_abi_file_constructor_and_vtk_writer(tmp_path):
    """PumiTally(mesh_filename, ...) and write(filename) at the C ABI
    (PAPER.md:265-270): bt_create_from_file + moves + bt_write_vtk /
    bt_write_flux_csv write the same bytes as the Python facade's writers
    (which match the reference's, tests/test_writers.py)."""
    import ctypes as C
    from paper_2504_19048_b200 import mesh as M
    L = _lib.load()
    m = build_cube_mesh(6)
    path = tmp_path / "cube6.tet"
    M.write_tetmesh(m, path)
    gen = np.random.default_rng(12)
    n = 3000
    pos = synth.uniform_box(gen, n)
    h = C.c_void_p()
    _lib.check(L.bt_create_from_file(str(path).encode(), n, 2, 0, C.byref(h)))
    mt = MeshTally(str(path), n, 2)  # the facade reads the file the same way
    s = _lib.Summary()
    for batch in range(2):
        _lib.check(L.bt_initialize_particle_location(h, pos.ctypes.data, pos.size,
                                                     _lib.BT_MEM_HOST, 0, C.byref(s)))
        mt.initialize_particle_location(pos)
        dest = np.ascontiguousarray(synth.flight_destinations(gen, pos, 5.0))
        fly = np.ones(n, np.int8)
        w = np.ascontiguousarray(0.5 + gen.random(n))
        g = np.ascontiguousarray(gen.integers(0, 2, n).astype(np.int32))
        _lib.check(L.bt_move_to_next_location(h, dest.ctypes.data, fly.ctypes.data, w.ctypes.data,
                                              g.ctypes.data, n, _lib.BT_MEM_HOST, C.byref(s)))
        mt.move_to_next_location(dest, fly, w, g)
        _lib.check(L.bt_finalize_batch(h, 0.0))
        mt.finalize_batch()
    # the C writers on the file-made handle vs the Python writers on its moments
    # (volumes of the mesh as read back: the file holds the oriented rows, whose
    # recomputed volumes may differ in the last bit, as in the reference)
    m = M.read_tetmesh(path)
    E, G = m.num_elements, 2
    sm, sq = np.empty(E * G), np.empty(E * G)
    _lib.check(L.bt_read_tally(h, _lib.BT_TALLY_SUM, sm.ctypes.data, E * G))
    _lib.check(L.bt_read_tally(h, _lib.BT_TALLY_SUM_SQ, sq.ctypes.data, E * G))
    from paper_2504_19048_b200 import FluxResult, write_flux_csv, write_vtk
    nb = 2
    bm = sm.reshape(E, G) / nb
    mean = bm / m.volumes[:, None]
    var = np.clip((sq.reshape(E, G) - sm.reshape(E, G) ** 2 / nb) / (nb - 1), 0.0, None)
    rel = np.zeros((E, G))
    nz = bm > 0
    rel[nz] = np.sqrt(var / nb)[nz] / bm[nz]
    fr = FluxResult(mean=mean, rel_error=rel)
    a, b = tmp_path / "c.vtk", tmp_path / "py.vtk"
    _lib.check(L.bt_write_vtk(h, str(a).encode(), None))
    write_vtk(m, fr, b)
    assert a.read_bytes() == b.read_bytes()
    a, b = tmp_path / "c.csv", tmp_path / "py.csv"
    _lib.check(L.bt_write_flux_csv(h, str(a).encode(), None))
    write_flux_csv(fr, b)
    assert a.read_bytes() == b.read_bytes()
    # a handle made from arrays (the facade's) needs the volumes; same bytes
    # as the facade's own write()
    assert L.bt_write_vtk(mt._h, str(a).encode(), None) == _lib.BT_EINVAL
    vol = np.ascontiguousarray(mt.mesh.volumes)
    _lib.check(L.bt_write_vtk(mt._h, str(a).encode(), vol.ctypes.data))
    mt.write(b)
    assert a.read_bytes() == b.read_bytes()
    L.bt_destroy(h)
    mt.close()


def test_create_grid_and_scoring_functions():
    """create_grid / score_track_length / score_collision / finalize_batch /
    flux (tally.py:47-152) on a standalone device grid, against the same
    arithmetic in numpy; the reference's argument errors."""
    from paper_2504_19048_b200 import (batch_totals, create_grid, finalize_batch, flux,
                                       score_collision, score_track_length)
    E, G = 50, 3
    grid = create_grid(E, G)
    ref = np.zeros(E * G)
    s = np.zeros(E * G)
    sq = np.zeros(E * G)
    gen = np.random.default_rng(4)
    for batch in range(3):
        score_track_length(grid, 7, 2, 0.5, 3.0)
        ref[7 * G + 2] += 0.5 * 3.0
        score_collision(grid, 8, 0, 2.0, 4.0)
        ref[8 * G + 0] += 2.0 / 4.0
        e = gen.integers(0, E, 1000)
        g = gen.integers(0, G, 1000)
        w = gen.random(1000)
        x = gen.random(1000) + 0.1
        score_track_length(grid, e, g, w, x)
        np.add.at(ref, e * G + g, w * x)
        assert np.allclose(batch_totals(grid).reshape(-1), ref, rtol=1e-12, atol=0)
        finalize_batch(grid, 10.0)
        s += ref / 10.0
        sq += (ref / 10.0) ** 2
        ref[:] = 0.0
    assert grid.batches_completed == 3
    assert np.allclose(grid.sum, s, rtol=1e-12) and np.allclose(grid.sum_sq, sq, rtol=1e-12)
    vol = np.full(E, 0.25)
    fr = flux(grid, vol)
    assert np.allclose(fr.mean, (s / 3).reshape(E, G) / 0.25, rtol=1e-12)
    with pytest.raises(IndexError):
        score_track_length(grid, E, 0, 1.0, 1.0)
    with pytest.raises(IndexError):
        score_track_length(grid, 0, G, 1.0, 1.0)
    with pytest.raises(ValueError):
        score_collision(grid, 0, 0, 1.0, 0.0)
    with pytest.raises(ValueError):
        finalize_batch(grid, 0.0)
    with pytest.raises(ValueError):
        create_grid(0, 1)


def test_grid_is_live_and_writable():
    """MeshTally.grid reads the device arrays on every access and writes
    through on assignment (the reference's grid is the live jitclass)."""
    from paper_2504_19048_b200 import batch_totals, score_track_length
    m = build_cube_mesh(5)
    gen = np.random.default_rng(9)
    n = 2000
    pos = synth.uniform_box(gen, n)
    mt = MeshTally(m, n)
    grid = mt.grid
    mt.initialize_particle_location(pos)
    mt.move_to_next_location(synth.flight_destinations(gen, pos, 5.0), np.ones(n, np.int8),
                             np.ones(n))
    live = grid.partials
    tot = float(np.asarray(live).sum())
    assert tot > 0 and tot == pytest.approx(float(mt.read_particles().seg_total.sum()), rel=1e-12)
    score_track_length(grid, 3, 0, 2.0, 0.25)
    assert float(np.asarray(live).sum()) == pytest.approx(tot + 0.5, rel=1e-12)
    live[0, :] = 0.0
    assert not batch_totals(grid).any()
    grid.sum[5] = 7.0
    assert grid.sum[5] == 7.0 and np.asarray(grid.sum).sum() == 7.0
    grid.batches_completed = 2
    assert mt.batches_completed == 2
    mt.close()


def test_gpu_adjacency_is_the_default_with_a_gpu():
    from paper_2504_19048_b200 import mesh as M
    assert _lib.device_count() >= 1
    a = M.build_cube_mesh(20, device=None)
    b = M.build_cube_mesh(20)  # "auto": native ingest, adjacency on GPU 0
    for f in ("elements", "adj_elem", "adj_face", "volumes", "centroids"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("pinned", [False, True])
def test_deferred_initialize_paths(pinned):
    """Host positions of >= 2^20 particles with BT_OPT_DEFER_INIT = 1: the
    initialize call parks part of them in pinned staging and the next call
    localizes them.  Every way the parked part can be consumed -- a move over all
    particles, a move over fewer (the rest settled after the walk), a readout
    in between, a second initialize on top -- must equal the undeferred path
    bit for bit."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(14)
    gen = np.random.default_rng(55)
    n = 3_000_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 4.0)
    fly = (gen.random(n) < 0.9).astype(np.int8)
    w = 0.5 + gen.random(n)

    def host(a):
        return torch.from_numpy(a).pin_memory().numpy() if pinned else a

    hp, hd, hf, hw = host(pos), host(dest), host(fly), host(w)
    runs = []
    for defer in (0, 1):
        mt = MeshTally(m, n)
        mt.set_option(_lib.BT_OPT_DEFER_INIT, defer)
        out = []
        mt.initialize_particle_location(hp)                 # then a full move
        out.append(mt.move_to_next_location(hd, hf, hw))
        out.append(mt.read_particles())
        mt.initialize_particle_location(hp)                 # then a short move
        k = n - 777_777
        out.append(mt.move_to_next_location(hd[:k], hf[:k], hw[:k]))
        out.append(mt.read_particles())
        mt.initialize_particle_location(hp)                 # then a readout
        out.append(mt.read_particles())
        mt.initialize_particle_location(hp[: n // 2])
        mt.initialize_particle_location(hp)                 # init on top of init
        out.append(mt.move_to_next_location(hd, hf, hw))
        out.append(mt.read_particles())
        out.append(mt.batch_totals().copy())
        runs.append(out)
        mt.close()
    a, b = runs
    for x, y in zip(a, b):
        if hasattr(x, "position"):
            for key in ("position", "element", "alive", "entry_face", "stuck", "outcome",
                        "seg_total"):
                assert np.array_equal(getattr(x, key), getattr(y, key)), key
        elif isinstance(x, np.ndarray):
            assert np.allclose(x, y, rtol=1e-9, atol=0)
        else:
            assert x == y


def test_device_libm_restatement_equals_host_libm():
    """bt_glibc_math (csrc/glibc_math.cuh on the device) against the host
    libm the reference calls, bit for bit: 3e5 transport arguments per
    function plus the branch thresholds' neighbourhoods."""
    import ctypes
    from paper_2504_19048_b200 import _lib
    L = _lib.load()
    libm = ctypes.CDLL("libm.so.6")
    fns = []
    for name in ("log", "sin", "cos"):
        f = getattr(libm, name)
        f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double]
        fns.append(f)
    gen = np.random.default_rng(77)
    u = (np.floor(gen.random(300_000) * 2.0**53) + 1.0) / 2.0**53
    edges = np.array([0.126, 0.855469, 2.426265, np.pi / 2, np.pi, 1.5 * np.pi, 2 * np.pi])
    near = (edges[:, None] * (1.0 + np.linspace(-1e-9, 1e-9, 2001))[None, :]).reshape(-1)
    args = {0: np.concatenate([u, 0.9375 + 0.125 * u[:50_000], [1.0]]),
            1: np.concatenate([2 * np.pi * u, near]), 2: np.concatenate([2 * np.pi * u, near])}
    for fn, x in args.items():
        x = np.ascontiguousarray(x)
        out = np.empty_like(x)
        st = L.bt_glibc_math(x.ctypes.data, x.size, fn, 0, out.ctypes.data)
        if st != 0:
            pytest.skip("library built without the host libm tables")
        want = np.array([fns[fn](float(v)) for v in x])
        bad = np.nonzero(out.view(np.uint64) != want.view(np.uint64))[0]
        assert bad.size == 0, (fn, x[bad[:5]], out[bad[:5]], want[bad[:5]])


def test_misaligned_device_flying_buffer():
    """A caller's int8 flying tensor that starts at an odd address (a view)
    is read in place by the walk's refill: the same results as an aligned
    one (a refill that copies the flags in 4-byte words must not change
    that)."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(12)
    gen = np.random.default_rng(202)
    n = 50_001
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 3.0)
    fly = (gen.random(n) < 0.8).astype(np.int8)
    w = 0.5 + gen.random(n)
    out = []
    for offset in (0, 1, 3):
        mt = MeshTally(m, n, digest=True)
        mt.initialize_particle_location(torch.from_numpy(pos).cuda())
        big = torch.zeros(n + 8, dtype=torch.int8, device="cuda")
        f = big[offset:offset + n]
        f.copy_(torch.from_numpy(fly).cuda())
        s = mt.move_to_next_location(torch.from_numpy(dest).cuda(), f, torch.from_numpy(w).cuda())
        out.append(((s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                     s.stuck_terminations), mt.read_particles(), mt.read_digest(),
                    mt.batch_totals().copy()))
        mt.close()
    for s, st, (d, c), t in out[1:]:
        assert s == out[0][0]
        for k in ("position", "element", "alive", "outcome", "seg_total"):
            assert np.array_equal(getattr(st, k), getattr(out[0][1], k)), k
        assert np.array_equal(d, out[0][2][0])
        den = np.maximum(np.abs(t), np.abs(out[0][3]))
        assert (np.abs(t - out[0][3]) <= 1e-9 * den).all()  # atomic summation order
