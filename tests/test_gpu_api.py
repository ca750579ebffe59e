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
