"""Parity of the MEASURED kernel and of the configurations the benches run.

The bench times the walk without digest bookkeeping
(``walk_staged_kernel<192, 2, DIG=false, DIRECT=true>``); the golden-case
tests run the digest build of the same template.  Here the digest-free
kernel is checked against the CPU oracle directly (states, ``seg_total`` and
per-bin tallies), and the configurations of BASELINE.json configs[2..4] that
exceed the oracle's reach are checked on samples (walks are independent per
particle, search.py:182-274, so a sample replayed on the oracle from the
same start state must match bit for bit):

* C2 (998,250 tets): 2e5 particles exhaustively, and the 1e7-particle bench
  move on a 20,000-particle sample;
* C4's two meshes beyond L2 (n = 95: 5,144,250 tets; n = 119: 10,110,954):
  1e7 particles, sampled; at n = 119 also the whole move against the
  literal-arithmetic walk (BT_OPT_EXACT_ONLY);
* C5 (toroidal shell 8 x 256 x 408 = 5,013,504 tets): 1e7 particles from a
  sector, a 10-move chain, sampled after every move;
* C3's largest point (1e8 particles on C2), sampled.

Bars: element, position, flags, outcome, ``seg_total`` and (where digests
run) the (element, exit face) sequence digests bit-exact; per-bin tallies
within 1e-9 relative (BASELINE.json north_star).
"""

import numpy as np
import pytest

import oracle as orc
from golden_cases import rel_close
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh, synth

pytestmark = pytest.mark.gpu

TALLY_RTOL = 1e-9
STATE = ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total")
SAMPLE = 20_000


def _summary(s):
    return (s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
            s.stuck_terminations)


def _device_move(mt, torch, dest, fly, w):
    return mt.move_to_next_location(torch.from_numpy(dest).cuda(), torch.from_numpy(fly).cuda(),
                                    torch.from_numpy(w).cuda())


def _oracle_from(m, pos, dest, fly, w):
    ref = orc.OracleTally(m, pos.shape[0], threads=orc.max_threads())
    ref.initialize_particle_location(pos)
    ref.seg_total[:] = 0.0  # grid localization has no trial-walk length
    r = ref.move_to_next_location(dest, fly, w)
    return ref, r


def _check_sample(st, idx, ref, keys=STATE):
    for k in keys:
        assert np.array_equal(getattr(st, k)[idx], getattr(ref, k)[:idx.size]), k


@pytest.mark.parametrize("sigma_t", [2.0, 100.0])
def test_bench_kernel_scored_path_exhaustive_c2(sigma_t):
    """The digest-free (benchmarked) kernel against the oracle on every
    particle of a 2e5-particle C2 move: summary, states, seg_total bit-exact,
    every tally bin within 1e-9."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 210)
    n = 200_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, sigma_t)
    w = 0.5 + gen.random(n)
    fly = (gen.random(n) < 0.95).astype(np.int8)
    mt = MeshTally(m, n)  # digest off: the bench's kernel
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    s = _device_move(mt, torch, dest, fly, w)
    st = mt.read_particles()
    ref, r = _oracle_from(m, pos, dest, fly, w)
    assert _summary(s) == tuple(r)
    _check_sample(st, np.arange(n), ref)
    ok, worst = rel_close(mt.batch_totals().reshape(-1), ref.batch_totals(), TALLY_RTOL)
    assert ok, worst
    assert mt.source_weight == w[fly != 0].sum()  # device-side pairwise sum, numpy's bits
    mt.finalize_batch()
    ref.finalize_batch()
    assert rel_close(mt.grid.sum, ref.sum, TALLY_RTOL)[0]
    assert rel_close(mt.grid.sum_sq, ref.sum_sq, TALLY_RTOL)[0]
    mt.close()


def test_bench_kernel_at_bench_size_c2():
    """The bench move itself (C2, 1e7 particles, uniform source, sigma_t = 2,
    device inputs) through the digest-free kernel: a 20,000-particle sample
    equals the oracle bit for bit; the whole move equals the digest kernel's
    (summary, states, every tally bin within 1e-9); path length is conserved."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(55)
    gen = synth.rng(synth.SEED + 211)
    n = 10_000_000
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 2.0)
    w = 0.5 + gen.random(n)
    fly = np.ones(n, np.int8)
    runs = []
    for digest in (False, True):
        mt = MeshTally(m, n, digest=digest)
        mt.initialize_particle_location(torch.from_numpy(pos).cuda())
        s = _device_move(mt, torch, dest, fly, w)
        runs.append((s, mt.read_particles(), mt.batch_totals().reshape(-1), mt.source_weight))
        mt.close()
    (s0, st0, t0, w0), (s1, st1, t1, w1) = runs
    assert _summary(s0) == _summary(s1)
    for k in STATE:
        assert np.array_equal(getattr(st0, k), getattr(st1, k)), k
    ok, worst = rel_close(t0, t1, TALLY_RTOL)
    assert ok, worst
    assert w0 == w1 == w.sum()
    tot = t0.sum()
    assert abs(tot - float((w * st0.seg_total).sum())) <= 1e-9 * tot
    idx = np.sort(gen.choice(n, SAMPLE, replace=False))
    ref, _ = _oracle_from(m, pos[idx], dest[idx], fly[idx], w[idx])
    _check_sample(st0, idx, ref)


def _c4_inputs(m, n, seed):
    gen = synth.rng(seed)
    pos = synth.uniform_box(gen, n)
    dest = synth.flight_destinations(gen, pos, 2.0)
    w = 0.5 + gen.random(n)
    return gen, pos, dest, w


@pytest.mark.parametrize("cells", [95, 119])
def test_c4_meshes_beyond_l2_sampled_parity(cells):
    """C4's L2-exceeding meshes (5.1M and 10.1M tets), 1e7 particles: the
    benchmarked (digest-free) kernel and the digest kernel agree on the whole
    move, and a 20,000-particle sample -- digests included -- equals the
    oracle bit for bit.  At n = 119 the whole move also equals the walk with
    every exit search in the reference's literal arithmetic."""
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(cells, device=0)
    n = 10_000_000
    gen, pos, dest, w = _c4_inputs(m, n, synth.SEED + 300 + cells)
    fly = np.ones(n, np.int8)
    modes = [(False, 0), (True, 0)] + ([(True, 1)] if cells == 119 else [])
    runs = []
    for digest, exact in modes:
        mt = MeshTally(m, n, digest=digest)
        mt.set_option(_lib.BT_OPT_EXACT_ONLY, exact)
        mt.initialize_particle_location(torch.from_numpy(pos).cuda())
        s = _device_move(mt, torch, dest, fly, w)
        dg = mt.read_digest() if digest else None
        runs.append((s, mt.read_particles(), mt.batch_totals().reshape(-1), dg))
        mt.close()
    s0, st0, t0, _ = runs[0]
    assert s0.events > 50 * n
    for s, st, t, dg in runs[1:]:
        assert _summary(s) == _summary(s0)
        for k in STATE:
            assert np.array_equal(getattr(st, k), getattr(st0, k)), k
        assert rel_close(t, t0, TALLY_RTOL)[0]
    if cells == 119:
        (d1, c1), (d2, c2) = runs[1][3], runs[2][3]
        assert np.array_equal(d1, d2) and np.array_equal(c1, c2)
    tot = t0.sum()
    assert abs(tot - float((w * st0.seg_total).sum())) <= 1e-9 * tot
    idx = np.sort(gen.choice(n, SAMPLE, replace=False))
    ref, _ = _oracle_from(m, pos[idx], dest[idx], fly[idx], w[idx])
    _check_sample(st0, idx, ref)
    d, c = runs[1][3]
    assert np.array_equal(d[idx], ref.digest) and np.array_equal(c[idx], ref.count)


def test_c5_torus_ten_move_chain_sampled_parity():
    """C5: the 5,013,504-tet toroidal shell (8 x 256 x 408 cells, R = 300,
    a = 100..120 cm), 1e7 particles from a shell sector, ten chained moves
    (flying = alive, sigma_t = 1/30 cm^-1) through the benchmarked kernel.
    A 20,000-particle sample follows on the oracle from the grid's placement
    and must match bit for bit after every move."""
    torch = pytest.importorskip("torch")
    from paper_2504_19048_b200 import build_torus_shell_mesh
    m = build_torus_shell_mesh(8, 256, 408, R=300.0, a_in=100.0, a_out=120.0)
    gen = np.random.default_rng(5)
    n = 10_000_000
    i = gen.integers(0, 8, n)
    j = gen.integers(0, 32, n)
    k = gen.integers(0, 51, n)
    elems = ((i * 256 + j) * 408 + k) * 6 + gen.integers(0, 6, n)
    pos = synth.points_in_elements(gen, m.vertices, m.elements, elems)
    idx = np.sort(gen.choice(n, SAMPLE, replace=False))
    mt = MeshTally(m, n)
    mt.initialize_particle_location(torch.from_numpy(pos).cuda())
    st = mt.read_particles()
    assert np.array_equal(st.element[idx], elems[idx])  # generic interior points
    ref = orc.OracleTally(m, idx.size, threads=orc.max_threads())
    ref.initialize_particle_location(pos[idx])
    found = ref.element >= 0  # the reference's walk loses points behind the hole
    assert np.array_equal(ref.element[found], elems[idx][found])
    for key in ("element", "alive", "position", "outcome", "entry_face", "stuck"):
        getattr(ref, key)[:] = getattr(st, key)[idx]  # continue from the grid's placement
    ref.seg_total[:] = 0.0
    cur = pos
    events = 0
    scored = 0.0  # sum over moves of w * (this move's path length)
    for move in range(10):
        dest = synth.flight_destinations(gen, cur, 1.0 / 30.0)
        fly = st.alive.astype(np.int8)
        w = 0.5 + gen.random(n)
        seg0 = st.seg_total
        s = _device_move(mt, torch, dest, fly, w)
        r = ref.move_to_next_location(dest[idx], fly[idx], w[idx])
        st = mt.read_particles()
        _check_sample(st, idx, ref)
        events += s.events
        assert r.events <= s.events
        scored += float((w * (st.seg_total - seg0)).sum())
        cur = st.position
    assert events > 10 * n
    tot = mt.batch_totals().sum()
    assert abs(tot - scored) <= 1e-9 * tot  # path-length conservation over the chain
    mt.close()


def test_c3_1e8_particles_sampled_parity():
    """C3's largest point: 1e8 particles on the C2 mesh, one move through the
    benchmarked kernel (inputs generated on the device).  20,000 random
    particles (position, element, alive) and the first 20,000 (every state
    field, seg_total) replayed on the oracle match bit for bit; counters add
    up; path length is conserved."""
    torch = pytest.importorskip("torch")
    import math
    m = build_cube_mesh(55)
    n = 100_000_000
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(synth.SEED + 400)
    pos = 0.05 + 0.9 * torch.rand(n, 3, generator=g, device=dev, dtype=torch.float64)
    mu = 2.0 * torch.rand(n, generator=g, device=dev, dtype=torch.float64) - 1.0
    phi = 2.0 * math.pi * torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    ell = -torch.log(1.0 - torch.rand(n, generator=g, device=dev, dtype=torch.float64)) / 2.0
    s_ = torch.sqrt(torch.clamp(1.0 - mu * mu, min=0.0))
    dest = pos + ell[:, None] * torch.stack([s_ * torch.cos(phi), s_ * torch.sin(phi), mu], 1)
    del mu, phi, ell, s_
    w = 0.5 + torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    fly = torch.ones(n, dtype=torch.int8, device=dev)
    gen = np.random.default_rng(401)
    idx = np.sort(gen.choice(n, SAMPLE, replace=False))
    it = torch.from_numpy(idx).to(dev)
    head = np.arange(SAMPLE)
    sample_in = {name: (t[it].cpu().numpy(), t[:SAMPLE].cpu().numpy())
                 for name, t in (("pos", pos), ("dest", dest), ("w", w))}
    mt = MeshTally(m, n)
    mt.initialize_particle_location(pos)
    s = mt.move_to_next_location(dest.contiguous(), fly, w)
    assert s.reached + s.boundary_exits + s.stuck_terminations == n
    assert s.events > 50 * n
    p_t, e_t, a_t = mt.particle_tensors()
    got = {"position": p_t[it].cpu().numpy(), "element": e_t[it].cpu().numpy(),
           "alive": a_t[it].cpu().numpy()}
    st_head = mt.read_particles(SAMPLE)
    tot = mt.batch_totals().sum()
    del pos, dest, fly
    for which, sel in ((0, idx), (1, head)):
        ref, _ = _oracle_from(m, sample_in["pos"][which], sample_in["dest"][which],
                              np.ones(SAMPLE, np.int8), sample_in["w"][which])
        if which == 0:
            for k, v in got.items():
                assert np.array_equal(v, getattr(ref, k)), k
        else:
            _check_sample(st_head, head, ref)
    # path-length conservation over all 1e8 particles
    seg = np.empty(n)
    _lib.check(mt._L.bt_read_particles(mt._h, n, None, None, None, None, None, None,
                                       seg.ctypes.data))
    wsum = float((w * torch.from_numpy(seg).to(dev)).sum().item())
    mt.close()
    assert abs(tot - wsum) <= 1e-9 * tot
