"""Listing-1 callback path on the GPU (bt_load_step / bt_trace_* through
MeshTally.trace_batch) vs the reference's trace_batch with the same
deterministic callback (tests/golden/callback_ref.npz)."""

import numpy as np
import pytest

from golden_cases import GOLDEN, rel_close
from paper_2504_19048_b200 import MeshTally, build_cube_mesh

pytestmark = pytest.mark.gpu

H0 = np.uint64(0xCBF29CE484222325)
HP = np.uint64(0x100000001B3)


def callback_decisions(sweep, particle, element, exit_face, next_element, particle_done):
    """Verbatim copy of oracle/gen_golden.py:callback_decisions (the reference
    side cannot be imported on the GPU box)."""
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
    next_element[jump] = np.asarray(element)[jump]


@pytest.mark.parametrize("name", ["cb_n6", "cb_plane"])
def test_trace_batch_matches_reference(name):
    g = np.load(GOLDEN / "callback_ref.npz")
    p = name + "_"
    m = build_cube_mesh(int(g[p + "mesh_n"]))
    k = g[p + "pos"].shape[0]
    modify = bool(g[p + "modify"])
    mt = MeshTally(m, k, 2, localize="walk", digest=True)
    mt.initialize_particle_location(g[p + "pos"])
    mt.load_step(g[p + "dest"], g[p + "fly"], g[p + "w"], g[p + "groups"])
    h = np.full(k, H0, dtype=np.uint64)
    cnt = np.zeros(k, np.int64)
    counts = []
    state = {"sweep": 0}

    def cb(ev):
        pid = np.asarray(ev.particle, dtype=np.int64)
        code = (np.asarray(ev.element, dtype=np.int64) * 8
                + np.asarray(ev.exit_face, dtype=np.int64) + 1).astype(np.uint64)
        with np.errstate(over="ignore"):
            h[pid] = (h[pid] ^ code) * HP
        cnt[pid] += 1
        counts.append(len(ev))
        if modify:
            callback_decisions(state["sweep"], ev.particle, ev.element, ev.exit_face,
                               ev.next_element, ev.particle_done)
        state["sweep"] += 1

    s = mt.trace_batch(cb)
    got = np.array([s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                    s.stuck_terminations])
    assert np.array_equal(got, g[p + "summary"]), (got, g[p + "summary"])
    assert counts == g[p + "sweep_counts"].tolist()
    assert np.array_equal(h, g[p + "digest"]) and np.array_equal(cnt, g[p + "count"])
    d, c = mt.read_digest(k)
    assert np.array_equal(d, g[p + "digest"]) and np.array_equal(c, g[p + "count"])
    st = mt.read_particles(k)
    for key in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
        assert np.array_equal(getattr(st, key), g[p + key]), key
    assert rel_close(mt.batch_totals().reshape(-1), g[p + "tally"], 1e-9)[0]


def test_trace_batch_device_events_and_errors():
    torch = pytest.importorskip("torch")
    g = np.load(GOLDEN / "callback_ref.npz")
    p = "cb_n6_"
    m = build_cube_mesh(int(g[p + "mesh_n"]))
    k = g[p + "pos"].shape[0]
    a = MeshTally(m, k, 2, localize="walk")
    b = MeshTally(m, k, 2, localize="walk")
    for mt in (a, b):
        mt.initialize_particle_location(g[p + "pos"])
        mt.load_step(g[p + "dest"], g[p + "fly"], g[p + "w"], g[p + "groups"])

    def kill_half(ev):  # works on numpy and torch views alike
        ev.particle_done[ev.particle % 2 == 1] = 1

    sa = a.trace_batch(kill_half)
    sb = b.trace_batch(kill_half, device_events=True)
    assert sa == sb
    assert np.array_equal(a.read_particles(k).position, b.read_particles(k).position)
    # unlocalized flying particle -> ValueError before any work
    c = MeshTally(m, 4)
    c.load_step(np.full((4, 3), 0.3), np.ones(4), np.ones(4))
    with pytest.raises(ValueError):
        c.trace_batch()
