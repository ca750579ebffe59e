"""Device transport (bt_transport_run) vs the reference's transport.run
(golden fixtures) and the CPU oracle, which is pinned bit-exact to it
(tests/test_transport_oracle.py).

* philox4x64-10 uniforms: bit-exact.
* Histories: the same sequence of operations, and -- with the host libm's
  log / sin / cos restated on the device (csrc/glibc_math.cuh, tables read
  from this image's glibc at build time) -- the same bits:
  test_transport_bit_exact_vs_reference requires every particle's final
  state, the event / collision / sweep counts and the balance weights to be
  the reference's exactly, the fluxes within 1e-9.
* A build without those tables (another libm) falls back to CUDA's
  functions; histories then diverge after a last-bit difference, and the
  statistical tests below carry the parity: per-history PAIRED differences
  (device minus reference, same particle, same random stream) of track
  length, random blocks consumed and outcome must have mean 0 within K
  standard errors (a 1% bias in the collision rate or the scatter sampling
  fails this at the sizes below).  With the tables they see 0 differences.
"""

import numpy as np
import pytest

import oracle as orc
from golden_cases import GOLDEN
from paper_2504_19048_b200 import build_cube_mesh
from paper_2504_19048_b200 import transport as T

pytestmark = pytest.mark.gpu

K = 4.0  # standard errors


def _exact_math():
    """The library carries the host libm restatement (bit-exact histories)."""
    from paper_2504_19048_b200 import _lib
    x = np.array([0.5])
    return _lib.load().bt_glibc_math(x.ctypes.data, 1, 0, 0, x.ctypes.data) == 0


def _paired_ok(a, b, what):
    """mean(a - b) within K standard errors of 0 (exactly 0 if all equal)."""
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    n = d.size
    se = d.std(ddof=1) / np.sqrt(n) if n > 1 else 0.0
    m = d.mean()
    print(f"  {what}: mean diff {m:.4g}, se {se:.3g}, diverged {(d != 0).mean():.3f}")
    assert abs(m) <= K * se + 1e-12 * max(1.0, float(np.abs(b).mean())), what
    return d


def _total_ok(total_a, total_b, d_last, nb, what):
    """A run total (all batches) against the reference's: the paired per-
    history differences of the last batch give its standard error."""
    se = np.sqrt(nb * float((d_last ** 2).sum()))
    print(f"  {what}: {total_a} vs {total_b}, K*se = {K * se:.4g}")
    assert abs(total_a - total_b) <= K * se + 1e-9 * abs(total_b), what


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "transport_ref.npz")


def test_device_philox_bit_exact(gold):
    u = T.uniform_blocks(gold["uni_key"].astype(np.uint64))
    assert np.array_equal(u, gold["uni_out"])


def _cfg(gold, name):
    p = name + "_"
    n_mesh, n, nb, seed = (int(x) for x in gold[p + "cfg"])
    d = gold[p + "dir"]
    box = gold[p + "box"]
    xs = T.CrossSections(gold[p + "sigma_t"], gold[p + "sigma_s"])
    return T.RunConfig(mesh_n=n_mesh, num_particles=n, num_batches=nb, seed=seed,
                       cross_sections=xs, source_box=(tuple(box[0]), tuple(box[1])),
                       source_direction=tuple(d) if d.size else None)


@pytest.mark.parametrize("name", ["t1g", "t2g", "tdir"])
def test_transport_statistical_parity(gold, name):
    p = name + "_"
    cfg = _cfg(gold, name)
    m = build_cube_mesh(cfg.mesh_n)
    r = T.run(cfg, m)
    n, nb = cfg.num_particles, cfg.num_batches
    # source localization is deterministic: identical source weight
    assert r.source_weight == float(gold[p + "source_weight"])
    # per-history agreement with the reference's final state (last batch)
    fs = r.final_state
    same = ((fs["rng_block"] == gold[p + "final_rng_block"])
            & (fs["outcome"] == gold[p + "final_outcome"])
            & (fs["position"] == gold[p + "final_position"]).all(axis=1)
            & (fs["group"] == gold[p + "final_group"]))
    frac = same.mean()
    for key in ("rng_block", "outcome", "group", "position", "direction", "element", "alive"):
        a, b = fs[key], gold[p + "final_" + key]
        eq = (a == b) if a.ndim == 1 else (a == b).all(axis=1)
        if not eq.all():
            j = int(np.nonzero(~eq)[0][0])
            print(f"  {name} {key}: {int((~eq).sum())} differ; first #{j}: {a[j]} vs {b[j]}")
    print(f"{name}: bit-identical histories {frac:.4f}; collisions {r.collisions} vs "
          f"{int(gold[p + 'collisions'])}; leaked {r.leaked_weight} vs "
          f"{float(gold[p + 'leaked_weight'])}")
    assert frac == 1.0 if _exact_math() else frac > 0.5
    # balance: every source particle leaks, is absorbed or stuck-killed
    assert r.leaked_weight + r.absorbed_weight + r.stuck_weight == r.source_weight
    # per-history paired differences (last batch) and the run totals
    d_seg = _paired_ok(fs["seg_total"], gold[p + "final_seg_total"], "track length") \
        if p + "final_seg_total" in gold else None
    d_blk = _paired_ok(fs["rng_block"], gold[p + "final_rng_block"], "random blocks")
    _paired_ok(fs["outcome"] == 2, gold[p + "final_outcome"] == 2, "leaked")
    _total_ok(r.collisions, float(gold[p + "collisions"]), d_blk / 2.0, nb, "collisions")
    if d_seg is not None:
        V = m.volumes[:, None]
        a = float((r.flux_track.mean * V).sum())
        b = float((gold[p + "flux_track_mean"] * V).sum())
        # integrated track-length flux = track length / (batches x source weight)
        _total_ok(a, b, d_seg / (nb * n), nb, "integrated track flux")
    # both estimators agree with each other (same physics): the collision
    # estimator's integral against the track-length one, within their
    # batch-to-batch errors
    V = m.volumes[:, None]
    a = float((r.flux_track.mean * V).sum())
    c = float((r.flux_collision.mean * V).sum())
    se = float((r.flux_track.rel_error * r.flux_track.mean * V).sum()
               + (r.flux_collision.rel_error * r.flux_collision.mean * V).sum())
    if nb >= 2:
        assert abs(a - c) <= K * se, (a, c, se)


@pytest.mark.parametrize("name", ["t1g", "t2g", "tdir"])
def test_transport_bit_exact_vs_reference(gold, name):
    """With the host libm's log / sin / cos restated on the device
    (csrc/glibc_math.cuh) every history is the reference's: final state of
    every particle (position, direction, element, group, outcome, RNG block
    counter, track length) bit for bit, the same collision and event counts,
    balance weights equal, flux of both estimators within 1e-9 (atomic
    summation order)."""
    if not _exact_math():
        pytest.skip("library built without the host libm tables")
    p = name + "_"
    cfg = _cfg(gold, name)
    m = build_cube_mesh(cfg.mesh_n)
    r = T.run(cfg, m)
    fs = r.final_state
    for key in ("position", "direction", "element", "group", "outcome", "alive", "rng_block"):
        a, b = fs[key], gold[p + "final_" + key]
        assert np.array_equal(a, b), key
    if p + "final_seg_total" in gold:
        assert np.array_equal(fs["seg_total"], gold[p + "final_seg_total"])
    for k in ("collisions", "events", "sweeps"):
        assert getattr(r, k) == int(gold[p + k]), k
    for k in ("source_weight", "leaked_weight", "absorbed_weight", "stuck_weight"):
        assert getattr(r, k) == float(gold[p + k]), k  # sums of unit weights: exact
    tl = float(gold[p + "track_length_total"])
    assert abs(r.track_length_total - tl) <= 1e-12 * tl
    for est, key in (("flux_track", "flux_track_mean"), ("flux_collision", "flux_col_mean")):
        a = getattr(r, est).mean.reshape(-1)
        b = gold[p + key].reshape(-1)
        den = np.maximum(np.abs(a), np.abs(b))
        assert (np.abs(a - b) <= 1e-9 * den).all(), est


def test_transport_vs_oracle_same_engine():
    """The oracle restatement and the device run side by side on a bigger
    paper-physics case (sigma_t = sigma_s = 100, n = 10 cube)."""
    cfg = T.RunConfig(mesh_n=10, num_particles=4000, num_batches=2, seed=5)
    m = build_cube_mesh(10)
    r = T.run(cfg, m)
    xs = cfg.cross_sections
    o = orc.transport_run(m, xs.sigma_t, xs.sigma_s, cfg.num_particles, cfg.num_batches,
                          cfg.seed, cfg.source_box)
    assert r.source_weight == o["source_weight"]
    same = (r.final_state["rng_block"] == o["rng_block"]) & \
        (r.final_state["position"] == o["position"][:cfg.num_particles]).all(axis=1)
    print("paper physics: identical histories", same.mean(), "events", r.events, o["events"],
          "collisions", r.collisions, o["collisions"])
    assert same.mean() == 1.0 if _exact_math() else same.mean() > 0.2
    fs = r.final_state
    n, nb = cfg.num_particles, cfg.num_batches
    d_seg = _paired_ok(fs["seg_total"], o["seg_total"][:n], "track length")
    d_blk = _paired_ok(fs["rng_block"], o["rng_block"][:n], "random blocks")
    _paired_ok(fs["outcome"] == 2, o["outcome"][:n] == 2, "leaked")
    _paired_ok(fs["outcome"] == 5, o["outcome"][:n] == 5, "absorbed")
    _total_ok(r.collisions, o["collisions"], d_blk / 2.0, nb, "collisions")
    _total_ok(r.events, o["events"], d_blk, nb, "events")
    _total_ok(r.track_length_total, o["track_length_total"], d_seg, nb, "track length")
