"""Pin the CPU oracle (oracle/walk_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the reference package
(oracle/gen_golden.py); every comparison here is bit-exact except the
multi-threaded tally (slab summation order).
"""

import numpy as np
import pytest

import oracle as orc
from golden_cases import GOLDEN, STATE_KEYS, WALK_CASES, load_walk_case, rel_close
from paper_2504_19048_b200 import mesh as mymesh


def test_geometry_kats_bit_exact():
    d = np.load(GOLDEN / "geometry_kat.npz")
    l, det = orc.bary([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [0.1, 0.2, 0.3])
    assert np.array_equal(l, d["spec_bary"])
    for i in range(d["bary_tets"].shape[0]):
        l, det = orc.bary(d["bary_tets"][i], d["bary_pts"][i])
        want = d["bary_out"][i]
        assert det == want[4]
        if det != 0.0:
            assert np.array_equal(l, want[:4])
    for i in range(d["fh_t"].shape[0]):
        t = orc.face_hit(d["fh_faces"][i], d["fh_orig"][i], d["fh_seg"][i])
        assert t == d["fh_t"][i] or (np.isnan(t) and np.isnan(d["fh_t"][i]))
    m3 = mymesh.build_cube_mesh(3)
    for i in range(d["xs_out"].shape[0]):
        k, f, t = orc.exit_search(m3, d["xs_elem"][i], d["xs_orig"][i], d["xs_dest"][i],
                                  d["xs_entry"][i])
        assert (k, f, t) == tuple(d["xs_out"][i]), i


def test_spec_exit_face_kat():
    # find_exit_face(o=(0.1,0.1,0.1), d=(0.1,0.1,-0.5)) on the
    # reference tet -> face 3, t = 0.16666666666666669
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=np.float64)
    e = np.array([[0, 1, 2, 3]], dtype=np.int32)
    m = mymesh.TetMesh.from_arrays(v, e)
    k, f, t = orc.exit_search(m, 0, [0.1, 0.1, 0.1], [0.1, 0.1, -0.5], -1)
    assert (k, f) == (1, 3) and t == 0.16666666666666669


def _run_case(case, threads=1):
    tal = orc.OracleTally(case.mesh, case.capacity, case.num_groups, threads=threads)
    for b in case.batches:
        tal.initialize_particle_location(b.init_positions)
        n = b.init_positions.shape[0]
        assert np.array_equal(tal.element[:n], b.init_element)
        assert np.array_equal(tal.alive[:n], b.init_alive)
        for mv in b.moves:
            seg0 = tal.seg_total[:n].copy()
            s = tal.move_to_next_location(mv.dest, mv.flying, mv.weights, mv.groups)
            yield tal, mv, np.array(s), tal.seg_total[:n] - seg0, n
        tal.finalize_batch()
        assert tal.source_weight == 0.0


@pytest.mark.parametrize("name", WALK_CASES)
def test_oracle_walk_matches_reference(name):
    case = load_walk_case(name)
    for tal, mv, summ, seg, n in _run_case(case):
        e = mv.expect
        assert np.array_equal(summ, e["summary"]), (summ, e["summary"])
        for k in STATE_KEYS:
            assert np.array_equal(getattr(tal, k)[:n], e[k]), k
        assert np.array_equal(tal.count[:n], e["count"])
        assert np.array_equal(tal.digest[:n], e["digest"])
        assert np.array_equal(seg, e["seg_delta"])
        # serial lockstep: identical summation order -> bitwise tally
        assert np.array_equal(tal.batch_totals(), e["tally"])


@pytest.mark.parametrize("name", ["c1_point_s2", "n6_uniform_g3"])
def test_oracle_threads_tally_tolerance(name):
    case = load_walk_case(name)
    last = None
    for tal, mv, summ, seg, n in _run_case(case, threads=4):
        assert np.array_equal(summ, mv.expect["summary"])
        assert np.array_equal(tal.digest[:n], mv.expect["digest"])
        ok, worst = rel_close(tal.batch_totals(), mv.expect["tally"], 1e-12)
        assert ok, worst
        last = tal
    assert rel_close(last.sum, case.batches[-1].sum, 1e-12)[0]
    assert rel_close(last.sum_sq, case.batches[-1].sum_sq, 1e-12)[0]
    mean, rel = last.flux()
    assert rel_close(mean, case.flux_mean.reshape(mean.shape), 1e-12)[0]
    # rel_error = sqrt((sq - s^2/n)/(n(n-1)))/mean cancels catastrophically when
    # batches agree, so a 1e-12 perturbation of the sums moves it by up to
    # ~sqrt(1e-12); compare it absolutely (it is a fraction in [0, 1]).
    assert np.abs(rel - case.flux_rel.reshape(rel.shape)).max() < 1e-5


def test_oracle_finalize_and_flux_bit_exact():
    case = load_walk_case("c1_point_s2")
    tal = None
    bi = 0
    for tal, mv, summ, seg, n in _run_case(case):
        pass
    mean, rel = tal.flux()
    assert np.array_equal(tal.sum, case.batches[-1].sum)
    assert np.array_equal(tal.sum_sq, case.batches[-1].sum_sq)
    assert np.array_equal(mean, case.flux_mean)
    assert np.array_equal(rel, case.flux_rel)


def test_oracle_localization_pathologies():
    d = np.load(GOLDEN / "localize_ref.npz")
    m = mymesh.build_cube_mesh(10)
    pts = d["points"]
    tal = orc.OracleTally(m, pts.shape[0])
    tal.initialize_particle_location(pts)
    assert np.array_equal(tal.element, d["element"])
    assert np.array_equal(tal.alive, d["alive"])
    assert np.array_equal(tal.outcome, d["outcome"])
    # lowest-id containing element (pkg/tests/oracles.py:36-57 semantics)
    # agrees with the walk on the generic subset
    ng = int(d["groups"][0])
    low = orc.locate_exhaustive(m, pts[:ng])
    assert np.array_equal(low, d["element"][:ng])
