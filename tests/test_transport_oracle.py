"""Pin the C restatement of the reference transport driver (SURVEY §8f row 1:
philox4x64-10, transport.run) to the reference's own outputs
(tests/golden/transport_ref.npz, written by oracle/gen_golden.py --transport)."""

import numpy as np
import pytest

import oracle as orc
from golden_cases import GOLDEN
from paper_2504_19048_b200 import build_cube_mesh


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLDEN / "transport_ref.npz")


def test_philox_kat(gold):
    for c, k, want in zip(gold["philox_ctr"].reshape(-1, 4), gold["philox_key"].reshape(-1, 2),
                          gold["philox_out"]):
        assert np.array_equal(orc.philox(c, k), want)
    # raw_block([0,0,0,0],[0,0]) (Random123 philox4x64-10 KAT)
    assert [hex(x) for x in orc.philox([0, 0, 0, 0], [0, 0])] == [
        "0x16554d9eca36314c", "0xdb20fe9d672d0fdc", "0xd7e772cee186176b", "0x7e68b68aec7ba23b"]


def test_uniform_block(gold):
    for (a, b, c, d), want in zip(gold["uni_key"], gold["uni_out"]):
        assert np.array_equal(orc.uniform_block(a, b, c, d), want)


@pytest.mark.parametrize("name", ["t1g", "t2g", "tdir"])
def test_transport_run_matches_reference(gold, name):
    p = name + "_"
    n_mesh, n, nb, seed = (int(x) for x in gold[p + "cfg"])
    m = build_cube_mesh(n_mesh)
    d = gold[p + "dir"]
    r = orc.transport_run(m, gold[p + "sigma_t"], gold[p + "sigma_s"], n, nb, seed,
                          gold[p + "box"], direction=d if d.size else None)
    for key in ("source_weight", "leaked_weight", "absorbed_weight", "stuck_weight",
                "collisions", "events", "sweeps", "track_length_total"):
        assert r[key] == float(gold[p + key]), key
    ng = gold[p + "sigma_t"].shape[0]
    mean, rel = orc.flux_from_moments(r["track_sum"], r["track_sum_sq"], nb, m.volumes, ng)
    assert np.array_equal(mean, gold[p + "flux_track_mean"])
    assert np.array_equal(rel, gold[p + "flux_track_rel"])
    mean, rel = orc.flux_from_moments(r["col_sum"], r["col_sum_sq"], nb, m.volumes, ng)
    assert np.array_equal(mean, gold[p + "flux_col_mean"])
    assert np.array_equal(rel, gold[p + "flux_col_rel"])
    for key in ("position", "direction", "element", "group", "alive", "outcome", "rng_block",
                "seg_total"):
        assert np.array_equal(r[key][:n], gold[p + "final_" + key]), key
