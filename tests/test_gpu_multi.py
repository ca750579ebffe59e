"""One handle over several GPUs (bt_create_multi; SURVEY §8b "ndev", §8e):
contiguous particle shards, replicated mesh, one NCCL all-reduce of the
tallies per batch.

On this one-GPU pool: devices=[0] runs the NCCL path (a one-rank
communicator), devices=[0, 0] / [0, 0, 0] run the shard fan-out with the
peer-copy reduction; both must reproduce the reference golden cases exactly
like a single-GPU handle.  The >= 2-GPU test runs where two GPUs are visible.
"""

import numpy as np
import pytest

from golden_cases import load_walk_case, rel_close
from paper_2504_19048_b200 import MeshTally, build_cube_mesh, synth
from test_gpu_parity import _check_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("name", ["c1_point_s2", "n6_uniform_g3", "c1_point_s100"])
def test_multi_handle_matches_reference(devices, name):
    _check_case(load_walk_case(name), "grid", devices=devices)


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_handle_equals_single_handle(devices):
    """Same inputs through a one-GPU handle and a sharded one: identical
    particle states and summaries, tallies within 1e-12, the same recorded
    source weight rule (first move with flying weight, decided globally:
    the first move here flies only particles of the first shard)."""
    m = build_cube_mesh(12)
    gen = np.random.default_rng(31)
    n = 30_001  # ragged shards
    pos = synth.uniform_box(gen, n)
    one = MeshTally(m, n, 2)
    many = MeshTally(m, n, 2, devices=devices)
    assert many.num_shards == len(devices)
    assert many.shard_bounds(0)[0] == 0 and many.shard_bounds(len(devices) - 1)[1] == n
    for t in (one, many):
        t.initialize_particle_location(pos)
    cur = pos
    for move in range(3):
        dest = synth.flight_destinations(gen, cur, 4.0)
        w = 0.5 + gen.random(n)
        g = gen.integers(0, 2, n).astype(np.int32)
        fly = np.ones(n, np.int8)
        if move == 0:
            fly[n // len(devices) // 2:] = 0
        count = n if move != 2 else n - 5000  # ragged count
        s1 = one.move_to_next_location(dest[:count], fly[:count], w[:count], g[:count])
        s2 = many.move_to_next_location(dest[:count], fly[:count], w[:count], g[:count])
        assert s1 == s2
        a, b = one.read_particles(n), many.read_particles(n)
        for k in ("position", "element", "alive", "entry_face", "stuck", "outcome", "seg_total"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), (move, k)
        assert rel_close(one.batch_totals(), many.batch_totals(), 1e-12)[0]
        assert many.source_weight == pytest.approx(one.source_weight, rel=1e-14)
        cur = a.position
    one.finalize_batch()
    many.finalize_batch()
    assert rel_close(one.grid.sum, many.grid.sum, 1e-12)[0]
    assert rel_close(one.grid.sum_sq, many.grid.sum_sq, 1e-12)[0]
    f1, f2 = one.flux(), many.flux()
    assert rel_close(f1.mean, f2.mean, 1e-12)[0]
    with pytest.raises(RuntimeError):
        many.finalize_batch()  # no source weight recorded after the finalize
    one.close()
    many.close()


def test_multi_handle_refuses_device_arrays_and_single_gpu_paths():
    torch = pytest.importorskip("torch")
    m = build_cube_mesh(4)
    mt = MeshTally(m, 10, devices=[0, 0])
    pos = torch.full((10, 3), 0.3123, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        mt.initialize_particle_location(pos)
    with pytest.raises(ValueError):
        mt.particle_tensors()
    mt.close()


def test_two_gpus():
    torch = pytest.importorskip("torch")
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    test_multi_handle_equals_single_handle([0, 1])
    _check_case(load_walk_case("c1_point_s2"), "grid", devices=[0, 1])
