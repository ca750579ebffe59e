"""World-size-2 CPU (gloo) test of the multi-GPU host logic: particle
sharding, per-rank walks, the per-batch tally/source-weight all-reduce and
summary reduction of ShardedMeshTally, with the CPU oracle standing in for the
per-GPU tally.  The result must equal one process walking every particle."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShard:
    """CPU tally with MeshTally's method surface (test stand-in)."""

    def __init__(self, mesh, n, groups):
        import oracle as orc
        self.t = orc.OracleTally(mesh, n, groups, threads=1)
        self.mesh = mesh

    def tally_tensor(self):
        return torch.from_numpy(self.t.partials[0])

    @property
    def source_weight(self):
        return self.t.source_weight

    @source_weight.setter
    def source_weight(self, w):
        self.t.source_weight = w

    def initialize_particle_location(self, pos):
        self.t.initialize_particle_location(pos)

    def move_to_next_location(self, d, f, w, g=None):
        from paper_2504_19048_b200.tally import TraceSummary
        s = self.t.move_to_next_location(d, f, w, g)
        return None if s is None else TraceSummary(*s)

    def finalize_batch(self, w):
        self.t.finalize_batch(w)

    def flux(self):
        return self.t.flux()

    def batch_totals(self):
        return self.t.batch_totals()


def _workload():
    from paper_2504_19048_b200 import build_cube_mesh, synth
    mesh = build_cube_mesh(8)
    gen = synth.rng(99)
    n = 3001  # odd: ragged shards
    pos = synth.uniform_box(gen, n)
    moves = []
    for _ in range(2):
        moves.append((synth.flight_destinations(gen, pos, 2.0), 0.5 + gen.random(n),
                      gen.integers(0, 2, n).astype(np.int32)))
    return mesh, pos, moves


def _fly(batch, move, n):
    fly = np.ones(n, np.int8)
    if batch == 1:
        fly[::3] = 0  # some particles sit out a move
    if batch == 2 and move == 0:
        fly[1000:] = 0  # only rank 0's shard flies: rank 1 must not record move 2
    return fly


NBATCH = 3


def _worker(rank, world, port, q):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle"), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19048_b200.distributed import ShardedMeshTally
        mesh, pos, moves = _workload()
        n = pos.shape[0]
        sh = ShardedMeshTally(mesh, n, 2, _tally_factory=OracleShard)
        out = []
        for batch in range(NBATCH):
            sh.initialize_particle_location(pos)
            sums = []
            for mv, (d, w, g) in enumerate(moves):
                s = sh.move_to_next_location(d, _fly(batch, mv, n), w, g)
                sums.append(tuple(s.__dict__.values()))
            sums.append(sh.source_weight)
            sh.finalize_batch()
            out.append(sums)
        mean, rel = sh.flux()
        q.put((rank, out, mean, rel, sh.lo, sh.hi))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_single_process():
    sys.path[:0] = [str(ROOT / "oracle")]
    import oracle as orc
    mesh, pos, moves = _workload()
    n = pos.shape[0]
    ref = orc.OracleTally(mesh, n, 2, threads=1)
    ref_out = []
    for batch in range(NBATCH):
        ref.initialize_particle_location(pos)
        sums = []
        for mv, (d, w, g) in enumerate(moves):
            sums.append(tuple(ref.move_to_next_location(d, _fly(batch, mv, n), w, g)))
        sums.append(ref.source_weight)
        ref.finalize_batch()
        ref_out.append(sums)
    rmean, rrel = ref.flux()

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    bounds = [(r[4], r[5]) for r in results]
    assert bounds == [(0, 1501), (1501, 3001)]
    for rank, out, mean, rel, lo, hi in results:
        # summaries: sums of counters, max of sweeps -> identical to one process;
        # the recorded source weight is the global first move's (two partial
        # sums: equal to the single-process pairwise sum within rounding)
        for got, want in zip(out, ref_out):
            assert got[:-1] == want[:-1]
            assert got[-1] == pytest.approx(want[-1], rel=1e-14)
        den = np.maximum(np.abs(mean), np.abs(rmean))
        assert (np.abs(mean - rmean) <= 1e-12 * den).all()
        assert np.abs(rel - rrel).max() < 1e-5


def test_shard_bounds():
    from paper_2504_19048_b200.distributed import shard_bounds
    assert [shard_bounds(10, r, 4) for r in range(4)] == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert [shard_bounds(2, r, 4) for r in range(4)] == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(ValueError):
        shard_bounds(10, 4, 4)
