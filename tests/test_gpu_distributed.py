"""ShardedMeshTally on the real CUDA path: two ranks sharing cuda:0 over gloo
(CUDA tensors; NCCL refuses two ranks on one GPU) and one rank over NCCL.
Results must match one MeshTally walking every particle (tallies within
1e-9 relative: only the summation order of the per-rank tallies differs)."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    from paper_2504_19048_b200 import build_cube_mesh, synth
    mesh = build_cube_mesh(9)
    gen = synth.rng(7)
    n = 20001
    pos = synth.uniform_box(gen, n)
    moves = [(synth.flight_destinations(gen, pos, 3.0), 0.5 + gen.random(n)) for _ in range(2)]
    return mesh, pos, moves


def _run(sh, pos, moves):
    n = pos.shape[0]
    sh.initialize_particle_location(pos)
    sums = []
    for d, w in moves:
        s = sh.move_to_next_location(d, np.ones(n, np.int8), w)
        sums.append((s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                     s.stuck_terminations))
    sh.finalize_batch()
    return sums, np.asarray(sh.flux().mean)


def _worker(rank, world, port, backend, q):
    sys.path[:0] = [str(ROOT)]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    kw = dict(device_id=torch.device("cuda", 0)) if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_2504_19048_b200.distributed import ShardedMeshTally
        mesh, pos, moves = _workload()
        sh = ShardedMeshTally(mesh, pos.shape[0], device=0)
        sums, mean = _run(sh, pos, moves)
        q.put((rank, sums, mean))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1)])
def test_sharded_cuda_tally_matches_single(backend, world):
    import torch.multiprocessing as mp
    from paper_2504_19048_b200 import MeshTally
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mesh, pos, moves = _workload()
    n = pos.shape[0]
    mt = MeshTally(mesh, n)
    mt.initialize_particle_location(pos)
    ref = []
    for d, w in moves:
        s = mt.move_to_next_location(d, np.ones(n, np.int8), w)
        ref.append((s.sweeps, s.events, s.reached, s.boundary_exits, s.stuck_recoveries,
                    s.stuck_terminations))
    mt.finalize_batch()
    mean_ref = np.asarray(mt.flux().mean)
    for rank, sums, mean in res:
        assert sums == ref
        den = np.maximum(np.abs(mean), np.abs(mean_ref))
        assert (np.abs(mean - mean_ref) <= 1e-9 * den).all()
