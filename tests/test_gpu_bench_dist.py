"""bench.py's N > 1 path (torchrun, one rank per GPU: particle shards, tally
all-reduce per batch, barrier + max-over-ranks timing, rank 0 prints the
line) executed end to end: two ranks sharing cuda:0 over gloo
(BENCH_SHARE_GPU=1), since NCCL refuses two ranks on one GPU."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_smoke():
    env = dict(os.environ, BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--particles", "300000", "--no-cpu-baseline",
           "--no-transport"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["global_particles"] == 600_000
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    # both ranks' crossings: ~57 per particle-move on C2 at sigma_t = 2
    assert 50 < d["value"] / d["particle_moves_per_s"] < 65
