"""Particle-sharded multi-GPU tally: one process per GPU, mesh replicated,
private tallies summed by one collective per batch.

The reference has no distribution; the paper describes
replicated geometry with independent particles and "a single all gather
before writing to disk".  Here each rank owns a contiguous
particle shard ``[r*ceil(N/P), (r+1)*ceil(N/P))``, walks it
with no data-path communication, and ``finalize_batch`` sums the per-GPU
tallies and recorded source weights with ``torch.distributed.all_reduce``
(NCCL over NVLink on B200, gloo in the CPU tests) before the on-device
finalize -- the device analogue of the reference's per-thread slab reduction
in ``_finalize`` (tally.py:86-90).

``TraceSummary`` counters are summed across ranks, except ``sweeps``, which is
the maximum (the lockstep sweep count of the union is the longest walk).
"""

from __future__ import annotations

import os

import numpy as np

from .tally import TraceSummary


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n particles for `rank` of `world`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    per = -(-int(n) // world)
    lo = min(rank * per, n)
    return lo, min(lo + per, n)


def reduce_summary(s: TraceSummary | None, device=None, group=None) -> TraceSummary:
    import torch
    import torch.distributed as dist
    v = [0] * 6 if s is None else [s.sweeps, s.events, s.reached, s.boundary_exits,
                                   s.stuck_recoveries, s.stuck_terminations]
    t = torch.tensor(v[1:], dtype=torch.int64, device=device)
    m = torch.tensor([v[0]], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    return TraceSummary(int(m.item()), *(int(x) for x in t.tolist()))


def reduce_tally_(tally, group=None) -> None:
    """In-place sum of the per-rank batch tallies (the one collective per batch)."""
    import torch.distributed as dist
    dist.all_reduce(tally, group=group)


def all_reduce_scalar(x: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist
    w = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(w, group=group)
    return float(w.item())


class _CudaArray:
    """__cuda_array_interface__ wrapper of a raw device pointer (zero-copy
    torch view of the library-owned tally)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_tally_tensor(mt, device):
    import torch
    n = mt.mesh.num_elements * mt.num_groups
    return torch.as_tensor(_CudaArray(mt.tally_device_ptr(), n), device=device)


class ShardedMeshTally:
    """``MeshTally`` semantics over a process group: callers pass the GLOBAL
    arrays (or this rank's slice with ``presharded=True``); every rank ends a
    batch with the global moments."""

    def __init__(self, mesh, num_particles: int, num_groups: int = 1, *, group=None,
                 device: int | None = None, presharded: bool = False, _tally_factory=None,
                 **kw):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.num_particles = int(num_particles)
        self.lo, self.hi = shard_bounds(self.num_particles, self.rank, self.world)
        self.presharded = presharded
        self._source_weight = 0.0
        if _tally_factory is None:
            from .tally import MeshTally
            if device is None:
                device = int(os.environ.get("LOCAL_RANK", self.rank))
            self.mt = MeshTally(mesh, max(1, self.hi - self.lo), num_groups, device=device, **kw)
            self.device = torch.device("cuda", device)
            self._tally = device_tally_tensor(self.mt, self.device)
        else:  # test hook: a CPU tally with the same methods + .tally_tensor()
            self.mt = _tally_factory(mesh, max(1, self.hi - self.lo), num_groups)
            self.device = torch.device("cpu")
            self._tally = self.mt.tally_tensor()

    @property
    def mesh(self):
        return self.mt.mesh

    def _local(self, a, count_global, per_particle):
        if self.presharded:
            return a
        a = np.asarray(a)
        lo = min(self.lo, count_global)
        hi = min(self.hi, count_global)
        flat = a.reshape(-1)
        return flat[lo * per_particle:hi * per_particle]

    def initialize_particle_location(self, positions) -> None:
        pos = np.asarray(positions, dtype=np.float64).reshape(-1)
        count = pos.size // 3
        if pos.size != 3 * count:
            raise ValueError(f"positions must hold 3*count = {3 * count} floats, got {pos.size}")
        self.mt.initialize_particle_location(self._local(pos, count, 3))
        self._source_weight = 0.0  # tally.py:245

    def move_to_next_location(self, destinations, flying, weights, groups=None):
        fly = np.asarray(flying).reshape(-1)
        count = fly.size
        if count == 0:  # tally.py:258-260: nothing moved, nothing recorded
            return None
        g = None if groups is None else self._local(groups, count, 1)
        recording = self._source_weight == 0.0
        if recording:
            self.mt.source_weight = 0.0  # this rank records this move's flying weight
        s = self.mt.move_to_next_location(self._local(destinations, count, 3),
                                          self._local(fly, count, 1),
                                          self._local(weights, count, 1), g)
        if recording:
            # The reference records the batch's source weight on the first move
            # whose flying weight is non-zero (tally.py:267-269) -- decided on
            # the GLOBAL move, so a rank whose shard is empty or not flying on
            # that move does not record a later one of its own.
            w = all_reduce_scalar(self.mt.source_weight if s is not None else 0.0,
                                  self.device, self.group)
            self._source_weight = w
            self.mt.source_weight = w if w != 0.0 else 0.0
        return reduce_summary(s, self.device, self.group)

    @property
    def source_weight(self) -> float:
        return self._source_weight

    def finalize_batch(self, source_weight: float | None = None) -> None:
        w = self._source_weight if source_weight is None else float(source_weight)
        if not w or w <= 0.0:
            raise RuntimeError("no source weight recorded for this batch; pass source_weight")
        reduce_tally_(self._tally, self.group)
        self.mt.finalize_batch(w)
        self._source_weight = 0.0

    def flux(self):
        return self.mt.flux()

    def batch_totals(self):
        return self.mt.batch_totals()
