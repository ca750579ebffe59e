"""Transport RNG-phase threshold sweep (BT_OPT_RNG_WAIT) on the paper's
verification physics.  The draws are keyed by block index, so
every setting must give the same integer totals (events, collisions, sweeps);
one JSON line per setting.
    python tools/transport_wait_sweep.py [particles] [waits, comma-separated]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh  # noqa: E402
from paper_2504_19048_b200 import transport as T  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
waits = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,4,8,12,16,20,24,32").split(",")]
mesh = build_cube_mesh(10)
cfg = T.RunConfig(mesh_n=10, num_particles=P, num_batches=2, seed=42)
ref = None
for rep in range(2):
    for w in waits:
        mt = MeshTally(mesh, P)
        if w:  # 0: leave the library's default (also for builds without the option)
            mt.set_option(_lib.BT_OPT_RNG_WAIT, w)
        T.run(T.RunConfig(mesh_n=10, num_particles=min(P, 20000), num_batches=1), mesh, tally=mt)
        mt.close()
        mt = MeshTally(mesh, P)
        if w:
            mt.set_option(_lib.BT_OPT_RNG_WAIT, w)
        r = T.run(cfg, mesh, tally=mt)
        key = (r.events, r.collisions, r.sweeps)
        if ref is None:
            ref = key
        print(json.dumps({"rng_wait": w, "rep": rep, "particles": P, "events": r.events,
                          "collisions": r.collisions, "sweeps": r.sweeps,
                          "t_transport_s": r.t_batch,
                          "events_per_s": r.events / r.t_batch,
                          "collisions_per_s": r.collisions / r.t_batch,
                          "same_totals": key == ref}), flush=True)
        mt.close()
