"""Device transport throughput on the paper's verification
physics (n=10 cube, sigma_t = sigma_s = 100/cm, source in 1/8 of
the domain), per launch variant; one JSON line per point.
    python tools/transport_bench.py [particles] [batches]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_19048_b200 import MeshTally, _lib, build_cube_mesh  # noqa: E402
from paper_2504_19048_b200 import transport as T  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mesh = build_cube_mesh(10)
for variant, label, wagg in ((0, "192x2", None), (0, "192x2", False), (1, "256x1", None)):
    cfg = T.RunConfig(mesh_n=10, num_particles=P, num_batches=B, seed=42)
    mt = MeshTally(mesh, P, warp_aggregate=wagg)
    mt.set_option(_lib.BT_OPT_BLOCKS_PER_SM, variant)
    T.run(cfg, mesh, tally=mt)  # warm-up
    mt.close()
    mt = MeshTally(mesh, P, warp_aggregate=wagg)
    mt.set_option(_lib.BT_OPT_BLOCKS_PER_SM, variant)
    r = T.run(cfg, mesh, tally=mt)
    print(json.dumps({"point": f"transport paper physics N={P}", "variant": label,
                      "warp_aggregate": "adaptive" if wagg is None else wagg,
                      "elements": mesh.num_elements, "particles": P, "batches": B,
                      "events": r.events, "collisions": r.collisions,
                      "t_transport_s": r.t_batch, "t_localization_s": r.t_localization,
                      "events_per_s": r.events / r.t_batch,
                      "collisions_per_s": r.collisions / r.t_batch,
                      "histories_per_s": P * B / r.t_batch}), flush=True)
    mt.close()
