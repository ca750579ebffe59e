"""Evidence for the walk's optional techniques named by the north star
(particle sorting by element, warp-aggregated __match_any_sync atomics, the
staged refill) on C2 (998,250 tets, 1e7 particles): a uniform source and a
point source (every particle starts in one element, the atomics' worst case),
each at sigma_t = 2 (long flights) and 100 (paper physics, ~1.4 crossings).
    python tools/options_sweep.py [--out profiles/r01_options.jsonl]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from sweep import run_point  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--particles", type=int, default=10_000_000)
ap.add_argument("--only", default=None, help="comma-separated option names to run")
args = ap.parse_args()

import torch  # noqa: E402

from paper_2504_19048_b200 import build_cube_mesh  # noqa: E402

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(7)
m = build_cube_mesh(55)
n = args.particles
uniform = 0.05 + 0.9 * torch.rand(n, 3, generator=gen, device=dev, dtype=torch.float64)
point = torch.tensor([[0.5123456789, 0.4876543211, 0.5031415926]], dtype=torch.float64,
                     device=dev).expand(n, 3).contiguous()
OPTS = [("default", {}), ("sort", {"sort": True}),
        ("warp_aggregate_always", {"warp_aggregate": True}),
        ("warp_aggregate_never", {"warp_aggregate": False}), ("unstaged", {"staged": False}),
        ("stage_kernel", {"staged": 1}), ("direct", {"staged": 2})]
res = []
for src_name, src in (("uniform", uniform), ("point", point)):
    for sigma in (2.0, 100.0):
        for name, kw in OPTS:
            if args.only and name not in args.only.split(","):
                continue
            r = run_point(m, src, sigma, 1, f"C2 {src_name} sigma_t={sigma:g} {name}", **kw)
            r.update(source=src_name, option=name)
            res.append(r)
if args.out:
    Path(args.out).write_text("\n".join(json.dumps(r) for r in res) + "\n")
