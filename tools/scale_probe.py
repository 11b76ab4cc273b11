"""Strong-scaling estimate on one GPU (development aid): config 5's per-rank share at G = 1, 2,
4, 8 ranks (4096 / G cloths of the same seeded stream, rank 0's slice) stepped device-resident;
efficiency(G) = T(4096) / (G x T(4096 / G)) is what the driver's scaling run would see if the
ranks' GPUs are independent (batch sharding has no data-path collective).
  python tools/scale_probe.py [--steps 300]"""
import argparse
import json
import sys

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=300)
ap.add_argument("--cfg", type=int, default=5)
args = ap.parse_args()
B = configs.CONFIGS[args.cfg].batch
t = {}
for G in (1, 2, 4, 8):
    cfg, scenes, p, x, v = configs.build(args.cfg, batch=B // G)
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        cb.benchmark(20, 3, "fast")
        sec = cb.benchmark(args.steps, 3, "fast")
    t[G] = sec / args.steps
    print(json.dumps({"G": G, "cloths": B // G, "us_per_step": t[G] * 1e6,
                      "efficiency": t[1] / (G * t[G])}), flush=True)
