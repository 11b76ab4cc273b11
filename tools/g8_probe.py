"""Config-5 share per GPU at small batches: device time per step of the default stepping vs
environment overrides (development aid for the strong-scaling shares).
  python tools/g8_probe.py [B ...]"""
import sys, json, os
sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs
for B in [int(a) for a in (sys.argv[1:] or [512, 1024])]:
    cfg, scenes, p, x, v = configs.build(5, batch=B)
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        cb.benchmark(20, 3, "fast")
        sec = cb.benchmark(300, 3, "fast")
    print(json.dumps({"B": B, "env": {k: os.environ.get(k) for k in ("SC_WAVE", "SC_GROUP_SMS", "SC_GROUP")}, "us": sec / 300 * 1e6}), flush=True)
