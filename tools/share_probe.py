"""Strong-scaling shares of config 5 (B / G cloths on one GPU) at the driver's 20 timed steps and
at the config's 300: device time per timestep under chunk-count / segment-length overrides
(development aid).  python tools/share_probe.py [B ...]"""
import json
import os
import sys

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

VARIANTS = [{}, {"SC_CHUNKS": "2"}, {"SC_CHUNKS": "8"}, {"SC_CHUNK_SEG_ROWS": "16"},
            {"SC_CHUNK_SEG_ROWS": "32"}, {"SC_CHUNK_SEG_ROWS": "64"}, {"SC_CHUNK_SEG_ROWS": "128"},
            {"SC_CHUNKS": "2", "SC_CHUNK_SEG_ROWS": "64"}, {"SC_CHUNKS": "8", "SC_CHUNK_SEG_ROWS": "32"}]
for B in [int(a) for a in (sys.argv[1:] or [512, 1024, 2048])]:
    cfg, scenes, p, x, v = configs.build(5, batch=B)
    for var in VARIANTS:
        for k in ("SC_CHUNKS", "SC_CHUNK_SEG_ROWS"):
            os.environ.pop(k, None)
        os.environ.update(var)
        res = {}
        with ClothBatch(scenes, p) as cb:
            for steps in (20, 300):
                cb.set_state(x, v)
                cb.benchmark(20, 3, "fast")
                best = min(cb.benchmark(steps, 3, "fast") for _ in range(3))
                res[steps] = round(best / steps * 1e6, 2)
        print(json.dumps({"B": B, "env": var, "us_per_step": res}), flush=True)
