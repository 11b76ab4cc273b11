"""FAST schedule independence: states after a few steps are bit-identical whatever the row
segmentation (a node's arithmetic does not depend on which unit computes it), plus the device
time per segmentation. usage: python tools/sched_check.py CFG... [--seg=0,8,15]  (0 = planner)"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

segs = ["0"]
args = []
for a in sys.argv[1:]:
    if a.startswith("--seg="):
        segs = a.split("=", 1)[1].split(",")
    else:
        args.append(int(a))
steps = 6
for cid in args or [2, 4, 5]:
    cfg, scenes, p, x, v = configs.build(cid, batch=min(configs.CONFIGS[cid].batch, 4096))
    out = {}
    for sr in segs:
        if sr == "0":
            os.environ.pop("SC_FAST_SEG_ROWS", None)
        else:
            os.environ["SC_FAST_SEG_ROWS"] = sr
        with ClothBatch(scenes, p) as cb:
            xs, vs = cb.rollout(x, v, steps, 0, "fast")
            cb.set_state(x, v)
            sec = cb.benchmark(50, 3, "fast")
        out[sr] = (xs, vs, sec / 50 * 1e6)
    nodes = cfg.batch * cfg.n * cfg.n
    ref = out[segs[0]]
    line = "cfg%d" % cid
    for sr in segs:
        same = all(np.array_equal(out[sr][i].view(np.uint32), ref[i].view(np.uint32)) for i in (0, 1))
        line += "  seg=%s %.1f us (%.1f%%)%s" % (sr, out[sr][2], 100 * nodes * 48 / (out[sr][2] * 1e-6) / 6454.6e9,
                                               "" if same else " MISMATCH")
    print(line, flush=True)
