"""FAST schedules (static segments / weighted by issue rank / dynamic claims): bit-identical
states after a few steps (a node's arithmetic does not depend on which unit computes it) and the
device time of each. usage: python tools/sched_check.py CFG... [--modes static,wt,dyn]"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

ENV = {"static": {"SC_FAST_DYN": "0", "SC_FAST_WT": "0"},
       "dyn": {"SC_FAST_DYN": "1", "SC_FAST_WT": "0"},
       "wt": {"SC_FAST_DYN": "0", "SC_FAST_WT": "1"}}
modes = ["static", "wt"]
args = []
for a in sys.argv[1:]:
    if a.startswith("--modes="):
        modes = a.split("=", 1)[1].split(",")
    else:
        args.append(int(a))
steps = 6
for cid in args or [2, 4, 5]:
    cfg, scenes, p, x, v = configs.build(cid, batch=min(configs.CONFIGS[cid].batch, 4096))
    out = {}
    for m in modes:
        os.environ.update(ENV[m])
        with ClothBatch(scenes, p) as cb:
            xs, vs = cb.rollout(x, v, steps, 0, "fast")
            cb.set_state(x, v)
            sec = cb.benchmark(50, 3, "fast")
        out[m] = (xs, vs, sec / 50 * 1e6)
    nodes = cfg.batch * cfg.n * cfg.n
    ref = out[modes[0]]
    line = "cfg%d" % cid
    for m in modes:
        same = all(np.array_equal(out[m][i].view(np.uint32), ref[i].view(np.uint32)) for i in (0, 1))
        line += "  %s %.1f us (%.1f%%)%s" % (m, out[m][2], 100 * nodes * 48 / (out[m][2] * 1e-6) / 6454.6e9,
                                           "" if same else " MISMATCH")
    print(line, flush=True)
