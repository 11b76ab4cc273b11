"""PBS (ground-truth mass-spring) step device time, f32 and f64 (development aid)."""
import sys

sys.path.insert(0, ".")
from paper_2403_12820_b200 import configs  # noqa: E402
from paper_2403_12820_b200.api import Context  # noqa: E402

for cid in [int(a) for a in sys.argv[1:]] or [2]:
    cfg, scenes, p, x, v = configs.build(cid, batch=min(configs.CONFIGS[cid].batch, 4096))
    for prec in ("f32", "f64"):
        with Context(scenes, p, precision=prec) as cb:
            cb.set_state(x, v)
            sec = cb.benchmark_sim(10, 2)
            print("cfg%d pbs %s %.1f us/step" % (cid, prec, sec / 10 * 1e6), flush=True)
