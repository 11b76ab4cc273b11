"""Device-timed config-5 stepping for short timed windows (the driver's `--steps 20`) under
several environment settings, inputs built once: prints us per timestep (best of 3) per setting.
Usage: python tools/k_probe.py K1,K2,.. "ENV=V,ENV2=V2" "ENV=V" ...   (empty string = defaults)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

Ks = [int(t) for t in sys.argv[1].split(",")]
cid = int(os.environ.get("PROBE_CONFIG", "5"))
cfg, scenes, p, x, v = configs.build(cid, threads=16)
nodes = cfg.batch * cfg.n * cfg.n
for spec in sys.argv[2:]:
    kv = [t.split("=") for t in spec.split(",") if t]
    for k, val in kv:
        os.environ[k] = val
    with ClothBatch(scenes, p) as cb:
        for K in Ks:
            best = None
            for _ in range(3):
                cb.set_state(x, v)
                cb.advance(5, 0, "fast")
                sec = cb.benchmark(K, 0, "fast")
                best = sec if best is None else min(best, sec)
            print("cfg%d K=%d %-40s %8.2f us/step  %.3e node-upd/s"
                  % (cid, K, spec or "default", best / K * 1e6, nodes * K / best), flush=True)
    for k, _ in kv:
        del os.environ[k]
