"""Quick device-timed throughput probe for the configs (development aid, not the bench)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("-")]
modes = ["parity", "fast", "fast-perstep"] if "--all" in sys.argv else ["fast", "fast-perstep"]
for cfg_id in [int(a) for a in (args or ["2"])]:
    t0 = time.time()
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=min(configs.CONFIGS[cfg_id].batch, 4096))
    t1 = time.time()
    with ClothBatch(scenes, p) as cb:
        for mode in modes:
            cb.set_state(x, v)
            cb.set_persistent(mode != "fast-perstep")
            steps = 50
            sec = cb.benchmark(steps, 3, "parity" if mode == "parity" else "fast")
            nodes = cfg.batch * cfg.n * cfg.n
            rate = nodes * steps / sec
            print("cfg%d %-12s %8.1f us/step  %.3e node-upd/s  %.1f%% of 6555 GB/s (48 B/node)"
                  % (cfg_id, mode, sec / steps * 1e6, rate, 100 * rate * 48 / 6555.2e9), flush=True)
    print("  (input generation %.1f s)" % (t1 - t0))
