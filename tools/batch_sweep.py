"""Per-step time of config 2's cloth at growing batch sizes (development aid): separates the
fixed per-step costs (launch, wave tail, segment prologue/epilogue) from the per-node rate."""
import sys

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for B in [int(b) for b in (sys.argv[2:] or ["16", "32", "64", "128", "256", "512"])]:
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=B)
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        cb.set_persistent(False)
        steps = 50
        sec = cb.benchmark(steps, 3, "fast")
        nodes = B * cfg.n * cfg.n
        print("cfg%d batch %5d  %8.1f us/step  %.3e node-upd/s  %.1f%% of roofline"
              % (cfg_id, B, sec / steps * 1e6, nodes * steps / sec,
                 100 * nodes * steps / sec * 48 / 6555.2e9), flush=True)
