import sys
sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs
cfg, scenes, p, x, v = configs.build(5)
for label in ["with planes", "planes removed"]:
    if label == "planes removed":
        for s in scenes:
            s.planes = []
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        cb.set_persistent(False)
        sec = cb.benchmark(30, 3, "fast")
        rate = cfg.batch * cfg.n * cfg.n * 30 / sec
        print("%-15s %8.1f us/step  %.1f%% of roofline" % (label, sec / 30 * 1e6, 100 * rate * 48 / 6555.2e9), flush=True)
