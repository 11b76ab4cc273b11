import sys, time
sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs
cfg, scenes, p, x, v = configs.build(2)
with ClothBatch(scenes, p) as cb:
    cb.set_state(x, v)
    out = []
    for i in range(12):
        sec = cb.benchmark(250, 0, "fast")
        out.append(round(sec / 250 * 1e6, 2))
    print("12 x 250 steps, us/step:", out)
    sec = cb.benchmark(3000, 0, "fast")
    print("one 3000-step call:", round(sec / 3000 * 1e6, 2))
    out = []
    for i in range(6):
        sec = cb.benchmark(250, 0, "fast")
        out.append(round(sec / 250 * 1e6, 2))
        time.sleep(0.2)
    print("6 x 250 with 0.2 s pauses:", out)
