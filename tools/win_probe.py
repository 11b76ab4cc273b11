import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2403_12820_b200 import ClothBatch, configs
cfg, scenes, p, x, v = configs.build(3)
with ClothBatch(scenes, p) as cb:
    for rep in range(2):
        cb.set_state(x, v)
        out = []
        for w in range(40):
            sec = cb.benchmark(10, 0, "fast")
            out.append(sec / 10 * 1e6)
        print(" ".join("%.1f" % t for t in out))
    cb.set_state(x, v)
    for w in range(12):
        cb.advance(10, 10 * w, "fast")
        xs, vs = cb.get_state()
        print(w * 10 + 10, "z range %.3f %.3f  |v|max %.3g  finite %s" % (xs[..., 2].min(), xs[..., 2].max(), np.abs(vs).max(), np.isfinite(xs).all()))
