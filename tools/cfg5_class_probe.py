"""Config 5 FAST step time with the mixed classes vs simple-only / plane-only cloth sets
(estimates what grouping cloths by boundary class could buy; development aid).
SC_ZSWIZZLE=0/1 in the environment forces the z layout (1 on a collider-free set runs the
general-finish kernel on it)."""
import sys

sys.path.insert(0, ".")
import paper_2403_12820_b200.configs as C  # noqa: E402
from paper_2403_12820_b200 import ClothBatch  # noqa: E402

base = C.cloth_kind
sets = {"mixed": base, "simple-only": lambda cfg, b: ("top_row", "corners")[b % 2],
        "plane-only": lambda cfg, b: "free"}
import os
STEPS = int(os.environ.get("PROBE_STEPS", "300"))
for label in (sys.argv[1:] or list(sets)):
    C.cloth_kind = sets[label]
    cfg, scenes, p, x, v = C.build(5)
    for persistent in (True, False):
        with ClothBatch(scenes, p) as cb:
            cb.set_persistent(persistent)
            cb.set_state(x, v)
            sec = cb.benchmark(STEPS, 3, "fast")
        print(label, "wave" if persistent else "stream", "%.1f us/step" % (sec / STEPS * 1e6),
              "%.3g node-updates/s" % (x.shape[0] * x.shape[1] * STEPS / sec), flush=True)
C.cloth_kind = base
