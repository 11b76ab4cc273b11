"""Bit-identity of two library builds on sphere-contact scenes (development aid): each build
(SC_B200_LIB, or "tree") steps the same contact-heavy scenes in its own process and prints a hash
of the states and masks; also times the contact phase of config 3 (timesteps 20-70).
  python tools/contact_ab.py LIB [LIB ...]"""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import hashlib, sys
sys.path.insert(0, %(root)r)
import numpy as np
from paper_2403_12820_b200 import ClothBatch, configs
from paper_2403_12820_b200.scene import SphereCollider
h = hashlib.sha256()
for n, cz, fr in ((256, -0.27, 0.0), (384, -0.29, 0.3), (128, -0.25, 0.0), (512, -0.31, 0.1)):
    cfg, scenes, p, x, v = configs.build(3, batch=1, n=n)
    scenes[0].colliders[:] = [SphereCollider(np.array([0.47, 0.52, cz]), 0.3, fr)]
    with ClothBatch(scenes, p) as cb:
        xs, vs = x, v
        for k in range(8):
            xs, vs, m = cb.rollout(xs, vs, 1, k, "fast", constrained=True)
            h.update(xs.tobytes()); h.update(vs.tobytes()); h.update(m.tobytes())
        xr, vr = cb.rollout(x, v, 12, 0, "fast")
        h.update(xr.tobytes()); h.update(vr.tobytes())
        touched = int(m.sum())
cfg, scenes, p, x, v = configs.build(3)
with ClothBatch(scenes, p) as cb:
    cb.set_state(x, v)
    cb.advance(20, 0, "fast")
    t = min(cb.benchmark(50, 0, "fast") for _ in range(1))
    xs, vs = cb.get_state()
    h.update(xs.tobytes())
print(h.hexdigest()[:16], "contacts(last scene) %%d, config 3 timesteps 20-70: %%.2f us/step" %% (touched, t / 50 * 1e6))
"""
for lib in sys.argv[1:]:
    env = dict(os.environ)
    if lib != "tree":
        env["SC_B200_LIB"] = os.path.abspath(lib)
    out = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=env,
                         capture_output=True, text=True, timeout=900)
    print("%-12s %s" % (os.path.basename(lib), out.stdout.strip() or out.stderr[-600:]), flush=True)
