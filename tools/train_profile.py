"""A few compute_loss calls (with gradients) for an ncu launch list of the training kernels."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import paper_2403_12820_b200 as ours  # noqa: E402
from golden_io import scene_arrays, to_scene  # noqa: E402
from make_golden import random_params, sheet  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rng = np.random.default_rng(1)
x0 = sheet(rng, n, n, 1.0 / (n - 1), 1e-3)
sc = scene_arrays(n, n, 1.0 / 240, mass=0.01, drag=0.02, plugs=(0, 1, 1), pin_nodes=[0, n - 1],
                  pin_anchors=x0[[0, n - 1]], stiffness=100.0, damping=0.1, spacing=1.0 / (n - 1))
frames = 200
fx = np.repeat(x0[None], frames, 0) + rng.normal(0, 1e-3, (frames, n * n, 3))
fv = rng.normal(0, 0.1, fx.shape)
with ours.Trainer(to_scene(sc, x0), ours.Trajectory(n, n, 1.0 / 240, 1.0 / (n - 1), fx, fv)) as t:
    t.sample_batch(batch, 1)
    p = ours.NetworkParams.from_scalars(random_params(rng, 0.05, True))
    for _ in range(3):
        t.compute_loss(p, 0.5)
print("ok")
