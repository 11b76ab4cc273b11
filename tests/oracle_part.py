"""Test helper: a `part` for paper_2403_12820_b200.DistributedTrainer computed on the CPU by the
training oracle (oracle/train_oracle.py + oracle.c), so the data-parallel orchestration can be
tested over gloo without a GPU. Same interface as dist_train.CudaPart."""
import math

import numpy as np

from golden_io import cloth_desc, params_c
from oracle import train_oracle as T
from oracle.pyoracle import Oracle

_OFF = T.OFFSETS


class OraclePart:
    def __init__(self, z, frames_x, frames_v):
        """z: fixture-style scene arrays (golden_io.scene_arrays); frames: [F][n][3] f64."""
        self.z, self.fx, self.fv = z, frames_x, frames_v
        self.nx, self.ny = int(z["nx"]), int(z["ny"])
        self.n = self.nx * self.ny
        self.frames = frames_x.shape[0]
        self.n_free = self.n - len(z["pin_nodes"])
        self.keep = []
        self.cd = cloth_desc(z, self.keep)
        self.oracle = Oracle()
        self.pinned = set(int(i) for i in z["pin_nodes"])

    def set_batch(self, indices):
        self.indices = [int(i) for i in indices]
        self.targets = [T.sample_targets(self.nx, self.ny, self.fx[k], self.fv[k], self.z)
                        for k in self.indices]

    def forward(self, params, b0, b1):
        self.b0 = b0
        p = params.scalars()
        pc = params_c(p)
        dt = float(self.z["dt"])
        inv_mass = 1.0 / float(self.z["mass"])
        self.pt, self.dm, self.res = [], [], []
        count, bad = 0, (-1, -1)
        for b in range(b0, b1):
            k = self.indices[b]
            x, v = self.fx[k], self.fv[k]
            imp = self.oracle.forward_impulse(self.nx, self.ny, pc, x, v)
            if bad[0] < 0:
                nf = np.where(~np.isfinite(imp).all(axis=1))[0]
                if len(nf):
                    bad = (b, int(nf[0]))
            applied = imp + self.oracle.plug_impulse(self.nx, self.ny, self.cd, x, v)
            xo, vo, mask = self.oracle.advance_with_impulse(self.nx, self.ny, self.cd, x, v, applied,
                                                            (k + 1) * dt)
            pt, dm = [0.0] * self.n, [0.0] * self.n
            rp, rd = np.zeros((self.n, 3)), np.zeros((self.n, 3))
            for i in range(self.n):
                if i in self.pinned:
                    continue
                r = [imp[i][q] - self.targets[b][i][q] * inv_mass for q in range(3)]
                pt[i] = T._dot(r, r)
                rp[i] = r
                if mask[i]:
                    continue
                rv = [vo[i][q] - self.fv[k + 1][i][q] for q in range(3)]
                rx = [xo[i][q] - self.fx[k + 1][i][q] for q in range(3)]
                dm[i] = T._dot(rv, rv) + T._dot(rx, rx)
                count += 1
                rd[i] = [rv[q] + rx[q] * dt for q in range(3)]
            self.pt.append(pt)
            self.dm.append(dm)
            self.res.append((rp, rd))
        return count, bad[0], bad[1]

    def chain(self, ps, ds):
        for j, (pt, dm) in enumerate(zip(self.pt, self.dm)):
            for i in range(self.n):
                ps += pt[i]
                ds += dm[i]
            if not (math.isfinite(ps) and math.isfinite(ds)):
                return ps, ds, self.b0 + j
        return ps, ds, -1

    def backward(self, params, alpha, count, batch, nb):
        p = params.scalars()
        phys_denom = 3.0 * float(batch) * self.n_free
        pc = 2.0 * alpha / phys_denom if self.n_free > 0 else 0.0
        dc = 2.0 * (1.0 - alpha) / (6.0 * float(count)) if count > 0 else 0.0
        out = np.zeros((nb, 53))
        for j in range(nb):
            k = self.indices[self.b0 + j]
            rp, rd = self.res[j]
            out[j] = T.backward_gradients(self.nx, self.ny, self.fx[k], self.fv[k], p,
                                          rp * pc + rd * dc)
        return out

    def diagnose(self, params, frame, node):
        from paper_2403_12820_b200.api import _diagnose_forward
        from golden_io import to_scene
        return _diagnose_forward(self.fx[frame], self.fv[frame], to_scene(self.z, self.fx[0]),
                                 params, node)
