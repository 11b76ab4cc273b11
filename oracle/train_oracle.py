"""TEST INFRASTRUCTURE ONLY — CPU restatement of the training path.

Plain Python double arithmetic in the reference's operation and summation order, for small
cases (a few hundred nodes); the per-node forward / plug / advance operators come from the C
restatement (oracle.c via pyoracle.Oracle, f64). Checked against the reference-generated fixture
tests/golden/train_f64.npz by tests/test_train_oracle.py. Nothing in the product imports this.

  sample_targets     train.cpp:111-124   (elastic_force / damping_force / pressure_force,
                                          kernels.hpp:86-155, each on a zero field)
  backward_gradients net.cpp:144-201     (fixed 1024-node chunks, chunk partials in order)
  compute_loss       train.cpp:129-209
"""
from __future__ import annotations

import math

import numpy as np

OFFSETS = [(1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, 1), (-1, -1), (1, -1),
           (2, 0), (0, 2), (-2, 0), (0, -2)]  # grid.cpp:14-27 canonical channel order
REST_MULT = [1.0] * 4 + [math.sqrt(2.0)] * 4 + [2.0] * 4


def _nb(i, c, nx, ny):
    ix, iy = i % nx, i // nx
    jx, jy = ix + OFFSETS[c][0], iy + OFFSETS[c][1]
    if 0 <= jx < nx and 0 <= jy < ny:
        return jy * nx + jx
    return -1


def _dot(a, b):
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]


def sample_targets(nx, ny, x, v, sc):
    """f_k * dt for one frame (train.cpp:111-124); sc: dict of the scene arrays (golden_io)."""
    n = nx * ny
    stiff, damp = float(sc["stiffness"]), float(sc["damping"])
    rest = [float(sc["spacing"]) * m for m in REST_MULT]
    mass, dt, drag, pressure = (float(sc["mass"]), float(sc["dt"]), float(sc["drag"]),
                                float(sc["pressure"]))
    plug_p, plug_g, plug_d = (int(p) for p in sc["plugs"])
    grav = [float(g) for g in sc["gravity"]]
    out = np.zeros((n, 3))
    for i in range(n):
        xi, vi = x[i].tolist(), v[i].tolist()
        E = [0.0, 0.0, 0.0]
        D = [0.0, 0.0, 0.0]
        for c in range(12):  # accumulate_elastic (kernels.hpp:86-108)
            j = _nb(i, c, nx, ny)
            if j < 0:
                continue
            d = [xi[k] - x[j][k] for k in range(3)]
            ln = math.sqrt(_dot(d, d))
            if ln == 0.0:
                raise ArithmeticError("elastic force: singular spring (coincident nodes) at node %d"
                                      % i)
            s = stiff * (ln - rest[c]) / ln
            E = [E[k] - d[k] * s for k in range(3)]
        for c in range(12):  # accumulate_damping (kernels.hpp:112-136)
            j = _nb(i, c, nx, ny)
            if j < 0:
                continue
            d = [xi[k] - x[j][k] for k in range(3)]
            ln = math.sqrt(_dot(d, d))
            if ln == 0.0:
                continue
            dr = [d[k] / ln for k in range(3)]
            dv = [vi[k] - v[j][k] for k in range(3)]
            s = damp * _dot(dv, dr)
            D = [D[k] - dr[k] * s for k in range(3)]
        f = [E[k] + D[k] for k in range(3)]
        if not plug_p:  # pressure_force on a zero field (kernels.hpp:142-155), added
            fp = [0.0, 0.0, 0.0]
            ix, iy = i % nx, i // nx
            if pressure != 0.0 and 1 <= ix <= nx - 2 and 1 <= iy <= ny - 2:
                e = [xi[k] - x[i + 1][k] for k in range(3)]
                nn = [xi[k] - x[i + nx][k] for k in range(3)]
                w = [xi[k] - x[i - 1][k] for k in range(3)]
                s_ = [xi[k] - x[i - nx][k] for k in range(3)]

                def cross(p, q):
                    return [p[1] * q[2] - p[2] * q[1], p[2] * q[0] - p[0] * q[2],
                            p[0] * q[1] - p[1] * q[0]]
                c1, c2, c3, c4 = cross(e, nn), cross(nn, w), cross(w, s_), cross(s_, e)
                fp = [0.0 + ((c1[k] + c2[k]) + c3[k] + c4[k]) * pressure for k in range(3)]
            f = [f[k] + fp[k] for k in range(3)]
        g = [0.0, 0.0, 0.0] if plug_g else grav
        dd = 0.0 if plug_d else drag
        out[i] = [((f[k] + g[k] * mass) - vi[k] * dd) * dt for k in range(3)]
    return out


def backward_gradients(nx, ny, x, v, p, upstream):
    """The 53 gradient sums (net.cpp:144-201); p: the 53 scalars in for_each_scalar order."""
    n = nx * ny
    gain, wl, wn, wd = p[0:12], p[12:24], p[27:39], p[39:51]
    alpha = p[52]
    total = [0.0] * 53
    for c0 in range(0, n, 1024):
        g = [0.0] * 53  # ParamGradients{} of this chunk
        for i in range(c0, min(n, c0 + 1024)):
            u = upstream[i].tolist()
            xi, vi = x[i].tolist(), v[i].tolist()
            for k in range(3):
                g[24 + k] += u[k]
            g[51] += _dot(u, vi)
            for c in range(12):
                j = _nb(i, c, nx, ny)
                if j < 0:
                    continue
                dx = [xi[k] - x[j][k] for k in range(3)]
                dv = [vi[k] - v[j][k] for k in range(3)]
                phi = [dx[k] * gain[c] for k in range(3)]
                xi_ = [dv[k] * gain[c] for k in range(3)]
                s, sp, sa = [0.0] * 3, [0.0] * 3, [0.0] * 3
                for k in range(3):
                    z = phi[k]
                    q = 1.0 + alpha * z * z
                    rq = 1.0 / math.sqrt(q)
                    s[k] = z * rq
                    sp[k] = rq / q
                    sa[k] = -0.5 * z * z * z * rq / q
                g[12 + c] += _dot(u, phi)
                g[27 + c] += _dot(u, s)
                g[39 + c] += _dot(u, [xi_[k] * s[k] for k in range(3)])
                kk = [(dx[k] * wl[c] + (sp[k] * dx[k]) * wn[c])
                      + (dv[k] * s[k] + xi_[k] * (sp[k] * dx[k])) * wd[c] for k in range(3)]
                g[c] += _dot(u, kk)
                aa = [sa[k] * wn[c] + (xi_[k] * sa[k]) * wd[c] for k in range(3)]
                g[52] += _dot(u, aa)
        total = [total[k] + g[k] * 1.0 for k in range(53)]
    return np.array(total)


def compute_loss(nx, ny, frames_x, frames_v, indices, targets, p, alpha, sc, cloth, oracle):
    """compute_loss (train.cpp:129-209) -> ((total, physics, data), 53 gradients); `cloth` the
    sc_cloth_desc and `oracle` a pyoracle.Oracle for the per-node f64 operators."""
    from golden_io import params_c
    n = nx * ny
    pc = params_c(p)
    dt = float(sc["dt"])
    inv_mass = 1.0 / float(sc["mass"])
    pinned = set(int(i) for i in sc["pin_nodes"])
    free_count = n - len(pinned)
    phys_sq = data_sq = 0.0
    data_count = 0
    res = []
    for b, k in enumerate(indices):
        x, v = frames_x[k], frames_v[k]
        imp = oracle.forward_impulse(nx, ny, pc, x, v)
        applied = imp + oracle.plug_impulse(nx, ny, cloth, x, v)
        xo, vo, mask = oracle.advance_with_impulse(nx, ny, cloth, x, v, applied, (k + 1) * dt)
        rp = np.zeros((n, 3))
        rd = np.zeros((n, 3))
        for i in range(n):
            if i in pinned:
                continue
            r = [imp[i][q] - targets[b][i][q] * inv_mass for q in range(3)]
            phys_sq += _dot(r, r)
            rp[i] = r
            if mask[i]:
                continue
            rv = [vo[i][q] - frames_v[k + 1][i][q] for q in range(3)]
            rx = [xo[i][q] - frames_x[k + 1][i][q] for q in range(3)]
            data_sq += _dot(rv, rv) + _dot(rx, rx)
            data_count += 1
            rd[i] = [rv[q] + rx[q] * dt for q in range(3)]
        res.append((rp, rd))
    phys_denom = 3.0 * len(indices) * free_count
    data_denom = 6.0 * data_count
    physics = phys_sq / phys_denom if free_count > 0 else 0.0
    data = data_sq / data_denom if data_count > 0 else 0.0
    total = alpha * physics + (1.0 - alpha) * data
    pcoef = 2.0 * alpha / phys_denom if free_count > 0 else 0.0
    dcoef = 2.0 * (1.0 - alpha) / data_denom if data_count > 0 else 0.0
    grads = [0.0] * 53
    for b, k in enumerate(indices):
        rp, rd = res[b]
        up = rp * pcoef + rd * dcoef
        g = backward_gradients(nx, ny, frames_x[k], frames_v[k], list(p), up)
        grads = [grads[q] + g[q] * 1.0 for q in range(53)]
    return np.array([total, physics, data]), np.array(grads)
