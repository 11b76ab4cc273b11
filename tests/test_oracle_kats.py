"""The reference's own known-answer tests for this path, restated against the C oracle (CPU).

The golden fixtures pin the oracle bit for bit to the reference build (test_oracle_golden.py);
these pin it independently of any fixture, with the reference's test logic:
  * cell vs a from-scratch evaluation in another association order, <= 1e-12
    (/root/reference/proj/tests/test_net.cpp:104-116, oracle cell_forward oracles.hpp:146-167);
  * zero weights -> zero impulse, the bias passes straight through (test_net.cpp:118-125);
  * nn_step = cell + gravity + drag closed form, <= 1e-14 (test_net.cpp:212-239);
  * sphere response: outside untouched, inside+approaching projected with the inward normal
    removed and the tangent scaled by 1 - friction, inside+receding projected with v kept, the
    centre left alone (test_sim.cpp:207-229);
  * pins exactly on the anchor path anchor + u * t (test_sim.cpp:190-205, 269-281).
"""
import ctypes as C

import numpy as np

from golden_io import cloth_desc, scene_arrays
from paper_2403_12820_b200 import _abi

OFFS = [(1, 0), (0, 1), (-1, 0), (0, -1), (1, 1), (-1, 1), (-1, -1), (1, -1), (2, 0), (0, 2),
        (-2, 0), (0, -2)]


def params(rng, zero=False):
    p = _abi.sc_params()
    for c in range(12):
        p.kernel_gain[c] = 1.0 if zero else rng.uniform(0.5, 1.5)
        p.linear_w[c] = 0.0 if zero else rng.normal(0, 0.3)
        p.nonlinear_w[c] = 0.0 if zero else rng.normal(0, 0.3)
        p.deriv_w[c] = 0.0 if zero else rng.normal(0, 0.3)
    for d in range(3):
        p.linear_b[d] = 0.0 if zero else rng.normal(0, 0.1)
    p.self_velocity_w = 0.0 if zero else rng.normal(0, 0.3)
    p.isru_alpha = 1.0 if zero else rng.uniform(0.5, 2.0)
    return p


def cell_from_scratch(x, v, nx, ny, p):
    """Per node: acc = b + v w_V, then += phi wL, += sigma wN, += (xi * sigma) wD per channel
    (three separate accumulations, unlike the reference's fused t = ... expression)."""
    out = np.zeros_like(x)
    g = np.array(p.kernel_gain[:])
    for iy in range(ny):
        for ix in range(nx):
            i = iy * nx + ix
            acc = np.array(p.linear_b[:]) + v[i] * p.self_velocity_w
            for c, (dx, dy) in enumerate(OFFS):
                jx, jy = ix + dx, iy + dy
                if not (0 <= jx < nx and 0 <= jy < ny):
                    continue
                j = jy * nx + jx
                phi = (x[i] - x[j]) * g[c]
                xi = (v[i] - v[j]) * g[c]
                sig = phi / np.sqrt(1.0 + p.isru_alpha * phi * phi)
                acc = acc + phi * p.linear_w[c]
                acc = acc + sig * p.nonlinear_w[c]
                acc = acc + (xi * sig) * p.deriv_w[c]
            out[i] = acc
    return out


def test_cell_matches_from_scratch_evaluation(oracle):
    rng = np.random.default_rng(17)
    for _ in range(8):
        nx, ny = int(rng.integers(3, 9)), int(rng.integers(3, 9))
        gx, gy = np.meshgrid(np.arange(nx) * 0.1, np.arange(ny) * 0.1)
        x = np.stack([gx.ravel(), gy.ravel(), np.zeros(nx * ny)], 1)
        x = x + rng.normal(0, 0.05, x.shape)
        v = rng.normal(0, 1.5, x.shape)
        p = params(rng)
        got = oracle.forward_impulse(nx, ny, p, x, v)
        want = cell_from_scratch(x, v, nx, ny, p)
        assert np.abs(got - want).max() <= 1e-12


def test_zero_weights_zero_impulse_and_bias_passthrough(oracle):
    nx = ny = 4
    gx, gy = np.meshgrid(np.arange(nx) * 0.1, np.arange(ny) * 0.1)
    x = np.stack([gx.ravel(), gy.ravel(), np.zeros(nx * ny)], 1)
    v = np.zeros_like(x)
    p = params(None, zero=True)
    for dt in (np.float64, np.float32):
        assert np.array_equal(oracle.forward_impulse(nx, ny, p, x.astype(dt), v.astype(dt)),
                              np.zeros_like(x, dt))
    p.linear_b[0], p.linear_b[1], p.linear_b[2] = 0.1, -0.2, 0.3
    out = oracle.forward_impulse(nx, ny, p, x, v)
    assert (out == np.array([0.1, -0.2, 0.3])).all()


def test_nn_step_plugs_gravity_and_drag_closed_form(oracle):
    nx = ny = 4
    dt, mass, drag, g = 0.01, 0.5, 0.3, np.array([0.0, 0.0, -9.8])
    keep = []
    cd = cloth_desc(scene_arrays(nx, ny, dt, mass=mass, drag=drag, gravity=g, plugs=(0, 1, 1)),
                    keep)
    gx, gy = np.meshgrid(np.arange(nx) * 0.1, np.arange(ny) * 0.1)
    x = np.stack([gx.ravel(), gy.ravel(), np.zeros(nx * ny)], 1)
    v = np.tile([0.2, -0.1, 0.4], (nx * ny, 1))
    xo, vo, _, _ = oracle.nn_step(nx, ny, cd, params(None, zero=True), x, v, dt)
    want_v = v + g * dt - v * (drag * dt / mass)
    assert np.linalg.norm(vo - want_v, axis=1).max() <= 1e-14
    assert np.linalg.norm(xo - (x + vo * dt), axis=1).max() <= 1e-14


def test_sphere_response_known_answers(oracle):
    # four nodes of a 2x2 grid at the KAT positions; dt = 0 keeps x' = x so the position pass
    # sees exactly the listed points (test_sim.cpp:207-229)
    keep = []
    cd = cloth_desc(scene_arrays(2, 2, 1.0, plugs=(0, 0, 0), spheres=[(0, 0, 0, 1.0, 0.25)]),
                    keep)
    cd.dt = 0.0
    x = np.array([[2.0, 0, 0], [0.5, 0, 0], [0, 0.5, 0], [0, 0, 0]])
    v = np.array([[-1.0, 0, 0], [-3, 2, 0], [0, 4, 1], [1, 1, 1]])
    xo, vo, m = oracle.advance_with_impulse(2, 2, cd, x, v, np.zeros_like(x), 0.0)
    assert (xo[0] == x[0]).all() and (vo[0] == v[0]).all() and m[0] == 0
    assert abs(np.linalg.norm(xo[1]) - 1.0) <= 1e-12 and abs(xo[1][0] - 1.0) <= 1e-12
    assert abs(vo[1][0]) <= 1e-12 and abs(vo[1][1] - 2.0 * 0.75) <= 1e-12 and m[1] == 1
    assert abs(np.linalg.norm(xo[2]) - 1.0) <= 1e-12 and (vo[2] == v[2]).all()
    assert (xo[3] == x[3]).all() and (vo[3] == v[3]).all() and m[3] == 0


def test_pins_follow_the_anchor_path_exactly(oracle):
    nx = ny = 4
    gx, gy = np.meshgrid(np.arange(nx) * 0.1, np.arange(ny) * 0.1)
    x0 = np.stack([gx.ravel(), gy.ravel(), np.zeros(nx * ny)], 1)
    anchors = x0[[12, 15]]
    u = np.array([0.3, 0.0, -0.1])
    keep = []
    cd = cloth_desc(scene_arrays(nx, ny, 1e-3, plugs=(0, 1, 0), pin_nodes=[12, 15],
                                 pin_anchors=anchors, pin_velocity=u), keep)
    rng = np.random.default_rng(5)
    p = params(rng)
    x, v = x0.copy(), np.zeros_like(x0)
    for k in range(9):
        x, v, m = oracle.rollout(nx, ny, [cd], p, x[None], v[None], 1, k)
        x, v = x[0], v[0]
        t = (k + 1) * 1e-3
        assert (x[12] == anchors[0] + u * t).all() and (x[15] == anchors[1] + u * t).all()
        assert (v[12] == u).all() and (v[15] == u).all() and m[0, 12] == 1 and m[0, 15] == 1
