"""The CPU oracle (oracle/oracle.c) against fixtures produced by the reference itself
(tests/golden/make_golden.py -> oracle/_ref, the unmodified reference sources). Bit-exact."""
import glob
import os

import numpy as np
import pytest

from golden_io import GOLDEN_DIR, cloth_desc, load, params_c

F32_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*_f32.npz")))


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("name", F32_CASES)
def test_oracle_f32_rollout_matches_reference_bitwise(oracle, name):
    z = load(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    pc = params_c(z["params"])
    x, v = z["x0"][None].copy(), z["v0"][None].copy()
    k = 0
    for cp in z["checkpoints"]:
        # step one at a time so every step's mask is checked too
        while k < cp:
            x, v, m = oracle.rollout(nx, ny, [cd], pc, x, v, 1, k)
            assert np.array_equal(m[0], z["masks"][k]), "mask differs at step %d" % (k + 1)
            k += 1
        assert bits_equal(x[0], z["x_%d" % cp]), "x differs after %d steps" % cp
        assert bits_equal(v[0], z["v_%d" % cp]), "v differs after %d steps" % cp


@pytest.mark.parametrize("name", F32_CASES)
def test_oracle_f32_impulse_matches_reference_bitwise(oracle, name):
    z = load(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    t1 = np.float32(1) * np.float32(float(z["dt"]))
    _, _, _, imp = oracle.nn_step(nx, ny, cd, params_c(z["params"]), z["x0"], z["v0"], t1)
    assert bits_equal(imp, z["impulse_step1"])


def test_oracle_forward_impulse_f64(oracle):
    z = load("forward_impulse_f64")
    t = 0
    while "fi%d_x" % t in z:
        nx, ny = (int(v) for v in z["fi%d_dims" % t])
        got = oracle.forward_impulse(nx, ny, params_c(z["fi%d_params" % t]), z["fi%d_x" % t],
                                     z["fi%d_v" % t])
        assert bits_equal(got, z["fi%d_out" % t])
        t += 1
    assert t >= 6


def test_oracle_f64_api(oracle):
    z = load("api_f64")
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    pc = params_c(z["params"])
    assert bits_equal(oracle.plug_impulse(nx, ny, cd, z["x0"], z["v0"]), z["plug"])
    xa, va, ma = oracle.advance_with_impulse(nx, ny, cd, z["x0"], z["v0"], z["imp"],
                                             float(z["adv_t"]))
    assert bits_equal(xa, z["adv_x"]) and bits_equal(va, z["adv_v"])
    assert np.array_equal(ma, z["adv_mask"])
    xs, vs, _, _ = oracle.nn_step(nx, ny, cd, pc, z["x0"], z["v0"], float(z["step_t"]))
    assert bits_equal(xs, z["step_x"]) and bits_equal(vs, z["step_v"])


def test_oracle_f64_rollout_frames(oracle):
    """rollout() (eval.cpp:86-103): frame 0 = apply_dirichlet(initial, 0), then nn_step with
    t_next = (k+1)*dt; every frame bit-exact."""
    z = load("api_f64")
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    pc = params_c(z["params"])
    x, v = z["x0"].copy(), z["v0"].copy()
    u = z["pin_velocity"]
    for k, i in enumerate(z["pin_nodes"]):
        x[i] = z["pin_anchors"][k] + u * 0.0
        v[i] = u
    fx, fv = z["frames_x"], z["frames_v"]
    assert bits_equal(x, fx[0]) and bits_equal(v, fv[0])
    dt = float(z["dt"])
    for k in range(fx.shape[0] - 1):
        x, v, _, _ = oracle.nn_step(nx, ny, cd, pc, x, v, (k + 1) * dt)
        assert bits_equal(x, fx[k + 1]) and bits_equal(v, fv[k + 1]), "frame %d" % (k + 1)


def test_golden_fixtures_exercise_contacts():
    """The sphere-drop fixture really collides (else the mask checks would be vacuous)."""
    z = load("sphere_drop_f32")
    per_step = z["masks"].sum(axis=1)
    assert per_step.max() > 50 and per_step[0] == len(z["pin_nodes"])


def test_oracle_pbs_matches_reference_bitwise(oracle):
    """Ground-truth mass-spring step (PBS, §8(f2)): the oracle's total_impulse and
    step_semi_implicit reproduce simulate_scene's frames (f64) and the benchmark_sim step
    sequence (f32) bit for bit."""
    z = load("pbs_sim64")
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    fx, fv = z["frames_x"], z["frames_v"]
    imp, sing = oracle.total_impulse(nx, ny, cd, fx[60], fv[60])
    assert sing == -1 and bits_equal(imp, z["imp60"])
    x, v = fx[0].copy(), fv[0].copy()
    for k in range(fx.shape[0] - 1):
        x, v, _, _ = oracle.pbs_step(nx, ny, cd, x, v, (k + 1) * float(z["dt"]))
        assert bits_equal(x, fx[k + 1]) and bits_equal(v, fv[k + 1]), "frame %d" % (k + 1)
    z = load("pbs_steps32")
    cd = cloth_desc(z, keep)
    x, v = z["x0"].copy(), z["v0"].copy()
    k = 0
    for cp in z["checkpoints"]:
        while k < cp:
            x, v, _, _ = oracle.pbs_step(nx, ny, cd, x, v, np.float32(k + 1) * np.float32(float(z["dt"])))
            k += 1
        assert bits_equal(x, z["x_%d" % cp]) and bits_equal(v, z["v_%d" % cp])


def test_oracle_pbs_singular_spring(oracle):
    z = load("pbs_sim64")
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    x = z["frames_x"][0].copy()
    x[17] = x[18]  # coincident E neighbours
    _, sing = oracle.total_impulse(nx, ny, cd, x, z["frames_v"][0])
    assert sing == 17
