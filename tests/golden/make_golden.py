"""Generate the golden fixtures under tests/golden/ from the REFERENCE ITSELF.

Every output array here comes from oracle/_ref/libstencilcloth_ref.so, i.e. the unmodified
reference sources (/root/reference/proj/src/*.cpp + include/cloth/detail/kernels.hpp) compiled
by oracle/Makefile and driven through oracle/ref_harness.cpp:
  * f32: the run_steps<float> step sequence (eval.cpp:48-59) of detail::forward_impulse<float>,
    add_plug_impulse<float>, advance_with_impulse<float>;
  * f64: the public API forward_impulse / plug_impulse / advance_with_impulse / nn_step /
    rollout (net.cpp:132-142,242-248, sim.cpp:100-148, eval.cpp:86-103).
Inputs are seeded numpy draws (np.random.default_rng) so the fixtures do not depend on the
product. Run from the repo root:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from golden_io import GOLDEN_DIR, cloth_desc, params_c, scene_arrays  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402
from paper_2403_12820_b200 import _abi  # noqa: E402

# the reference is only needed to generate; tests import the helpers below without it
R = Reference() if __name__ == "__main__" else None


def sheet(rng, nx, ny, spacing, noise, origin=(0.0, 0.0, 0.0)):
    ix = np.tile(np.arange(nx, dtype=np.float64), ny)
    iy = np.repeat(np.arange(ny, dtype=np.float64), nx)
    x = np.stack([origin[0] + spacing * ix, origin[1] + spacing * iy,
                  origin[2] + 0.0 * ix], axis=1)
    return x + rng.normal(0.0, noise, x.shape)


def random_params(rng, sigma=0.05, gains=False, alpha=1.0):
    s = np.zeros(53)
    s[0:12] = rng.uniform(0.5, 1.5, 12) if gains else 1.0
    s[12:51] = rng.normal(0.0, sigma, 39)
    s[51] = rng.normal(0.0, sigma)
    s[52] = alpha
    return s


def save(name, **arrays):
    os.makedirs(GOLDEN_DIR, exist_ok=True)
    path = os.path.join(GOLDEN_DIR, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, "%.1f KB" % (os.path.getsize(path) / 1024))


def f32_case(name, rng, sc, params, x0, v0, checkpoints):
    """run_steps<float> from (x0, v0): x, v after each checkpoint step count and the mask of
    every step (one-step calls with the right k so t_next matches)."""
    keep = []
    nx, ny = int(sc["nx"]), int(sc["ny"])
    cd = cloth_desc(sc, keep)
    pc = params_c(params)
    x = x0.astype(np.float32)
    v = v0.astype(np.float32)
    out = dict(sc, params=params, x0=x, v0=v, checkpoints=np.array(checkpoints, np.int64))
    masks = []
    k = 0
    for cp in checkpoints:
        while k < cp:
            x, v, m = R.rollout_f32(nx, ny, [cd], pc, x.reshape(1, -1, 3), v.reshape(1, -1, 3), 1,
                                    k)
            x, v = x[0], v[0]
            masks.append(m[0])
            k += 1
        out["x_%d" % cp] = x.copy()
        out["v_%d" % cp] = v.copy()
    out["masks"] = np.array(masks, np.uint8)
    # one step with the impulse exposed, from the input state (per-step parity)
    xo, vo, m, imp = R.step_f32(nx, ny, cd, pc, x0.astype(np.float32), v0.astype(np.float32),
                                np.float32(1) * np.float32(float(sc["dt"])))
    out["impulse_step1"] = imp
    save(name, **out)


def main():
    rng = np.random.default_rng(20240319)

    # 1) config-1-shaped: 32x32, corners pinned, gravity, hidden-8 weights, 100 steps
    nx = ny = 32
    x0 = sheet(rng, nx, ny, 1.0 / 31, 1e-3).astype(np.float32).astype(np.float64)
    pins = [(ny - 1) * nx, (ny - 1) * nx + nx - 1]
    sc = scene_arrays(nx, ny, 1.0 / 240, pin_nodes=pins, pin_anchors=x0[pins])
    p = random_params(rng)
    p[12 + 8:12 + 12] = 0.0   # linear skip channels
    p[27 + 8:27 + 12] = 0.0   # nonlinear
    p[39 + 8:39 + 12] = 0.0   # deriv
    f32_case("cfg1_f32", rng, sc, p, x0, np.zeros_like(x0), [1, 10, 100])

    # 2) ragged 20x13 sheet dropped on a sphere with friction, moving pins, all three plugs,
    #    non-unit gains and alpha != 1, small weights so the sheet really falls onto the ball
    nx, ny = 20, 13
    sp = 0.05
    x0 = sheet(rng, nx, ny, sp, 2e-4, origin=(-0.475, -0.3, 0.32)).astype(np.float32).astype(
        np.float64)
    pins = [0, nx - 1]
    sc = scene_arrays(nx, ny, 2e-3, mass=0.02, drag=0.05, pressure=0.8, gravity=(0.3, 0.0, -9.8),
                      plugs=(1, 1, 1), pin_nodes=pins, pin_anchors=x0[pins],
                      pin_velocity=(0.05, 0.0, -0.02), spheres=[(0.0, 0.0, 0.0, 0.25, 0.3)])
    p = random_params(rng, sigma=0.002, gains=True, alpha=1.3)
    f32_case("sphere_drop_f32", rng, sc, p, x0, np.zeros_like(x0), [1, 5, 20, 80, 150])

    # 3) tiny / ragged grids (edge cases of the channel masks), 10 steps each
    for (nx, ny) in [(2, 2), (3, 2), (2, 7), (5, 3)]:
        x0 = sheet(rng, nx, ny, 0.1, 1e-2).astype(np.float32).astype(np.float64)
        v0 = rng.normal(0.0, 0.1, x0.shape).astype(np.float32).astype(np.float64)
        sc = scene_arrays(nx, ny, 1e-2, mass=0.5, drag=0.3, plugs=(0, 1, 1),
                          pin_nodes=[nx * ny - 1], pin_anchors=x0[[nx * ny - 1]])
        p = random_params(rng, sigma=0.3, gains=True, alpha=0.7)
        f32_case("tiny_%dx%d_f32" % (nx, ny), rng, sc, p, x0, v0, [1, 10])

    # 4) f64 public API: forward_impulse on random 3..8 grids (test_net.cpp:104-116 shapes),
    #    plug_impulse / advance_with_impulse (+ mask) / nn_step, and a 30-frame rollout
    out = {}
    for t in range(6):
        nx, ny = int(rng.integers(3, 9)), int(rng.integers(3, 9))
        x = sheet(rng, nx, ny, 0.1, 0.05)
        v = rng.uniform(-1.5, 1.5, x.shape)
        p = random_params(rng, sigma=0.4, gains=True, alpha=float(rng.uniform(0.5, 2.0)))
        out["fi%d_dims" % t] = np.array([nx, ny])
        out["fi%d_x" % t], out["fi%d_v" % t], out["fi%d_params" % t] = x, v, p
        out["fi%d_out" % t] = R.forward_impulse_f64(nx, ny, params_c(p), x, v)
    save("forward_impulse_f64", **out)

    nx, ny = 9, 7
    x0 = sheet(rng, nx, ny, 0.05, 1e-3, origin=(-0.2, -0.15, 0.27))
    v0 = rng.normal(0.0, 0.05, x0.shape)
    pins = [3, 4, 60]
    sc = scene_arrays(nx, ny, 1e-3, mass=0.01, drag=0.02, pressure=-1.5, gravity=(0, 0, -9.8),
                      plugs=(1, 1, 1), pin_nodes=pins, pin_anchors=x0[pins] + 0.01,
                      pin_velocity=(0.0, 0.1, -0.05),
                      spheres=[(0.0, 0.0, 0.0, 0.25, 0.25), (0.1, 0.05, 0.05, 0.2, 0.0)])
    keep = []
    cd = cloth_desc(sc, keep)
    p = random_params(rng, sigma=0.01, gains=True, alpha=1.1)
    pc = params_c(p)
    imp = rng.normal(0.0, 0.5, x0.shape)
    plug = R.plug_impulse_f64(nx, ny, cd, x0, v0)
    xa, va, ma = R.advance_with_impulse_f64(nx, ny, cd, x0, v0, imp, 0.0123)
    xs, vs = R.nn_step_f64(nx, ny, cd, pc, x0, v0, 0.004)
    fx, fv = R.rollout_f64(nx, ny, cd, pc, x0, v0, 120)
    save("api_f64", **sc, params=p, x0=x0, v0=v0, imp=imp, plug=plug, adv_x=xa, adv_v=va,
         adv_mask=ma, adv_t=np.float64(0.0123), step_x=xs, step_v=vs, step_t=np.float64(0.004),
         frames_x=fx, frames_v=fv)


def pbs_main():
    """Ground-truth mass-spring step (PBS) fixtures from the reference."""
    rng = np.random.default_rng(20240320)
    # f64 simulate_scene: a sheet dropped on a sphere with friction, a moving pin, pressure,
    # drag (like acceptance criterion 6's ball scene, smaller)
    nx, ny = 12, 10
    sp = 0.05
    x0 = sheet(rng, nx, ny, sp, 1e-3, origin=(-0.275, -0.225, 0.28))
    v0 = np.zeros_like(x0)
    pins = [0, nx - 1]
    sc = scene_arrays(nx, ny, 4e-4, mass=0.01, drag=0.01, pressure=0.7, gravity=(0.0, 0.0, -9.8),
                      plugs=(0, 0, 0), pin_nodes=pins, pin_anchors=x0[pins],
                      pin_velocity=(0.02, 0.0, 0.0), spheres=[(0.0, 0.0, 0.0, 0.25, 0.3)],
                      stiffness=40.0, damping=0.2, spacing=sp)
    keep = []
    cd = cloth_desc(sc, keep)
    fx, fv = R.simulate_f64(nx, ny, cd, x0, v0, 150)
    xs, vs = fx[60].copy(), fv[60].copy()
    imp = R.total_impulse_f64(nx, ny, cd, xs, vs)
    save("pbs_sim64", **sc, x0=x0, v0=v0, frames_x=fx, frames_v=fv, imp60=imp)
    # f32: the benchmark_sim step sequence (run_steps<float>, params == nullptr)
    x32 = x0.astype(np.float32)
    v32 = np.zeros_like(x32)
    outs = {}
    xk, vk = x32, v32
    k = 0
    for cp in (1, 20, 100):
        xk, vk = R.pbs_rollout_f32(nx, ny, cd, xk, vk, cp - k, k)
        k = cp
        outs["x_%d" % cp], outs["v_%d" % cp] = xk.copy(), vk.copy()
    save("pbs_steps32", **sc, x0=x32, v0=v32, checkpoints=np.array([1, 20, 100]), **outs)


def train_config(**kw):
    c = _abi.sc_train_config()
    base = dict(alpha=0.5, batch_size=8, epochs=12, schedule_kind=0, lr0=1e-2, gamma=0.5,
                interval=5, floor=1e-5, period=1000, seed=3, de_population=6, de_generations=2,
                de_bound=4.0, de_cross_prob=0.9, de_diff_weight=0.7, de_probe_batch=4,
                checkpoint_interval=500, freeze_mask=0)
    base.update(kw)
    for k, v in base.items():
        setattr(c, k, v)
    return c


def train_main():
    """Training forward/backward fixtures from the reference's own
    sample_batch / compute_loss / backward_gradients / train_loop (train.cpp, net.cpp)."""
    rng = np.random.default_rng(20240321)
    nx, ny = 12, 10
    sp = 0.05
    x0 = sheet(rng, nx, ny, sp, 1e-3, origin=(-0.275, -0.225, 0.28))
    pins = [0, nx - 1]
    sc = scene_arrays(nx, ny, 1e-3, mass=0.01, drag=0.03, pressure=0.4, gravity=(0.0, 0.0, -9.8),
                      plugs=(0, 1, 1), pin_nodes=pins, pin_anchors=x0[pins],
                      pin_velocity=(0.02, 0.0, 0.0), spheres=[(0.0, 0.0, 0.0, 0.25, 0.3)],
                      stiffness=40.0, damping=0.2, spacing=sp)
    keep = []
    cd = cloth_desc(sc, keep)
    fx, fv = R.simulate_f64(nx, ny, cd, x0, np.zeros_like(x0), 60)
    idx, tgt = R.sample_batch(nx, ny, cd, fx, fv, 16, 77)
    p = random_params(rng, sigma=0.05, gains=True, alpha=1.2)
    loss, grads = R.compute_loss(nx, ny, cd, fx, fv, 16, 77, params_c(p), 0.3)
    bx, by = 40, 30  # two backward chunks of 1024 nodes
    bxs = sheet(rng, bx, by, 0.1, 0.03)
    bvs = rng.uniform(-1.0, 1.0, bxs.shape)
    bup = rng.normal(0.0, 1.0, bxs.shape)
    bp = random_params(rng, sigma=0.4, gains=True, alpha=0.8)
    bgrads = R.backward_gradients(bx, by, bxs, bvs, params_c(bp), bup)
    cfg = train_config()
    tp, ttr, thist = R.train(nx, ny, cd, fx, fv, cfg)
    flat = (list(tp.kernel_gain) + list(tp.linear_w) + list(tp.linear_b) + list(tp.nonlinear_w)
            + list(tp.deriv_w) + [tp.self_velocity_w, tp.isru_alpha])
    save("train_f64", **sc, frames_x=fx, frames_v=fv, batch_seed=np.uint64(77), batch_idx=idx,
         targets=tgt, params=p, loss_alpha=np.float64(0.3), loss=loss, grads=grads,
         bwd_dims=np.array([bx, by]), bwd_x=bxs, bwd_v=bvs, bwd_up=bup, bwd_params=bp,
         bwd_grads=bgrads, train_params=np.array(flat), train_trainable=ttr, train_history=thist)


if __name__ == "__main__":
    if "--train" in sys.argv:
        train_main()
        sys.exit(0)
    if "--pbs" not in sys.argv:
        main()
    pbs_main()
    train_main()
