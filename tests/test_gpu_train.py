"""GPU training forward/backward (§8(f1)) against the reference: sample_batch targets, compute_loss
(loss + 53 gradients), backward_gradients, the full train_loop and the error texts — all
bit-identical (float64, the reference's association order; see csrc/train.cu)."""
import numpy as np
import pytest

import paper_2403_12820_b200 as ours
from golden_io import cloth_desc, load, params_c, to_scene
from make_golden import random_params, sheet, train_config

pytestmark = pytest.mark.gpu


def bits(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def fixture_trainer(z):
    scene = to_scene(z, z["frames_x"][0])
    traj = ours.Trajectory(int(z["nx"]), int(z["ny"]), float(z["dt"]), float(z["spacing"]),
                           z["frames_x"], z["frames_v"])
    return scene, traj


def test_sample_batch_and_loss_match_fixture():
    z = load("train_f64")
    scene, traj = fixture_trainer(z)
    with ours.Trainer(scene, traj) as t:
        idx, tgt = t.sample_batch(16, 77, targets=True)
        assert np.array_equal(idx, z["batch_idx"])
        assert bits(tgt, z["targets"])
        p = ours.NetworkParams.from_scalars(z["params"])
        loss, g = t.compute_loss(p, float(z["loss_alpha"]))
        assert bits([loss.total, loss.physics, loss.data], z["loss"])
        assert bits(g.flat, z["grads"])
        loss2, none = t.compute_loss(p, float(z["loss_alpha"]), grads=False)
        assert none is None and loss2 == loss


def test_backward_matches_fixture():
    z = load("train_f64")
    bx, by = (int(v) for v in z["bwd_dims"])
    g = ours.backward_gradients(bx, by, z["bwd_x"], z["bwd_v"],
                                ours.NetworkParams.from_scalars(z["bwd_params"]), z["bwd_up"])
    assert bits(g.flat, z["bwd_grads"])


def test_train_loop_matches_fixture():
    z = load("train_f64")
    scene, traj = fixture_trainer(z)
    cfg = ours.TrainConfig(alpha=0.5, batch_size=8, epochs=12, seed=3,
                           schedule=ours.ScheduleConfig(lr0=1e-2, gamma=0.5, interval=5),
                           de=ours.DeConfig(population=6, generations=2, probe_batch=4))
    r = ours.train_loop(cfg, scene, traj)
    assert bits(r.params.scalars(), z["train_params"])
    assert [int(t) for t in r.params.trainable] == [int(t) for t in z["train_trainable"]]
    hist = np.array([[h.step, h.lr, h.physics, h.data, h.total] for h in r.history])
    assert bits(hist, z["train_history"])
    assert r.opt.step == 12


def _scene_case(rng, nx, ny, plugs, pressure, spheres, pin_velocity, steps=40):
    from golden_io import scene_arrays
    sp = 0.05
    x0 = sheet(rng, nx, ny, sp, 1e-3, origin=(-0.5 * sp * (nx - 1), -0.5 * sp * (ny - 1), 0.27))
    pins = [0, nx - 1, nx * ny - 1]
    sc = scene_arrays(nx, ny, 1e-3, mass=0.02, drag=0.05, pressure=pressure,
                      gravity=(0.1, 0.0, -9.8), plugs=plugs, pin_nodes=pins,
                      pin_anchors=x0[pins], pin_velocity=pin_velocity, spheres=spheres,
                      stiffness=30.0, damping=0.1, spacing=sp)
    return sc, x0


CASES = [
    # (nx, ny, plugs, pressure, spheres, pin velocity, alpha, batch)
    (12, 9, (0, 1, 1), 0.5, [(0.0, 0.0, 0.0, 0.25, 0.3)], (0.02, 0.0, 0.0), 0.5, 12),
    (7, 5, (1, 0, 0), -0.8, [], (0.0, 0.0, 0.0), 1.0, 6),
    (40, 33, (0, 0, 1), 0.0, [(0.1, 0.0, -0.1, 0.3, 0.0)], (0.0, 0.01, 0.0), 0.0, 20),
    (9, 8, (1, 1, 1), 0.3, [(0.0, 0.0, 0.0, 0.25, 1.0), (0.05, 0.02, 0.1, 0.1, 0.5)],
     (0.0, 0.0, -0.03), 0.25, 30),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_compute_loss_matches_reference(reference, case):
    nx, ny, plugs, pressure, spheres, pv, alpha, batch = CASES[case]
    rng = np.random.default_rng(100 + case)
    sc, x0 = _scene_case(rng, nx, ny, plugs, pressure, spheres, pv)
    keep = []
    cd = cloth_desc(sc, keep)
    fx, fv = reference.simulate_f64(nx, ny, cd, x0, np.zeros_like(x0), 40)
    scene = to_scene(sc, x0)
    traj = ours.Trajectory(nx, ny, float(sc["dt"]), float(sc["spacing"]), fx, fv)
    with ours.Trainer(scene, traj) as t:
        for trial, seed in enumerate((5, 2**40 + 3)):
            p = random_params(rng, sigma=[0.02, 0.3][trial], gains=True,
                              alpha=float(rng.uniform(0.5, 2.0)))
            ridx, rtgt = reference.sample_batch(nx, ny, cd, fx, fv, batch, seed)
            rloss, rg = reference.compute_loss(nx, ny, cd, fx, fv, batch, seed, params_c(p), alpha)
            idx, tgt = t.sample_batch(batch, seed, targets=True)
            assert np.array_equal(idx, ridx) and bits(tgt, rtgt)
            loss, g = t.compute_loss(ours.NetworkParams.from_scalars(p), alpha)
            assert bits([loss.total, loss.physics, loss.data], rloss), (loss, rloss)
            assert bits(g.flat, rg)


@pytest.mark.parametrize("dims", [(3, 2), (33, 31), (64, 64), (100, 41)])
def test_backward_matches_reference(reference, dims):
    nx, ny = dims
    rng = np.random.default_rng(nx * 1000 + ny)
    x = sheet(rng, nx, ny, 0.1, 0.03)
    v = rng.uniform(-1.0, 1.0, x.shape)
    up = rng.normal(0.0, 1.0, x.shape)
    p = random_params(rng, sigma=0.4, gains=True, alpha=1.7)
    rg = reference.backward_gradients(nx, ny, x, v, params_c(p), up)
    g = ours.backward_gradients(nx, ny, x, v, ours.NetworkParams.from_scalars(p), up)
    assert bits(g.flat, rg)


def test_loss_errors_match_reference(reference):
    nx, ny, plugs, pressure, spheres, pv, alpha, batch = CASES[0]
    rng = np.random.default_rng(7)
    sc, x0 = _scene_case(rng, nx, ny, plugs, pressure, spheres, pv)
    keep = []
    cd = cloth_desc(sc, keep)
    fx, fv = reference.simulate_f64(nx, ny, cd, x0, np.zeros_like(x0), 40)
    traj = ours.Trajectory(nx, ny, float(sc["dt"]), float(sc["spacing"]), fx, fv)
    huge = random_params(rng, sigma=1.0, gains=True)
    huge[12:24] = 1e305   # linear branch overflows
    big = random_params(rng, sigma=1.0, gains=True)
    big[24:27] = 1e200    # finite impulse, the squared residual overflows
    with ours.Trainer(to_scene(sc, x0), traj) as t:
        t.sample_batch(batch, 11)
        for p in (huge, big):
            with pytest.raises(ArithmeticError) as r:
                reference.compute_loss(nx, ny, cd, fx, fv, batch, 11, params_c(p), alpha)
            with pytest.raises(ours.NumericsError) as o:
                t.compute_loss(ours.NetworkParams.from_scalars(p), alpha)
            assert str(o.value) == str(r.value)
        bad = ours.NetworkParams.from_scalars(huge)
        bad.isru_alpha = 0.0
        with pytest.raises(ours.ConfigError, match="^isru_alpha: must be > 0$"):
            t.compute_loss(bad, alpha)


def test_train_cosine_and_freeze_match_reference(reference):
    z = load("train_f64")
    keep = []
    cd = cloth_desc(z, keep)
    nx, ny = int(z["nx"]), int(z["ny"])
    cfg = train_config(schedule_kind=1, period=7, epochs=10, seed=11, alpha=0.8,
                       freeze_mask=(1 << 2) | (1 << 5), de_population=5, de_generations=1)
    rp, rtr, rh = reference.train(nx, ny, cd, z["frames_x"], z["frames_v"], cfg)
    scene, traj = fixture_trainer(z)
    mine = ours.TrainConfig(alpha=0.8, batch_size=8, epochs=10, seed=11,
                            schedule=ours.ScheduleConfig(kind=ours.ScheduleKind.Cosine, lr0=1e-2,
                                                         gamma=0.5, interval=5, period=7),
                            de=ours.DeConfig(population=5, generations=1, probe_batch=4),
                            freeze=[ours.ParamGroup.Bias, ours.ParamGroup.SelfVelocity])
    r = ours.train_loop(mine, scene, traj)
    flat = (list(rp.kernel_gain) + list(rp.linear_w) + list(rp.linear_b) + list(rp.nonlinear_w)
            + list(rp.deriv_w) + [rp.self_velocity_w, rp.isru_alpha])
    assert bits(r.params.scalars(), flat)
    assert [int(t) for t in r.params.trainable] == rtr.tolist()
    assert bits([[h.step, h.lr, h.physics, h.data, h.total] for h in r.history], rh)
    # resume (fine-tune mode): continues the optimizer state, no pre-search
    r2 = ours.train_loop(ours.TrainConfig(alpha=0.8, batch_size=8, epochs=3, seed=11), scene, traj,
                         resume=r)
    assert r2.opt.step == 13 and r2.history[0].step == 10


def test_gradient_check_matches_reference_module():
    import os
    import sys
    ref_pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                           "_ref")
    if not os.path.isdir(os.path.join(ref_pkg, "stencilcloth")):
        pytest.skip("reference module not built")
    sys.path.insert(0, ref_pkg)
    import stencilcloth as sc
    for args in ((8, 8, 7, 1e-6), (5, 9, 3, 1e-5)):
        assert ours.gradient_check(*args) == sc.gradient_check(*args)
    assert ours.gradient_check() < 1e-5


def test_train_binding_checkpoint_bytes_match_reference(tmp_path):
    """The reference module's own train() and ours on the same parsed scene and simulated
    trajectory: the CKP1 files of the two results are byte-identical (parameters, trainable
    flags and the DE brackets)."""
    import os
    import sys
    ref_pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                           "_ref")
    if not os.path.isdir(os.path.join(ref_pkg, "stencilcloth")):
        pytest.skip("reference module not built")
    sys.path.insert(0, ref_pkg)
    import stencilcloth as sc
    text = """{"name": "ckp_train", "grid": {"nx": 10, "ny": 8, "spacing": 0.05,
      "origin": [-0.2, -0.15, 0.3], "plane": "xy"},
      "material": {"stiffness": 30.0, "damping": 0.05, "mass": 0.01,
                   "gravity": [0.0, 0.0, -9.8], "drag": 0.02, "pressure": 0.2},
      "time": {"dt": 0.001, "steps": 40}, "pins": {"nodes": ["top_left", "top_right"]},
      "colliders": [{"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 0.25,
                     "friction": 0.3}]}"""
    rscene = sc.parse_scene(text)
    rtraj = sc.simulate(rscene)
    kw = dict(alpha=0.4, batch_size=6, epochs=8, seed=5, lr0=2e-2, de_population=5,
              de_generations=2, de_probe=4)
    rparams, rhist = sc.train(rscene, rtraj, **kw)
    scene = ours.parse_scene(text)
    traj = ours.simulate(scene)
    assert bits(traj.frames_x, np.stack([rtraj.positions(f) for f in range(rtraj.frame_count)]))
    params, hist = ours.train(scene, traj, **kw)
    assert bits(np.array(hist), np.array(rhist))
    pr, po = str(tmp_path / "ref.ckpt"), str(tmp_path / "ours.ckpt")
    rc = sc.Checkpoint()
    rc.params = rparams
    rc.step = kw["epochs"]
    sc.save_checkpoint(pr, rc)
    ours.save_checkpoint(po, ours.Checkpoint(params, None, kw["epochs"], ""))
    assert open(po, "rb").read() == open(pr, "rb").read()


def test_distributed_trainer_single_rank_matches_trainer():
    """DistributedTrainer over the GPU part with one rank = Trainer (compute_loss and run)."""
    z = load("train_f64")
    scene, traj = fixture_trainer(z)
    p = ours.NetworkParams.from_scalars(z["params"])
    with ours.Trainer(scene, traj) as t:
        t.set_batch(z["batch_idx"])
        want, wg = t.compute_loss(p, 0.3)
        cfg = ours.TrainConfig(alpha=0.5, batch_size=8, epochs=6, seed=3,
                               de=ours.DeConfig(population=5, generations=2, probe_batch=4))
        rw = t.run(cfg)
    part = ours.CudaPart(scene, traj)
    d = ours.DistributedTrainer(part)
    d.set_batch(z["batch_idx"])
    got, gg = d.compute_loss(p, 0.3)
    assert bits([got.total, got.physics, got.data], [want.total, want.physics, want.data])
    assert bits(gg.flat, wg.flat)
    r = d.run(cfg)
    assert bits(r.params.scalars(), rw.params.scalars())
    assert r.params.brackets == rw.params.brackets
    assert bits([[h.step, h.lr, h.physics, h.data, h.total] for h in r.history],
                [[h.step, h.lr, h.physics, h.data, h.total] for h in rw.history])
    part.close()


def test_parts_combine_exactly():
    """Two GPU parts of one batch (two ranks emulated in one process, one after the other):
    count summed, loss chain handed over, per-transition gradients summed in order — equal to
    the single-part compute_loss bit for bit."""
    z = load("train_f64")
    scene, traj = fixture_trainer(z)
    p = ours.NetworkParams.from_scalars(z["params"])
    idx = list(z["batch_idx"])
    B, m = len(idx), 7
    with ours.Trainer(scene, traj) as t:
        t.set_batch(idx)
        want, wg = t.compute_loss(p, 0.3)
    a, b = ours.CudaPart(scene, traj), ours.CudaPart(scene, traj)
    a.set_batch(idx)
    b.set_batch(idx)
    ca, bad_a, _ = a.forward(p, 0, m)
    cb, bad_b, _ = b.forward(p, m, B)
    assert bad_a < 0 and bad_b < 0
    ps, ds, bl = a.chain(0.0, 0.0)
    ps, ds, bl2 = b.chain(ps, ds)
    assert bl < 0 and bl2 < 0
    count = ca + cb
    per_b = np.concatenate([a.backward(p, 0.3, count, B, m), b.backward(p, 0.3, count, B, B - m)])
    g = [0.0] * 53
    for row in per_b.tolist():
        g = [g[s] + row[s] * 1.0 for s in range(53)]
    assert bits(g, wg.flat)
    free = scene.nx * scene.ny - len(scene.bc.nodes)
    physics = ps / (3.0 * B * free)
    data = ds / (6.0 * count)
    assert bits([physics, data], [want.physics, want.data])
    a.close()
    b.close()
