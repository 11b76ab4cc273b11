"""GPU parity: the sm_100a kernels (through the C-ABI) against the reference's golden fixtures
and the CPU oracle.

Bars (north_star in BASELINE.json):
  * PARITY mode: bit-exact x, v and `constrained` masks vs the reference templates, every step
    and over full rollouts (f32 and f64).
  * FAST mode (f32): per step from identical input states, |a - b| <= 1e-5 * max(|b|, rms(b))
    per component plane (relative error against the element, floored at the field's RMS so
    that accidental cancellations near zero are not over-weighted); masks identical.
"""
import glob
import os

import numpy as np
import pytest

from golden_io import GOLDEN_DIR, cloth_desc, load, params_c, to_scene

pytestmark = pytest.mark.gpu

F32_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*_f32.npz")))
FAST_RTOL = 1e-5


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.view(np.uint8), b.view(np.uint8))


def fast_close(a, b, rtol=FAST_RTOL, normwise=1e-6):
    """Per component plane |a - b| <= rtol * max(|b|, rms(b)) and max|a - b| / max|b| <=
    normwise (test_gpu_fullsize.py explains why the floor is the field's RMS)."""
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    rms = np.sqrt(np.mean(b * b, axis=0))
    scale = np.maximum(np.abs(b), rms[None, :])
    err = np.abs(a - b)
    ok = (err <= rtol * scale).all() and err.max() <= normwise * max(np.abs(b).max(), 1e-300)
    return bool(ok), float((err / np.maximum(scale, 1e-300)).max())


def golden_ctx(z, precision="f32"):
    from paper_2403_12820_b200 import Context, NetworkParams
    return Context(to_scene(z), NetworkParams.from_scalars(z["params"]), precision)


@pytest.mark.parametrize("name", F32_CASES)
def test_parity_f32_every_step_bitwise(name):
    z = load(name)
    with golden_ctx(z) as ctx:
        x, v = z["x0"][None], z["v0"][None]
        k = 0
        for cp in z["checkpoints"]:
            while k < cp:
                x, v, m = ctx.rollout(x, v, 1, k, "parity", constrained=True)
                assert np.array_equal(m[0], z["masks"][k]), "mask differs at step %d" % (k + 1)
                k += 1
            assert bits_equal(x[0], z["x_%d" % cp]), "x differs after %d steps" % cp
            assert bits_equal(v[0], z["v_%d" % cp]), "v differs after %d steps" % cp


@pytest.mark.parametrize("name", F32_CASES)
def test_parity_f32_device_resident_rollout_bitwise(name):
    z = load(name)
    last = int(z["checkpoints"][-1])
    with golden_ctx(z) as ctx:
        x, v, m = ctx.rollout(z["x0"][None], z["v0"][None], last, 0, "parity", constrained=True)
        assert bits_equal(x[0], z["x_%d" % last]) and bits_equal(v[0], z["v_%d" % last])
        assert np.array_equal(m[0], z["masks"][last - 1])
        # chunked rollouts continue time exactly (k0 offsets)
        first = int(z["checkpoints"][0])
        x1, v1 = ctx.rollout(z["x0"][None], z["v0"][None], first, 0, "parity")
        x2, v2 = ctx.rollout(x1, v1, last - first, first, "parity")
        assert bits_equal(x2[0], z["x_%d" % last]) and bits_equal(v2[0], z["v_%d" % last])


@pytest.mark.parametrize("name", F32_CASES)
def test_fast_f32_per_step_within_tolerance(name, oracle):
    """FAST mode from identical (reference) input states at every checkpoint."""
    z = load(name)
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    pc = params_c(z["params"])
    dt = np.float32(float(z["dt"]))
    states = [(0, z["x0"], z["v0"])] + [(int(c), z["x_%d" % c], z["v_%d" % c])
                                         for c in z["checkpoints"][:-1]]
    with golden_ctx(z) as ctx:
        for k, xs, vs in states:
            xo, vo, m, _ = oracle.nn_step(nx, ny, cd, pc, xs, vs, np.float32(k + 1) * dt)
            xf, vf, mf = ctx.rollout(xs[None], vs[None], 1, k, "fast", constrained=True)
            okx, ex = fast_close(xf[0], xo)
            okv, ev = fast_close(vf[0], vo)
            assert okx and okv, "step %d: rel err x %.3g v %.3g" % (k + 1, ex, ev)
            assert np.array_equal(mf[0], m), "mask differs at step %d" % (k + 1)


def test_f64_public_api_bitwise():
    import paper_2403_12820_b200 as sc
    z = load("api_f64")
    scene = to_scene(z, z["x0"])
    scene.initial_v = z["v0"].copy()
    p = sc.NetworkParams.from_scalars(z["params"])
    assert bits_equal(sc.plug_impulse(scene, z["x0"], z["v0"]), z["plug"])
    xa, va, ma = sc.advance_with_impulse(scene, z["x0"], z["v0"], z["imp"], float(z["adv_t"]),
                                         constrained=True)
    assert bits_equal(xa, z["adv_x"]) and bits_equal(va, z["adv_v"])
    assert np.array_equal(ma, z["adv_mask"])
    xs, vs = sc.nn_step(p, scene, z["x0"], z["v0"], float(z["step_t"]))
    assert bits_equal(xs, z["step_x"]) and bits_equal(vs, z["step_v"])
    traj = sc.rollout(p, scene, steps=z["frames_x"].shape[0] - 1)
    assert len(traj) == z["frames_x"].shape[0]
    for f in range(len(traj)):
        assert bits_equal(traj.positions(f), z["frames_x"][f]), "frame %d" % f
        assert bits_equal(traj.velocities(f), z["frames_v"][f]), "frame %d" % f


def test_f64_forward_impulse_bitwise():
    import paper_2403_12820_b200 as sc
    z = load("forward_impulse_f64")
    t = 0
    while "fi%d_x" % t in z:
        nx, ny = (int(v) for v in z["fi%d_dims" % t])
        scene = sc.Scene(nx, ny, 0.1, z["fi%d_x" % t])
        scene.dt = 1e-3
        p = sc.NetworkParams.from_scalars(z["fi%d_params" % t])
        got = sc.forward_impulse(p, scene, z["fi%d_x" % t], z["fi%d_v" % t])
        assert bits_equal(got, z["fi%d_out" % t])
        t += 1


@pytest.mark.parametrize("cfg_id,n,batch,steps", [(1, 32, 1, 100), (2, 40, 5, 30), (3, 64, 1, 60),
                                                   (4, 48, 1, 30), (5, 24, 7, 40)])
def test_configs_parity_vs_oracle_bitwise(oracle, cfg_id, n, batch, steps):
    """Every BASELINE config's dynamics (shrunk grid/batch) bit-exact against the oracle,
    including the plane-collider extension of config 5 (oracle-only parity)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xo, vo, mo = oracle.rollout(n, n, cds, p.to_c(), x, v, steps)
    with ClothBatch(scenes, p) as cb:
        xg, vg, mg = cb.rollout(x, v, steps, 0, "parity", constrained=True)
    assert bits_equal(xg, xo) and bits_equal(vg, vo)
    assert np.array_equal(mg, mo)


@pytest.mark.parametrize("cfg_id,n,batch", [(2, 256, 4), (3, 1024, 1), (5, 128, 9), (1, 32, 1)])
def test_configs_fast_per_step(oracle, cfg_id, n, batch):
    """FAST mode at the configs' real grid sizes: per step from identical input states (the
    oracle's state after a few steps), within tolerance; masks identical."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xs, vs, _ = oracle.rollout(n, n, cds, p.to_c(), x, v, 3)
    xo, vo, mo = oracle.rollout(n, n, cds, p.to_c(), xs, vs, 1, 3)
    with ClothBatch(scenes, p) as cb:
        xf, vf, mf = cb.rollout(xs, vs, 1, 3, "fast", constrained=True)
    okx, ex = fast_close(xf, xo)
    okv, ev = fast_close(vf, vo)
    assert okx and okv, "rel err x %.3g v %.3g" % (ex, ev)
    assert np.array_equal(mf, mo)


def test_fast_short_rollout_drift_bounded(oracle):
    """Short FAST rollout vs the bit-exact path: the drift stays at rounding level over 10
    steps on config 2's cloth size (random-weight dynamics are chaotic over long horizons)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(2, batch=2, n=256)
    with ClothBatch(scenes, p) as cb:
        xp, vp = cb.rollout(x, v, 10, 0, "parity")
        xf, vf = cb.rollout(x, v, 10, 0, "fast")
    okx, ex = fast_close(xf, xp, 1e-5, normwise=1e-5)
    okv, ev = fast_close(vf, vp, 1e-5, normwise=1e-5)
    print("10-step FAST drift (rms-floored relative): x %.3g v %.3g" % (ex, ev))
    assert okx and okv, "10-step drift x %.3g v %.3g" % (ex, ev)


def test_full_config2_batch_properties():
    """Config 2 at full size (64 x 256^2) in FAST mode: finite, pins exactly on their anchors,
    deterministic run to run."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(2)
    with ClothBatch(scenes, p) as cb:
        x1, v1 = cb.rollout(x, v, 20, 0, "fast")
        x2, v2 = cb.rollout(x, v, 20, 0, "fast")
    assert bits_equal(x1, x2) and bits_equal(v1, v2)
    assert np.isfinite(x1).all() and np.isfinite(v1).all()
    top = np.arange((cfg.n - 1) * cfg.n, cfg.n * cfg.n)
    assert np.array_equal(x1[:, top], x[:, top])
    assert not np.any(v1[:, top])


def test_errors_map_to_reference_exceptions():
    import paper_2403_12820_b200 as sc
    z = load("api_f64")
    scene = to_scene(z, z["x0"])
    p = sc.NetworkParams.from_scalars(z["params"])
    bad = p.copy()
    bad.isru_alpha = 0.0
    with pytest.raises(ValueError):
        sc.forward_impulse(bad, scene, z["x0"], z["v0"])
    with pytest.raises(ValueError):
        sc.forward_impulse(p, scene, z["x0"][:-1], z["v0"][:-1])
    inf = p.copy()
    inf.linear_w[0] = np.inf
    with pytest.raises(ArithmeticError, match="linear"):
        sc.forward_impulse(inf, scene, z["x0"], z["v0"])
    s2 = to_scene(z, z["x0"])
    s2.bc.nodes = [5, 3, 1]
    s2.bc.anchors = np.zeros((3, 3))
    with pytest.raises(ValueError, match="strictly increasing"):
        sc.Context(s2, p)


def test_rollout_divergence_reports_frame():
    """eval.cpp:98-99: a finite impulse that drives the state non-finite is reported as
    "rollout diverged: non-finite state at frame k"; a non-finite impulse names the branch
    (net.cpp:30-51)."""
    import paper_2403_12820_b200 as sc
    scene = sc.Scene(6, 6, 0.1, sc.build_grid(6, 6, 0.1))
    scene.dt = 1e10
    p = sc.NetworkParams()
    p.linear_b = np.array([1e300, 0.0, 0.0])  # v' = 1e300, x' = x + 1e310 -> inf
    with pytest.raises(ArithmeticError, match="rollout diverged: non-finite state at frame 1"):
        sc.rollout(p, scene, steps=3)
    scene.dt = 1.0
    p = sc.NetworkParams()
    p.linear_b = np.array([1.0, 1.0, 1.0])
    p.self_velocity_w = 1e200  # v*wV overflows in the impulse of frame 3
    with pytest.raises(ArithmeticError, match=r"network impulse non-finite at node \d+ \(derivative"):
        sc.rollout(p, scene, steps=5)


def test_zero_weights_bias_passthrough():
    """test_net.cpp:118-125 on the GPU: zero weights give a zero impulse; the bias passes
    straight through exactly."""
    import paper_2403_12820_b200 as sc
    x = sc.build_grid(4, 4, 0.1)
    scene = sc.Scene(4, 4, 0.1, x)
    scene.dt = 1e-3
    p = sc.NetworkParams()
    assert not np.any(sc.forward_impulse(p, scene, x, np.zeros_like(x)))
    p.linear_b = np.array([0.1, -0.2, 0.3])
    out = sc.forward_impulse(p, scene, x, np.zeros_like(x))
    assert np.array_equal(out, np.tile(p.linear_b, (16, 1)))


def test_benchmark_net_reports_throughput():
    import paper_2403_12820_b200 as sc
    z = load("cfg1_f32")
    scene = to_scene(z, z["x0"].astype(np.float64))
    p = sc.NetworkParams.from_scalars(z["params"])
    for prec in ("f32", "f64"):
        r = sc.benchmark_net(p, scene, 5, 2, prec)
        assert r.steps == 5 and r.seconds > 0 and r.steps_per_second > 0
    with pytest.raises(ValueError):
        sc.benchmark_net(p, scene, 0, 0)


@pytest.mark.parametrize("cfg_id,n,batch,steps", [(2, 256, 8, 25), (3, 256, 1, 30), (5, 128, 12, 21),
                                                   (1, 32, 1, 40)])
def test_fast_persistent_kernel_matches_per_step_launches(monkeypatch, cfg_id, n, batch, steps):
    """The multi-step FAST kernel (the wavefront kernel for narrow cloths, one launch) gives
    bit-identical states to one launch per step (same per-node arithmetic and order); config 1's
    cloth is held on the wavefront kernel (SC_SMALL=0: the small-cloth kernel is FAST-tolerance
    equal only, tests/test_gpu_small.py)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    monkeypatch.setenv("SC_SMALL", "0")
    monkeypatch.setenv("SC_WAVE_MIN_CLOTHS", "1")  # the wavefront kernel at these batch sizes
    monkeypatch.setenv("SC_WAVE_MIN_STEPS", "1")  # ... and step counts
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    with ClothBatch(scenes, p) as cb:
        cb.set_persistent(True)
        xa, va = cb.rollout(x, v, steps, 0, "fast")
        la = cb.launch_count()
        cb.set_persistent(False)
        xb, vb = cb.rollout(x, v, steps, 0, "fast")
        lb = cb.launch_count() - la
    assert bits_equal(xa, xb) and bits_equal(va, vb)
    assert lb >= steps  # the per-step path really launched per step


def test_fast_general_alpha_and_pair_gains(oracle):
    """FAST mode with alpha != 1 and non-unit gains that are equal within each channel pair
    (the channel-pair sharing precondition): the ALPHA1 = false kernel variant, per step within
    tolerance, masks identical. Unequal pair gains fall back to the (bit-exact) PARITY kernel."""
    from paper_2403_12820_b200 import ClothBatch, configs
    from paper_2403_12820_b200.scene import NEGATED_CHANNEL
    cfg, scenes, p, x, v = configs.build(3, batch=1, n=96)
    rng = np.random.default_rng(3)
    gains = rng.uniform(0.6, 1.4, 12)
    for c in range(12):
        gains[NEGATED_CHANNEL[c]] = gains[min(c, NEGATED_CHANNEL[c])]
    p.kernel_gain = gains
    p.isru_alpha = 1.7
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xs, vs, _ = oracle.rollout(96, 96, cds, p.to_c(), x, v, 4)
    xo, vo, mo = oracle.rollout(96, 96, cds, p.to_c(), xs, vs, 1, 4)
    with ClothBatch(scenes, p) as cb:
        l0 = cb.launch_count()
        xf, vf, mf = cb.rollout(xs, vs, 1, 4, "fast", constrained=True)
    okx, ex = fast_close(xf, xo)
    okv, ev = fast_close(vf, vo)
    assert okx and okv, "rel err x %.3g v %.3g" % (ex, ev)
    assert np.array_equal(mf, mo)
    # the FAST result is not bit-identical to PARITY here (it really ran the FAST kernel)
    assert not (bits_equal(xf, xo) and bits_equal(vf, vo))
    # unequal pair gains: FAST requests run the bit-exact PARITY kernel instead
    p.kernel_gain = rng.uniform(0.6, 1.4, 12)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xo2, vo2, _ = oracle.rollout(96, 96, cds, p.to_c(), xs, vs, 1, 4)
    with ClothBatch(scenes, p) as cb:
        xf2, vf2 = cb.rollout(xs, vs, 1, 4, "fast")
    assert bits_equal(xf2, xo2) and bits_equal(vf2, vo2)
