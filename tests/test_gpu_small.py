"""The small-cloth FAST kernel (csrc/small_kernels.cu: <= 1024 nodes per cloth, one CTA per
cloth, one thread per node, every timestep of the advance in one launch) against the C oracle —
the per-node evaluation follows the reference's channel order (forward_impulse<T>,
kernels.hpp:265-282; add_plug_impulse / advance_with_impulse, kernels.hpp:179-252) in FAST
arithmetic, so the bar is the FAST tolerance, not bit identity with the row-pass kernels."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def rel_errors(a, b):
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    err = np.abs(a - b)
    rms = np.sqrt(np.mean(b * b, axis=0))
    return float((err / np.maximum(np.abs(b), rms)).max()), float(err.max() / np.abs(b).max())


# config 1 (32^2, corner pins), config 3's dynamics shrunk (sphere, friction 0), config 5's mixed
# classes shrunk (top row / corners / free onto the plane), a ragged 20 x 30 grid
CASES = [(1, 32, 1), (3, 32, 3), (5, 32, 6), (2, 24, 2)]


@pytest.mark.parametrize("cfg_id,n,batch", CASES)
def test_small_two_steps_vs_oracle(oracle, cfg_id, n, batch):
    """Two timesteps (one small-kernel launch) from the oracle's state after 20 steps, against
    two oracle steps: per component within 1e-5 of max(|b|, rms(b)) per step (2e-5 for two)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    pc = p.to_c()
    xs, vs, _ = oracle.rollout(n, n, cds, pc, x, v, 20)
    xo, vo, _ = oracle.rollout(n, n, cds, pc, xs, vs, 2, 20)
    with ClothBatch(scenes, p) as cb:
        l0 = cb.launch_count()
        xf, vf = cb.rollout(xs, vs, 2, 20, "fast")
        launches = cb.launch_count() - l0
    ex, nx_ = rel_errors(xf, xo)
    ev, nv = rel_errors(vf, vo)
    print("small kernel cfg%d n=%d: x %.3g / %.3g, v %.3g / %.3g" % (cfg_id, n, ex, nx_, ev, nv))
    assert ex <= 2e-5 and ev <= 2e-5
    assert launches <= 3  # layout in + one small-kernel launch + layout out


def test_small_config1_rollout_one_launch(oracle):
    """Config 1's 100-step rollout: one kernel launch for the stepping, split-independent
    (k0 continuation bit-identical), and within a short-horizon drift bound of the oracle."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(1)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    with ClothBatch(scenes, p) as cb:
        l0 = cb.launch_count()
        xa, va = cb.rollout(x, v, 100, 0, "fast")
        la = cb.launch_count() - l0
        x1, v1 = cb.rollout(x, v, 37, 0, "fast")
        x2, v2 = cb.rollout(x1, v1, 63, 37, "fast")
        xb, vb = cb.rollout(x, v, 10, 0, "fast")
    assert la <= 3
    assert bits_equal(x2, xa) and bits_equal(v2, va)
    xo, vo, _ = oracle.rollout(32, 32, cds, p.to_c(), x, v, 10)
    drift = max(rel_errors(xb, xo)[1], rel_errors(vb, vo)[1])
    print("config 1, 10 FAST steps vs oracle: normwise drift %.3g" % drift)
    assert drift <= 1e-4
    assert np.isfinite(xa).all() and np.isfinite(va).all()


def test_small_disabled_by_env(monkeypatch):
    """SC_SMALL=0 (read at set_scene) routes config 1 through the wavefront kernel: one launch
    as well, results within the FAST tolerance of the small kernel's."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(1)
    with ClothBatch(scenes, p) as cb:
        xa, va = cb.rollout(x, v, 2, 0, "fast")
    monkeypatch.setenv("SC_SMALL", "0")
    with ClothBatch(scenes, p) as cb:
        xb, vb = cb.rollout(x, v, 2, 0, "fast")
    assert not (bits_equal(xa, xb) and bits_equal(va, vb))  # really a different kernel
    assert rel_errors(xa, xb)[0] <= 2e-5 and rel_errors(va, vb)[0] <= 2e-5
