"""Parity at the BASELINE configs' full sizes (reference run_steps<float>,
eval.cpp:48-59):

  * every cloth of configs 2 (64 x 256^2) and 5 (4096 x 128^2, all three boundary classes), the
    1024^2 cloth of config 3 and the 8192^2 cloth of config 4, from the initial state and from
    the state after 10 steps: one PARITY step is bit-exact with the C oracle (x, v and the
    contact mask), and one FAST step is within the FAST bar of it;
  * config 3's full 500-step PARITY rollout equals the reference itself (oracle/_ref, the
    unmodified reference sources) bit for bit, final contact mask included.

FAST bar (north_star: "per-step outputs within 1e-5 relative"): per component plane,
|a - b| <= 1e-5 * max(|b|, rms(b)), and the normwise error max|a - b| / max|b| <= 1e-6. The
measured maxima are printed (DESIGN.md §2 lists them per config). SURVEY §8(d)(ii)'s alternative
floor of 1e-6 * rms(b) is reported, not asserted: outputs that are the difference of O(rms)
quantities (a velocity crossing zero) carry an absolute rounding error of ~1 ulp of the rms in
any non-bit-exact evaluation order, which that floor turns into relative errors up to ~0.1.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAST_RTOL = 1e-5
FAST_NORMWISE = 1e-6


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def oracle_step(o, n, cds, pc, x, v, k, threads=16):
    """One run_steps step (t_next = (k+1) dt) of every cloth on the C oracle, cloth-parallel."""
    B = x.shape[0]
    xo, vo = np.empty_like(x), np.empty_like(v)
    mo = np.empty((B, n * n), np.uint8)
    per = max(1, (B + threads - 1) // threads)

    def work(b0, b1):
        a, b, m = o.rollout(n, n, cds[b0:b1], pc, x[b0:b1], v[b0:b1], 1, k)
        xo[b0:b1], vo[b0:b1], mo[b0:b1] = a, b, m

    ts = [threading.Thread(target=work, args=(i, min(B, i + per))) for i in range(0, B, per)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return xo, vo, mo


def errors(a, b):
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    rms = np.sqrt(np.mean(b * b, axis=0))
    err = np.abs(a - b)
    return {"rms_floor": float((err / np.maximum(np.abs(b), rms)).max()),
            "tight_floor": float((err / np.maximum(np.abs(b), 1e-6 * rms)).max()),
            "normwise": float(err.max() / np.abs(b).max())}


@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg_id", [2, 3, 4, 5])
def test_fullsize_step_parity_and_fast(cfg_id, oracle):
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(cfg_id, threads=16)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    pc = p.to_c()
    n = cfg.n
    with ClothBatch(scenes, p) as cb:
        xs, vs, kdone = x, v, 0
        for k in (0, 10):
            if k > kdone:
                xs, vs = cb.rollout(xs, vs, k - kdone, kdone, "parity")
                kdone = k
            xp, vp, mp = cb.rollout(xs, vs, 1, k, "parity", constrained=True)
            xf, vf, mf = cb.rollout(xs, vs, 1, k, "fast", constrained=True)
            xo, vo, mo = oracle_step(oracle, n, cds, pc, xs, vs, k)
            assert bits_equal(xp, xo) and bits_equal(vp, vo), "config %d step %d" % (cfg_id, k + 1)
            assert np.array_equal(mp.reshape(mo.shape), mo)
            assert np.array_equal(mf.reshape(mo.shape), mo)
            ex, ev = errors(xf, xo), errors(vf, vo)
            print("config %d step %d FAST x %s v %s" % (cfg_id, k + 1, ex, ev))
            for e in (ex, ev):
                assert e["rms_floor"] <= FAST_RTOL and e["normwise"] <= FAST_NORMWISE, (ex, ev)
            assert np.isfinite(xo).all() and np.isfinite(vo).all()


@pytest.mark.timeout(600)
def test_config3_full_rollout_equals_reference(reference):
    """500 PARITY steps of the 1024^2 cloth dropped on its sphere against the reference's own
    templates at T = float (oracle/_ref, node-parallel OpenMP), bit for bit."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(3, threads=16)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xr, vr, mr = reference.rollout_f32(cfg.n, cfg.n, cds, p.to_c(), x, v, cfg.steps)
    with ClothBatch(scenes, p) as cb:
        xg, vg, mg = cb.rollout(x, v, cfg.steps, 0, "parity", constrained=True)
    assert bits_equal(xg, xr) and bits_equal(vg, vr)
    assert np.array_equal(mg.reshape(np.asarray(mr).shape), mr)
    assert mg.any()  # the sheet really reached the sphere
    print("config 3: 500 steps bit-exact, %d contact nodes at the end, max |v| %.3g"
          % (int(mg.sum()), float(np.abs(vg).max())))
