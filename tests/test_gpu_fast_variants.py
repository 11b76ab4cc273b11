"""FAST kernel variants and schedules on the GPU: the simple-finish kernels (no collider / mask:
the collider-free configs' hot path) within tolerance of the oracle per step, and every kernel
variant / row segmentation bit-identical to every other (a node's arithmetic does not depend on
which unit, register budget or wave computes it; fast_kernels.cu plan_fast / fast_step_kernel)."""
import numpy as np
import pytest

from test_gpu_parity import bits_equal, fast_close

pytestmark = pytest.mark.gpu


def _build(cfg_id, n, batch):
    from paper_2403_12820_b200 import configs
    return configs.build(cfg_id, batch=batch, n=n)


@pytest.mark.parametrize("cfg_id,n,batch,wide", [(2, 256, 4, "auto"), (4, 512, 1, "1"),
                                                 (4, 512, 1, "0"), (2, 256, 2, "1")])
def test_fast_simple_finish_per_step(oracle, monkeypatch, cfg_id, n, batch, wide):
    """No mask output and no collider: the GEN = false kernels (16-CTA and wide-register),
    per step from identical input states, within the FAST tolerance of the oracle."""
    from paper_2403_12820_b200 import ClothBatch
    if wide != "auto":
        monkeypatch.setenv("SC_FAST_WIDE", wide)
    cfg, scenes, p, x, v = _build(cfg_id, n, batch)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xs, vs, _ = oracle.rollout(n, n, cds, p.to_c(), x, v, 3)
    xo, vo, _ = oracle.rollout(n, n, cds, p.to_c(), xs, vs, 1, 3)
    with ClothBatch(scenes, p) as cb:
        xf, vf = cb.rollout(xs, vs, 1, 3, "fast")
    okx, ex = fast_close(xf, xo)
    okv, ev = fast_close(vf, vo)
    assert okx and okv, "rel err x %.3g v %.3g" % (ex, ev)


@pytest.mark.parametrize("cfg_id,n,batch", [(4, 512, 1), (2, 256, 4), (5, 128, 6)])
def test_fast_variants_and_segmentations_bit_identical(monkeypatch, cfg_id, n, batch):
    """8-step FAST rollouts: 16-CTA vs wide-register kernel, planner's segmentation vs short and
    long forced segments — all bit-identical."""
    from paper_2403_12820_b200 import ClothBatch
    cfg, scenes, p, x, v = _build(cfg_id, n, batch)
    runs = []
    for wide, seg in (("0", None), ("1", None), ("0", "5"), ("1", "40"), ("0", "64")):
        monkeypatch.setenv("SC_FAST_WIDE", wide)
        if seg is None:
            monkeypatch.delenv("SC_FAST_SEG_ROWS", raising=False)
        else:
            monkeypatch.setenv("SC_FAST_SEG_ROWS", seg)
        with ClothBatch(scenes, p) as cb:
            runs.append(cb.rollout(x, v, 8, 0, "fast"))
    x0, v0 = runs[0]
    assert np.isfinite(x0).all() and np.isfinite(v0).all()
    for xr, vr in runs[1:]:
        assert bits_equal(xr, x0) and bits_equal(vr, v0)


@pytest.mark.parametrize("n,cz,friction", [(256, -0.27, 0.0), (384, -0.29, 0.3), (128, -0.25, 0.0)])
def test_sphere_broad_phase_keeps_contacts_exact(oracle, n, cz, friction):
    """The one-sphere finish skips the collider response for warp rows whose nodes are provably
    outside the sphere (fast_rowpass.cuh sphere_near). A sphere whose cap cuts the sheet from the
    first step gives rows entirely outside, rows entirely inside and rows where only some lanes
    touch: per step from identical input states the contact masks equal the oracle's and the
    states stay within the FAST tolerance, with and without the mask output (the sphere-only and
    the general-dispatch instantiations)."""
    from paper_2403_12820_b200 import ClothBatch
    from paper_2403_12820_b200.scene import SphereCollider
    cfg, scenes, p, x, v = _build(3, n, 1)
    scenes[0].colliders[:] = [SphereCollider(np.array([0.47, 0.52, cz]), 0.3, friction)]
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xs, vs = x, v
    touched = 0
    with ClothBatch(scenes, p) as cb:
        for k in range(6):
            xo, vo, mo = oracle.rollout(n, n, cds, p.to_c(), xs, vs, 1, k)
            xf, vf, mf = cb.rollout(xs, vs, 1, k, "fast", constrained=True)
            xg, vg = cb.rollout(xs, vs, 1, k, "fast")
            assert np.array_equal(mf, mo), "contact mask differs at step %d" % k
            assert bits_equal(xg, xf) and bits_equal(vg, vf)
            okx, ex = fast_close(xf, xo)
            okv, ev = fast_close(vf, vo)
            assert okx and okv, "step %d rel err x %.3g v %.3g" % (k, ex, ev)
            touched = max(touched, int(mo.sum()))
            xs, vs = xo, vo
    pins = len(scenes[0].bc.nodes)
    assert pins < touched < n * n // 2, "contacts %d: the scene must mix touching and free rows" % touched
