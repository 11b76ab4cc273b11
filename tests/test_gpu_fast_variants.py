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
