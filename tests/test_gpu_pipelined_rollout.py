"""The host -> host FAST rollout with overlapped transfers (capi.cu rollout_pipelined: chunks of
cloths on their own streams, page-locked host arrays) against the plain path: bit-identical
states, odd and even step counts, plain and z-swizzled layouts, 2- and 4-chunk splits."""
import numpy as np
import pytest

from test_gpu_parity import bits_equal

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg_id,n,batch,steps", [(2, 256, 8, 9), (2, 128, 32, 12),
                                                  (5, 128, 9, 9), (1, 32, 16, 10)])
def test_pipelined_rollout_bit_identical(monkeypatch, cfg_id, n, batch, steps):
    from paper_2403_12820_b200 import ClothBatch, configs
    from paper_2403_12820_b200.api import pinned_empty
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    xp, vp = pinned_empty(x.shape), pinned_empty(v.shape)
    xp[...] = x
    vp[...] = v
    with ClothBatch(scenes, p) as cb:
        xa, va = cb.rollout(x, v, steps, 3, "fast")  # pageable: plain path
        l0 = cb.launch_count()
        xo, vo = pinned_empty(x.shape), pinned_empty(v.shape)
        xb, vb = cb.rollout(xp, vp, steps, 3, "fast", out=(xo, vo))  # pipelined
        lp = cb.launch_count() - l0
        monkeypatch.setenv("SC_PIPELINE", "0")
        xc, vc = cb.rollout(xp, vp, steps, 3, "fast")
    assert xb is xo and vb is vo
    assert bits_equal(xb, xa) and bits_equal(vb, va)
    assert bits_equal(xc, xa) and bits_equal(vc, va)
    assert lp >= 2 * steps  # the pipelined path ran (one launch per chunk and step)
