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
        cb.set_persistent(False)  # the streaming kernel's chunked pipeline (not the wavefront)
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


@pytest.mark.parametrize("cfg_id,n,batch", [(2, 128, 16), (5, 128, 12), (2, 256, 9)])
def test_chunked_stepping_bit_identical_to_whole_batch(monkeypatch, cfg_id, n, batch):
    """Device-resident FAST stepping in concurrent cloth chunks (capi.cu chunked_fast_steps)
    against one whole-batch launch per step: bit-identical states."""
    from paper_2403_12820_b200 import ClothBatch, configs
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n)
    out = {}
    for k in ("0", "2", "4"):
        monkeypatch.setenv("SC_CHUNKS", k)
        with ClothBatch(scenes, p) as cb:
            cb.set_persistent(False)  # streaming kernel: chunked launches per step
            cb.set_state(x, v)
            l0 = cb.launch_count()
            cb.advance(11, 0, "fast")
            out[k] = cb.get_state() + (cb.launch_count() - l0,)
    x0, v0, n0 = out["0"]
    assert n0 >= 11
    for k in ("2", "4"):
        xk, vk, nk = out[k]
        assert nk == n0 + 11 * (min(int(k), batch // 2) - 1)  # K launches per step
        assert bits_equal(xk, x0) and bits_equal(vk, v0)


def test_chunked_stepping_vs_oracle(oracle):
    """Two FAST steps of 8 config-2 cloths (chunked: 2 chunks) from the oracle's state after 3
    steps, within the FAST tolerance of the oracle's next two steps."""
    from paper_2403_12820_b200 import ClothBatch, configs
    from test_gpu_parity import fast_close
    n, batch = 256, 8
    cfg, scenes, p, x, v = configs.build(2, batch=batch, n=n)
    keep = []
    cds = [s.cloth_desc(keep) for s in scenes]
    xs, vs, _ = oracle.rollout(n, n, cds, p.to_c(), x, v, 3)
    xo, vo, _ = oracle.rollout(n, n, cds, p.to_c(), xs, vs, 2, 3)
    with ClothBatch(scenes, p) as cb:
        cb.set_state(xs, vs)
        l0 = cb.launch_count()
        cb.advance(2, 3, "fast")
        assert cb.launch_count() - l0 >= 4  # 2 chunks x 2 steps
        xf, vf = cb.get_state()
    okx, ex = fast_close(xf, xo, 1e-5, normwise=2e-6)
    okv, ev = fast_close(vf, vo, 1e-5, normwise=2e-6)
    assert okx and okv, "rel err x %.3g v %.3g" % (ex, ev)


@pytest.mark.parametrize("cfg_id,chunks,batch,steps", [(5, "2", 300, 14), (5, "4", 600, 25),
                                                     (2, "3", 151, 2), (2, "2", 200, 9),
                                                     (5, "ramp", 600, 200)])
def test_wave_pipelined_rollout_bit_identical(monkeypatch, cfg_id, chunks, batch, steps):
    """The wavefront context's host -> host rollout in cloth chunks (capi.cu
    rollout_wave_pipelined: H2D / step / D2H of different chunks overlapped; config 5's mixed
    classes as class groups per chunk) against the plain path and the streaming kernel:
    bit-identical. "ramp": the default long-rollout chunking (capi.cu pipeline_bounds: chunks of
    148, 304, 148 cloths for 600 cloths x 200 steps on 148 SMs)."""
    from paper_2403_12820_b200 import ClothBatch, configs
    from paper_2403_12820_b200.api import pinned_empty
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=128)
    xp, vp = pinned_empty(x.shape), pinned_empty(v.shape)
    xp[...] = x
    vp[...] = v
    monkeypatch.setenv("SC_WAVE_MIN_CLOTHS", "1")  # the wavefront pipeline at these batch sizes
    monkeypatch.setenv("SC_WAVE_MIN_STEPS", "1")  # ... and step counts
    if chunks != "ramp":
        monkeypatch.setenv("SC_WAVE_CHUNKS", chunks)
    else:
        monkeypatch.delenv("SC_WAVE_CHUNKS", raising=False)
    with ClothBatch(scenes, p) as cb:
        xa, va = cb.rollout(x, v, steps, 3, "fast")  # pageable: one wavefront launch
        l0 = cb.launch_count()
        xo, vo = pinned_empty(x.shape), pinned_empty(v.shape)
        xb, vb = cb.rollout(xp, vp, steps, 3, "fast", out=(xo, vo))  # pinned: chunked, overlapped
        lp = cb.launch_count() - l0
        cb.set_persistent(False)
        xc, vc = cb.rollout(x, v, steps, 3, "fast")
    assert bits_equal(xb, xa) and bits_equal(vb, va)
    assert bits_equal(xc, xa) and bits_equal(vc, va)
    K = 3 if chunks == "ramp" else int(chunks)
    if cfg_id == 5:  # per chunk: layout in + wavefront + `steps` streaming launches + layout out
        assert lp == K * (3 + steps)
    else:  # layout in + wavefront + layout out per chunk
        assert lp == 3 * K


@pytest.mark.parametrize("cfg_id,n,band,steps", [(4, 512, "64", 37), (4, 384, "32", 150),
                                                 (3, 512, "48", 40), (4, 256, "16", 2)])
def test_band_pipelined_rollout_bit_identical(monkeypatch, cfg_id, n, band, steps):
    """The single-cloth host -> host rollout as a diagonal wavefront over row bands (capi.cu
    rollout_band_pipelined: band i+1 uploads while the levels computable from bands <= i step,
    finished rows download behind later bands) against the plain path: bit-identical. Small
    bands (SC_BAND_ROWS) put many bands on a test-sized grid; 2 * steps > the band height and
    steps > ny / 2 exercise the staircase's empty and clipped launches."""
    from paper_2403_12820_b200 import ClothBatch, configs
    from paper_2403_12820_b200.api import pinned_empty
    cfg, scenes, p, x, v = configs.build(cfg_id, batch=1, n=n)
    xp, vp = pinned_empty(x.shape), pinned_empty(v.shape)
    xp[...] = x
    vp[...] = v
    monkeypatch.setenv("SC_BAND_ROWS", band)
    with ClothBatch(scenes, p) as cb:
        xa, va = cb.rollout(x, v, steps, 3, "fast")  # pageable: plain path
        l0 = cb.launch_count()
        xo, vo = pinned_empty(x.shape), pinned_empty(v.shape)
        xb, vb = cb.rollout(xp, vp, steps, 3, "fast", out=(xo, vo))  # pinned: band pipeline
        lp = cb.launch_count() - l0
        monkeypatch.setenv("SC_PIPELINE", "0")
        xc, vc = cb.rollout(xp, vp, steps, 3, "fast")
    assert bits_equal(xb, xa) and bits_equal(vb, va)
    assert bits_equal(xc, xa) and bits_equal(vc, va)
    assert lp > steps + 2  # several row-range launches per level: the band path ran
