"""Row-strip contexts on one GPU (ranks emulated sequentially: no kernel waits on another):
stepping each strip, then packing / unpacking the halo rows through device buffers, must give
bit-identical states to the whole-cloth context, in PARITY and FAST mode."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("cfg_id,n,world,steps,mode", [(4, 256, 3, 8, "fast"),
                                                         (4, 128, 4, 6, "parity"),
                                                         (3, 96, 2, 8, "fast"),
                                                         (3, 64, 3, 5, "parity")])
def test_strips_match_whole_cloth(cfg_id, n, world, steps, mode):
    import torch

    from paper_2403_12820_b200 import ClothBatch, configs, strips

    cfg, scenes, p, x, v = configs.build(cfg_id, batch=1, n=n)
    with ClothBatch(scenes, p) as whole:
        xw, vw = whole.rollout(x, v, steps, 0, mode)
    ctxs, spans = [], []
    for r in range(world):
        row0, rows = strips.strip_bounds(n, world, r)
        g0, g1 = strips.local_window(n, row0, rows)
        sc = configs.make_scene(cfg, 0, x[0][g0 * n:g1 * n].astype(np.float64), row0=g0)
        c = ClothBatch([sc], p, strip=(row0, rows))
        c.set_state(x[0][g0 * n:g1 * n], v[0][g0 * n:g1 * n])
        ctxs.append(c)
        spans.append((row0, rows, g0, g1))
    m = ctxs[0].halo_elems()
    bufs = [[torch.zeros(m, device="cuda") for _ in range(2)] for _ in range(world)]
    for k in range(steps):
        for c, (row0, rows, _, _) in zip(ctxs, spans):
            c.strip_step(k, row0, row0 + rows, mode)
        for c in ctxs:
            c.sync()
        for r, c in enumerate(ctxs):
            if r > 0:
                c.halo_pack(0, bufs[r][0].data_ptr())
            if r < world - 1:
                c.halo_pack(1, bufs[r][1].data_ptr())
            c.sync()
        for r, c in enumerate(ctxs):
            if r > 0:  # my low ghosts <- rank r-1's high rows
                c.halo_unpack(0, bufs[r - 1][1].data_ptr())
            if r < world - 1:  # my high ghosts <- rank r+1's low rows
                c.halo_unpack(1, bufs[r + 1][0].data_ptr())
            c.sync()
            c.strip_commit()
    for c, (row0, rows, g0, g1) in zip(ctxs, spans):
        xs, vs = c.get_state()
        own = slice((row0 - g0) * n, (row0 + rows - g0) * n)
        glob = slice(row0 * n, (row0 + rows) * n)
        assert bits_equal(xs[0][own], xw[0][glob]) and bits_equal(vs[0][own], vw[0][glob])
        c.close()
