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


@pytest.mark.parametrize("cfg_id,n,world,steps", [(4, 256, 3, 8), (3, 96, 2, 6), (4, 128, 4, 5)])
def test_fused_peer_exchange_matches_whole_cloth(cfg_id, n, world, steps):
    """transport='peer': each strip's FAST kernel stores its boundary rows straight into the
    neighbours' ghost rows (here: contexts of one process linked by raw pointers; each step is
    synchronised before the next context runs, so no kernel ever waits on one not yet launched)."""
    from paper_2403_12820_b200 import ClothBatch, configs, strips

    cfg, scenes, p, x, v = configs.build(cfg_id, batch=1, n=n)
    with ClothBatch(scenes, p) as whole:
        xw, vw = whole.rollout(x, v, steps, 0, "fast")
    ctxs, spans = [], []
    for r in range(world):
        row0, rows = strips.strip_bounds(n, world, r)
        g0, g1 = strips.local_window(n, row0, rows)
        sc = configs.make_scene(cfg, 0, x[0][g0 * n:g1 * n].astype(np.float64), row0=g0)
        c = ClothBatch([sc], p, strip=(row0, rows))
        c.set_state(x[0][g0 * n:g1 * n], v[0][g0 * n:g1 * n])
        ctxs.append(c)
        spans.append((row0, rows, g0, g1))
    for r in range(world - 1):
        ctxs[r].set_peer(1, ctxs[r + 1].peer_export(), ipc=False)
        ctxs[r + 1].set_peer(0, ctxs[r].peer_export(), ipc=False)
    for k in range(steps):
        for c in ctxs:
            c.peer_step(k)
            c.sync()
    for c, (row0, rows, g0, g1) in zip(ctxs, spans):
        xs, vs = c.get_state()
        own = slice((row0 - g0) * n, (row0 + rows - g0) * n)
        glob = slice(row0 * n, (row0 + rows) * n)
        assert bits_equal(xs[0][own], xw[0][glob]) and bits_equal(vs[0][own], vw[0][glob])
        c.close()


def test_peer_link_validation():
    from paper_2403_12820_b200 import ClothBatch, ConfigError, configs, strips

    n, world = 64, 3
    cfg, scenes, p, x, v = configs.build(4, batch=1, n=n)
    ctx = []
    for r in range(world):
        row0, rows = strips.strip_bounds(n, world, r)
        g0, g1 = strips.local_window(n, row0, rows)
        sc = configs.make_scene(cfg, 0, x[0][g0 * n:g1 * n].astype(np.float64), row0=g0)
        c = ClothBatch([sc], p, strip=(row0, rows))
        c.set_state(x[0][g0 * n:g1 * n], v[0][g0 * n:g1 * n])
        ctx.append(c)
    with pytest.raises(ConfigError, match="not adjacent"):
        ctx[0].set_peer(1, ctx[2].peer_export(), ipc=False)
    with pytest.raises(ConfigError, match="no peer linked"):
        ctx[1].peer_step(0)
    ctx[0].set_peer(1, ctx[1].peer_export(), ipc=False)
    with pytest.raises(ConfigError, match="FAST f32"):
        ctx[0].peer_step(0, "parity")
    for c in ctx:
        c.close()
