"""Row-strip decomposition host logic (paper_2403_12820_b200/strips.py) on CPU: world_size 2
and 3 gloo process groups, the oracle as the per-rank compute engine, halo rows exchanged with
strips.exchange(). The assembled owned rows must equal the single-domain oracle rollout bit for
bit — the property the GPU path (same strip_bounds / halo_plan / exchange, NCCL) relies on."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

NX, NY, STEPS = 12, 23, 6


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    from golden_io import cloth_desc, params_c, scene_arrays
    rng = np.random.default_rng(7)
    ix = np.tile(np.arange(NX), NY)
    iy = np.repeat(np.arange(NY), NX)
    x = np.stack([ix / (NX - 1), iy / (NX - 1), 0.0 * ix], 1) + rng.normal(0, 1e-3, (NX * NY, 3))
    x = x.astype(np.float32)
    v = rng.normal(0, 0.05, x.shape).astype(np.float32)
    pins = list(range((NY - 1) * NX, NY * NX)) + [NX // 2]
    p = np.zeros(53)
    p[0:12] = 1.0
    p[12:52] = rng.normal(0, 0.05, 40)
    p[52] = 1.0
    z = scene_arrays(NX, NY, 1.0 / 240, pin_nodes=sorted(pins),
                     pin_anchors=x[sorted(pins)].astype(np.float64),
                     spheres=[(0.5, 0.4, -0.05, 0.2, 0.1)])
    return x, v, p, z, cloth_desc, params_c


def _block_desc(z, g0, g1, cloth_desc):
    """The scene restricted to local rows [g0, g1): pins translated to block-local indices."""
    zz = dict(z)
    nodes, anchors = [], []
    for n, a in zip(z["pin_nodes"], z["pin_anchors"]):
        if g0 <= n // NX < g1:
            nodes.append(n - g0 * NX)
            anchors.append(a)
    zz["pin_nodes"] = np.array(nodes, np.int32)
    zz["pin_anchors"] = np.array(anchors, np.float64).reshape(-1, 3)
    keep = []
    return cloth_desc(zz, keep), keep


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, v, p, z, cloth_desc, params_c = _problem()
        from oracle.pyoracle import Oracle
        from paper_2403_12820_b200 import strips
        orc = Oracle()
        row0, rows = strips.strip_bounds(NY, world, rank)
        g0, g1 = strips.local_window(NY, row0, rows)
        cd, keep = _block_desc(z, g0, g1, cloth_desc)
        pc = params_c(p)
        xl = x[g0 * NX:g1 * NX].copy()
        vl = v[g0 * NX:g1 * NX].copy()
        send_lo, send_hi, recv_lo, recv_hi = strips.halo_plan(NY, world, rank)
        n = strips.HALO * NX * 6
        bufs = [torch.zeros(n) for _ in range(4)]

        def pack(xa, va, rr, buf):
            sl = slice((rr[0] - g0) * NX, (rr[1] - g0) * NX)
            buf.copy_(torch.from_numpy(np.concatenate([xa[sl].ravel(), va[sl].ravel()])))

        def unpack(xa, va, rr, buf):
            sl = slice((rr[0] - g0) * NX, (rr[1] - g0) * NX)
            h = buf.numpy()
            xa[sl] = h[:n // 2].reshape(-1, 3)
            va[sl] = h[n // 2:].reshape(-1, 3)

        for k in range(STEPS):
            xn, vn, _, _ = orc.nn_step(NX, g1 - g0, cd, pc, xl, vl,
                                       np.float32(k + 1) * np.float32(float(z["dt"])))
            if send_lo:
                pack(xn, vn, send_lo, bufs[0])
            if send_hi:
                pack(xn, vn, send_hi, bufs[1])
            for w in strips.exchange(rank, world, bufs[0], bufs[1], bufs[2], bufs[3]):
                w.wait()
            if recv_lo:
                unpack(xn, vn, recv_lo, bufs[2])
            if recv_hi:
                unpack(xn, vn, recv_hi, bufs[3])
            xl, vl = xn, vn
        own = slice((row0 - g0) * NX, (row0 + rows - g0) * NX)
        q.put((rank, row0, rows, xl[own].copy(), vl[own].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_decomposition_matches_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x, v, p, z, cloth_desc, params_c = _problem()
    from oracle.pyoracle import Oracle
    keep = []
    xo, vo, _ = Oracle().rollout(NX, NY, [cloth_desc(z, keep)], params_c(p), x[None], v[None],
                                 STEPS)
    covered = 0
    for rank, row0, rows, xs, vs in results:
        sl = slice(row0 * NX, (row0 + rows) * NX)
        assert np.array_equal(xs.view(np.uint32), xo[0][sl].view(np.uint32)), rank
        assert np.array_equal(vs.view(np.uint32), vo[0][sl].view(np.uint32)), rank
        covered += rows
    assert covered == NY


def test_strip_bounds_cover_and_halo_plan():
    from paper_2403_12820_b200 import strips
    for ny, world in [(8192, 8), (23, 3), (100, 7), (4, 2)]:
        spans = [strips.strip_bounds(ny, world, r) for r in range(world)]
        assert spans[0][0] == 0 and sum(r for _, r in spans) == ny
        for (a0, n0), (a1, _) in zip(spans, spans[1:]):
            assert a0 + n0 == a1
        for r in range(world):
            sl, sh, rl, rh = strips.halo_plan(ny, world, r)
            assert (sl is None) == (r == 0) and (rh is None) == (r == world - 1)
            if r > 0:  # what I receive below is what rank-1 sends above
                assert rl == strips.halo_plan(ny, world, r - 1)[1]
    with pytest.raises(ValueError):
        strips.strip_bounds(3, 2, 0)
