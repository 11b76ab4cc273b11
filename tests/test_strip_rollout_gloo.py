"""The real row-strip driver, StripRollout._step (paper_2403_12820_b200/strips.py), on CPU over
gloo process groups of 2 and 3 ranks. Each rank drives an oracle-backed stand-in for its strip
context (same strip_step / halo_pack / halo_unpack / strip_commit surface as the GPU context),
so the very sequencing code the NCCL path runs — boundary rows first, halo pack, the batched
isend/irecv, interior rows while the halo is in flight, wait, unpack, commit — is exercised
with real message passing. The assembled owned rows must equal the single-domain oracle rollout
bit for bit (reference halo depth: the 2-row stencil reach, grid.cpp:24-27; per-step loop
eval.cpp:62-65)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

NX, NY, STEPS = 12, 23, 7


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
    rng = np.random.default_rng(11)
    ix = np.tile(np.arange(NX), NY)
    iy = np.repeat(np.arange(NY), NX)
    x = np.stack([ix / (NX - 1), iy / (NX - 1), 0.0 * ix], 1) + rng.normal(0, 1e-3, (NX * NY, 3))
    x = x.astype(np.float32)
    v = rng.normal(0, 0.05, x.shape).astype(np.float32)
    pins = sorted(list(range((NY - 1) * NX, NY * NX)) + [NX // 2, 9 * NX + 3])
    p = np.zeros(53)
    p[0:12] = 1.0
    p[12:52] = rng.normal(0, 0.05, 40)
    p[52] = 1.0
    z = scene_arrays(NX, NY, 1.0 / 240, pin_nodes=pins, pin_anchors=x[pins].astype(np.float64),
                     spheres=[(0.5, 0.4, -0.05, 0.2, 0.1)])
    return x, v, p, z, cloth_desc, params_c


class OracleStripCtx:
    """A strip context computed by the C oracle: the local window (owned rows + up to 2 ghost
    rows per side) as a stand-alone grid with the pins translated to window-local nodes; owned
    rows are >= 2 rows from any window edge that is not the cloth's own edge, so every owned row
    sees exactly the neighbourhood it has in the whole cloth."""

    def __init__(self, z, pc, row0, rows, g0, g1, cloth_desc, orc):
        self.u0, self.u1, self.g0, self.g1 = row0, row0 + rows, g0, g1
        zz = dict(z)
        nodes, anchors = [], []
        for n, a in zip(z["pin_nodes"], z["pin_anchors"]):
            if g0 <= n // NX < g1:
                nodes.append(n - g0 * NX)
                anchors.append(a)
        zz["pin_nodes"] = np.array(nodes, np.int32)
        zz["pin_anchors"] = np.array(anchors, np.float64).reshape(-1, 3)
        self.keep = []
        self.cd = cloth_desc(zz, self.keep)
        self.pc, self.orc = pc, orc
        self.dt = np.float32(float(z["dt"]))
        self.cur = self.nxt = None
        self.calls = []

    def set_state(self, x, v):
        self.cur = (np.array(x, np.float32), np.array(v, np.float32))
        self.nxt = (self.cur[0].copy(), self.cur[1].copy())

    def get_state(self):
        return self.cur[0].copy(), self.cur[1].copy()

    def halo_elems(self):
        return 2 * NX * 6

    def _rows(self, arrs, g):  # global row -> slice of the window arrays
        return slice((g - self.g0) * NX, (g - self.g0 + 1) * NX)

    def strip_step(self, k, r_begin, r_end, mode, stream):
        assert self.u0 <= r_begin <= r_end <= self.u1
        self.calls.append(("step", r_begin, r_end))
        nyw = self.g1 - self.g0
        xo, vo, _, _ = self.orc.nn_step(NX, nyw, self.cd, self.pc, self.cur[0], self.cur[1],
                                        np.float32(k + 1) * self.dt)
        sl = slice((r_begin - self.g0) * NX, (r_end - self.g0) * NX)
        self.nxt[0][sl] = xo[sl]
        self.nxt[1][sl] = vo[sl]

    def _buf(self, ptr):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(2 * NX * 6,))

    def halo_pack(self, side, ptr, stream):
        self.calls.append(("pack", side))
        g = self.u0 if side == 0 else self.u1 - 2
        buf = self._buf(ptr)
        for r in range(2):
            s = self._rows(self.nxt, g + r)
            buf[r * 6 * NX:(r * 6 + 3) * NX] = self.nxt[0][s].ravel()
            buf[(r * 6 + 3) * NX:(r + 1) * 6 * NX] = self.nxt[1][s].ravel()

    def halo_unpack(self, side, ptr, stream):
        self.calls.append(("unpack", side))
        g = self.u0 - 2 if side == 0 else self.u1
        buf = self._buf(ptr)
        for r in range(2):
            s = self._rows(self.nxt, g + r)
            self.nxt[0][s] = buf[r * 6 * NX:(r * 6 + 3) * NX].reshape(NX, 3)
            self.nxt[1][s] = buf[(r * 6 + 3) * NX:(r + 1) * 6 * NX].reshape(NX, 3)

    def strip_commit(self):
        self.calls.append(("commit",))
        self.cur = self.nxt
        self.nxt = (self.cur[0].copy(), self.cur[1].copy())

    def close(self):
        pass


def _worker(rank, world, port, q):
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
        pc = params_c(p)
        ctx = OracleStripCtx(z, pc, row0, rows, g0, g1, cloth_desc, orc)

        class _Scene:  # StripRollout reads only ny from the scene when a ctx is given
            ny = NY

        sr = strips.StripRollout(_Scene(), None, x[g0 * NX:g1 * NX], v[g0 * NX:g1 * NX], rank,
                                 world, mode="parity", ctx=ctx)
        for k in range(STEPS):
            sr.step(k)
        xs, vs = sr.state()
        own = slice((row0 - g0) * NX, (row0 - g0 + rows) * NX)
        q.put((rank, row0, rows, xs[own], vs[own], ctx.calls[:12]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strip_rollout_step_over_gloo_matches_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x, v, p, z, cloth_desc, params_c = _problem()
    from oracle.pyoracle import Oracle
    keep = []
    xo, vo, _ = Oracle().rollout(NX, NY, [cloth_desc(z, keep)], params_c(p), x[None], v[None],
                                 STEPS)
    xg, vg = np.empty_like(x), np.empty_like(v)
    for rank, row0, rows, xs, vs, calls in res:
        xg[row0 * NX:(row0 + rows) * NX] = xs
        vg[row0 * NX:(row0 + rows) * NX] = vs
        # the driver's order within a step: boundary rows, packs, interior, unpacks, commit
        kinds = [c[0] for c in calls[:calls.index(("commit",)) + 1]]
        first_interior = max(i for i, c in enumerate(kinds) if c == "step")
        assert all(c == "step" for c in kinds[:kinds.index("pack")]) if "pack" in kinds else True
        assert kinds.index("pack") < first_interior < kinds.index("unpack") if "pack" in kinds \
            else True
    assert np.array_equal(xg.view(np.uint32), xo[0].view(np.uint32))
    assert np.array_equal(vg.view(np.uint32), vo[0].view(np.uint32))
