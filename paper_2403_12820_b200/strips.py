"""Row-strip domain decomposition of one tall cloth across ranks.

Rank r owns global rows [row0, row0 + rows) of an ny-row cloth and keeps up to two ghost rows on
each side (the stencil reaches +-2 rows: the skip channels N2/S2, reference grid.cpp:24-27).
Per step:
  1. the two boundary rows next to each neighbour are stepped first,
  2. they are packed and exchanged with the neighbours (batch_isend_irecv: NCCL over NVLink on
     GPUs, gloo in the CPU tests) while
  3. the interior rows are stepped (they never read ghost rows), then
  4. the received rows land in the ghost rows and the state buffers swap.
Nodes, pins and masks keep their GLOBAL indices; only the state buffer is local, so every row
is computed with exactly the arithmetic of the single-GPU kernel (bit-identical results).

transport="peer" (FAST mode) replaces steps 1-4 by one fused kernel per step: the boundary rows
are stored straight into the neighbours' ghost rows through CUDA IPC mappings of their state
buffers (NVLink peer stores), with a completion-flag handshake instead of NCCL
(sc_ctx_peer_step, csrc/capi.cu). The handles are exchanged once with all_gather_object.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

HALO = 2  # stencil radius in rows


def strip_bounds(ny: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous row strips, the first ny % world ranks taking one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("strip_bounds: bad rank/world")
    base, extra = divmod(ny, world)
    if base < HALO:
        raise ValueError("strip_bounds: each strip needs at least %d rows" % HALO)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def local_window(ny: int, row0: int, rows: int) -> Tuple[int, int]:
    """Global rows [g0, g1) held locally: the owned rows plus up to HALO ghost rows per side."""
    return max(0, row0 - HALO), min(ny, row0 + rows + HALO)


def halo_plan(ny: int, world: int, rank: int):
    """(send_lo, send_hi, recv_lo, recv_hi) global row ranges of this rank's exchange; None when
    the side has no neighbour. send_lo goes to rank-1 (its high ghosts), send_hi to rank+1."""
    row0, rows = strip_bounds(ny, world, rank)
    send_lo = (row0, row0 + HALO) if rank > 0 else None
    send_hi = (row0 + rows - HALO, row0 + rows) if rank < world - 1 else None
    recv_lo = (row0 - HALO, row0) if rank > 0 else None
    recv_hi = (row0 + rows, row0 + rows + HALO) if rank < world - 1 else None
    return send_lo, send_hi, recv_lo, recv_hi


def exchange(rank: int, world: int, send_lo, send_hi, recv_lo, recv_hi, group=None) -> list:
    """Post the halo send/recv pairs as one batch (tensors: contiguous, same shape per pair).
    Returns the works to wait on."""
    import torch.distributed as dist

    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, send_lo, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_lo, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, send_hi, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_hi, rank + 1, group))
    return dist.batch_isend_irecv(ops) if ops else []


class StripRollout:
    """One rank's strip of a tall cloth on its GPU, stepped with halo exchange over NCCL.

    x_local / v_local: AoS f32 state of the local window rows (ghosts included). The scene is
    the cloth's global descriptor (global pins; positions not needed)."""

    def __init__(self, scene, params, x_local, v_local, rank: int, world: int, device: int = 0,
                 group=None, mode: str = "fast", transport: str = "nccl", ctx=None):
        """ctx: a strip context to drive instead of the GPU one (the CPU tests pass an
        oracle-backed stand-in with the same strip_step / halo_pack / halo_unpack /
        strip_commit surface; its halo buffers are then host tensors and there is no stream)."""
        import torch

        from .api import ClothBatch

        if transport not in ("nccl", "peer"):
            raise ValueError("transport: 'nccl' or 'peer'")
        if transport == "peer" and mode != "fast":
            raise ValueError("transport 'peer' runs the FAST kernel")
        self.rank, self.world, self.group, self.mode = rank, world, group, mode
        self.transport = transport if world > 1 else "nccl"  # one strip: nothing to exchange
        self.ny = scene.ny
        self.row0, self.rows = strip_bounds(scene.ny, world, rank)
        self.g0, self.g1 = local_window(scene.ny, self.row0, self.rows)
        if ctx is None:
            self.ctx = ClothBatch([scene], params, "f32", device, strip=(self.row0, self.rows))
            dev = torch.device("cuda", device)
        else:
            if self.transport == "peer":
                raise ValueError("transport 'peer' needs the GPU context")
            self.ctx = ctx
            dev = torch.device("cpu")
        self.ctx.set_state(x_local, v_local)
        n = self.ctx.halo_elems()
        self.send_lo, self.send_hi, self.recv_lo, self.recv_hi = (
            torch.zeros(n, dtype=torch.float32, device=dev) for _ in range(4))
        # a real (non-legacy) stream: kernels, packs and NCCL all order on it
        self.stream = torch.cuda.Stream(device=dev) if ctx is None else None
        if transport == "peer" and world > 1:
            import torch.distributed as dist
            exports = [None] * world
            dist.all_gather_object(exports, self.ctx.peer_export(), group=group)
            if rank > 0:
                self.ctx.set_peer(0, exports[rank - 1], ipc=True)
            if rank < world - 1:
                self.ctx.set_peer(1, exports[rank + 1], ipc=True)
            dist.barrier(group=group)

    @staticmethod
    def link_local(lower: "StripRollout", upper: "StripRollout") -> None:
        """Link two strips held by one process (same device) for the fused peer path."""
        lower.ctx.set_peer(1, upper.ctx.peer_export(), ipc=False)
        upper.ctx.set_peer(0, lower.ctx.peer_export(), ipc=False)

    def step(self, k: int) -> None:
        import torch

        if self.stream is None:
            self._step(k, None)
            return
        with torch.cuda.stream(self.stream):
            self._step(k, self.stream.cuda_stream)

    def _step(self, k: int, stream: int) -> None:
        if self.transport == "peer":
            self.ctx.peer_step(k, self.mode, stream)
            return
        r0, r1 = self.row0, self.row0 + self.rows
        lo_end = min(r1, r0 + HALO) if self.rank > 0 else r0
        hi_beg = max(lo_end, r1 - HALO) if self.rank < self.world - 1 else r1
        # 1. boundary rows first
        if lo_end > r0:
            self.ctx.strip_step(k, r0, lo_end, self.mode, stream)
        if r1 > hi_beg:
            self.ctx.strip_step(k, hi_beg, r1, self.mode, stream)
        # 2. ship them (NCCL orders itself after the work queued so far on this stream)
        if self.rank > 0:
            self.ctx.halo_pack(0, self.send_lo.data_ptr(), stream)
        if self.rank < self.world - 1:
            self.ctx.halo_pack(1, self.send_hi.data_ptr(), stream)
        works = exchange(self.rank, self.world, self.send_lo, self.send_hi, self.recv_lo,
                         self.recv_hi, self.group) if self.world > 1 else []
        # 3. interior rows overlap the transfer
        if hi_beg > lo_end:
            self.ctx.strip_step(k, lo_end, hi_beg, self.mode, stream)
        # 4. ghosts in, swap
        for w in works:
            w.wait()
        if self.rank > 0:
            self.ctx.halo_unpack(0, self.recv_lo.data_ptr(), stream)
        if self.rank < self.world - 1:
            self.ctx.halo_unpack(1, self.recv_hi.data_ptr(), stream)
        self.ctx.strip_commit()

    def state(self):
        if self.stream is not None:
            self.stream.synchronize()
        return self.ctx.get_state()

    def close(self) -> None:
        self.ctx.close()
