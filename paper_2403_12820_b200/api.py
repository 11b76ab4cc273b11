"""Reference-compatible compute API over the C-ABI (include/stencilcloth_b200.h).

Drop-in functions for the reference's path (reference paths under /root/reference/proj):
  forward_impulse(params, scene, positions, velocities)   bindings.cpp:147-154, net.cpp:132-142
  plug_impulse(scene, positions, velocities)              sim.cpp:100-106
  advance_with_impulse(scene, x, v, impulse, t_next)      sim.cpp:134-148
  nn_step(params, scene, x, v, t_next)                    net.cpp:242-248
  rollout(params, scene, steps=-1)                        bindings.cpp:163-164, eval.cpp:86-103
  benchmark_net(params, scene, steps, warmup, precision)  eval.cpp:155-158
They run the sm_100a kernels in PARITY mode at double precision by default, i.e. bit-identical
to the reference's double-precision templates. `ClothBatch` is the batched, device-resident
f32 engine the benchmarks drive (run_steps<float>, eval.cpp:35-67, over many cloths at once).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Union

import numpy as np

from . import _abi
from .scene import (ConfigError, NetworkParams, NumericsError, Scene, Trajectory,
                    STENCIL_OFFSETS)

PRECISIONS = {"f32": _abi.SC_F32, "f64": _abi.SC_F64}
MODES = {"parity": _abi.SC_MODE_PARITY, "fast": _abi.SC_MODE_FAST}


class CudaError(RuntimeError):
    """Device / driver failure (SC_ERR_CUDA). There is no CPU fallback."""


def _raise(lib, code: int) -> None:
    if code == _abi.SC_OK:
        return
    msg = (lib.sc_last_error() or b"").decode()
    if code == _abi.SC_ERR_CONFIG:
        raise ConfigError(msg)
    if code == _abi.SC_ERR_NUMERICS:
        raise NumericsError(msg)
    if code == _abi.SC_ERR_CUDA:
        raise CudaError(msg)
    raise RuntimeError(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Context:
    """One device context bound to a batch of same-size cloths and one parameter set."""

    def __init__(self, scenes: Union[Scene, Sequence[Scene]], params: Optional[NetworkParams] = None,
                 precision: str = "f64", device: int = 0, strip: Optional[tuple] = None):
        self.lib = _abi.load()
        scenes = [scenes] if isinstance(scenes, Scene) else list(scenes)
        if not scenes:
            raise ConfigError("batch: must be >= 1")
        nx, ny = scenes[0].nx, scenes[0].ny
        for s in scenes:
            if (s.nx, s.ny) != (nx, ny):
                raise ConfigError("batch: all cloths must share one grid size")
        if precision not in PRECISIONS:
            raise ConfigError("precision: must be 'f32' or 'f64'")
        self.scenes, self.nx, self.ny, self.batch = scenes, nx, ny, len(scenes)
        self.precision = precision
        self.dtype = np.float32 if precision == "f32" else np.float64
        h = C.c_void_p()
        _raise(self.lib, self.lib.sc_ctx_create(device, PRECISIONS[precision], C.byref(h)))
        self.h = h
        self.strip = strip
        if strip is not None:
            _raise(self.lib, self.lib.sc_ctx_set_strip(self.h, int(strip[0]), int(strip[1])))
        keep: list = []
        descs = (_abi.sc_cloth_desc * self.batch)(*[s.cloth_desc(keep) for s in scenes])
        sd = _abi.sc_scene_desc(nx, ny, self.batch, C.cast(descs, C.POINTER(_abi.sc_cloth_desc)))
        _raise(self.lib, self.lib.sc_ctx_set_scene(self.h, C.byref(sd)))
        if params is not None:
            self.set_params(params)

    # -- lifecycle --
    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.sc_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def local_rows(self) -> int:
        if self.strip is None:
            return self.ny
        r0, n = self.strip
        g0 = max(0, r0 - 2)
        return min(self.ny, r0 + n + 2) - g0

    def _arr(self, a, rows: Optional[int] = None) -> np.ndarray:
        rows = self.local_rows if rows is None else rows
        a = np.ascontiguousarray(a, dtype=self.dtype)
        if a.size != self.batch * rows * self.nx * 3:
            raise ConfigError("state shape does not match the grid topology")
        return a

    def _empty(self) -> np.ndarray:
        return np.empty((self.batch, self.local_rows * self.nx, 3), dtype=self.dtype)

    def set_params(self, params: NetworkParams) -> None:
        c = params.to_c()
        _raise(self.lib, self.lib.sc_ctx_set_params(self.h, C.byref(c)))

    def set_state(self, x, v) -> None:
        x, v = self._arr(x), self._arr(v)
        _raise(self.lib, self.lib.sc_ctx_set_state(self.h, _ptr(x), _ptr(v)))

    def get_state(self):
        x, v = self._empty(), self._empty()
        _raise(self.lib, self.lib.sc_ctx_get_state(self.h, _ptr(x), _ptr(v)))
        return x, v

    def advance(self, steps: int, k0: int = 0, mode: str = "parity") -> None:
        _raise(self.lib, self.lib.sc_ctx_advance(self.h, int(steps), int(k0), MODES[mode]))

    def set_persistent(self, on: bool) -> None:
        _raise(self.lib, self.lib.sc_ctx_set_persistent(self.h, int(bool(on))))

    def set_health_checks(self, on: bool) -> None:
        _raise(self.lib, self.lib.sc_ctx_set_health_checks(self.h, int(bool(on))))

    def sync(self) -> None:
        _raise(self.lib, self.lib.sc_ctx_sync(self.h))

    def health(self):
        fi = np.zeros(self.batch, np.int32)
        fn = np.zeros(self.batch, np.int32)
        fs = np.zeros(self.batch, np.int32)
        _raise(self.lib, self.lib.sc_ctx_get_health(self.h, _ptr(fi), _ptr(fn), _ptr(fs)))
        return fi, fn, fs

    def rollout(self, x0, v0, steps: int, k0: int = 0, mode: str = "parity",
                constrained: bool = False, out=None):
        """`out`: optional preallocated (x, v) result arrays. With page-locked inputs and
        outputs (`pinned_empty`) a FAST rollout overlaps its transfers with the stepping."""
        x0, v0 = self._arr(x0), self._arr(v0)
        if out is None:
            xo, vo = self._empty(), self._empty()
        else:
            xo, vo = out
            if (xo.dtype != self.dtype or vo.dtype != self.dtype or not xo.flags.c_contiguous
                    or not vo.flags.c_contiguous or xo.size != self.batch * self.local_rows * self.nx * 3
                    or vo.size != xo.size):
                raise ConfigError("out: expected two C-contiguous state arrays of the context dtype")
        m = np.zeros((self.batch, self.nx * self.ny), np.uint8) if constrained else None
        _raise(self.lib, self.lib.sc_rollout(self.h, _ptr(x0), _ptr(v0), int(steps), int(k0),
                                             MODES[mode], _ptr(xo), _ptr(vo), _ptr(m)))
        return (xo, vo, m) if constrained else (xo, vo)

    def rollout_frames(self, x0, v0, steps: int, stride: int = 1, mode: str = "parity",
                       out=None):
        """Frames 0, stride, 2*stride, ... as [frames][batch][node][3] arrays. ``out`` = (fx, fv)
        writes into caller arrays; page-locked ones (pinned_empty) take the D2H copies directly,
        pageable ones go through the context's two pinned staging slots (overlapped)."""
        x0, v0 = self._arr(x0), self._arr(v0)
        nf = steps // stride + 1
        shape = (nf,) + (self.batch, self.local_rows * self.nx, 3)
        if out is None:
            fx = np.empty(shape, self.dtype)
            fv = np.empty_like(fx)
        else:
            fx, fv = out
            for a in (fx, fv):
                if a.shape != shape or a.dtype != self.dtype or not a.flags.c_contiguous:
                    raise ConfigError("frames: out arrays must be C-contiguous %s %s"
                                      % (self.dtype.__name__, shape))
        _raise(self.lib, self.lib.sc_rollout_frames(self.h, _ptr(x0), _ptr(v0), int(steps),
                                                    int(stride), MODES[mode], _ptr(fx), _ptr(fv)))
        return fx, fv

    def forward_impulse(self, x, v) -> np.ndarray:
        x, v = self._arr(x), self._arr(v)
        out = self._empty()
        _raise(self.lib, self.lib.sc_forward_impulse(self.h, _ptr(x), _ptr(v), _ptr(out)))
        return out

    def plug_impulse(self, x, v) -> np.ndarray:
        x, v = self._arr(x), self._arr(v)
        out = self._empty()
        _raise(self.lib, self.lib.sc_plug_impulse(self.h, _ptr(x), _ptr(v), _ptr(out)))
        return out

    def advance_with_impulse(self, x, v, impulse, t_next: float, constrained: bool = False):
        x, v, imp = self._arr(x), self._arr(v), self._arr(impulse)
        xo, vo = self._empty(), self._empty()
        m = np.zeros((self.batch, self.nx * self.ny), np.uint8) if constrained else None
        _raise(self.lib, self.lib.sc_advance_with_impulse(self.h, _ptr(x), _ptr(v), _ptr(imp),
                                                          float(t_next), _ptr(xo), _ptr(vo),
                                                          _ptr(m)))
        return (xo, vo, m) if constrained else (xo, vo)

    def nn_step(self, x, v, t_next: float, mode: str = "parity", constrained: bool = False):
        x, v = self._arr(x), self._arr(v)
        xo, vo = self._empty(), self._empty()
        m = np.zeros((self.batch, self.nx * self.ny), np.uint8) if constrained else None
        _raise(self.lib, self.lib.sc_nn_step(self.h, _ptr(x), _ptr(v), float(t_next),
                                             MODES[mode], _ptr(xo), _ptr(vo), _ptr(m)))
        return (xo, vo, m) if constrained else (xo, vo)

    # -- ground-truth mass-spring step (PBS) --
    def total_impulse(self, x, v) -> np.ndarray:
        x, v = self._arr(x), self._arr(v)
        out = self._empty()
        _raise(self.lib, self.lib.sc_total_impulse(self.h, _ptr(x), _ptr(v), _ptr(out)))
        return out

    def total_force(self, x, v) -> np.ndarray:
        x, v = self._arr(x), self._arr(v)
        out = self._empty()
        _raise(self.lib, self.lib.sc_total_force(self.h, _ptr(x), _ptr(v), _ptr(out)))
        return out

    def pbs_step(self, x, v, t_next: float, constrained: bool = False):
        x, v = self._arr(x), self._arr(v)
        xo, vo = self._empty(), self._empty()
        m = np.zeros((self.batch, self.nx * self.ny), np.uint8) if constrained else None
        _raise(self.lib, self.lib.sc_pbs_step(self.h, _ptr(x), _ptr(v), float(t_next), _ptr(xo),
                                              _ptr(vo), _ptr(m)))
        return (xo, vo, m) if constrained else (xo, vo)

    def simulate_frames(self, x0, v0, steps: int, stride: int = 1):
        x0, v0 = self._arr(x0), self._arr(v0)
        nf = steps // stride + 1
        fx = np.empty((nf,) + (self.batch, self.local_rows * self.nx, 3), self.dtype)
        fv = np.empty_like(fx)
        _raise(self.lib, self.lib.sc_simulate_frames(self.h, _ptr(x0), _ptr(v0), int(steps),
                                                     int(stride), _ptr(fx), _ptr(fv)))
        return fx, fv

    def benchmark_sim(self, steps: int, warmup: int) -> float:
        sec = C.c_double()
        _raise(self.lib, self.lib.sc_benchmark_sim(self.h, int(steps), int(warmup), C.byref(sec)))
        return sec.value

    def benchmark(self, steps: int, warmup: int, mode: str = "parity") -> float:
        sec = C.c_double()
        _raise(self.lib, self.lib.sc_benchmark(self.h, int(steps), int(warmup), MODES[mode],
                                               C.byref(sec)))
        return sec.value

    def benchmark_launches(self, steps: int, k0: int = 0, mode: str = "fast") -> np.ndarray:
        ms = np.zeros(int(steps), np.float32)
        _raise(self.lib, self.lib.sc_benchmark_launches(self.h, int(steps), int(k0), MODES[mode],
                                                        _ptr(ms)))
        return ms

    def launch_count(self) -> int:
        return int(self.lib.sc_ctx_launch_count(self.h))

    # -- strip decomposition helpers --
    def halo_elems(self) -> int:
        return int(self.lib.sc_ctx_halo_elems(self.h))

    def halo_pack(self, side: int, dev_ptr: int, stream: Optional[int] = None) -> None:
        _raise(self.lib, self.lib.sc_ctx_halo_pack(self.h, side, C.c_void_p(dev_ptr),
                                                   C.c_void_p(stream) if stream else None))

    def halo_unpack(self, side: int, dev_ptr: int, stream: Optional[int] = None) -> None:
        _raise(self.lib, self.lib.sc_ctx_halo_unpack(self.h, side, C.c_void_p(dev_ptr),
                                                     C.c_void_p(stream) if stream else None))

    def strip_step(self, k: int, r_begin: int, r_end: int, mode: str = "fast",
                   stream: Optional[int] = None) -> None:
        _raise(self.lib, self.lib.sc_ctx_strip_step(self.h, int(k), int(r_begin), int(r_end),
                                                    MODES[mode],
                                                    C.c_void_p(stream) if stream else None))

    def peer_export(self) -> bytes:
        """This strip context's IPC handles / pointers (sc_ctx_peer_export) as bytes."""
        e = _abi.sc_peer_export()
        _raise(self.lib, self.lib.sc_ctx_peer_export(self.h, C.byref(e)))
        return bytes(e)

    def set_peer(self, side: int, export: bytes, ipc: bool = True) -> None:
        """Link the neighbour strip on `side` (0: below, 1: above) from its peer_export()."""
        e = _abi.sc_peer_export.from_buffer_copy(export)
        _raise(self.lib, self.lib.sc_ctx_set_peer(self.h, int(side), C.byref(e), 1 if ipc else 0))

    def peer_step(self, k: int, mode: str = "fast", stream: Optional[int] = None) -> None:
        """One fused step: boundary rows stored straight into the linked neighbours' ghost rows."""
        _raise(self.lib, self.lib.sc_ctx_peer_step(self.h, int(k), MODES[mode],
                                                   C.c_void_p(stream) if stream else None))

    def strip_commit(self) -> None:
        _raise(self.lib, self.lib.sc_ctx_strip_commit(self.h))

    def stream(self) -> int:
        return int(self.lib.sc_ctx_stream(self.h) or 0)


# ---------------------------------------------------------------- reference-style API ----

class _PinnedBlock:
    def __init__(self, nbytes: int):
        self.lib = _abi.load()
        p = C.c_void_p()
        _raise(self.lib, self.lib.sc_host_alloc(max(1, nbytes), C.byref(p)))
        self.ptr = p.value

    def __del__(self):
        if getattr(self, "ptr", None):
            self.lib.sc_host_free(C.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """Uninitialised page-locked (cudaHostAlloc) numpy array; the block is freed with the array.
    Frame and state transfers into such arrays are direct DMA, no staging copy."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    blk = _PinnedBlock(n)
    buf = (C.c_char * max(1, n)).from_address(blk.ptr)
    buf._owner = blk  # keep the allocation alive as long as any view of it
    return np.frombuffer(buf, dt, count=int(np.prod(shape))).reshape(shape)


def _state2(a, n: int, name: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ConfigError(name + ": expected an (n, 3) array")
    return a


def _check_shape(x, v, scene: Scene):
    if x.shape[0] != v.shape[0]:
        raise ConfigError("positions and velocities disagree on the node count")
    if x.shape[0] != scene.node_count:
        raise ConfigError("state shape does not match the grid topology")


def _check_alpha(params: NetworkParams):
    if not params.isru_alpha > 0.0:
        raise ConfigError("isru_alpha: must be > 0")


def _diagnose_forward(x, v, scene: Scene, p: NetworkParams, node: int) -> str:
    """Names the branch with a non-finite value at one node, like diagnose_forward
    (net.cpp:30-51). Failure path only: formats the error message."""
    nx, ny = scene.nx, scene.ny
    ix, iy = node % nx, node // nx
    with np.errstate(all="ignore"):
        lin = np.array(p.linear_b, dtype=np.float64)
        non = np.zeros(3)
        der = v[node] * p.self_velocity_w
        for c, (dx, dy, _) in enumerate(STENCIL_OFFSETS):
            jx, jy = ix + dx, iy + dy
            if not (0 <= jx < nx and 0 <= jy < ny):
                continue
            j = jy * nx + jx
            phi = (x[node] - x[j]) * p.kernel_gain[c]
            xi = (v[node] - v[j]) * p.kernel_gain[c]
            s = phi / np.sqrt(1.0 + p.isru_alpha * phi * phi)
            lin = lin + phi * p.linear_w[c]
            non = non + s * p.nonlinear_w[c]
            der = der + xi * s * p.deriv_w[c]
    branch = ("linear" if not np.all(np.isfinite(lin)) else
              "nonlinear" if not np.all(np.isfinite(non)) else "derivative")
    return "network impulse non-finite at node %d (%s branch)" % (node, branch)


def forward_impulse(params: NetworkParams, scene: Scene, positions, velocities,
                    device: int = 0) -> np.ndarray:
    """Per-node impulse of the three-branch cell, float64 (net.cpp:132-142)."""
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    _check_alpha(params)
    with Context(scene, params, "f64", device) as ctx:
        out = ctx.forward_impulse(x, v)[0]
        fi, fn, _ = ctx.health()
    if fi[0] >= 0:
        raise NumericsError(_diagnose_forward(x, v, scene, params, int(fn[0])))
    return out


def plug_impulse(scene: Scene, positions, velocities, device: int = 0) -> np.ndarray:
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    with Context(scene, None, "f64", device) as ctx:
        return ctx.plug_impulse(x, v)[0]


def advance_with_impulse(scene: Scene, positions, velocities, impulse, t_next: float,
                         constrained: bool = False, device: int = 0):
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    imp = _state2(impulse, 0, "impulse")
    _check_shape(x, v, scene)
    if imp.shape != x.shape:
        raise ConfigError("impulse field shape does not match the state")
    with Context(scene, None, "f64", device) as ctx:
        r = ctx.advance_with_impulse(x, v, imp, t_next, constrained)
    if constrained:
        return r[0][0], r[1][0], r[2][0]
    return r[0][0], r[1][0]


def nn_step(params: NetworkParams, scene: Scene, positions, velocities, t_next: float,
            device: int = 0):
    """One network step to the frame at t_next (net.cpp:242-248); returns (x, v)."""
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    _check_alpha(params)
    with Context(scene, params, "f64", device) as ctx:
        xo, vo = ctx.nn_step(x, v, t_next)
        fi, fn, _ = ctx.health()
    if fi[0] >= 0:
        raise NumericsError(_diagnose_forward(x, v, scene, params, int(fn[0])))
    return xo[0], vo[0]


def apply_dirichlet(x: np.ndarray, v: np.ndarray, scene: Scene, t: float):
    """Pins to the anchor path at time t (sim.cpp:108-117)."""
    x, v = x.copy(), v.copy()
    u = scene.bc.pin_velocity()
    for k, i in enumerate(scene.bc.nodes):
        x[i] = scene.bc.anchor_at(k, t)
        v[i] = u
    return x, v


def rollout(params: NetworkParams, scene: Scene, steps: int = -1, device: int = 0) -> Trajectory:
    """Closed-loop rollout storing every frame (eval.cpp:86-103), bit-identical to the
    reference's double-precision rollout."""
    scene.validate()
    _check_alpha(params)
    if steps < 0:
        steps = scene.steps
    x0, v0 = apply_dirichlet(scene.initial_x, scene.initial_v, scene, 0.0)
    with Context(scene, params, "f64", device) as ctx:
        fx, fv = ctx.rollout_frames(x0, v0, steps, 1, "parity")
        fi, fn, fs = ctx.health()
    bad_imp, bad_state = int(fi[0]), int(fs[0])
    if bad_imp >= 0 and (bad_state < 0 or bad_imp <= bad_state):
        k = bad_imp - 1
        raise NumericsError(_diagnose_forward(fx[k, 0], fv[k, 0], scene, params, int(fn[0])))
    if bad_state >= 0:
        raise NumericsError("rollout diverged: non-finite state at frame %d" % bad_state)
    return Trajectory(scene.nx, scene.ny, scene.dt, scene.spacing, fx[:, 0], fv[:, 0])


@dataclass
class BenchResult:
    """eval.hpp:38-44."""
    steps: int
    warmup: int
    precision: str
    seconds: float
    steps_per_second: float


def benchmark_net(params: NetworkParams, scene: Scene, steps: int, warmup: int,
                  precision: str = "f32", mode: str = "parity", device: int = 0) -> BenchResult:
    """Device-timed run_steps loop (eval.cpp:69-82,155-158) from the scene's initial state."""
    scene.validate()
    if steps < 1:
        raise ConfigError("bench: steps must be >= 1")
    if warmup < 0:
        raise ConfigError("bench: warmup must be >= 0")
    with Context(scene, params, precision, device) as ctx:
        ctx.set_state(scene.initial_x, scene.initial_v)
        sec = ctx.benchmark(steps, warmup, mode)
    return BenchResult(steps, warmup, precision, sec, steps / max(sec, 1e-12))


# ---------------------------------------------- ground-truth mass-spring step (PBS, §8 f2) ----

def _force_terms(x: np.ndarray, v: np.ndarray, scene: Scene):
    """The four force terms of total_force (sim.cpp:77-88) in float64, vectorised; used only on
    the failure path to name the term that went non-finite (diagnose_divergence, sim.cpp:23-48)."""
    nx, ny = scene.nx, scene.ny
    m = scene.material
    X = x.reshape(ny, nx, 3)
    Vv = v.reshape(ny, nx, 3)
    el = np.zeros_like(X)
    da = np.zeros_like(X)
    with np.errstate(all="ignore"):
        for dx, dy, mult in STENCIL_OFFSETS:
            rest = scene.spacing * mult
            ys = slice(max(0, -dy), ny - max(0, dy))
            xs = slice(max(0, -dx), nx - max(0, dx))
            yj = slice(max(0, dy), ny + min(0, dy))
            xj = slice(max(0, dx), nx + min(0, dx))
            d = X[ys, xs] - X[yj, xj]
            ln = np.sqrt((d * d).sum(-1, keepdims=True))
            el[ys, xs] -= d * (m.stiffness * (ln - rest) / ln)
            dr = d / ln
            da[ys, xs] -= dr * (m.damping * ((Vv[ys, xs] - Vv[yj, xj]) * dr).sum(-1, keepdims=True))
        pr = np.zeros_like(X)
        if m.pressure != 0.0:
            c = X[1:-1, 1:-1]
            e, n = c - X[1:-1, 2:], c - X[2:, 1:-1]
            w, s = c - X[1:-1, :-2], c - X[:-2, 1:-1]
            pr[1:-1, 1:-1] = (np.cross(e, n) + np.cross(n, w) + np.cross(w, s) + np.cross(s, e)) * m.pressure
        ex = m.gravity * m.mass - Vv * m.drag
    return [(name, t.reshape(-1, 3)) for name, t in
            (("elastic", el), ("damping", da), ("pressure", pr), ("external", ex))]


def _diagnose_divergence(x, v, scene: Scene) -> str:
    for name, f in _force_terms(x, v, scene):
        bad = np.where(~np.isfinite(f).all(axis=1))[0]
        if len(bad):
            return "%s force non-finite at node %d (reduce dt or stiffness)" % (name, bad[0])
    return "non-finite state update (reduce dt or stiffness)"


def total_impulse(scene: Scene, positions, velocities, device: int = 0) -> np.ndarray:
    """Total force scaled by dt/m (sim.cpp:90-98), float64, bit-identical to the reference."""
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    with Context(scene, None, "f64", device) as ctx:
        return ctx.total_impulse(x, v)[0]


def total_force(scene: Scene, positions, velocities, device: int = 0) -> np.ndarray:
    """Sum of the elastic, damping, pressure and external forces (sim.cpp:84-96; binding
    total_force, bindings.cpp:156-161), float64, bit-identical to the reference."""
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    with Context(scene, None, "f64", device) as ctx:
        return ctx.total_force(x, v)[0]


def step_semi_implicit(scene: Scene, positions, velocities, t_next: float, device: int = 0):
    """One ground-truth step to the frame at t_next (sim.cpp:150-155); returns (x, v)."""
    x, v = _state2(positions, 0, "positions"), _state2(velocities, 0, "velocities")
    _check_shape(x, v, scene)
    with Context(scene, None, "f64", device) as ctx:
        try:
            xo, vo = ctx.pbs_step(x, v, t_next)
        except NumericsError as e:
            if "singular" in str(e):
                raise
            raise NumericsError(_diagnose_divergence(x, v, scene)) from None
    return xo[0], vo[0]


def simulate(scene: Scene, device: int = 0) -> Trajectory:
    """simulate_scene (sim.cpp:157-175): scene.steps ground-truth steps from the pinned initial
    state, every frame stored; bit-identical to the reference, including its error text."""
    scene.validate()
    x0, v0 = apply_dirichlet(scene.initial_x, scene.initial_v, scene, 0.0)
    with Context(scene, None, "f64", device) as ctx:
        fx, fv = ctx.simulate_frames(x0, v0, scene.steps, 1)
        fs, fn, fstate = ctx.health()
    sing, state = int(fs[0]), int(fstate[0])
    if sing >= 0 and (state < 0 or sing <= state):
        raise NumericsError("simulation diverged at frame %d: elastic force: singular spring "
                            "(coincident nodes) at node %d" % (sing, int(fn[0])))
    if state >= 0:
        raise NumericsError("simulation diverged at frame %d: %s" % (
            state, _diagnose_divergence(fx[state - 1, 0], fv[state - 1, 0], scene)))
    return Trajectory(scene.nx, scene.ny, scene.dt, scene.spacing, fx[:, 0], fv[:, 0])


def benchmark_sim(scene: Scene, steps: int, warmup: int, precision: str = "f32",
                  device: int = 0) -> BenchResult:
    """Device-timed ground-truth stepping (benchmark_sim, eval.cpp:151-153)."""
    scene.validate()
    if steps < 1:
        raise ConfigError("bench: steps must be >= 1")
    if warmup < 0:
        raise ConfigError("bench: warmup must be >= 0")
    with Context(scene, None, precision, device) as ctx:
        ctx.set_state(scene.initial_x, scene.initial_v)
        sec = ctx.benchmark_sim(steps, warmup)
    return BenchResult(steps, warmup, precision, sec, steps / max(sec, 1e-12))


class ClothBatch(Context):
    """Batched device-resident engine: B same-size cloths stepped together (f32 by default)."""

    def __init__(self, scenes: Sequence[Scene], params: NetworkParams, precision: str = "f32",
                 device: int = 0, strip: Optional[tuple] = None):
        super().__init__(scenes, params, precision, device, strip)

    def rollout_trajectories(self, steps: int, stride: int = 1, mode: str = "fast",
                             pinned: bool = True) -> List[Trajectory]:
        """Batched closed-loop rollout from every scene's pinned initial state (the batched form of
        rollout, eval.cpp:86-103), one Trajectory per cloth holding frames 0, stride, 2*stride,
        ... . Frame output streams off the device behind the stepping (§8(f3)); f32 frames are
        widened to the Trajectory's double fields like read_trajectory does for CLT1 v2 files."""
        x0 = np.stack([apply_dirichlet(s.initial_x, s.initial_v, s, 0.0)[0] for s in self.scenes])
        v0 = np.stack([apply_dirichlet(s.initial_x, s.initial_v, s, 0.0)[1] for s in self.scenes])
        nf = steps // stride + 1
        shape = (nf, self.batch, self.local_rows * self.nx, 3)
        out = (pinned_empty(shape, self.dtype), pinned_empty(shape, self.dtype)) if pinned else None
        fx, fv = self.rollout_frames(x0, v0, steps, stride, mode, out=out)
        return [Trajectory(self.nx, self.ny, s.dt * stride, s.spacing,
                           fx[:, b].astype(np.float64), fv[:, b].astype(np.float64))
                for b, s in enumerate(self.scenes)]
