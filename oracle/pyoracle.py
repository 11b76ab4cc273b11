"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU checkers.

  liboracle.so                 plain-C restatement of the path (oracle/oracle.c)
  _ref/libstencilcloth_ref.so  the UNMODIFIED reference sources compiled by oracle/Makefile,
                               driven through oracle/ref_harness.cpp

Importable only from tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs. Nothing in the product package imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np


def _load_abi_types():
    """The C-ABI struct layouts (paper_2403_12820_b200/_abi.py) loaded as a standalone module:
    importing the package would load libstencilcloth_b200.so, and the checker side (tests'
    oracle, bench.py's reference arm) must run without the product library."""
    import importlib.util
    import sys
    # registered under its package name, so a later `import paper_2403_12820_b200` reuses this
    # very module (one set of ctypes classes for both sides)
    name = "paper_2403_12820_b200._abi"
    if name in sys.modules:
        return sys.modules[name]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2403_12820_b200", "_abi.py")
    spec = importlib.util.spec_from_file_location(name, path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


_abi = _load_abi_types()

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstencilcloth_ref.so")

_P = C.c_void_p
_I = C.c_int
_CD = C.POINTER(_abi.sc_cloth_desc)
_PR = C.POINTER(_abi.sc_params)


def build(quiet: bool = True) -> None:
    """make -C oracle (liboracle.so always; _ref only where /root/reference exists)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    """The C restatement, at float or double."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.lib = C.CDLL(ORACLE_SO)
        for sfx, T in (("f32", C.c_float), ("f64", C.c_double)):
            getattr(self.lib, "orc_forward_impulse_" + sfx).argtypes = [_I, _I, _PR, _P, _P, _P]
            getattr(self.lib, "orc_plug_impulse_" + sfx).argtypes = [_I, _I, _CD, _P, _P, _P]
            getattr(self.lib, "orc_advance_with_impulse_" + sfx).argtypes = [
                _I, _I, _CD, _P, _P, _P, T, _P, _P, _P]
            getattr(self.lib, "orc_nn_step_" + sfx).argtypes = [
                _I, _I, _CD, _PR, _P, _P, T, _P, _P, _P, _P]
            getattr(self.lib, "orc_rollout_" + sfx).argtypes = [
                _I, _I, _I, _CD, _PR, _P, _P, _I, _I, _P]
            for fn in ("orc_forward_impulse_", "orc_plug_impulse_", "orc_advance_with_impulse_",
                       "orc_nn_step_", "orc_rollout_"):
                getattr(self.lib, fn + sfx).restype = None
            getattr(self.lib, "orc_total_impulse_" + sfx).argtypes = [_I, _I, _CD, _P, _P, _P]
            getattr(self.lib, "orc_total_impulse_" + sfx).restype = C.c_long
            getattr(self.lib, "orc_pbs_step_" + sfx).argtypes = [_I, _I, _CD, _P, _P, T, _P, _P, _P]
            getattr(self.lib, "orc_pbs_step_" + sfx).restype = C.c_long

    @staticmethod
    def _dt(a):
        return "f32" if a.dtype == np.float32 else "f64"

    def forward_impulse(self, nx, ny, params, x, v):
        out = np.empty_like(x)
        getattr(self.lib, "orc_forward_impulse_" + self._dt(x))(nx, ny, C.byref(params), _p(x),
                                                                _p(v), _p(out))
        return out

    def plug_impulse(self, nx, ny, cloth, x, v):
        out = np.empty_like(x)
        getattr(self.lib, "orc_plug_impulse_" + self._dt(x))(nx, ny, C.byref(cloth), _p(x), _p(v),
                                                             _p(out))
        return out

    def advance_with_impulse(self, nx, ny, cloth, x, v, imp, t_next):
        xo, vo = np.empty_like(x), np.empty_like(v)
        m = np.zeros(nx * ny, np.uint8)
        getattr(self.lib, "orc_advance_with_impulse_" + self._dt(x))(
            nx, ny, C.byref(cloth), _p(x), _p(v), _p(imp), t_next, _p(xo), _p(vo), _p(m))
        return xo, vo, m

    def nn_step(self, nx, ny, cloth, params, x, v, t_next):
        xo, vo, imp = np.empty_like(x), np.empty_like(v), np.empty_like(x)
        m = np.zeros(nx * ny, np.uint8)
        getattr(self.lib, "orc_nn_step_" + self._dt(x))(
            nx, ny, C.byref(cloth), C.byref(params), _p(x), _p(v), t_next, _p(xo), _p(vo), _p(m),
            _p(imp))
        return xo, vo, m, imp

    def total_impulse(self, nx, ny, cloth, x, v):
        """(impulse, first singular node or -1)."""
        out = np.empty_like(x)
        sing = getattr(self.lib, "orc_total_impulse_" + self._dt(x))(nx, ny, C.byref(cloth), _p(x),
                                                                     _p(v), _p(out))
        return out, int(sing)

    def pbs_step(self, nx, ny, cloth, x, v, t_next):
        """step_semi_implicit: (x', v', mask, first singular node or -1)."""
        xo, vo = np.empty_like(x), np.empty_like(v)
        m = np.zeros(nx * ny, np.uint8)
        sing = getattr(self.lib, "orc_pbs_step_" + self._dt(x))(nx, ny, C.byref(cloth), _p(x),
                                                                _p(v), t_next, _p(xo), _p(vo),
                                                                _p(m))
        return xo, vo, m, int(sing)

    def rollout(self, nx, ny, cloths, params, x, v, steps, k0=0):
        """run_steps<T> sequence over a batch; returns (x, v, last-step mask)."""
        x, v = np.array(x, copy=True), np.array(v, copy=True)
        batch = len(cloths)
        arr = (_abi.sc_cloth_desc * batch)(*cloths)
        m = np.zeros((batch, nx * ny), np.uint8)
        getattr(self.lib, "orc_rollout_" + self._dt(x))(
            nx, ny, batch, C.cast(arr, _CD), C.byref(params), _p(x), _p(v), steps, k0, _p(m))
        return x, v, m


class Reference:
    """The reference's own code (oracle/_ref), through oracle/ref_harness.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build it with `make -C oracle ref` where "
                                    "/root/reference exists)")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [_I]
        L.ref_rollout_f32.argtypes = [_I, _I, _I, _CD, _PR, _P, _P, _I, _I, _P]
        L.ref_rollout_tmpl_f64.argtypes = [_I, _I, _I, _CD, _PR, _P, _P, _I, _I, _P]
        L.ref_step_f32.argtypes = [_I, _I, _CD, _PR, _P, _P, C.c_float, _P, _P, _P, _P]
        L.ref_forward_impulse_f64.argtypes = [_I, _I, _PR, _P, _P, _P]
        L.ref_plug_impulse_f64.argtypes = [_I, _I, _CD, _P, _P, _P]
        L.ref_advance_with_impulse_f64.argtypes = [_I, _I, _CD, _P, _P, _P, C.c_double, _P, _P,
                                                   _P]
        L.ref_nn_step_f64.argtypes = [_I, _I, _CD, _PR, _P, _P, C.c_double, _P, _P]
        L.ref_rollout_f64.argtypes = [_I, _I, _CD, _PR, _P, _P, _I, _P, _P]
        L.ref_benchmark_net.argtypes = [_I, _I, _CD, _PR, _P, _P, _I, _I, _I, _I,
                                        C.POINTER(C.c_double)]
        L.ref_total_impulse_f64.argtypes = [_I, _I, _CD, _P, _P, _P]
        L.ref_pbs_step_f64.argtypes = [_I, _I, _CD, _P, _P, C.c_double, _P, _P]
        L.ref_simulate_f64.argtypes = [_I, _I, _CD, _P, _P, _I, _P, _P]
        L.ref_pbs_rollout_f32.argtypes = [_I, _I, _CD, _P, _P, _I, _I]
        L.ref_benchmark_sim.argtypes = [_I, _I, _CD, _P, _P, _I, _I, _I, _I, C.POINTER(C.c_double)]
        L.ref_benchmark_net_cloth_parallel.argtypes = [_I, _I, _I, _CD, _PR, _P, _P, _I, _I,
                                                       C.POINTER(C.c_double),
                                                       C.POINTER(C.c_double)]
        _TC = C.POINTER(_abi.sc_train_config)
        L.ref_sample_batch.argtypes = [_I, _I, _CD, _I, _P, _P, _I, C.c_uint64, _P, _P]
        L.ref_compute_loss.argtypes = [_I, _I, _CD, _I, _P, _P, _I, C.c_uint64, _PR, C.c_double,
                                       _I, _P, _P]
        L.ref_backward_gradients.argtypes = [_I, _I, _P, _P, _PR, _P, _P]
        L.ref_train.argtypes = [_I, _I, _CD, _I, _P, _P, _TC, _PR, _P, _P, _P]

    def _ck(self, rc):
        if rc != 0:
            msg = (self.lib.ref_last_error() or b"").decode()
            if rc == 1:
                raise ValueError(msg)
            if rc == 2:
                raise ArithmeticError(msg)
            raise RuntimeError(msg)

    def rollout_f32(self, nx, ny, cloths, params, x, v, steps, k0=0):
        x = np.ascontiguousarray(x, np.float32).copy()
        v = np.ascontiguousarray(v, np.float32).copy()
        batch = len(cloths)
        arr = (_abi.sc_cloth_desc * batch)(*cloths)
        m = np.zeros((batch, nx * ny), np.uint8)
        self._ck(self.lib.ref_rollout_f32(nx, ny, batch, C.cast(arr, _CD), C.byref(params), _p(x),
                                          _p(v), steps, k0, _p(m)))
        return x, v, m

    def rollout_tmpl_f64(self, nx, ny, cloths, params, x, v, steps, k0=0):
        x = np.ascontiguousarray(x, np.float64).copy()
        v = np.ascontiguousarray(v, np.float64).copy()
        batch = len(cloths)
        arr = (_abi.sc_cloth_desc * batch)(*cloths)
        m = np.zeros((batch, nx * ny), np.uint8)
        self._ck(self.lib.ref_rollout_tmpl_f64(nx, ny, batch, C.cast(arr, _CD), C.byref(params),
                                               _p(x), _p(v), steps, k0, _p(m)))
        return x, v, m

    def step_f32(self, nx, ny, cloth, params, x, v, t_next):
        xo, vo, imp = (np.empty_like(x) for _ in range(3))
        m = np.zeros(nx * ny, np.uint8)
        self._ck(self.lib.ref_step_f32(nx, ny, C.byref(cloth), C.byref(params), _p(x), _p(v),
                                       t_next, _p(xo), _p(vo), _p(m), _p(imp)))
        return xo, vo, m, imp

    def forward_impulse_f64(self, nx, ny, params, x, v):
        out = np.empty_like(x)
        self._ck(self.lib.ref_forward_impulse_f64(nx, ny, C.byref(params), _p(x), _p(v), _p(out)))
        return out

    def plug_impulse_f64(self, nx, ny, cloth, x, v):
        out = np.empty_like(x)
        self._ck(self.lib.ref_plug_impulse_f64(nx, ny, C.byref(cloth), _p(x), _p(v), _p(out)))
        return out

    def advance_with_impulse_f64(self, nx, ny, cloth, x, v, imp, t_next):
        xo, vo = np.empty_like(x), np.empty_like(v)
        m = np.zeros(nx * ny, np.uint8)
        self._ck(self.lib.ref_advance_with_impulse_f64(nx, ny, C.byref(cloth), _p(x), _p(v),
                                                       _p(imp), t_next, _p(xo), _p(vo), _p(m)))
        return xo, vo, m

    def nn_step_f64(self, nx, ny, cloth, params, x, v, t_next):
        xo, vo = np.empty_like(x), np.empty_like(v)
        self._ck(self.lib.ref_nn_step_f64(nx, ny, C.byref(cloth), C.byref(params), _p(x), _p(v),
                                          t_next, _p(xo), _p(vo)))
        return xo, vo

    def rollout_f64(self, nx, ny, cloth, params, x0, v0, steps):
        n = nx * ny
        fx = np.empty((steps + 1, n, 3))
        fv = np.empty_like(fx)
        self._ck(self.lib.ref_rollout_f64(nx, ny, C.byref(cloth), C.byref(params), _p(x0), _p(v0),
                                          steps, _p(fx), _p(fv)))
        return fx, fv

    def total_impulse_f64(self, nx, ny, cloth, x, v):
        out = np.empty_like(x)
        self._ck(self.lib.ref_total_impulse_f64(nx, ny, C.byref(cloth), _p(x), _p(v), _p(out)))
        return out

    def pbs_step_f64(self, nx, ny, cloth, x, v, t_next):
        xo, vo = np.empty_like(x), np.empty_like(v)
        self._ck(self.lib.ref_pbs_step_f64(nx, ny, C.byref(cloth), _p(x), _p(v), t_next, _p(xo),
                                           _p(vo)))
        return xo, vo

    def simulate_f64(self, nx, ny, cloth, x0, v0, steps):
        n = nx * ny
        fx = np.empty((steps + 1, n, 3))
        fv = np.empty_like(fx)
        self._ck(self.lib.ref_simulate_f64(nx, ny, C.byref(cloth), _p(x0), _p(v0), steps, _p(fx),
                                           _p(fv)))
        return fx, fv

    def pbs_rollout_f32(self, nx, ny, cloth, x, v, steps, k0=0):
        x = np.ascontiguousarray(x, np.float32).copy()
        v = np.ascontiguousarray(v, np.float32).copy()
        self._ck(self.lib.ref_pbs_rollout_f32(nx, ny, C.byref(cloth), _p(x), _p(v), steps, k0))
        return x, v

    def benchmark_sim(self, nx, ny, cloth, x0, v0, steps, warmup, f64=False, threads=1):
        sec = C.c_double()
        self._ck(self.lib.ref_benchmark_sim(nx, ny, C.byref(cloth), _p(x0), _p(v0), steps, warmup,
                                            int(f64), threads, C.byref(sec)))
        return sec.value

    def benchmark_net(self, nx, ny, cloth, params, x0, v0, steps, warmup, f64=False, threads=1):
        sec = C.c_double()
        self._ck(self.lib.ref_benchmark_net(nx, ny, C.byref(cloth), C.byref(params), _p(x0),
                                            _p(v0), steps, warmup, int(f64), threads,
                                            C.byref(sec)))
        return sec.value

    def benchmark_net_cloth_parallel(self, nx, ny, cloths, params, x0, v0, steps, warmup):
        batch = len(cloths)
        arr = (_abi.sc_cloth_desc * batch)(*cloths)
        mx, wall = C.c_double(), C.c_double()
        self._ck(self.lib.ref_benchmark_net_cloth_parallel(
            nx, ny, batch, C.cast(arr, _CD), C.byref(params), _p(x0), _p(v0), steps, warmup,
            C.byref(mx), C.byref(wall)))
        return mx.value, wall.value

    # ---- training (train.cpp / net.cpp:144-201) -------------------------------------------
    def sample_batch(self, nx, ny, cloth, fx, fv, batch_size, seed):
        fx = np.ascontiguousarray(fx, np.float64)
        fv = np.ascontiguousarray(fv, np.float64)
        idx = np.empty(batch_size, np.int32)
        tgt = np.empty((batch_size, nx * ny, 3))
        self._ck(self.lib.ref_sample_batch(nx, ny, C.byref(cloth), fx.shape[0], _p(fx), _p(fv),
                                           batch_size, seed, _p(idx), _p(tgt)))
        return idx, tgt

    def compute_loss(self, nx, ny, cloth, fx, fv, batch_size, seed, params, alpha, grads=True):
        fx = np.ascontiguousarray(fx, np.float64)
        fv = np.ascontiguousarray(fv, np.float64)
        loss = np.empty(3)
        g = np.empty(53)
        self._ck(self.lib.ref_compute_loss(nx, ny, C.byref(cloth), fx.shape[0], _p(fx), _p(fv),
                                           batch_size, seed, C.byref(params), alpha, int(grads),
                                           _p(loss), _p(g)))
        return loss, (g if grads else None)

    def backward_gradients(self, nx, ny, x, v, params, upstream):
        g = np.empty(53)
        self._ck(self.lib.ref_backward_gradients(
            nx, ny, _p(np.ascontiguousarray(x, np.float64)), _p(np.ascontiguousarray(v, np.float64)),
            C.byref(params), _p(np.ascontiguousarray(upstream, np.float64)), _p(g)))
        return g

    def train(self, nx, ny, cloth, fx, fv, cfg):
        fx = np.ascontiguousarray(fx, np.float64)
        fv = np.ascontiguousarray(fv, np.float64)
        out = _abi.sc_params()
        tr = np.zeros(7, np.uint8)
        hist = np.zeros((cfg.epochs, 5))
        br = np.zeros(14)
        self._ck(self.lib.ref_train(nx, ny, C.byref(cloth), fx.shape[0], _p(fx), _p(fv),
                                    C.byref(cfg), C.byref(out), _p(tr), _p(hist), _p(br)))
        self.last_brackets = br
        return out, tr, hist
