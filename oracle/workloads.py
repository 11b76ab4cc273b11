"""TEST / BENCH INFRASTRUCTURE ONLY — the five BASELINE.json workloads built on the checker side.

bench.py's reference arm and cpu_baseline time the reference's own CPU code (oracle/_ref) on
these inputs; they must not load the product library, so this module rebuilds the workloads
from oracle/gen.c (a restatement of the reference's Rng, rng.hpp:13-47) with the repo's frozen
conventions. tests/test_workloads.py checks that the inputs are
identical, draw for draw and field for field, to paper_2403_12820_b200.configs.

The reference has no plane collider (spheres only, io.cpp:321-322): config 5's free-falling
class runs without its plane on the reference side (`plane=False` below), which is stated in
the bench line.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from .pyoracle import ORACLE_SO, _abi
from .pyoracle import build as _build_oracle

DT = 1.0 / 240.0


@dataclass(frozen=True)
class Workload:
    name: str
    n: int
    batch: int
    steps: int
    seed: int
    pins: str        # "corners" | "top_row" | "mixed"
    wind: bool
    sphere: bool
    hidden8: bool


WORKLOADS = {
    1: Workload("cfg1_32x32_b1", 32, 1, 100, 0, "corners", False, False, True),
    2: Workload("cfg2_256x256_b64", 256, 64, 1000, 1, "top_row", True, False, False),
    3: Workload("cfg3_1024x1024_sphere", 1024, 1, 500, 2, "corners", False, True, False),
    4: Workload("cfg4_8192x8192", 8192, 1, 200, 3, "top_row", False, False, False),
    5: Workload("cfg5_128x128_b4096_mixed", 128, 4096, 300, 4, "mixed", True, False, False),
}

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(ORACLE_SO):
            _build_oracle()
        lib = C.CDLL(ORACLE_SO)
        lib.orc_rng_mix.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_rng_mix.restype = C.c_uint64
        lib.orc_rng_uniform01.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        lib.orc_rng_normal.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_void_p]
        lib.orc_gen_sheet.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_double, C.c_double, C.c_void_p]
        for f in ("orc_rng_uniform01", "orc_rng_normal", "orc_gen_sheet"):
            getattr(lib, f).restype = None
        _LIB = lib
    return _LIB


def mix(seed: int, stream: int) -> int:
    return int(_lib().orc_rng_mix(seed, stream))


def uniforms(stream_seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    _lib().orc_rng_uniform01(stream_seed, count, out.ctypes.data_as(C.c_void_p))
    return out


def normals(stream_seed: int, count: int, sigma: float) -> np.ndarray:
    out = np.empty(count, np.float64)
    _lib().orc_rng_normal(stream_seed, count, sigma, out.ctypes.data_as(C.c_void_p))
    return out


def sheet(seed: int, cloth: int, n: int, row0: int = 0, rows: Optional[int] = None,
          sigma: float = 1e-3) -> np.ndarray:
    rows = n - row0 if rows is None else rows
    out = np.empty((rows * n, 3), np.float32)
    _lib().orc_gen_sheet(seed, cloth, n, row0, rows, 1.0 / (n - 1), sigma,
                         out.ctypes.data_as(C.c_void_p))
    return out


def params(w: Workload, sigma: float = 0.05) -> "_abi.sc_params":
    """The 40 trainable scalars ~ N(0, sigma) in for_each_scalar order (net.hpp:72-81),
    gains 1, alpha 1 (net.cpp:81-93); hidden8: skip channels 8..11 zeroed."""
    v = normals(mix(w.seed, 1), 40, sigma)
    p = _abi.sc_params()
    for c in range(12):
        keep = not (w.hidden8 and c >= 8)
        p.kernel_gain[c] = 1.0
        p.linear_w[c] = v[c] if keep else 0.0
        p.nonlinear_w[c] = v[15 + c] if keep else 0.0
        p.deriv_w[c] = v[27 + c] if keep else 0.0
    for d in range(3):
        p.linear_b[d] = v[12 + d]
    p.self_velocity_w = v[39]
    p.isru_alpha = 1.0
    return p


def wind(w: Workload, cloth: int) -> np.ndarray:
    u = uniforms(mix(w.seed, 2 + cloth), 3)
    z = 2.0 * u[0] - 1.0
    phi = 2.0 * math.pi * u[1]
    r = math.sqrt(max(0.0, 1.0 - z * z))
    return (2.0 * u[2]) * np.array([r * math.cos(phi), r * math.sin(phi), z])


def kind(w: Workload, b: int) -> str:
    return w.pins if w.pins != "mixed" else ("top_row", "corners", "free")[b % 3]


def pin_nodes(k: str, n: int) -> List[int]:
    if k == "top_row":
        return [(n - 1) * n + ix for ix in range(n)]
    if k == "corners":
        return [(n - 1) * n, (n - 1) * n + n - 1]
    return []


def cloth_desc(w: Workload, b: int, x0: np.ndarray, keep: list, plane: bool = True):
    """sc_cloth_desc of cloth b (x0: its f32 initial positions, AoS)."""
    n = w.n
    d = _abi.sc_cloth_desc()
    d.dt, d.mass, d.drag, d.pressure = DT, 1.0, 0.0, 0.0
    g = np.array([0.0, 0.0, -9.8]) + (wind(w, b) if w.wind else 0.0)
    for i in range(3):
        d.gravity[i] = float(g[i])
        d.pin_velocity[i] = 0.0
    d.plug_pressure, d.plug_gravity, d.plug_drag = 0, 1, 0
    nodes = np.asarray(pin_nodes(kind(w, b), n), np.int32)
    anchors = x0[nodes].astype(np.float64) if len(nodes) else np.zeros((0, 3))
    anchors = np.ascontiguousarray(anchors)
    sph = (_abi.sc_sphere * 1)()
    pl = (_abi.sc_plane * 1)()
    d.n_spheres = 0
    if w.sphere:
        u = uniforms(mix(w.seed, 0x20000 + b), 2)
        for i, c in enumerate((u[0], u[1], -0.35)):
            sph[0].center[i] = float(c)
        sph[0].radius, sph[0].friction = 0.3, 0.0
        d.n_spheres = 1
    d.n_planes = 0
    if plane and kind(w, b) == "free":
        pl[0].height, pl[0].friction = -0.5, 0.0
        d.n_planes = 1
    keep += [nodes, anchors, sph, pl]
    d.n_pins = len(nodes)
    d.pin_nodes = nodes.ctypes.data_as(C.POINTER(C.c_int32))
    d.pin_anchors = anchors.ctypes.data_as(C.POINTER(C.c_double))
    d.spheres = C.cast(sph, C.POINTER(_abi.sc_sphere))
    d.planes = C.cast(pl, C.POINTER(_abi.sc_plane))
    d.stiffness, d.damping, d.spacing = 0.0, 0.0, 1.0 / (n - 1)
    return d


def build(cfg_id: int, batch: Optional[int] = None, cloth0: int = 0, plane: bool = True,
          n: Optional[int] = None):
    """(workload, cloth descriptors, keep-alive list, params, x0 [B][n*n][3] f32, v0 zeros);
    n: shrink the grid to n x n (tests)."""
    w = WORKLOADS[cfg_id]
    if n is not None:
        w = Workload(w.name + "_n%d" % n, n, w.batch, w.steps, w.seed, w.pins, w.wind, w.sphere,
                     w.hidden8)
    B = w.batch if batch is None else batch
    x = np.empty((B, w.n * w.n, 3), np.float32)
    keep: list = []
    cds = []
    for i in range(B):
        x[i] = sheet(w.seed, cloth0 + i, w.n)
        cds.append(cloth_desc(w, cloth0 + i, x[i], keep, plane))
    return w, cds, keep, params(w), x, np.zeros_like(x)
