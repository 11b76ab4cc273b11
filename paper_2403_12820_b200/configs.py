"""The five BASELINE.json workloads as seeded synthetic inputs (SURVEY.md §8(d) mapping).

Conventions (frozen):
  * Grid: build_grid(n, n, 1/(n-1), 0, XY) (grid.cpp:83-138) + N(0, 1e-3) noise on every
    component, per-(cloth,row) streams (csrc/host_gen.cpp). v0 = 0.
  * Weights: the 40 trainable scalars ~ N(0, 0.05) in for_each_scalar order (net.hpp:72-81:
    linear[12], bias[3], nonlinear[12], deriv[12], self_velocity) from stream mix(seed, 1);
    gains = 1, alpha = 1 (net.cpp:81-93). "Hidden 8, 3x3" (config 1) = skip channels 8..11
    zeroed; "hidden 16/32" = the full 12-channel reference cell (the only cell it has).
  * Dynamics: gravity plugged, g_eff = (0,0,-9.8) + wind (summed in double, cast once), wind
    direction uniform on the sphere, magnitude U(0,2), per cloth from stream mix(seed, 2+b).
    dt = 1/240, mass 1, no drag / pressure plug.
  * Pins: "top" = row iy = ny-1 (io.cpp:85-111); anchors captured AFTER the noise.
  * Config 3 sphere: R = 0.3, friction 0, centre (U(0,1), U(0,1), -0.35).
  * Config 5: cloth b's class = b mod 3 -> top_row / top corners / free + plane z = -0.5.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _abi
from .scene import NetworkParams, PlaneCollider, PlugForce, Scene, SphereCollider

DT = 1.0 / 240.0


@dataclass(frozen=True)
class Config:
    name: str
    n: int             # grid is n x n
    batch: int
    steps: int
    seed: int
    pins: str          # "corners" | "top_row" | "mixed"
    wind: bool
    sphere: bool
    hidden8: bool      # zero the skip channels (3x3 footprint)
    description: str


CONFIGS = {
    1: Config("cfg1_32x32_b1", 32, 1, 100, 0, "corners", False, False, True,
              "1 x 32^2, two top corners pinned, gravity, 100 steps, hidden 8 (3x3)"),
    2: Config("cfg2_256x256_b64", 256, 64, 1000, 1, "top_row", True, False, False,
              "64 x 256^2, top row pinned, gravity + wind, 1000 steps"),
    3: Config("cfg3_1024x1024_sphere", 1024, 1, 500, 2, "corners", False, True, False,
              "1 x 1024^2, two corners pinned, sphere R=0.3 under the cloth, 500 steps"),
    4: Config("cfg4_8192x8192", 8192, 1, 200, 3, "top_row", False, False, False,
              "1 x 8192^2, top row pinned, gravity, 200 steps"),
    5: Config("cfg5_128x128_b4096_mixed", 128, 4096, 300, 4, "mixed", True, False, False,
              "4096 x 128^2, mixed BCs (top row / corners / free onto plane z=-0.5), wind"),
}


def _lib():
    return _abi.load()


def mix(seed: int, stream: int) -> int:
    return int(_lib().sc_rng_mix(C.c_uint64(seed), C.c_uint64(stream)))


def normals(stream_seed: int, count: int, sigma: float) -> np.ndarray:
    out = np.empty(count, np.float64)
    _lib().sc_rng_normal(C.c_uint64(stream_seed), count, sigma, out.ctypes.data_as(C.c_void_p))
    return out


def uniforms(stream_seed: int, count: int) -> np.ndarray:
    out = np.empty(count, np.float64)
    _lib().sc_rng_uniform01(C.c_uint64(stream_seed), count, out.ctypes.data_as(C.c_void_p))
    return out


def make_params(seed: int, hidden8: bool = False, sigma: float = 0.05) -> NetworkParams:
    w = normals(mix(seed, 1), 40, sigma)
    p = NetworkParams()
    p.linear_w = w[0:12].copy()
    p.linear_b = w[12:15].copy()
    p.nonlinear_w = w[15:27].copy()
    p.deriv_w = w[27:39].copy()
    p.self_velocity_w = float(w[39])
    if hidden8:
        p.linear_w[8:] = 0.0
        p.nonlinear_w[8:] = 0.0
        p.deriv_w[8:] = 0.0
    return p


def sheet(seed: int, cloth: int, n: int, row0: int = 0, rows: Optional[int] = None,
          sigma: float = 1e-3, f32: bool = True, f64: bool = False, threads: int = 0):
    """Noisy flat sheet rows [row0, row0+rows) of cloth `cloth` as AoS (rows*n, 3) arrays."""
    rows = n - row0 if rows is None else rows
    threads = threads or min(32, os.cpu_count() or 1)
    a32 = np.empty((rows * n, 3), np.float32) if f32 else None
    a64 = np.empty((rows * n, 3), np.float64) if f64 else None
    _lib().sc_gen_sheet(C.c_uint64(seed), cloth, n, n, row0, rows, 1.0 / (n - 1), sigma,
                        a32.ctypes.data_as(C.c_void_p) if f32 else None,
                        a64.ctypes.data_as(C.c_void_p) if f64 else None, threads)
    return a32, a64


def wind(seed: int, cloth: int) -> np.ndarray:
    u = uniforms(mix(seed, 2 + cloth), 3)
    z = 2.0 * u[0] - 1.0
    phi = 2.0 * math.pi * u[1]
    r = math.sqrt(max(0.0, 1.0 - z * z))
    return (2.0 * u[2]) * np.array([r * math.cos(phi), r * math.sin(phi), z])


def pin_nodes(kind: str, n: int) -> List[int]:
    if kind == "top_row":
        return [(n - 1) * n + ix for ix in range(n)]
    if kind == "corners":
        return [(n - 1) * n, (n - 1) * n + n - 1]
    if kind == "free":
        return []
    raise ValueError(kind)


def cloth_kind(cfg: Config, b: int) -> str:
    if cfg.pins != "mixed":
        return cfg.pins
    return ("top_row", "corners", "free")[b % 3]


def make_scene(cfg: Config, b: int, x0: Optional[np.ndarray], row0: int = 0) -> Scene:
    """Scene of cloth b. x0: its initial positions as AoS rows [row0, row0 + len(x0)/n) (the
    whole cloth when row0 == 0 and all rows are given; then it becomes scene.initial_x). Pin
    anchors are the noisy initial positions of the pinned nodes (captured after the noise),
    rounded through f32 exactly like the f32 state."""
    n = cfg.n
    rows = 0 if x0 is None else x0.shape[0] // n
    whole = x0 is not None and row0 == 0 and rows == n
    s = Scene(n, n, 1.0 / (n - 1), x0 if whole else None, name=cfg.name)
    s.dt = DT
    s.steps = cfg.steps
    s.material.mass = 1.0
    g = np.array([0.0, 0.0, -9.8])
    if cfg.wind:
        g = g + wind(cfg.seed, b)
    s.material.gravity = g
    s.plug_forces = [PlugForce.Gravity]
    kind = cloth_kind(cfg, b)
    nodes = pin_nodes(kind, n)
    s.bc.nodes = nodes
    if nodes:
        anchors = np.zeros((len(nodes), 3))
        for k, node in enumerate(nodes):
            lr = node // n - row0
            if x0 is not None and 0 <= lr < rows:
                anchors[k] = x0[lr * n + node % n]
            else:  # pinned row outside the given rows: from its own noise stream
                a32, _ = sheet(cfg.seed, b, n, node // n, 1, threads=1)
                anchors[k] = a32[node % n]
        s.bc.anchors = anchors.astype(np.float32).astype(np.float64)
    if cfg.sphere:
        u = uniforms(mix(cfg.seed, 0x20000 + b), 2)
        s.colliders.append(SphereCollider(np.array([u[0], u[1], -0.35]), 0.3, 0.0))
    if kind == "free":
        s.planes.append(PlaneCollider(-0.5, 0.0))
    return s


def build(cfg_id: int, batch: Optional[int] = None, cloth0: int = 0, n: Optional[int] = None,
          threads: int = 0) -> Tuple[Config, List[Scene], NetworkParams, np.ndarray, np.ndarray]:
    """Scenes, params and the f32 initial state [B][n*n][3] for cloths cloth0..cloth0+batch of a
    config (optionally shrunk to an n x n grid for tests)."""
    cfg = CONFIGS[cfg_id]
    if n is not None:
        cfg = Config(cfg.name + "_n%d" % n, n, cfg.batch, cfg.steps, cfg.seed, cfg.pins, cfg.wind,
                     cfg.sphere, cfg.hidden8, cfg.description)
    B = cfg.batch if batch is None else batch
    x = np.empty((B, cfg.n * cfg.n, 3), np.float32)
    scenes = []
    for i in range(B):
        b = cloth0 + i
        a32, _ = sheet(cfg.seed, b, cfg.n, threads=threads)
        x[i] = a32
        scenes.append(make_scene(cfg, b, a32.astype(np.float64)))
    v = np.zeros_like(x)
    return cfg, scenes, make_params(cfg.seed, cfg.hidden8), x, v
