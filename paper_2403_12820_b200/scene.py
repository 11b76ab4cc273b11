"""Scene / parameter / trajectory types of the reference's public API, host side.

Mirrors (reference paths under /root/reference/proj):
  NetworkParams          include/cloth/net.hpp:35-54, src/net.cpp:81-93 (defaults)
  MaterialParams         include/cloth/grid.hpp:65-76, src/grid.cpp:73-81 (validate)
  BoundarySpec / Pins    include/cloth/scene.hpp:13-29
  SphereCollider         include/cloth/scene.hpp:31-35
  Scene                  include/cloth/scene.hpp:43-60, src/scene.cpp:23-61 (validate)
  Trajectory             include/cloth/scene.hpp:62-74
  build_grid             src/grid.cpp:83-138
  parse_scene/load_scene src/io.cpp:30-119 (helpers, selectors), :199-371 (schema)
  params_fingerprint     src/eval.cpp:135-149
These are plain data + validation; all stepping happens in the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import math
import struct
import sys
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

K_CHANNELS = 12
# canonical channel order E,N,W,S,NE,NW,SW,SE,E2,N2,W2,S2 (grid.cpp:14-30)
STENCIL_OFFSETS = [
    (1, 0, 1.0), (0, 1, 1.0), (-1, 0, 1.0), (0, -1, 1.0),
    (1, 1, math.sqrt(2.0)), (-1, 1, math.sqrt(2.0)), (-1, -1, math.sqrt(2.0)), (1, -1, math.sqrt(2.0)),
    (2, 0, 2.0), (0, 2, 2.0), (-2, 0, 2.0), (0, -2, 2.0),
]
NEGATED_CHANNEL = [2, 3, 0, 1, 6, 7, 4, 5, 10, 11, 8, 9]  # grid.cpp:32-35


class ConfigError(ValueError):
    """cloth::ConfigError (error.hpp:17-21); pybind maps it to ValueError (bindings.cpp:64)."""


class IoError(OSError):
    """cloth::IoError (error.hpp:23-27); pybind maps it to OSError (bindings.cpp:65)."""


class NumericsError(ArithmeticError):
    """cloth::NumericsError (error.hpp:29-33); pybind maps it to ArithmeticError (bindings.cpp:66)."""


def channel_order_hash() -> int:
    """FNV-1a over "%d,%d,%.17g;" per offset (grid.cpp:37-49)."""
    h = 0xCBF29CE484222325
    for dx, dy, m in STENCIL_OFFSETS:
        for b in ("%d,%d,%.17g;" % (dx, dy, m)).encode():
            h ^= b
            h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


class ParamGroup(enum.IntEnum):
    """net.hpp:14-22."""
    Kernel = 0
    Linear = 1
    Bias = 2
    Nonlinear = 3
    Deriv = 4
    SelfVelocity = 5
    Alpha = 6


class NetworkParams:
    """All 53 network-cell scalars (net.hpp:35-54). Default: unit kernel gains, alpha = 1, zero
    weights; kernel and alpha frozen (net.cpp:81-93)."""

    kScalarCount = 53

    def __init__(self):
        self.kernel_gain = np.ones(K_CHANNELS)
        self.linear_w = np.zeros(K_CHANNELS)
        self.linear_b = np.zeros(3)
        self.nonlinear_w = np.zeros(K_CHANNELS)
        self.deriv_w = np.zeros(K_CHANNELS)
        self.self_velocity_w = 0.0
        self.isru_alpha = 1.0
        self.trainable = [True] * 7
        self.trainable[ParamGroup.Kernel] = False
        self.trainable[ParamGroup.Alpha] = False
        # InitBracket per group (net.hpp:28-31), set by the DE pre-search (train.cpp:296-310)
        self.brackets = [(-1.0, 1.0)] * 7

    def scalars(self) -> List[float]:
        """for_each_scalar order (net.hpp:72-81)."""
        return ([float(v) for v in self.kernel_gain] + [float(v) for v in self.linear_w]
                + [float(v) for v in self.linear_b] + [float(v) for v in self.nonlinear_w]
                + [float(v) for v in self.deriv_w] + [float(self.self_velocity_w),
                                                       float(self.isru_alpha)])

    @classmethod
    def from_scalars(cls, s: Sequence[float]) -> "NetworkParams":
        if len(s) != cls.kScalarCount:
            raise ConfigError("params: expected 53 scalars")
        p = cls()
        s = [float(v) for v in s]
        p.kernel_gain = np.array(s[0:12])
        p.linear_w = np.array(s[12:24])
        p.linear_b = np.array(s[24:27])
        p.nonlinear_w = np.array(s[27:39])
        p.deriv_w = np.array(s[39:51])
        p.self_velocity_w = s[51]
        p.isru_alpha = s[52]
        return p

    @property
    def fingerprint(self) -> str:
        return params_fingerprint(self)

    def to_c(self) -> _abi.sc_params:
        c = _abi.sc_params()
        for name in ("kernel_gain", "linear_w", "nonlinear_w", "deriv_w"):
            arr = getattr(c, name)
            for i, v in enumerate(getattr(self, name)):
                arr[i] = float(v)
        for i in range(3):
            c.linear_b[i] = float(self.linear_b[i])
        c.self_velocity_w = float(self.self_velocity_w)
        c.isru_alpha = float(self.isru_alpha)
        return c

    def copy(self) -> "NetworkParams":
        p = NetworkParams.from_scalars(self.scalars())
        p.trainable = list(self.trainable)
        p.brackets = list(self.brackets)
        return p

    def is_trainable(self, g: "ParamGroup") -> bool:
        return bool(self.trainable[int(g)])

    def set_trainable(self, g: "ParamGroup", on: bool) -> None:
        self.trainable[int(g)] = bool(on)


def params_fingerprint(p: NetworkParams) -> str:
    """FNV-1a over the little-endian bytes of the 53 doubles (eval.cpp:135-149)."""
    h = 0xCBF29CE484222325
    for v in p.scalars():
        for b in struct.pack("<d", v):
            h ^= b
            h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


@dataclass
class MaterialParams:
    stiffness: float = 0.0
    damping: float = 0.0
    mass: float = 1.0
    gravity: np.ndarray = field(default_factory=lambda: np.zeros(3))
    drag: float = 0.0
    pressure: float = 0.0

    def validate(self) -> None:  # grid.cpp:73-81
        f = math.isfinite
        if not f(self.stiffness) or self.stiffness < 0.0:
            raise ConfigError("material.stiffness: must be a finite value >= 0")
        if not f(self.damping) or self.damping < 0.0:
            raise ConfigError("material.damping: must be a finite value >= 0")
        if not f(self.mass) or self.mass <= 0.0:
            raise ConfigError("material.mass: must be a finite value > 0")
        if not np.all(np.isfinite(self.gravity)):
            raise ConfigError("material.gravity: components must be finite")
        if not f(self.drag) or self.drag < 0.0:
            raise ConfigError("material.drag: must be a finite value >= 0")
        if not f(self.pressure):
            raise ConfigError("material.pressure: must be finite")


class PlugForce(enum.Enum):
    """scene.hpp:38."""
    Pressure = "pressure"
    Gravity = "gravity"
    Drag = "drag"


@dataclass
class SphereCollider:
    center: np.ndarray
    radius: float
    friction: float = 0.0


@dataclass
class PlaneCollider:
    """Extension (no reference counterpart): plane z = height, normal +z."""
    height: float
    friction: float = 0.0


@dataclass
class BoundarySpec:
    nodes: List[int] = field(default_factory=list)       # sorted, unique
    anchors: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    motion: Optional[np.ndarray] = None                  # PinMotion.velocity or None

    def pin_velocity(self) -> np.ndarray:
        return np.array(self.motion, dtype=np.float64) if self.motion is not None else np.zeros(3)

    def anchor_at(self, k: int, t: float) -> np.ndarray:
        a = np.asarray(self.anchors[k], dtype=np.float64)
        return a + self.pin_velocity() * t if self.motion is not None else a.copy()


class Scene:
    """cloth::Scene (scene.hpp:43-60) for one cloth on an nx-by-ny grid."""

    def __init__(self, nx: int, ny: int, spacing: float, positions: Optional[np.ndarray],
                 velocities: Optional[np.ndarray] = None, name: str = ""):
        """positions None: a descriptor-only scene (e.g. one rank's strip of a huge cloth,
        whose state lives on the device); the reference-style rollout() needs positions."""
        self.name = name
        self.nx, self.ny, self.spacing = int(nx), int(ny), float(spacing)
        if positions is None:
            self.initial_x = self.initial_v = None
        else:
            self.initial_x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
            self.initial_v = (np.zeros_like(self.initial_x) if velocities is None else
                              np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3))
        self.material = MaterialParams()
        self.dt = 0.0
        self.steps = 0
        self.bc = BoundarySpec()
        self.colliders: List[SphereCollider] = []
        self.planes: List[PlaneCollider] = []
        self.plug_forces: List[PlugForce] = []

    # ---- pybind-compatible accessors (bindings.cpp:69-89) ----
    @property
    def node_count(self) -> int:
        return self.nx * self.ny

    @property
    def pinned_nodes(self) -> List[int]:
        return list(self.bc.nodes)

    def initial_positions(self) -> np.ndarray:
        return self.initial_x.copy()

    def plugs(self, f: PlugForce) -> bool:
        return f in self.plug_forces

    def max_springs_per_node(self) -> int:
        """GridTopology::max_springs_per_node (grid.cpp:62-66). A node's valid-channel count
        depends only on its distance to each edge clamped at the stencil radius 2, so a few
        representative columns/rows cover every class."""
        def reps(n):
            return sorted({i for i in (0, 1, 2, n // 2, n - 3, n - 2, n - 1) if 0 <= i < n})
        best = 0
        for iy in reps(self.ny):
            for ix in reps(self.nx):
                cnt = sum(1 for dx, dy, _ in STENCIL_OFFSETS
                          if 0 <= ix + dx < self.nx and 0 <= iy + dy < self.ny)
                best = max(best, cnt)
        return best

    def stable_dt(self) -> float:  # scene.cpp:17-21
        k_row = self.material.stiffness * self.max_springs_per_node()
        if k_row <= 0.0:
            return math.inf
        return 0.5 * math.sqrt(self.material.mass / k_row)

    @property
    def spring_count(self) -> int:
        nx, ny = self.nx, self.ny
        return ((nx - 1) * ny + nx * (ny - 1) + 2 * (nx - 1) * (ny - 1)
                + max(nx - 2, 0) * ny + nx * max(ny - 2, 0))

    def validate(self) -> None:  # scene.cpp:23-61
        if self.nx < 2:
            raise ConfigError("grid.nx: must be >= 2")
        if self.ny < 2:
            raise ConfigError("grid.ny: must be >= 2")
        if not self.spacing > 0.0:
            raise ConfigError("grid.spacing: must be > 0")
        n = self.node_count
        if self.initial_x is None:
            raise ConfigError("initial state: scene has no initial positions")
        if self.initial_x.shape != (n, 3) or self.initial_v.shape != (n, 3):
            raise ConfigError("initial state: node count does not match the grid")
        if not (np.all(np.isfinite(self.initial_x)) and np.all(np.isfinite(self.initial_v))):
            raise ConfigError("initial state: non-finite component")
        self.material.validate()
        if not (self.dt > 0.0) or not math.isfinite(self.dt):
            raise ConfigError("time.dt: must be a finite value > 0")
        if self.steps < 0:
            raise ConfigError("time.steps: must be >= 0")
        anchors = np.asarray(self.bc.anchors, dtype=np.float64).reshape(-1, 3)
        if len(anchors) != len(self.bc.nodes):
            raise ConfigError("pins: anchor list does not match the node list")
        for k, i in enumerate(self.bc.nodes):
            if i < 0 or i >= n:
                raise ConfigError("pins.nodes[%d]: index out of range" % k)
            if k > 0 and self.bc.nodes[k - 1] >= i:
                raise ConfigError("pins.nodes: must be strictly increasing (sorted, unique)")
            if not np.all(np.isfinite(anchors[k])):
                raise ConfigError("pins.anchors[%d]: non-finite component" % k)
        if self.bc.motion is not None and not np.all(np.isfinite(self.bc.motion)):
            raise ConfigError("pins.motion.velocity: components must be finite")
        for k, s in enumerate(self.colliders):
            path = "colliders[%d]" % k
            if not np.all(np.isfinite(s.center)):
                raise ConfigError(path + ".center: components must be finite")
            if not (s.radius > 0.0) or not math.isfinite(s.radius):
                raise ConfigError(path + ".radius: must be a finite value > 0")
            if not (0.0 <= s.friction <= 1.0):
                raise ConfigError(path + ".friction: must be in [0, 1]")
        for k, q in enumerate(self.planes):
            path = "planes[%d]" % k
            if not math.isfinite(q.height):
                raise ConfigError(path + ".height: must be finite")
            if not (0.0 <= q.friction <= 1.0):
                raise ConfigError(path + ".friction: must be in [0, 1]")
        if len(set(self.plug_forces)) != len(self.plug_forces):
            raise ConfigError("plug_forces: duplicate entry")

    def __repr__(self) -> str:
        return "<Scene %s %dx%d>" % (self.name or "?", self.nx, self.ny)

    # ---- C descriptor ----
    def cloth_desc(self, keep: list) -> _abi.sc_cloth_desc:
        """sc_cloth_desc for this scene; arrays it points to are appended to `keep`."""
        d = _abi.sc_cloth_desc()
        d.dt = float(self.dt)
        d.mass = float(self.material.mass)
        d.drag = float(self.material.drag)
        d.pressure = float(self.material.pressure)
        for i in range(3):
            d.gravity[i] = float(self.material.gravity[i])
        d.plug_pressure = int(self.plugs(PlugForce.Pressure))
        d.plug_gravity = int(self.plugs(PlugForce.Gravity))
        d.plug_drag = int(self.plugs(PlugForce.Drag))
        nodes = np.ascontiguousarray(self.bc.nodes, dtype=np.int32)
        anchors = np.ascontiguousarray(np.asarray(self.bc.anchors, dtype=np.float64).reshape(-1, 3))
        keep += [nodes, anchors]
        d.n_pins = len(nodes)
        d.pin_nodes = nodes.ctypes.data_as(C.POINTER(C.c_int32))
        d.pin_anchors = anchors.ctypes.data_as(C.POINTER(C.c_double))
        u = self.bc.pin_velocity()
        for i in range(3):
            d.pin_velocity[i] = float(u[i])
        sph = (_abi.sc_sphere * max(1, len(self.colliders)))()
        for k, s in enumerate(self.colliders):
            for i in range(3):
                sph[k].center[i] = float(s.center[i])
            sph[k].radius = float(s.radius)
            sph[k].friction = float(s.friction)
        pl = (_abi.sc_plane * max(1, len(self.planes)))()
        for k, q in enumerate(self.planes):
            pl[k].height = float(q.height)
            pl[k].friction = float(q.friction)
        keep += [sph, pl]
        d.n_spheres = len(self.colliders)
        d.spheres = C.cast(sph, C.POINTER(_abi.sc_sphere))
        d.n_planes = len(self.planes)
        d.planes = C.cast(pl, C.POINTER(_abi.sc_plane))
        d.stiffness = float(self.material.stiffness)
        d.damping = float(self.material.damping)
        d.spacing = float(self.spacing)
        return d


class Trajectory:
    """Ordered frames (scene.hpp:62-74; pybind surface bindings.cpp:82-103)."""

    def __init__(self, nx: int, ny: int, dt: float, spacing: float,
                 frames_x: np.ndarray, frames_v: np.ndarray):
        self.nx, self.ny, self.dt, self.spacing = nx, ny, dt, spacing
        self.frames_x = frames_x  # [frames][n][3]
        self.frames_v = frames_v

    @property
    def frame_count(self) -> int:
        return int(self.frames_x.shape[0])

    def __len__(self) -> int:
        return self.frame_count

    def _check(self, f: int) -> None:
        if f < 0 or f >= self.frame_count:
            raise ConfigError("frame index out of range")

    def validate(self) -> None:
        """Trajectory::validate (scene.cpp:63-75), same checks and messages."""
        if self.nx < 2 or self.ny < 2:
            raise ConfigError("trajectory: grid dimensions must be >= 2")
        if not (self.dt > 0.0):
            raise ConfigError("trajectory: dt must be > 0")
        if not (self.spacing > 0.0):
            raise ConfigError("trajectory: spacing must be > 0")
        if self.frame_count < 1:
            raise ConfigError("trajectory: needs at least one frame")
        n = self.nx * self.ny
        fx, fv = np.asarray(self.frames_x), np.asarray(self.frames_v)
        if fx.ndim != 3 or fx.shape[1:] != (n, 3) or fv.shape != fx.shape:
            raise ConfigError("trajectory: frame 0 has the wrong node count")
        bad = ~(np.isfinite(fx).all(axis=(1, 2)) & np.isfinite(fv).all(axis=(1, 2)))
        if bad.any():
            raise ConfigError("trajectory: frame %d has non-finite components"
                              % int(np.argmax(bad)))

    def positions(self, frame: int) -> np.ndarray:
        self._check(frame)
        return np.array(self.frames_x[frame], dtype=np.float64)

    def velocities(self, frame: int) -> np.ndarray:
        self._check(frame)
        return np.array(self.frames_v[frame], dtype=np.float64)

    def __repr__(self) -> str:
        return "<Trajectory %dx%d, %d frames>" % (self.nx, self.ny, self.frame_count)


class GridPlane(enum.Enum):
    XY = "xy"
    XZ = "xz"
    YZ = "yz"


def build_grid(nx: int, ny: int, spacing: float, origin=(0.0, 0.0, 0.0),
               plane: GridPlane = GridPlane.XY) -> np.ndarray:
    """Flat sheet positions [n][3] of build_grid (grid.cpp:83-138): node iy*nx+ix at
    origin + (spacing*ix, spacing*iy) in the chosen plane."""
    if nx < 2:
        raise ConfigError("grid.nx: must be >= 2")
    if ny < 2:
        raise ConfigError("grid.ny: must be >= 2")
    if not (spacing > 0.0) or not math.isfinite(spacing):
        raise ConfigError("grid.spacing: must be a finite value > 0")
    origin = np.asarray(origin, dtype=np.float64)
    if not np.all(np.isfinite(origin)):
        raise ConfigError("grid.origin: components must be finite")
    ix = np.tile(np.arange(nx, dtype=np.float64), ny)
    iy = np.repeat(np.arange(ny, dtype=np.float64), nx)
    a, b = spacing * ix, spacing * iy
    x = np.empty((nx * ny, 3))
    z = np.zeros_like(a)
    cols = {GridPlane.XY: (a, b, z), GridPlane.XZ: (a, z, b), GridPlane.YZ: (z, a, b)}[plane]
    for d in range(3):
        x[:, d] = origin[d] + cols[d]
    return x


# ------------------------------------------------------------------ JSON scenes (io.cpp) ----

def _fail(path: str, what: str):
    raise ConfigError("%s: %s" % (path, what))


def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _num(v, path):
    if not _is_num(v):
        _fail(path, "expected a number")
    return float(v)


def _pos(v, path):
    d = _num(v, path)
    if not (d > 0.0) or not math.isfinite(d):
        _fail(path, "must be a finite value > 0")
    return d


def _nonneg(v, path):
    d = _num(v, path)
    if not (d >= 0.0) or not math.isfinite(d):
        _fail(path, "must be a finite value >= 0")
    return d


def _int(v, path):
    if not isinstance(v, int) or isinstance(v, bool):
        _fail(path, "expected an integer")
    return int(v)


def _vec3(v, path):
    if not isinstance(v, list) or len(v) != 3:
        _fail(path, "expected an array of 3 numbers")
    out = np.zeros(3)
    for d in range(3):
        c = _num(v[d], "%s[%d]" % (path, d))
        if not math.isfinite(c):
            _fail(path, "components must be finite")
        out[d] = c
    return out


def _require(obj, path, key):
    if key not in obj:
        _fail(path + "." + key if path else "." + key, "missing required field")
    return obj[key]


def _reject_unknown(obj, path, allowed):
    for key in obj:
        if key not in allowed:
            _fail(key if not path else path + "." + key, "unknown field")


def _select_nodes(name: str, nx: int, ny: int, path: str, out: list) -> None:
    """Named pin selectors; "top" is the iy = ny-1 row (io.cpp:85-119)."""
    def row(iy):
        out.extend(iy * nx + ix for ix in range(nx))

    def col(ix):
        out.extend(iy * nx + ix for iy in range(ny))

    if name == "edges":
        row(0); row(ny - 1); col(0); col(nx - 1)
    elif name == "top_row":
        row(ny - 1)
    elif name == "bottom_row":
        row(0)
    elif name == "left_column":
        col(0)
    elif name == "right_column":
        col(nx - 1)
    elif name == "top_left":
        out.append((ny - 1) * nx)
    elif name == "top_right":
        out.append((ny - 1) * nx + nx - 1)
    elif name == "bottom_left":
        out.append(0)
    elif name == "bottom_right":
        out.append(nx - 1)
    else:
        _fail(path, 'unknown node selector "%s"' % name)


def parse_scene(json_text: str) -> Scene:
    """parse_scene_config (io.cpp:199-359): strict schema, unknown keys rejected."""
    try:
        root = json.loads(json_text)
    except json.JSONDecodeError as e:
        raise ConfigError("scene config is not valid JSON: %s" % e) from None
    if not isinstance(root, dict):
        raise ConfigError("scene config: top level must be an object")
    _reject_unknown(root, "", {"name", "grid", "material", "time", "pins", "colliders",
                               "plug_forces"})
    name = ""
    if "name" in root:
        if not isinstance(root["name"], str):
            _fail("name", "expected a string")
        name = root["name"]
    grid = _require(root, "", "grid")
    if not isinstance(grid, dict):
        _fail("grid", "expected an object")
    _reject_unknown(grid, "grid", {"nx", "ny", "spacing", "origin", "plane"})
    nx = _int(_require(grid, "grid", "nx"), "grid.nx")
    ny = _int(_require(grid, "grid", "ny"), "grid.ny")
    spacing = _pos(_require(grid, "grid", "spacing"), "grid.spacing")
    origin = _vec3(grid["origin"], "grid.origin") if "origin" in grid else np.zeros(3)
    plane = GridPlane.XY
    if "plane" in grid:
        if not isinstance(grid["plane"], str):
            _fail("grid.plane", "expected a string")
        try:
            plane = GridPlane(grid["plane"])
        except ValueError:
            _fail("grid.plane", 'must be one of "xy", "xz", "yz"')
    x0 = build_grid(nx, ny, spacing, origin, plane)
    s = Scene(nx, ny, spacing, x0, name=name)

    mat = _require(root, "", "material")
    if not isinstance(mat, dict):
        _fail("material", "expected an object")
    _reject_unknown(mat, "material", {"stiffness", "damping", "mass", "gravity", "drag",
                                      "pressure", "pressure_side"})
    m = s.material
    m.stiffness = _nonneg(_require(mat, "material", "stiffness"), "material.stiffness")
    m.damping = _nonneg(_require(mat, "material", "damping"), "material.damping")
    m.mass = _pos(_require(mat, "material", "mass"), "material.mass")
    if "gravity" in mat:
        m.gravity = _vec3(mat["gravity"], "material.gravity")
    if "drag" in mat:
        m.drag = _nonneg(mat["drag"], "material.drag")
    pressure = _nonneg(mat["pressure"], "material.pressure") if "pressure" in mat else 0.0
    if "pressure_side" in mat:
        side = _int(mat["pressure_side"], "material.pressure_side")
        if side not in (1, -1):
            _fail("material.pressure_side", "must be 1 or -1")
        pressure *= side
    m.pressure = pressure

    tm = _require(root, "", "time")
    if not isinstance(tm, dict):
        _fail("time", "expected an object")
    _reject_unknown(tm, "time", {"dt", "steps"})
    s.steps = _int(_require(tm, "time", "steps"), "time.steps")
    if s.steps < 0:
        _fail("time.steps", "must be >= 0")
    if "dt" in tm:
        s.dt = _pos(tm["dt"], "time.dt")
    else:
        s.dt = s.stable_dt()
        if not math.isfinite(s.dt):
            _fail("time.dt", "required when stiffness is 0 (no stability bound to default to)")

    if "pins" in root:
        pins = root["pins"]
        if not isinstance(pins, dict):
            _fail("pins", "expected an object")
        _reject_unknown(pins, "pins", {"nodes", "motion"})
        nodes = _require(pins, "pins", "nodes")
        sel: list = []

        def add(entry, path):
            if isinstance(entry, str):
                _select_nodes(entry, nx, ny, path, sel)
            elif isinstance(entry, int) and not isinstance(entry, bool):
                sel.append(int(entry))
            else:
                _fail(path, "expected a node index or a selector string")

        if isinstance(nodes, list):
            for k, e in enumerate(nodes):
                add(e, "pins.nodes[%d]" % k)
        else:
            add(nodes, "pins.nodes")
        sel = sorted(set(sel))
        for i in sel:
            if i < 0 or i >= nx * ny:
                _fail("pins.nodes", "index out of range")
        s.bc.nodes = sel
        s.bc.anchors = s.initial_x[sel].copy() if sel else np.zeros((0, 3))
        if "motion" in pins:
            mo = pins["motion"]
            if not isinstance(mo, dict):
                _fail("pins.motion", "expected an object")
            _reject_unknown(mo, "pins.motion", {"velocity"})
            s.bc.motion = _vec3(_require(mo, "pins.motion", "velocity"), "pins.motion.velocity")

    if "colliders" in root:
        cols = root["colliders"]
        if not isinstance(cols, list):
            _fail("colliders", "expected an array")
        for k, c in enumerate(cols):
            path = "colliders[%d]" % k
            if not isinstance(c, dict):
                _fail(path, "expected an object")
            _reject_unknown(c, path, {"type", "center", "radius", "friction"})
            typ = _require(c, path, "type")
            if not isinstance(typ, str) or typ != "sphere":
                _fail(path + ".type", 'only "sphere" is supported')
            sp = SphereCollider(_vec3(_require(c, path, "center"), path + ".center"),
                                _pos(_require(c, path, "radius"), path + ".radius"))
            if "friction" in c:
                sp.friction = _num(c["friction"], path + ".friction")
                if not (0.0 <= sp.friction <= 1.0):
                    _fail(path + ".friction", "must be in [0, 1]")
            s.colliders.append(sp)

    if "plug_forces" in root:
        plugs = root["plug_forces"]
        if not isinstance(plugs, list):
            _fail("plug_forces", "expected an array")
        for k, p in enumerate(plugs):
            path = "plug_forces[%d]" % k
            if not isinstance(p, str):
                _fail(path, "expected a string")
            try:
                s.plug_forces.append(PlugForce(p))
            except ValueError:
                _fail(path, 'must be one of "pressure", "gravity", "drag"')

    s.validate()
    if s.dt > s.stable_dt():
        print("warning: %s: dt %.6g exceeds the explicit-integration stability bound %.6g"
              % (s.name or "scene", s.dt, s.stable_dt()), file=sys.stderr)
    return s


def load_scene(path: str) -> Scene:
    """load_scene (io.cpp:361-371)."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise IoError("cannot open scene config " + path) from None
    try:
        return parse_scene(text)
    except ConfigError as e:
        raise ConfigError(path + ": " + str(e)) from None
