"""Training of the network cell on the GPU: the reference's training surface
(train.hpp, net.hpp:57-68,118-126; Python binding `train` / `gradient_check`,
bindings.cpp:168-212) over the native trainer in csrc/train.cu.

Trainer         one scene + its ground-truth trajectory resident on the device
  .sample_batch   sample_batch (train.cpp:91-127): the reference's RNG draws, device targets
  .compute_loss   compute_loss (train.cpp:129-209): hybrid loss + the 53 gradient sums
  .run            train_loop (train.cpp:343-375): DE pre-search, Adam, schedule (native C++)
train           the binding `stencilcloth.train(scene, trajectory, ...)` -> (params, history)
backward_gradients / gradient_check   net.cpp:144-240
Everything is float64 and bit-identical to the reference (tests/test_gpu_train.py).
"""
from __future__ import annotations

import ctypes as C
import enum
import functools
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from .api import _ptr, _raise
from .scene import (ConfigError, NetworkParams, ParamGroup, Scene, Trajectory, build_grid)

K_SCALARS = 53


class ScheduleKind(enum.IntEnum):
    Step = 0
    Cosine = 1


@dataclass
class ScheduleConfig:
    """ScheduleConfig (train.hpp:16-26)."""
    kind: ScheduleKind = ScheduleKind.Step
    lr0: float = 1e-2
    gamma: float = 0.5
    interval: int = 250
    floor: float = 1e-5
    period: int = 1000


@dataclass
class DeConfig:
    """DeConfig (train.hpp:33-40)."""
    population: int = 64
    generations: int = 60
    bound: float = 4.0
    cross_prob: float = 0.9
    diff_weight: float = 0.7
    probe_batch: int = 32


@dataclass
class TrainConfig:
    """TrainConfig (train.hpp:42-53)."""
    alpha: float = 0.5
    batch_size: int = 128
    epochs: int = 2000
    schedule: ScheduleConfig = field(default_factory=ScheduleConfig)
    seed: int = 0
    de: DeConfig = field(default_factory=DeConfig)
    checkpoint_interval: int = 500
    freeze: List[ParamGroup] = field(default_factory=list)

    def to_c(self) -> _abi.sc_train_config:
        c = _abi.sc_train_config()
        c.alpha, c.batch_size, c.epochs = float(self.alpha), int(self.batch_size), int(self.epochs)
        s = self.schedule
        c.schedule_kind = int(s.kind)
        c.lr0, c.gamma, c.interval = float(s.lr0), float(s.gamma), int(s.interval)
        c.floor, c.period = float(s.floor), int(s.period)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        d = self.de
        c.de_population, c.de_generations = int(d.population), int(d.generations)
        c.de_bound, c.de_cross_prob = float(d.bound), float(d.cross_prob)
        c.de_diff_weight, c.de_probe_batch = float(d.diff_weight), int(d.probe_batch)
        c.checkpoint_interval = int(self.checkpoint_interval)
        c.freeze_mask = functools.reduce(lambda m, g: m | (1 << int(g)), self.freeze, 0)
        return c


@dataclass
class LossValue:
    """LossValue (train.hpp:72-76)."""
    total: float = 0.0
    physics: float = 0.0
    data: float = 0.0


class ParamGradients:
    """ParamGradients (net.hpp:57-68) over the flat for_each_gradient order."""

    def __init__(self, flat: np.ndarray):
        self.flat = np.asarray(flat, np.float64)
        f = self.flat
        self.kernel, self.linear, self.bias = f[0:12], f[12:24], f[24:27]
        self.nonlinear, self.deriv = f[27:39], f[39:51]
        self.self_velocity, self.alpha = float(f[51]), float(f[52])

    def __repr__(self) -> str:
        return "<ParamGradients |g|=%.6g>" % float(np.linalg.norm(self.flat))


@dataclass
class AdamState:
    """AdamState (train.hpp:118-123)."""
    m: np.ndarray = field(default_factory=lambda: np.zeros(K_SCALARS))
    v: np.ndarray = field(default_factory=lambda: np.zeros(K_SCALARS))
    step: int = 0

    def to_c(self) -> _abi.sc_adam_state:
        c = _abi.sc_adam_state()
        for i in range(K_SCALARS):
            c.m[i], c.v[i] = float(self.m[i]), float(self.v[i])
        c.step = int(self.step)
        return c

    @classmethod
    def from_c(cls, c: _abi.sc_adam_state) -> "AdamState":
        return cls(np.array(c.m[:]), np.array(c.v[:]), int(c.step))


@dataclass
class LossRow:
    """LossRow (train.hpp:125-131)."""
    step: int
    lr: float
    physics: float
    data: float
    total: float


@dataclass
class TrainResult:
    """TrainResult (train.hpp:133-137)."""
    params: NetworkParams
    opt: AdamState
    history: List[LossRow]


def _params_from_c(c: _abi.sc_params, trainable: Sequence[int]) -> NetworkParams:
    p = NetworkParams.from_scalars(list(c.kernel_gain) + list(c.linear_w) + list(c.linear_b)
                                   + list(c.nonlinear_w) + list(c.deriv_w)
                                   + [c.self_velocity_w, c.isru_alpha])
    p.trainable = [bool(t) for t in trainable]
    return p


class Trainer:
    """One scene and its ground-truth trajectory, resident on the GPU."""

    def __init__(self, scene: Scene, trajectory: Trajectory, device: int = 0):
        scene.validate()
        trajectory.validate()
        if (trajectory.nx, trajectory.ny) != (scene.nx, scene.ny):
            raise ConfigError("state shape does not match the grid topology")
        self.lib = _abi.load()
        self.scene, self.trajectory = scene, trajectory
        keep: list = []
        desc = (_abi.sc_cloth_desc * 1)(scene.cloth_desc(keep))
        sd = _abi.sc_scene_desc(scene.nx, scene.ny, 1, C.cast(desc, C.POINTER(_abi.sc_cloth_desc)))
        fx = np.ascontiguousarray(trajectory.frames_x, np.float64)
        fv = np.ascontiguousarray(trajectory.frames_v, np.float64)
        h = C.c_void_p()
        _raise(self.lib, self.lib.sc_trainer_create(device, C.byref(sd), trajectory.frame_count,
                                                    _ptr(fx), _ptr(fv), C.byref(h)))
        self.h = h
        self.n = scene.nx * scene.ny
        self.batch_indices: Optional[np.ndarray] = None

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.sc_trainer_destroy(self.h)
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

    def sample_batch(self, batch_size: int, rng_seed: int, targets: bool = False):
        """sample_batch with a fresh Rng(rng_seed); returns the indices (and the f_k*dt targets
        [batch][node][3] when asked). The batch becomes the current one."""
        idx = np.empty(max(batch_size, 0), np.int32)
        tgt = np.empty((max(batch_size, 0), self.n, 3)) if targets else None
        _raise(self.lib, self.lib.sc_trainer_sample_batch(
            self.h, int(batch_size), int(rng_seed) & 0xFFFFFFFFFFFFFFFF, _ptr(idx), _ptr(tgt)))
        self.batch_indices = idx
        return (idx, tgt) if targets else idx

    def set_batch(self, indices: Sequence[int]) -> None:
        idx = np.ascontiguousarray(indices, np.int32)
        _raise(self.lib, self.lib.sc_trainer_set_batch(self.h, _ptr(idx), len(idx)))
        self.batch_indices = idx

    def compute_loss(self, params: NetworkParams, alpha: float, grads: bool = True
                     ) -> Tuple[LossValue, Optional[ParamGradients]]:
        out = np.empty(3)
        g = np.empty(K_SCALARS) if grads else None
        pc = params.to_c()
        _raise(self.lib, self.lib.sc_trainer_compute_loss(self.h, C.byref(pc), float(alpha),
                                                          _ptr(out), _ptr(g)))
        return LossValue(*map(float, out)), (ParamGradients(g) if grads else None)

    def run(self, cfg: TrainConfig, resume: Optional[TrainResult] = None) -> TrainResult:
        """train_loop (train.cpp:343-375); `resume` continues from its params / optimizer state
        (fine-tune mode, no pre-search)."""
        c = cfg.to_c()
        out = _abi.sc_params()
        tr = np.zeros(7, np.uint8)
        hist = np.zeros((max(cfg.epochs, 1), 5))
        opt = (resume.opt if resume else AdamState()).to_c()
        rp = resume.params.to_c() if resume else None
        rtr = np.array([1 if t else 0 for t in resume.params.trainable], np.uint8) if resume \
            else None
        br = np.zeros(14)
        _raise(self.lib, self.lib.sc_trainer_run(
            self.h, C.byref(c), C.byref(rp) if rp is not None else None, _ptr(rtr),
            C.byref(opt), C.byref(out), _ptr(tr), _ptr(hist), _ptr(br)))
        history = [LossRow(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]))
                   for r in hist[:cfg.epochs]]
        params = _params_from_c(out, tr)
        if resume is not None:  # fine-tune mode keeps the resumed parameters' brackets
            params.brackets = list(resume.params.brackets)
        else:
            params.brackets = [(float(br[2 * g]), float(br[2 * g + 1])) for g in range(7)]
        return TrainResult(params, AdamState.from_c(opt), history)


def sample_indices(frames: int, batch_size: int, rng_seed: int) -> np.ndarray:
    """The index draw of sample_batch (train.cpp:98-109) on the host: batch_size distinct
    transition indices from Rng(rng_seed) over a frames-long trajectory."""
    lib = _abi.load()
    idx = np.empty(max(batch_size, 0), np.int32)
    _raise(lib, lib.sc_sample_indices(int(frames), int(batch_size),
                                      int(rng_seed) & 0xFFFFFFFFFFFFFFFF, _ptr(idx)))
    return idx


def train_loop(cfg: TrainConfig, scene: Scene, trajectory: Trajectory,
               resume: Optional[TrainResult] = None, device: int = 0) -> TrainResult:
    """train_loop (train.hpp:145-154)."""
    with Trainer(scene, trajectory, device) as t:
        return t.run(cfg, resume)


def train(scene: Scene, trajectory: Trajectory, alpha: float = 0.5, batch_size: int = 128,
          epochs: int = 2000, seed: int = 0, lr0: float = 1e-2, de_population: int = 64,
          de_generations: int = 60, de_probe: int = 32, device: int = 0):
    """The binding `stencilcloth.train` (bindings.cpp:168-187): (params, history) with history
    rows (step, lr, physics, data, total)."""
    cfg = TrainConfig(alpha=alpha, batch_size=batch_size, epochs=epochs, seed=seed,
                      schedule=ScheduleConfig(lr0=lr0),
                      de=DeConfig(population=de_population, generations=de_generations,
                                  probe_batch=de_probe))
    r = train_loop(cfg, scene, trajectory, device=device)
    return r.params, [(h.step, h.lr, h.physics, h.data, h.total) for h in r.history]


def backward_gradients(nx: int, ny: int, positions, velocities, params: NetworkParams,
                       upstream, device: int = 0) -> ParamGradients:
    """backward_gradients (net.cpp:144-201) of sum(upstream . forward_impulse) for one state."""
    n = nx * ny
    arrs = []
    for a in (positions, velocities, upstream):
        a = np.ascontiguousarray(a, np.float64)
        if a.shape != (n, 3):
            raise ConfigError("upstream cotangent shape does not match the state"
                              if len(arrs) == 2 else
                              "state shape does not match the grid topology")
        arrs.append(a)
    if not (params.isru_alpha > 0.0):
        raise ConfigError("isru_alpha: must be > 0")
    lib = _abi.load()
    g = np.empty(K_SCALARS)
    pc = params.to_c()
    _raise(lib, lib.sc_backward_gradients(device, nx, ny, _ptr(arrs[0]), _ptr(arrs[1]),
                                          C.byref(pc), _ptr(arrs[2]), _ptr(g)))
    return ParamGradients(g)


class Rng:
    """cloth::Rng (rng.hpp:13-47) over std::mt19937_64 outputs drawn natively."""

    def __init__(self, seed: int, prefetch: int = 4096):
        self.seed, self.pos, self.buf = int(seed) & 0xFFFFFFFFFFFFFFFF, 0, np.empty(0, np.uint64)
        self._fill(prefetch)

    def _fill(self, count: int) -> None:
        out = np.empty(count, np.uint64)
        _abi.load().sc_mt64_fill(self.seed, count, _ptr(out))
        self.buf = out

    def next_u64(self) -> int:
        if self.pos >= len(self.buf):
            self._fill(2 * len(self.buf))
        v = int(self.buf[self.pos])
        self.pos += 1
        return v

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def uniform_below(self, n: int) -> int:
        """Rejection-sampled uniform integer in [0, n) (rng.hpp:20-27)."""
        m = 0xFFFFFFFFFFFFFFFF
        limit = m - m % n
        while True:
            r = self.next_u64()
            if r < limit:
                return r % n

    @staticmethod
    def mix(seed: int, stream: int) -> int:
        """Rng::mix (rng.hpp:36-42), splitmix64 finaliser over the pair."""
        m = 0xFFFFFFFFFFFFFFFF
        z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & m
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        return z ^ (z >> 31)


def gradient_check(nx: int = 8, ny: int = 8, seed: int = 7, eps: float = 1e-6,
                   device: int = 0) -> float:
    """The binding `gradient_check` (bindings.cpp:189-212) -> finite_diff_check (net.cpp:203-240):
    worst relative error of the GPU backward against central differences of sum |impulse|^2."""
    from .api import forward_impulse

    if not (eps > 0.0):
        raise ConfigError("finite_diff_check: eps must be > 0")
    rng = Rng(seed)
    x = build_grid(nx, ny, 0.1)
    v = np.zeros_like(x)
    for i in range(nx * ny):
        for d in range(3):
            x[i, d] += rng.uniform(-0.03, 0.03)
            v[i, d] = rng.uniform(-1.0, 1.0)
    p = NetworkParams()
    for c in range(12):
        p.kernel_gain[c] = rng.uniform(0.5, 1.5)
        p.linear_w[c] = rng.uniform(-0.5, 0.5)
        p.nonlinear_w[c] = rng.uniform(-0.5, 0.5)
        p.deriv_w[c] = rng.uniform(-0.5, 0.5)
    for d in range(3):
        p.linear_b[d] = rng.uniform(-0.3, 0.3)
    p.self_velocity_w = rng.uniform(-0.5, 0.5)
    p.isru_alpha = rng.uniform(0.5, 2.0)
    p.trainable = [True] * 7
    scene = Scene(nx, ny, 0.1, x)
    scene.dt = 1.0  # forward_impulse reads only the topology

    def loss(q: NetworkParams) -> float:
        out = forward_impulse(q, scene, x, v, device=device)
        s = 0.0
        for o in out.tolist():
            s += (o[0] * o[0] + o[1] * o[1]) + o[2] * o[2]
        return s

    out = forward_impulse(p, scene, x, v, device=device)
    analytic = backward_gradients(nx, ny, x, v, p, out * 2.0, device).flat
    worst = 0.0
    base = p.scalars()
    for idx in range(K_SCALARS):
        probe = list(base)
        probe[idx] = base[idx] + eps
        hi = loss(NetworkParams.from_scalars(probe))
        probe[idx] = base[idx] - eps
        lo = loss(NetworkParams.from_scalars(probe))
        fd = (hi - lo) / (2.0 * eps)
        ga = float(analytic[idx])
        scale = max(abs(ga), abs(fd))
        if scale < 1e-12:
            continue
        worst = max(worst, abs(ga - fd) / scale)
    return worst
