"""Data-parallel training across ranks, bit-identical to one device ("a batch
of independent transitions is truly data-parallel ... a deterministic fixed-order reduction of
53 gradient sums").

Each rank holds the scene and the whole trajectory and computes a contiguous share of every
batch's transitions ("part", `CudaPart` over the sc_trainer_part_* C-ABI). compute_loss
(train.cpp:129-209) is then combined so the result does not depend on the number of ranks:

  * data count:  all-reduce of integers (exact);
  * loss sums:   the reference's single left-to-right chain, run part after part (rank r starts
                 from rank r-1's running sums: a hand-over of two doubles, not a reduction);
  * gradients:   every rank's per-transition totals are all-gathered and summed in transition
                 order on every rank — the reference's grads->add_scaled(g, 1.0) loop — instead
                 of an all-reduce, whose association order would depend on the world size;
  * errors:      the first failing transition over all parts, with the reference's precedence.

`DistributedTrainer.run` restates train_loop (train.cpp:212-375: DE pre-search, schedule, Adam)
on the host around that compute_loss; with one rank it reproduces `Trainer.run` / the reference's
train_loop bit for bit. The part object is pluggable (the CPU tests drive the same orchestration
over gloo with a test-side part built on the oracle).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import List, Optional, Sequence

import numpy as np

from .api import _ptr, _raise
from .scene import ConfigError, NetworkParams, NumericsError, ParamGroup
from .training import (AdamState, LossRow, LossValue, ParamGradients, Rng, TrainConfig,
                       TrainResult, Trainer, sample_indices)

K_DE_STREAM = 0xDE5EA4C400000001
K_PROBE_STREAM = 0xDE5EA4C400000002
BETA1, BETA2, EPS = 0.9, 0.999, 1e-8


class CudaPart:
    """One rank's share of compute_loss on its GPU (sc_trainer_part_*)."""

    def __init__(self, scene, trajectory, device: int = 0):
        self.t = Trainer(scene, trajectory, device)
        self.lib = self.t.lib
        self.frames = trajectory.frame_count
        self.n_free = scene.nx * scene.ny - len(scene.bc.nodes)

    def set_batch(self, indices: Sequence[int]) -> None:
        self.t.set_batch(indices)

    def forward(self, params: NetworkParams, b0: int, b1: int):
        cnt = C.c_uint64()
        bad = np.full(2, -1, np.int32)
        pc = params.to_c()
        _raise(self.lib, self.lib.sc_trainer_part_forward(self.t.h, C.byref(pc), b0, b1,
                                                          C.byref(cnt), _ptr(bad)))
        return int(cnt.value), int(bad[0]), int(bad[1])

    def chain(self, ps: float, ds: float):
        sin = np.array([ps, ds])
        sout = np.zeros(2)
        bad = np.full(1, -1, np.int32)
        _raise(self.lib, self.lib.sc_trainer_part_chain(self.t.h, _ptr(sin), _ptr(sout), _ptr(bad)))
        return float(sout[0]), float(sout[1]), int(bad[0])

    def backward(self, params: NetworkParams, alpha: float, count: int, batch: int, nb: int):
        out = np.zeros((nb, 53))
        pc = params.to_c()
        _raise(self.lib, self.lib.sc_trainer_part_backward(self.t.h, C.byref(pc), float(alpha),
                                                           int(count), int(batch), _ptr(out)))
        return out

    def diagnose(self, params: NetworkParams, frame: int, node: int) -> str:
        buf = C.create_string_buffer(256)
        pc = params.to_c()
        _raise(self.lib, self.lib.sc_trainer_diagnose_forward(self.t.h, C.byref(pc), int(frame),
                                                              int(node), buf, 256))
        return buf.value.decode()

    def close(self) -> None:
        self.t.close()


class _Comm:
    """The few exchanges compute_loss needs, over a torch.distributed group (or none)."""

    def __init__(self, group=None):
        self.group = group
        try:
            import torch.distributed as dist
            self.dist = dist if dist.is_available() and dist.is_initialized() else None
        except ImportError:
            self.dist = None
        if self.dist is None:
            self.rank, self.world = 0, 1
        else:
            self.rank = self.dist.get_rank(group)
            self.world = self.dist.get_world_size(group)
        self.device = "cpu"
        if self.dist is not None and self.dist.get_backend(group) == "nccl":
            import torch
            self.device = torch.device("cuda", torch.cuda.current_device())

    def _t(self, values, dtype):
        import torch
        return torch.tensor(values, dtype=dtype, device=self.device)

    def _g(self, r: int) -> int:  # group rank -> global rank
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def sum_int(self, v: int) -> int:
        if self.world == 1:
            return v
        import torch
        t = self._t([v], torch.int64)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def gather_pairs(self, a: int, b: int) -> List[tuple]:
        if self.world == 1:
            return [(a, b)]
        import torch
        t = self._t([a, b], torch.int64)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [(int(x[0]), int(x[1])) for x in out]

    def chain(self, run):
        """Run `run(ps, ds) -> (ps, ds, bad)` rank after rank; everyone gets the final triple."""
        if self.world == 1:
            return run(0.0, 0.0)
        import torch
        state = self._t([0.0, 0.0, -1.0], torch.float64)
        if self.rank > 0:
            self.dist.recv(state, src=self._g(self.rank - 1), group=self.group)
        ps, ds, bad = float(state[0]), float(state[1]), int(state[2])
        if bad < 0:
            ps, ds, bad = run(ps, ds)
        state = self._t([ps, ds, float(bad)], torch.float64)
        if self.rank < self.world - 1:
            self.dist.send(state, dst=self._g(self.rank + 1), group=self.group)
        self.dist.broadcast(state, src=self._g(self.world - 1), group=self.group)
        return float(state[0]), float(state[1]), int(state[2])

    def gather_rows(self, rows: np.ndarray, counts: List[int]) -> np.ndarray:
        """Concatenate every rank's [k_r, 53] block in rank order."""
        if self.world == 1:
            return rows
        import torch
        width = max(counts)
        t = torch.zeros((width, rows.shape[1]), dtype=torch.float64, device=self.device)
        if len(rows):
            t[:len(rows)] = torch.from_numpy(rows).to(self.device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return np.concatenate([o[:c].cpu().numpy() for o, c in zip(out, counts)], axis=0)


class DistributedTrainer:
    """compute_loss and train_loop over the ranks of `group` (each with its own part)."""

    def __init__(self, part, group=None):
        self.part = part
        self.comm = _Comm(group)
        self.indices: List[int] = []

    def _span(self, B: int, r: int):
        w = self.comm.world
        return r * B // w, (r + 1) * B // w

    def set_batch(self, indices: Sequence[int]) -> None:
        self.indices = [int(i) for i in indices]
        self.part.set_batch(self.indices)

    def compute_loss(self, params: NetworkParams, alpha: float, grads: bool = True):
        """compute_loss (train.cpp:129-209) of the current batch, identical on every rank."""
        if not (params.isru_alpha > 0.0):
            raise ConfigError("isru_alpha: must be > 0")
        B = len(self.indices)
        if B == 0:
            raise ConfigError("compute_loss: empty batch")
        b0, b1 = self._span(B, self.comm.rank)
        if b1 > b0:
            cnt, bad_b, bad_node = self.part.forward(params, b0, b1)
        else:
            cnt, bad_b, bad_node = 0, -1, -1
        count = self.comm.sum_int(cnt)
        fwd = [pr for pr in self.comm.gather_pairs(bad_b, bad_node) if pr[0] >= 0]
        bf, bnode = min(fwd) if fwd else (-1, -1)
        ps, ds, bl = self.comm.chain(
            lambda p, d: self.part.chain(p, d) if b1 > b0 else (p, d, -1))
        # element b's forward_impulse throws before b's loss check (train.cpp:146-182)
        if bf >= 0 and (bl < 0 or bf <= bl):
            raise NumericsError(self.part.diagnose(params, self.indices[bf], bnode))
        if bl >= 0:
            raise NumericsError("non-finite loss at batch element %d (frame %d)"
                                % (bl, self.indices[bl]))
        free = self.part.n_free
        phys_denom = 3.0 * float(B) * free
        data_denom = 6.0 * float(count)
        physics = ps / phys_denom if free > 0 else 0.0
        data = ds / data_denom if count > 0 else 0.0
        loss = LossValue(alpha * physics + (1.0 - alpha) * data, physics, data)
        if not grads:
            return loss, None
        local = (self.part.backward(params, alpha, count, B, b1 - b0) if b1 > b0
                 else np.zeros((0, 53)))
        counts = [self._span(B, r)[1] - self._span(B, r)[0] for r in range(self.comm.world)]
        per_b = self.comm.gather_rows(local, counts)
        g = [0.0] * 53
        for row in per_b.tolist():  # grads->add_scaled(g_b, 1.0) in transition order
            g = [g[s] + row[s] * 1.0 for s in range(53)]
        return loss, ParamGradients(np.array(g))

    # ---- train_loop (train.cpp:54-63, 212-375) on the host ----------------------------------
    @staticmethod
    def _validate(cfg: TrainConfig, transitions: int) -> None:
        def bad(m):
            raise ConfigError(m)
        s, d = cfg.schedule, cfg.de
        if not (0.0 <= cfg.alpha <= 1.0):
            bad("train.alpha: must be in [0, 1]")
        if cfg.batch_size < 1:
            bad("train.batch_size: must be >= 1")
        if cfg.batch_size > transitions:
            bad("train.batch_size: exceeds the %d available transitions" % transitions)
        if cfg.epochs < 1:
            bad("train.epochs: must be >= 1")
        if not (s.lr0 > 0.0):
            bad("train.lr0: must be > 0")
        if not (0.0 < s.gamma <= 1.0):
            bad("train.gamma: must be in (0, 1]")
        if s.interval < 1:
            bad("train.interval: must be >= 1")
        if s.period < 1:
            bad("train.period: must be >= 1")
        if not (s.floor >= 0.0):
            bad("train.floor: must be >= 0")
        if d.population < 4:
            bad("train.de.population: must be >= 4")
        if d.generations < 0:
            bad("train.de.generations: must be >= 0")
        if not (d.bound > 0.0):
            bad("train.de.bound: must be > 0")
        if not (0.0 <= d.cross_prob <= 1.0):
            bad("train.de.cross_prob: must be in [0, 1]")
        if not (0.0 < d.diff_weight <= 2.0):
            bad("train.de.diff_weight: must be in (0, 2]")
        if d.probe_batch < 1:
            bad("train.de.probe_batch: must be >= 1")
        if cfg.checkpoint_interval < 1:
            bad("train.checkpoint_interval: must be >= 1")

    @staticmethod
    def _lr(cfg: TrainConfig, step: int) -> float:
        s = cfg.schedule
        if int(s.kind) == 0:
            return s.lr0 * math.pow(s.gamma, float(step // s.interval))
        if step >= s.period:
            return s.floor
        return s.floor + (s.lr0 - s.floor) * 0.5 * (1.0 + math.cos(math.pi * step / s.period))

    @staticmethod
    def _adam(p: NetworkParams, grads: ParamGradients, opt: AdamState, lr: float) -> None:
        opt.step += 1
        c1 = 1.0 - math.pow(BETA1, float(opt.step))
        c2 = 1.0 - math.pow(BETA2, float(opt.step))
        flat = p.scalars()
        groups = [0] * 12 + [1] * 12 + [2] * 3 + [3] * 12 + [4] * 12 + [5, 6]
        for s in range(53):
            if not p.trainable[groups[s]]:
                continue
            g = float(grads.flat[s])
            opt.m[s] = BETA1 * opt.m[s] + (1.0 - BETA1) * g
            opt.v[s] = BETA2 * opt.v[s] + (1.0 - BETA2) * g * g
            m_hat = opt.m[s] / c1
            v_hat = opt.v[s] / c2
            flat[s] -= lr * m_hat / (math.sqrt(v_hat) + EPS)
        q = NetworkParams.from_scalars(flat)
        p.kernel_gain, p.linear_w, p.linear_b = q.kernel_gain, q.linear_w, q.linear_b
        p.nonlinear_w, p.deriv_w = q.nonlinear_w, q.deriv_w
        p.self_velocity_w, p.isru_alpha = q.self_velocity_w, q.isru_alpha

    @staticmethod
    def _decode(z):
        def scale(v):
            return (1.0 if v >= 0.0 else -1.0) * math.pow(10.0, abs(v) - 2.0)
        return (scale(z[0]), scale(z[1]), scale(z[2]), scale(z[3]), scale(z[4]),
                math.pow(10.0, z[5] / 2.0))

    def _de_preprocess(self, cfg: TrainConfig, rng: Rng) -> NetworkParams:
        transitions = self.part.frames - 1
        probe = sample_indices(self.part.frames, min(cfg.de.probe_batch, transitions),
                               Rng.mix(cfg.seed, K_PROBE_STREAM))
        self.set_batch(probe)

        def objective(z):
            lin, bias, non, der, selfv, alpha = self._decode(z)
            p = NetworkParams()
            p.linear_w = np.full(12, lin)
            p.linear_b = np.full(3, bias)
            p.nonlinear_w = np.full(12, non)
            p.deriv_w = np.full(12, der)
            p.self_velocity_w = selfv
            p.isru_alpha = alpha
            try:
                return self.compute_loss(p, cfg.alpha, grads=False)[0].total
            except NumericsError:
                return 1e300

        dim, bound, pop_n = 6, cfg.de.bound, cfg.de.population
        lo, hi = [-bound] * dim, [bound] * dim
        seed = [[-bound + (float(rng.uniform_below(6)) + 0.5) * (2.0 * bound / 6.0)
                 for _ in range(dim)] for _ in range(pop_n)]
        clamp = (lambda v, a, b: a if v < a else (b if b < v else v))
        pop = [[clamp(seed[p][d], lo[d], hi[d]) for d in range(dim)] for p in range(pop_n)]
        value = [objective(pop[p]) for p in range(pop_n)]
        for _ in range(cfg.de.generations):
            for p in range(pop_n):
                a = rng.uniform_below(pop_n)
                while a == p:
                    a = rng.uniform_below(pop_n)
                b = rng.uniform_below(pop_n)
                while b == p or b == a:
                    b = rng.uniform_below(pop_n)
                c = rng.uniform_below(pop_n)
                while c == p or c == a or c == b:
                    c = rng.uniform_below(pop_n)
                forced = rng.uniform_below(dim)
                trial = [0.0] * dim
                for d in range(dim):
                    if rng.uniform01() < cfg.de.cross_prob or d == forced:
                        trial[d] = clamp(pop[a][d] + cfg.de.diff_weight * (pop[b][d] - pop[c][d]),
                                         lo[d], hi[d])
                    else:
                        trial[d] = pop[p][d]
                tv = objective(trial)
                if tv <= value[p]:
                    pop[p], value[p] = trial, tv
        best = 0
        for p in range(1, pop_n):
            if value[p] < value[best]:
                best = p
        lin, bias, non, der, selfv, alpha = self._decode(pop[best])

        def bracket(v):
            w = max(abs(v), 0.05)
            return (v - w, v + w)
        params = NetworkParams()
        ab = bracket(alpha)
        params.brackets = [(1.0, 1.0), bracket(lin), bracket(bias), bracket(non), bracket(der),
                           bracket(selfv), (max(ab[0], 1e-3), ab[1])]
        params.isru_alpha = alpha
        flat = params.scalars()
        groups = [0] * 12 + [1] * 12 + [2] * 3 + [3] * 12 + [4] * 12 + [5, 6]
        for s in range(53):
            g = groups[s]
            if params.trainable[g]:
                flat[s] = rng.uniform(*params.brackets[g])
        q = NetworkParams.from_scalars(flat)
        q.brackets = params.brackets
        return q

    def run(self, cfg: TrainConfig, resume: Optional[TrainResult] = None) -> TrainResult:
        """train_loop (train.cpp:343-375) with the data-parallel compute_loss."""
        self._validate(cfg, self.part.frames - 1)
        if resume is not None:
            params = resume.params.copy()
            opt = AdamState(np.array(resume.opt.m, dtype=np.float64),
                            np.array(resume.opt.v, dtype=np.float64), int(resume.opt.step))
        else:
            params = self._de_preprocess(cfg, Rng(Rng.mix(cfg.seed, K_DE_STREAM)))
            opt = AdamState()
        for g in cfg.freeze:
            params.trainable[int(g)] = False
        opt.m = [float(v) for v in opt.m]
        opt.v = [float(v) for v in opt.v]
        start = opt.step
        history: List[LossRow] = []
        for e in range(cfg.epochs):
            step = start + e
            lr = self._lr(cfg, step)
            self.set_batch(sample_indices(self.part.frames, cfg.batch_size,
                                          Rng.mix(cfg.seed, step)))
            try:
                loss, grads = self.compute_loss(params, cfg.alpha)
            except NumericsError as err:
                raise NumericsError("%s [optimizer step %d]" % (err, step)) from None
            self._adam(params, grads, opt, lr)
            history.append(LossRow(step, lr, loss.physics, loss.data, loss.total))
        opt.m, opt.v = np.array(opt.m), np.array(opt.v)
        return TrainResult(params, opt, history)
