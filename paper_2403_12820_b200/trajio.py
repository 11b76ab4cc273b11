"""Frame output and evaluation of rollouts.

* CLT1 trajectory files (io.cpp:375-459): magic "CLT1", u32 version (1 = f64, 2 = f32 payload),
  u32 nx, u32 ny, u32 frames, f64 dt, f64 spacing, then per frame the positions [n][3] and the
  velocities [n][3], little-endian; written through a ``path + ".tmp"`` sibling renamed into
  place (io.cpp:160-182). Reader checks and error texts follow read_trajectory (io.cpp:401-445)
  and read_trajectory_file's "PATH: " prefix (io.cpp:451-459).
* export_obj (io.cpp:463-491) and write_eval_csv (io.cpp:608-619).
* evaluate (eval.cpp:105-133): the per-frame node sums of |x_test - x_ref| run on the GPU
  (sc_evaluate_frames, csrc/eval.cu); the bbox diagonal, the normalisation and the mean are
  the reference's own host expressions.
File I/O is host byte work on numpy views (no per-node Python loops).
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _abi
from .scene import ConfigError, IoError, NumericsError, Trajectory

MAGIC = b"CLT1"
_HEADER = struct.Struct("<4sIIIIdd")  # magic, version, nx, ny, frames, dt, spacing


def _atomic_write(path: str, write) -> None:
    """atomic_write (io.cpp:160-182)."""
    tmp = path + ".tmp"
    try:
        f = open(tmp, "wb")
    except OSError:
        raise IoError("cannot open %s for writing" % tmp) from None
    try:
        with f:
            write(f)
            f.flush()
    except BaseException:
        try:
            os.remove(tmp)
        except OSError:
            pass
        raise
    try:
        os.replace(tmp, path)
    except OSError:
        try:
            os.remove(tmp)
        except OSError:
            pass
        raise IoError("cannot rename %s to %s" % (tmp, path)) from None


def trajectory_bytes_header(traj: Trajectory, version: int) -> bytes:
    return _HEADER.pack(MAGIC, version, traj.nx, traj.ny, traj.frame_count, float(traj.dt),
                        float(traj.spacing))


def write_trajectory(out, traj: Trajectory, version: int = 1) -> None:
    """write_trajectory (io.cpp:375-399) into a binary stream."""
    traj.validate()
    if version not in (1, 2):
        raise IoError("unsupported trajectory version %d" % version)
    out.write(trajectory_bytes_header(traj, version))
    dt = np.dtype("<f8") if version == 1 else np.dtype("<f4")
    # per frame: x block then v block (the reference's field order)
    fx, fv = np.asarray(traj.frames_x), np.asarray(traj.frames_v)
    payload = np.empty((traj.frame_count, 2) + fx.shape[1:], dt)
    payload[:, 0] = fx  # f64 -> f32 is the reference's static_cast (round to nearest)
    payload[:, 1] = fv
    out.write(memoryview(np.ascontiguousarray(payload)).cast("B"))


def save_trajectory(path: str, trajectory: Trajectory, version: int = 1) -> None:
    """write_trajectory_file (io.cpp:447-449; binding save_trajectory, bindings.cpp:139)."""
    _atomic_write(path, lambda f: write_trajectory(f, trajectory, version))


def read_trajectory(buf: bytes) -> Trajectory:
    """read_trajectory (io.cpp:401-445) over the file's bytes."""
    def need(n, what, off):
        if len(buf) - off < n:
            raise IoError("truncated file: expected %d more bytes of %s" % (n, what))

    need(4, "trajectory magic", 0)
    if buf[:4] != MAGIC:
        raise IoError("not a trajectory file (bad magic)")
    need(4, "trajectory version", 4)
    (version,) = struct.unpack_from("<I", buf, 4)
    if version not in (1, 2):
        raise IoError("unsupported trajectory version %d" % version)
    off = 8
    vals = []
    for fmt in ("<I", "<I", "<I", "<d", "<d"):
        need(struct.calcsize(fmt), "trajectory header", off)
        vals.append(struct.unpack_from(fmt, buf, off)[0])
        off += struct.calcsize(fmt)
    nx_u, ny_u, frames, dt, spacing = vals
    nx, ny = np.int32(np.uint32(nx_u)).item(), np.int32(np.uint32(ny_u)).item()  # static_cast<int>
    if nx < 2 or ny < 2 or nx > 65536 or ny > 65536:
        raise IoError("trajectory header: implausible grid %dx%d" % (nx, ny))
    if frames < 1:
        raise IoError("trajectory header: zero frames")
    n = nx * ny
    esize = 8 if version == 1 else 4
    expected = frames * n * 6 * esize
    available = len(buf) - off
    if available < expected:
        raise IoError("truncated trajectory: header declares %d payload bytes, found %d"
                      % (expected, available))
    dt_ = np.dtype("<f8") if version == 1 else np.dtype("<f4")
    payload = np.frombuffer(buf, dt_, count=frames * n * 6, offset=off).reshape(frames, 2, n, 3)
    traj = Trajectory(nx, ny, dt, spacing, payload[:, 0].astype(np.float64),
                      payload[:, 1].astype(np.float64))
    traj.validate()
    return traj


def load_trajectory(path: str) -> Trajectory:
    """read_trajectory_file (io.cpp:451-459; binding load_trajectory, bindings.cpp:141)."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError("cannot open trajectory %s" % path) from None
    try:
        return read_trajectory(buf)
    except IoError as e:
        raise IoError("%s: %s" % (path, e)) from None


def export_obj(path: str, trajectory: Trajectory, frame: int) -> None:
    """export_obj_file (io.cpp:463-491): %.17g vertices, quads split lower-left/upper-right."""
    trajectory.validate()
    if frame < 0 or frame >= trajectory.frame_count:
        raise ConfigError("obj export: frame %d not in [0, %d]"
                          % (frame, trajectory.frame_count - 1))
    x = np.asarray(trajectory.frames_x[frame], np.float64)
    nx, ny = trajectory.nx, trajectory.ny

    def write(f):
        f.write("".join("v %s %s %s\n" % (_g17(p[0]), _g17(p[1]), _g17(p[2]))
                        for p in x.tolist()).encode())
        iy, ix = np.meshgrid(np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
        a = (iy * nx + ix + 1).ravel()
        lines = []
        for av in a.tolist():
            b, c, d = av + 1, av + nx + 1, av + nx
            lines.append("f %d %d %d\nf %d %d %d\n" % (av, b, c, av, c, d))
        f.write("".join(lines).encode())

    _atomic_write(path, write)


def _g17(v: float) -> str:
    return "%.17g" % v


@dataclass
class EvalReport:
    """EvalReport (eval.hpp:19-25; binding bindings.cpp:122-127)."""
    scene_id: str = ""
    checkpoint_id: str = ""
    frame_error_pct: List[float] = field(default_factory=list)
    mean_error_pct: float = 0.0
    final_error_pct: float = 0.0


def write_eval_csv(path: str, report: EvalReport) -> None:
    """write_eval_csv (io.cpp:608-619)."""
    def write(f):
        rows = ["scene,%s" % report.scene_id, "checkpoint,%s" % report.checkpoint_id,
                "frame,error_pct"]
        rows += ["%d,%s" % (i, _g17(e)) for i, e in enumerate(report.frame_error_pct)]
        rows += ["mean,%s" % _g17(report.mean_error_pct), "final,%s" % _g17(report.final_error_pct)]
        f.write(("\n".join(rows) + "\n").encode())

    _atomic_write(path, write)


def bbox_diagonal(x: np.ndarray) -> float:
    """bbox_diagonal (eval.cpp:20-31): |hi - lo| with Vec3::norm's sqrt(x*x + y*y + z*z)."""
    d = np.asarray(x, np.float64).max(axis=0) - np.asarray(x, np.float64).min(axis=0)
    return float(np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]))


def evaluate(test: Trajectory, reference: Trajectory, device: int = 0) -> EvalReport:
    """evaluate_rollout (eval.cpp:105-133; binding evaluate, bindings.cpp:165). The node sums
    run on the GPU in double (a fixed-order tree instead of the reference's left-to-right sum:
    the per-frame value agrees to ~1e-15 relative, see tests/test_gpu_eval.py)."""
    test.validate()
    reference.validate()
    if test.nx != reference.nx or test.ny != reference.ny:
        raise ConfigError("evaluate: trajectories have different grid shapes")
    if test.frame_count != reference.frame_count:
        raise ConfigError("evaluate: trajectories have different frame counts (%d vs %d)"
                          % (test.frame_count, reference.frame_count))
    diag = bbox_diagonal(reference.frames_x[0])
    if not (diag > 0.0):
        raise NumericsError("evaluate: reference frame 0 has a degenerate bounding box")
    frames = test.frame_count
    n = test.nx * test.ny
    a = np.ascontiguousarray(test.frames_x, np.float64)
    b = np.ascontiguousarray(reference.frames_x, np.float64)
    sums = np.empty(frames, np.float64)
    lib = _abi.load()
    st = lib.sc_evaluate_frames(device, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                frames, n, sums.ctypes.data_as(C.c_void_p))
    if st != 0:
        from .api import CudaError
        msg = (lib.sc_eval_last_error() or b"").decode()
        if st == 1:  # SC_ERR_CONFIG
            raise ConfigError(msg)
        raise CudaError(msg)
    rep = EvalReport()
    denom = float(n) * diag
    rep.frame_error_pct = [100.0 * float(s) / denom for s in sums]
    total = 0.0
    for e in rep.frame_error_pct:
        total += e
    rep.mean_error_pct = total / float(len(rep.frame_error_pct))
    rep.final_error_pct = rep.frame_error_pct[-1]
    return rep


# ---- checkpoints (CKP1, io.cpp:495-606) and the loss CSV (io.cpp:596-604) ---------------------

CKP_MAGIC = b"CKP1"
GROUP_NAMES = ("kernel", "linear", "bias", "nonlinear", "deriv", "self_velocity", "alpha")
GROUP_SIZES = (12, 12, 3, 12, 12, 1, 1)


@dataclass
class Checkpoint:
    """Checkpoint (io.hpp:36-45; binding bindings.cpp:129-133): parameters with trainable flags
    and init brackets, the optional Adam state, the step counter and a config echo."""
    params: object = None
    opt: object = None
    step: int = 0
    config_echo: str = ""


def _group_slices():
    out, k = [], 0
    for n in GROUP_SIZES:
        out.append(slice(k, k + n))
        k += n
    return out


def save_checkpoint(path: str, checkpoint: Checkpoint) -> None:
    """save_checkpoint (io.cpp:495-530), atomic write."""
    from .scene import NetworkParams, channel_order_hash

    p = checkpoint.params if checkpoint.params is not None else NetworkParams()
    flat = p.scalars()
    echo = checkpoint.config_echo.encode() if isinstance(checkpoint.config_echo, str) \
        else bytes(checkpoint.config_echo)

    def write(f):
        f.write(CKP_MAGIC)
        f.write(struct.pack("<IQqI", 1, channel_order_hash(), int(checkpoint.step), len(echo)))
        f.write(echo)
        f.write(struct.pack("<I", len(GROUP_NAMES)))
        for g, (name, sl) in enumerate(zip(GROUP_NAMES, _group_slices())):
            lo, hi = p.brackets[g]
            vals = flat[sl]
            f.write(struct.pack("<B", len(name)) + name.encode())
            f.write(struct.pack("<BddI", 1 if p.trainable[g] else 0, float(lo), float(hi), len(vals)))
            f.write(struct.pack("<%dd" % len(vals), *vals))
        o = checkpoint.opt
        f.write(struct.pack("<B", 1 if o is not None else 0))
        if o is not None:
            f.write(struct.pack("<q", int(o.step)))
            f.write(np.ascontiguousarray(o.m, "<f8").tobytes())
            f.write(np.ascontiguousarray(o.v, "<f8").tobytes())

    _atomic_write(path, write)


def load_checkpoint(path: str) -> Checkpoint:
    """load_checkpoint (io.cpp:532-590): every validation and error text of the reference."""
    from .scene import NetworkParams, channel_order_hash
    from .training import AdamState

    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError("cannot open checkpoint %s" % path) from None
    pos = [0]

    def take(fmt, what):
        n = struct.calcsize(fmt)
        if len(buf) - pos[0] < n:
            raise IoError("truncated file: expected %d more bytes of %s" % (n, what))
        v = struct.unpack_from(fmt, buf, pos[0])
        pos[0] += n
        return v[0] if len(v) == 1 else v

    def take_bytes(n, what):
        if len(buf) - pos[0] < n:
            raise IoError("truncated file: expected %d more bytes of %s" % (n, what))
        b = buf[pos[0]:pos[0] + n]
        pos[0] += n
        return b

    try:
        if take_bytes(4, "checkpoint magic") != CKP_MAGIC:
            raise IoError("not a checkpoint file (bad magic)")
        version = take("<I", "checkpoint version")
        if version != 1:
            raise IoError("unsupported checkpoint version %d" % version)
        if take("<Q", "channel order hash") != channel_order_hash():
            raise IoError("checkpoint was written against a different stencil channel ordering")
        ckp = Checkpoint(params=NetworkParams())
        ckp.step = take("<q", "step counter")
        echo_len = take("<I", "config echo length")
        if echo_len > (1 << 20):
            raise IoError("checkpoint config echo implausibly large")
        ckp.config_echo = take_bytes(echo_len, "config echo").decode("utf-8", "surrogateescape")
        groups = take("<I", "group count")
        if groups != len(GROUP_NAMES):
            raise IoError("checkpoint declares %d parameter groups, expected %d"
                          % (groups, len(GROUP_NAMES)))
        flat = [0.0] * 53
        for g, (expected, sl) in enumerate(zip(GROUP_NAMES, _group_slices())):
            name_len = take("<B", "group name length")
            name = take_bytes(name_len, "group name").decode("utf-8", "surrogateescape")
            if name != expected:
                raise IoError('checkpoint group %d is "%s", expected "%s"' % (g, name, expected))
            ckp.params.trainable[g] = take("<B", "trainable flag") != 0
            lo = take("<d", "bracket")
            hi = take("<d", "bracket")
            ckp.params.brackets[g] = (lo, hi)
            count = take("<I", "group scalar count")
            if count != GROUP_SIZES[g]:
                raise IoError('checkpoint group "%s" has %d scalars, expected %d'
                              % (name, count, GROUP_SIZES[g]))
            vals = take_bytes(8 * count, "group scalars")
            flat[sl] = list(struct.unpack("<%dd" % count, vals))
        trainable, brackets = ckp.params.trainable, ckp.params.brackets
        ckp.params = NetworkParams.from_scalars(flat)
        ckp.params.trainable, ckp.params.brackets = trainable, brackets
        if not (ckp.params.isru_alpha > 0.0):
            raise IoError("checkpoint isru_alpha must be > 0")
        if take("<B", "optimizer flag") != 0:
            step = take("<q", "optimizer step")
            m = np.frombuffer(take_bytes(8 * 53, "optimizer moments"), "<f8").copy()
            v = np.frombuffer(take_bytes(8 * 53, "optimizer moments"), "<f8").copy()
            ckp.opt = AdamState(m, v, step)
        return ckp
    except IoError as e:
        raise IoError("%s: %s" % (path, e)) from None


def write_loss_csv(path: str, rows) -> None:
    """write_loss_csv (io.cpp:596-604): rows of LossRow or (step, lr, physics, data, total)."""
    def write(f):
        lines = ["step,lr,physics,data,total"]
        for r in rows:
            t = (r.step, r.lr, r.physics, r.data, r.total) if hasattr(r, "step") else tuple(r)
            lines.append("%d,%s,%s,%s,%s" % (int(t[0]), _g17(t[1]), _g17(t[2]), _g17(t[3]),
                                             _g17(t[4])))
        f.write(("\n".join(lines) + "\n").encode())

    _atomic_write(path, write)
