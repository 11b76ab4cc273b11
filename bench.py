#!/usr/bin/env python
"""Throughput of the network-cell rollout step (arXiv 2403.12820 reference path) on B200.

Metric (BASELINE.json): cloth node-updates/s (nodes x timesteps / s), whole job over all GPUs,
and the fraction of the HBM roofline (48 algorithmic bytes per node-update: fp32 x and v read
once and written once per timestep).

Workload: BASELINE config 5 by default — 4096 independent 128x128 cloths, mixed boundary
conditions (top row pinned / two top corners / free onto the plane z = -0.5), gravity + per-cloth
wind, dt = 1/240, 300 timesteps, the reference's 12-channel cell with N(0, 0.05) weights
(SURVEY.md §8(d) mapping); it is the largest single-GPU config and the one BASELINE quotes its
1/2/4/8-GPU sweep on. `--config 2|3|4|1` runs the others. One bench "step" = one timestep of
the whole batch; the K timed steps run device-resident (config 5: one wavefront launch that
advances all K timesteps, csrc/wave_kernels.cu, beside the streaming launches of its plane
cloths; config 1: one small-cloth launch, csrc/small_kernels.cu).

Multi-GPU (one process per GPU): configs 2 and 5 shard the fixed batch B/G per rank (strong
scaling, no data-path collective; `--scaling weak` gives every rank the whole batch instead),
config 4 splits its 8192^2 cloth into row strips with a 2-row halo exchange per step over NCCL;
configs 1 and 3 are replicas only. `--gpus N` without an outer torchrun spawns the N ranks
itself and fails when fewer GPUs are visible.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the unmodified
reference sources, benchmark_net's own timer) on all host cores, on bounded samples of the same
config, with inputs built on the checker side (oracle/workloads.py: the product library is never
loaded); under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_NODE_UPDATE = 48  # fp32 x, v: 24 B read + 24 B written per node per timestep
DEFAULT_CONFIG = 5
# config.workload of both arms (ours and --impl reference print the same string; the reference
# arm never imports the product package, tests/test_bench_cli.py keeps this table and
# paper_2403_12820_b200.configs in step)
WORKLOAD_LABEL = {
    1: "cfg1: 1 x 32^2, two top corners pinned, gravity, 100 steps, hidden 8 (3x3)",
    2: "cfg2: 64 x 256^2, top row pinned, gravity + wind, 1000 steps",
    3: "cfg3: 1 x 1024^2, two corners pinned, sphere R=0.3 under the cloth, 500 steps",
    4: "cfg4: 1 x 8192^2, top row pinned, gravity, 200 steps",
    5: "cfg5: 4096 x 128^2, mixed BCs (top row / corners / free onto plane z=-0.5), wind",
}
WORKLOAD_KEY = {1: "cfg1_32x32", 2: "cfg2_64x256x256", 3: "cfg3_1024x1024", 4: "cfg4_8192x8192",
                5: "cfg5_4096x128x128"}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons during the timed region: one NVML sample when the region
    opens, one every 10 ms from a thread while it runs, one when it closes (so even a region
    shorter than the sampling period is covered); nvidia-smi polling when NVML is unavailable."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, set(reasons))
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._max = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def sample(self):
        if self._nv is not None:
            nv = self._nv
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                active = {name for name, const in self.REASONS if r & getattr(nv, const)}
                self.samples.append((float(sm), self._max, active))
                return
            except Exception:
                pass
        try:
            out = subprocess.run(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            v = [x.strip() for x in out.stdout.strip().split(",")]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            self.samples.append((float(v[0]), float(v[1]),
                                 {names[i] for i in range(4) if v[2 + i].lower() == "active"}))
        except Exception:
            pass

    def _run(self):
        while not self._stop.wait(0.01 if self._nv is not None else 0.2):
            self.sample()

    def __enter__(self):
        self.sample()
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        self.sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_min_mhz": min(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*[s[2] for s in self.samples])),
                "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "0"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# Test hook (never a measurement): SC_BENCH_SHARE_GPU=1 runs every rank on GPU 0 with a gloo
# process group, so the multi-rank path (batch shares, barriers, max over ranks, rank-0 output)
# can be exercised on a one-GPU box (tests/test_gpu_bench_ranks.py). Batch-sharded and replica
# configs only: their ranks never wait on each other's kernels. The line says "shared_gpu".
SHARE_GPU = os.environ.get("SC_BENCH_SHARE_GPU") == "1"


def _spawn(args) -> int:
    """--gpus N without an outer torchrun: launch the N ranks ourselves (same arguments)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and not SHARE_GPU:
        print(json.dumps({"error": "bench.py --gpus %d: only %d GPU(s) visible; refusing to "
                          "measure fewer ranks than asked" % (args.gpus, have)}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=%d" % args.gpus, "--master-addr=127.0.0.1",
           "--master-port=%d" % _free_port(), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _traffic(kernel: str, workload: str, steps: int):
    """DRAM bytes per node-update of the dominant kernel from the committed ncu capture
    (profiles/traffic.json: the bench's own launch). For the wavefront kernel the state crosses
    HBM once per pass of W timesteps, so the capture's bytes per (node x pass) are rescaled to
    this launch's ceil(K / W) passes."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get("%s:%s" % (kernel, workload))
        if not e:
            return None, None
        if kernel == "wave_kernel":
            W = e["levels"]
            per_node_pass = e["dram_bytes"] / (e["nodes"] * -(-e["steps"] // W))
            return per_node_pass * -(-steps // W) / steps, e.get("source")
        return e["dram_bytes"] / e["node_updates"], e.get("source")
    except Exception:
        return None, None


def _cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ reference CPU path ------
_REF_INPUTS = {}


def reference_sample(ref, cid: int, cores: int, steps: int, warmup: int = 1):
    """benchmark_net (eval.cpp:155-158) on a bounded sample of config `cid`, inputs from the
    checker-side generator (oracle/workloads.py). Batched configs: `cores` cloths, one
    std::thread each (the cloth-parallel variant: reference code unchanged, global thread count
    1). Single-cloth configs: the one cloth, node-parallel on `cores` threads (the reference's
    own parallel_for). Returns (node-updates, seconds, description)."""
    from oracle import workloads as W
    import numpy as np

    w = W.WORKLOADS[cid]
    if cid not in _REF_INPUTS:
        nb = cores if w.batch > 1 else 1
        # no plane collider in the reference (io.cpp:321-322): config 5's free cloths fall freely
        _, cds, keep, pc, x, v = W.build(cid, batch=nb, plane=False)
        _REF_INPUTS[cid] = (cds, keep, pc, np.ascontiguousarray(x, np.float64),
                            np.ascontiguousarray(v, np.float64))
    cds, _, pc, x64, v64 = _REF_INPUTS[cid]
    n = w.n
    if w.batch > 1:
        mx, _ = ref.benchmark_net_cloth_parallel(n, n, cds, pc, x64, v64, steps, warmup)
        return len(cds) * n * n * steps, mx, "%d cloths x %d timesteps, cloth-parallel" % (
            len(cds), steps)
    sec = ref.benchmark_net(n, n, cds[0], pc, x64[0], v64[0], steps, warmup, threads=cores)
    return n * n * steps, sec, "1 cloth x %d timesteps, node-parallel on %d threads" % (steps, cores)


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from oracle.pyoracle import REF_SO, Reference
    from oracle import workloads as W

    cid = args.config
    w = W.WORKLOADS[cid]
    if not os.path.exists(REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
        return 0
    ref = Reference()
    cores = _cpu_cores()
    n0, s0, _ = reference_sample(ref, cid, cores, 1, 0)
    per_ts = s0
    per_step = args.ref_budget / max(1, args.steps + args.warmup)
    ts = max(1, min(w.steps, int(per_step / max(per_ts, 1e-6))))
    for _ in range(args.warmup):
        reference_sample(ref, cid, cores, ts, 0)
    total_nodes, total_sec = 0, 0.0
    desc = ""
    for _ in range(args.steps):
        n, sec, desc = reference_sample(ref, cid, cores, ts, 0)
        total_nodes += n
        total_sec += sec
    value = total_nodes / total_sec
    sample = ("each step: %s of config %d (%dx%d), reference benchmark_net timer%s"
              % (desc, cid, w.n, w.n, "; free cloths without the plane collider (the reference "
                 "has none)" if cid == 5 else ""))
    line = {
        "impl": "reference", "metric": "cloth node-updates/s", "value": value,
        "unit": "node-updates/s", "n_gpus": max(world, args.gpus), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total_sec / args.steps,
        "higher_is_better": True, "scaling": "strong" if cid in (2, 4, 5) else "replicas",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_LABEL[cid], "grid": "%dx%d" % (w.n, w.n),
                   "sample_per_step": desc,
                   "sample_of": "a bounded sample of the same workload per step (every cloth and "
                                "timestep of it costs the same; its full size takes minutes per "
                                "rollout on the CPU)",
                   "parallelism": "cpu, %d host threads" % cores},
        "cpu_baseline": {"value": value, "unit": "node-updates/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "node-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(cid: int, seconds: float):
    """The reference CPU path timed on this host (rank 0, N = 1), a ~`seconds` sample."""
    try:
        from oracle.pyoracle import Reference
        ref = Reference()
        cores = _cpu_cores()
        _, s0, _ = reference_sample(ref, cid, cores, 1, 1)
        ts = max(1, min(4000, int(seconds / max(s0, 1e-6))))
        n, s, desc = reference_sample(ref, cid, cores, ts, 1)
        return {"value": n / s, "unit": "node-updates/s", "cores": cores, "kind": "reference",
                "sample": "%s of config %d, reference benchmark_net timer, %.1f s%s" % (
                    desc, cid, s, "; free cloths without the plane (none in the reference)"
                    if cid == 5 else "")}
    except Exception as e:  # the box may lack the prebuilt reference library
        return {"value": None, "unit": "node-updates/s", "cores": _cpu_cores(),
                "kind": "reference", "sample": "unavailable: %s" % e}


# ------------------------------------------------------------------ our GPU path ------------
def _e2e_batch(cb, x, v, steps, barrier, max_over_ranks, calls):
    """The reference-facing C-ABI call with host buffers: sc_rollout of `steps` timesteps from
    pinned host x0/v0 to host x/v (H2D + steps + D2H inside the timed region)."""
    import ctypes as C

    import numpy as np

    from paper_2403_12820_b200 import _abi

    lib = _abi.load()
    nbytes = x.nbytes
    bufs = []
    for _ in range(4):
        ptr = C.c_void_p()
        assert lib.sc_host_alloc(nbytes, C.byref(ptr)) == 0
        bufs.append(ptr)
    arrs = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), shape=x.shape) for p in bufs]
    arrs[0][...] = x
    arrs[1][...] = v
    rc = lib.sc_rollout(cb.h, bufs[0], bufs[1], 2, 0, 1, bufs[2], bufs[3], None)  # warm
    assert rc == 0, lib.sc_last_error()
    barrier()
    t = []
    for _ in range(calls):
        t0 = time.perf_counter()
        rc = lib.sc_rollout(cb.h, bufs[0], bufs[1], steps, 0, 1, bufs[2], bufs[3], None)
        t.append(time.perf_counter() - t0)
        assert rc == 0, lib.sc_last_error()
    barrier()
    sec = max_over_ranks(min(t))
    finite = bool(np.isfinite(arrs[2]).all() and np.isfinite(arrs[3]).all())
    for p in bufs:
        lib.sc_host_free(p)
    return sec, 2 * nbytes, 2 * nbytes, finite


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2403_12820_b200 import ClothBatch, configs, strips

    if SHARE_GPU and args.config == 4 and world > 1:
        print(json.dumps({"error": "SC_BENCH_SHARE_GPU: config 4's row strips exchange halos "
                          "over NCCL; not on a shared GPU"}), flush=True)
        return 2
    dev = 0 if SHARE_GPU else local
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if SHARE_GPU else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    cid = args.config
    cfg = configs.CONFIGS[cid]
    K = args.steps
    mode = args.mode
    peak, peak_src = _peaks()
    extra = {}
    if cid != 4 or world == 1:
        # ---- independent cloths: a B/G shard per rank (strong), the whole batch per rank (weak),
        # or replicas of a single-cloth config ----
        if cfg.batch > 1 and args.scaling == "strong":
            b0, b1 = cfg.batch * rank // world, cfg.batch * (rank + 1) // world
            scaling = "strong"
        elif cid == 4:  # N = 1: the whole 8192^2 cloth in one context (strips only for N > 1)
            b0, b1 = 0, 1
            scaling = "strong"
        else:
            b0, b1 = (cfg.batch * rank, cfg.batch * (rank + 1)) if cfg.batch > 1 else (0, 1)
            scaling = "weak" if cfg.batch > 1 else "replicas"
        B = b1 - b0
        _, scenes, params, x, v = configs.build(cid, batch=B, cloth0=b0, threads=16)
        nodes_rank = B * cfg.n * cfg.n
        cb = ClothBatch(scenes, params, device=dev)
        cb.set_state(x, v)
        cb.advance(args.warmup, 0, mode)
        cb.sync()
        barrier()
        launches0 = cb.launch_count()
        nvtx = os.environ.get("SC_BENCH_NVTX") == "1"  # ncu --replay-mode range capture
        with ClockSampler(dev) as clocks:
            # CUDA events on the context stream around exactly the K timed timesteps
            if nvtx:
                torch.cuda.nvtx.range_push("bench_timed")
            sec = cb.benchmark(K, 0, mode)
            if nvtx:
                torch.cuda.synchronize()
                torch.cuda.nvtx.range_pop()
        launches = cb.launch_count() - launches0
        barrier()
        sec_max = max_over_ranks(sec)
        n_coll = sum(1 for s in scenes if s.colliders or s.planes)
        if mode != "fast":
            kernel = "parity_kernel"
        elif launches == 1:
            # one launch for all K timesteps: the small-cloth kernel (<= 1024 nodes per cloth,
            # csrc/small_kernels.cu) or the wavefront kernel (nx <= 128, csrc/wave_kernels.cu)
            kernel = "small_kernel" if cfg.n * cfg.n <= 1024 else "wave_kernel"
        elif launches == K + 1 and 0 < n_coll < B:
            kernel = "wave_kernel+fast_step_kernel"  # class groups, concurrent (capi.cu)
        else:
            kernel = "fast_step_kernel"
        region_nu = nodes_rank * K
        cb.set_state(x, v)
        ps = max(3, min(K, 10))
        extra["parity_mode"] = {
            "value": world * nodes_rank * ps / cb.benchmark(ps, 1, "parity") if scaling != "replicas"
            else nodes_rank * ps / cb.benchmark(ps, 1, "parity"),
            "unit": "node-updates/s", "note": "bit-exact with the reference f32 templates"}
        # one user call = one rollout of the config's own length (the reference's rollout /
        # benchmark_net call on this workload), whatever K the device-timed region uses
        T = cfg.steps
        e2e_sec, hb, db, finite = _e2e_batch(cb, x, v, T, barrier, max_over_ranks, args.e2e_calls)
        total_nodes = world * nodes_rank if scaling != "replicas" else nodes_rank
        if scaling == "strong":
            total_nodes = cfg.batch * cfg.n * cfg.n
        e2e = {"value": total_nodes * T / e2e_sec, "unit": "node-updates/s",
               "h2d_bytes_per_step": hb / T, "d2h_bytes_per_step": db / T,
               "call": "sc_rollout host->host, one rollout of the config's %d timesteps per call "
                       "(pinned buffers; per-step bytes = the state's in / out over %d)" % (T, T),
               "finite": finite}
        cb.close()
        assert WORKLOAD_LABEL[cid] == "cfg%d: %s" % (cid, cfg.description)
        conf = {"workload": WORKLOAD_LABEL[cid], "cloths": cfg.batch,
                "cloths_per_gpu": B, "grid": "%dx%d" % (cfg.n, cfg.n), "nodes_per_gpu": nodes_rank,
                **({"shared_gpu": "test hook: every rank on GPU 0 (not a measurement)"}
                   if SHARE_GPU and world > 1 else {}),
                "timesteps_per_step": 1, "mode": mode,
                "timed_window": "%d timesteps, %.1f ms%s" % (
                    K, 1e3 * sec, " (below the ~50 ms after which HBM-bound streaming steps meet "
                    "the board's power cap; the config's own %d-step rollout, e2e, takes the "
                    "temporally blocked kernel)" % cfg.steps if kernel == "fast_step_kernel"
                    and cid == 5 else ""),
                "l2": "no flush: state %.1f MB per GPU%s" % (
                    24e-6 * nodes_rank, " > 126 MB L2" if 24e-6 * nodes_rank > 126 else
                    " (L2-resident: configs 1/3 are small by definition)"),
                "parallelism": ("one GPU, whole cloth" if cid == 4 else
                                "dp%d: %d cloths per GPU, no collective" % (world, B)
                                if scaling != "replicas" else "replicas only (one cloth)")}
    else:
        # ---- one 8192^2 cloth in row strips, halo rows over NCCL each step ----
        scaling = "strong"
        row0, rows = strips.strip_bounds(cfg.n, world, rank)
        g0, g1 = strips.local_window(cfg.n, row0, rows)
        xl, _ = configs.sheet(cfg.seed, 0, cfg.n, g0, g1 - g0)
        scene = configs.make_scene(cfg, 0, xl.astype(np.float64), row0=g0)
        params = configs.make_params(cfg.seed, cfg.hidden8)
        sr = strips.StripRollout(scene, params, xl, np.zeros_like(xl), rank, world, local,
                                 mode=mode, transport=args.transport if mode == "fast" else "nccl")
        nodes_rank = rows * cfg.n
        total_nodes = cfg.n * cfg.n
        for k in range(args.warmup):
            sr.step(k)
        sr.stream.synchronize()
        barrier()
        l0 = sr.ctx.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clocks:
            ev0.record(sr.stream)
            for k in range(args.warmup, args.warmup + K):
                sr.step(k)
            ev1.record(sr.stream)
            ev1.synchronize()
        launches = sr.ctx.launch_count() - l0
        barrier()
        sec = ev0.elapsed_time(ev1) * 1e-3
        sec_max = max_over_ranks(sec)
        kernel = "fast_step_kernel" if mode == "fast" else "parity_kernel"
        region_nu = nodes_rank * K
        n_coll, B = 0, 1
        barrier()
        T = cfg.steps  # one rollout of the config's own length per call, as for N = 1
        t0 = time.perf_counter()
        sr.ctx.set_state(xl, np.zeros_like(xl))
        for k in range(T):
            sr.step(k)
        sr.state()
        e2e_sec = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": total_nodes * T / e2e_sec, "unit": "node-updates/s",
               "h2d_bytes_per_step": 2 * xl.nbytes / T,
               "d2h_bytes_per_step": 2 * xl.nbytes / T,
               "call": "set_state (host) + %d strip steps + get_state (host)" % T}
        sr.close()
        conf = {"workload": WORKLOAD_LABEL[4], "grid": "8192x8192",
                "nodes_per_gpu": nodes_rank, "timesteps_per_step": 1, "mode": mode,
                "l2": "no flush: state 2 x %.0f MB >> 126 MB L2" % (24e-6 * nodes_rank),
                "parallelism": "%d row strips, 2-row halo per step %s" % (
                    world, "stored into the neighbours' ghost rows over peer memory (fused)"
                    if sr.transport == "peer" else "over NCCL")}

    value = total_nodes * K / sec_max
    # the timed region on this GPU: algorithmic bytes of all its node-updates over the region's
    # CUDA-event time (launch gaps included); the dominant kernel(s) run the whole region
    achieved = BYTES_PER_NODE_UPDATE * region_nu / sec / 1e9
    if kernel == "wave_kernel+fast_step_kernel" and _traffic(kernel, WORKLOAD_KEY[cid], K)[0]:
        traffic_per_nu, traffic_src = _traffic(kernel, WORKLOAD_KEY[cid], K)  # range capture
    elif kernel == "wave_kernel+fast_step_kernel":
        tw, src_w = _traffic("wave_kernel", WORKLOAD_KEY[cid], K)
        ts, src_s = _traffic("fast_step_kernel", WORKLOAD_KEY[cid], K)
        traffic_per_nu = ((B - n_coll) * tw + n_coll * ts) / B if tw and ts else None
        traffic_src = "%s (collider-free cloths) + %s (collider cloths)" % (src_w, src_s)
    else:
        traffic_per_nu, traffic_src = _traffic(kernel, WORKLOAD_KEY[cid], K)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": traffic_per_nu * region_nu if traffic_per_nu else None,
                "traffic_source": traffic_src, "kernel": kernel, "peak_source": peak_src,
                "algorithmic_bytes": BYTES_PER_NODE_UPDATE * region_nu,
                "launches": int(launches), "region_ms": sec * 1e3,
                "per": "the timed region: %d timesteps of this GPU's cloths" % K}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cid, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": "cloth node-updates/s", "value": value, "unit": "node-updates/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec_max / K, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": conf, "roofline": roofline, "hbm_fraction": achieved / peak,
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="timed timesteps (0: the config's own)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "parity"], default="fast")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=DEFAULT_CONFIG)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="batched configs: fixed batch split over the GPUs, or a batch per GPU")
    ap.add_argument("--e2e-calls", type=int, default=2)
    ap.add_argument("--transport", choices=["nccl", "peer"], default="nccl",
                    help="config 4 halo exchange: NCCL send/recv or the fused peer-store kernel")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="CPU seconds for the whole --impl reference run")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.steps <= 0:
        from oracle.workloads import WORKLOADS
        args.steps = WORKLOADS[args.config].steps
    world, rank, local = _dist()
    if args.impl == "reference":
        return run_reference(args, max(world, 1), rank)
    if world == 0:
        if args.gpus > 1:
            return _spawn(args)
        world = 1
    elif world != args.gpus:
        print("bench.py: WORLD_SIZE=%d overrides --gpus %d" % (world, args.gpus), file=sys.stderr)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
