#!/usr/bin/env python
"""Throughput of the network-cell rollout step (arXiv 2403.12820 reference path) on B200.

Metric (BASELINE.json): cloth node-updates/s (nodes x timesteps / s), whole job over all GPUs,
and the fraction of the HBM roofline (48 algorithmic bytes per node-update: fp32 x and v read
once and written once per timestep).

Workload (N=1 and per rank under torchrun): BASELINE config 2 — 64 independent 256x256 cloths,
top row pinned, gravity + per-cloth wind, dt = 1/240, the reference's 12-channel cell with
N(0, 0.05) weights (SURVEY.md §8(d) mapping). One bench "step" = one timestep of the whole
batch (one fused-kernel launch). Multi-GPU: every rank owns its own 64 cloths (cloth ids
64*rank .. 64*rank+63 of the same seeded stream), no data-path collective -> weak scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the unmodified
reference sources, benchmark_net's own timer) cloth-parallel on all host cores, on bounded
samples of the same workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_NODE_UPDATE = 48  # fp32 x, v: 24 B read + 24 B written per node per timestep
CONFIG_ID = 2  # default workload; --config 4 (row strips) / 5 (4096 cloths) also run


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled every 10 ms (NVML, in-process) during the timed
    region; falls back to nvidia-smi polling when NVML is unavailable."""

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

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                active = {name for name, const in self.REASONS if r & getattr(nv, const)}
                self.samples.append((float(sm), float(mx), active))
                self._stop.wait(0.01)
            nv.nvmlShutdown()
        except Exception:
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    v = [x.strip() for x in out.stdout.strip().split(",")]
                    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                             "sw_power_cap"]
                    self.samples.append((float(v[0]), float(v[1]),
                                         {names[i] for i in range(4) if v[2 + i].lower() == "active"}))
                except Exception:
                    pass
                self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        time.sleep(0.02)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_min_mhz": min(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(set().union(*[s[2] for s in self.samples])),
                "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _traffic(kernel: str, workload: str):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(workload) if kernel == "fast_step_kernel" else t.get(kernel + ":" + workload)
        if e and e.get("workload") == workload:
            return e.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


def _cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


_REF_INPUTS = {}


def reference_sample(ref, cores: int, steps: int, warmup: int = 1, cloth0: int = 0):
    """benchmark_net (eval.cpp:155-158) on `cores` config-2 cloths, one thread each (the
    cloth-parallel variant: reference code unchanged, global thread count 1). Inputs are
    generated once per (cores, cloth0) and reused across samples."""
    from paper_2403_12820_b200 import configs
    import numpy as np

    key = (cores, cloth0)
    if key not in _REF_INPUTS:
        cfg, scenes, p, x, v = configs.build(CONFIG_ID, batch=cores, cloth0=cloth0)
        keep: list = []
        cds = [s.cloth_desc(keep) for s in scenes]
        _REF_INPUTS[key] = (cfg, cds, keep, p.to_c(), np.ascontiguousarray(x, np.float64),
                            np.ascontiguousarray(v, np.float64))
    cfg, cds, _, pc, x64, v64 = _REF_INPUTS[key]
    mx, wall = ref.benchmark_net_cloth_parallel(cfg.n, cfg.n, cds, pc, x64, v64, steps, warmup)
    nodes = cores * cfg.n * cfg.n * steps
    return nodes, mx, wall


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from oracle.pyoracle import Reference
    from paper_2403_12820_b200 import configs

    cfg = configs.CONFIGS[CONFIG_ID]
    ref = Reference()
    cores = _cpu_cores()
    # size every step's sample so the whole --steps K --warmup W run takes ~args.ref_budget
    # seconds of CPU time (each step: `cores` cloths x ts timesteps, ts >= 1)
    n0, s0, _ = reference_sample(ref, cores, 2, 1)
    per_ts = s0 / 2
    per_step = args.ref_budget / max(1, args.steps + args.warmup)
    ts = max(1, min(200, int(per_step / max(per_ts, 1e-6))))
    for _ in range(args.warmup):
        reference_sample(ref, cores, ts, 0)
    total_nodes, total_sec, times = 0, 0.0, []
    for _ in range(args.steps):
        n, sec, _ = reference_sample(ref, cores, ts, 0)
        total_nodes += n
        total_sec += sec
        times.append(sec)
    value = total_nodes / total_sec
    sample = ("%d cloths x %d timesteps of config 2 (256x256) per step, one std::thread per "
              "cloth, reference benchmark_net timer" % (cores, ts))
    line = {
        "impl": "reference", "metric": "cloth node-updates/s", "value": value,
        "unit": "node-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_sec / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.description, "grid": "256x256", "cloths_sampled": cores,
                   "timesteps_per_sample": ts, "parallelism": "cpu cloth-parallel"},
        "cpu_baseline": {"value": value, "unit": "node-updates/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "node-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _e2e_batch(cb, x, v, steps, mode, world, max_over_ranks, barrier, calls):
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
    cb.rollout(arrs[0], arrs[1], 2, 0, mode)  # warm the path
    barrier()
    t = []
    for _ in range(calls):
        t0 = time.perf_counter()
        rc = lib.sc_rollout(cb.h, bufs[0], bufs[1], steps, 0, 1 if mode == "fast" else 0,
                            bufs[2], bufs[3], None)
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

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    cid = args.config
    cfg = configs.CONFIGS[cid]
    mode = args.mode
    peak, peak_src = _peaks()
    kernel = "fast_step_kernel" if mode == "fast" else "parity_kernel"
    extra = {}
    if cid in (2, 5):
        # ---- batch sharding: every rank owns the config's batch (cloth ids B*rank ..) ----
        B = cfg.batch
        _, scenes, params, x, v = configs.build(cid, batch=B, cloth0=rank * B)
        nodes_rank = B * cfg.n * cfg.n
        cb = ClothBatch(scenes, params, device=local)
        cb.set_state(x, v)
        cb.advance(args.warmup, 0, mode)
        cb.sync()
        barrier()
        launches0 = cb.launch_count()
        with ClockSampler(local) as clocks:
            sec = cb.benchmark(args.steps, 0, mode)  # CUDA events around exactly K launches
            cb.sync()
        launches = cb.launch_count() - launches0
        barrier()
        sec_max = max_over_ranks(sec)
        # one timestep = the fused kernel over the whole batch, issued as `chunks` concurrent
        # cloth-chunk launches (capi.cu chunked_fast_steps); its average duration over the timed
        # region is region / steps (inter-launch gaps included, i.e. conservative)
        avg_launch_s = sec / args.steps
        extra["launches_per_step"] = launches / args.steps
        cb.set_state(x, v)
        ps = max(5, min(args.steps, 20))
        parity_value = world * nodes_rank * ps / cb.benchmark(ps, 2, "parity")
        extra["parity_mode"] = {"value": parity_value, "unit": "node-updates/s",
                                "note": "bit-exact with the reference f32 templates"}
        e2e_steps = cfg.steps
        e2e_sec, hb, db, finite = _e2e_batch(cb, x, v, e2e_steps, mode, world, max_over_ranks,
                                             barrier, args.e2e_calls)
        e2e = {"value": world * nodes_rank * e2e_steps / e2e_sec, "unit": "node-updates/s",
               "h2d_bytes_per_step": hb / e2e_steps, "d2h_bytes_per_step": db / e2e_steps,
               "call": "sc_rollout host->host, %d timesteps per call (pinned buffers)"
                       % e2e_steps, "finite": finite}
        cb.close()
        conf = {"workload": "cfg%d: %s" % (cid, cfg.description), "cloths_per_gpu": B,
                "grid": "%dx%d" % (cfg.n, cfg.n), "nodes_per_gpu": nodes_rank,
                "timesteps_per_step": 1, "mode": mode,
                "l2": "no flush: ping-pong state 2 x %.1f MB > 126 MB L2" % (24e-6 * nodes_rank),
                "parallelism": "dp%d batch-sharded, no collective" % world}
        scaling = "weak"
    elif cid == 4:
        # ---- one 8192^2 cloth in row strips, halo rows over NCCL each step ----
        row0, rows = strips.strip_bounds(cfg.n, world, rank)
        g0, g1 = strips.local_window(cfg.n, row0, rows)
        xl, _ = configs.sheet(cfg.seed, 0, cfg.n, g0, g1 - g0)
        scene = configs.make_scene(cfg, 0, xl.astype(np.float64), row0=g0)
        params = configs.make_params(cfg.seed, cfg.hidden8)
        sr = strips.StripRollout(scene, params, xl, np.zeros_like(xl), rank, world, local,
                                 mode=mode, transport=args.transport if mode == "fast" else "nccl")
        nodes_rank = rows * cfg.n
        for k in range(args.warmup):
            sr.step(k)
        barrier()
        l0 = sr.ctx.launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clocks:
            ev0.record(sr.stream)
            for k in range(args.warmup, args.warmup + args.steps):
                sr.step(k)
            ev1.record(sr.stream)
            ev1.synchronize()
        launches = sr.ctx.launch_count() - l0
        barrier()
        sec = ev0.elapsed_time(ev1) * 1e-3
        sec_max = max_over_ranks(sec)
        avg_launch_s = sec / args.steps  # one interior launch dominates each step
        t0 = time.perf_counter()
        sr.ctx.set_state(xl, np.zeros_like(xl))
        for k in range(args.steps):
            sr.step(k)
        sr.state()
        e2e_sec = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": world * nodes_rank * args.steps / e2e_sec, "unit": "node-updates/s",
               "h2d_bytes_per_step": 2 * xl.nbytes / args.steps,
               "d2h_bytes_per_step": 2 * xl.nbytes / args.steps,
               "call": "set_state (host) + %d strip steps + get_state (host)" % args.steps}
        sr.close()
        conf = {"workload": "cfg4: " + cfg.description, "grid": "8192x8192",
                "nodes_per_gpu": nodes_rank, "timesteps_per_step": 1, "mode": mode,
                "l2": "no flush: state 2 x %.0f MB >> 126 MB L2" % (24e-6 * nodes_rank),
                "parallelism": "%d row strips, 2-row halo per step %s" % (
                    world, "stored into the neighbours' ghost rows over peer memory (fused)"
                    if sr.transport == "peer" else "over NCCL")}
        scaling = "strong"
    else:
        raise SystemExit("--config must be 2, 4 or 5")

    value = world * nodes_rank * args.steps / sec_max if cid != 4 else \
        cfg.n * cfg.n * args.steps / sec_max
    achieved = BYTES_PER_NODE_UPDATE * nodes_rank / avg_launch_s / 1e9
    workload = {2: "cfg2_64x256x256", 4: "cfg4_8192x8192", 5: "cfg5_4096x128x128"}[cid]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": _traffic(kernel, workload),
                "kernel": kernel, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": BYTES_PER_NODE_UPDATE * nodes_rank,
                "avg_launch_ms": avg_launch_s * 1e3,
                "per": "timestep of the whole batch (its cloth-chunk launches run concurrently)"}

    # ---- CPU baseline: reference CPU path on this host, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cid == 2:
        try:
            from oracle.pyoracle import Reference
            ref = Reference()
            cores = _cpu_cores()
            n0, s0, _ = reference_sample(ref, cores, 2, 1)
            ts = max(1, min(4000, int(args.cpu_seconds / max(s0 / 2, 1e-6))))
            n, s, wall = reference_sample(ref, cores, ts, 1)
            cpu = {"value": n / s, "unit": "node-updates/s", "cores": cores, "kind": "reference",
                   "sample": "%d config-2 cloths (256x256) x %d timesteps, cloth-parallel "
                             "(one std::thread per cloth), reference benchmark_net timer, "
                             "%.1f s" % (cores, ts, s)}
        except Exception as e:  # the box may lack the prebuilt reference library
            cpu = {"value": None, "unit": "node-updates/s", "cores": _cpu_cores(),
                   "kind": "reference", "sample": "unavailable: %s" % e}

    if rank == 0:
        line = {
            "metric": "cloth node-updates/s", "value": value, "unit": "node-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec_max / args.steps, "higher_is_better": True,
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
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["fast", "parity"], default="fast")
    ap.add_argument("--config", type=int, choices=[2, 4, 5], default=CONFIG_ID)
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
    world, rank, local = _dist()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
