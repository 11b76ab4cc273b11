"""Timeline of one pinned host -> host sc_rollout (CUPTI through torch.profiler: every kernel and
copy of the library on every stream). Prints the wall span, the union of kernel time, the H2D /
D2H busy time, the GPU idle gaps and the exposed head / tail, so the gap between the e2e and the
device-resident rate can be attributed. Usage: python tools/rollout_trace.py [config] [steps]
(env knobs such as SC_BAND_ROWS apply). Runs on the GPU box."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402
from paper_2403_12820_b200.api import pinned_empty  # noqa: E402


def union(iv):
    iv = sorted(iv)
    tot, cs, ce = 0.0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    cfg = configs.CONFIGS[cid]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.steps
    _, scenes, p, x, v = configs.build(cid, threads=16)
    xp, vp = pinned_empty(x.shape), pinned_empty(v.shape)
    xp[...] = x
    vp[...] = v
    xo, vo = pinned_empty(x.shape), pinned_empty(v.shape)
    nodes = x.shape[0] * x.shape[1] if x.ndim == 3 else x.size // 3
    with ClothBatch(scenes, p) as cb:
        cb.set_state(x, v)
        sec = cb.benchmark(steps, 0, "fast")
        cb.rollout(xp, vp, 2, 0, "fast", out=(xo, vo))
        t0 = time.perf_counter()
        cb.rollout(xp, vp, steps, 0, "fast", out=(xo, vo))
        wall = time.perf_counter() - t0
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            cb.rollout(xp, vp, steps, 0, "fast", out=(xo, vo))
            torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern, h2d, d2h = [], [], []
    for e in ev:
        iv = (e.time_range.start, e.time_range.end)
        n = e.name.lower()
        if "memcpy" in n and ("htod" in n or "host to device" in n):
            h2d.append(iv)
        elif "memcpy" in n and ("dtoh" in n or "device to host" in n):
            d2h.append(iv)
        elif "memcpy" not in n and "memset" not in n:
            kern.append(iv)
    t_lo = min(s for s, _ in kern + h2d + d2h)
    t_hi = max(e for _, e in kern + h2d + d2h)
    print("config %d, %d steps, %d nodes" % (cid, steps, nodes))
    print("device-resident stepping (benchmark): %.2f ms -> %.3e node-updates/s"
          % (sec * 1e3, nodes * steps / sec))
    print("e2e wall: %.2f ms -> %.3e node-updates/s (%.3f x)"
          % (wall * 1e3, nodes * steps / wall, sec / wall))
    print("traced span: %.2f ms; kernels %d, union %.2f ms; H2D %d, busy %.2f ms; D2H %d, busy "
          "%.2f ms" % ((t_hi - t_lo) / 1e3, len(kern), union(kern) / 1e3, len(h2d),
                       union(h2d) / 1e3, len(d2h), union(d2h) / 1e3))
    k_lo = min(s for s, _ in kern)
    k_hi = max(e for _, e in kern)
    print("head (first copy -> first kernel): %.2f ms; tail (last kernel -> last copy): %.2f ms"
          % ((k_lo - t_lo) / 1e3, (t_hi - k_hi) / 1e3))
    print("kernel idle inside [first, last kernel]: %.2f ms"
          % ((k_hi - k_lo - union(kern)) / 1e3))
    names = {}
    for e in ev:
        if "memcpy" in e.name.lower():
            continue
        d = names.setdefault(e.name[:60], [0, 0.0])
        d[0] += 1
        d[1] += e.time_range.end - e.time_range.start
    for k, (cnt, tot) in sorted(names.items(), key=lambda t: -t[1][1])[:8]:
        print("  %6d x %9.2f ms  %s" % (cnt, tot / 1e3, k))


if __name__ == "__main__":
    main()
