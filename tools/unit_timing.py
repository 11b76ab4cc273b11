"""Debug: start/end time of every FAST-kernel unit (one launch of config 2) -> ramp/tail view."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, _abi, configs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lib = _abi.load()
lib.sc_debug_unit_timing.argtypes = [C.c_void_p]
lib.sc_debug_units.argtypes = [C.c_void_p]
lib.sc_debug_units.restype = C.c_int64
cfg, scenes, p, x, v = configs.build(cid)
with ClothBatch(scenes, p) as cb:
    cb.set_state(x, v)
    units = lib.sc_debug_units(cb.h)
    buf = torch.zeros(3 * units, dtype=torch.int64, device="cuda")
    cb.advance(5, 0, "fast")
    cb.sync()
    lib.sc_debug_unit_timing(C.c_void_p(buf.data_ptr()))
    cb.advance(1, 5, "fast")
    cb.sync()
    lib.sc_debug_unit_timing(None)
raw = buf.cpu().numpy().reshape(-1, 3)
ids = raw[:, 2]
sm = (ids >> 32).astype(np.int64)
warp = (ids & 0xFFFFFFFF).astype(np.int64)
t = raw[:, :2].astype(np.float64)
t -= t[:, 0].min()
dur = t[:, 1] - t[:, 0]
print("units", units, "span %.1f us" % (t[:, 1].max() / 1e3))
print("start: min %.1f  p50 %.1f  p90 %.1f  max %.1f us" % tuple(np.percentile(t[:, 0], [0, 50, 90, 100]) / 1e3))
print("end:   min %.1f  p10 %.1f  p50 %.1f  p90 %.1f  max %.1f us" % tuple(np.percentile(t[:, 1], [0, 10, 50, 90, 100]) / 1e3))
print("dur:   min %.1f  p10 %.1f  p50 %.1f  p90 %.1f  max %.1f us" % tuple(np.percentile(dur, [0, 10, 50, 90, 100]) / 1e3))
# busy-warp profile over time
grid = np.linspace(0, t[:, 1].max(), 21)
busy = [int(((t[:, 0] <= g) & (t[:, 1] > g)).sum()) for g in grid]
print("active units over time:", busy)

# duration vs SM occupancy and warp slot (SMSP = warpid % 4)
per_sm = np.bincount(sm, minlength=sm.max() + 1)
d_us = dur / 1e3
print("units per SM: min %d max %d" % (per_sm[per_sm > 0].min(), per_sm.max()))
for k in sorted(set(per_sm[sm])):
    sel = per_sm[sm] == k
    print("  SMs with %d units: mean dur %.1f us (n=%d)" % (k, d_us[sel].mean(), sel.sum()))
smsp = warp % 4
for q in range(4):
    sel = smsp == q
    print("  smsp %d: mean dur %.1f us, n %d" % (q, d_us[sel].mean(), sel.sum()))
# warps per (sm, smsp)
key = sm * 4 + smsp
cnt = np.bincount(key)
for c in sorted(set(cnt[key])):
    sel = cnt[key] == c
    print("  SMSPs holding %d warps: mean dur %.1f us (n=%d)" % (c, d_us[sel].mean(), sel.sum()))
sm_mean = np.array([d_us[sm == i].mean() for i in range(sm.max() + 1) if (sm == i).any()])
print("per-SM mean duration: min %.1f p50 %.1f max %.1f" % (sm_mean.min(), np.median(sm_mean), sm_mean.max()))
print("within-SM spread (max-min) median %.1f us" % np.median([d_us[sm == i].max() - d_us[sm == i].min() for i in range(sm.max() + 1) if (sm == i).any()]))
# duration vs launch order (blockIdx): warps launched earlier get issue priority
order = np.arange(len(d_us))
rank = order * 16 // len(d_us)
print("mean duration by launch-order sixteenth:", [round(float(d_us[rank == r].mean()), 1) for r in range(16)])
np.save("gpurun_out/unit_timing_%d.npy" % cid, np.stack([t[:, 0], t[:, 1], sm, warp]))
