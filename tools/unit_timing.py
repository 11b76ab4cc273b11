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
    buf = torch.zeros(2 * units, dtype=torch.int64, device="cuda")
    cb.advance(5, 0, "fast")
    cb.sync()
    lib.sc_debug_unit_timing(C.c_void_p(buf.data_ptr()))
    cb.advance(1, 5, "fast")
    cb.sync()
    lib.sc_debug_unit_timing(None)
t = buf.cpu().numpy().reshape(-1, 2).astype(np.float64)
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
