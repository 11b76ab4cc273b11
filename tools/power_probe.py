"""Power, clocks and throttle bits (NVML, every 5 ms) during a long FAST benchmark of config 2."""
import sys
import threading
import time

import pynvml as nv

sys.path.insert(0, ".")
from paper_2403_12820_b200 import ClothBatch, configs  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sample():
    t0 = time.time()
    while not stop.is_set():
        samples.append((time.time() - t0, nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                        nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM),
                        nv.nvmlDeviceGetCurrentClocksEventReasons(h),
                        nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU)))
        time.sleep(0.005)


cfg, scenes, p, x, v = configs.build(2)
with ClothBatch(scenes, p) as cb:
    cb.set_state(x, v)
    cb.benchmark(50, 0, "fast")
    th = threading.Thread(target=sample)
    th.start()
    time.sleep(0.05)
    out = []
    for i in range(12):
        sec = cb.benchmark(250, 0, "fast")
        out.append(round(sec / 250 * 1e6, 2))
    stop.set()
    th.join()
print("us/step per 250-step call:", out)
print("limit W", nv.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0)
for s in samples[::4]:
    print("t=%.3f P=%.0fW sm=%d mem=%d reasons=0x%x T=%dC" % s)
