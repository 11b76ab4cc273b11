"""Config 3 device time per timestep (500-step rollout and the contact window, timesteps 20-70)
for library builds (SC_B200_LIB or "tree"), alternated (development aid)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, %(root)r)
from paper_2403_12820_b200 import ClothBatch, configs
cfg, scenes, p, x, v = configs.build(3)
with ClothBatch(scenes, p) as cb:
    best = 1e9
    for _ in range(3):
        cb.set_state(x, v); cb.advance(5, 0, "fast")
        best = min(best, cb.benchmark(500, 0, "fast"))
    cb.set_state(x, v); cb.advance(20, 0, "fast")
    c = cb.benchmark(50, 0, "fast")
    cb.set_state(x, v); cb.advance(150, 0, "fast")
    f = cb.benchmark(100, 0, "fast")
print("500 steps %%.2f  contact 20-70 %%.2f  free 150-250 %%.2f us/step" %% (best / 500 * 1e6, c / 50 * 1e6, f / 100 * 1e6))
"""
for rep in range(2):
    for lib in sys.argv[1:]:
        env = dict(os.environ)
        if lib != "tree":
            env["SC_B200_LIB"] = os.path.abspath(lib)
        out = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}], env=env, capture_output=True, text=True, timeout=900)
        print("%-12s %s" % (os.path.basename(lib), out.stdout.strip() or out.stderr[-400:]), flush=True)
