"""A/B device timing of library builds (development aid, not the bench).

  python tools/ab_perf.py [--reps 2] [--cases c5,c5s,c5p,c2,c3,c4] LIB [LIB ...]

LIB = a path to a libstencilcloth_b200.so build or "tree" (the in-tree library). Each (case,
lib) runs in its own process (SC_B200_LIB selects the build), alternating libs, and prints the
device time per timestep of the FAST stepping as the bench does it (ClothBatch.benchmark).
Cases: c5 = config 5 (mixed classes, class-grouped), c5s / c5p = config-5 batches of only
collider-free / only plane cloths (wavefront and streaming), c2 / c3 / c4 = configs 2 / 3 / 4,
c1 = config 1.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
sys.path.insert(0, %(root)r)
import paper_2403_12820_b200.configs as C
from paper_2403_12820_b200 import ClothBatch
case = %(case)r
steps_over = %(steps)d
cid = {"c1": 1, "c2": 2, "c3": 3, "c4": 4}.get(case, 5)
if case == "c5s":
    C.cloth_kind = lambda cfg, b: ("top_row", "corners")[b %% 2]
elif case == "c5p":
    C.cloth_kind = lambda cfg, b: "free"
cfg, scenes, p, x, v = C.build(cid)
steps = steps_over or cfg.steps
res = {}
for persistent in ((True, False) if case in ("c5s", "c5p") else (True,)):
    with ClothBatch(scenes, p) as cb:
        cb.set_persistent(persistent)
        cb.set_state(x, v)
        cb.benchmark(min(steps, 20), 3, "fast")
        sec = cb.benchmark(steps, 3, "fast")
    res["wave" if persistent else "stream"] = sec / steps * 1e6
print(json.dumps(res))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--cases", default="c5,c5s,c5p,c2,c3,c4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--steps", type=int, default=0)
    args = ap.parse_args()
    for case in args.cases.split(","):
        for rep in range(args.reps):
            for lib in args.libs:
                env = dict(os.environ)
                if lib != "tree":
                    env["SC_B200_LIB"] = os.path.abspath(lib)
                code = CHILD % {"root": ROOT, "case": case, "steps": args.steps}
                out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                                     text=True, timeout=900)
                line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-400:]
                print("%-4s rep%d %-28s %s" % (case, rep, os.path.basename(lib), line), flush=True)


if __name__ == "__main__":
    main()
