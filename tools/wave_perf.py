"""Device-resident FAST throughput: wavefront kernel (levels 8 / 12 / 16) vs the streaming
per-step kernel, on full-size BASELINE workloads (node-updates/s, CUDA-event timed).

  python tools/wave_perf.py [--configs 5,1] [--steps 300] [--levels 8,12,16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="5")
    ap.add_argument("--steps", type=int, default=0, help="0: the config's own length")
    ap.add_argument("--levels", default="8,12,16")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--n", type=int, default=0, help="shrink / grow the grid to n x n")
    args = ap.parse_args()
    from paper_2403_12820_b200 import ClothBatch, configs

    for cid in [int(c) for c in args.configs.split(",")]:
        cfg, scenes, p, x, v = configs.build(cid, batch=args.batch or None, threads=16,
                                             n=args.n or None)
        steps = args.steps or cfg.steps
        nodes = x.shape[0] * x.shape[1]
        runs = [("stream", None)] + [("wave%s" % l, l) for l in args.levels.split(",")]
        for name, lev in runs:
            if lev:
                os.environ["SC_WAVE_LEVELS"] = lev
            with ClothBatch(scenes, p) as cb:
                cb.set_persistent(lev is not None)
                cb.set_state(x, v)
                best = None
                for _ in range(args.reps):
                    sec = cb.benchmark(steps, 3, "fast")
                    best = sec if best is None else min(best, sec)
            print(json.dumps({"config": cid, "kernel": name, "steps": steps, "nodes": nodes,
                              "ms": best * 1e3, "node_updates_per_s": nodes * steps / best,
                              "hbm_roofline_frac_48B": nodes * steps * 48 / best / 6454.6e9}),
                  flush=True)
        os.environ.pop("SC_WAVE_LEVELS", None)


if __name__ == "__main__":
    main()
