"""FAST-mode error report at the BASELINE configs' full sizes (GPU box).

For each config: roll the full batch forward k steps in PARITY mode (bit-exact with the
reference, tests/test_gpu_parity.py), then from that state take ONE step with the C oracle
(oracle/oracle.c, multi-threaded over cloths) and ONE step with the FAST kernel, and report
  * PARITY step == oracle step bit for bit (also at full size),
  * max |a-b| / max(|b|, f * rms(b)) per component plane for f = 1 (the round-1 gate) and
    f = 1e-6, the count of elements above 1e-5 under the latter,
  * the normwise error max|a-b| / max|b|,
  * masks identical.
Prints one JSON line per (config, k).

  python tools/fast_error_report.py [--configs 1,2,3,4,5] [--ks 0,10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def oracle_step(o, n, cds, pc, x, v, k, threads=16):
    B = x.shape[0]
    xo, vo = np.empty_like(x), np.empty_like(v)
    mo = np.empty((B, n * n), np.uint8)
    per = (B + threads - 1) // threads

    def work(b0, b1):
        # rollout of 1 step starting at step index k (t_next = (k+1) dt)
        a, b, m = o.rollout(n, n, cds[b0:b1], pc, x[b0:b1], v[b0:b1], 1, k)
        xo[b0:b1], vo[b0:b1], mo[b0:b1] = a, b, m

    ts = [threading.Thread(target=work, args=(i, min(B, i + per))) for i in range(0, B, per)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return xo, vo, mo


def errs(a, b):
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    rms = np.sqrt(np.mean(b * b, axis=0))
    err = np.abs(a - b)
    out = {}
    for f, tag in ((1.0, "rms_floor"), (1e-6, "tight_floor")):
        r = err / np.maximum(np.abs(b), f * rms[None, :])
        out[tag] = float(r.max())
        if tag == "tight_floor":
            out["tight_over_1e-5"] = int((r > 1e-5).sum())
            i = int(np.argmax(r))
            out["tight_worst"] = {"a": float(a.flat[i]), "b": float(b.flat[i]),
                                  "rms": float(rms[i % 3])}
    out["normwise"] = float(err.max() / np.abs(b).max())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--ks", default="0,10")
    args = ap.parse_args()
    from oracle.pyoracle import Oracle
    from paper_2403_12820_b200 import ClothBatch, configs

    o = Oracle()
    for cid in [int(c) for c in args.configs.split(",")]:
        t0 = time.time()
        cfg, scenes, p, x, v = configs.build(cid, threads=16)
        keep = []
        cds = [s.cloth_desc(keep) for s in scenes]
        pc = p.to_c()
        n = cfg.n
        with ClothBatch(scenes, p, device=0) as cb:
            xs, vs, kdone = x, v, 0
            for k in sorted(int(s) for s in args.ks.split(",")):
                if k > kdone:
                    xs, vs = cb.rollout(xs, vs, k - kdone, kdone, "parity")
                    kdone = k
                xp, vp, mp = cb.rollout(xs, vs, 1, k, "parity", constrained=True)
                xf, vf, mf = cb.rollout(xs, vs, 1, k, "fast", constrained=True)
                xo, vo, mo = oracle_step(o, n, cds, pc, xs, vs, k)
                line = {"config": cid, "k": k, "nodes": int(x.shape[0] * n * n),
                        "parity_bitexact": bool(np.array_equal(xp.view(np.uint32), xo.view(np.uint32))
                                                and np.array_equal(vp.view(np.uint32), vo.view(np.uint32))),
                        "parity_mask": bool(np.array_equal(mp.reshape(mo.shape), mo)),
                        "fast_mask": bool(np.array_equal(mf.reshape(mo.shape), mo)),
                        "x": errs(xf, xo), "v": errs(vf, vo),
                        "max_abs_v": float(np.abs(vo).max()),
                        "seconds": round(time.time() - t0, 1)}
                print(json.dumps(line), flush=True)
        del x, v, xs, vs


if __name__ == "__main__":
    main()
