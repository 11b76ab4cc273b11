"""Training throughput: the native GPU train loop vs the reference's train_loop on the host cores,
same scene / trajectory / TrainConfig, and the final parameters compared bit for bit.

  python tools/train_bench.py [--n 32] [--frames 201] [--batch 128] [--epochs 50]
                              [--de-pop 16] [--de-gen 4] [--ref-threads 0]
Prints one JSON line. The reference arm needs oracle/_ref (built where /root/reference exists).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import paper_2403_12820_b200 as ours  # noqa: E402
from golden_io import cloth_desc, scene_arrays, to_scene  # noqa: E402
from make_golden import sheet, train_config  # noqa: E402
from oracle.pyoracle import Reference  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--frames", type=int, default=201)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--epochs", type=int, default=50)
    ap.add_argument("--de-pop", type=int, default=16)
    ap.add_argument("--de-gen", type=int, default=4)
    ap.add_argument("--probe", type=int, default=32)
    ap.add_argument("--ref-threads", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    n = a.n
    rng = np.random.default_rng(5)
    sp = 1.0 / (n - 1)
    x0 = sheet(rng, n, n, sp, 1e-3, origin=(-0.5, -0.5, 0.35))
    pins = [n * (n - 1), n * n - 1]
    sc = scene_arrays(n, n, 1.0 / 240, mass=0.01, drag=0.02, pressure=0.0, plugs=(0, 1, 1),
                      pin_nodes=pins, pin_anchors=x0[pins], spheres=[(0.0, 0.0, 0.0, 0.3, 0.2)],
                      stiffness=200.0, damping=0.05, spacing=sp)
    keep = []
    cd = cloth_desc(sc, keep)
    R = Reference()
    fx, fv = R.simulate_f64(n, n, cd, x0, np.zeros_like(x0), a.frames - 1)
    scene = to_scene(sc, x0)
    traj = ours.Trajectory(n, n, float(sc["dt"]), sp, fx, fv)
    cfg = ours.TrainConfig(alpha=0.5, batch_size=a.batch, epochs=a.epochs, seed=1,
                           de=ours.DeConfig(population=a.de_pop, generations=a.de_gen,
                                            probe_batch=a.probe))
    with ours.Trainer(scene, traj) as t:
        t.run(ours.TrainConfig(alpha=0.5, batch_size=a.batch, epochs=2, seed=9,
                               de=ours.DeConfig(population=4, generations=0, probe_batch=4)))
        t0 = time.perf_counter()
        r = t.run(cfg)
        gpu_s = time.perf_counter() - t0
        # per-call compute_loss time (grads) at this batch, device-synchronous
        t.sample_batch(a.batch, 3)
        t.compute_loss(r.params, 0.5)
        t0 = time.perf_counter()
        for _ in range(20):
            t.compute_loss(r.params, 0.5)
        loss_ms = (time.perf_counter() - t0) / 20 * 1e3
    evals = a.de_pop * (a.de_gen + 1)
    out = {"workload": "train_loop %dx%d, %d frames, batch %d, %d epochs, DE %dx%d (probe %d)"
           % (n, n, a.frames, a.batch, a.epochs, a.de_pop, a.de_gen + 1, a.probe),
           "gpu_seconds": round(gpu_s, 4), "gpu_compute_loss_ms": round(loss_ms, 4),
           "loss_evaluations": evals + a.epochs}
    if not a.no_ref:
        threads = a.ref_threads or os.cpu_count()
        R.lib.ref_set_threads(threads)
        c = train_config(alpha=0.5, batch_size=a.batch, epochs=a.epochs, seed=1,
                         de_population=a.de_pop, de_generations=a.de_gen, de_probe_batch=a.probe,
                         interval=250)
        t0 = time.perf_counter()
        rp, _, _ = R.train(n, n, cd, fx, fv, c)
        ref_s = time.perf_counter() - t0
        flat = (list(rp.kernel_gain) + list(rp.linear_w) + list(rp.linear_b)
                + list(rp.nonlinear_w) + list(rp.deriv_w) + [rp.self_velocity_w, rp.isru_alpha])
        out.update({"ref_seconds": round(ref_s, 4), "ref_threads": threads,
                    "speedup": round(ref_s / gpu_s, 2),
                    "params_bit_identical": bool(np.array_equal(
                        np.array(r.params.scalars()).view(np.uint64),
                        np.array(flat).view(np.uint64)))})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
