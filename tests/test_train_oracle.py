"""The training restatement (oracle/train_oracle.py) pinned against the reference-generated
fixture (tests/golden/train_f64.npz, made by oracle/_ref): targets, loss, gradients and a
multi-chunk backward pass, bit for bit. CPU only."""
import numpy as np

from golden_io import cloth_desc, load
from oracle import train_oracle as T


def bits(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_targets_match_fixture():
    z = load("train_f64")
    nx, ny = int(z["nx"]), int(z["ny"])
    for b, k in enumerate(z["batch_idx"]):
        tg = T.sample_targets(nx, ny, z["frames_x"][k], z["frames_v"][k], z)
        assert bits(tg, z["targets"][b]), b


def test_loss_and_gradients_match_fixture(oracle):
    z = load("train_f64")
    nx, ny = int(z["nx"]), int(z["ny"])
    keep = []
    cd = cloth_desc(z, keep)
    loss, grads = T.compute_loss(nx, ny, z["frames_x"], z["frames_v"], list(z["batch_idx"]),
                                 z["targets"], list(z["params"]), float(z["loss_alpha"]), z, cd,
                                 oracle)
    assert bits(loss, z["loss"])
    assert bits(grads, z["grads"])


def test_backward_two_chunks_matches_fixture():
    z = load("train_f64")
    bx, by = (int(v) for v in z["bwd_dims"])
    g = T.backward_gradients(bx, by, z["bwd_x"], z["bwd_v"], list(z["bwd_params"]), z["bwd_up"])
    assert bits(g, z["bwd_grads"])
