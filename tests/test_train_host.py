"""Host side of training (§8(f1)) without a GPU: the sample_batch index draw and the Rng mirror
against the reference, the TrainConfig ABI layout, validation texts, and the training fixture
pinned against the reference itself."""
import ctypes as C

import numpy as np
import pytest

import paper_2403_12820_b200 as ours
from paper_2403_12820_b200 import _abi
from golden_io import cloth_desc, load, params_c


def test_config_struct_layout():
    assert C.sizeof(_abi.sc_train_config) == 120
    assert C.sizeof(_abi.sc_adam_state) == 53 * 16 + 8
    c = ours.TrainConfig(freeze=[ours.ParamGroup.Bias, ours.ParamGroup.Deriv]).to_c()
    assert c.freeze_mask == (1 << 2) | (1 << 4)
    assert (c.batch_size, c.epochs, c.de_population, c.de_probe_batch) == (128, 2000, 64, 32)


@pytest.mark.parametrize("frames,batch,seed", [(61, 16, 77), (2, 1, 0), (500, 128, 2**63 + 5),
                                               (33, 32, 12345)])
def test_sample_indices_match_reference(reference, frames, batch, seed):
    z = load("train_f64")
    keep = []
    cd = cloth_desc(z, keep)
    nx, ny = int(z["nx"]), int(z["ny"])
    fx = np.zeros((frames, nx * ny, 3))
    fx[:] = z["frames_x"][0]
    idx, _ = reference.sample_batch(nx, ny, cd, fx, fx * 0, batch, seed)
    mine = ours.sample_indices(frames, batch, seed)
    assert np.array_equal(mine, idx)
    assert len(set(mine.tolist())) == batch


def test_sample_indices_errors():
    with pytest.raises(ours.ConfigError, match=r"^batch size 9 not in \[1, 8\]$"):
        ours.sample_indices(9, 9, 1)
    with pytest.raises(ours.ConfigError, match=r"^batch size 0 not in \[1, 8\]$"):
        ours.sample_indices(9, 0, 1)
    with pytest.raises(ours.ConfigError, match="^trajectory has no transitions to sample$"):
        ours.sample_indices(1, 1, 1)


def test_fixture_pinned_to_reference(reference):
    z = load("train_f64")
    keep = []
    cd = cloth_desc(z, keep)
    nx, ny = int(z["nx"]), int(z["ny"])
    idx, tgt = reference.sample_batch(nx, ny, cd, z["frames_x"], z["frames_v"], 16, 77)
    assert np.array_equal(idx, z["batch_idx"]) and np.array_equal(tgt, z["targets"])
    loss, g = reference.compute_loss(nx, ny, cd, z["frames_x"], z["frames_v"], 16, 77,
                                     params_c(z["params"]), float(z["loss_alpha"]))
    assert np.array_equal(loss, z["loss"]) and np.array_equal(g, z["grads"])
    bx, by = (int(v) for v in z["bwd_dims"])
    bg = reference.backward_gradients(bx, by, z["bwd_x"], z["bwd_v"], params_c(z["bwd_params"]),
                                      z["bwd_up"])
    assert np.array_equal(bg, z["bwd_grads"])


def test_rng_mirror_uniform_draws():
    # Rng::uniform01 = (u64 >> 11) * 2^-53 over std::mt19937_64; the standard fixes the 10000th
    # output of a default-seeded (5489) engine
    from paper_2403_12820_b200.training import Rng
    r = Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042
    r = Rng(1)
    u = [r.uniform01() for _ in range(1000)]
    assert all(0.0 <= x < 1.0 for x in u)


def test_trainer_rejects_bad_inputs():
    z = load("train_f64")
    from golden_io import to_scene
    scene = to_scene(z, z["frames_x"][0])
    t = ours.Trajectory(3, 3, 1e-3, 0.05, np.zeros((2, 9, 3)), np.zeros((2, 9, 3)))
    with pytest.raises(ours.ConfigError, match="state shape does not match the grid topology"):
        ours.Trainer(scene, t)
    bad = ours.Trajectory(12, 10, 1e-3, 0.05, np.full((2, 120, 3), np.nan), np.zeros((2, 120, 3)))
    with pytest.raises(ours.ConfigError, match="trajectory: frame 0 has non-finite components"):
        ours.Trainer(scene, bad)
