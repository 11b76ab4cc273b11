"""Drop-in adapter (integration/stencilcloth_b200_adapter.cpp): the reference's OWN Python API
objects (stencilcloth.Scene / NetworkParams, built from /root/reference into oracle/_ref) go
straight into the B200 path and come back as the reference's own Trajectory type."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref")

SCENE = """
{
  "name": "dropin_sheet",
  "grid": {"nx": 14, "ny": 11, "spacing": 0.04, "origin": [-0.26, -0.2, 0.31], "plane": "xy"},
  "material": {"stiffness": 30.0, "damping": 0.05, "mass": 0.01, "gravity": [0.2, 0.0, -9.8],
               "drag": 0.02, "pressure": 0.5},
  "time": {"dt": 0.001, "steps": 60},
  "pins": {"nodes": ["top_left", "top_right"], "motion": {"velocity": [0.0, 0.05, 0.0]}},
  "colliders": [{"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 0.25, "friction": 0.4}],
  "plug_forces": ["gravity", "drag", "pressure"]
}
"""


def _modules():
    if not os.path.isdir(os.path.join(REF_PKG, "stencilcloth")):
        pytest.skip("reference module not built (integration/Makefile needs /root/reference)")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import stencilcloth as sc
    import stencilcloth_b200_adapter as gpu
    return sc, gpu


def _trained_params(sc, scene):
    """Non-trivial weights through the reference's own API (a few training epochs)."""
    traj = sc.simulate(scene)
    params, _ = sc.train(scene, traj, alpha=0.5, batch_size=8, epochs=3, seed=5,
                         de_population=6, de_generations=2, de_probe=4)
    return params


def test_adapter_imports_and_refuses_without_gpu():
    sc, gpu = _modules()
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by test_dropin_rollout_bitwise")
    except ImportError:
        pass
    scene = sc.parse_scene(SCENE)
    with pytest.raises(RuntimeError):  # no CPU fallback
        gpu.rollout(sc.NetworkParams(), scene, 2)


@pytest.mark.gpu
def test_dropin_rollout_bitwise():
    sc, gpu = _modules()
    scene = sc.parse_scene(SCENE)
    params = _trained_params(sc, scene)
    assert any(v != 0.0 for v in params.scalars()[12:51])
    ref = sc.rollout(params, scene, 10)
    got = gpu.rollout(params, scene, 10)
    assert type(got) is type(ref) and len(got) == len(ref) == 11
    for f in range(len(ref)):
        assert np.array_equal(got.positions(f), ref.positions(f)), f
        assert np.array_equal(got.velocities(f), ref.velocities(f)), f
    # past the horizon these weights blow up: the same exception type and text as the reference
    with pytest.raises(ArithmeticError) as e_ref:
        sc.rollout(params, scene, 60)
    with pytest.raises(ArithmeticError) as e_gpu:
        gpu.rollout(params, scene, 60)
    assert str(e_gpu.value) == str(e_ref.value)
    x, v = ref.positions(7), ref.velocities(7)
    assert np.array_equal(gpu.forward_impulse(params, scene, x, v),
                          sc.forward_impulse(params, scene, x, v))
    with pytest.raises(ValueError):
        gpu.forward_impulse(params, scene, x[:-1], v[:-1])
