"""Ground-truth mass-spring step (PBS) on the GPU: total_impulse,
step_semi_implicit and simulate_scene bit-exact against fixtures made by the reference build,
f64 and f32, including the reference's error messages."""
import numpy as np
import pytest

from golden_io import cloth_desc, load, to_scene

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(
        a.view(np.uint8), b.view(np.uint8))


def _scene(z):
    s = to_scene(z, z["x0"])
    s.initial_v = np.array(z["v0"], np.float64)
    s.steps = z["frames_x"].shape[0] - 1 if "frames_x" in z else 0
    return s


def test_pbs_f64_public_api_bitwise():
    import paper_2403_12820_b200 as sc
    z = load("pbs_sim64")
    scene = _scene(z)
    fx, fv = z["frames_x"], z["frames_v"]
    assert bits_equal(sc.total_impulse(scene, fx[60], fv[60]), z["imp60"])
    x1, v1 = sc.step_semi_implicit(scene, fx[30], fv[30], 31 * scene.dt)
    assert bits_equal(x1, fx[31]) and bits_equal(v1, fv[31])
    traj = sc.simulate(scene)
    assert len(traj) == fx.shape[0]
    for f in range(len(traj)):
        assert bits_equal(traj.positions(f), fx[f]), f
        assert bits_equal(traj.velocities(f), fv[f]), f


def test_pbs_f32_step_sequence_bitwise():
    from paper_2403_12820_b200 import Context
    z = load("pbs_steps32")
    scene = to_scene(z, z["x0"].astype(np.float64))
    with Context(scene, None, "f32") as ctx:
        last = int(z["checkpoints"][-1])
        fx, fv = ctx.simulate_frames(z["x0"][None], z["v0"][None], last, 1)
        for cp in z["checkpoints"]:
            assert bits_equal(fx[cp, 0], z["x_%d" % cp]) and bits_equal(fv[cp, 0], z["v_%d" % cp])
        sec = ctx.benchmark_sim(5, 1)
        assert sec > 0


def test_pbs_errors_match_reference(reference):
    import paper_2403_12820_b200 as sc
    z = load("pbs_sim64")
    nx, ny = int(z["nx"]), int(z["ny"])
    # coincident connected nodes: the singular-spring message of the elastic pass
    scene = _scene(z)
    scene.initial_x = scene.initial_x.copy()
    scene.initial_x[17] = scene.initial_x[18]
    scene.steps = 3
    keep = []
    cd = cloth_desc(z, keep)
    with pytest.raises(ArithmeticError) as e_ref:
        reference.simulate_f64(nx, ny, cd, scene.initial_x, scene.initial_v, 3)
    with pytest.raises(ArithmeticError) as e_gpu:
        sc.simulate(scene)
    assert str(e_gpu.value) == str(e_ref.value)
    # an unstable dt: the term diagnosis of diagnose_divergence (sim.cpp:23-48)
    zz = dict(z)
    zz["dt"] = np.float64(0.5)
    scene = _scene(zz)
    scene.steps = 40
    cd = cloth_desc(zz, keep)
    with pytest.raises(ArithmeticError) as e_ref:
        reference.simulate_f64(nx, ny, cd, scene.initial_x, scene.initial_v, 40)
    with pytest.raises(ArithmeticError) as e_gpu:
        sc.simulate(scene)
    assert str(e_gpu.value) == str(e_ref.value)


def test_total_force_matches_reference_module():
    """total_force (sim.cpp:84-96) through the reference's own binding, bit for bit, including
    its singular-spring error text."""
    import os
    import sys
    ref_pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle",
                           "_ref")
    if not os.path.isdir(os.path.join(ref_pkg, "stencilcloth")):
        pytest.skip("reference module not built")
    sys.path.insert(0, ref_pkg)
    import stencilcloth as ref
    import paper_2403_12820_b200 as sc
    text = """{"name": "tf", "grid": {"nx": 11, "ny": 9, "spacing": 0.05,
      "origin": [-0.25, -0.2, 0.3], "plane": "xy"},
      "material": {"stiffness": 40.0, "damping": 0.3, "mass": 0.02,
                   "gravity": [0.1, 0.0, -9.8], "drag": 0.05, "pressure": 0.7},
      "time": {"dt": 0.001, "steps": 10}, "pins": {"nodes": ["top_left"]}}"""
    rscene = ref.parse_scene(text)
    scene = sc.parse_scene(text)
    rng = np.random.default_rng(4)
    x = rscene.initial_positions() + rng.normal(0, 0.01, (99, 3))
    v = rng.normal(0, 0.5, (99, 3))
    assert bits_equal(sc.total_force(scene, x, v), ref.total_force(rscene, x, v))
    x[5] = x[6]  # coincident connected pair
    with pytest.raises(ArithmeticError) as r:
        ref.total_force(rscene, x, v)
    with pytest.raises(sc.NumericsError) as o:
        sc.total_force(scene, x, v)
    assert str(o.value) == str(r.value)
