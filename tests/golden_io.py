"""Golden-fixture (de)serialisation shared by tests/golden/make_golden.py and the tests.

A fixture .npz holds one cloth scene as plain arrays (so it does not depend on the product's
input generator), the 53 parameters, the input state and the reference's outputs.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2403_12820_b200 import _abi

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def scene_arrays(nx, ny, dt, mass=1.0, drag=0.0, pressure=0.0, gravity=(0, 0, -9.8),
                 plugs=(0, 1, 0), pin_nodes=(), pin_anchors=None, pin_velocity=(0, 0, 0),
                 spheres=(), planes=(), stiffness=0.0, damping=0.0, spacing=None):
    return dict(
        stiffness=np.float64(stiffness), damping=np.float64(damping),
        spacing=np.float64(spacing if spacing is not None else 1.0 / (nx - 1)),
        nx=np.int64(nx), ny=np.int64(ny), dt=np.float64(dt), mass=np.float64(mass),
        drag=np.float64(drag), pressure=np.float64(pressure),
        gravity=np.asarray(gravity, np.float64), plugs=np.asarray(plugs, np.int64),
        pin_nodes=np.asarray(pin_nodes, np.int32),
        pin_anchors=np.asarray(pin_anchors if pin_anchors is not None else np.zeros((0, 3)),
                               np.float64).reshape(-1, 3),
        pin_velocity=np.asarray(pin_velocity, np.float64),
        spheres=np.asarray(spheres, np.float64).reshape(-1, 5),
        planes=np.asarray(planes, np.float64).reshape(-1, 2),
    )


def cloth_desc(z, keep: list, prefix: str = "") -> _abi.sc_cloth_desc:
    g = lambda k: z[prefix + k]  # noqa: E731
    d = _abi.sc_cloth_desc()
    d.dt, d.mass, d.drag, d.pressure = float(g("dt")), float(g("mass")), float(g("drag")), float(
        g("pressure"))
    for i in range(3):
        d.gravity[i] = float(g("gravity")[i])
        d.pin_velocity[i] = float(g("pin_velocity")[i])
    d.plug_pressure, d.plug_gravity, d.plug_drag = (int(v) for v in g("plugs"))
    nodes = np.ascontiguousarray(g("pin_nodes"), np.int32)
    anchors = np.ascontiguousarray(g("pin_anchors"), np.float64)
    sph_a = np.asarray(g("spheres")).reshape(-1, 5)
    pl_a = np.asarray(g("planes")).reshape(-1, 2)
    sph = (_abi.sc_sphere * max(1, len(sph_a)))()
    for k, row in enumerate(sph_a):
        for i in range(3):
            sph[k].center[i] = float(row[i])
        sph[k].radius, sph[k].friction = float(row[3]), float(row[4])
    pl = (_abi.sc_plane * max(1, len(pl_a)))()
    for k, row in enumerate(pl_a):
        pl[k].height, pl[k].friction = float(row[0]), float(row[1])
    keep += [nodes, anchors, sph, pl]
    d.n_pins = len(nodes)
    d.pin_nodes = nodes.ctypes.data_as(C.POINTER(C.c_int32))
    d.pin_anchors = anchors.ctypes.data_as(C.POINTER(C.c_double))
    d.n_spheres = len(sph_a)
    d.spheres = C.cast(sph, C.POINTER(_abi.sc_sphere))
    d.n_planes = len(pl_a)
    d.planes = C.cast(pl, C.POINTER(_abi.sc_plane))
    # fixtures written before the PBS fields existed default to no springs
    d.stiffness = float(z[prefix + "stiffness"]) if prefix + "stiffness" in z else 0.0
    d.damping = float(z[prefix + "damping"]) if prefix + "damping" in z else 0.0
    nx = int(z[prefix + "nx"])
    d.spacing = float(z[prefix + "spacing"]) if prefix + "spacing" in z else 1.0 / (nx - 1)
    return d


def params_c(scalars) -> _abi.sc_params:
    s = [float(v) for v in scalars]
    p = _abi.sc_params()
    for i in range(12):
        p.kernel_gain[i] = s[i]
        p.linear_w[i] = s[12 + i]
        p.nonlinear_w[i] = s[27 + i]
        p.deriv_w[i] = s[39 + i]
    for i in range(3):
        p.linear_b[i] = s[24 + i]
    p.self_velocity_w = s[51]
    p.isru_alpha = s[52]
    return p


def to_scene(z, x0=None):
    """paper_2403_12820_b200.Scene for a fixture (for the Python API tests)."""
    from paper_2403_12820_b200 import PlaneCollider, PlugForce, Scene, SphereCollider

    nx, ny = int(z["nx"]), int(z["ny"])
    s = Scene(nx, ny, float(z["spacing"]) if "spacing" in z else 1.0 / (nx - 1), x0)
    s.dt = float(z["dt"])
    if "stiffness" in z:
        s.material.stiffness = float(z["stiffness"])
        s.material.damping = float(z["damping"])
    s.material.mass = float(z["mass"])
    s.material.drag = float(z["drag"])
    s.material.pressure = float(z["pressure"])
    s.material.gravity = np.array(z["gravity"], np.float64)
    s.plug_forces = [f for f, on in zip((PlugForce.Pressure, PlugForce.Gravity, PlugForce.Drag),
                                        z["plugs"]) if on]
    s.bc.nodes = [int(i) for i in z["pin_nodes"]]
    s.bc.anchors = np.array(z["pin_anchors"], np.float64).reshape(-1, 3)
    pv = np.array(z["pin_velocity"], np.float64)
    s.bc.motion = pv if np.any(pv != 0) else None
    s.colliders = [SphereCollider(np.array(r[:3]), float(r[3]), float(r[4]))
                   for r in np.asarray(z["spheres"]).reshape(-1, 5)]
    s.planes = [PlaneCollider(float(r[0]), float(r[1]))
                for r in np.asarray(z["planes"]).reshape(-1, 2)]
    return s


def load(name: str):
    return np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
