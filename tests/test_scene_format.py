"""The Python scene model / JSON parser (paper_2403_12820_b200/scene.py, a restatement of
io.cpp:30-371 and scene.cpp:23-61) against the reference's own parser (its pybind module built
from /root/reference into oracle/_ref by integration/Makefile), plus the reference-type helpers
(NetworkParams defaults and scalar order, fingerprint, channel hash)."""
import os
import sys

import numpy as np
import pytest

import paper_2403_12820_b200 as mine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref")

SCENES = [
    """{"name": "a", "grid": {"nx": 9, "ny": 6, "spacing": 0.05, "origin": [0.1, -0.2, 0.3],
        "plane": "xz"}, "material": {"stiffness": 20, "damping": 0.1, "mass": 0.02,
        "gravity": [0, -9.8, 0], "drag": 0.01, "pressure": 1.5, "pressure_side": -1},
        "time": {"dt": 0.001, "steps": 12}, "pins": {"nodes": ["top_row", 3, "bottom_left"],
        "motion": {"velocity": [0.1, 0, 0]}},
        "colliders": [{"type": "sphere", "center": [0, 0, 0], "radius": 0.2, "friction": 0.3}],
        "plug_forces": ["gravity", "pressure"]}""",
    """{"grid": {"nx": 5, "ny": 7, "spacing": 0.1, "plane": "yz"},
        "material": {"stiffness": 10, "damping": 0, "mass": 1}, "time": {"steps": 3},
        "pins": {"nodes": "edges"}}""",
    """{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 0, "damping": 0,
        "mass": 2, "drag": 0.5}, "time": {"dt": 0.01, "steps": 0},
        "pins": {"nodes": ["top_left", "top_right", "left_column", "right_column"]},
        "plug_forces": ["drag"]}""",
]

BAD = [
    '{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}, "color": 3}',
    '{"grid": {"nx": 1, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}}',
    '{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}, "pins": {"nodes": "middle"}}',
    '{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}, "colliders": [{"type": "box", "center": [0,0,0], "radius": 1}]}',
    '{"grid": {"nx": 4.0, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}}',
    '{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 0, "damping": 0, "mass": 1}, "time": {"steps": 1}}',
    '{"grid": {"nx": 4, "ny": 4, "spacing": 0.2}, "material": {"stiffness": 1, "damping": 0, "mass": 1}, "time": {"steps": 1}, "plug_forces": ["gravity", "gravity"]}',
    "{",
]


def _ref():
    if not os.path.isdir(os.path.join(REF_PKG, "stencilcloth")):
        pytest.skip("reference module not built (integration/Makefile needs /root/reference)")
    if REF_PKG not in sys.path:
        sys.path.insert(0, REF_PKG)
    import stencilcloth
    return stencilcloth


@pytest.mark.parametrize("text", SCENES)
def test_parse_scene_matches_reference_parser(text):
    sc = _ref()
    r = sc.parse_scene(text)
    m = mine.parse_scene(text)
    assert (m.nx, m.ny, m.spacing, m.dt, m.steps) == (r.nx, r.ny, r.spacing, r.dt, r.steps)
    assert m.node_count == r.node_count and m.spring_count == r.spring_count
    assert m.pinned_nodes == list(r.pinned_nodes)
    assert np.array_equal(m.initial_positions(), r.initial_positions())
    assert m.stable_dt() == r.stable_dt()


@pytest.mark.parametrize("text", BAD)
def test_parse_errors_match_reference(text):
    sc = _ref()
    with pytest.raises(ValueError) as e_ref:
        sc.parse_scene(text)
    with pytest.raises(ValueError) as e_mine:
        mine.parse_scene(text)
    # same offending field path at the front of the message (io.cpp:30-49)
    assert str(e_mine.value).split(":")[0] == str(e_ref.value).split(":")[0]


def test_network_params_defaults_and_fingerprint():
    sc = _ref()
    r, m = sc.NetworkParams(), mine.NetworkParams()
    assert list(r.scalars()) == m.scalars()
    assert r.fingerprint == m.fingerprint
    assert sc.channel_order_hash() == mine.channel_order_hash()
