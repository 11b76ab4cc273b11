"""The checker-side workload generator (oracle/workloads.py over oracle/gen.c, used by
bench.py's reference arm so it never loads the product library) reproduces the product's
seeded inputs (paper_2403_12820_b200.configs over csrc/host_gen.cpp) exactly: the same
mt19937_64 draws (rng.hpp:13-47), sheets, weights, wind, pins, anchors and colliders."""
import numpy as np
import pytest

from oracle import workloads as W


def test_rng_streams_match_product():
    from paper_2403_12820_b200 import configs
    for seed, stream in ((0, 0), (1, 7), (4, 0x10005), (12345, 2**40 + 3)):
        m = W.mix(seed, stream)
        assert m == configs.mix(seed, stream)
        assert np.array_equal(W.uniforms(m, 1000), configs.uniforms(m, 1000))
        assert np.array_equal(W.normals(m, 1001, 0.05), configs.normals(m, 1001, 0.05))


@pytest.mark.parametrize("cfg_id,n,batch", [(1, 32, 1), (2, 64, 4), (3, 48, 2), (4, 40, 1),
                                            (5, 32, 6)])
def test_workloads_match_product_configs(cfg_id, n, batch):
    from paper_2403_12820_b200 import configs
    _, scenes, p, x, v = configs.build(cfg_id, batch=batch, n=n, cloth0=3)
    w, cds, keep, pc, xw, vw = W.build(cfg_id, batch=batch, n=n, cloth0=3)
    assert np.array_equal(x.view(np.uint32), xw.view(np.uint32)) and not vw.any()
    q = p.to_c()
    for f in ("kernel_gain", "linear_w", "nonlinear_w", "deriv_w", "linear_b"):
        assert list(getattr(q, f)) == list(getattr(pc, f)), f
    assert q.self_velocity_w == pc.self_velocity_w and q.isru_alpha == pc.isru_alpha
    keep2 = []
    for s, d in zip(scenes, cds):
        e = s.cloth_desc(keep2)
        for f in ("dt", "mass", "drag", "pressure", "plug_pressure", "plug_gravity", "plug_drag",
                  "n_pins", "n_spheres", "n_planes", "spacing"):
            assert getattr(e, f) == getattr(d, f), f
        assert list(e.gravity) == list(d.gravity) and list(e.pin_velocity) == list(d.pin_velocity)
        for k in range(d.n_pins):
            assert e.pin_nodes[k] == d.pin_nodes[k]
            assert [e.pin_anchors[3 * k + i] for i in range(3)] == \
                [d.pin_anchors[3 * k + i] for i in range(3)]
        for k in range(d.n_spheres):
            assert list(e.spheres[k].center) == list(d.spheres[k].center)
            assert (e.spheres[k].radius, e.spheres[k].friction) == \
                (d.spheres[k].radius, d.spheres[k].friction)
        for k in range(d.n_planes):
            assert (e.planes[k].height, e.planes[k].friction) == \
                (d.planes[k].height, d.planes[k].friction)


def test_sheet_rows_are_partition_independent():
    a = W.sheet(3, 0, 40)
    b = W.sheet(3, 0, 40, row0=17, rows=9)
    assert np.array_equal(a[17 * 40:26 * 40], b)
