// Python drop-in for the reference's rollout / forward_impulse (python/bindings.cpp:147-164):
// a pybind11 module compiled against the reference headers that accepts the reference's OWN
// `stencilcloth.Scene` / `stencilcloth.NetworkParams` objects (pybind11 shares the type
// registrations of stencilcloth._core) and runs the B200 kernels through the C-ABI
// (include/stencilcloth_b200.h), returning the reference's own `stencilcloth.Trajectory`.
//
//   import stencilcloth as sc, stencilcloth_b200_adapter as gpu
//   traj = gpu.rollout(params, scene, steps)      # was: sc.rollout(params, scene, steps)
//
// Built by integration/Makefile where /root/reference exists (output in oracle/_ref/, which is
// git-ignored and travels to the GPU box). Double precision, PARITY mode: bit-identical frames.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "cloth/error.hpp"
#include "cloth/grid.hpp"
#include "cloth/net.hpp"
#include "cloth/scene.hpp"
#include "stencilcloth_b200.h"

namespace py = pybind11;

namespace {

void check(int rc) {
  if (rc == SC_OK) return;
  const std::string msg = sc_last_error();
  if (rc == SC_ERR_CONFIG) throw cloth::ConfigError(msg);
  if (rc == SC_ERR_NUMERICS) throw cloth::NumericsError(msg);
  throw std::runtime_error("stencilcloth_b200: " + msg);
}

struct Ctx {
  sc_ctx* h = nullptr;
  ~Ctx() { sc_ctx_destroy(h); }
};

sc_params to_c(const cloth::NetworkParams& p) {
  sc_params c{};
  for (int i = 0; i < SC_CHANNELS; ++i) {
    c.kernel_gain[i] = p.kernel_gain[i];
    c.linear_w[i] = p.linear_w[i];
    c.nonlinear_w[i] = p.nonlinear_w[i];
    c.deriv_w[i] = p.deriv_w[i];
  }
  c.linear_b[0] = p.linear_b.x;
  c.linear_b[1] = p.linear_b.y;
  c.linear_b[2] = p.linear_b.z;
  c.self_velocity_w = p.self_velocity_w;
  c.isru_alpha = p.isru_alpha;
  return c;
}

// The per-cloth part of cloth::Scene (scene.hpp:43-60) as the C-ABI descriptor.
struct Desc {
  sc_cloth_desc d{};
  std::vector<int32_t> pins;
  std::vector<double> anchors;
  std::vector<sc_sphere> spheres;
};

void fill(const cloth::Scene& s, Desc& out) {
  sc_cloth_desc& d = out.d;
  d.dt = s.dt;
  d.mass = s.material.mass;
  d.drag = s.material.drag;
  d.pressure = s.material.pressure;
  d.gravity[0] = s.material.gravity.x;
  d.gravity[1] = s.material.gravity.y;
  d.gravity[2] = s.material.gravity.z;
  // Scene::plugs (scene.cpp:13-15) lives in stencilcloth._core with hidden visibility
  auto plugs = [&](cloth::PlugForce f) {
    return std::find(s.plug_forces.begin(), s.plug_forces.end(), f) != s.plug_forces.end();
  };
  d.plug_pressure = plugs(cloth::PlugForce::Pressure);
  d.plug_gravity = plugs(cloth::PlugForce::Gravity);
  d.plug_drag = plugs(cloth::PlugForce::Drag);
  out.pins.assign(s.bc.nodes.begin(), s.bc.nodes.end());
  for (const cloth::Vec3& a : s.bc.anchors) out.anchors.insert(out.anchors.end(), {a.x, a.y, a.z});
  d.n_pins = static_cast<int32_t>(out.pins.size());
  d.pin_nodes = out.pins.data();
  d.pin_anchors = out.anchors.data();
  const cloth::Vec3 u = s.bc.pin_velocity();
  d.pin_velocity[0] = u.x;
  d.pin_velocity[1] = u.y;
  d.pin_velocity[2] = u.z;
  for (const cloth::SphereCollider& c : s.colliders)
    out.spheres.push_back({{c.center.x, c.center.y, c.center.z}, c.radius, c.friction});
  d.n_spheres = static_cast<int32_t>(out.spheres.size());
  d.spheres = out.spheres.data();
  d.n_planes = 0;
  d.planes = nullptr;
}

void bind(Ctx& c, const cloth::Scene& s, const cloth::NetworkParams& p) {
  check(sc_ctx_create(0, SC_F64, &c.h));
  Desc desc;
  fill(s, desc);
  sc_scene_desc sd{s.topology.nx, s.topology.ny, 1, &desc.d};
  check(sc_ctx_set_scene(c.h, &sd));
  const sc_params pc = to_c(p);
  check(sc_ctx_set_params(c.h, &pc));
}

// Branch naming of a non-finite cell impulse (net.cpp:30-51), failure path only.
std::string diagnose(const double* x, const double* v, const cloth::Scene& s,
                     const cloth::NetworkParams& p, int node) {
  static const int off[12][2] = {{1, 0},  {0, 1},  {-1, 0}, {0, -1}, {1, 1},  {-1, 1},
                                 {-1, -1}, {1, -1}, {2, 0},  {0, 2},  {-2, 0}, {0, -2}};
  const int nx = s.topology.nx, ny = s.topology.ny, ix = node % nx, iy = node / nx;
  double lin[3] = {p.linear_b.x, p.linear_b.y, p.linear_b.z}, non[3] = {0, 0, 0}, der[3];
  for (int d = 0; d < 3; ++d) der[d] = v[3 * node + d] * p.self_velocity_w;
  for (int c = 0; c < 12; ++c) {
    const int jx = ix + off[c][0], jy = iy + off[c][1];
    if (jx < 0 || jx >= nx || jy < 0 || jy >= ny) continue;
    const int j = jy * nx + jx;
    for (int d = 0; d < 3; ++d) {
      const double phi = (x[3 * node + d] - x[3 * j + d]) * p.kernel_gain[c];
      const double xi = (v[3 * node + d] - v[3 * j + d]) * p.kernel_gain[c];
      const double sg = phi / std::sqrt(1.0 + p.isru_alpha * phi * phi);
      lin[d] += phi * p.linear_w[c];
      non[d] += sg * p.nonlinear_w[c];
      der[d] += xi * sg * p.deriv_w[c];
    }
  }
  auto fin = [](const double* a) {
    return std::isfinite(a[0]) && std::isfinite(a[1]) && std::isfinite(a[2]);
  };
  const char* branch = !fin(lin) ? "linear" : (!fin(non) ? "nonlinear" : "derivative");
  return "network impulse non-finite at node " + std::to_string(node) + " (" + branch +
         " branch)";
}

cloth::Trajectory rollout(const cloth::NetworkParams& p, const cloth::Scene& s, int steps) {
  if (!(p.isru_alpha > 0.0)) throw cloth::ConfigError("isru_alpha: must be > 0");
  if (steps < 0) steps = s.steps;
  const size_t n = static_cast<size_t>(s.topology.node_count());
  if (s.initial.x.size() != n || s.initial.v.size() != n)
    throw cloth::ConfigError("initial state: node count does not match the grid");
  // frame 0 = apply_dirichlet(initial, bc, 0) (eval.cpp:95, sim.cpp:108-117)
  std::vector<double> x0(3 * n), v0(3 * n);
  std::memcpy(x0.data(), s.initial.x.data(), sizeof(double) * 3 * n);
  std::memcpy(v0.data(), s.initial.v.data(), sizeof(double) * 3 * n);
  const cloth::Vec3 u = s.bc.pin_velocity();
  for (size_t k = 0; k < s.bc.nodes.size(); ++k) {
    const cloth::Vec3 a = s.bc.anchor_at(k, 0.0);
    const size_t i = static_cast<size_t>(s.bc.nodes[k]);
    x0[3 * i] = a.x, x0[3 * i + 1] = a.y, x0[3 * i + 2] = a.z;
    v0[3 * i] = u.x, v0[3 * i + 1] = u.y, v0[3 * i + 2] = u.z;
  }
  Ctx c;
  bind(c, s, p);
  const size_t frames = static_cast<size_t>(steps) + 1;
  std::vector<double> fx(frames * 3 * n), fv(frames * 3 * n);
  check(sc_rollout_frames(c.h, x0.data(), v0.data(), steps, 1, SC_MODE_PARITY, fx.data(),
                          fv.data()));
  int32_t bi = -1, bn = -1, bs = -1;
  check(sc_ctx_get_health(c.h, &bi, &bn, &bs));
  if (bi >= 0 && (bs < 0 || bi <= bs))
    throw cloth::NumericsError(diagnose(fx.data() + 3 * n * (bi - 1),
                                        fv.data() + 3 * n * (bi - 1), s, p, bn));
  if (bs >= 0)
    throw cloth::NumericsError("rollout diverged: non-finite state at frame " +
                               std::to_string(bs));
  cloth::Trajectory t;
  t.nx = s.topology.nx;
  t.ny = s.topology.ny;
  t.dt = s.dt;
  t.spacing = s.topology.spacing;
  t.frames.resize(frames);
  for (size_t f = 0; f < frames; ++f) {
    t.frames[f].x.resize(n);
    t.frames[f].v.resize(n);
    std::memcpy(t.frames[f].x.data(), fx.data() + 3 * n * f, sizeof(double) * 3 * n);
    std::memcpy(t.frames[f].v.data(), fv.data() + 3 * n * f, sizeof(double) * 3 * n);
  }
  return t;
}

py::array_t<double> forward_impulse(const cloth::NetworkParams& p, const cloth::Scene& s,
                                    const py::array_t<double, py::array::c_style |
                                                                  py::array::forcecast>& x,
                                    const py::array_t<double, py::array::c_style |
                                                                  py::array::forcecast>& v) {
  if (x.ndim() != 2 || x.shape(1) != 3) throw cloth::ConfigError("positions: expected an (n, 3) array");
  if (v.ndim() != 2 || v.shape(1) != 3) throw cloth::ConfigError("velocities: expected an (n, 3) array");
  if (x.shape(0) != v.shape(0))
    throw cloth::ConfigError("positions and velocities disagree on the node count");
  if (x.shape(0) != s.topology.node_count())
    throw cloth::ConfigError("state shape does not match the grid topology");
  if (!(p.isru_alpha > 0.0)) throw cloth::ConfigError("isru_alpha: must be > 0");
  Ctx c;
  bind(c, s, p);
  py::array_t<double> out({x.shape(0), py::ssize_t(3)});
  check(sc_forward_impulse(c.h, x.data(), v.data(), out.mutable_data()));
  int32_t bi = -1, bn = -1, bs = -1;
  check(sc_ctx_get_health(c.h, &bi, &bn, &bs));
  if (bi >= 0) throw cloth::NumericsError(diagnose(x.data(), v.data(), s, p, bn));
  return out;
}

}  // namespace

PYBIND11_MODULE(stencilcloth_b200_adapter, m) {
  m.doc() = "B200 (sm_100a) drop-in for stencilcloth.rollout / forward_impulse";
  py::module_::import("stencilcloth");  // registers Scene / NetworkParams / Trajectory + errors
  m.def("rollout", &rollout, py::arg("params"), py::arg("scene"), py::arg("steps") = -1,
        py::call_guard<py::gil_scoped_release>());
  m.def("forward_impulse", &forward_impulse, py::arg("params"), py::arg("scene"),
        py::arg("positions"), py::arg("velocities"));
}
