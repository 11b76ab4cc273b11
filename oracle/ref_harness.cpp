// TEST INFRASTRUCTURE ONLY — C-ABI harness over the UNMODIFIED reference implementation.
//
// oracle/Makefile compiles this file together with the reference's own sources, in place
// under /root/reference/proj/src (grid, scene, sim, net, eval, io, threads — cli.cpp is left
// out because CLI11 is absent), into oracle/_ref/libstencilcloth_ref.so. Nothing here
// re-implements the arithmetic: every number comes from the reference templates
//   detail::forward_impulse<T> / add_plug_impulse<T> / advance_with_impulse<T>
//   (include/cloth/detail/kernels.hpp:179-282)
// or its public API (forward_impulse net.cpp:132-142, nn_step net.cpp:242-248,
// advance_with_impulse sim.cpp:134-148, rollout eval.cpp:86-103, benchmark_net
// eval.cpp:155-158). The f32 rollout replicates the 4-line run_steps<float> sequence
// (eval.cpp:48-59), which lives in an anonymous namespace and returns only seconds.
//
// Used by tests/golden/make_golden.py (fixture generation), the tests, and bench.py's
// `--impl reference` / cpu_baseline legs (the reference CPU path timed on the host).
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cloth/detail/kernels.hpp"
#include "cloth/detail/net_kernel.hpp"
#include "cloth/error.hpp"
#include "cloth/eval.hpp"
#include "cloth/io.hpp"
#include "cloth/net.hpp"
#include "cloth/sim.hpp"
#include "cloth/threads.hpp"
#include "cloth/train.hpp"

#include "../include/stencilcloth_b200.h"

using namespace cloth;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

NetworkParams to_params(const sc_params* p) {
  NetworkParams q;
  for (int c = 0; c < kChannels; ++c) {
    q.kernel_gain[c] = p->kernel_gain[c];
    q.linear_w[c] = p->linear_w[c];
    q.nonlinear_w[c] = p->nonlinear_w[c];
    q.deriv_w[c] = p->deriv_w[c];
  }
  q.linear_b = {p->linear_b[0], p->linear_b[1], p->linear_b[2]};
  q.self_velocity_w = p->self_velocity_w;
  q.isru_alpha = p->isru_alpha;
  return q;
}

// A reference Scene for one cloth descriptor. Initial state: the given positions/velocities
// (double), else the flat build_grid sheet.
Scene to_scene(int nx, int ny, const sc_cloth_desc* cd, const double* x0, const double* v0) {
  GridInit g = build_grid(nx, ny, cd->spacing > 0.0 ? cd->spacing : 1.0 / (nx - 1), Vec3{},
                          GridPlane::XY);
  Scene s;
  s.name = "harness";
  s.topology = std::move(g.topology);
  s.initial = std::move(g.state);
  const size_t n = static_cast<size_t>(nx) * ny;
  if (x0)
    for (size_t i = 0; i < n; ++i) s.initial.x[i] = {x0[3 * i], x0[3 * i + 1], x0[3 * i + 2]};
  if (v0)
    for (size_t i = 0; i < n; ++i) s.initial.v[i] = {v0[3 * i], v0[3 * i + 1], v0[3 * i + 2]};
  s.material.stiffness = cd->stiffness;
  s.material.damping = cd->damping;
  s.material.mass = cd->mass;
  s.material.drag = cd->drag;
  s.material.pressure = cd->pressure;
  s.material.gravity = {cd->gravity[0], cd->gravity[1], cd->gravity[2]};
  s.dt = cd->dt;
  s.steps = 0;
  for (int p = 0; p < cd->n_pins; ++p) {
    s.bc.nodes.push_back(cd->pin_nodes[p]);
    s.bc.anchors.push_back(
        {cd->pin_anchors[3 * p], cd->pin_anchors[3 * p + 1], cd->pin_anchors[3 * p + 2]});
  }
  if (cd->pin_velocity[0] != 0.0 || cd->pin_velocity[1] != 0.0 || cd->pin_velocity[2] != 0.0)
    s.bc.motion = PinMotion{{cd->pin_velocity[0], cd->pin_velocity[1], cd->pin_velocity[2]}};
  for (int k = 0; k < cd->n_spheres; ++k) {
    const sc_sphere& sp = cd->spheres[k];
    s.colliders.push_back({{sp.center[0], sp.center[1], sp.center[2]}, sp.radius, sp.friction});
  }
  if (cd->plug_pressure) s.plug_forces.push_back(PlugForce::Pressure);
  if (cd->plug_gravity) s.plug_forces.push_back(PlugForce::Gravity);
  if (cd->plug_drag) s.plug_forces.push_back(PlugForce::Drag);
  return s;
}

template <typename T>
void copy_in(std::vector<VecT<T>>& dst, const T* src, size_t n) {
  dst.resize(n);
  for (size_t i = 0; i < n; ++i) dst[i] = {src[3 * i], src[3 * i + 1], src[3 * i + 2]};
}

template <typename T>
void copy_out(T* dst, const std::vector<VecT<T>>& src) {
  for (size_t i = 0; i < src.size(); ++i) {
    dst[3 * i] = src[i].x;
    dst[3 * i + 1] = src[i].y;
    dst[3 * i + 2] = src[i].z;
  }
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return SC_OK;
  } catch (const ConfigError& e) {
    return fail(SC_ERR_CONFIG, e.what());
  } catch (const NumericsError& e) {
    return fail(SC_ERR_NUMERICS, e.what());
  } catch (const std::exception& e) {
    return fail(SC_ERR_STATE, e.what());
  }
}

// run_steps<T> step sequence (eval.cpp:48-59) for one cloth, state advanced in place.
template <typename T>
void run_cloth(int nx, int ny, const sc_cloth_desc* cd, const NetworkParams& params, T* x, T* v,
               int steps, int k0, uint8_t* constrained_last) {
  const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
  const auto kernel = detail::make_scene_kernel<T>(scene);
  const detail::NetKernel<T> net = detail::make_net_kernel<T>(params);
  const size_t n = static_cast<size_t>(nx) * ny;
  std::vector<VecT<T>> xs, vs, xn(n), vn(n), imp(n);
  copy_in(xs, x, n);
  copy_in(vs, v, n);
  for (int k = k0; k < k0 + steps; ++k) {
    const T t_next = static_cast<T>(k + 1) * kernel.dt;
    detail::forward_impulse(xs.data(), vs.data(), scene.topology, net, imp.data());
    detail::add_plug_impulse(xs.data(), vs.data(), kernel, imp.data());
    detail::advance_with_impulse(xs.data(), vs.data(), imp.data(), kernel, t_next, xn.data(),
                                 vn.data(),
                                 (constrained_last && k == k0 + steps - 1) ? constrained_last
                                                                            : nullptr);
    xs.swap(xn);
    vs.swap(vn);
  }
  copy_out(x, xs);
  copy_out(v, vs);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_set_threads(int n) { set_thread_count(n); }
int ref_threads(void) { return thread_count(); }

// run_steps<float>/<double> sequence over a batch (eval.cpp:35-67), state in place.
int ref_rollout_f32(int nx, int ny, int batch, const sc_cloth_desc* cloths, const sc_params* p,
                    float* x, float* v, int steps, int k0, uint8_t* constrained_last) {
  return guarded([&] {
    const NetworkParams params = to_params(p);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (int b = 0; b < batch; ++b) {
      if (cloths[b].n_planes > 0) throw ConfigError("planes: no reference implementation");
      run_cloth<float>(nx, ny, &cloths[b], params, x + 3 * n * b, v + 3 * n * b, steps, k0,
                       constrained_last ? constrained_last + n * b : nullptr);
    }
  });
}

int ref_rollout_tmpl_f64(int nx, int ny, int batch, const sc_cloth_desc* cloths,
                         const sc_params* p, double* x, double* v, int steps, int k0,
                         uint8_t* constrained_last) {
  return guarded([&] {
    const NetworkParams params = to_params(p);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (int b = 0; b < batch; ++b) {
      if (cloths[b].n_planes > 0) throw ConfigError("planes: no reference implementation");
      run_cloth<double>(nx, ny, &cloths[b], params, x + 3 * n * b, v + 3 * n * b, steps, k0,
                        constrained_last ? constrained_last + n * b : nullptr);
    }
  });
}

// One f32 step with the impulse exposed (forward + plug), the advance mask, from the
// reference templates.
int ref_step_f32(int nx, int ny, const sc_cloth_desc* cd, const sc_params* p, const float* x,
                 const float* v, float t_next, float* xo, float* vo, uint8_t* constrained,
                 float* impulse) {
  return guarded([&] {
    if (cd->n_planes > 0) throw ConfigError("planes: no reference implementation");
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    const auto kernel = detail::make_scene_kernel<float>(scene);
    const auto net = detail::make_net_kernel<float>(to_params(p));
    const size_t n = static_cast<size_t>(nx) * ny;
    std::vector<Vec3f> xs, vs, xn(n), vn(n), imp(n);
    copy_in(xs, x, n);
    copy_in(vs, v, n);
    detail::forward_impulse(xs.data(), vs.data(), scene.topology, net, imp.data());
    detail::add_plug_impulse(xs.data(), vs.data(), kernel, imp.data());
    detail::advance_with_impulse(xs.data(), vs.data(), imp.data(), kernel, t_next, xn.data(),
                                 vn.data(), constrained);
    copy_out(xo, xn);
    copy_out(vo, vn);
    if (impulse) copy_out(impulse, imp);
  });
}

// ---- the reference's public double-precision API ----------------------------------------

int ref_forward_impulse_f64(int nx, int ny, const sc_params* p, const double* x,
                            const double* v, double* out) {
  return guarded([&] {
    const GridInit g = build_grid(nx, ny, 1.0 / (nx - 1), Vec3{}, GridPlane::XY);
    ClothState s;
    copy_in(s.x, x, static_cast<size_t>(nx) * ny);
    copy_in(s.v, v, static_cast<size_t>(nx) * ny);
    copy_out(out, forward_impulse(s, g.topology, to_params(p)));
  });
}

int ref_plug_impulse_f64(int nx, int ny, const sc_cloth_desc* cd, const double* x,
                         const double* v, double* out) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    ClothState s;
    copy_in(s.x, x, static_cast<size_t>(nx) * ny);
    copy_in(s.v, v, static_cast<size_t>(nx) * ny);
    copy_out(out, plug_impulse(s, scene));
  });
}

int ref_advance_with_impulse_f64(int nx, int ny, const sc_cloth_desc* cd, const double* x,
                                 const double* v, const double* imp, double t_next, double* xo,
                                 double* vo, uint8_t* constrained) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    const size_t n = static_cast<size_t>(nx) * ny;
    ClothState s;
    copy_in(s.x, x, n);
    copy_in(s.v, v, n);
    Vec3Field impulse;
    copy_in(impulse, imp, n);
    std::vector<uint8_t> mask;
    const ClothState out =
        advance_with_impulse(s, impulse, scene, t_next, constrained ? &mask : nullptr);
    copy_out(xo, out.x);
    copy_out(vo, out.v);
    if (constrained) std::memcpy(constrained, mask.data(), n);
  });
}

int ref_nn_step_f64(int nx, int ny, const sc_cloth_desc* cd, const sc_params* p,
                    const double* x, const double* v, double t_next, double* xo, double* vo) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    ClothState s;
    copy_in(s.x, x, static_cast<size_t>(nx) * ny);
    copy_in(s.v, v, static_cast<size_t>(nx) * ny);
    const ClothState out = nn_step(s, scene, to_params(p), t_next);
    copy_out(xo, out.x);
    copy_out(vo, out.v);
  });
}

// rollout (eval.cpp:86-103): frames [(steps+1)][n][3]; frame 0 = apply_dirichlet(initial, 0).
int ref_rollout_f64(int nx, int ny, const sc_cloth_desc* cd, const sc_params* p,
                    const double* x0, const double* v0, int steps, double* frames_x,
                    double* frames_v) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, x0, v0);
    const Trajectory t = rollout(to_params(p), scene, steps);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (int f = 0; f < t.frame_count(); ++f) {
      copy_out(frames_x + 3 * n * f, t.frames[static_cast<size_t>(f)].x);
      copy_out(frames_v + 3 * n * f, t.frames[static_cast<size_t>(f)].v);
    }
  });
}

// ---- the ground-truth mass-spring step (PBS) --------------------------------------------

int ref_total_impulse_f64(int nx, int ny, const sc_cloth_desc* cd, const double* x,
                          const double* v, double* out) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    ClothState s;
    copy_in(s.x, x, static_cast<size_t>(nx) * ny);
    copy_in(s.v, v, static_cast<size_t>(nx) * ny);
    copy_out(out, total_impulse(s, scene));
  });
}

int ref_pbs_step_f64(int nx, int ny, const sc_cloth_desc* cd, const double* x, const double* v,
                     double t_next, double* xo, double* vo) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    ClothState s;
    copy_in(s.x, x, static_cast<size_t>(nx) * ny);
    copy_in(s.v, v, static_cast<size_t>(nx) * ny);
    const ClothState out = step_semi_implicit(s, scene, t_next);
    copy_out(xo, out.x);
    copy_out(vo, out.v);
  });
}

// simulate_scene (sim.cpp:157-175): frames [(steps+1)][n][3].
int ref_simulate_f64(int nx, int ny, const sc_cloth_desc* cd, const double* x0, const double* v0,
                     int steps, double* frames_x, double* frames_v) {
  return guarded([&] {
    Scene scene = to_scene(nx, ny, cd, x0, v0);
    scene.steps = steps;
    const Trajectory t = simulate_scene(scene);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (int f = 0; f < t.frame_count(); ++f) {
      copy_out(frames_x + 3 * n * f, t.frames[static_cast<size_t>(f)].x);
      copy_out(frames_v + 3 * n * f, t.frames[static_cast<size_t>(f)].v);
    }
  });
}

// run_steps<float> with params == nullptr (eval.cpp:53-55): the benchmark_sim sequence.
int ref_pbs_rollout_f32(int nx, int ny, const sc_cloth_desc* cd, float* x, float* v, int steps,
                        int k0) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, nullptr, nullptr);
    const auto kernel = detail::make_scene_kernel<float>(scene);
    const size_t n = static_cast<size_t>(nx) * ny;
    std::vector<Vec3f> xs, vs, xn(n), vn(n), imp(n);
    copy_in(xs, x, n);
    copy_in(vs, v, n);
    for (int k = k0; k < k0 + steps; ++k) {
      detail::total_impulse(xs.data(), vs.data(), kernel, imp.data());
      detail::advance_with_impulse(xs.data(), vs.data(), imp.data(), kernel,
                                   static_cast<float>(k + 1) * kernel.dt, xn.data(), vn.data(),
                                   nullptr);
      xs.swap(xn);
      vs.swap(vn);
    }
    copy_out(x, xs);
    copy_out(v, vs);
  });
}

int ref_benchmark_sim(int nx, int ny, const sc_cloth_desc* cd, const double* x0,
                      const double* v0, int steps, int warmup, int f64, int threads,
                      double* seconds) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, x0, v0);
    const int before = thread_count();
    set_thread_count(threads);
    const BenchResult r =
        benchmark_sim(scene, steps, warmup, f64 ? Precision::F64 : Precision::F32);
    set_thread_count(before);
    *seconds = r.seconds;
  });
}

// benchmark_net (eval.cpp:155-158) — the reference's own timer around run_steps<T>.
// threads: node-parallel OpenMP thread count for this call (CLOTHSIM_THREADS semantics).
int ref_benchmark_net(int nx, int ny, const sc_cloth_desc* cd, const sc_params* p,
                      const double* x0, const double* v0, int steps, int warmup, int f64,
                      int threads, double* seconds) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, x0, v0);
    const int before = thread_count();
    set_thread_count(threads);
    const BenchResult r = benchmark_net(to_params(p), scene, steps, warmup,
                                        f64 ? Precision::F64 : Precision::F32);
    set_thread_count(before);
    *seconds = r.seconds;
  });
}

// Cloth-parallel variant: `ncloth` independent cloths, one std::thread each with the global
// thread count at 1 (reference code unchanged). Returns the wall time of the slowest cloth's
// benchmark_net timed region and the wall time of the whole parallel region.
int ref_benchmark_net_cloth_parallel(int nx, int ny, int ncloth, const sc_cloth_desc* cloths,
                                     const sc_params* p, const double* x0, const double* v0,
                                     int steps, int warmup, double* max_seconds,
                                     double* wall_seconds) {
  return guarded([&] {
    const int before = thread_count();
    set_thread_count(1);
    const NetworkParams params = to_params(p);
    const size_t n = static_cast<size_t>(nx) * ny;
    std::vector<Scene> scenes;
    for (int b = 0; b < ncloth; ++b)
      scenes.push_back(to_scene(nx, ny, &cloths[b], x0 ? x0 + 3 * n * b : nullptr,
                                v0 ? v0 + 3 * n * b : nullptr));
    std::vector<double> secs(static_cast<size_t>(ncloth), 0.0);
    std::atomic<int> err{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int b = 0; b < ncloth; ++b)
      pool.emplace_back([&, b] {
        try {
          secs[static_cast<size_t>(b)] =
              benchmark_net(params, scenes[static_cast<size_t>(b)], steps, warmup,
                            Precision::F32)
                  .seconds;
        } catch (...) {
          err = 1;
        }
      });
    for (auto& t : pool) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    set_thread_count(before);
    if (err) throw NumericsError("cloth-parallel benchmark failed");
    double mx = 0.0;
    for (double s : secs) mx = std::max(mx, s);
    *max_seconds = mx;
    *wall_seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// ---- training (train.cpp, net.cpp:144-201): the reference's own sample_batch / compute_loss /
// backward_gradients / train_loop over a trajectory given as [frames][n][3] arrays.
namespace {
Trajectory make_traj(int nx, int ny, const sc_cloth_desc* cd, int frames, const double* fx,
                     const double* fv) {
  Trajectory t;
  t.nx = nx;
  t.ny = ny;
  t.dt = cd->dt;
  t.spacing = cd->spacing > 0.0 ? cd->spacing : 1.0 / (nx - 1);
  const size_t n = static_cast<size_t>(nx) * ny;
  t.frames.resize(static_cast<size_t>(frames));
  for (int f = 0; f < frames; ++f) {
    copy_in(t.frames[static_cast<size_t>(f)].x, fx + 3 * n * f, n);
    copy_in(t.frames[static_cast<size_t>(f)].v, fv + 3 * n * f, n);
  }
  return t;
}
void flat_grads(const ParamGradients& g, double* out) {
  ParamGradients c = g;
  int k = 0;
  for_each_gradient(c, [&](ParamGroup, int, double& v) { out[k++] = v; });
}
}  // namespace

extern "C" {

int ref_sample_batch(int nx, int ny, const sc_cloth_desc* cd, int frames, const double* fx,
                     const double* fv, int batch_size, uint64_t seed, int32_t* idx_out,
                     double* force_dt_out) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, fx, fv);
    const Trajectory traj = make_traj(nx, ny, cd, frames, fx, fv);
    Rng rng(seed);
    const TrainBatch b = sample_batch(traj, scene, batch_size, rng);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (size_t k = 0; k < b.indices.size(); ++k) {
      if (idx_out) idx_out[k] = b.indices[k];
      if (force_dt_out) copy_out(force_dt_out + 3 * n * k, b.force_dt[k]);
    }
  });
}

int ref_compute_loss(int nx, int ny, const sc_cloth_desc* cd, int frames, const double* fx,
                     const double* fv, int batch_size, uint64_t seed, const sc_params* p,
                     double alpha, int want_grads, double* loss_out, double* grads_out) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, fx, fv);
    const Trajectory traj = make_traj(nx, ny, cd, frames, fx, fv);
    Rng rng(seed);
    TrainBatch b = sample_batch(traj, scene, batch_size, rng);
    b.traj = &traj;
    b.scene = &scene;
    ParamGradients g;
    const LossValue l = compute_loss(to_params(p), b, alpha, want_grads ? &g : nullptr);
    loss_out[0] = l.total;
    loss_out[1] = l.physics;
    loss_out[2] = l.data;
    if (want_grads) flat_grads(g, grads_out);
  });
}

int ref_backward_gradients(int nx, int ny, const double* x, const double* v, const sc_params* p,
                           const double* upstream, double* grads_out) {
  return guarded([&] {
    const GridInit g = build_grid(nx, ny, 1.0, Vec3{}, GridPlane::XY);
    ClothState s;
    const size_t n = static_cast<size_t>(nx) * ny;
    copy_in(s.x, x, n);
    copy_in(s.v, v, n);
    Vec3Field u;
    copy_in(u, upstream, n);
    flat_grads(backward_gradients(s, g.topology, to_params(p), u), grads_out);
  });
}

int ref_train(int nx, int ny, const sc_cloth_desc* cd, int frames, const double* fx,
              const double* fv, const sc_train_config* c, sc_params* params_out,
              uint8_t* trainable_out, double* history_out, double* brackets_out) {
  return guarded([&] {
    const Scene scene = to_scene(nx, ny, cd, fx, fv);
    const Trajectory traj = make_traj(nx, ny, cd, frames, fx, fv);
    TrainConfig cfg;
    cfg.alpha = c->alpha;
    cfg.batch_size = c->batch_size;
    cfg.epochs = c->epochs;
    cfg.schedule.kind = c->schedule_kind ? ScheduleKind::Cosine : ScheduleKind::Step;
    cfg.schedule.lr0 = c->lr0;
    cfg.schedule.gamma = c->gamma;
    cfg.schedule.interval = c->interval;
    cfg.schedule.floor = c->floor;
    cfg.schedule.period = c->period;
    cfg.seed = c->seed;
    cfg.de.population = c->de_population;
    cfg.de.generations = c->de_generations;
    cfg.de.bound = c->de_bound;
    cfg.de.cross_prob = c->de_cross_prob;
    cfg.de.diff_weight = c->de_diff_weight;
    cfg.de.probe_batch = c->de_probe_batch;
    cfg.checkpoint_interval = c->checkpoint_interval;
    for (int g = 0; g < kParamGroups; ++g)
      if (c->freeze_mask & (1u << g)) cfg.freeze.push_back(static_cast<ParamGroup>(g));
    const TrainResult r = train_loop(cfg, scene, traj);
    NetworkParams q = r.params;
    int k = 0;
    double flat[NetworkParams::kScalarCount];
    for_each_scalar(q, [&](ParamGroup, int, double& v) { flat[k++] = v; });
    for (int i = 0; i < kChannels; ++i) {
      params_out->kernel_gain[i] = flat[i];
      params_out->linear_w[i] = flat[12 + i];
      params_out->nonlinear_w[i] = flat[27 + i];
      params_out->deriv_w[i] = flat[39 + i];
    }
    for (int d = 0; d < 3; ++d) params_out->linear_b[d] = flat[24 + d];
    params_out->self_velocity_w = flat[51];
    params_out->isru_alpha = flat[52];
    for (int g = 0; g < kParamGroups; ++g) {
      if (trainable_out) trainable_out[g] = q.is_trainable(static_cast<ParamGroup>(g)) ? 1 : 0;
      if (brackets_out) {
        brackets_out[2 * g] = q.brackets[static_cast<size_t>(g)].lo;
        brackets_out[2 * g + 1] = q.brackets[static_cast<size_t>(g)].hi;
      }
    }
    if (history_out)
      for (size_t e = 0; e < r.history.size(); ++e) {
        history_out[5 * e] = r.history[e].step;
        history_out[5 * e + 1] = r.history[e].lr;
        history_out[5 * e + 2] = r.history[e].physics;
        history_out[5 * e + 3] = r.history[e].data;
        history_out[5 * e + 4] = r.history[e].total;
      }
  });
}

}  // extern "C"

// Scene JSON parsing through the reference parser (io.cpp:199-359), for checking the Python
// mirror's parser. Returns counts; arrays are filled when non-null and large enough.
int ref_parse_scene(const char* json_text, int* nx, int* ny, double* spacing, double* dt,
                    int* steps, double* material /*stiffness,damping,mass,drag,pressure,gx,gy,gz*/,
                    int* n_pins, int* pins, double* anchors, int pins_cap, int* n_spheres,
                    double* spheres /*cx,cy,cz,r,fr*/, int spheres_cap, int* plugs /*p,g,d*/,
                    double* initial_x) {
  return guarded([&] {
    const Scene s = parse_scene_config(json_text);
    *nx = s.topology.nx;
    *ny = s.topology.ny;
    *spacing = s.topology.spacing;
    *dt = s.dt;
    *steps = s.steps;
    const double m[8] = {s.material.stiffness, s.material.damping, s.material.mass,
                         s.material.drag,      s.material.pressure, s.material.gravity.x,
                         s.material.gravity.y, s.material.gravity.z};
    std::memcpy(material, m, sizeof m);
    *n_pins = static_cast<int>(s.bc.nodes.size());
    for (int k = 0; k < *n_pins && k < pins_cap; ++k) {
      pins[k] = s.bc.nodes[static_cast<size_t>(k)];
      anchors[3 * k] = s.bc.anchors[static_cast<size_t>(k)].x;
      anchors[3 * k + 1] = s.bc.anchors[static_cast<size_t>(k)].y;
      anchors[3 * k + 2] = s.bc.anchors[static_cast<size_t>(k)].z;
    }
    *n_spheres = static_cast<int>(s.colliders.size());
    for (int k = 0; k < *n_spheres && k < spheres_cap; ++k) {
      const SphereCollider& c = s.colliders[static_cast<size_t>(k)];
      const double row[5] = {c.center.x, c.center.y, c.center.z, c.radius, c.friction};
      std::memcpy(spheres + 5 * k, row, sizeof row);
    }
    plugs[0] = s.plugs(PlugForce::Pressure);
    plugs[1] = s.plugs(PlugForce::Gravity);
    plugs[2] = s.plugs(PlugForce::Drag);
    if (initial_x) copy_out(initial_x, s.initial.x);
  });
}

}  // extern "C"
