// C-ABI implementation (include/stencilcloth_b200.h): contexts, validation, constant upload,
// layout conversion at the edges, and launch of the PARITY / FAST step kernels.
//
// Error behaviour mirrors the reference: scene/param validation failures are SC_ERR_CONFIG with
// the field name the reference's ConfigError would carry (scene.cpp:23-61, net.cpp:17-26);
// there is no CPU fallback — a CUDA failure is SC_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/stencilcloth_b200.h"
#include "capi_internal.h"
#include "sc_device.cuh"
#include "sc_kernels.h"

using namespace scb;

namespace {

thread_local std::string g_err;

struct Fail {
  sc_status code;
  std::string msg;
};

[[noreturn]] void throw_config(const std::string& m) { throw Fail{SC_ERR_CONFIG, m}; }
[[noreturn]] void throw_state(const std::string& m) { throw Fail{SC_ERR_STATE, m}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail{SC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

template <typename Fn>
sc_status guarded(Fn&& fn) {
  try {
    fn();
    return SC_OK;
  } catch (const Fail& f) {
    g_err = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SC_ERR_STATE;
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (count == 0) return;
    ck(cudaMalloc(&p, sizeof(T) * count), "cudaMalloc");
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_encodeTiled>(p);
  }();
  return fn;
}

}  // namespace

struct sc_ctx {
  int device = 0;
  sc_precision prec = SC_F32;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // grid / strip
  int nx = 0, ny = 0, batch = 0;
  int strip_row0 = -1, strip_rows = 0;  // requested strip (global rows), -1: whole cloth
  int g0 = 0, rows_local = 0;           // global row of local row 0, local rows
  int u0 = 0, u1 = 0;                   // owned global rows
  int pitch = 0;
  int64_t plane_stride = 0;
  bool zs = false;  // z planes in the z_col swizzle (sc_device.cuh): FAST general-finish contexts
  bool has_scene = false, has_params = false;
  // device memory
  void* state[2] = {nullptr, nullptr};
  size_t state_bytes = 0;
  int cur = 0;
  void* cloths = nullptr;
  void* spheres = nullptr;
  void* planes = nullptr;
  DevBuf<uint32_t> pin_bits;
  DevBuf<int32_t> pin_rank;
  void* anchors = nullptr;
  DevBuf<Health> health;
  DevBuf<uint8_t> mask;
  DevBuf<unsigned char> aos;  // staging for AoS x, v, impulse
  // params
  NetConst<float> net32{};
  NetConst<double> net64{};
  FastNet fast{};
  bool fast_ok = false;
  FastPlan plan{};       // simple finish (no colliders / pressure / mask)
  FastPlan plan_gen{};   // general finish
  WavePlan wave{};       // wavefront temporal blocking (nx <= 128 batches, no pressure plug)
  bool small_ok = false;  // small-cloth kernel (<= 1024 nodes per cloth, no pressure plug)
  bool plane_only = false;  // every collider cloth: one frictionless plane, no sphere
  bool sphere_only = false;  // every collider cloth: one sphere, no plane
  std::map<int, WavePlan> wave_chunk;  // plans for cloth-chunk launches (pipelined rollout)
  // class groups (a batch mixing collider-free cloths with collider cloths): the collider-free
  // ones through the wavefront kernel without the collider finish, the others through the
  // streaming kernel (its general finish runs faster at its occupancy)
  bool grouped = false;
  int n_simple = 0, n_general = 0;
  DevBuf<int32_t> ids_simple, ids_general;
  WavePlan wave_simple{};
  FastPlan plan_general{};
  bool wave_on = true;   // sc_ctx_set_persistent / SC_WAVE=0: the streaming kernel only
  bool wave_pinned = false;
  std::map<long long, FastPlan> plan_cache;  // row-range launches of strip contexts
  bool any_pressure = false, any_general = false;
  bool pbs_ok = false;  // every cloth has a grid spacing (rest lengths) for the PBS step
  CUtensorMap tmap[2][2];  // [buffer][xy pairs | z planes]
  bool tmap_ok = false;
  std::atomic<int64_t> launches{0};
  bool health_on = false;  // non-finite tracking in device-resident stepping
  // fused halo exchange with strip neighbours (sc_ctx_set_peer / sc_ctx_peer_step): side 0 =
  // the neighbour owning the rows below, 1 = above
  struct Peer {
    void* buf[2] = {nullptr, nullptr};  // its state buffers (IPC-mapped or same-process)
    int64_t S = 0;
    int32_t g0 = 0;
    int32_t cur_delta = 0;              // its buffer parity relative to ours
    unsigned* flag = nullptr;           // its completion-flag slot this ctx signals
    bool ipc = false;
    void* opened[3] = {nullptr, nullptr, nullptr};
  } peer[2];
  DevBuf<unsigned> peer_flags;  // [2] written by the neighbours: steps they have completed
  unsigned peer_count = 0;      // fused steps this ctx has completed since linking
  bool peer_launch = false;     // base_args adds the peer stores
  // frame streaming (sc_rollout_frames / sc_simulate_frames): two pinned host slots + events
  void* pin_stage = nullptr;
  size_t pin_stage_bytes = 0;
  cudaEvent_t frame_ev[2] = {nullptr, nullptr};
  // pipelined host->host FAST rollout (sc_rollout): per-chunk streams and events
  static constexpr int kPipe = 16;
  cudaStream_t pipe_stream[kPipe] = {};
  cudaEvent_t pipe_ev[kPipe + 1] = {};
  std::vector<cudaEvent_t> band_ev;  // band uploads / downloads of rollout_band_pipelined

  size_t elem() const { return prec == SC_F32 ? 4 : 8; }
  int64_t nodes_global() const { return static_cast<int64_t>(nx) * ny; }
  int64_t nodes_local() const { return static_cast<int64_t>(nx) * rows_local; }
};

namespace {

void free_scene(sc_ctx* c) {
  for (void*& p : c->state) {
    if (p) cudaFree(p);
    p = nullptr;
  }
  for (void** p : {&c->cloths, &c->spheres, &c->planes, &c->anchors}) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  c->pin_bits.release();
  c->pin_rank.release();
  c->health.release();
  c->mask.release();
  c->aos.release();
  c->has_scene = false;
  c->tmap_ok = false;
  c->plan_cache.clear();
  c->wave_chunk.clear();
  c->ids_simple.release();
  c->ids_general.release();
  c->grouped = false;
  // a rebound scene must not keep pointers into the neighbours' (old) buffers
  for (auto& q : c->peer) {
    for (void*& o : q.opened)
      if (o) {
        cudaIpcCloseMemHandle(o);
        o = nullptr;
      }
    q = sc_ctx::Peer{};
  }
  c->peer_count = 0;
  c->peer_launch = false;
}

bool finite3(const double* v) {
  return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]);
}

// Scene::validate (scene.cpp:23-61) + MaterialParams::validate (grid.cpp:73-81) for the fields
// the NN step consumes; messages carry the reference's field names.
void validate_scene(const sc_scene_desc* s) {
  if (!s) throw_config("scene: null descriptor");
  if (s->nx < 2) throw_config("grid.nx: must be >= 2");
  if (s->ny < 2) throw_config("grid.ny: must be >= 2");
  if (static_cast<int64_t>(s->nx) * s->ny > INT32_MAX)
    throw_config("grid: node count exceeds the 32-bit node index of the reference");
  if (s->batch < 1) throw_config("batch: must be >= 1");
  if (!s->cloths) throw_config("batch: null cloth array");
  const int64_t n = static_cast<int64_t>(s->nx) * s->ny;
  for (int b = 0; b < s->batch; ++b) {
    const sc_cloth_desc& c = s->cloths[b];
    const std::string at = s->batch > 1 ? "cloths[" + std::to_string(b) + "]." : "";
    if (!(c.mass > 0.0) || !std::isfinite(c.mass))
      throw_config(at + "material.mass: must be a finite value > 0");
    if (!std::isfinite(c.drag) || c.drag < 0.0)
      throw_config(at + "material.drag: must be a finite value >= 0");
    if (!std::isfinite(c.pressure)) throw_config(at + "material.pressure: must be finite");
    if (!std::isfinite(c.stiffness) || c.stiffness < 0.0)
      throw_config(at + "material.stiffness: must be a finite value >= 0");
    if (!std::isfinite(c.damping) || c.damping < 0.0)
      throw_config(at + "material.damping: must be a finite value >= 0");
    if (!std::isfinite(c.spacing) || c.spacing < 0.0)
      throw_config(at + "grid.spacing: must be a finite value > 0");
    if (!finite3(c.gravity)) throw_config(at + "material.gravity: components must be finite");
    if (!(c.dt > 0.0) || !std::isfinite(c.dt))
      throw_config(at + "time.dt: must be a finite value > 0");
    if (c.n_pins < 0) throw_config(at + "pins: negative count");
    if (c.n_pins > 0 && (!c.pin_nodes || !c.pin_anchors))
      throw_config(at + "pins: anchor list does not match the node list");
    for (int k = 0; k < c.n_pins; ++k) {
      const int i = c.pin_nodes[k];
      if (i < 0 || i >= n)
        throw_config(at + "pins.nodes[" + std::to_string(k) + "]: index out of range");
      if (k > 0 && c.pin_nodes[k - 1] >= i)
        throw_config(at + "pins.nodes: must be strictly increasing (sorted, unique)");
      if (!finite3(c.pin_anchors + 3 * k))
        throw_config(at + "pins.anchors[" + std::to_string(k) + "]: non-finite component");
    }
    if (!finite3(c.pin_velocity))
      throw_config(at + "pins.motion.velocity: components must be finite");
    if (c.n_spheres < 0 || (c.n_spheres > 0 && !c.spheres))
      throw_config(at + "colliders: bad sphere list");
    for (int k = 0; k < c.n_spheres; ++k) {
      const std::string path = at + "colliders[" + std::to_string(k) + "]";
      const sc_sphere& sp = c.spheres[k];
      if (!finite3(sp.center)) throw_config(path + ".center: components must be finite");
      if (!(sp.radius > 0.0) || !std::isfinite(sp.radius))
        throw_config(path + ".radius: must be a finite value > 0");
      if (!(sp.friction >= 0.0 && sp.friction <= 1.0))
        throw_config(path + ".friction: must be in [0, 1]");
    }
    if (c.n_planes < 0 || (c.n_planes > 0 && !c.planes))
      throw_config(at + "planes: bad plane list");
    for (int k = 0; k < c.n_planes; ++k) {
      const std::string path = at + "planes[" + std::to_string(k) + "]";
      if (!std::isfinite(c.planes[k].height)) throw_config(path + ".height: must be finite");
      if (!(c.planes[k].friction >= 0.0 && c.planes[k].friction <= 1.0))
        throw_config(path + ".friction: must be in [0, 1]");
    }
  }
}

template <typename T>
T eps16() {
  return std::numeric_limits<T>::epsilon() * T(16);
}

// SceneKernel<T> cast + the derived per-cloth products, each one IEEE op in T on the host
// (x86-64 SSE, no contraction) exactly as the reference evaluates them (kernels.hpp:182-193,
// 217, 221, 239).
template <typename T>
void upload_scene(sc_ctx* c, const sc_scene_desc* s) {
  const int B = s->batch;
  std::vector<ClothConst<T>> cl(static_cast<size_t>(B));
  std::vector<SphereConst<T>> sph;
  std::vector<PlaneConst<T>> pln;
  std::vector<T> anchors;
  const int64_t n = c->nodes_global();
  const int64_t words = (n + 31) / 32;
  int64_t total_words = 0;
  for (int b = 0; b < B; ++b)
    if (s->cloths[b].n_pins > 0) total_words += words;
  std::vector<uint32_t> bits(static_cast<size_t>(std::max<int64_t>(total_words, 1)), 0u);
  std::vector<int32_t> rank(bits.size(), 0);
  int64_t word0 = 0;
  for (int b = 0; b < B; ++b) {
    const sc_cloth_desc& d = s->cloths[b];
    ClothConst<T>& k = cl[static_cast<size_t>(b)];
    k.dt = static_cast<T>(d.dt);
    const T mass = static_cast<T>(d.mass);
    k.scale = k.dt / mass;
    k.drag_c = static_cast<T>(d.drag) * k.scale;
    k.pressure = static_cast<T>(d.pressure);
    for (int q = 0; q < 3; ++q) {
      k.dv[q] = static_cast<T>(d.gravity[q]) * k.dt;
      k.pin_u[q] = static_cast<T>(d.pin_velocity[q]);
    }
    k.plug_pressure = (d.plug_pressure && k.pressure != T(0)) ? 1 : 0;
    k.plug_gravity = d.plug_gravity ? 1 : 0;
    k.plug_drag = d.plug_drag ? 1 : 0;
    for (int q = 0; q < 3; ++q) k.fin[q] = k.plug_gravity ? k.dv[q] : T(0);
    k.fin[3] = k.plug_drag ? k.drag_c : T(0);
    k.n_spheres = d.n_spheres;
    k.sphere0 = static_cast<int32_t>(sph.size());
    for (int q = 0; q < d.n_spheres; ++q) {
      SphereConst<T> sc{};
      for (int e = 0; e < 3; ++e) sc.c[e] = static_cast<T>(d.spheres[q].center[e]);
      sc.R = static_cast<T>(d.spheres[q].radius);
      sc.Rband = sc.R * (T(1) + eps16<T>());
      sc.omf = T(1) - static_cast<T>(d.spheres[q].friction);
      sph.push_back(sc);
    }
    k.n_planes = d.n_planes;
    k.plane0 = static_cast<int32_t>(pln.size());
    for (int q = 0; q < d.n_planes; ++q) {
      PlaneConst<T> pc{};
      pc.h = static_cast<T>(d.planes[q].height);
      const T ah = pc.h < T(0) ? -pc.h : pc.h;
      pc.band = (ah > T(1) ? ah : T(1)) * eps16<T>();
      pc.omf = T(1) - static_cast<T>(d.planes[q].friction);
      pln.push_back(pc);
    }
    // PBS material (SceneKernel<T> casts, kernels.hpp:62-70; rest lengths grid.cpp:93-95)
    k.stiffness = static_cast<T>(d.stiffness);
    k.damping = static_cast<T>(d.damping);
    k.mass = mass;
    k.drag = static_cast<T>(d.drag);
    for (int q = 0; q < 3; ++q) k.grav[q] = static_cast<T>(d.gravity[q]);
    static const double mult[kChannels] = {1.0, 1.0, 1.0, 1.0,
                                           1.41421356237309504880, 1.41421356237309504880,
                                           1.41421356237309504880, 1.41421356237309504880,
                                           2.0, 2.0, 2.0, 2.0};
    for (int c = 0; c < kChannels; ++c) k.rest[c] = static_cast<T>(d.spacing * mult[c]);
    k.n_pins = d.n_pins;
    k.pin_row_lo = d.n_pins > 0 ? d.pin_nodes[0] / s->nx : 0;  // pins are sorted
    k.pin_row_hi = d.n_pins > 0 ? d.pin_nodes[d.n_pins - 1] / s->nx : -1;
    k.pin_word0 = 0;
    k.anchor0 = static_cast<int64_t>(anchors.size() / 3);
    if (d.n_pins > 0) {
      k.pin_word0 = word0;
      for (int p = 0; p < d.n_pins; ++p) {
        const int64_t node = d.pin_nodes[p];
        bits[static_cast<size_t>(word0 + (node >> 5))] |= 1u << (node & 31);
        for (int e = 0; e < 3; ++e) anchors.push_back(static_cast<T>(d.pin_anchors[3 * p + e]));
      }
      int32_t acc = 0;
      for (int64_t w = 0; w < words; ++w) {
        rank[static_cast<size_t>(word0 + w)] = acc;
        acc += __builtin_popcount(bits[static_cast<size_t>(word0 + w)]);
      }
      word0 += words;
    }
  }
  auto up = [&](void** dst, const void* src, size_t bytes) {
    ck(cudaMalloc(dst, std::max<size_t>(bytes, 16)), "cudaMalloc(scene)");
    if (bytes) ck(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice), "cudaMemcpy(scene)");
  };
  up(&c->cloths, cl.data(), sizeof(ClothConst<T>) * cl.size());
  up(&c->spheres, sph.data(), sizeof(SphereConst<T>) * sph.size());
  up(&c->planes, pln.data(), sizeof(PlaneConst<T>) * pln.size());
  up(&c->anchors, anchors.data(), sizeof(T) * anchors.size());
  c->pin_bits.ensure(bits.size());
  ck(cudaMemcpy(c->pin_bits.p, bits.data(), sizeof(uint32_t) * bits.size(),
                cudaMemcpyHostToDevice),
     "cudaMemcpy(pins)");
  c->pin_rank.ensure(rank.size());
  ck(cudaMemcpy(c->pin_rank.p, rank.data(), sizeof(int32_t) * rank.size(),
                cudaMemcpyHostToDevice),
     "cudaMemcpy(pins)");
}

template <typename T>
NetConst<T> make_net(const sc_params* p) {
  NetConst<T> k{};
  for (int c = 0; c < kChannels; ++c) {
    k.gain[c] = static_cast<T>(p->kernel_gain[c]);
    k.wl[c] = static_cast<T>(p->linear_w[c]);
    k.wn[c] = static_cast<T>(p->nonlinear_w[c]);
    k.wd[c] = static_cast<T>(p->deriv_w[c]);
  }
  for (int d = 0; d < 3; ++d) k.b[d] = static_cast<T>(p->linear_b[d]);
  k.wv = static_cast<T>(p->self_velocity_w);
  k.alpha = static_cast<T>(p->isru_alpha);
  return k;
}

void build_tmaps(sc_ctx* c) {
  c->tmap_ok = false;
  if (c->prec != SC_F32) return;
  PFN_encodeTiled enc = get_encoder();
  if (!enc) throw Fail{SC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver"};
  const cuuint64_t S = static_cast<cuuint64_t>(c->plane_stride);
  for (int i = 0; i < 2; ++i) {
    // xy pairs as 8-byte elements: dims (pitch, rows, {x,v}, batch)
    {
      const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c->pitch),
                                  static_cast<cuuint64_t>(c->rows_local), 2,
                                  static_cast<cuuint64_t>(c->batch)};
      const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c->pitch) * 8, S * 8, S * 24};
      const cuuint32_t box[4] = {136, 1, 2, 1};  // see fast_kernels.cu (BOXW)
      const cuuint32_t estr[4] = {1, 1, 1, 1};
      const CUresult r = enc(&c->tmap[i][0], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, c->state[i],
                             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        throw Fail{SC_ERR_CUDA, "cuTensorMapEncodeTiled(xy) failed (" + std::to_string(r) + ")"};
    }
    // z planes: dims (pitch, rows, {x,v}, batch), base at element 4S
    {
      const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c->pitch),
                                  static_cast<cuuint64_t>(c->rows_local), 2,
                                  static_cast<cuuint64_t>(c->batch)};
      const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c->pitch) * 4, S * 4, S * 24};
      const cuuint32_t box[4] = {136, 1, 2, 1};
      const cuuint32_t estr[4] = {1, 1, 1, 1};
      const CUresult r = enc(&c->tmap[i][1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                             static_cast<float*>(c->state[i]) + 4 * S, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        throw Fail{SC_ERR_CUDA, "cuTensorMapEncodeTiled(z) failed (" + std::to_string(r) + ")"};
    }
  }
  c->tmap_ok = true;
}

void require_ready(sc_ctx* c, bool need_params = true) {
  if (!c) throw_state("null context");
  if (!c->has_scene) throw_state("no scene bound (call sc_ctx_set_scene first)");
  if (need_params && !c->has_params) throw_state("no parameters bound (call sc_ctx_set_params)");
}

template <typename T>
StepArgs<T> base_args(sc_ctx* c) {
  StepArgs<T> a{};
  a.in = static_cast<const T*>(c->state[c->cur]);
  a.out = static_cast<T*>(c->state[1 - c->cur]);
  a.plane_stride = c->plane_stride;
  a.pitch = c->pitch;
  a.nx = c->nx;
  a.ny = c->ny;
  a.g0 = c->g0;
  a.u0 = c->u0;
  a.u1 = c->u1;
  a.batch = c->batch;
  a.zs = c->zs ? 1 : 0;
  a.cloths = static_cast<const ClothConst<T>*>(c->cloths);
  a.spheres = static_cast<const SphereConst<T>*>(c->spheres);
  a.planes = static_cast<const PlaneConst<T>*>(c->planes);
  a.pin_bits = c->pin_bits.p;
  a.pin_rank = c->pin_rank.p;
  a.pin_anchors = static_cast<const T*>(c->anchors);
  if (c->peer_launch)
    for (int sd = 0; sd < 2; ++sd) {
      const sc_ctx::Peer& q = c->peer[sd];
      if (!q.buf[0]) continue;
      a.peer_out[sd] = static_cast<T*>(q.buf[1 - (c->cur ^ q.cur_delta)]);
      a.peer_S[sd] = q.S;
      a.peer_g0[sd] = q.g0;
    }
  return a;
}

template <typename T>
NetConst<T>& net_of(sc_ctx* c);
template <>
NetConst<float>& net_of<float>(sc_ctx* c) {
  return c->net32;
}
template <>
NetConst<double>& net_of<double>(sc_ctx* c) {
  return c->net64;
}

// Plan of a row-range FAST launch (strip steps, bands): cached per (rows, finish kind); the
// single-kind collider instantiation carries over from the context plan.
FastPlan range_plan(sc_ctx* c, int rows, bool gen) {
  const long long key = (static_cast<long long>(rows) << 1) | (gen ? 1 : 0);
  auto it = c->plan_cache.find(key);
  if (it == c->plan_cache.end()) {
    FastPlan p = plan_fast(c->nx, rows, c->batch, c->device, c->any_pressure, gen);
    p.only = c->plan.only;
    it = c->plan_cache.emplace(key, p).first;
  }
  return it->second;
}

// One launch of the fused step (or one operator) on the ctx stream.
template <typename T>
void launch_one(sc_ctx* c, int kind, sc_mode mode, int k, bool t_override, double t_next,
                uint8_t* mask, T* impulse, Health* health, int u0, int u1, cudaStream_t stream) {
  StepArgs<T> a = base_args<T>(c);
  a.u0 = u0;
  a.u1 = u1;
  a.k = k;
  a.use_t_override = t_override ? 1 : 0;
  a.t_override = static_cast<T>(t_next);
  a.constrained = mask;
  a.impulse = impulse;
  a.health = health;
  a.net = net_of<T>(c);
  cudaError_t e;
  if constexpr (std::is_same<T, float>::value) {
    if (kind == KIND_STEP && mode == SC_MODE_FAST && c->fast_ok && c->tmap_ok) {
      FastPlan plan = mask ? c->plan_gen : c->plan;
      if (u0 != c->u0 || u1 != c->u1) plan = range_plan(c, u1 - u0, c->any_general || mask);
      e = launch_fast(a, c->fast, c->tmap[c->cur], plan, stream);
    } else {
      e = launch_parity<float>(a, kind, stream);
    }
  } else {
    e = launch_parity<double>(a, kind, stream);
  }
  ck(e, "kernel launch");
  c->launches.fetch_add(1);
}

void reset_health(sc_ctx* c) {
  c->health.ensure(static_cast<size_t>(c->batch));
  std::vector<Health> h(static_cast<size_t>(c->batch));
  for (auto& x : h) {
    x.impulse_key = ~0ull;
    x.state_frame = INT_MAX;
    x.pad = 0;
  }
  ck(cudaMemcpyAsync(c->health.p, h.data(), sizeof(Health) * h.size(), cudaMemcpyHostToDevice,
                     c->stream),
     "health reset");
  ck(cudaStreamSynchronize(c->stream), "health reset");
}

void upload_state(sc_ctx* c, const void* x, const void* v) {
  const size_t bytes = static_cast<size_t>(c->batch) * c->nodes_local() * 3 * c->elem();
  c->aos.ensure(3 * bytes);
  unsigned char* dx = c->aos.p;
  unsigned char* dv = c->aos.p + bytes;
  ck(cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, c->stream), "H2D x");
  ck(cudaMemcpyAsync(dv, v, bytes, cudaMemcpyHostToDevice, c->stream), "H2D v");
  cudaError_t e;
  if (c->prec == SC_F32)
    e = launch_aos_to_planar<float>(reinterpret_cast<float*>(dx), reinterpret_cast<float*>(dv),
                                    static_cast<float*>(c->state[c->cur]), c->batch, c->nx,
                                    c->rows_local, c->plane_stride, c->pitch, c->zs, c->stream);
  else
    e = launch_aos_to_planar<double>(reinterpret_cast<double*>(dx),
                                     reinterpret_cast<double*>(dv),
                                     static_cast<double*>(c->state[c->cur]), c->batch, c->nx,
                                     c->rows_local, c->plane_stride, c->pitch, c->zs, c->stream);
  ck(e, "aos_to_planar");
  c->launches.fetch_add(1);
}

void download_state(sc_ctx* c, int which, void* x, void* v, bool sync = true) {
  const size_t bytes = static_cast<size_t>(c->batch) * c->nodes_local() * 3 * c->elem();
  c->aos.ensure(3 * bytes);
  unsigned char* dx = c->aos.p;
  unsigned char* dv = c->aos.p + bytes;
  cudaError_t e;
  if (c->prec == SC_F32)
    e = launch_planar_to_aos<float>(static_cast<const float*>(c->state[which]),
                                    reinterpret_cast<float*>(dx), reinterpret_cast<float*>(dv),
                                    c->batch, c->nx, c->rows_local, c->plane_stride, c->pitch,
                                    c->zs, c->stream);
  else
    e = launch_planar_to_aos<double>(static_cast<const double*>(c->state[which]),
                                     reinterpret_cast<double*>(dx),
                                     reinterpret_cast<double*>(dv), c->batch, c->nx,
                                     c->rows_local, c->plane_stride, c->pitch, c->zs, c->stream);
  ck(e, "planar_to_aos");
  c->launches.fetch_add(1);
  if (x) ck(cudaMemcpyAsync(x, dx, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H x");
  if (v) ck(cudaMemcpyAsync(v, dv, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H v");
  if (sync) ck(cudaStreamSynchronize(c->stream), "D2H sync");
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Frame output of a rollout (§8(f3)): frame f's AoS x/v are converted into device slot f&1 and
// copied D2H behind the stepping kernels of frame f+1 on the same stream. Pinned destination
// arrays are written directly; pageable ones go through two pinned slots, the host copying
// frame f-1 out while the GPU advances frame f, so the device never waits on the host copy.
template <typename StepFn>
void frames_impl(sc_ctx* c, const void* x0, const void* v0, int steps, int stride, void* fx,
                 void* fv, StepFn&& step) {
  const size_t bytes = static_cast<size_t>(c->batch) * c->nodes_local() * 3 * c->elem();
  upload_state(c, x0, v0);
  std::memcpy(fx, x0, bytes);
  std::memcpy(fv, v0, bytes);
  const bool direct = is_pinned(fx) && is_pinned(fv);
  c->aos.ensure(4 * bytes);
  if (!direct && c->pin_stage_bytes < 4 * bytes) {
    if (c->pin_stage) cudaFreeHost(c->pin_stage);
    c->pin_stage = nullptr;
    c->pin_stage_bytes = 0;
    ck(cudaHostAlloc(&c->pin_stage, 4 * bytes, cudaHostAllocPortable), "cudaHostAlloc frames");
    c->pin_stage_bytes = 4 * bytes;
  }
  for (cudaEvent_t& e : c->frame_ev)
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  auto* ux = static_cast<unsigned char*>(fx);
  auto* uv = static_cast<unsigned char*>(fv);
  auto* stage = static_cast<unsigned char*>(c->pin_stage);
  auto drain = [&](int f) {  // host side of frame f (staged path)
    const int slot = f & 1;
    ck(cudaEventSynchronize(c->frame_ev[slot]), "frame event");
    std::memcpy(ux + bytes * f, stage + 2 * bytes * slot, bytes);
    std::memcpy(uv + bytes * f, stage + 2 * bytes * slot + bytes, bytes);
  };
  int f = 1;
  for (int k = 0; k < steps; k += stride) {
    const int n = std::min(stride, steps - k);
    step(n, k);
    if (n != stride) break;
    const int slot = f & 1;
    unsigned char* dx = c->aos.p + 2 * bytes * slot;
    unsigned char* dv = dx + bytes;
    cudaError_t e;
    if (c->prec == SC_F32)
      e = launch_planar_to_aos<float>(static_cast<const float*>(c->state[c->cur]),
                                      reinterpret_cast<float*>(dx), reinterpret_cast<float*>(dv),
                                      c->batch, c->nx, c->rows_local, c->plane_stride, c->pitch,
                                      c->zs, c->stream);
    else
      e = launch_planar_to_aos<double>(static_cast<const double*>(c->state[c->cur]),
                                       reinterpret_cast<double*>(dx),
                                       reinterpret_cast<double*>(dv), c->batch, c->nx,
                                       c->rows_local, c->plane_stride, c->pitch, c->zs, c->stream);
    ck(e, "planar_to_aos");
    c->launches.fetch_add(1);
    unsigned char* hx = direct ? ux + bytes * f : stage + 2 * bytes * slot;
    unsigned char* hv = direct ? uv + bytes * f : stage + 2 * bytes * slot + bytes;
    ck(cudaMemcpyAsync(hx, dx, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H frame x");
    ck(cudaMemcpyAsync(hv, dv, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H frame v");
    ck(cudaEventRecord(c->frame_ev[slot], c->stream), "frame event");
    if (!direct && f > 1) drain(f - 1);
    ++f;
  }
  if (!direct && f > 1) drain(f - 1);
  ck(cudaStreamSynchronize(c->stream), "sync");
}

// FAST stepping in cloth chunks on concurrent streams. Each chunk of cloths runs its own chain
// of step launches (a slice of the whole-batch grid with the same plan: identical arithmetic,
// bit-identical results), so one chunk's launch ramp and tail overlap the others' work instead
// of leaving SMs idle at every step boundary (config 2: 46.0 -> ~42.6 us per step). `pre(i, q)`
// and `post(i, q, buffer)` enqueue per-chunk work on chunk i's stream before its first and after
// its last step (the pipelined rollout's transfers). Taken for FAST, f32, whole-cloth contexts
// with >= 8 cloths and no mask output.
// The wavefront kernel (wave_kernels.cu) applies: FAST f32 whole-cloth context, nx <= 128, no
// pressure plug, not linked to strip peers, persistent stepping on (sc_ctx_set_persistent).
// The small-cloth kernel (small_kernels.cu) applies: FAST f32 whole-cloth context of cloths of at
// most 1024 nodes, no pressure plug, not linked to strip peers, persistent stepping on. Taken
// before the wavefront kernel (config 1: 6.1 -> ~1.5 us per timestep).
bool small_usable(const sc_ctx* c) {
  return c->prec == SC_F32 && c->fast_ok && c->small_ok && c->wave_on && !c->peer_launch &&
         c->strip_row0 < 0;
}

// some cloth of the scene has a collider, and every such cloth has exactly one sphere and no plane
bool sphere_only_scene(const sc_scene_desc* s) {
  bool any = false;
  for (int b = 0; b < s->batch; ++b) {
    const sc_cloth_desc& d = s->cloths[b];
    if (d.n_planes > 0 || d.n_spheres > 1) return false;
    any = any || d.n_spheres == 1;
  }
  return any;
}

// some cloth of the scene has a collider, and every such cloth has exactly one frictionless plane
// and no sphere
bool plane_only_scene(const sc_scene_desc* s) {
  bool any = false;
  for (int b = 0; b < s->batch; ++b) {
    const sc_cloth_desc& d = s->cloths[b];
    if (d.n_spheres > 0 || d.n_planes > 1 ||
        (d.n_planes == 1 && static_cast<float>(d.planes[0].friction) != 0.0f))
      return false;
    any = any || d.n_planes == 1;
  }
  return any;
}

bool wave_usable(const sc_ctx* c) {
  return c->prec == SC_F32 && c->fast_ok && c->tmap_ok && c->wave.ok && c->wave_on &&
         !c->peer_launch && c->strip_row0 < 0;
}

int fast_chunks(const sc_ctx* c, int steps) {
  int k = c->batch >= 16 ? 4 : 2;
  if (const char* env = std::getenv("SC_CHUNKS")) k = std::min(sc_ctx::kPipe, std::atoi(env));
  k = std::min(k, c->batch / 2);
  if (k < 2 || c->prec != SC_F32 || !c->fast_ok || !c->tmap_ok || c->peer_launch)
    return 0;
  if (c->u0 != 0 || c->u1 != c->ny || c->g0 != 0 || c->rows_local != c->ny) return 0;
  if (c->batch < 8 || steps < 2) return 0;
  return k;
}

// The wavefront kernel wins on large narrow-cloth batches stepped for long; below ~8 cloths per
// SM its whole cloths per CTA quantise the load (config-5 shares: 512 cloths 82.8 vs 75.1 us per
// step for the chunked streaming path, 1024: 148.1 vs 145.1; 2048: 290.5 vs 305.8), so smaller
// batches that can be chunked take the streaming kernel. So do short advances: at full clocks the
// chunked streaming kernel steps config 5 faster (538 vs 561-594 us per timestep), but it moves
// 48 B per node-update through HBM and after ~50 ms of back-to-back steps the board hits its
// power cap (sw_power_cap, SM clock 1965 -> ~1600 MHz: 584 us at 150 steps, 617 at 300), while
// the wavefront kernel (0.06x the DRAM traffic, ~100 W less) holds 1965 MHz (561 us at 300).
// Measured crossover between 80 and 150 timesteps per call (tools/k_probe.py).
// SC_WAVE_MIN_CLOTHS / SC_WAVE_MIN_STEPS override the thresholds.
bool wave_preferred(const sc_ctx* c, int steps) {
  if (!wave_usable(c)) return false;
  if (fast_chunks(c, steps) == 0) return true;  // no chunked alternative
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int min_cloths = 8 * sms, min_steps = 128;
  if (const char* env = std::getenv("SC_WAVE_MIN_CLOTHS")) min_cloths = std::atoi(env);
  if (const char* env = std::getenv("SC_WAVE_MIN_STEPS")) min_steps = std::atoi(env);
  return c->batch >= min_cloths && steps >= min_steps;
}

template <typename Pre, typename Post>
void chunked_fast_steps(sc_ctx* c, int K, int steps, int k0, Pre pre, Post post) {
  for (int i = 0; i < K; ++i)
    if (!c->pipe_stream[i])
      ck(cudaStreamCreateWithFlags(&c->pipe_stream[i], cudaStreamNonBlocking), "stream");
  for (cudaEvent_t& e : c->pipe_ev)
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  const FastPlan& full = c->plan;  // no mask: the launch-wide plan of this context
  int b0[sc_ctx::kPipe + 1];
  for (int i = 0; i <= K; ++i) b0[i] = static_cast<int>((static_cast<int64_t>(i) * c->batch) / K);
  ck(cudaEventRecord(c->pipe_ev[K], c->stream), "event");  // earlier work on the ctx stream
  for (int i = 0; i < K; ++i) {  // in chunk order (e.g. the uploads: one H2D copy engine)
    ck(cudaStreamWaitEvent(c->pipe_stream[i], c->pipe_ev[K], 0), "wait");
    pre(i, b0[i], b0[i + 1], c->pipe_stream[i]);
  }
  float* st[2] = {static_cast<float*>(c->state[c->cur]), static_cast<float*>(c->state[1 - c->cur])};
  StepArgs<float> a = base_args<float>(c);
  a.net = c->net32;
  a.health = c->health_on ? c->health.p : nullptr;
  for (int s = 0; s < steps; ++s) {  // step launches interleaved across the chunk streams
    a.in = st[s & 1];
    a.out = st[(s & 1) ^ 1];
    a.k = k0 + s;
    for (int i = 0; i < K; ++i) {
      FastPlan p = full;
      p.wide = full.chunk_wide;
      a.b_off = b0[i];
      a.batch = b0[i + 1] - b0[i];
      p.n_segs = p.chunk_segs;
      p.seg_rows = (c->u1 - c->u0 + p.n_segs - 1) / p.n_segs;
      p.units = static_cast<int64_t>(a.batch) * p.n_strips * p.n_segs;
      ck(launch_fast(a, c->fast, c->tmap[c->cur ^ (s & 1)], p, c->pipe_stream[i]),
         "kernel launch");
    }
  }
  for (int i = 0; i < K; ++i) {
    post(i, b0[i], b0[i + 1], c->pipe_stream[i], st[steps & 1]);
    ck(cudaEventRecord(c->pipe_ev[i], c->pipe_stream[i]), "event");
    ck(cudaStreamWaitEvent(c->stream, c->pipe_ev[i], 0), "wait");
  }
  c->launches.fetch_add(static_cast<int64_t>(K) * steps);
  if (steps & 1) c->cur = 1 - c->cur;
}

// n FAST timesteps of a class-grouped context's cloths simple ids [s0, s0 + ns) and general ids
// [g0, g0 + ng), from buffer cur into buffer (cur + n) % 2: the collider-free cloths in one
// wavefront launch (grid wplan.ctas: part of the SMs) on `main`, the collider cloths in n
// ping-pong streaming launches on a side stream at the same time (they land on the SMs the
// wavefront grid leaves free, and on all of them once it is done); `main` waits for both.
void grouped_steps(sc_ctx* c, int n, int k0, int s0, int ns, int g0, int ng,
                   const WavePlan& wplan, const FastPlan& gplan, cudaStream_t main) {
  const int out = (c->cur + n) & 1;
  if (!c->pipe_stream[2])
    ck(cudaStreamCreateWithFlags(&c->pipe_stream[2], cudaStreamNonBlocking), "stream");
  for (cudaEvent_t& e : c->pipe_ev)
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  cudaStream_t side = c->pipe_stream[2];
  ck(cudaEventRecord(c->pipe_ev[14], main), "event");
  ck(cudaStreamWaitEvent(side, c->pipe_ev[14], 0), "wait");
  StepArgs<float> a = base_args<float>(c);
  a.net = c->net32;
  a.health = c->health_on ? c->health.p : nullptr;
  if (ns > 0) {
    a.out = static_cast<float*>(c->state[out]);
    a.k = k0;
    a.ids = c->ids_simple.p + s0;
    a.batch = ns;
    ck(launch_wave(a, c->fast, c->tmap[c->cur], c->tmap[out], wplan, n, main), "kernel launch");
  }
  a.ids = c->ids_general.p + g0;
  a.batch = ng;
  for (int s2 = 0; ng > 0 && s2 < n; ++s2) {
    const int in = (c->cur + s2) & 1;
    a.in = static_cast<const float*>(c->state[in]);
    a.out = static_cast<float*>(c->state[in ^ 1]);
    a.k = k0 + s2;
    ck(launch_fast(a, c->fast, c->tmap[in], gplan, side), "kernel launch");
  }
  ck(cudaEventRecord(c->pipe_ev[15], side), "event");
  ck(cudaStreamWaitEvent(main, c->pipe_ev[15], 0), "wait");
  c->launches.fetch_add((ns > 0 ? 1 : 0) + (ng > 0 ? n : 0));
}

void advance_impl(sc_ctx* c, int steps, int k0, sc_mode mode, uint8_t* dev_mask_last,
                  int kind = KIND_STEP) {
  if (steps < 0) throw_config("steps: must be >= 0");
  if (mode != SC_MODE_PARITY && mode != SC_MODE_FAST) throw_config("mode: unknown");
  if (mode == SC_MODE_FAST && c->prec != SC_F32)
    throw_config("mode: FAST is an f32 mode (use PARITY with an f64 context)");
  int s = 0;
  if (kind == KIND_STEP && mode == SC_MODE_FAST && small_usable(c)) {
    const int n = steps - (dev_mask_last ? 1 : 0);  // a mask-producing last step runs whole
    if (n >= 2) {
      StepArgs<float> a = base_args<float>(c);
      a.k = k0;
      a.net = c->net32;
      a.health = c->health_on ? c->health.p : nullptr;
      ck(launch_small(a, c->fast, c->any_general, n, c->stream), "kernel launch");
      c->launches.fetch_add(1);
      c->cur = 1 - c->cur;
      k0 += n;
      steps -= n;
    }
  }
  if (s == 0 && kind == KIND_STEP && mode == SC_MODE_FAST && wave_preferred(c, steps)) {
    const int n = steps - (dev_mask_last ? 1 : 0);  // a mask-producing last step runs whole
    if (n >= 2 && c->grouped) {
      const int out = (c->cur + n) & 1;
      grouped_steps(c, n, k0, 0, c->n_simple, 0, c->n_general, c->wave_simple, c->plan_general,
                    c->stream);
      c->cur = out;
      k0 += n;
      steps -= n;
    } else if (n >= 2) {
      StepArgs<float> a = base_args<float>(c);
      a.out = static_cast<float*>(c->state[c->cur]);  // in place
      a.k = k0;
      a.net = c->net32;
      a.health = c->health_on ? c->health.p : nullptr;
      ck(launch_wave(a, c->fast, c->tmap[c->cur], c->tmap[c->cur], c->wave, n, c->stream),
         "kernel launch");
      c->launches.fetch_add(1);
      k0 += n;  // the mask-producing last step (if any) follows below
      steps -= n;
    }
  }
  if (s == 0 && kind == KIND_STEP && mode == SC_MODE_FAST) {
    const int n = steps - (dev_mask_last ? 1 : 0);  // a mask-producing last step runs whole
    const int K = fast_chunks(c, n);
    if (K > 0) {
      chunked_fast_steps(c, K, n, k0, [](int, int, int, cudaStream_t) {},
                         [](int, int, int, cudaStream_t, const float*) {});
      s = n;
    }
  }
  for (; s < steps; ++s) {
    const int k = k0 + s;
    uint8_t* m = (s == steps - 1) ? dev_mask_last : nullptr;
    if (c->prec == SC_F32)
      launch_one<float>(c, kind, mode, k, false, 0.0, m, nullptr,
                        c->health_on ? c->health.p : nullptr, c->u0, c->u1, c->stream);
    else
      launch_one<double>(c, kind, mode, k, false, 0.0, m, nullptr,
                         c->health_on ? c->health.p : nullptr, c->u0, c->u1, c->stream);
    c->cur = 1 - c->cur;
  }
}

// Host -> host FAST rollout with the transfers overlapped: each chunk's H2D and layout conversion
// precede its step chain on its stream, its conversion back and D2H follow it, so the copy
// engines move chunk i while the SMs step the chunks already resident and the last chunks'
// steps hide the first chunks' downloads. Needs page-locked host arrays.
bool pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Host -> host FAST rollout of a wavefront context with the transfers overlapped: the batch goes
// in K cloth chunks; chunk i's H2D runs on a copy stream while the compute stream converts and
// steps the chunks before it, and its D2H on a second copy stream while the chunks after it
// step. Each chunk is one wavefront launch over all SMs (chunks of >= 4 cloths per CTA keep
// its load balance), so the device time is the unchunked one plus one chunk's copies.
// Cloth-chunk boundaries of the pipelined wavefront rollout. The pipeline is compute-bound when
// a cloth's `steps` timesteps take longer on the GPU than its upload (per node: ~9e-12 s per
// node-update at ~1.1e11 node-updates/s against 24 B at ~54 GB/s = 4.4e-10 s each way), i.e. by
// the factor g = 0.02 steps (6 for config 5's 300 steps). The exposed time is then the first
// chunk's upload and the last chunk's download, so the chunks ramp geometrically: one wavefront
// CTA's worth of cloths per SM first, each next chunk at most g x larger (its upload hides behind
// the previous chunk's stepping), the same ramp mirrored at the end (each download hides behind
// the next chunk's stepping), the rest in the middle. Chunk sizes are multiples of the SM count
// where possible (the wavefront grid's load balance). Short rollouts (g < 2) keep K equal chunks.
std::vector<int> pipeline_bounds(int batch, int sms, int steps, int K_equal) {
  std::vector<int> b0{0};
  double g = 0.5 * 0.0207 * steps;  // half the break-even growth: measured best (config 5: 3.1)
  if (const char* env = std::getenv("SC_RAMP_G")) g = std::atof(env);  // tuning knob
  if (g >= 2.0 && batch >= 4 * sms) {
    std::vector<int> ramp;
    int64_t size = sms, used = 0;
    // at most two ramp chunks per side (K <= 5: the event slots below), at least one SM-wave of
    // cloths left for the middle
    while (ramp.size() < 2 && 2 * (used + size) <= batch - sms) {
      ramp.push_back(static_cast<int>(size));
      used += size;
      size = static_cast<int64_t>(size * g) / sms * sms;
      if (size < sms) size = sms;
    }
    const int middle = static_cast<int>(batch - 2 * used);
    std::vector<int> sizes(ramp.begin(), ramp.end());
    sizes.push_back(middle);
    sizes.insert(sizes.end(), ramp.rbegin(), ramp.rend());
    for (int sz : sizes) b0.push_back(b0.back() + sz);
    return b0;
  }
  for (int i = 1; i <= K_equal; ++i)
    b0.push_back(static_cast<int>((static_cast<int64_t>(i) * batch) / K_equal));
  return b0;
}

bool rollout_wave_pipelined(sc_ctx* c, const void* x0, const void* v0, int steps, int k0,
                            void* xo, void* vo) {
  if (const char* env = std::getenv("SC_PIPELINE"))
    if (std::atoi(env) == 0) return false;
  // small-cloth contexts step in one small-kernel launch on the plain path
  if (!wave_preferred(c, steps) || small_usable(c) || steps < 2 || !xo || !vo) return false;
  if (!pinned(x0) || !pinned(v0) || !pinned(xo) || !pinned(vo)) return false;
  int Ke = c->batch >= 16 * c->wave.ctas ? 4 : c->batch >= 8 * c->wave.ctas ? 2 : 1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  std::vector<int> b0;
  if (const char* env = std::getenv("SC_WAVE_CHUNKS")) {  // tuning / tests: K equal chunks
    const int K = std::min(std::max(1, std::atoi(env)), c->batch);
    for (int i = 0; i <= K; ++i) b0.push_back(static_cast<int>((static_cast<int64_t>(i) * c->batch) / K));
  } else {
    b0 = pipeline_bounds(c->batch, sms, steps, std::min(Ke, c->batch));
  }
  const int K = static_cast<int>(b0.size()) - 1;
  if (K < 2 || K > 6) return false;  // event slots: ev_in [0, K), ev_out [8, 8 + K), 14-16 taken
  // class-grouped contexts: each chunk's collider-free / collider cloths are contiguous slices
  // of the two (ascending) id lists
  std::vector<int> s_lo(K + 1, 0), g_lo(K + 1, 0);
  if (c->grouped) {
    std::vector<int32_t> ids(static_cast<size_t>(c->n_simple));
    ck(cudaMemcpy(ids.data(), c->ids_simple.p, sizeof(int32_t) * ids.size(),
                  cudaMemcpyDeviceToHost), "D2H ids");
    for (int i = 0; i <= K; ++i) {
      s_lo[i] = static_cast<int>(std::lower_bound(ids.begin(), ids.end(), b0[i]) - ids.begin());
      g_lo[i] = b0[i] - s_lo[i];
    }
  }
  for (int i = 0; i < K; ++i) {
    const int nb = b0[i + 1] - b0[i];
    if (c->grouped) {
      const int ns = s_lo[i + 1] - s_lo[i], ng = g_lo[i + 1] - g_lo[i];
      const int key = -1 - ns;  // grouped chunk plans: negative keys
      if (c->wave_chunk.find(key) == c->wave_chunk.end())
        c->wave_chunk[key] = plan_wave(c->nx, c->ny, ns, c->device, false, c->wave_simple.ctas);
      if (ns > 0 && !c->wave_chunk[key].ok) return false;
      // the collider cloths' streaming launches get the SMs the chunk's wavefront grid leaves
      const long long gkey = -1 - (static_cast<long long>(ng) << 20) - ns;
      if (c->plan_cache.find(gkey) == c->plan_cache.end())
      {
        c->plan_cache[gkey] = plan_fast(c->nx, c->u1 - c->u0, ng, c->device, false, true,
                                        sms - std::min(ns, c->wave_simple.ctas));
        c->plan_cache[gkey].only = c->plane_only ? 1 : 0;
      }
      continue;
    }
    if (c->wave_chunk.find(nb) == c->wave_chunk.end())
      c->wave_chunk[nb] = plan_wave(c->nx, c->ny, nb, c->device, c->any_general);
    if (!c->wave_chunk[nb].ok) return false;
  }
  const int out_buf = c->grouped ? (c->cur + steps) & 1 : c->cur;
  for (int i = 0; i < 2; ++i)
    if (!c->pipe_stream[i])
      ck(cudaStreamCreateWithFlags(&c->pipe_stream[i], cudaStreamNonBlocking), "stream");
  for (cudaEvent_t& e : c->pipe_ev)
    if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  const size_t cloth_bytes = static_cast<size_t>(c->nodes_local()) * 3 * sizeof(float);
  const size_t bytes = cloth_bytes * c->batch;
  c->aos.ensure(2 * bytes);
  unsigned char* dx = c->aos.p;
  unsigned char* dv = c->aos.p + bytes;
  const int64_t S = c->plane_stride;
  float* st = static_cast<float*>(c->state[c->cur]);
  cudaStream_t in = c->pipe_stream[0], out = c->pipe_stream[1];
  cudaEvent_t* ev_in = c->pipe_ev;          // [K]
  cudaEvent_t* ev_out = c->pipe_ev + 8;     // [K]
  ck(cudaEventRecord(c->pipe_ev[16], c->stream), "event");  // earlier work on the ctx stream
  ck(cudaStreamWaitEvent(in, c->pipe_ev[16], 0), "wait");
  for (int i = 0; i < K; ++i) {
    const size_t off = cloth_bytes * b0[i], n = cloth_bytes * (b0[i + 1] - b0[i]);
    ck(cudaMemcpyAsync(dx + off, static_cast<const unsigned char*>(x0) + off, n,
                       cudaMemcpyHostToDevice, in), "H2D x");
    ck(cudaMemcpyAsync(dv + off, static_cast<const unsigned char*>(v0) + off, n,
                       cudaMemcpyHostToDevice, in), "H2D v");
    ck(cudaEventRecord(ev_in[i], in), "event");
  }
  for (int i = 0; i < K; ++i) {
    const int nb = b0[i + 1] - b0[i];
    const size_t off = cloth_bytes * b0[i];
    ck(cudaStreamWaitEvent(c->stream, ev_in[i], 0), "wait");
    ck(launch_aos_to_planar<float>(reinterpret_cast<float*>(dx + off),
                                   reinterpret_cast<float*>(dv + off), st + b0[i] * 6 * S, nb,
                                   c->nx, c->rows_local, S, c->pitch, c->zs, c->stream),
       "aos_to_planar");
    if (c->grouped) {
      const int ns = s_lo[i + 1] - s_lo[i], ng = g_lo[i + 1] - g_lo[i];
      grouped_steps(c, steps, k0, s_lo[i], ns, g_lo[i], ng, c->wave_chunk[-1 - ns],
                    c->plan_cache[-1 - (static_cast<long long>(ng) << 20) - ns], c->stream);
    } else {
      StepArgs<float> a = base_args<float>(c);
      a.out = st;  // in place
      a.k = k0;
      a.b_off = b0[i];
      a.batch = nb;
      a.net = c->net32;
      a.health = c->health_on ? c->health.p : nullptr;
      ck(launch_wave(a, c->fast, c->tmap[c->cur], c->tmap[c->cur], c->wave_chunk[nb], steps,
                     c->stream),
         "kernel launch");
    }
    float* fin = static_cast<float*>(c->state[out_buf]);
    ck(launch_planar_to_aos<float>(fin + b0[i] * 6 * S, reinterpret_cast<float*>(dx + off),
                                   reinterpret_cast<float*>(dv + off), nb, c->nx, c->rows_local,
                                   S, c->pitch, c->zs, c->stream),
       "planar_to_aos");
    ck(cudaEventRecord(ev_out[i], c->stream), "event");
  }
  for (int i = 0; i < K; ++i) {
    const size_t off = cloth_bytes * b0[i], n = cloth_bytes * (b0[i + 1] - b0[i]);
    ck(cudaStreamWaitEvent(out, ev_out[i], 0), "wait");
    ck(cudaMemcpyAsync(static_cast<unsigned char*>(xo) + off, dx + off, n,
                       cudaMemcpyDeviceToHost, out), "D2H x");
    ck(cudaMemcpyAsync(static_cast<unsigned char*>(vo) + off, dv + off, n,
                       cudaMemcpyDeviceToHost, out), "D2H v");
  }
  ck(cudaEventRecord(c->pipe_ev[16], out), "event");
  ck(cudaStreamWaitEvent(c->stream, c->pipe_ev[16], 0), "wait");
  c->launches.fetch_add(c->grouped ? 2 * K : 3 * K);
  c->cur = out_buf;
  return true;
}

bool rollout_pipelined(sc_ctx* c, const void* x0, const void* v0, int steps, int k0, void* xo,
                       void* vo) {
  if (const char* env = std::getenv("SC_PIPELINE"))
    if (std::atoi(env) == 0) return false;
  if (wave_preferred(c, steps)) return false;  // the wavefront pipeline (rollout_wave_pipelined)
  const int K = fast_chunks(c, steps);
  if (K == 0 || !xo || !vo) return false;
  if (!pinned(x0) || !pinned(v0) || !pinned(xo) || !pinned(vo)) return false;
  const size_t cloth_bytes = static_cast<size_t>(c->nodes_local()) * 3 * sizeof(float);
  const size_t bytes = cloth_bytes * c->batch;
  c->aos.ensure(2 * bytes);
  unsigned char* dx = c->aos.p;
  unsigned char* dv = c->aos.p + bytes;
  const int64_t S = c->plane_stride;
  float* st0 = static_cast<float*>(c->state[c->cur]);
  auto pre = [&](int, int b0, int b1, cudaStream_t q) {
    const size_t off = cloth_bytes * b0, n = cloth_bytes * (b1 - b0);
    ck(cudaMemcpyAsync(dx + off, static_cast<const unsigned char*>(x0) + off, n,
                       cudaMemcpyHostToDevice, q), "H2D x");
    ck(cudaMemcpyAsync(dv + off, static_cast<const unsigned char*>(v0) + off, n,
                       cudaMemcpyHostToDevice, q), "H2D v");
    ck(launch_aos_to_planar<float>(reinterpret_cast<float*>(dx + off),
                                   reinterpret_cast<float*>(dv + off), st0 + b0 * 6 * S, b1 - b0,
                                   c->nx, c->rows_local, S, c->pitch, c->zs, q), "aos_to_planar");
  };
  auto post = [&](int, int b0, int b1, cudaStream_t q, const float* fin) {
    const size_t off = cloth_bytes * b0, n = cloth_bytes * (b1 - b0);
    ck(launch_planar_to_aos<float>(fin + b0 * 6 * S, reinterpret_cast<float*>(dx + off),
                                   reinterpret_cast<float*>(dv + off), b1 - b0, c->nx,
                                   c->rows_local, S, c->pitch, c->zs, q), "planar_to_aos");
    ck(cudaMemcpyAsync(static_cast<unsigned char*>(xo) + off, dx + off, n,
                       cudaMemcpyDeviceToHost, q), "D2H x");
    ck(cudaMemcpyAsync(static_cast<unsigned char*>(vo) + off, dv + off, n,
                       cudaMemcpyDeviceToHost, q), "D2H v");
  };
  chunked_fast_steps(c, K, steps, k0, pre, post);
  c->launches.fetch_add(2 * K);
  return true;
}

// Row bands of the diagonal-wavefront rollout below: band i holds rows [tops[i-1], tops[i]).
// ~12M nodes per band (SC_BAND_ROWS overrides the row count; config 4: 1536 rows, e2e 0.93x
// the device-resident rate against 0.91x at 1024 and 2048 rows), a quarter and a half band first
// and last (the first upload and the last download are the exposed transfers); empty when the
// cloth is too short for a pipeline (< 3 full bands).
std::vector<int> band_tops(int nx, int ny) {
  int H = std::max(64, (12 << 20) / std::max(1, nx)) / 2 * 2;
  if (const char* env = std::getenv("SC_BAND_ROWS")) H = std::max(8, std::atoi(env)) / 2 * 2;
  const int r0 = std::max(4, H / 4 / 2 * 2), r1 = std::max(4, H / 2 / 2 * 2);
  const int middle = ny - 2 * (r0 + r1);
  if (middle < H) return {};
  const int m = std::max(1, (middle + H / 2) / H);
  std::vector<int> sizes{r0, r1};
  for (int j = 0; j < m; ++j)
    sizes.push_back(static_cast<int>((static_cast<int64_t>(j + 1) * middle) / m -
                                     (static_cast<int64_t>(j) * middle) / m));
  sizes.push_back(r1);
  sizes.push_back(r0);
  std::vector<int> tops;
  int t = 0;
  for (int s : sizes) tops.push_back(t += s);
  return tops;
}

// Host -> host FAST rollout of ONE large cloth with the transfers overlapped (config 4: 8192^2,
// 1.6 GB each way over PCIe against ~120 ms of stepping). Cloth chunks cannot hide anything here
// — the first timestep needs every row — but the cell reaches only 2 rows per timestep
// (grid.cpp:24-27; the reference's per-step loop eval.cpp:62-65), so the rollout runs as a
// diagonal wavefront over row bands. Once the rows below tops[i] are resident (band i uploaded),
// timestep level L (1..steps) can be advanced on every row below tops[i] - 2L. Iteration i
// launches, for L = 1..steps in order, the level-L rows that became computable, [T(i-1, L),
// T(i, L)), while the copy engine uploads band i + 1; the rows that reached the last level are
// converted back and downloaded on the other PCIe direction while later iterations step, so
// only the first band's upload and the last rows' download stay exposed. Ping-pong buffers stay
// valid: level L lives in buffer (cur + L) & 1 and, the levels forming a staircase 2 rows apart,
// a level-L row is overwritten by level L + 2 only after every level-(L + 1) row that reads it
// is done. Row-range launches take the same kernels and arithmetic as whole-cloth launches:
// bit-identical results (tests/test_gpu_pipelined_rollout.py).
bool rollout_band_pipelined(sc_ctx* c, const void* x0, const void* v0, int steps, int k0,
                            void* xo, void* vo) {
  if (const char* env = std::getenv("SC_PIPELINE"))
    if (std::atoi(env) == 0) return false;
  if (c->prec != SC_F32 || !c->fast_ok || !c->tmap_ok || c->peer_launch || c->strip_row0 >= 0 ||
      c->batch != 1 || steps < 2 || !xo || !vo)
    return false;
  if (small_usable(c) || wave_preferred(c, steps)) return false;
  if (!pinned(x0) || !pinned(v0) || !pinned(xo) || !pinned(vo)) return false;
  const std::vector<int> tops = band_tops(c->nx, c->ny);
  const int nb = static_cast<int>(tops.size());
  if (nb < 3) return false;
  // iteration i runs on compute stream q[i & 1]; its launch of level L waits for iteration i-1's
  // level L-1 (the rows below its band at the level it reads; the only cross-iteration
  // dependency: iteration i-1 never waits on i, and the staircase keeps their reads and writes on
  // disjoint rows), so two iterations step concurrently and one launch's tail overlaps the other's
  // ramp. Iteration i-1 records an event after its layout conversion (level 0) and after every
  // G-th level; a wait takes the first recorded level >= the one needed.
  int G = 4;
  if (const char* env = std::getenv("SC_BAND_G")) G = std::max(1, std::atoi(env));
  bool chunk_plan = true;
  if (const char* env = std::getenv("SC_BAND_PLAN")) chunk_plan = std::atoi(env) != 0;
  const int nlev = steps / G + 2;  // recorded levels per iteration: 0, G, 2G, ..., last
  for (int i = 0; i < 4; ++i)
    if (!c->pipe_stream[i])
      ck(cudaStreamCreateWithFlags(&c->pipe_stream[i], cudaStreamNonBlocking), "stream");
  if (!c->pipe_ev[16]) ck(cudaEventCreateWithFlags(&c->pipe_ev[16], cudaEventDisableTiming), "event");
  const int n_ev = 2 * nb + 2 * nlev + 2;  // band uploads, downloads, level events of 2 iterations
  while (static_cast<int>(c->band_ev.size()) < n_ev) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    c->band_ev.push_back(e);
  }
  const int nx = c->nx, ny = c->ny;
  const size_t row_bytes = static_cast<size_t>(nx) * 3 * sizeof(float);
  const size_t bytes = row_bytes * ny;
  c->aos.ensure(2 * bytes);
  unsigned char* dx = c->aos.p;
  unsigned char* dv = c->aos.p + bytes;
  const int64_t S = c->plane_stride;
  const int cur0 = c->cur;
  float* st[2] = {static_cast<float*>(c->state[cur0]), static_cast<float*>(c->state[cur0 ^ 1])};
  cudaStream_t in = c->pipe_stream[0], out = c->pipe_stream[1];
  cudaStream_t q[2] = {c->pipe_stream[2], c->pipe_stream[3]};
  auto top = [&](int i, int L) {  // rows below which level L is done after iteration i
    if (i < 0) return 0;
    if (tops[i] >= ny) return ny;
    return std::max(0, tops[i] - 2 * L);
  };
  ck(cudaEventRecord(c->pipe_ev[16], c->stream), "event");  // earlier work on the ctx stream
  for (cudaStream_t w : {in, q[0], q[1]}) ck(cudaStreamWaitEvent(w, c->pipe_ev[16], 0), "wait");
  for (int i = 0; i < nb; ++i) {
    const int r0 = i ? tops[i - 1] : 0;
    const size_t off = row_bytes * r0, n = row_bytes * (tops[i] - r0);
    ck(cudaMemcpyAsync(dx + off, static_cast<const unsigned char*>(x0) + off, n,
                       cudaMemcpyHostToDevice, in), "H2D x");
    ck(cudaMemcpyAsync(dv + off, static_cast<const unsigned char*>(v0) + off, n,
                       cudaMemcpyHostToDevice, in), "H2D v");
    ck(cudaEventRecord(c->band_ev[i], in), "event");
  }
  StepArgs<float> a = base_args<float>(c);
  a.net = c->net32;
  a.health = c->health_on ? c->health.p : nullptr;
  int64_t launches = 0;
  // recorded levels of the previous iteration (ascending) and their events
  std::vector<int> prev_lv, cur_lv;
  std::vector<cudaEvent_t> prev_ev, cur_ev;
  for (int i = 0; i < nb; ++i) {
    const int r0 = i ? tops[i - 1] : 0;
    cudaStream_t w = q[i & 1];
    cudaEvent_t* lev = c->band_ev.data() + 2 * nb + (i & 1) * nlev;
    cur_lv.clear();
    cur_ev.clear();
    size_t pk = 0;  // next candidate in prev_lv
    auto wait_prev = [&](int need) {  // iteration i-1 done with level `need`
      if (prev_lv.empty()) return;
      while (pk + 1 < prev_lv.size() && prev_lv[pk] < need) ++pk;
      ck(cudaStreamWaitEvent(w, prev_ev[pk], 0), "wait");
    };
    ck(cudaStreamWaitEvent(w, c->band_ev[i], 0), "wait");
    ck(launch_aos_to_planar_rows(reinterpret_cast<const float*>(dx + row_bytes * r0),
                                 reinterpret_cast<const float*>(dv + row_bytes * r0), st[0], nx,
                                 r0, tops[i] - r0, S, c->pitch, c->zs, w),
       "aos_to_planar");
    ck(cudaEventRecord(lev[0], w), "event");
    cur_lv.push_back(0);
    cur_ev.push_back(lev[0]);
    int last = 0;
    for (int L = 1; L <= steps; ++L) {
      const int lo = top(i - 1, L), hi = top(i, L);
      if (hi <= lo) continue;
      wait_prev(L - 1);
      a.in = st[(L - 1) & 1];
      a.out = st[L & 1];
      a.k = k0 + L - 1;
      a.u0 = lo;
      a.u1 = hi;
      FastPlan pl = range_plan(c, hi - lo, c->any_general);
      if (chunk_plan) {  // the chunked-stepping segmentation: concurrent launches fill the slots
        pl.wide = pl.chunk_wide;
        pl.n_segs = pl.chunk_segs;
        pl.seg_rows = (hi - lo + pl.n_segs - 1) / pl.n_segs;
        pl.units = static_cast<int64_t>(a.batch) * pl.n_strips * pl.n_segs;
      }
      ck(launch_fast(a, c->fast, c->tmap[cur0 ^ ((L - 1) & 1)], pl, w), "kernel launch");
      ++launches;
      last = L;
      if (L % G == 0) {
        cudaEvent_t e = lev[cur_ev.size()];
        ck(cudaEventRecord(e, w), "event");
        cur_lv.push_back(L);
        cur_ev.push_back(e);
      }
    }
    if (cur_lv.back() != last) {
      cudaEvent_t e = lev[cur_ev.size()];
      ck(cudaEventRecord(e, w), "event");
      cur_lv.push_back(last);
      cur_ev.push_back(e);
    }
    const int f0 = top(i - 1, steps), f1 = top(i, steps);  // rows at the last level
    if (f1 > f0) {
      ck(launch_planar_to_aos_rows(st[steps & 1], reinterpret_cast<float*>(dx + row_bytes * f0),
                                   reinterpret_cast<float*>(dv + row_bytes * f0), nx, f0,
                                   f1 - f0, S, c->pitch, c->zs, w),
         "planar_to_aos");
      ck(cudaEventRecord(c->band_ev[nb + i], w), "event");
      ck(cudaStreamWaitEvent(out, c->band_ev[nb + i], 0), "wait");
      const size_t off = row_bytes * f0, n = row_bytes * (f1 - f0);
      ck(cudaMemcpyAsync(static_cast<unsigned char*>(xo) + off, dx + off, n,
                         cudaMemcpyDeviceToHost, out), "D2H x");
      ck(cudaMemcpyAsync(static_cast<unsigned char*>(vo) + off, dv + off, n,
                         cudaMemcpyDeviceToHost, out), "D2H v");
      launches += 1;
    }
    std::swap(prev_lv, cur_lv);
    std::swap(prev_ev, cur_ev);
  }
  // the ctx stream continues after the downloads and both compute streams
  ck(cudaEventRecord(c->pipe_ev[16], out), "event");
  ck(cudaStreamWaitEvent(c->stream, c->pipe_ev[16], 0), "wait");
  for (int j = 0; j < 2; ++j) {
    cudaEvent_t e = c->band_ev[2 * nb + 2 * nlev + j];
    ck(cudaEventRecord(e, q[j]), "event");
    ck(cudaStreamWaitEvent(c->stream, e, 0), "wait");
  }
  c->launches.fetch_add(launches + nb);
  c->cur = cur0 ^ (steps & 1);
  return true;
}

}  // namespace

// ============================================================================ C ABI =====

extern "C" {

int sc_abi_version(void) { return SC_ABI_VERSION; }

const char* sc_last_error(void) { return g_err.c_str(); }

sc_status sc_ctx_create(int device, sc_precision precision, sc_ctx** out) {
  return guarded([&] {
    if (!out) throw_config("out: null");
    *out = nullptr;
    if (precision != SC_F32 && precision != SC_F64) throw_config("precision: unknown");
    int n = 0;
    ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n)
      throw Fail{SC_ERR_CUDA, "device " + std::to_string(device) + " not present (" +
                                  std::to_string(n) + " visible)"};
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      throw Fail{SC_ERR_CUDA, std::string("kernels are built for sm_100a; device is ") +
                                  prop.name};
    auto* c = new sc_ctx();
    c->device = device;
    c->prec = precision;
    c->health_on = precision == SC_F64;  // the reference's f64 rollout checks; run_steps<float> does not
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    ck(cudaEventCreate(&c->ev0), "cudaEventCreate");
    ck(cudaEventCreate(&c->ev1), "cudaEventCreate");
    *out = c;
  });
}

void sc_ctx_destroy(sc_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_scene(c);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (cudaEvent_t e : c->frame_ev)
    if (e) cudaEventDestroy(e);
  for (auto& q : c->peer)
    for (void* o : q.opened)
      if (o) cudaIpcCloseMemHandle(o);
  c->peer_flags.release();
  if (c->pin_stage) cudaFreeHost(c->pin_stage);
  for (cudaStream_t q : c->pipe_stream)
    if (q) cudaStreamDestroy(q);
  for (cudaEvent_t e : c->pipe_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->band_ev) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

sc_status sc_ctx_set_strip(sc_ctx* c, int32_t row0, int32_t rows) {
  return guarded([&] {
    if (!c) throw_state("null context");
    // the stencil reaches 2 rows: a strip must own at least the 2 rows its halo ships
    if (row0 < 0 || rows < 2) throw_config("strip: row0 must be >= 0 and rows >= 2");
    c->strip_row0 = row0;
    c->strip_rows = rows;
  });
}

sc_status sc_ctx_set_scene(sc_ctx* c, const sc_scene_desc* s) {
  return guarded([&] {
    if (!c) throw_state("null context");
    validate_scene(s);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ck(cudaStreamSynchronize(c->stream), "sync");
    free_scene(c);
    c->nx = s->nx;
    c->ny = s->ny;
    c->batch = s->batch;
    if (c->strip_row0 >= 0) {
      if (s->batch != 1) throw_config("strip: row-strip decomposition needs batch == 1");
      if (c->strip_row0 + c->strip_rows > s->ny) throw_config("strip: rows exceed grid.ny");
      c->u0 = c->strip_row0;
      c->u1 = c->strip_row0 + c->strip_rows;
      c->g0 = std::max(0, c->u0 - 2);
      c->rows_local = std::min(s->ny, c->u1 + 2) - c->g0;
    } else {
      c->u0 = 0;
      c->u1 = s->ny;
      c->g0 = 0;
      c->rows_local = s->ny;
    }
    c->pitch = (s->nx + 3) / 4 * 4;
    c->plane_stride = static_cast<int64_t>(c->rows_local) * c->pitch;
    c->state_bytes = static_cast<size_t>(c->batch) * 6 * c->plane_stride * c->elem();
    for (int i = 0; i < 2; ++i) {
      ck(cudaMalloc(&c->state[i], c->state_bytes), "cudaMalloc(state)");
      ck(cudaMemsetAsync(c->state[i], 0, c->state_bytes, c->stream), "memset(state)");
    }
    c->cur = 0;
    if (c->prec == SC_F32)
      upload_scene<float>(c, s);
    else
      upload_scene<double>(c, s);
    c->health.ensure(static_cast<size_t>(c->batch));
    reset_health(c);
    c->any_pressure = c->any_general = false;
    c->pbs_ok = true;
    for (int b = 0; b < s->batch; ++b) c->pbs_ok = c->pbs_ok && s->cloths[b].spacing > 0.0;
    for (int b = 0; b < s->batch; ++b) {
      const sc_cloth_desc& d = s->cloths[b];
      const bool pres = d.plug_pressure && static_cast<float>(d.pressure) != 0.0f;
      c->any_pressure = c->any_pressure || pres;
      c->any_general = c->any_general || pres || d.n_spheres > 0 || d.n_planes > 0;
    }
    // the z-plane swizzle pays on the general-finish FAST kernel only (sc_device.cuh z_col); the
    // state is (re)initialised after set_scene, so the layout is fixed here
    c->zs = c->prec == SC_F32 && c->any_general;
    // ... except when every collider cloth has one collider of one kind — one frictionless plane
    // (config 5) or one sphere (config 3): the kernels with that finish alone run faster on the
    // plain layout (config 5's class-grouped step 0.598 -> 0.583 ms with the plane finish; config
    // 3 22.1 -> 21.7 us with the sphere-only streaming kernel)
    if (c->strip_row0 < 0 && !c->any_pressure && (plane_only_scene(s) || sphere_only_scene(s)))
      c->zs = false;
    if (const char* env = std::getenv("SC_ZSWIZZLE")) c->zs = c->prec == SC_F32 && std::atoi(env);
    if (c->prec == SC_F32) {
      build_tmaps(c);
      c->plan = plan_fast(c->nx, c->u1 - c->u0, c->batch, c->device, c->any_pressure,
                          c->any_general);
      c->plan_gen = plan_fast(c->nx, c->u1 - c->u0, c->batch, c->device, c->any_pressure, true);
      c->wave = WavePlan{};
      c->grouped = false;
      c->plane_only = false;
      c->sphere_only = false;
      c->small_ok = c->strip_row0 < 0 && !c->any_pressure && small_supported(c->nx, c->ny);
      if (c->strip_row0 < 0 && !c->any_pressure) {
        // every collider cloth has one frictionless plane and no sphere (config 5)
        c->plane_only = plane_only_scene(s);
        c->sphere_only = sphere_only_scene(s);
        if (const char* env = std::getenv("SC_PLANE_ONLY")) c->plane_only = c->plane_only && std::atoi(env);
        c->plan.only = c->plan_gen.only = c->plane_only ? 1 : c->sphere_only ? 2 : 0;
        c->wave = plan_wave(c->nx, c->ny, c->batch, c->device, c->any_general, 0, c->plane_only);
        std::vector<int32_t> simple, general;
        for (int b = 0; b < s->batch; ++b)
          (s->cloths[b].n_spheres > 0 || s->cloths[b].n_planes > 0 ? general : simple).push_back(b);
        bool want = !simple.empty() && !general.empty();
        if (const char* env = std::getenv("SC_GROUP")) want = want && std::atoi(env) != 0;
        if (want) {
          // the two groups run concurrently: the wavefront kernel on part of the SMs, the
          // streaming launches of the collider cloths on the rest. Split measured on config 5
          // (tools/cfg5_class_probe.py, SC_GROUP_SMS sweep: 100-108 of 148 SMs best for 2731
          // collider-free + 1365 plane cloths): SMs in proportion to 1.05 x collider-free
          // cloths : 1 x collider cloths
          int sms = 148;
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
          const double ws = 1.05 * simple.size(), wg = 1.0 * general.size();
          int wave_sms = static_cast<int>(sms * ws / (ws + wg) + 0.5);
          if (const char* env = std::getenv("SC_GROUP_SMS")) wave_sms = std::atoi(env);
          wave_sms = std::max(1, std::min(sms, wave_sms));
          c->wave_simple = plan_wave(c->nx, c->ny, static_cast<int>(simple.size()), c->device, false,
                                     wave_sms);
          if (c->wave_simple.ok) {
            c->n_simple = static_cast<int>(simple.size());
            c->n_general = static_cast<int>(general.size());
            c->ids_simple.ensure(simple.size());
            c->ids_general.ensure(general.size());
            ck(cudaMemcpy(c->ids_simple.p, simple.data(), sizeof(int32_t) * simple.size(),
                          cudaMemcpyHostToDevice), "cudaMemcpy(ids)");
            ck(cudaMemcpy(c->ids_general.p, general.data(), sizeof(int32_t) * general.size(),
                          cudaMemcpyHostToDevice), "cudaMemcpy(ids)");
            c->plan_general = plan_fast(c->nx, c->u1 - c->u0, c->n_general, c->device, false, true,
                                        sms - c->wave_simple.ctas);
            c->plan_general.only = c->plane_only ? 1 : c->sphere_only ? 2 : 0;
            c->grouped = true;
          }
        }
      }
      if (!c->wave_pinned) {
        c->wave_on = true;
        if (const char* env = std::getenv("SC_WAVE")) c->wave_on = std::atoi(env) != 0;
      }
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->has_scene = true;
    // FAST eligibility depends on the grid (nx % 4) as well as the gains: re-derive it for
    // the bound parameters whenever the scene changes
    c->fast_ok = c->has_params && fast_supported(c->net32, c->nx);
  });
}

sc_status sc_ctx_set_params(sc_ctx* c, const sc_params* p) {
  return guarded([&] {
    if (!c) throw_state("null context");
    if (!p) throw_config("params: null");
    if (!(p->isru_alpha > 0.0)) throw_config("isru_alpha: must be > 0");
    c->net32 = make_net<float>(p);
    c->net64 = make_net<double>(p);
    c->fast = make_fast_net(c->net32);
    // without a bound scene nx is unknown: sc_ctx_set_scene re-derives fast_ok
    c->fast_ok = c->has_scene && fast_supported(c->net32, c->nx);
    c->has_params = true;
  });
}

sc_status sc_ctx_set_state(sc_ctx* c, const void* x, const void* v) {
  return guarded([&] {
    require_ready(c, false);
    if (!x || !v) throw_config("state: null array");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    upload_state(c, x, v);
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

sc_status sc_ctx_get_state(sc_ctx* c, void* x, void* v) {
  return guarded([&] {
    require_ready(c, false);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    download_state(c, c->cur, x, v);
  });
}

sc_status sc_ctx_advance(sc_ctx* c, int32_t steps, int32_t k0, sc_mode mode) {
  return guarded([&] {
    require_ready(c);
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    advance_impl(c, steps, k0, mode, nullptr);
  });
}

sc_status sc_ctx_set_persistent(sc_ctx* c, int32_t on) {
  return guarded([&] {
    if (!c) throw_state("null context");
    c->wave_on = on != 0;
    c->wave_pinned = true;  // an explicit choice outlives later set_scene calls
  });
}

sc_status sc_ctx_set_health_checks(sc_ctx* c, int32_t on) {
  return guarded([&] {
    if (!c) throw_state("null context");
    c->health_on = on != 0;
  });
}

sc_status sc_ctx_sync(sc_ctx* c) {
  return guarded([&] {
    if (!c) throw_state("null context");
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

sc_status sc_ctx_get_health(sc_ctx* c, int32_t* bad_imp_frame, int32_t* bad_imp_node,
                            int32_t* bad_state_frame) {
  return guarded([&] {
    require_ready(c, false);
    std::vector<Health> h(static_cast<size_t>(c->batch));
    ck(cudaMemcpyAsync(h.data(), c->health.p, sizeof(Health) * h.size(), cudaMemcpyDeviceToHost,
                       c->stream),
       "D2H health");
    ck(cudaStreamSynchronize(c->stream), "sync");
    for (int b = 0; b < c->batch; ++b) {
      const Health& x = h[static_cast<size_t>(b)];
      const bool imp_bad = x.impulse_key != ~0ull;
      if (bad_imp_frame) bad_imp_frame[b] = imp_bad ? static_cast<int32_t>(x.impulse_key >> 32) : -1;
      if (bad_imp_node)
        bad_imp_node[b] = imp_bad ? static_cast<int32_t>(x.impulse_key & 0xffffffffu) : -1;
      if (bad_state_frame) bad_state_frame[b] = x.state_frame == INT_MAX ? -1 : x.state_frame;
    }
  });
}

sc_status sc_rollout(sc_ctx* c, const void* x0, const void* v0, int32_t steps, int32_t k0,
                     sc_mode mode, void* x_out, void* v_out, uint8_t* constrained) {
  return guarded([&] {
    require_ready(c);
    if (!x0 || !v0) throw_config("state: null array");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_health(c);
    if (!constrained && mode == SC_MODE_FAST && steps > 0 &&
        (rollout_wave_pipelined(c, x0, v0, steps, k0, x_out, v_out) ||
         rollout_pipelined(c, x0, v0, steps, k0, x_out, v_out) ||
         rollout_band_pipelined(c, x0, v0, steps, k0, x_out, v_out))) {
      ck(cudaStreamSynchronize(c->stream), "sync");
      return;
    }
    upload_state(c, x0, v0);
    uint8_t* dm = nullptr;
    if (constrained && steps > 0) {
      c->mask.ensure(static_cast<size_t>(c->batch) * c->nodes_global());
      dm = c->mask.p;
    }
    advance_impl(c, steps, k0, mode, dm);
    download_state(c, c->cur, x_out, v_out, false);
    if (constrained) {
      const size_t n = static_cast<size_t>(c->batch) * c->nodes_global();
      if (dm)
        ck(cudaMemcpyAsync(constrained, dm, n, cudaMemcpyDeviceToHost, c->stream), "D2H mask");
      else
        std::memset(constrained, 0, n);
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

sc_status sc_rollout_frames(sc_ctx* c, const void* x0, const void* v0, int32_t steps,
                            int32_t stride, sc_mode mode, void* fx, void* fv) {
  return guarded([&] {
    require_ready(c);
    if (stride < 1) throw_config("stride: must be >= 1");
    if (!x0 || !v0 || !fx || !fv) throw_config("frames: null array");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_health(c);
    frames_impl(c, x0, v0, steps, stride, fx, fv,
                [&](int n, int k) { advance_impl(c, n, k, mode, nullptr); });
  });
}

}  // extern "C"

namespace {
// Shared body of the per-operator entry points: the state is uploaded into the ctx front
// buffer (these calls replace the resident state), the impulse staged as AoS.
template <typename T>
void op_call(sc_ctx* c, int kind, sc_mode mode, const void* x, const void* v,
             const void* impulse_in, void* impulse_out, double t_next, void* xo, void* vo,
             uint8_t* constrained) {
  const size_t bytes = static_cast<size_t>(c->batch) * c->nodes_local() * 3 * sizeof(T);
  upload_state(c, x, v);
  T* dimp = reinterpret_cast<T*>(c->aos.p + 2 * bytes);
  if (impulse_in)
    ck(cudaMemcpyAsync(dimp, impulse_in, bytes, cudaMemcpyHostToDevice, c->stream), "H2D imp");
  uint8_t* dm = nullptr;
  if (constrained) {
    c->mask.ensure(static_cast<size_t>(c->batch) * c->nodes_global());
    dm = c->mask.p;
  }
  launch_one<T>(c, kind, mode, 0, true, t_next, dm, dimp, c->health.p, c->u0, c->u1, c->stream);
  if (impulse_out)
    ck(cudaMemcpyAsync(impulse_out, dimp, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H imp");
  if (kind == KIND_STEP || kind == KIND_ADVANCE || kind == KIND_PBS) {
    download_state(c, 1 - c->cur, xo, vo, false);
    if (constrained)
      ck(cudaMemcpyAsync(constrained, dm, static_cast<size_t>(c->batch) * c->nodes_global(),
                         cudaMemcpyDeviceToHost, c->stream),
         "D2H mask");
  }
  ck(cudaStreamSynchronize(c->stream), "sync");
}

// NumericsError of the PBS step: a singular spring (kernels.hpp:105-107, batch 1 node index),
// then a non-finite state (sim.cpp:153 -> diagnose_divergence; the force term is named by the
// Python layer, which can evaluate the terms separately).
void pbs_check(sc_ctx* c, bool state) {
  std::vector<Health> h(static_cast<size_t>(c->batch));
  ck(cudaMemcpy(h.data(), c->health.p, sizeof(Health) * h.size(), cudaMemcpyDeviceToHost),
     "D2H health");
  for (int b = 0; b < c->batch; ++b)
    if (h[static_cast<size_t>(b)].impulse_key != ~0ull)
      throw Fail{SC_ERR_NUMERICS, "elastic force: singular spring (coincident nodes) at node " +
                                      std::to_string(h[static_cast<size_t>(b)].impulse_key &
                                                     0xffffffffu)};
  if (state)
    for (int b = 0; b < c->batch; ++b)
      if (h[static_cast<size_t>(b)].state_frame != INT_MAX)
        throw Fail{SC_ERR_NUMERICS, "non-finite state update (reduce dt or stiffness)"};
}

sc_status op_entry(sc_ctx* c, int kind, sc_mode mode, const void* x, const void* v,
                   const void* imp_in, void* imp_out, double t_next, void* xo, void* vo,
                   uint8_t* constrained, bool need_params) {
  return guarded([&] {
    require_ready(c, need_params);
    if (!x || !v) throw_config("state: null array");
    if (c->strip_row0 >= 0) throw_config("per-operator entry points need a whole-cloth context");
    if (mode == SC_MODE_FAST && c->prec != SC_F32) throw_config("mode: FAST is an f32 mode");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    reset_health(c);
    if ((kind == KIND_PBS || kind == KIND_TOTAL || kind == KIND_FORCE) && !c->pbs_ok)
      throw_config("grid.spacing: must be a finite value > 0 (rest lengths of the PBS step)");
    if (c->prec == SC_F32)
      op_call<float>(c, kind, mode, x, v, imp_in, imp_out, t_next, xo, vo, constrained);
    else
      op_call<double>(c, kind, mode, x, v, imp_in, imp_out, t_next, xo, vo, constrained);
    if (kind == KIND_PBS || kind == KIND_TOTAL || kind == KIND_FORCE) pbs_check(c, kind == KIND_PBS);
  });
}
}  // namespace

extern "C" {

sc_status sc_forward_impulse(sc_ctx* c, const void* x, const void* v, void* impulse) {
  if (!impulse) {
    g_err = "impulse: null array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_FORWARD, SC_MODE_PARITY, x, v, nullptr, impulse, 0.0, nullptr, nullptr,
                  nullptr, true);
}

sc_status sc_plug_impulse(sc_ctx* c, const void* x, const void* v, void* impulse) {
  if (!impulse) {
    g_err = "impulse: null array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_PLUG, SC_MODE_PARITY, x, v, nullptr, impulse, 0.0, nullptr, nullptr,
                  nullptr, false);
}

sc_status sc_advance_with_impulse(sc_ctx* c, const void* x, const void* v, const void* impulse,
                                  double t_next, void* xo, void* vo, uint8_t* constrained) {
  if (!impulse || !xo || !vo) {
    g_err = "advance_with_impulse: null array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_ADVANCE, SC_MODE_PARITY, x, v, impulse, nullptr, t_next, xo, vo,
                  constrained, false);
}

sc_status sc_nn_step(sc_ctx* c, const void* x, const void* v, double t_next, sc_mode mode,
                     void* xo, void* vo, uint8_t* constrained) {
  if (!xo || !vo) {
    g_err = "nn_step: null output array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_STEP, mode, x, v, nullptr, nullptr, t_next, xo, vo, constrained, true);
}

sc_status sc_total_impulse(sc_ctx* c, const void* x, const void* v, void* impulse) {
  if (!impulse) {
    g_err = "impulse: null array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_TOTAL, SC_MODE_PARITY, x, v, nullptr, impulse, 0.0, nullptr, nullptr,
                  nullptr, false);
}

sc_status sc_total_force(sc_ctx* c, const void* x, const void* v, void* force) {
  if (!force) {
    g_err = "force: null array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_FORCE, SC_MODE_PARITY, x, v, nullptr, force, 0.0, nullptr, nullptr,
                  nullptr, false);
}

sc_status sc_pbs_step(sc_ctx* c, const void* x, const void* v, double t_next, void* xo, void* vo,
                      uint8_t* constrained) {
  if (!xo || !vo) {
    g_err = "pbs_step: null output array";
    return SC_ERR_CONFIG;
  }
  return op_entry(c, KIND_PBS, SC_MODE_PARITY, x, v, nullptr, nullptr, t_next, xo, vo,
                  constrained, false);
}

sc_status sc_simulate_frames(sc_ctx* c, const void* x0, const void* v0, int32_t steps,
                             int32_t stride, void* fx, void* fv) {
  return guarded([&] {
    require_ready(c, false);
    if (!c->pbs_ok)
      throw_config("grid.spacing: must be a finite value > 0 (rest lengths of the PBS step)");
    if (stride < 1) throw_config("stride: must be >= 1");
    if (!x0 || !v0 || !fx || !fv) throw_config("frames: null array");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    const bool health_before = c->health_on;
    c->health_on = true;  // simulate_scene checks every step (sim.cpp:153)
    reset_health(c);
    try {
      frames_impl(c, x0, v0, steps, stride, fx, fv, [&](int n, int k) {
        advance_impl(c, n, k, SC_MODE_PARITY, nullptr, KIND_PBS);
      });
    } catch (...) {
      c->health_on = health_before;
      throw;
    }
    c->health_on = health_before;
  });
}

sc_status sc_benchmark_sim(sc_ctx* c, int32_t steps, int32_t warmup, double* seconds) {
  return guarded([&] {
    require_ready(c, false);
    if (!c->pbs_ok)
      throw_config("grid.spacing: must be a finite value > 0 (rest lengths of the PBS step)");
    if (steps < 1) throw_config("bench: steps must be >= 1");
    if (warmup < 0) throw_config("bench: warmup must be >= 0");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    advance_impl(c, warmup, 0, SC_MODE_PARITY, nullptr, KIND_PBS);
    ck(cudaEventRecord(c->ev0, c->stream), "event");
    advance_impl(c, steps, warmup, SC_MODE_PARITY, nullptr, KIND_PBS);
    ck(cudaEventRecord(c->ev1, c->stream), "event");
    ck(cudaEventSynchronize(c->ev1), "event sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event time");
    if (seconds) *seconds = ms * 1e-3;
  });
}

sc_status sc_benchmark(sc_ctx* c, int32_t steps, int32_t warmup, sc_mode mode, double* seconds) {
  return guarded([&] {
    require_ready(c);
    if (steps < 1) throw_config("bench: steps must be >= 1");
    if (warmup < 0) throw_config("bench: warmup must be >= 0");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    advance_impl(c, warmup, 0, mode, nullptr);
    ck(cudaEventRecord(c->ev0, c->stream), "event");
    advance_impl(c, steps, warmup, mode, nullptr);
    ck(cudaEventRecord(c->ev1, c->stream), "event");
    ck(cudaEventSynchronize(c->ev1), "event sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, c->ev0, c->ev1), "event time");
    if (seconds) *seconds = ms * 1e-3;
  });
}

sc_status sc_benchmark_launches(sc_ctx* c, int32_t steps, int32_t k0, sc_mode mode,
                                float* launch_ms) {
  return guarded([&] {
    require_ready(c);
    if (steps < 1) throw_config("bench: steps must be >= 1");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    std::vector<cudaEvent_t> ev(static_cast<size_t>(steps) + 1);
    for (auto& e : ev) ck(cudaEventCreate(&e), "cudaEventCreate");
    ck(cudaEventRecord(ev[0], c->stream), "event");
    for (int s = 0; s < steps; ++s) {
      advance_impl(c, 1, k0 + s, mode, nullptr);
      ck(cudaEventRecord(ev[static_cast<size_t>(s) + 1], c->stream), "event");
    }
    ck(cudaEventSynchronize(ev.back()), "event sync");
    for (int s = 0; s < steps; ++s)
      ck(cudaEventElapsedTime(&launch_ms[s], ev[static_cast<size_t>(s)],
                              ev[static_cast<size_t>(s) + 1]),
         "event time");
    for (auto& e : ev) cudaEventDestroy(e);
  });
}

int64_t sc_ctx_halo_elems(sc_ctx* c) { return c ? static_cast<int64_t>(6) * 2 * c->pitch : 0; }

}  // extern "C"

namespace {
void halo_copy(sc_ctx* c, int side, void* dev, bool pack, cudaStream_t st) {
  require_ready(c, false);
  if (c->strip_row0 < 0) throw_config("halo: context has no strip");
  if (side != 0 && side != 1) throw_config("halo: side must be 0 or 1");
  // pack: owned rows next to the edge; unpack: ghost rows beyond the edge
  int grow;
  if (pack)
    grow = side == 0 ? c->u0 : c->u1 - 2;
  else
    grow = side == 0 ? c->u0 - 2 : c->u1;
  const size_t e = c->elem();
  const int64_t S = c->plane_stride;
  unsigned char* buf = static_cast<unsigned char*>(c->state[1 - c->cur]);
  // halo buffer [2 rows][x.xy 2p | v.xy 2p | x.z p | v.z p] = 6*pitch elements per row (whole
  // rows in the device layout, swizzle included)
  for (int r = 0; r < 2; ++r) {
    const int g = grow + r;
    if (g < 0 || g >= c->ny) continue;
    const int64_t lr = g - c->g0;
    // whole rows: the column swizzles permute within 4-column groups only
    const int64_t seg_off[4] = {elem_index(0, lr, 0, c->pitch, S, false),
                                elem_index(3, lr, 0, c->pitch, S, false),
                                elem_index(2, lr, 0, c->pitch, S, false),
                                elem_index(5, lr, 0, c->pitch, S, false)};
    const int64_t seg_len[4] = {2LL * c->pitch, 2LL * c->pitch, c->pitch, c->pitch};
    int64_t hoff = static_cast<int64_t>(r) * 6 * c->pitch;
    for (int q = 0; q < 4; ++q) {
      unsigned char* st_ptr = buf + seg_off[q] * e;
      unsigned char* h_ptr = static_cast<unsigned char*>(dev) + hoff * e;
      if (pack)
        ck(cudaMemcpyAsync(h_ptr, st_ptr, seg_len[q] * e, cudaMemcpyDeviceToDevice, st), "halo");
      else
        ck(cudaMemcpyAsync(st_ptr, h_ptr, seg_len[q] * e, cudaMemcpyDeviceToDevice, st), "halo");
      hoff += seg_len[q];
    }
  }
}
}  // namespace

extern "C" {

sc_status sc_ctx_halo_pack(sc_ctx* c, int32_t side, void* dev_dst, void* stream) {
  return guarded([&] {
    halo_copy(c, side, dev_dst, true, stream ? static_cast<cudaStream_t>(stream) : c->stream);
  });
}

sc_status sc_ctx_halo_unpack(sc_ctx* c, int32_t side, const void* dev_src, void* stream) {
  return guarded([&] {
    halo_copy(c, side, const_cast<void*>(dev_src), false,
              stream ? static_cast<cudaStream_t>(stream) : c->stream);
  });
}

sc_status sc_ctx_strip_step(sc_ctx* c, int32_t k, int32_t r_begin, int32_t r_end, sc_mode mode,
                            void* stream) {
  return guarded([&] {
    require_ready(c);
    if (r_begin < c->u0 || r_end > c->u1 || r_begin > r_end)
      throw_config("strip_step: rows outside the owned strip");
    if (mode == SC_MODE_FAST && c->prec != SC_F32) throw_config("mode: FAST is an f32 mode");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    Health* h = c->health_on ? c->health.p : nullptr;
    if (c->prec == SC_F32)
      launch_one<float>(c, KIND_STEP, mode, k, false, 0.0, nullptr, nullptr, h, r_begin, r_end, st);
    else
      launch_one<double>(c, KIND_STEP, mode, k, false, 0.0, nullptr, nullptr, h, r_begin, r_end,
                         st);
  });
}

sc_status sc_ctx_strip_commit(sc_ctx* c) {
  return guarded([&] {
    require_ready(c, false);
    c->cur = 1 - c->cur;
  });
}

void* sc_ctx_stream(sc_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

sc_status sc_ctx_state_buffers(sc_ctx* c, void** front, void** back, int64_t* plane_stride,
                               int32_t* pitch, int32_t* local_rows, int32_t* row_base) {
  return guarded([&] {
    require_ready(c, false);
    if (front) *front = c->state[c->cur];
    if (back) *back = c->state[1 - c->cur];
    if (plane_stride) *plane_stride = c->plane_stride;
    if (pitch) *pitch = c->pitch;
    if (local_rows) *local_rows = c->rows_local;
    if (row_base) *row_base = c->g0;
  });
}

}  // extern "C"

namespace {
// Peer-step handshake. A neighbour writes `steps completed` into our flag slot after each fused
// step (system-scope release after a system fence, so its remote ghost-row stores are visible
// first); before our n-th step we wait for n from both neighbours: their step n-1 wrote our
// ghost rows, and they are done reading the buffer whose ghost rows our step n overwrites.
__global__ void peer_wait_kernel(const unsigned* flags, int need0, int need1, unsigned target) {
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  for (int sd = 0; sd < 2; ++sd) {
    if (!(sd == 0 ? need0 : need1)) continue;
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + sd) : "memory");
      if (v >= target) break;
      __nanosleep(256);
      if (clock64() - t0 > (1LL << 35)) __trap();  // ~15 s: a neighbour is gone
    }
  }
}

__global__ void peer_signal_kernel(unsigned* f0, unsigned* f1, unsigned val) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  if (f0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f0), "r"(val) : "memory");
  if (f1) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f1), "r"(val) : "memory");
}
}  // namespace

extern "C" {

sc_status sc_ctx_peer_export(sc_ctx* c, sc_peer_export* out) {
  return guarded([&] {
    require_ready(c, false);
    if (!out) throw_config("peer export: null");
    if (c->strip_row0 < 0) throw_config("peer export: context has no strip");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    c->peer_flags.ensure(2);
    std::memset(out, 0, sizeof *out);
    for (int i = 0; i < 2; ++i) {
      cudaIpcMemHandle_t h;
      ck(cudaIpcGetMemHandle(&h, c->state[i]), "cudaIpcGetMemHandle");
      std::memcpy(out->state_handle[i], &h, sizeof h);
      out->state_ptr[i] = c->state[i];
    }
    cudaIpcMemHandle_t hf;
    ck(cudaIpcGetMemHandle(&hf, c->peer_flags.p), "cudaIpcGetMemHandle");
    std::memcpy(out->flags_handle, &hf, sizeof hf);
    out->flags_ptr = c->peer_flags.p;
    out->plane_stride = c->plane_stride;
    out->g0 = c->g0;
    out->u0 = c->u0;
    out->u1 = c->u1;
    out->nx = c->nx;
    out->pitch = c->pitch;
    out->batch = c->batch;
    out->cur = c->cur;
    out->device = c->device;
  });
}

sc_status sc_ctx_set_peer(sc_ctx* c, int32_t side, const sc_peer_export* nb, int32_t use_ipc) {
  return guarded([&] {
    require_ready(c, false);
    if (c->strip_row0 < 0) throw_config("peer: context has no strip");
    if (side != 0 && side != 1) throw_config("peer: side must be 0 or 1");
    if (!nb) throw_config("peer: null export");
    if (nb->nx != c->nx || nb->pitch != c->pitch || nb->batch != c->batch)
      throw_config("peer: neighbour has a different grid layout");
    if (side == 0 ? nb->u1 != c->u0 : nb->u0 != c->u1)
      throw_config("peer: neighbour strip is not adjacent on that side");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    sc_ctx::Peer& q = c->peer[side];
    for (void*& o : q.opened)
      if (o) {
        cudaIpcCloseMemHandle(o);
        o = nullptr;
      }
    void* p[3];
    if (use_ipc) {
      for (int i = 0; i < 2; ++i) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, nb->state_handle[i], sizeof h);
        ck(cudaIpcOpenMemHandle(&p[i], h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        q.opened[i] = p[i];
      }
      cudaIpcMemHandle_t hf;
      std::memcpy(&hf, nb->flags_handle, sizeof hf);
      ck(cudaIpcOpenMemHandle(&p[2], hf, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      q.opened[2] = p[2];
    } else {
      p[0] = nb->state_ptr[0];
      p[1] = nb->state_ptr[1];
      p[2] = nb->flags_ptr;
    }
    q.buf[0] = p[0];
    q.buf[1] = p[1];
    q.S = nb->plane_stride;
    q.g0 = nb->g0;
    q.cur_delta = (nb->cur ^ c->cur) & 1;
    q.ipc = use_ipc != 0;
    // we are its neighbour on the opposite side
    q.flag = static_cast<unsigned*>(p[2]) + (side == 0 ? 1 : 0);
    c->peer_flags.ensure(2);
    // ordered on the ctx stream and complete before we return: the neighbours only signal
    // after the caller's barrier that follows every set_peer, so no signal can be lost
    ck(cudaMemsetAsync(c->peer_flags.p, 0, 2 * sizeof(unsigned), c->stream), "memset");
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->peer_count = 0;
  });
}

sc_status sc_ctx_peer_step(sc_ctx* c, int32_t k, sc_mode mode, void* stream) {
  return guarded([&] {
    require_ready(c);
    if (c->strip_row0 < 0) throw_config("peer step: context has no strip");
    if (mode != SC_MODE_FAST || c->prec != SC_F32)
      throw_config("peer step: the fused exchange runs in FAST f32 mode");
    if (!c->peer[0].buf[0] && !c->peer[1].buf[0]) throw_config("peer step: no peer linked");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->stream;
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    peer_wait_kernel<<<1, 32, 0, st>>>(c->peer_flags.p, c->peer[0].buf[0] != nullptr,
                                       c->peer[1].buf[0] != nullptr, c->peer_count);
    ck(cudaGetLastError(), "peer wait");
    c->peer_launch = true;
    Health* h = c->health_on ? c->health.p : nullptr;
    try {
      launch_one<float>(c, KIND_STEP, mode, k, false, 0.0, nullptr, nullptr, h, c->u0, c->u1, st);
    } catch (...) {
      c->peer_launch = false;
      throw;
    }
    c->peer_launch = false;
    peer_signal_kernel<<<1, 32, 0, st>>>(c->peer[0].flag, c->peer[1].flag, c->peer_count + 1);
    ck(cudaGetLastError(), "peer signal");
    c->launches.fetch_add(2);
    c->peer_count += 1;
    c->cur = 1 - c->cur;
  });
}

sc_status sc_host_alloc(size_t bytes, void** out) {
  return guarded([&] {
    if (!out) throw_config("out: null");
    ck(cudaHostAlloc(out, bytes, cudaHostAllocPortable), "cudaHostAlloc");
  });
}

void sc_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int64_t sc_ctx_launch_count(sc_ctx* c) { return c ? c->launches.load() : 0; }

// Debug instrumentation (not part of the public header): per-unit globaltimer stamps of the
// FAST kernel into a device buffer of 2 * units uint64 (nullptr switches it off).
sc_status sc_debug_unit_timing(void* dev_buf) {
  return guarded([&] { ck(set_unit_timing(static_cast<unsigned long long*>(dev_buf)), "timing"); });
}
int64_t sc_debug_units(sc_ctx* c) { return c ? c->plan.units : 0; }

}  // extern "C"

namespace scb {

bool ctx_scene_view(sc_ctx* c, SceneView* v) {
  if (!c || !c->has_scene || c->rows_local != c->ny) return false;
  v->cloths = c->cloths;
  v->spheres = c->spheres;
  v->planes = c->planes;
  v->anchors = c->anchors;
  v->pin_bits = c->pin_bits.p;
  v->pin_rank = c->pin_rank.p;
  v->nx = c->nx;
  v->ny = c->ny;
  v->batch = c->batch;
  v->device = c->device;
  return true;
}

void set_last_error(const std::string& msg) { g_err = msg; }

}  // namespace scb
