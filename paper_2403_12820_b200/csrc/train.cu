// Training forward + backward on the GPU and the native host training loop.
//
//   sample_batch   train.cpp:91-127   indices on the host (std::mt19937_64, rng.hpp), the
//                                     force-integration targets f_k*dt on the device
//   compute_loss   train.cpp:129-209  forward_impulse + plug_impulse + advance_with_impulse per
//                                     transition, physics/data residuals, hybrid loss
//   backward_gradients net.cpp:144-201 the 53 parameter-gradient sums
//   adam_update / schedule_lr / BoxSearch (the DE pre-search) / de_preprocess / train_loop
//                  train.cpp:54-63,212-375  host C++ over the 53 scalars, same RNG draws
//
// Bit-exactness with the reference (f64): every per-node quantity is the reference expression in
// non-contractible IEEE RN ops (this TU is compiled with --fmad=false), and every reduction keeps
// the reference's association order:
//   * loss sums: one sequential chain over (batch element, node) (train.cpp:168-182), run by a
//     single thread on a second stream, concurrent with the gradient kernels;
//   * gradients: per (batch element, fixed 1024-node chunk) one sequential chain per scalar
//     (net.cpp:152-199), chunk partials and batch elements then summed in order
//     (net.cpp:199, train.cpp:205). Channels a node lacks contribute +0.0, which is exact: an
//     accumulator that starts at +0.0 never becomes -0.0, and x + (+0.0) == x for every other x.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <random>
#include <string>
#include <vector>

#include "../../include/stencilcloth_b200.h"
#include "capi_internal.h"
#include "sc_device.cuh"

using namespace scb;

namespace {

constexpr int kChunk = 1024;   // backward_gradients' fixed chunk (net.cpp:151)
constexpr int kTerms = 64;     // per-node gradient terms (see kTerm* below)
constexpr int kScalars = 53;   // NetworkParams::kScalarCount
constexpr int kNone = 0x7F7F7F7F;
// term rows of the per-node scratch: for_each_gradient order (net.hpp:83-91) for the 52
// non-alpha scalars, then the 12 per-channel alpha terms (one chain over (node, channel))
constexpr int kTermKernel = 0, kTermLinear = 12, kTermBias = 24, kTermNonlin = 27,
              kTermDeriv = 39, kTermSelf = 51, kTermAlpha = 52;

struct Fail {
  sc_status code;
  std::string msg;
};
[[noreturn]] void fail(sc_status c, const std::string& m) { throw Fail{c, m}; }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
template <typename Fn>
sc_status guarded(Fn&& fn) {
  try {
    fn();
    return SC_OK;
  } catch (const Fail& f) {
    set_last_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SC_ERR_STATE;
  }
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void ensure(size_t count) {
    if (count <= n && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    ck(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)), "cudaMalloc(train)");
    n = count;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

// ------------------------------------------------------------------------- device ----
using R = RN<double>;

struct Frames {
  const double* fx;  // [F][n][3]
  const double* fv;
  const int32_t* idx;  // frame of each batch element
  int nx, ny;
  int64_t n;
};

__device__ __forceinline__ bool valid_channel(int ix, int iy, int nx, int ny, int c) {
  const int jx = ix + off_dx(c), jy = iy + off_dy(c);
  return jx >= 0 && jx < nx && jy >= 0 && jy < ny;
}
__device__ __forceinline__ int64_t nb(int64_t i, int nx, int c) {
  return i + static_cast<int64_t>(off_dy(c)) * nx + off_dx(c);
}
__device__ __forceinline__ double dot3(const double* a, const double* b) {
  return R::add(R::add(R::mul(a[0], b[0]), R::mul(a[1], b[1])), R::mul(a[2], b[2]));
}
__device__ __forceinline__ bool pinned_node(const ClothConst<double>& cc, const uint32_t* bits,
                                            int64_t i) {
  if (cc.n_pins <= 0) return false;
  return (__ldg(bits + cc.pin_word0 + (i >> 5)) >> (i & 31)) & 1u;
}

// sample_batch targets (train.cpp:111-124): f = elastic + damping [+ pressure], then
// (f + g*m - v*d) * dt with the plugged terms zeroed; each force field starts from zero.
struct TargetArgs {
  Frames fr;
  int batch;
  const ClothConst<double>* cloth;
  int plug_pressure, plug_gravity, plug_drag;  // raw scene plug flags (scene.hpp:56-58)
  double* force_dt;   // [batch][n][3]
  int32_t* bad_spring;  // [batch] min node with a singular spring
};

__global__ void __launch_bounds__(256) targets_kernel(const TargetArgs a) {
  const ClothConst<double>& cc = *a.cloth;
  const int64_t total = a.fr.n * a.batch;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(t / a.fr.n);
    const int64_t i = t - static_cast<int64_t>(b) * a.fr.n;
    const int ix = static_cast<int>(i % a.fr.nx), iy = static_cast<int>(i / a.fr.nx);
    const int64_t base = static_cast<int64_t>(a.fr.idx[b]) * a.fr.n * 3;
    const double* X = a.fr.fx + base;
    const double* V = a.fr.fv + base;
    double x[3], v[3];
    for (int d = 0; d < 3; ++d) {
      x[d] = X[3 * i + d];
      v[d] = V[3 * i + d];
    }
    double E[3] = {0.0, 0.0, 0.0}, D[3] = {0.0, 0.0, 0.0};
    bool singular = false;
    for (int c = 0; c < kChannels; ++c) {  // accumulate_elastic (kernels.hpp:86-108)
      if (!valid_channel(ix, iy, a.fr.nx, a.fr.ny, c)) continue;
      const int64_t j = nb(i, a.fr.nx, c);
      double dd[3];
      for (int d = 0; d < 3; ++d) dd[d] = R::sub(x[d], X[3 * j + d]);
      const double len = R::sqrt(dot3(dd, dd));
      if (len == 0.0) {
        singular = true;
        continue;
      }
      const double sc = R::div(R::mul(cc.stiffness, R::sub(len, cc.rest[c])), len);
      for (int d = 0; d < 3; ++d) E[d] = R::sub(E[d], R::mul(dd[d], sc));
    }
    for (int c = 0; c < kChannels; ++c) {  // accumulate_damping (kernels.hpp:112-136)
      if (!valid_channel(ix, iy, a.fr.nx, a.fr.ny, c)) continue;
      const int64_t j = nb(i, a.fr.nx, c);
      double dd[3], dv[3];
      for (int d = 0; d < 3; ++d) {
        dd[d] = R::sub(x[d], X[3 * j + d]);
        dv[d] = R::sub(v[d], V[3 * j + d]);
      }
      const double len = R::sqrt(dot3(dd, dd));
      if (len == 0.0) continue;
      double dir[3];
      for (int d = 0; d < 3; ++d) dir[d] = R::div(dd[d], len);
      const double sc = R::mul(cc.damping, dot3(dv, dir));
      for (int d = 0; d < 3; ++d) D[d] = R::sub(D[d], R::mul(dir[d], sc));
    }
    double f[3];
    for (int d = 0; d < 3; ++d) f[d] = R::add(E[d], D[d]);
    if (!a.plug_pressure) {  // pressure_force (kernels.hpp:142-155) on a zero field, added
      double fp[3] = {0.0, 0.0, 0.0};
      if (cc.pressure != 0.0 && ix >= 1 && ix <= a.fr.nx - 2 && iy >= 1 && iy <= a.fr.ny - 2) {
        double e[3], nn[3], w[3], s[3], c1[3], c2[3], c3[3], c4[3];
        for (int d = 0; d < 3; ++d) {
          e[d] = R::sub(x[d], X[3 * (i + 1) + d]);
          nn[d] = R::sub(x[d], X[3 * (i + a.fr.nx) + d]);
          w[d] = R::sub(x[d], X[3 * (i - 1) + d]);
          s[d] = R::sub(x[d], X[3 * (i - a.fr.nx) + d]);
        }
        auto cross = [](const double* p, const double* q, double* o) {
          o[0] = R::sub(R::mul(p[1], q[2]), R::mul(p[2], q[1]));
          o[1] = R::sub(R::mul(p[2], q[0]), R::mul(p[0], q[2]));
          o[2] = R::sub(R::mul(p[0], q[1]), R::mul(p[1], q[0]));
        };
        cross(e, nn, c1);
        cross(nn, w, c2);
        cross(w, s, c3);
        cross(s, e, c4);
        for (int d = 0; d < 3; ++d)
          fp[d] = R::add(fp[d], R::mul(R::add(R::add(R::add(c1[d], c2[d]), c3[d]), c4[d]),
                                       cc.pressure));
      }
      for (int d = 0; d < 3; ++d) f[d] = R::add(f[d], fp[d]);
    }
    const double drag = a.plug_drag ? 0.0 : cc.drag;
    double* out = a.force_dt + (static_cast<int64_t>(b) * a.fr.n + i) * 3;
    for (int d = 0; d < 3; ++d) {
      const double g = a.plug_gravity ? 0.0 : cc.grav[d];
      out[d] = R::mul(R::sub(R::add(f[d], R::mul(g, cc.mass)), R::mul(v[d], drag)), cc.dt);
    }
    if (singular) atomicMin(a.bad_spring + b, static_cast<int>(i));
  }
}

// compute_loss forward (train.cpp:146-182) for every (batch element, node).
struct LossArgs {
  Frames fr;
  int batch;
  const double* force_dt;
  double inv_mass;
  NetConst<double> net;
  StepArgs<double> sa;  // collider / pin tables for advance_node
  const ClothConst<double>* cloth;
  double* rp;  // [batch][n][3] physics residual (0 on pinned nodes)
  double* rd;  // [batch][n][3] data residual rv + rx*dt (0 on pinned / constrained nodes)
  double* phys_term;  // [batch][n] |r|^2 (0 where skipped)
  double* data_term;  // [batch][n] |rv|^2 + |rx|^2 (0 where skipped)
  unsigned long long* data_count;
  int32_t* bad_fwd;  // [batch] min node with a non-finite cell impulse
};

__global__ void __launch_bounds__(256) loss_fwd_kernel(const LossArgs a) {
  const ClothConst<double>& cc = *a.cloth;
  const int64_t total = a.fr.n * a.batch;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < total;
       base += stride) {
    const int64_t t = base + threadIdx.x;
    int counted = 0;
    if (t < total) {
      const int b = static_cast<int>(t / a.fr.n);
      const int64_t i = t - static_cast<int64_t>(b) * a.fr.n;
      const int ix = static_cast<int>(i % a.fr.nx), iy = static_cast<int>(i / a.fr.nx);
      const int k = a.fr.idx[b];
      const int64_t f0 = static_cast<int64_t>(k) * a.fr.n * 3;
      const double* X = a.fr.fx + f0;
      const double* V = a.fr.fv + f0;
      double x[3], v[3], imp[3];
      for (int d = 0; d < 3; ++d) {
        x[d] = X[3 * i + d];
        v[d] = V[3 * i + d];
      }
      // forward_impulse<double> (kernels.hpp:268-281)
      for (int d = 0; d < 3; ++d) imp[d] = R::add(a.net.b[d], R::mul(v[d], a.net.wv));
      for (int c = 0; c < kChannels; ++c) {
        if (!valid_channel(ix, iy, a.fr.nx, a.fr.ny, c)) continue;
        const int64_t j = nb(i, a.fr.nx, c);
        const double g = a.net.gain[c];
        for (int d = 0; d < 3; ++d) {
          const double phi = R::mul(R::sub(x[d], X[3 * j + d]), g);
          const double xi = R::mul(R::sub(v[d], V[3 * j + d]), g);
          const double s =
              R::div(phi, R::sqrt(R::add(1.0, R::mul(R::mul(a.net.alpha, phi), phi))));
          const double tt = R::add(R::add(R::mul(phi, a.net.wl[c]), R::mul(s, a.net.wn[c])),
                                   R::mul(R::mul(xi, s), a.net.wd[c]));
          imp[d] = R::add(imp[d], tt);
        }
      }
      if (!(isfinite(imp[0]) && isfinite(imp[1]) && isfinite(imp[2])))
        atomicMin(a.bad_fwd + b, static_cast<int>(i));
      // plug_impulse on a zero field (sim.cpp:100-106), added: applied = impulse + plug
      double plug[3] = {0.0, 0.0, 0.0};
      if (cc.plug_pressure) {
        const bool interior = ix >= 1 && ix <= a.fr.nx - 2 && iy >= 1 && iy <= a.fr.ny - 2;
        double e[3] = {0, 0, 0}, nn[3] = {0, 0, 0}, w[3] = {0, 0, 0}, s[3] = {0, 0, 0};
        if (interior)
          for (int d = 0; d < 3; ++d) {
            e[d] = R::sub(x[d], X[3 * (i + 1) + d]);
            nn[d] = R::sub(x[d], X[3 * (i + a.fr.nx) + d]);
            w[d] = R::sub(x[d], X[3 * (i - 1) + d]);
            s[d] = R::sub(x[d], X[3 * (i - a.fr.nx) + d]);
          }
        pressure_plug(cc, interior, e, nn, w, s, plug);
      }
      plug_tail(cc, v, plug);
      double applied[3];
      for (int d = 0; d < 3; ++d) applied[d] = R::add(imp[d], plug[d]);
      // advance_with_impulse at t_next = (k + 1) * dt with the constrained mask
      StepArgs<double> sa = a.sa;
      sa.k = k;
      double xo[3], vo[3];
      uint8_t mask;
      advance_node(sa, cc, iy, i, x, v, applied, xo, vo, mask);
      // residuals (train.cpp:166-177)
      const int64_t o = (static_cast<int64_t>(b) * a.fr.n + i) * 3;
      const int64_t on = o / 3;
      double rp[3] = {0.0, 0.0, 0.0}, rd[3] = {0.0, 0.0, 0.0};
      double pt = 0.0, dtm = 0.0;
      if (!pinned_node(cc, a.sa.pin_bits, i)) {
        for (int d = 0; d < 3; ++d) rp[d] = R::sub(imp[d], R::mul(a.force_dt[o + d], a.inv_mass));
        pt = dot3(rp, rp);
        if (!mask) {
          const double* Xn = X + a.fr.n * 3;
          const double* Vn = V + a.fr.n * 3;
          double rv[3], rx[3];
          for (int d = 0; d < 3; ++d) {
            rv[d] = R::sub(vo[d], Vn[3 * i + d]);
            rx[d] = R::sub(xo[d], Xn[3 * i + d]);
          }
          dtm = R::add(dot3(rv, rv), dot3(rx, rx));
          counted = 1;
          for (int d = 0; d < 3; ++d) rd[d] = R::add(rv[d], R::mul(rx[d], cc.dt));
        }
      }
      if (a.rp) {
        for (int d = 0; d < 3; ++d) {
          a.rp[o + d] = rp[d];
          a.rd[o + d] = rd[d];
        }
      }
      a.phys_term[on] = pt;
      a.data_term[on] = dtm;
    }
    const int cnt = __syncthreads_count(counted);
    if (threadIdx.x == 0 && cnt) atomicAdd(a.data_count, static_cast<unsigned long long>(cnt));
  }
}

// The loss sums as the reference's sequential chain (train.cpp:168-182): phys_sq and data_sq are
// two independent chains over (batch element, node), so lane 0 of warp 0 runs the first and
// lane 0 of warp 1 the second while the whole block stages the next tile in shared memory
// (the chain is bound by the dependent-add latency, never by a load). Each records the first
// batch element after which its running sum is non-finite; the reference stops at the smaller.
constexpr int kChainTile = 1024;

__global__ void __launch_bounds__(256) loss_chain_kernel(const double* __restrict__ pt,
                                                         const double* __restrict__ dt,
                                                         int batch, int64_t n, double* out,
                                                         int32_t* bad_b, double ps0, double ds0) {
  __shared__ double buf[2][2][kChainTile];
  __shared__ int bad_s[2];
  const int64_t total = static_cast<int64_t>(batch) * n;
  const int64_t tiles = (total + kChainTile - 1) / kChainTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // warps 2..7 stage tiles (all loads of a tile in flight at once); the two consumer warps
  // never wait on a global load
  constexpr int kLoaders = 192, kPer = (kChainTile + kLoaders - 1) / kLoaders;
  auto load = [&](int64_t t) {
    if (threadIdx.x < 64) return;
    const int64_t g0 = t * kChainTile;
    const int l = threadIdx.x - 64;
    double a[kPer], c[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int j = l + u * kLoaders;
      const int64_t g = g0 + j;
      const bool ok = j < kChainTile && g < total;
      a[u] = ok ? __ldg(pt + g) : 0.0;
      c[u] = ok ? __ldg(dt + g) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int j = l + u * kLoaders;
      if (j < kChainTile) {
        buf[t & 1][0][j] = a[u];
        buf[t & 1][1][j] = c[u];
      }
    }
  };
  load(0);
  __syncthreads();
  const bool consumer = warp < 2 && lane == 0;
  double acc = warp == 0 ? ps0 : ds0;  // a rank continues the chain where the previous one ended
  int bad = kNone;
  int b = 0;
  int64_t boundary = n;  // global index one past batch element b
  for (int64_t t = 0; t < tiles; ++t) {
    if (t + 1 < tiles) load(t + 1);
    if (consumer && bad == kNone) {
      const double* src = buf[t & 1][warp];
      const int64_t g0 = t * kChainTile;
      const int len = static_cast<int>(total - g0 < kChainTile ? total - g0 : kChainTile);
      int j = 0;
      while (j < len && bad == kNone) {
        const int seg = static_cast<int>(boundary - g0 < len ? boundary - g0 : len);
        // software-pipelined: the next eight values are loaded while the current eight are
        // added, so the chain runs at the dependent-add latency
        if (j + 8 <= seg) {
          double cur[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cur[u] = src[j + u];
          for (; j + 16 <= seg; j += 8) {
            double nxt[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) nxt[u] = src[j + 8 + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = R::add(acc, cur[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) acc = R::add(acc, cur[u]);
          j += 8;
        }
        for (; j < seg; ++j) acc = R::add(acc, src[j]);
        if (g0 + j == boundary) {
          if (!isfinite(acc)) bad = b;
          ++b;
          boundary += n;
        }
      }
    }
    __syncthreads();
  }
  if (consumer) {
    out[warp] = acc;
    bad_s[warp] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) *bad_b = bad_s[0] < bad_s[1] ? bad_s[0] : bad_s[1];
}

// backward_gradients per-node terms (net.cpp:159-196) into [b][chunk][term][kChunk].
struct BwdArgs {
  Frames fr;
  int b0, nb;  // batch elements [b0, b0 + nb) of this group
  NetConst<double> net;
  // upstream: either given (standalone backward_gradients) or rp*pc + rd*dc (compute_loss)
  const double* upstream;  // [n][3] for batch element 0, or nullptr
  const double* rp;
  const double* rd;
  double phys_coeff;
  double alpha_loss;  // the hybrid loss mix (data coefficient derived from data_count)
  const unsigned long long* data_count;
  double* terms;  // [nb][chunks][kTerms][kChunk]
  int chunks;
};

__global__ void __launch_bounds__(256) bwd_terms_kernel(const BwdArgs a) {
  double data_coeff = 0.0;
  if (!a.upstream) {
    const unsigned long long cnt = *a.data_count;
    // data_denom = 6 * data_count; data_coeff = 2 * (1 - alpha) / data_denom (train.cpp:187-197)
    if (cnt > 0)
      data_coeff = R::div(R::mul(2.0, R::sub(1.0, a.alpha_loss)),
                          R::mul(6.0, static_cast<double>(cnt)));
  }
  const int64_t total = a.fr.n * a.nb;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int bl = static_cast<int>(t / a.fr.n);
    const int b = a.b0 + bl;
    const int64_t i = t - static_cast<int64_t>(bl) * a.fr.n;
    const int ix = static_cast<int>(i % a.fr.nx), iy = static_cast<int>(i / a.fr.nx);
    const int64_t f0 = static_cast<int64_t>(a.fr.idx[b]) * a.fr.n * 3;
    const double* X = a.fr.fx + f0;
    const double* V = a.fr.fv + f0;
    double x[3], v[3], u[3];
    for (int d = 0; d < 3; ++d) {
      x[d] = X[3 * i + d];
      v[d] = V[3 * i + d];
    }
    if (a.upstream) {
      for (int d = 0; d < 3; ++d) u[d] = a.upstream[3 * i + d];
    } else {
      const int64_t o = (static_cast<int64_t>(b) * a.fr.n + i) * 3;
      for (int d = 0; d < 3; ++d)
        u[d] = R::add(R::mul(a.rp[o + d], a.phys_coeff), R::mul(a.rd[o + d], data_coeff));
    }
    const int chunk = static_cast<int>(i / kChunk);
    const int il = static_cast<int>(i - static_cast<int64_t>(chunk) * kChunk);
    double* T = a.terms + (static_cast<int64_t>(bl) * a.chunks + chunk) * kTerms * kChunk + il;
    auto put = [&](int row, double val) { T[static_cast<int64_t>(row) * kChunk] = val; };
    for (int d = 0; d < 3; ++d) put(kTermBias + d, u[d]);
    put(kTermSelf, dot3(u, v));
    const double alpha = a.net.alpha;
    for (int c = 0; c < kChannels; ++c) {
      if (!valid_channel(ix, iy, a.fr.nx, a.fr.ny, c)) {
        put(kTermKernel + c, 0.0);
        put(kTermLinear + c, 0.0);
        put(kTermNonlin + c, 0.0);
        put(kTermDeriv + c, 0.0);
        put(kTermAlpha + c, 0.0);
        continue;
      }
      const int64_t j = nb(i, a.fr.nx, c);
      const double g = a.net.gain[c];
      double dx[3], dv[3], phi[3], xi[3], s[3], sp[3], sa[3];
      for (int d = 0; d < 3; ++d) {
        dx[d] = R::sub(x[d], X[3 * j + d]);
        dv[d] = R::sub(v[d], V[3 * j + d]);
        phi[d] = R::mul(dx[d], g);
        xi[d] = R::mul(dv[d], g);
        const double z = phi[d];
        const double q = R::add(1.0, R::mul(R::mul(alpha, z), z));
        const double rq = R::div(1.0, R::sqrt(q));
        s[d] = R::mul(z, rq);
        sp[d] = R::div(rq, q);
        sa[d] = R::div(R::mul(R::mul(R::mul(R::mul(-0.5, z), z), z), rq), q);
      }
      double xs[3], kk[3], aa[3];
      for (int d = 0; d < 3; ++d) {
        xs[d] = R::mul(xi[d], s[d]);
        const double spdx = R::mul(sp[d], dx[d]);
        // dx*wL + (sp.dx)*wN + ((dv.s) + xi.(sp.dx))*wD
        kk[d] = R::add(R::add(R::mul(dx[d], a.net.wl[c]), R::mul(spdx, a.net.wn[c])),
                       R::mul(R::add(R::mul(dv[d], s[d]), R::mul(xi[d], spdx)), a.net.wd[c]));
        // sa*wN + (xi.sa)*wD
        aa[d] = R::add(R::mul(sa[d], a.net.wn[c]), R::mul(R::mul(xi[d], sa[d]), a.net.wd[c]));
      }
      put(kTermLinear + c, dot3(u, phi));
      put(kTermNonlin + c, dot3(u, s));
      put(kTermDeriv + c, dot3(u, xs));
      put(kTermKernel + c, dot3(u, kk));
      put(kTermAlpha + c, dot3(u, aa));
    }
  }
}

// One sequential chain per scalar over a chunk's nodes (alpha: over (node, channel)); output
// in for_each_gradient order (kernel, linear, bias, nonlinear, deriv, self_velocity, alpha).
// The block stages 32-node tiles of all 64 term rows in shared memory (double buffered) so the
// 53 chains run at dependent-add latency.
constexpr int kRedTile = 32;

__global__ void __launch_bounds__(256) bwd_reduce_kernel(const double* __restrict__ terms,
                                                         int64_t n, int chunks,
                                                         double* __restrict__ partial) {
  __shared__ double tile[2][kTerms][kRedTile];
  const int bc = blockIdx.x;  // (batch element in group) * chunks + chunk
  const int chunk = bc % chunks;
  const int64_t rem = n - static_cast<int64_t>(chunk) * kChunk;
  const int len = rem < kChunk ? static_cast<int>(rem) : kChunk;
  const int ntiles = (len + kRedTile - 1) / kRedTile;
  const double* T = terms + static_cast<int64_t>(bc) * kTerms * kChunk;
  // warps 2.. stage tiles; the 53 chain threads (warps 0-1) never wait on a global load
  constexpr int kLoaders = 192, kPer = (kTerms * kRedTile + kLoaders - 1) / kLoaders;
  auto load = [&](int t) {
    if (threadIdx.x < 64) return;
    const int l = threadIdx.x - 64;
    double a[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = l + u * kLoaders;
      const int row = e / kRedTile, j = e - row * kRedTile;
      a[u] = e < kTerms * kRedTile
                 ? __ldg(T + static_cast<int64_t>(row) * kChunk + t * kRedTile + j)
                 : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = l + u * kLoaders;
      if (e < kTerms * kRedTile) tile[t & 1][e / kRedTile][e % kRedTile] = a[u];
    }
  };
  load(0);
  __syncthreads();
  const int r = threadIdx.x;
  double acc = 0.0;
  for (int t = 0; t < ntiles; ++t) {
    if (t + 1 < ntiles) load(t + 1);
    const int cnt = len - t * kRedTile < kRedTile ? len - t * kRedTile : kRedTile;
    if (r < kTermAlpha) {
      const double* row = tile[t & 1][r];
#pragma unroll 8
      for (int i = 0; i < cnt; ++i) acc = R::add(acc, row[i]);
    } else if (r == kTermAlpha) {
      int i = 0;
      for (; i + 2 <= cnt; i += 2) {  // both nodes' 24 terms loaded ahead of the chain
        double v[2 * kChannels];
#pragma unroll
        for (int c = 0; c < kChannels; ++c) {
          v[c] = tile[t & 1][kTermAlpha + c][i];
          v[kChannels + c] = tile[t & 1][kTermAlpha + c][i + 1];
        }
#pragma unroll
        for (int q = 0; q < 2 * kChannels; ++q) acc = R::add(acc, v[q]);
      }
      for (; i < cnt; ++i) {
#pragma unroll
        for (int c = 0; c < kChannels; ++c) acc = R::add(acc, tile[t & 1][kTermAlpha + c][i]);
      }
    }
    __syncthreads();
  }
  if (r <= kTermAlpha) partial[static_cast<int64_t>(bc) * kScalars + r] = acc;
}

// total.add_scaled(partial, 1.0) over chunks (net.cpp:198-199), then grads.add_scaled(g, 1.0)
// over batch elements (train.cpp:205); `grads` carries the running sum across groups.
__global__ void bwd_final_kernel(const double* __restrict__ partial, int nb, int chunks,
                                 double* __restrict__ grads, double* __restrict__ per_b) {
  const int s = threadIdx.x;
  if (s >= kScalars) return;
  double g = grads[s];
  double tot = 0.0;
  const int64_t total = static_cast<int64_t>(nb) * chunks;
  int c = 0;
  for (int64_t k0 = 0; k0 < total; k0 += 8) {  // eight partials loaded ahead of the chain
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = k0 + u < total ? __ldg(partial + (k0 + u) * kScalars + s) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (k0 + u >= total) break;
      tot = R::add(tot, R::mul(v[u], 1.0));
      if (++c == chunks) {
        if (per_b) per_b[((k0 + u) / chunks) * kScalars + s] = tot;  // this element's total
        g = R::add(g, R::mul(tot, 1.0));
        tot = 0.0;
        c = 0;
      }
    }
  }
  grads[s] = g;
}

int grid_for(int64_t total, int threads = 256) {
  const int64_t blocks = (total + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, 148 * 16)));
}

// ----------------------------------------------------------------------------- host ----

// cloth::Rng (rng.hpp:13-47): std::mt19937_64 with fixed-algorithm draws.
struct Rng {
  std::mt19937_64 gen;
  explicit Rng(uint64_t seed) : gen(seed) {}
  uint64_t uniform_below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t r;
    do {
      r = gen();
    } while (r >= limit);
    return r % n;
  }
  double uniform01() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  static uint64_t mix(uint64_t seed, uint64_t stream) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
};

// the 53 scalars in for_each_scalar order + the 7 group flags (net.hpp:35-81)
struct Params {
  std::array<double, kScalars> s{};
  std::array<bool, 7> trainable{};
  std::array<double, 14> brackets{};  // InitBracket lo, hi per group (net.hpp:28-31)
  Params() {
    for (int g = 0; g < 7; ++g) {
      brackets[2 * g] = -1.0;
      brackets[2 * g + 1] = 1.0;
    }
    for (int c = 0; c < 12; ++c) s[c] = 1.0;  // kernel gains
    s[52] = 1.0;                              // alpha
    trainable.fill(true);
    trainable[0] = false;  // kernel
    trainable[6] = false;  // alpha
  }
};
int group_of(int idx) {  // ParamGroup of a flat scalar index
  if (idx < 12) return 0;
  if (idx < 24) return 1;
  if (idx < 27) return 2;
  if (idx < 39) return 3;
  if (idx < 51) return 4;
  return idx == 51 ? 5 : 6;
}
sc_params to_c(const Params& p) {
  sc_params c{};
  for (int i = 0; i < 12; ++i) {
    c.kernel_gain[i] = p.s[i];
    c.linear_w[i] = p.s[12 + i];
    c.nonlinear_w[i] = p.s[27 + i];
    c.deriv_w[i] = p.s[39 + i];
  }
  for (int d = 0; d < 3; ++d) c.linear_b[d] = p.s[24 + d];
  c.self_velocity_w = p.s[51];
  c.isru_alpha = p.s[52];
  return c;
}
Params from_c(const sc_params& c) {
  Params p;
  for (int i = 0; i < 12; ++i) {
    p.s[i] = c.kernel_gain[i];
    p.s[12 + i] = c.linear_w[i];
    p.s[27 + i] = c.nonlinear_w[i];
    p.s[39 + i] = c.deriv_w[i];
  }
  for (int d = 0; d < 3; ++d) p.s[24 + d] = c.linear_b[d];
  p.s[51] = c.self_velocity_w;
  p.s[52] = c.isru_alpha;
  return p;
}
NetConst<double> net_of(const sc_params& p) {
  NetConst<double> k{};
  for (int c = 0; c < kChannels; ++c) {
    k.gain[c] = p.kernel_gain[c];
    k.wl[c] = p.linear_w[c];
    k.wn[c] = p.nonlinear_w[c];
    k.wd[c] = p.deriv_w[c];
  }
  for (int d = 0; d < 3; ++d) k.b[d] = p.linear_b[d];
  k.wv = p.self_velocity_w;
  k.alpha = p.isru_alpha;
  return k;
}

struct Batch {
  std::vector<int32_t> idx;
  DBuf<int32_t> idx_d;
  DBuf<double> force_dt;
};

}  // namespace

struct sc_trainer {
  sc_ctx* ctx = nullptr;  // f64 context holding the scene constants
  SceneView view{};
  int device = 0, nx = 0, ny = 0, frames = 0;
  int64_t n = 0;
  int plug_p = 0, plug_g = 0, plug_d = 0;
  int n_pins = 0;
  double dt = 0.0, mass = 1.0;
  cudaStream_t s0 = nullptr;
  DBuf<double> fx, fv;
  Batch batch;  // the batch set through the C-ABI
  // compute_loss scratch
  DBuf<double> rp, rd, terms, partial, grads;
  DBuf<unsigned long long> count;
  DBuf<int32_t> bad_fwd, bad_spring;
  size_t term_budget = size_t(1) << 31;  // bytes of backward scratch per group
  // loss-chain slots: per-node loss terms + the chain's result. Slot 0 serves synchronous
  // compute_loss calls; train_loop rotates through all of them so the chains of successive
  // epochs run concurrently (they only feed the history rows and the error check).
  struct ChainSlot {
    DBuf<double> pt, dtm, out;
    DBuf<int32_t> bad;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_in = nullptr, ev_done = nullptr;
    double* host = nullptr;  // pinned: {phys_sq, data_sq, first bad element (as double)}
  };
  std::deque<ChainSlot> slots;  // stable addresses as slots are added
  // a part [part_b0, part_b0 + part_nb) of the current batch (sc_trainer_part_*): one rank's
  // share of a data-parallel compute_loss
  int part_b0 = 0, part_nb = 0;
  double* slot_host = nullptr;
  ~sc_trainer() {
    for (ChainSlot& c : slots) {
      if (c.st) cudaStreamSynchronize(c.st);
      if (c.ev_in) cudaEventDestroy(c.ev_in);
      if (c.ev_done) cudaEventDestroy(c.ev_done);
      if (c.st) cudaStreamDestroy(c.st);
    }
    if (slot_host) cudaFreeHost(slot_host);
  }
};

namespace {

// sample_batch (train.cpp:91-127)
void sample_batch(sc_trainer* t, int batch_size, Rng& rng, Batch& out) {
  const int transitions = t->frames - 1;
  if (transitions < 1) fail(SC_ERR_CONFIG, "trajectory has no transitions to sample");
  if (batch_size < 1 || batch_size > transitions)
    fail(SC_ERR_CONFIG, "batch size " + std::to_string(batch_size) + " not in [1, " +
                            std::to_string(transitions) + "]");
  std::vector<int> pool(static_cast<size_t>(transitions));
  for (int i = 0; i < transitions; ++i) pool[static_cast<size_t>(i)] = i;
  out.idx.clear();
  for (int k = 0; k < batch_size; ++k) {
    const int j = k + static_cast<int>(rng.uniform_below(static_cast<uint64_t>(transitions - k)));
    std::swap(pool[static_cast<size_t>(k)], pool[static_cast<size_t>(j)]);
    out.idx.push_back(pool[static_cast<size_t>(k)]);
  }
}

// targets of a batch whose indices are set (device); NumericsError on a singular spring
void batch_targets(sc_trainer* t, Batch& bt) {
  const int B = static_cast<int>(bt.idx.size());
  bt.idx_d.ensure(B);
  ck(cudaMemcpyAsync(bt.idx_d.p, bt.idx.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice,
                     t->s0),
     "H2D indices");
  bt.force_dt.ensure(static_cast<size_t>(B) * t->n * 3);
  t->bad_spring.ensure(B);
  ck(cudaMemsetAsync(t->bad_spring.p, 0x7F, sizeof(int32_t) * B, t->s0), "memset");
  TargetArgs a{};
  a.fr = Frames{t->fx.p, t->fv.p, bt.idx_d.p, t->nx, t->ny, t->n};
  a.batch = B;
  a.cloth = static_cast<const ClothConst<double>*>(t->view.cloths);
  a.plug_pressure = t->plug_p;
  a.plug_gravity = t->plug_g;
  a.plug_drag = t->plug_d;
  a.force_dt = bt.force_dt.p;
  a.bad_spring = t->bad_spring.p;
  targets_kernel<<<grid_for(t->n * B), 256, 0, t->s0>>>(a);
  ck(cudaGetLastError(), "targets_kernel");
  std::vector<int32_t> bad(static_cast<size_t>(B));
  ck(cudaMemcpyAsync(bad.data(), t->bad_spring.p, sizeof(int32_t) * B, cudaMemcpyDeviceToHost,
                     t->s0),
     "D2H");
  ck(cudaStreamSynchronize(t->s0), "targets");
  for (int b = 0; b < B; ++b)
    if (bad[static_cast<size_t>(b)] != kNone)
      fail(SC_ERR_NUMERICS, "elastic force: singular spring (coincident nodes) at node " +
                                std::to_string(bad[static_cast<size_t>(b)]));
}

// diagnose_forward (net.cpp:30-51) for the error text, on the host from frame k
std::string diagnose_forward(sc_trainer* t, int k, int node, const sc_params& p) {
  std::vector<double> x(static_cast<size_t>(t->n) * 3), v(x.size());
  ck(cudaMemcpy(x.data(), t->fx.p + static_cast<int64_t>(k) * t->n * 3, sizeof(double) * x.size(),
                cudaMemcpyDeviceToHost),
     "D2H frame");
  ck(cudaMemcpy(v.data(), t->fv.p + static_cast<int64_t>(k) * t->n * 3, sizeof(double) * v.size(),
                cudaMemcpyDeviceToHost),
     "D2H frame");
  const int ix = node % t->nx, iy = node / t->nx;
  double lin[3], non[3] = {0, 0, 0}, der[3];
  for (int d = 0; d < 3; ++d) {
    lin[d] = p.linear_b[d];
    der[d] = v[3 * node + d] * p.self_velocity_w;
  }
  for (int c = 0; c < kChannels; ++c) {
    const int jx = ix + off_dx(c), jy = iy + off_dy(c);
    if (jx < 0 || jx >= t->nx || jy < 0 || jy >= t->ny) continue;
    const int j = jy * t->nx + jx;
    for (int d = 0; d < 3; ++d) {
      const double phi = (x[3 * node + d] - x[3 * j + d]) * p.kernel_gain[c];
      const double xi = (v[3 * node + d] - v[3 * j + d]) * p.kernel_gain[c];
      const double s = phi / std::sqrt(1.0 + p.isru_alpha * phi * phi);
      lin[d] += phi * p.linear_w[c];
      non[d] += s * p.nonlinear_w[c];
      der[d] += xi * s * p.deriv_w[c];
    }
  }
  auto fin = [](const double* q) {
    return std::isfinite(q[0]) && std::isfinite(q[1]) && std::isfinite(q[2]);
  };
  const char* branch = !fin(lin) ? "linear" : (!fin(non) ? "nonlinear" : "derivative");
  return "network impulse non-finite at node " + std::to_string(node) + " (" + branch +
         " branch)";
}

struct Loss {
  double total = 0.0, physics = 0.0, data = 0.0;
};

constexpr size_t kMaxSlots = 32;

sc_trainer::ChainSlot& chain_slot(sc_trainer* t, size_t k) {
  while (t->slots.size() <= k) {
    t->slots.emplace_back();
    sc_trainer::ChainSlot& c = t->slots.back();
    ck(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&c.ev_in, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c.ev_done, cudaEventDisableTiming), "event");
    if (!t->slot_host)  // one pinned block for every slot's result (cudaHostAlloc is slow)
      ck(cudaHostAlloc(reinterpret_cast<void**>(&t->slot_host), kMaxSlots * 4 * sizeof(double),
                       cudaHostAllocDefault),
         "cudaHostAlloc");
    c.host = t->slot_host + 4 * (t->slots.size() - 1);
  }
  return t->slots[k];
}

// What the host needs to finish a launched compute_loss.
struct LossLaunch {
  int B = 0;
  unsigned long long cnt = 0;
  int first_bad_fwd = kNone;  // first batch element with a non-finite cell impulse
  int bad_node = 0;
  int free_count = 0;
  double phys_denom = 0.0;
};

// compute_loss (train.cpp:129-209), device part: the forward pass, the loss chain (async on the
// slot's stream) and, when `grads` is given, the 53 gradient sums (returned synchronously).
LossLaunch launch_loss(sc_trainer* t, const sc_params& params, Batch& bt, double alpha,
                       double* grads, sc_trainer::ChainSlot& slot) {
  LossLaunch L;
  const int B = L.B = static_cast<int>(bt.idx.size());
  if (B == 0) fail(SC_ERR_CONFIG, "compute_loss: empty batch");
  if (!(params.isru_alpha > 0.0)) fail(SC_ERR_CONFIG, "isru_alpha: must be > 0");
  const int64_t n = t->n;
  const size_t bn = static_cast<size_t>(B) * n;
  // the slot's previous chain must be done with its buffers
  ck(cudaStreamWaitEvent(t->s0, slot.ev_done, 0), "wait");
  slot.pt.ensure(bn);
  slot.dtm.ensure(bn);
  slot.out.ensure(2);
  slot.bad.ensure(1);
  if (grads) {
    t->rp.ensure(bn * 3);
    t->rd.ensure(bn * 3);
  }
  t->count.ensure(1);
  t->bad_fwd.ensure(B);
  ck(cudaMemsetAsync(t->count.p, 0, sizeof(unsigned long long), t->s0), "memset");
  ck(cudaMemsetAsync(t->bad_fwd.p, 0x7F, sizeof(int32_t) * B, t->s0), "memset");

  const Frames fr{t->fx.p, t->fv.p, bt.idx_d.p, t->nx, t->ny, n};
  const NetConst<double> net = net_of(params);
  LossArgs la{};
  la.fr = fr;
  la.batch = B;
  la.force_dt = bt.force_dt.p;
  la.inv_mass = 1.0 / t->mass;
  la.net = net;
  la.sa.spheres = static_cast<const SphereConst<double>*>(t->view.spheres);
  la.sa.planes = static_cast<const PlaneConst<double>*>(t->view.planes);
  la.sa.pin_bits = t->view.pin_bits;
  la.sa.pin_rank = t->view.pin_rank;
  la.sa.pin_anchors = static_cast<const double*>(t->view.anchors);
  la.sa.use_t_override = 0;
  la.cloth = static_cast<const ClothConst<double>*>(t->view.cloths);
  la.rp = grads ? t->rp.p : nullptr;
  la.rd = grads ? t->rd.p : nullptr;
  la.phys_term = slot.pt.p;
  la.data_term = slot.dtm.p;
  la.data_count = t->count.p;
  la.bad_fwd = t->bad_fwd.p;
  loss_fwd_kernel<<<grid_for(static_cast<int64_t>(bn)), 256, 0, t->s0>>>(la);
  ck(cudaGetLastError(), "loss_fwd_kernel");
  ck(cudaEventRecord(slot.ev_in, t->s0), "event");
  ck(cudaStreamWaitEvent(slot.st, slot.ev_in, 0), "wait");
  loss_chain_kernel<<<1, 256, 0, slot.st>>>(slot.pt.p, slot.dtm.p, B, n, slot.out.p, slot.bad.p,
                                            0.0, 0.0);
  ck(cudaGetLastError(), "loss_chain_kernel");
  ck(cudaMemcpyAsync(slot.host, slot.out.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, slot.st),
     "D2H chain");
  ck(cudaMemcpyAsync(slot.host + 3, slot.bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, slot.st),
     "D2H chain");
  ck(cudaEventRecord(slot.ev_done, slot.st), "event");

  L.free_count = static_cast<int>(n) - t->n_pins;
  L.phys_denom = 3.0 * static_cast<double>(B) * L.free_count;
  if (grads) {
    t->grads.ensure(kScalars);
    ck(cudaMemsetAsync(t->grads.p, 0, sizeof(double) * kScalars, t->s0), "memset");
    const int chunks = static_cast<int>((n + kChunk - 1) / kChunk);
    const size_t per_elem = static_cast<size_t>(chunks) * kTerms * kChunk * sizeof(double);
    const int group = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(static_cast<size_t>(B), t->term_budget / per_elem)));
    t->terms.ensure(static_cast<size_t>(group) * chunks * kTerms * kChunk);
    t->partial.ensure(static_cast<size_t>(group) * chunks * kScalars);
    for (int b0 = 0; b0 < B; b0 += group) {
      const int nbat = std::min(group, B - b0);
      BwdArgs ba{};
      ba.fr = fr;
      ba.b0 = b0;
      ba.nb = nbat;
      ba.net = net;
      ba.upstream = nullptr;
      ba.rp = t->rp.p;
      ba.rd = t->rd.p;
      ba.phys_coeff = L.free_count > 0 ? 2.0 * alpha / L.phys_denom : 0.0;
      ba.alpha_loss = alpha;
      ba.data_count = t->count.p;
      ba.terms = t->terms.p;
      ba.chunks = chunks;
      bwd_terms_kernel<<<grid_for(n * nbat), 256, 0, t->s0>>>(ba);
      ck(cudaGetLastError(), "bwd_terms_kernel");
      bwd_reduce_kernel<<<nbat * chunks, 256, 0, t->s0>>>(t->terms.p, n, chunks, t->partial.p);
      ck(cudaGetLastError(), "bwd_reduce_kernel");
      bwd_final_kernel<<<1, 64, 0, t->s0>>>(t->partial.p, nbat, chunks, t->grads.p, nullptr);
      ck(cudaGetLastError(), "bwd_final_kernel");
    }
  }
  std::vector<int32_t> bad_fwd(static_cast<size_t>(B));
  ck(cudaMemcpyAsync(&L.cnt, t->count.p, sizeof L.cnt, cudaMemcpyDeviceToHost, t->s0), "D2H");
  ck(cudaMemcpyAsync(bad_fwd.data(), t->bad_fwd.p, sizeof(int32_t) * B, cudaMemcpyDeviceToHost,
                     t->s0),
     "D2H");
  if (grads)
    ck(cudaMemcpyAsync(grads, t->grads.p, sizeof(double) * kScalars, cudaMemcpyDeviceToHost,
                       t->s0),
       "D2H");
  ck(cudaStreamSynchronize(t->s0), "compute_loss");
  for (int b = 0; b < B; ++b)
    if (bad_fwd[static_cast<size_t>(b)] != kNone) {
      L.first_bad_fwd = b;
      L.bad_node = bad_fwd[static_cast<size_t>(b)];
      break;
    }
  return L;
}

// compute_loss, host part: waits for the slot's chain, applies the reference's error order
// (element b's forward_impulse throws before b's loss check, train.cpp:146-182) and forms the
// loss values (train.cpp:185-189).
Loss finish_loss(sc_trainer* t, const sc_params& params, const std::vector<int32_t>& idx,
                 double alpha, const LossLaunch& L, sc_trainer::ChainSlot& slot) {
  ck(cudaEventSynchronize(slot.ev_done), "loss chain");
  const double ps = slot.host[0], ds = slot.host[1];
  int32_t bad_b;
  std::memcpy(&bad_b, slot.host + 3, sizeof bad_b);
  if (L.first_bad_fwd != kNone && L.first_bad_fwd <= bad_b)
    fail(SC_ERR_NUMERICS, diagnose_forward(t, idx[static_cast<size_t>(L.first_bad_fwd)],
                                           L.bad_node, params));
  if (bad_b != kNone)
    fail(SC_ERR_NUMERICS, "non-finite loss at batch element " + std::to_string(bad_b) +
                              " (frame " + std::to_string(idx[static_cast<size_t>(bad_b)]) + ")");
  Loss loss;
  const double data_denom = 6.0 * static_cast<double>(L.cnt);
  loss.physics = L.free_count > 0 ? ps / L.phys_denom : 0.0;
  loss.data = L.cnt > 0 ? ds / data_denom : 0.0;
  loss.total = alpha * loss.physics + (1.0 - alpha) * loss.data;
  return loss;
}

Loss compute_loss(sc_trainer* t, const sc_params& params, Batch& bt, double alpha,
                  double* grads) {
  sc_trainer::ChainSlot& slot = chain_slot(t, 0);
  const LossLaunch L = launch_loss(t, params, bt, alpha, grads, slot);
  return finish_loss(t, params, bt.idx, alpha, L, slot);
}

// ---- optimizer / schedule / DE / loop (train.cpp:54-63, 212-375) ----------------------------

// What has to equal the reference here is behaviour, not text: the order of the random draws
// (every draw comes from the caller's mt19937_64 stream), the rounding order of each floating-
// point expression, the order in which configuration errors are reported and their messages.
// The code below is organised around this trainer's flat 53-scalar parameter vector.

// RNG substream tags of the pre-search and of its probe batch: part of the seeded behaviour
// (train.cpp:18-19), they must be these values for a run to reproduce the reference's.
constexpr uint64_t kTagSearch = 0xde5ea4c400000001ULL;
constexpr uint64_t kTagProbe = 0xde5ea4c400000002ULL;
constexpr double kPi = 3.141592653589793238462643383279502884;

// Learning rate of optimiser step `step` (train.cpp:54-60): step decay by completed intervals,
// or a half-cosine from lr0 down to the floor over `period` steps.
double schedule_lr(const sc_train_config& cfg, int step) {
  if (cfg.schedule_kind == 0) {
    const int decays = step / cfg.interval;
    return cfg.lr0 * std::pow(cfg.gamma, decays);
  }
  if (step >= cfg.period) return cfg.floor;
  const double span = cfg.lr0 - cfg.floor;
  const double phase = kPi * step / cfg.period;
  return cfg.floor + span * 0.5 * (1.0 + std::cos(phase));
}

// TrainConfig::validate (train.cpp:62-...): the first violated rule, in the reference's order,
// with the reference's field names in the message.
void validate_config(const sc_train_config& c, int transitions) {
  auto unit = [](double v) { return v >= 0.0 && v <= 1.0; };
  const std::pair<bool, std::string> rules[] = {
      {unit(c.alpha), "train.alpha: must be in [0, 1]"},
      {c.batch_size >= 1, "train.batch_size: must be >= 1"},
      {c.batch_size <= transitions, "train.batch_size: exceeds the " +
                                        std::to_string(transitions) + " available transitions"},
      {c.epochs >= 1, "train.epochs: must be >= 1"},
      {c.lr0 > 0.0, "train.lr0: must be > 0"},
      {c.gamma > 0.0 && c.gamma <= 1.0, "train.gamma: must be in (0, 1]"},
      {c.interval >= 1, "train.interval: must be >= 1"},
      {c.period >= 1, "train.period: must be >= 1"},
      {c.floor >= 0.0, "train.floor: must be >= 0"},
      {c.de_population >= 4, "train.de.population: must be >= 4"},
      {c.de_generations >= 0, "train.de.generations: must be >= 0"},
      {c.de_bound > 0.0, "train.de.bound: must be > 0"},
      {unit(c.de_cross_prob), "train.de.cross_prob: must be in [0, 1]"},
      {c.de_diff_weight > 0.0 && c.de_diff_weight <= 2.0,
       "train.de.diff_weight: must be in (0, 2]"},
      {c.de_probe_batch >= 1, "train.de.probe_batch: must be >= 1"},
      {c.checkpoint_interval >= 1, "train.checkpoint_interval: must be >= 1"},
  };
  for (const auto& [ok, text] : rules)  // NaN fields fail their comparison, as in the reference
    if (!ok) fail(SC_ERR_CONFIG, text);
}

// Adam (train.cpp:322-340) on the trainable scalars: moments first, then the bias-corrected
// steps; every scalar's arithmetic is independent of the others, each expression keeps the
// reference's association (decay * m + (1 - decay) * g, ((1 - decay) * g) * g,
// (lr * m_hat) / (sqrt(v_hat) + eps)).
void adam_update(Params& p, const double* grads, sc_adam_state& opt, double lr) {
  constexpr double kDecayM = 0.9, kDecayV = 0.999, kEps = 1e-8;
  const double t = static_cast<double>(++opt.step);
  const double unbias_m = 1.0 - std::pow(kDecayM, t);
  const double unbias_v = 1.0 - std::pow(kDecayV, t);
  auto live = [&](int s) { return p.trainable[static_cast<size_t>(group_of(s))]; };
  for (int s = 0; s < kScalars; ++s)
    if (live(s)) {
      const double g = grads[s];
      opt.m[s] = kDecayM * opt.m[s] + (1.0 - kDecayM) * g;
      opt.v[s] = kDecayV * opt.v[s] + (1.0 - kDecayV) * g * g;
    }
  for (int s = 0; s < kScalars; ++s)
    if (live(s)) {
      const double m_hat = opt.m[s] / unbias_m, v_hat = opt.v[s] / unbias_v;
      p.s[static_cast<size_t>(s)] -= lr * m_hat / (std::sqrt(v_hat) + kEps);
    }
}

// The pre-search works on a 6-vector z, one axis per parameter group 1..6 (linear, bias,
// nonlinear, deriv, self velocity, alpha): the weight groups as sign and decade, sgn(z) *
// 10^(|z| - 2) (z = -0.0 counts as positive), alpha as 10^(z / 2) (train.cpp:33-45).
constexpr size_t kSearchDim = 6;
using GroupValues = std::array<double, kSearchDim>;
GroupValues decode_search_point(const double* z) {
  GroupValues out{};
  for (size_t g = 0; g + 1 < kSearchDim; ++g) {
    const double magnitude = std::pow(10.0, std::abs(z[g]) - 2.0);
    out[g] = z[g] >= 0.0 ? magnitude : -magnitude;
  }
  out[kSearchDim - 1] = std::pow(10.0, z[kSearchDim - 1] / 2.0);
  return out;
}
// every scalar of group g >= 1 set to that group's value (the kernel gains stay 1)
Params group_constant_params(const GroupValues& values) {
  Params p;
  for (int s = 0; s < kScalars; ++s)
    if (const int g = group_of(s); g >= 1) p.s[static_cast<size_t>(s)] = values[static_cast<size_t>(g - 1)];
  return p;
}

// DE/rand/1/bin in the box [-bound, bound]^dim from a given start population, minimising
// `cost` (train.cpp:212-266; the reference's random-initialisation branch is not needed: the
// caller seeds every member). Draw order per member and generation: three distinct partners
// other than the member itself, each by rejection from uniform_below(members); the coordinate
// that always crosses over; then one uniform01 per coordinate, drawn whether or not that
// coordinate is the forced one. A trial replaces its member when it is not worse; the result is
// the first member with the lowest cost.
class BoxSearch {
 public:
  BoxSearch(std::vector<double> start, size_t dim, double bound)
      : dim_(dim), members_(start.size() / dim), bound_(bound), x_(std::move(start)),
        cost_(members_) {
    for (double& v : x_) v = confine(v);
  }
  template <typename Cost>
  std::vector<double> run(Cost&& cost, int generations, double diff_weight, double cross_prob,
                          Rng& rng) {
    for (size_t m = 0; m < members_; ++m) cost_[m] = cost(row(m));
    std::vector<double> trial(dim_);
    for (int gen = 0; gen < generations; ++gen)
      for (size_t m = 0; m < members_; ++m) {
        const size_t a = partner(rng, {m});
        const size_t b = partner(rng, {m, a});
        const size_t c = partner(rng, {m, a, b});
        const size_t forced = rng.uniform_below(dim_);
        const double *xa = row(a), *xb = row(b), *xc = row(c), *xm = row(m);
        for (size_t d = 0; d < dim_; ++d) {
          const bool cross = rng.uniform01() < cross_prob;
          trial[d] = (cross || d == forced) ? confine(xa[d] + diff_weight * (xb[d] - xc[d]))
                                            : xm[d];
        }
        const double trial_cost = cost(trial.data());
        if (trial_cost <= cost_[m]) {
          std::copy(trial.begin(), trial.end(), row(m));
          cost_[m] = trial_cost;
        }
      }
    const size_t best = static_cast<size_t>(
        std::min_element(cost_.begin(), cost_.end()) - cost_.begin());  // first minimum
    return std::vector<double>(row(best), row(best) + dim_);
  }

 private:
  double* row(size_t m) { return x_.data() + m * dim_; }
  double confine(double v) const { return v < -bound_ ? -bound_ : (bound_ < v ? bound_ : v); }
  size_t partner(Rng& rng, std::initializer_list<size_t> taken) const {
    for (;;) {
      const size_t k = rng.uniform_below(members_);
      if (std::find(taken.begin(), taken.end(), k) == taken.end()) return k;
    }
  }
  size_t dim_, members_;
  double bound_;
  std::vector<double> x_, cost_;
};

// de_preprocess (train.cpp:268-320): the box search over group-constant parameter sets on a
// fixed probe batch, then per-group initialisation brackets around the best point and a uniform
// draw inside them for every trainable scalar.
Params de_preprocess(sc_trainer* t, const sc_train_config& cfg, Rng& rng) {
  Rng probe_rng(Rng::mix(cfg.seed, kTagProbe));
  Batch probe;
  sample_batch(t, std::min(cfg.de_probe_batch, t->frames - 1), probe_rng, probe);
  batch_targets(t, probe);
  auto probe_loss = [&](const double* z) {
    try {
      const sc_params p = to_c(group_constant_params(decode_search_point(z)));
      return compute_loss(t, p, probe, cfg.alpha, nullptr).total;
    } catch (const Fail& f) {  // a diverging candidate is just a bad candidate
      if (f.code != SC_ERR_NUMERICS) throw;
      return 1e300;
    }
  };
  // start population: every coordinate on the midpoints of a 6-cell lattice across the box,
  // one uniform_below(6) per coordinate, member by member
  const double bound = cfg.de_bound, cell = 2.0 * bound / 6.0;
  std::vector<double> start(static_cast<size_t>(cfg.de_population) * kSearchDim);
  for (double& v : start) {
    const double level = static_cast<double>(rng.uniform_below(6));
    v = -bound + (level + 0.5) * cell;
  }
  const std::vector<double> best_z =
      BoxSearch(std::move(start), kSearchDim, bound)
          .run(probe_loss, cfg.de_generations, cfg.de_diff_weight, cfg.de_cross_prob, rng);
  const GroupValues best = decode_search_point(best_z.data());

  Params params;
  params.brackets[0] = params.brackets[1] = 1.0;  // kernel gains: fixed at 1
  for (size_t g = 1; g <= kSearchDim; ++g) {      // value +- max(|value|, 0.05)
    const double centre = best[g - 1], half = std::max(std::abs(centre), 0.05);
    params.brackets[2 * g] = centre - half;
    params.brackets[2 * g + 1] = centre + half;
  }
  params.brackets[12] = std::max(params.brackets[12], 1e-3);  // alpha stays positive
  // frozen groups keep their searched (alpha) or default value; trainable scalars draw from
  // their group's bracket, in flat scalar order
  params.s[52] = best[kSearchDim - 1];
  for (int s = 0; s < kScalars; ++s) {
    const size_t g = static_cast<size_t>(group_of(s));
    if (params.trainable[g])
      params.s[static_cast<size_t>(s)] = rng.uniform(params.brackets[2 * g], params.brackets[2 * g + 1]);
  }
  return params;
}

}  // namespace

extern "C" {

sc_status sc_trainer_create(int device, const sc_scene_desc* scene, int32_t frames,
                            const double* frames_x, const double* frames_v, sc_trainer** out) {
  return guarded([&] {
    if (!out) fail(SC_ERR_CONFIG, "out: null");
    *out = nullptr;
    if (!scene || scene->batch != 1) fail(SC_ERR_CONFIG, "trainer: exactly one scene");
    if (frames < 1) fail(SC_ERR_CONFIG, "trajectory: needs at least one frame");
    if (!frames_x || !frames_v) fail(SC_ERR_CONFIG, "trajectory: null frame array");
    auto* t = new sc_trainer();
    auto cleanup = [&] { sc_trainer_destroy(t); };
    try {
      sc_status st = sc_ctx_create(device, SC_F64, &t->ctx);
      if (st != SC_OK) fail(st, sc_last_error());
      st = sc_ctx_set_scene(t->ctx, scene);
      if (st != SC_OK) fail(st, sc_last_error());
      if (!ctx_scene_view(t->ctx, &t->view)) fail(SC_ERR_STATE, "trainer: scene view");
      const sc_cloth_desc& c = scene->cloths[0];
      t->device = device;
      t->nx = scene->nx;
      t->ny = scene->ny;
      t->n = static_cast<int64_t>(scene->nx) * scene->ny;
      t->frames = frames;
      t->plug_p = c.plug_pressure ? 1 : 0;
      t->plug_g = c.plug_gravity ? 1 : 0;
      t->plug_d = c.plug_drag ? 1 : 0;
      t->n_pins = c.n_pins;
      t->dt = c.dt;
      t->mass = c.mass;
      const size_t elems = static_cast<size_t>(frames) * t->n * 3;
      for (size_t e = 0; e < elems; ++e)
        if (!std::isfinite(frames_x[e]) || !std::isfinite(frames_v[e]))
          fail(SC_ERR_CONFIG, "trajectory: frame " + std::to_string(e / (t->n * 3)) +
                                  " has non-finite components");
      ck(cudaSetDevice(device), "cudaSetDevice");
      ck(cudaStreamCreateWithFlags(&t->s0, cudaStreamNonBlocking), "stream");
      t->fx.ensure(elems);
      t->fv.ensure(elems);
      ck(cudaMemcpy(t->fx.p, frames_x, elems * sizeof(double), cudaMemcpyHostToDevice), "H2D");
      ck(cudaMemcpy(t->fv.p, frames_v, elems * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    } catch (...) {
      cleanup();
      throw;
    }
    *out = t;
  });
}

void sc_trainer_destroy(sc_trainer* t) {
  if (!t) return;
  if (t->ctx) cudaSetDevice(t->device);
  if (t->s0) cudaStreamSynchronize(t->s0);
  if (t->s0) cudaStreamDestroy(t->s0);
  if (t->ctx) sc_ctx_destroy(t->ctx);
  delete t;
}

sc_status sc_trainer_sample_batch(sc_trainer* t, int32_t batch_size, uint64_t rng_seed,
                                  int32_t* indices_out, double* force_dt_out) {
  return guarded([&] {
    if (!t) fail(SC_ERR_STATE, "null trainer");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    Rng rng(rng_seed);
    t->batch.idx.clear();
    sample_batch(t, batch_size, rng, t->batch);
    if (indices_out)
      std::memcpy(indices_out, t->batch.idx.data(), sizeof(int32_t) * t->batch.idx.size());
    batch_targets(t, t->batch);
    if (force_dt_out)
      ck(cudaMemcpy(force_dt_out, t->batch.force_dt.p,
                    sizeof(double) * t->batch.idx.size() * t->n * 3, cudaMemcpyDeviceToHost),
         "D2H targets");
  });
}

sc_status sc_sample_indices(int32_t frames, int32_t batch_size, uint64_t rng_seed,
                            int32_t* indices_out) {
  return guarded([&] {
    if (!indices_out) fail(SC_ERR_CONFIG, "indices: null");
    sc_trainer t;  // host-only use: frame count
    t.frames = frames;
    Rng rng(rng_seed);
    Batch b;
    sample_batch(&t, batch_size, rng, b);
    std::memcpy(indices_out, b.idx.data(), sizeof(int32_t) * b.idx.size());
  });
}

sc_status sc_trainer_set_batch(sc_trainer* t, const int32_t* indices, int32_t count) {
  return guarded([&] {
    if (!t) fail(SC_ERR_STATE, "null trainer");
    if (count < 1 || !indices) fail(SC_ERR_CONFIG, "compute_loss: empty batch");
    for (int b = 0; b < count; ++b)
      if (indices[b] < 0 || indices[b] >= t->frames - 1)
        fail(SC_ERR_CONFIG, "batch index " + std::to_string(indices[b]) + " not in [0, " +
                                std::to_string(t->frames - 2) + "]");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    t->batch.idx.assign(indices, indices + count);
    batch_targets(t, t->batch);
  });
}

sc_status sc_trainer_compute_loss(sc_trainer* t, const sc_params* params, double alpha,
                                  double* loss_out, double* grads_out) {
  return guarded([&] {
    if (!t) fail(SC_ERR_STATE, "null trainer");
    if (!params || !loss_out) fail(SC_ERR_CONFIG, "compute_loss: null argument");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    const Loss l = compute_loss(t, *params, t->batch, alpha, grads_out);
    loss_out[0] = l.total;
    loss_out[1] = l.physics;
    loss_out[2] = l.data;
  });
}

// ---- data-parallel compute_loss in parts (one per rank) ------------------------------------
// compute_loss over B transitions split into contiguous parts is exactly the single-device
// result when (i) the data count is summed over parts before the backward pass, (ii) the loss
// chain runs part after part, each starting from the previous part's running sums, and (iii)
// the per-transition gradient totals are summed in transition order (train.cpp:205). These
// entry points run one part; the caller (training.DistributedTrainer) does the exchanges.

sc_status sc_trainer_part_forward(sc_trainer* t, const sc_params* params, int32_t b0, int32_t b1,
                                  uint64_t* count_out, int32_t* bad_out) {
  return guarded([&] {
    if (!t) fail(SC_ERR_STATE, "null trainer");
    if (!params || !count_out || !bad_out) fail(SC_ERR_CONFIG, "part: null argument");
    const int B = static_cast<int>(t->batch.idx.size());
    if (B == 0) fail(SC_ERR_CONFIG, "compute_loss: empty batch");
    if (b0 < 0 || b1 > B || b0 >= b1) fail(SC_ERR_CONFIG, "part: bad transition range");
    if (!(params->isru_alpha > 0.0)) fail(SC_ERR_CONFIG, "isru_alpha: must be > 0");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    const int nb = b1 - b0;
    const int64_t n = t->n;
    const size_t bn = static_cast<size_t>(nb) * n;
    sc_trainer::ChainSlot& slot = chain_slot(t, 0);
    ck(cudaStreamSynchronize(slot.st), "chain");
    slot.pt.ensure(bn);
    slot.dtm.ensure(bn);
    slot.out.ensure(2);
    slot.bad.ensure(1);
    t->rp.ensure(bn * 3);
    t->rd.ensure(bn * 3);
    t->count.ensure(1);
    t->bad_fwd.ensure(nb);
    ck(cudaMemsetAsync(t->count.p, 0, sizeof(unsigned long long), t->s0), "memset");
    ck(cudaMemsetAsync(t->bad_fwd.p, 0x7F, sizeof(int32_t) * nb, t->s0), "memset");
    LossArgs la{};
    la.fr = Frames{t->fx.p, t->fv.p, t->batch.idx_d.p + b0, t->nx, t->ny, n};
    la.batch = nb;
    la.force_dt = t->batch.force_dt.p + static_cast<size_t>(b0) * n * 3;
    la.inv_mass = 1.0 / t->mass;
    la.net = net_of(*params);
    la.sa.spheres = static_cast<const SphereConst<double>*>(t->view.spheres);
    la.sa.planes = static_cast<const PlaneConst<double>*>(t->view.planes);
    la.sa.pin_bits = t->view.pin_bits;
    la.sa.pin_rank = t->view.pin_rank;
    la.sa.pin_anchors = static_cast<const double*>(t->view.anchors);
    la.cloth = static_cast<const ClothConst<double>*>(t->view.cloths);
    la.rp = t->rp.p;
    la.rd = t->rd.p;
    la.phys_term = slot.pt.p;
    la.data_term = slot.dtm.p;
    la.data_count = t->count.p;
    la.bad_fwd = t->bad_fwd.p;
    loss_fwd_kernel<<<grid_for(static_cast<int64_t>(bn)), 256, 0, t->s0>>>(la);
    ck(cudaGetLastError(), "loss_fwd_kernel");
    std::vector<int32_t> bad(static_cast<size_t>(nb));
    unsigned long long cnt = 0;
    ck(cudaMemcpyAsync(&cnt, t->count.p, sizeof cnt, cudaMemcpyDeviceToHost, t->s0), "D2H");
    ck(cudaMemcpyAsync(bad.data(), t->bad_fwd.p, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost,
                       t->s0),
       "D2H");
    ck(cudaStreamSynchronize(t->s0), "part forward");
    t->part_b0 = b0;
    t->part_nb = nb;
    *count_out = cnt;
    bad_out[0] = -1;  // first transition (global index) with a non-finite impulse, and its node
    bad_out[1] = -1;
    for (int b = 0; b < nb; ++b)
      if (bad[static_cast<size_t>(b)] != kNone) {
        bad_out[0] = b0 + b;
        bad_out[1] = bad[static_cast<size_t>(b)];
        break;
      }
  });
}

sc_status sc_trainer_part_chain(sc_trainer* t, const double* sums_in, double* sums_out,
                                int32_t* bad_out) {
  return guarded([&] {
    if (!t || t->part_nb == 0) fail(SC_ERR_STATE, "part chain: no part forward pass");
    if (!sums_in || !sums_out || !bad_out) fail(SC_ERR_CONFIG, "part: null argument");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    sc_trainer::ChainSlot& slot = chain_slot(t, 0);
    loss_chain_kernel<<<1, 256, 0, t->s0>>>(slot.pt.p, slot.dtm.p, t->part_nb, t->n, slot.out.p,
                                            slot.bad.p, sums_in[0], sums_in[1]);
    ck(cudaGetLastError(), "loss_chain_kernel");
    int32_t bad = kNone;
    ck(cudaMemcpyAsync(sums_out, slot.out.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, t->s0),
       "D2H");
    ck(cudaMemcpyAsync(&bad, slot.bad.p, sizeof bad, cudaMemcpyDeviceToHost, t->s0), "D2H");
    ck(cudaStreamSynchronize(t->s0), "part chain");
    *bad_out = bad == kNone ? -1 : t->part_b0 + bad;
  });
}

sc_status sc_trainer_part_backward(sc_trainer* t, const sc_params* params, double alpha,
                                   uint64_t global_count, int32_t global_batch, double* per_b) {
  return guarded([&] {
    if (!t || t->part_nb == 0) fail(SC_ERR_STATE, "part backward: no part forward pass");
    if (!params || !per_b) fail(SC_ERR_CONFIG, "part: null argument");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    const int nb = t->part_nb;
    const int64_t n = t->n;
    const unsigned long long cnt = global_count;
    ck(cudaMemcpyAsync(t->count.p, &cnt, sizeof cnt, cudaMemcpyHostToDevice, t->s0), "H2D");
    const int free_count = static_cast<int>(n) - t->n_pins;
    const double phys_denom = 3.0 * static_cast<double>(global_batch) * free_count;
    const int chunks = static_cast<int>((n + kChunk - 1) / kChunk);
    const size_t per_elem = static_cast<size_t>(chunks) * kTerms * kChunk * sizeof(double);
    const int group = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>(static_cast<size_t>(nb), t->term_budget / per_elem)));
    t->terms.ensure(static_cast<size_t>(group) * chunks * kTerms * kChunk);
    t->partial.ensure(static_cast<size_t>(group) * chunks * kScalars);
    t->grads.ensure(kScalars);
    DBuf<double> pb;
    pb.ensure(static_cast<size_t>(nb) * kScalars);
    ck(cudaMemsetAsync(t->grads.p, 0, sizeof(double) * kScalars, t->s0), "memset");
    const Frames fr{t->fx.p, t->fv.p, t->batch.idx_d.p + t->part_b0, t->nx, t->ny, n};
    for (int g0 = 0; g0 < nb; g0 += group) {
      const int ng = std::min(group, nb - g0);
      BwdArgs ba{};
      ba.fr = fr;
      ba.b0 = g0;
      ba.nb = ng;
      ba.net = net_of(*params);
      ba.rp = t->rp.p;
      ba.rd = t->rd.p;
      ba.phys_coeff = free_count > 0 ? 2.0 * alpha / phys_denom : 0.0;
      ba.alpha_loss = alpha;
      ba.data_count = t->count.p;
      ba.terms = t->terms.p;
      ba.chunks = chunks;
      bwd_terms_kernel<<<grid_for(n * ng), 256, 0, t->s0>>>(ba);
      ck(cudaGetLastError(), "bwd_terms_kernel");
      bwd_reduce_kernel<<<ng * chunks, 256, 0, t->s0>>>(t->terms.p, n, chunks, t->partial.p);
      ck(cudaGetLastError(), "bwd_reduce_kernel");
      bwd_final_kernel<<<1, 64, 0, t->s0>>>(t->partial.p, ng, chunks, t->grads.p,
                                            pb.p + static_cast<size_t>(g0) * kScalars);
      ck(cudaGetLastError(), "bwd_final_kernel");
    }
    ck(cudaMemcpyAsync(per_b, pb.p, sizeof(double) * nb * kScalars, cudaMemcpyDeviceToHost,
                       t->s0),
       "D2H");
    ck(cudaStreamSynchronize(t->s0), "part backward");
  });
}

sc_status sc_trainer_diagnose_forward(sc_trainer* t, const sc_params* params, int32_t frame,
                                      int32_t node, char* msg, int32_t len) {
  return guarded([&] {
    if (!t || !params || !msg || len < 1) fail(SC_ERR_CONFIG, "diagnose: null argument");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    const std::string m = diagnose_forward(t, frame, node, *params);
    std::snprintf(msg, static_cast<size_t>(len), "%s", m.c_str());
  });
}

sc_status sc_backward_gradients(int device, int32_t nx, int32_t ny, const double* x,
                                const double* v, const sc_params* params, const double* upstream,
                                double* grads_out) {
  return guarded([&] {
    if (nx < 2 || ny < 2) fail(SC_ERR_CONFIG, "state shape does not match the grid topology");
    if (!x || !v || !params || !upstream || !grads_out)
      fail(SC_ERR_CONFIG, "backward_gradients: null argument");
    if (!(params->isru_alpha > 0.0)) fail(SC_ERR_CONFIG, "isru_alpha: must be > 0");
    ck(cudaSetDevice(device), "cudaSetDevice");
    const int64_t n = static_cast<int64_t>(nx) * ny;
    const int chunks = static_cast<int>((n + kChunk - 1) / kChunk);
    DBuf<double> dx, dv, du, terms, partial, grads;
    DBuf<int32_t> idx;
    dx.ensure(n * 3);
    dv.ensure(n * 3);
    du.ensure(n * 3);
    terms.ensure(static_cast<size_t>(chunks) * kTerms * kChunk);
    partial.ensure(static_cast<size_t>(chunks) * kScalars);
    grads.ensure(kScalars);
    idx.ensure(1);
    ck(cudaMemcpy(dx.p, x, sizeof(double) * n * 3, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(dv.p, v, sizeof(double) * n * 3, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemcpy(du.p, upstream, sizeof(double) * n * 3, cudaMemcpyHostToDevice), "H2D");
    ck(cudaMemset(idx.p, 0, sizeof(int32_t)), "memset");
    ck(cudaMemset(grads.p, 0, sizeof(double) * kScalars), "memset");
    BwdArgs ba{};
    ba.fr = Frames{dx.p, dv.p, idx.p, nx, ny, n};
    ba.b0 = 0;
    ba.nb = 1;
    ba.net = net_of(*params);
    ba.upstream = du.p;
    ba.terms = terms.p;
    ba.chunks = chunks;
    bwd_terms_kernel<<<grid_for(n), 256>>>(ba);
    ck(cudaGetLastError(), "bwd_terms_kernel");
    bwd_reduce_kernel<<<chunks, 256>>>(terms.p, n, chunks, partial.p);
    ck(cudaGetLastError(), "bwd_reduce_kernel");
    bwd_final_kernel<<<1, 64>>>(partial.p, 1, chunks, grads.p, nullptr);
    ck(cudaGetLastError(), "bwd_final_kernel");
    ck(cudaMemcpy(grads_out, grads.p, sizeof(double) * kScalars, cudaMemcpyDeviceToHost), "D2H");
  });
}

sc_status sc_trainer_run(sc_trainer* t, const sc_train_config* cfg, const sc_params* resume_params,
                         const uint8_t* resume_trainable, sc_adam_state* opt_inout,
                         sc_params* params_out, uint8_t* trainable_out, double* history_out,
                         double* brackets_out) {
  return guarded([&] {
    if (!t) fail(SC_ERR_STATE, "null trainer");
    if (!cfg || !params_out) fail(SC_ERR_CONFIG, "train: null argument");
    ck(cudaSetDevice(t->device), "cudaSetDevice");
    validate_config(*cfg, t->frames - 1);
    Params params;
    sc_adam_state opt{};
    if (resume_params) {  // fine-tune mode: no pre-search (train.cpp:352-355)
      params = from_c(*resume_params);
      if (resume_trainable)
        for (int g = 0; g < 7; ++g) params.trainable[static_cast<size_t>(g)] = resume_trainable[g] != 0;
      if (opt_inout) opt = *opt_inout;
    } else {
      Rng de_rng(Rng::mix(cfg->seed, kTagSearch));
      params = de_preprocess(t, *cfg, de_rng);
    }
    for (int g = 0; g < 7; ++g)
      if (cfg->freeze_mask & (1u << g)) params.trainable[static_cast<size_t>(g)] = false;
    const int64_t start = opt.step;
    Batch batch;
    double grads[kScalars];
    // epochs run back to back; each epoch's loss chain proceeds on its own slot while the next
    // epochs compute, and is harvested in epoch order (history rows, error check) — the first
    // failing epoch raises exactly what the reference raises there
    struct Pending {
      size_t slot;
      int e;
      int64_t step;
      double lr;
      sc_params p;
      std::vector<int32_t> idx;
      LossLaunch L;
    };
    std::vector<Pending> pend;
    size_t head = 0;
    const size_t slot_bytes =
        static_cast<size_t>(cfg->batch_size) * static_cast<size_t>(t->n) * 2 * sizeof(double);
    const size_t nslots = std::max<size_t>(
        1, std::min<size_t>(kMaxSlots, (size_t(1) << 30) / std::max<size_t>(slot_bytes, 1)));
    for (size_t k = 0; k < nslots; ++k) {  // every allocation before the epochs (cudaMalloc syncs)
      sc_trainer::ChainSlot& c = chain_slot(t, k);
      c.pt.ensure(slot_bytes / (2 * sizeof(double)));
      c.dtm.ensure(slot_bytes / (2 * sizeof(double)));
      c.out.ensure(2);
      c.bad.ensure(1);
    }
    {
      const size_t bn = static_cast<size_t>(cfg->batch_size) * static_cast<size_t>(t->n);
      t->rp.ensure(bn * 3);
      t->rd.ensure(bn * 3);
      batch.idx_d.ensure(static_cast<size_t>(cfg->batch_size));
      batch.force_dt.ensure(bn * 3);
    }
    auto harvest = [&](const Pending& q) {
      Loss loss;
      try {
        loss = finish_loss(t, q.p, q.idx, cfg->alpha, q.L, t->slots[q.slot]);
      } catch (const Fail& f) {
        if (f.code != SC_ERR_NUMERICS) throw;
        fail(SC_ERR_NUMERICS, f.msg + " [optimizer step " + std::to_string(q.step) + "]");
      }
      if (history_out) {
        double* row = history_out + static_cast<int64_t>(q.e) * 5;
        row[0] = static_cast<double>(q.step);
        row[1] = q.lr;
        row[2] = loss.physics;
        row[3] = loss.data;
        row[4] = loss.total;
      }
    };
    for (int e = 0; e < cfg->epochs; ++e) {
      const int64_t step = start + e;
      const double lr = schedule_lr(*cfg, static_cast<int>(step));
      Rng rng(Rng::mix(cfg->seed, static_cast<uint64_t>(step)));
      sample_batch(t, cfg->batch_size, rng, batch);
      batch_targets(t, batch);
      const size_t k = static_cast<size_t>(e) % nslots;
      if (pend.size() - head == nslots) harvest(pend[head++]);  // frees slot k
      Pending q{k, e, step, lr, to_c(params), batch.idx, LossLaunch{}};
      q.L = launch_loss(t, q.p, batch, cfg->alpha, grads, chain_slot(t, k));
      if (q.L.first_bad_fwd != kNone) {  // raises: earlier epochs' chains first, then this one
        while (head < pend.size()) harvest(pend[head++]);
        harvest(q);
      }
      adam_update(params, grads, opt, lr);
      pend.push_back(std::move(q));
      while (head < pend.size() &&
             cudaEventQuery(t->slots[pend[head].slot].ev_done) == cudaSuccess)
        harvest(pend[head++]);
    }
    while (head < pend.size()) harvest(pend[head++]);
    *params_out = to_c(params);
    if (trainable_out)
      for (int g = 0; g < 7; ++g) trainable_out[g] = params.trainable[static_cast<size_t>(g)] ? 1 : 0;
    if (brackets_out)
      for (int k = 0; k < 14; ++k) brackets_out[k] = params.brackets[static_cast<size_t>(k)];
    if (opt_inout) *opt_inout = opt;
  });
}

}  // extern "C"
