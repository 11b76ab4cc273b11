// Device-side definitions shared by the PARITY and FAST step kernels.
//
// HBM layout: one ctx holds `batch` cloths; cloth b owns a block of 6*S elements
// (S = plane_stride = rows_local * pitch, pitch = nx rounded up to 4) holding, row-major,
//   [x.xy: S interleaved (x,y) pairs][v.xy: S pairs][x.z: S][v.z: S]
// i.e. the x/y components of a node sit next to each other (one 8-byte element) so the FAST
// kernel processes them as packed f32x2 pairs, while z is a plain plane. Validity masks, pins
// and collider constants come from (ix, iy) or small per-cloth tables, so a step moves exactly
// 48 B per node (f32): x and v read once and written once.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace scb {

constexpr int kChannels = 12;

// canonical channel order E,N,W,S,NE,NW,SW,SE,E2,N2,W2,S2 (reference grid.cpp:14-30)
__host__ __device__ constexpr int off_dx(int c) {
  return c == 0 ? 1 : c == 1 ? 0 : c == 2 ? -1 : c == 3 ? 0 : c == 4 ? 1 : c == 5 ? -1
       : c == 6 ? -1 : c == 7 ? 1 : c == 8 ? 2 : c == 9 ? 0 : c == 10 ? -2 : 0;
}
__host__ __device__ constexpr int off_dy(int c) {
  return c == 0 ? 0 : c == 1 ? 1 : c == 2 ? 0 : c == 3 ? -1 : c == 4 ? 1 : c == 5 ? 1
       : c == 6 ? -1 : c == 7 ? -1 : c == 8 ? 0 : c == 9 ? 2 : c == 10 ? 0 : -2;
}

// Column swizzles of the planes: within every aligned group of 4 columns whose
// group index has bit 2 set (columns with bit 4 set), the two 2-column halves are swapped. A
// FAST-kernel lane owns one group; with this layout the lanes of a quarter-warp read their
// 16-byte window pieces from 8 distinct bank groups (the plain layout puts lanes l and l+4 on
// the same banks). Pure permutation within a group: any row segment of whole groups is
// contiguous, and every access goes through elem_index / xy_col.
__host__ __device__ __forceinline__ int64_t xy_col(int64_t c) { return c ^ ((c >> 3) & 2); }
// The same for the z planes with group-index bit 3 (columns with bit 5 set), in contexts whose
// FAST launches take the general (collider / pressure / mask) finish (`zs`): a lane's 8-byte
// window pieces (its own two halves and the neighbour halves of its halo) then come from 16
// distinct bank pairs in every half-warp (the plain layout puts lanes l and l+8 on one pair).
// Measured: config 5 (plane colliders) 696 -> 657 us/step; the simple-finish kernel is faster on
// the plain layout (config 2: 45.9 vs 46.8 us), so collider-free contexts keep it.
__host__ __device__ __forceinline__ int64_t z_col(int64_t c, bool zs) {
  return zs ? c ^ ((c >> 4) & 2) : c;
}

// Element index of component p (0..5 = x.x x.y x.z v.x v.y v.z) of local row r, column c
// within one cloth's block (see the layout above).
__host__ __device__ __forceinline__ int64_t elem_index(int p, int64_t r, int64_t c, int64_t pitch,
                                                       int64_t S, bool zs) {
  const int64_t rc = r * pitch + z_col(c, zs);
  const int64_t rx = r * pitch + xy_col(c);
  switch (p) {
    case 0: return 2 * rx;
    case 1: return 2 * rx + 1;
    case 2: return 4 * S + rc;
    case 3: return 2 * S + 2 * rx;
    case 4: return 2 * S + 2 * rx + 1;
    default: return 5 * S + rc;
  }
}

// IEEE round-to-nearest primitives that can never be contracted into FMA. The parity kernels
// and the shared plug/advance stage use only these, so they reproduce the reference's x86
// SSE scalar arithmetic bit for bit.
template <typename T>
struct RN;
template <>
struct RN<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ bool finite(float a) { return isfinite(a); }
};
template <>
struct RN<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
  static __device__ __forceinline__ bool finite(double a) { return isfinite(a); }
};

// NetKernel<T> (reference kernels.hpp:255-260), cast once on the host (net_kernel.hpp:8-22).
template <typename T>
struct NetConst {
  T gain[kChannels], wl[kChannels], wn[kChannels], wd[kChannels];
  T b[3];
  T wv, alpha;
};

// Per-cloth SceneKernel<T> constants (kernels.hpp:41-56) with the derived products the
// reference computes in T inside add_plug_impulse / advance_with_impulse precomputed on the
// host with the same single IEEE operation (so they are bit-identical).
template <typename T>
struct ClothConst {
  // FAST simple finish: plugged gravity impulse (or 0) x3, plugged drag coefficient (or 0)
  T fin[4];
  T dt;
  T scale;     // dt / mass                          (kernels.hpp:182)
  T drag_c;    // drag * scale                       (kernels.hpp:193)
  T pressure;  //                                    (kernels.hpp:183)
  T dv[3];     // gravity * dt                       (kernels.hpp:189)
  T pin_u[3];  // pin velocity                       (kernels.hpp:248-249)
  int32_t plug_pressure;  // plugged AND pressure != 0 (kernels.hpp:183)
  int32_t plug_gravity, plug_drag;
  int32_t n_spheres, sphere0, n_planes, plane0;
  int32_t n_pins;
  int32_t pin_row_lo, pin_row_hi;  // rows holding pins (skip the bitmap lookup elsewhere)
  // ground-truth mass-spring step (PBS): MaterialParams cast to T (kernels.hpp:62-70)
  T stiffness, damping, mass, drag;
  T grav[3];
  T rest[kChannels];  // topology rest lengths spacing * {1, sqrt2, 2} cast to T (kernels.hpp:69-70)
  int64_t pin_word0;  // first word of this cloth's pin bitmap / rank prefix
  int64_t anchor0;    // first anchor (x3) of this cloth
};

template <typename T>
struct SphereConst {
  T c[3];
  T R;
  T Rband;  // R * (1 + 16 eps)          (kernels.hpp:217, contact_band :23-28)
  T omf;    // 1 - friction              (kernels.hpp:221,239)
};

// Plane z = h, normal +z (extension; no reference counterpart).
template <typename T>
struct PlaneConst {
  T h;
  T band;  // max(|h|, 1) * 16 eps: velocity-level contact when x.z - h <= band
  T omf;
};

struct Health {
  // min over (frame << 32 | node) of non-finite cell impulses (net.cpp:139-140) — for the PBS
  // step: of singular springs (kernels.hpp:96-107); ~0 if none
  unsigned long long impulse_key;
  int32_t state_frame;  // first frame with a non-finite x' or v' (eval.cpp:98-99); INT_MAX
  int32_t pad;
};

template <typename T>
struct StepArgs {
  const T* in;
  T* out;
  int64_t plane_stride;  // elements per plane per cloth
  int32_t pitch;
  int32_t nx, ny;        // global grid
  int32_t g0;            // global row of local row 0
  int32_t u0, u1;        // global rows to update [u0, u1)
  int32_t batch;
  int32_t b_off;         // FAST launches over cloths [b_off, b_off + batch) (pipelined rollout)
  const int32_t* ids;    // FAST launches: cloth b of the launch is ids[b] (class groups), or b
  int32_t zs;            // z planes carry the z_col swizzle (contexts on the general finish)
  int32_t k;             // step index: t_next = T(k+1) * dt
  int32_t use_t_override;
  T t_override;
  const ClothConst<T>* cloths;
  const SphereConst<T>* spheres;
  const PlaneConst<T>* planes;
  const uint32_t* pin_bits;
  const int32_t* pin_rank;  // prefix popcount per bitmap word
  const T* pin_anchors;
  uint8_t* constrained;     // [batch][ny*nx] global node index, or nullptr
  T* impulse;               // planar [batch][3][local plane] or nullptr (forward-only output)
  Health* health;           // [batch] or nullptr
  // fused halo exchange (FAST strips with peer neighbours): the two owned rows next to side s
  // are also stored into that neighbour's output buffer (peer_out[s], its plane stride and row
  // base), i.e. straight into its ghost rows over NVLink. nullptr: no peer on that side.
  T* peer_out[2];
  int64_t peer_S[2];
  int32_t peer_g0[2];
  NetConst<T> net;
};

// ---- shared per-node tail -----------------------------------------------------------------
// plug_tail: gravity + drag of add_plug_impulse (kernels.hpp:188-195), applied after pressure.
// advance_node: advance_with_impulse for one node (kernels.hpp:210-251).
// Exactly the reference operation order, in non-contractible IEEE ops.
template <typename T>
__device__ __forceinline__ void plug_tail(const ClothConst<T>& cc, const T v[3], T imp[3]) {
  using R = RN<T>;
  if (cc.plug_gravity) {
#pragma unroll
    for (int d = 0; d < 3; ++d) imp[d] = R::add(imp[d], cc.dv[d]);
  }
  if (cc.plug_drag) {
#pragma unroll
    for (int d = 0; d < 3; ++d) imp[d] = R::sub(imp[d], R::mul(v[d], cc.drag_c));
  }
}

// The collider responses of advance_with_impulse, one collider and one node per call, so the
// FAST collider finish can run them collider-outer / node-inner with the same per-node sequence.
template <typename T>
__device__ __forceinline__ void sphere_velocity(const SphereConst<T>& sp, const T x[3], T vv[3],
                                                uint8_t& mask) {  // kernels.hpp:213-225
  using R = RN<T>;
  T r[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) r[d] = R::sub(x[d], sp.c[d]);
  const T dist = R::sqrt(R::add(R::add(R::mul(r[0], r[0]), R::mul(r[1], r[1])), R::mul(r[2], r[2])));
  if (dist > T(0) && dist <= sp.Rband) {
    const T vn = R::div(R::add(R::add(R::mul(vv[0], r[0]), R::mul(vv[1], r[1])), R::mul(vv[2], r[2])), dist);
    if (vn < T(0)) {
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const T nrm = R::div(r[d], dist);
        vv[d] = R::mul(R::sub(vv[d], R::mul(nrm, vn)), sp.omf);
      }
      mask = 1;
    }
  }
}
template <typename T>
__device__ __forceinline__ void plane_velocity(const PlaneConst<T>& pl, const T x[3], T vv[3],
                                               uint8_t& mask) {
  using R = RN<T>;
  if (R::sub(x[2], pl.h) <= pl.band && vv[2] < T(0)) {
    const T vn = vv[2];
    vv[0] = R::mul(vv[0], pl.omf);
    vv[1] = R::mul(vv[1], pl.omf);
    vv[2] = R::mul(R::sub(vv[2], vn), pl.omf);
    mask = 1;
  }
}
template <typename T>
__device__ __forceinline__ void sphere_position(const SphereConst<T>& sp, T xo[3], T vo[3],
                                                uint8_t& mask) {  // kernels.hpp:229-244
  using R = RN<T>;
  T r[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) r[d] = R::sub(xo[d], sp.c[d]);
  const T dist = R::sqrt(R::add(R::add(R::mul(r[0], r[0]), R::mul(r[1], r[1])), R::mul(r[2], r[2])));
  if (dist > T(0) && dist < sp.R) {
    T nrm[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      nrm[d] = R::div(r[d], dist);
      xo[d] = R::add(sp.c[d], R::mul(nrm[d], sp.R));
    }
    const T vn = R::add(R::add(R::mul(vo[0], nrm[0]), R::mul(vo[1], nrm[1])), R::mul(vo[2], nrm[2]));
    if (vn < T(0)) {
#pragma unroll
      for (int d = 0; d < 3; ++d) vo[d] = R::mul(R::sub(vo[d], R::mul(nrm[d], vn)), sp.omf);
    }
    mask = 1;
  }
}
template <typename T>
__device__ __forceinline__ void plane_position(const PlaneConst<T>& pl, T xo[3], T vo[3],
                                               uint8_t& mask) {
  using R = RN<T>;
  if (xo[2] < pl.h) {
    xo[2] = pl.h;
    const T vn = vo[2];
    if (vn < T(0)) {
      vo[0] = R::mul(vo[0], pl.omf);
      vo[1] = R::mul(vo[1], pl.omf);
      vo[2] = R::mul(R::sub(vo[2], vn), pl.omf);
    }
    mask = 1;
  }
}
// Dirichlet re-pin (kernels.hpp:245-251): bitmap + rank prefix -> anchor slot
template <typename T>
__device__ __forceinline__ void repin_t(const StepArgs<T>& a, const ClothConst<T>& cc, int row,
                                        int64_t gnode, T t_next, T xo[3], T vo[3], uint8_t& mask) {
  using R = RN<T>;
  if (cc.n_pins > 0 && row >= cc.pin_row_lo && row <= cc.pin_row_hi) {
    const int64_t w = cc.pin_word0 + (gnode >> 5);
    const uint32_t bits = __ldg(a.pin_bits + w);
    const uint32_t bit = 1u << (gnode & 31);
    if (bits & bit) {
      const int64_t slot = cc.anchor0 + __ldg(a.pin_rank + w) + __popc(bits & (bit - 1u));
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        vo[d] = cc.pin_u[d];
        xo[d] = R::add(__ldg(a.pin_anchors + 3 * slot + d), R::mul(cc.pin_u[d], t_next));
      }
      mask = 1;
    }
  }
}
template <typename T>
__device__ __forceinline__ void repin(const StepArgs<T>& a, const ClothConst<T>& cc, int row,
                                      int64_t gnode, T xo[3], T vo[3], uint8_t& mask) {
  using R = RN<T>;
  if (cc.n_pins > 0 && row >= cc.pin_row_lo && row <= cc.pin_row_hi) {
    const T t_next = a.use_t_override ? a.t_override : R::mul(T(a.k + 1), cc.dt);
    repin_t(a, cc, row, gnode, t_next, xo, vo, mask);
  }
}

template <typename T>
__device__ __forceinline__ void advance_node(const StepArgs<T>& a, const ClothConst<T>& cc,
                                             int row, int64_t gnode, const T x[3], const T v[3],
                                             const T imp[3], T xo[3], T vo[3], uint8_t& mask) {
  using R = RN<T>;
  mask = 0;
  T vv[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) vv[d] = R::add(v[d], imp[d]);
  // velocity-level response on the OLD positions (kernels.hpp:213-225)
  for (int s = 0; s < cc.n_spheres; ++s) sphere_velocity(a.spheres[cc.sphere0 + s], x, vv, mask);
  for (int q = 0; q < cc.n_planes; ++q) plane_velocity(a.planes[cc.plane0 + q], x, vv, mask);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    vo[d] = vv[d];
    xo[d] = R::add(x[d], R::mul(vv[d], cc.dt));
  }
  // position-level intersection elimination (kernels.hpp:229-244)
  for (int s = 0; s < cc.n_spheres; ++s) sphere_position(a.spheres[cc.sphere0 + s], xo, vo, mask);
  for (int q = 0; q < cc.n_planes; ++q) plane_position(a.planes[cc.plane0 + q], xo, vo, mask);
  repin(a, cc, row, gnode, xo, vo, mask);  // Dirichlet re-pin last
}

// ---- pressure plug (accumulate_pressure kernels.hpp:142-155 + scaling :183-187) -----------
// e,n,w,s are x_i - x_{E,N,W,S}; only interior nodes get the cross products, the others a
// zero force; the reference then adds f*scale to every node.
template <typename T>
__device__ __forceinline__ void pressure_plug(const ClothConst<T>& cc, bool interior,
                                              const T e[3], const T n[3], const T w[3],
                                              const T s[3], T imp[3]) {
  using R = RN<T>;
  T f[3] = {T(0), T(0), T(0)};
  if (interior) {
    auto cross = [](const T* p, const T* q, T* o) {
      o[0] = R::sub(R::mul(p[1], q[2]), R::mul(p[2], q[1]));
      o[1] = R::sub(R::mul(p[2], q[0]), R::mul(p[0], q[2]));
      o[2] = R::sub(R::mul(p[0], q[1]), R::mul(p[1], q[0]));
    };
    T c1[3], c2[3], c3[3], c4[3];
    cross(e, n, c1);
    cross(n, w, c2);
    cross(w, s, c3);
    cross(s, e, c4);
#pragma unroll
    for (int d = 0; d < 3; ++d) f[d] = R::mul(R::add(R::add(R::add(c1[d], c2[d]), c3[d]), c4[d]), cc.pressure);
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) imp[d] = R::add(imp[d], R::mul(f[d], cc.scale));
}

}  // namespace scb
