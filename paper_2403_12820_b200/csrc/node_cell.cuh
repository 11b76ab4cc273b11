// FAST per-node cell and finish of the small-cloth kernel (small_kernels.cu): one thread
// evaluates one node's twelve channels in the reference order (forward_impulse<T>, kernels.hpp:265-282; masked channels skipped) in FAST
// arithmetic (FMA, rsqrt.approx ISRU, gains folded into the weights as in fast_kernels.cu), then
// the plug tail and advance (add_plug_impulse / advance_with_impulse, kernels.hpp:179-252): the
// simple finish's contracted chain for collider-free cloths, the IEEE chain of sc_device.cuh for
// cloths with colliders (same contact decisions as PARITY), the Dirichlet re-pin last.
#pragma once

#include "fast_rowpass.cuh"
#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {
namespace nodecell {

// canonical channel order E,N,W,S,NE,NW,SW,SE,E2,N2,W2,S2 (grid.cpp:14-30)
// (functions, so the offsets fold to immediates after unrolling: no constant-bank arrays)
__host__ __device__ constexpr int kDx(int c) {
  return c == 0 ? 1 : c == 2 ? -1 : c == 4 ? 1 : c == 5 ? -1 : c == 6 ? -1 : c == 7 ? 1
       : c == 8 ? 2 : c == 10 ? -2 : 0;
}
__host__ __device__ constexpr int kDy(int c) {
  return c == 1 ? 1 : c == 3 ? -1 : c == 4 ? 1 : c == 5 ? 1 : c == 6 ? -1 : c == 7 ? -1
       : c == 9 ? 2 : c == 11 ? -2 : 0;
}

// acc = b + v wV + sum over valid channels c of dx (wL' + r (wN' + dv wD')), per component.
// nb(c, d) returns component d (0..5: x then v) of channel c's neighbour.
template <bool ALPHA1, typename NB>
__device__ __forceinline__ void cell(const FastNet& f, const float (&x)[3], const float (&v)[3],
                                     uint32_t valid, NB nb, float (&acc)[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) acc[d] = fmaf(v[d], f.wv, f.b[d]);
#pragma unroll
  for (int c = 0; c < kChannels; ++c) {
    if (!((valid >> c) & 1u)) continue;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float dx = x[d] - nb(c, d);
      const float dv = v[d] - nb(c, 3 + d);
      const float q = ALPHA1 ? fmaf(dx, dx, 1.0f) : fmaf(dx * f.alpha[c], dx, 1.0f);
      const float r = fastrow::rsqrt_q(q);
      const float w = fmaf(r, fmaf(dv, f.wd[c], f.wn[c]), f.wl[c]);
      acc[d] = fmaf(dx, w, acc[d]);
    }
  }
}

// plug tail + advance + re-pin of one node from its cell impulse `acc` (modified); mk: contact
// mask (0 / 1). Health records as the row-pass finishes do.
template <bool GEN>
__device__ __forceinline__ void finish(const StepArgs<float>& a, const ClothConst<float>& cc,
                                       bool simple, int b, int k, int row, int64_t gnode,
                                       float t_next, const float (&x)[3], const float (&v)[3],
                                       float (&acc)[3], float (&xo)[3], float (&vo)[3],
                                       uint8_t& mk) {
  if (a.health && !(isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]))) {
    const unsigned long long key = (static_cast<unsigned long long>(k + 1) << 32) |
                                   static_cast<unsigned long long>(gnode);
    atomicMin(&a.health[b].impulse_key, key);
  }
  mk = 0;
  if (!GEN || simple) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float imp = fmaf(v[d], -cc.fin[3], acc[d] + cc.fin[d]);
      vo[d] = v[d] + imp;
      xo[d] = fmaf(vo[d], cc.dt, x[d]);
    }
  } else {
    plug_tail(cc, v, acc);
    float vv[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) vv[d] = __fadd_rn(v[d], acc[d]);
    for (int q = 0; q < cc.n_spheres; ++q) sphere_velocity(a.spheres[cc.sphere0 + q], x, vv, mk);
    for (int q = 0; q < cc.n_planes; ++q) plane_velocity(a.planes[cc.plane0 + q], x, vv, mk);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      vo[d] = vv[d];
      xo[d] = __fadd_rn(x[d], __fmul_rn(vv[d], cc.dt));
    }
    for (int q = 0; q < cc.n_spheres; ++q) sphere_position(a.spheres[cc.sphere0 + q], xo, vo, mk);
    for (int q = 0; q < cc.n_planes; ++q) plane_position(a.planes[cc.plane0 + q], xo, vo, mk);
  }
  repin_t(a, cc, row, gnode, t_next, xo, vo, mk);  // Dirichlet re-pin last
  if (a.health && !(isfinite(xo[0]) && isfinite(xo[1]) && isfinite(xo[2]) && isfinite(vo[0]) &&
                    isfinite(vo[1]) && isfinite(vo[2])))
    atomicMin(&a.health[b].state_frame, k + 1);
}

}  // namespace nodecell
}  // namespace scb
