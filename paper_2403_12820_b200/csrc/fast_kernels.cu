// FAST-mode fused step kernel (f32): forward_impulse -> add_plug_impulse -> advance_with_impulse
// in one pass over HBM (reference kernels.hpp:179-282 driven by eval.cpp:48-59).
//
// Design:
//  * Warp = one 128-column strip of one cloth, marching upward over a segment of rows. Each lane
//    owns 4 consecutive columns (float4 in every plane).
//  * Rows are staged in a 6-slot shared-memory ring by TMA (cp.async.bulk.tensor.3d, one box of
//    136 columns x 1 row x 6 planes per row starting at the 16-byte-aligned column x0-4 — TMA
//    rejects unaligned starts — with negative / past-the-end coordinates zero-filled), two rows
//    ahead of use, so HBM latency hides behind the arithmetic.
//  * Edge sharing: the 12 stencil channels are 6 undirected edge types (E, E2, N, N2, NE, NW).
//    Each edge's difference, ISRU (one MUFU.RSQ) and derivative product are computed once and
//    pushed into both endpoint accumulators (isru is odd and differences are antisymmetric, so
//    the negated channel's term follows from the same values; grid.cpp:32-35).
//  * Accumulators of rows R-2, R-1, R live in registers; row R-2 is complete after step R and is
//    finished (plug, integrate, collide, pin) with the same IEEE-exact code as PARITY mode and
//    stored with STG.128. The cell sum itself uses FMA + rsqrt and a different summation order,
//    hence "within 1e-5 relative per step" instead of bit-exact.
#include <cuda.h>

#include <algorithm>

#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

constexpr int FW = 4;              // columns per lane
constexpr int STRIP = 32 * FW;     // columns per warp
constexpr int BOXW = STRIP + 8;    // staged columns x0-4 .. x0+131 (2-column halo + alignment)
constexpr int RING = 5;            // staged rows: R-3 .. R+1 (one row of prefetch)
constexpr int ROW_BYTES = 6 * BOXW * 4;            // bytes one TMA box delivers (6 planes)
constexpr int ROWF = ((ROW_BYTES + 127) / 128) * 32;  // ring slot stride in floats (128 B aligned)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_row(float* dst, const CUtensorMap* map, int c0, int c1,
                                             int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// rsqrt without the denormal fix-up rsqrtf() carries under -ftz=false: q = 1 + a dx^2 >= 1.
__device__ __forceinline__ float rsqrt_q(float q) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return r;
}

// Edge contribution to its origin node a (channel ca) and far node b (channel cb = -ca):
//   a: acc += dx*wL'_ca + s*(wN'_ca + dv*wD'_ca)
//   b: acc += dx*(-wL'_cb) + s*(dv*wD'_cb - wN'_cb)
// with dx = x_a - x_b, dv = v_a - v_b, s = dx * rsqrt(1 + alpha'_c dx^2) and the gains folded
// into the primed weights (wL' = g wL, wN' = g wN, wD' = g^2 wD, alpha' = alpha g^2).
// Invalid edges (an endpoint outside the grid) arrive with dx = dv = 0 and contribute exactly 0.
template <bool ALPHA1, bool PA, bool PB>
__device__ __forceinline__ void edge(const FastNet& f, int ca, int cb, float dx, float dv,
                                     float& acc_a, float& acc_b) {
  const float q = ALPHA1 ? fmaf(dx, dx, 1.0f) : fmaf(dx * f.alpha[ca], dx, 1.0f);
  const float s = dx * rsqrt_q(q);
  if (PA) {
    const float t = fmaf(dv, f.wd[ca], f.wn[ca]);
    acc_a = fmaf(dx, f.wl[ca], acc_a);
    acc_a = fmaf(s, t, acc_a);
  }
  if (PB) {
    const float t = fmaf(dv, f.wd[cb], f.nwn[cb]);
    acc_b = fmaf(dx, f.nwl[cb], acc_b);
    acc_b = fmaf(s, t, acc_b);
  }
}

// Lane window of a staged row: columns ix0-2 .. ix0+5 <-> box index 4*lane+2 .. 4*lane+9.
__device__ __forceinline__ void load8(const float* base, int lane, float* o) {
  const float2 l = *reinterpret_cast<const float2*>(base + FW * lane + 2);
  const float4 m = *reinterpret_cast<const float4*>(base + FW * lane + 4);
  const float2 r = *reinterpret_cast<const float2*>(base + FW * lane + 8);
  o[0] = l.x; o[1] = l.y; o[2] = m.x; o[3] = m.y; o[4] = m.z; o[5] = m.w; o[6] = r.x; o[7] = r.y;
}

__device__ __forceinline__ void load4(const float* base, int lane, float* o) {
  const float4 m = *reinterpret_cast<const float4*>(base + FW * lane + 4);
  o[0] = m.x; o[1] = m.y; o[2] = m.z; o[3] = m.w;
}

// All edges of one component whose upper endpoint lies on row R, pushed into the accumulators
// of rows R-2 (A0), R-1 (A1), R (A2). mL / mRt zero the edges that leave the grid through the
// strip's left / right boundary lane; GENERAL additionally applies the row masks of the first
// and last two rows of the cloth (uniform per step).
template <bool ALPHA1, bool GENERAL, bool TAIL>
__device__ __forceinline__ void comp_pass(const FastNet& f, const float* rowR, const float* row1,
                                          const float* row2, int lane, float mL, float mRt,
                                          float mR, float m1, float m2, float (&A0)[4],
                                          float (&A1)[4], float (&A2)[4], int d) {
  float xr[8], vr[8], x1[8], v1[8], x2[4], v2[4];
  load8(rowR + d * BOXW, lane, xr);
  load8(rowR + (3 + d) * BOXW, lane, vr);
  load8(row1 + d * BOXW, lane, x1);
  load8(row1 + (3 + d) * BOXW, lane, v1);
  load4(row2 + d * BOXW, lane, x2);
  load4(row2 + (3 + d) * BOXW, lane, v2);
  if (TAIL) {
    // rows R >= y1 are not owned: only the pushes into rows R-1, R-2 (a-sides of the edges
    // that reach up to row R) are still needed
    float dummy = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      edge<ALPHA1, true, false>(f, 1, 3, x1[k + 2] - xr[k + 2], v1[k + 2] - vr[k + 2], A1[k],
                                dummy);
      edge<ALPHA1, true, false>(f, 9, 11, x2[k] - xr[k + 2], v2[k] - vr[k + 2], A0[k], dummy);
    }
#pragma unroll
    for (int e = 1; e < 5; ++e) {
      float dx = x1[e + 1] - xr[e + 2], dv = v1[e + 1] - vr[e + 2];
      if (e == 4) {
        dx *= mRt;
        dv *= mRt;
      }
      edge<ALPHA1, true, false>(f, 4, 6, dx, dv, A1[e - 1], dummy);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float dx = x1[e + 2] - xr[e + 1], dv = v1[e + 2] - vr[e + 1];
      if (e == 0) {
        dx *= mL;
        dv *= mL;
      }
      edge<ALPHA1, true, false>(f, 5, 7, dx, dv, A1[e], dummy);
    }
    return;
  }
  // init row R: b + v*wV
#pragma unroll
  for (int k = 0; k < 4; ++k) A2[k] = fmaf(vr[k + 2], f.wv, f.b[d]);

  float dummy = 0.0f;
  auto mask_of = [&](int e, int lo, int hi, float row) -> float {
    // lane-column mask for slot e of an edge family whose slots < lo / > hi may leave the grid
    float m = e < lo ? mL : (e > hi ? mRt : 1.0f);
    return GENERAL ? m * row : m;
  };
  // E edges in row R: a = col ix0-1+e (j = e+1), b = col ix0+e (j = e+2)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = xr[e + 1] - xr[e + 2], dv = vr[e + 1] - vr[e + 2];
    if (GENERAL || e == 0 || e == 4) {
      const float m = mask_of(e, 1, 3, mR);
      dx *= m;
      dv *= m;
    }
    if (e == 0) edge<ALPHA1, false, true>(f, 0, 2, dx, dv, dummy, A2[0]);
    else if (e == 4) edge<ALPHA1, true, false>(f, 0, 2, dx, dv, A2[3], dummy);
    else edge<ALPHA1, true, true>(f, 0, 2, dx, dv, A2[e - 1 < 0 ? 0 : e - 1], A2[e > 3 ? 3 : e]);
  }
  // E2 edges in row R: a = col ix0-2+e (j = e), b = col ix0+e (j = e+2)
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    float dx = xr[e] - xr[e + 2], dv = vr[e] - vr[e + 2];
    if (GENERAL || e <= 1 || e >= 4) {
      const float m = mask_of(e, 2, 3, mR);
      dx *= m;
      dv *= m;
    }
    if (e <= 1) edge<ALPHA1, false, true>(f, 8, 10, dx, dv, dummy, A2[e]);
    else if (e >= 4) edge<ALPHA1, true, false>(f, 8, 10, dx, dv, A2[e - 2], dummy);
    else edge<ALPHA1, true, true>(f, 8, 10, dx, dv, A2[e - 2], A2[e]);
  }
  // N edges (R-1 -> R) and N2 edges (R-2 -> R), owned columns
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float dx = x1[k + 2] - xr[k + 2], dv = v1[k + 2] - vr[k + 2];
    if (GENERAL) {
      dx *= m1;
      dv *= m1;
    }
    edge<ALPHA1, true, true>(f, 1, 3, dx, dv, A1[k], A2[k]);
    float dx2 = x2[k] - xr[k + 2], dv2 = v2[k] - vr[k + 2];
    if (GENERAL) {
      dx2 *= m2;
      dv2 *= m2;
    }
    edge<ALPHA1, true, true>(f, 9, 11, dx2, dv2, A0[k], A2[k]);
  }
  // NE edges: a = (ix0-1+e, R-1) (j = e+1), b = (ix0+e, R) (j = e+2)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = x1[e + 1] - xr[e + 2], dv = v1[e + 1] - vr[e + 2];
    if (GENERAL || e == 0 || e == 4) {
      const float m = mask_of(e, 1, 3, m1);
      dx *= m;
      dv *= m;
    }
    if (e == 0) edge<ALPHA1, false, true>(f, 4, 6, dx, dv, dummy, A2[0]);
    else if (e == 4) edge<ALPHA1, true, false>(f, 4, 6, dx, dv, A1[3], dummy);
    else edge<ALPHA1, true, true>(f, 4, 6, dx, dv, A1[e - 1 < 0 ? 0 : e - 1], A2[e > 3 ? 3 : e]);
  }
  // NW edges: a = (ix0+e, R-1) (j = e+2), b = (ix0+e-1, R) (j = e+1)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = x1[e + 2] - xr[e + 1], dv = v1[e + 2] - vr[e + 1];
    if (GENERAL || e == 0 || e == 4) {
      const float m = mask_of(e, 1, 3, m1);
      dx *= m;
      dv *= m;
    }
    if (e == 0) edge<ALPHA1, true, false>(f, 5, 7, dx, dv, A1[0], dummy);
    else if (e == 4) edge<ALPHA1, false, true>(f, 5, 7, dx, dv, dummy, A2[3]);
    else edge<ALPHA1, true, true>(f, 5, 7, dx, dv, A1[e > 3 ? 3 : e], A2[e - 1 < 0 ? 0 : e - 1]);
  }
}

template <bool ALPHA1>
__global__ void __launch_bounds__(32) fast_step_kernel(const __grid_constant__ CUtensorMap tmap,
                                                      const StepArgs<float> a, const FastNet f,
                                                      const int n_strips, const int seg_rows,
                                                      const int n_segs) {
  extern __shared__ __align__(128) float ring[];  // [RING][6][BOXW] (slot stride ROWF)
  __shared__ __align__(8) uint64_t full[RING];
  __shared__ float scratch[32][13];  // per-lane impulse staging for the collider finish

  const int lane = threadIdx.x;
  const int unit = blockIdx.x;
  const int seg = unit % n_segs;
  const int strip = (unit / n_segs) % n_strips;
  const int b = unit / (n_segs * n_strips);
  const int y0 = a.u0 + seg * seg_rows;
  const int y1 = min(y0 + seg_rows, a.u1);
  if (y0 >= y1) return;
  const int x0 = strip * STRIP;
  const int ix0 = x0 + FW * lane;
  const int nx = a.nx, ny = a.ny;

  // Rows y0-2 .. y1+1 pass through the ring; arithmetic starts at row y0 (the two rows below
  // only feed rows < y0) and the last two steps (rows y1, y1+1) only finish rows y1-2, y1-1.
  const int r_first = y0 - 2;
  const int r_last = y1 + 1;

  if (lane == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int row) {  // lane 0 only
    const int t = row - r_first;
    uint64_t* bar = &full[t % RING];
    mbar_expect_tx(bar, ROW_BYTES);
    tma_load_row(ring + (t % RING) * ROWF, &tmap, x0 - 4, row - a.g0, 6 * b, bar);
  };
  if (lane == 0) {
    issue(r_first);
    issue(r_first + 1);
    issue(r_first + 2);
  }
  mbar_wait(&full[0], 0);
  mbar_wait(&full[1], 0);

  // nx % 4 == 0 (fast_supported): only a strip's outermost lanes own edges leaving the grid
  const float mL = ix0 >= 1 ? 1.0f : 0.0f;
  const float mRt = ix0 + 4 < nx ? 1.0f : 0.0f;
  const bool lane_live = ix0 < nx;

  const ClothConst<float> cc = a.cloths[b];
  const bool simple = cc.n_spheres == 0 && cc.n_planes == 0 && !cc.plug_pressure &&
                      a.constrained == nullptr;
  const int64_t nodes = static_cast<int64_t>(nx) * ny;
  float* out_b = a.out + static_cast<int64_t>(b) * 6 * a.plane_stride;
  const float t_next = a.use_t_override ? a.t_override : __fmul_rn(float(a.k + 1), cc.dt);

  float A0[3][4], A1[3][4], A2[3][4];  // [component][column] for rows R-2, R-1, R
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int k = 0; k < 4; ++k) A0[d][k] = A1[d][k] = A2[d][k] = 0.0f;

#pragma unroll 1
  for (int R = y0; R <= r_last; ++R) {
    const int t = R - r_first;
    __syncwarp();
    if (lane == 0 && R + 1 <= r_last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(R + 1);
    }
    mbar_wait(&full[t % RING], (t / RING) & 1);

    const float* rowR = ring + (t % RING) * ROWF;
    const float* row1 = ring + ((t + RING - 1) % RING) * ROWF;
    const float* row2 = ring + ((t + RING - 2) % RING) * ROWF;
    if (R >= y1) {
      if (R < ny) {
#pragma unroll
        for (int d = 0; d < 3; ++d)
          comp_pass<ALPHA1, false, true>(f, rowR, row1, row2, lane, mL, mRt, 1.f, 1.f, 1.f,
                                         A0[d], A1[d], A2[d], d);
      }
    } else if (R >= 2) {
#pragma unroll
      for (int d = 0; d < 3; ++d)
        comp_pass<ALPHA1, false, false>(f, rowR, row1, row2, lane, mL, mRt, 1.f, 1.f, 1.f, A0[d],
                                        A1[d], A2[d], d);
    } else {
      const float m1 = R >= 1 ? 1.f : 0.f;
#pragma unroll
      for (int d = 0; d < 3; ++d)
        comp_pass<ALPHA1, true, false>(f, rowR, row1, row2, lane, mL, mRt, 1.f, m1, 0.f, A0[d],
                                       A1[d], A2[d], d);
    }

    // row R-2 is complete: plug, integrate, collide, pin, store
    const int Rf = R - 2;
    if (Rf >= y0 && Rf < y1 && lane_live) {
      float xs[3][4], vs[3][4];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        load4(row2 + d * BOXW, lane, xs[d]);
        load4(row2 + (3 + d) * BOXW, lane, vs[d]);
      }
      float xo[3][4], vo[3][4];
      if (simple) {
        // add_plug_impulse gravity/drag + advance without colliders, IEEE-exact like PARITY
#pragma unroll
        for (int k = 0; k < 4; ++k) {
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            float imp = A0[d][k];
            if (cc.plug_gravity) imp = __fadd_rn(imp, cc.dv[d]);
            if (cc.plug_drag) imp = __fsub_rn(imp, __fmul_rn(vs[d][k], cc.drag_c));
            const float vv = __fadd_rn(vs[d][k], imp);
            vo[d][k] = vv;
            xo[d][k] = __fadd_rn(xs[d][k], __fmul_rn(vv, cc.dt));
          }
        }
        if (cc.n_pins > 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t gnode = static_cast<int64_t>(Rf) * nx + ix0 + k;
            const int64_t w = cc.pin_word0 + (gnode >> 5);
            const uint32_t bits = __ldg(a.pin_bits + w);
            const uint32_t bit = 1u << (gnode & 31);
            if (bits & bit) {
              const int64_t slot = cc.anchor0 + __ldg(a.pin_rank + w) + __popc(bits & (bit - 1u));
#pragma unroll
              for (int d = 0; d < 3; ++d) {
                vo[d][k] = cc.pin_u[d];
                xo[d][k] = __fadd_rn(__ldg(a.pin_anchors + 3 * slot + d),
                                     __fmul_rn(cc.pin_u[d], t_next));
              }
            }
          }
        }
        if (a.health) {
          bool fin_imp = true, fin = true;
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              fin_imp = fin_imp && isfinite(A0[d][k]);
              fin = fin && isfinite(xo[d][k]) && isfinite(vo[d][k]);
            }
          if (!fin_imp) {
            for (int k = 0; k < 4; ++k)
              if (!(isfinite(A0[0][k]) && isfinite(A0[1][k]) && isfinite(A0[2][k]))) {
                const unsigned long long key = (static_cast<unsigned long long>(a.k + 1) << 32) |
                                               static_cast<unsigned long long>(Rf * nx + ix0 + k);
                atomicMin(&a.health[b].impulse_key, key);
                break;
              }
          }
          if (!fin) atomicMin(&a.health[b].state_frame, a.k + 1);
        }
        float* o = out_b + static_cast<int64_t>(Rf - a.g0) * a.pitch + ix0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          *reinterpret_cast<float4*>(o + d * a.plane_stride) =
              make_float4(xo[d][0], xo[d][1], xo[d][2], xo[d][3]);
          *reinterpret_cast<float4*>(o + (3 + d) * a.plane_stride) =
              make_float4(vo[d][0], vo[d][1], vo[d][2], vo[d][3]);
        }
      } else {
        // colliders / pressure / mask: one node at a time (compact code, same IEEE-exact chain)
        const float* rs = ring + ((t + RING - 3) % RING) * ROWF;  // row Rf-1
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < 4; ++k) scratch[lane][d * 4 + k] = A0[d][k];  // own row only
        float* o = out_b + static_cast<int64_t>(Rf - a.g0) * a.pitch;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const int ix = ix0 + k;
          const int j = FW * lane + 4 + k;
          const int64_t gnode = static_cast<int64_t>(Rf) * nx + ix;
          float px[3], pv[3], imp[3], po[3], qo[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            px[d] = row2[d * BOXW + j];
            pv[d] = row2[(3 + d) * BOXW + j];
            imp[d] = scratch[lane][d * 4 + k];
          }
          if (a.health && !(isfinite(imp[0]) && isfinite(imp[1]) && isfinite(imp[2]))) {
            const unsigned long long key = (static_cast<unsigned long long>(a.k + 1) << 32) |
                                           static_cast<unsigned long long>(gnode);
            atomicMin(&a.health[b].impulse_key, key);
          }
          if (cc.plug_pressure) {
            const bool interior = ix >= 1 && ix <= nx - 2 && Rf >= 1 && Rf <= ny - 2;
            float e[3], n[3], w[3], sv[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              e[d] = __fsub_rn(px[d], row2[d * BOXW + j + 1]);
              n[d] = __fsub_rn(px[d], row1[d * BOXW + j]);
              w[d] = __fsub_rn(px[d], row2[d * BOXW + j - 1]);
              sv[d] = __fsub_rn(px[d], rs[d * BOXW + j]);
            }
            pressure_plug(cc, interior, e, n, w, sv, imp);
          }
          plug_tail(cc, pv, imp);
          uint8_t mk;
          advance_node(a, cc, gnode, px, pv, imp, po, qo, mk);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            o[d * a.plane_stride + ix] = po[d];
            o[(3 + d) * a.plane_stride + ix] = qo[d];
          }
          if (a.constrained) a.constrained[b * nodes + gnode] = mk;
          if (a.health && !(isfinite(po[0]) && isfinite(po[1]) && isfinite(po[2]) &&
                            isfinite(qo[0]) && isfinite(qo[1]) && isfinite(qo[2])))
            atomicMin(&a.health[b].state_frame, a.k + 1);
        }
      }
    }
    // rotate accumulator rows
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        A0[d][k] = A1[d][k];
        A1[d][k] = A2[d][k];
      }
  }
}

}  // namespace

FastNet make_fast_net(const NetConst<float>& n) {
  FastNet f{};
  for (int c = 0; c < kChannels; ++c) {
    const float g = n.gain[c];
    f.wl[c] = g * n.wl[c];
    f.wn[c] = g * n.wn[c];
    f.wd[c] = (g * g) * n.wd[c];
    f.nwl[c] = -f.wl[c];
    f.nwn[c] = -f.wn[c];
    f.alpha[c] = n.alpha * (g * g);
  }
  for (int d = 0; d < 3; ++d) f.b[d] = n.b[d];
  f.wv = n.wv;
  f.alpha1 = 1;
  for (int c = 0; c < kChannels; ++c)
    if (f.alpha[c] != 1.0f) f.alpha1 = 0;
  return f;
}

bool fast_supported(const NetConst<float>& net, int nx) {
  if (nx % 4 != 0) return false;  // the strip column masks assume whole float4 columns
  static const int neg[kChannels] = {2, 3, 0, 1, 6, 7, 4, 5, 10, 11, 8, 9};
  for (int c = 0; c < kChannels; ++c)
    if (net.gain[c] != net.gain[neg[c]]) return false;
  return true;
}

size_t fast_smem_bytes() { return sizeof(float) * RING * ROWF; }

FastPlan plan_fast(int nx, int rows, int batch, int device) {
  FastPlan p{};
  p.n_strips = (nx + STRIP - 1) / STRIP;
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t smem = fast_smem_bytes();
  cudaFuncSetAttribute(fast_step_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaFuncSetAttribute(fast_step_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fast_step_kernel<true>, 32, smem);
  if (occ < 1) occ = 1;
  const int64_t slots = static_cast<int64_t>(sms) * occ;
  const int64_t columns = static_cast<int64_t>(batch) * p.n_strips;
  // choose the number of row segments maximising wave efficiency, discounting the ~0.6-row
  // warm-up each segment pays, with segments of at least 8 rows
  double best = -1.0;
  int best_segs = 1;
  const int max_segs = std::max(1, rows / 8);
  for (int segs = 1; segs <= max_segs && segs <= 4096; ++segs) {
    const int seg_rows = (rows + segs - 1) / segs;
    const int real_segs = (rows + seg_rows - 1) / seg_rows;
    const int64_t units = columns * real_segs;
    const int64_t waves = (units + slots - 1) / slots;
    const double fill = static_cast<double>(units) / static_cast<double>(waves * slots);
    const double work = static_cast<double>(rows) / (static_cast<double>(real_segs) * seg_rows);
    const double warm = static_cast<double>(seg_rows) / (seg_rows + 0.6);
    const double eff = fill * work * warm;
    if (eff > best + 1e-9) {
      best = eff;
      best_segs = real_segs;
    }
  }
  p.seg_rows = (rows + best_segs - 1) / best_segs;
  p.n_segs = (rows + p.seg_rows - 1) / p.seg_rows;
  p.units = columns * p.n_segs;
  p.smem = smem;
  return p;
}

cudaError_t launch_fast(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tmap,
                        const FastPlan& p, cudaStream_t stream) {
  const int rows = a.u1 - a.u0;
  if (rows <= 0 || a.batch <= 0) return cudaSuccess;
  if (f.alpha1)
    fast_step_kernel<true><<<static_cast<unsigned>(p.units), 32, p.smem, stream>>>(
        *tmap, a, f, p.n_strips, p.seg_rows, p.n_segs);
  else
    fast_step_kernel<false><<<static_cast<unsigned>(p.units), 32, p.smem, stream>>>(
        *tmap, a, f, p.n_strips, p.seg_rows, p.n_segs);
  return cudaGetLastError();
}

}  // namespace scb
