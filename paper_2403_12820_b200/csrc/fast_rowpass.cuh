// FAST-mode row pass shared by the streaming step kernel (fast_kernels.cu) and the wavefront
// temporal-blocking kernel (wave_kernels.cu): staged-row layout, lane windows, the edge-shared
// cell evaluation of one row of a 128-column strip (reference kernels.hpp:265-282, restated
// with one ISRU per undirected edge), and the per-lane finish arithmetic. Both kernels call
// exactly these functions, so their per-step results are bit-identical.
#pragma once

#include <cuda.h>

#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {
namespace fastrow {

constexpr int FW = 4;              // columns per lane
constexpr int STRIP = 32 * FW;     // columns per warp
constexpr int BOXW = STRIP + 8;    // staged columns x0-4 .. x0+131 (2-column halo + alignment)
// staged rows: R-3 .. R+1 (RING = 5, when some cloth plugs pressure, whose finish reads row
// R-3) or R-2 .. R+1 (RING = 4); one row of prefetch
// ring slot (floats): [x.xy: BOXW pairs][v.xy: BOXW pairs][x.z: BOXW][v.z: BOXW]
constexpr int XY_X = 0, XY_V = 2 * BOXW, Z_X = 4 * BOXW, Z_V = 5 * BOXW;
constexpr int XY_BYTES = 4 * BOXW * 4;                 // first TMA box
constexpr int ROW_BYTES = 6 * BOXW * 4;                // both boxes
constexpr int ROWF = ((ROW_BYTES + 127) / 128) * 32;   // slot stride in floats (128 B aligned)
static_assert((XY_BYTES % 128) == 0, "z box must start 128-byte aligned");

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

// try_wait suspend-time hint: a warp whose TMA row has not landed sleeps (NANOSLEEP.SYNCS, woken
// by the barrier) instead of spinning on issue slots its SM's other warps could use
constexpr uint32_t kSuspendHintNs = 1000000;

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(kSuspendHintNs)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(float* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// one lane of the (converged) warp, without reading %tid (no S2R in the row loop)
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}

// rsqrt without the denormal fix-up rsqrtf() carries under -ftz=false: q = 1 + a dx^2 >= 1.
__device__ __forceinline__ float rsqrt_q(float q) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return r;
}

// ---- f32 / packed f32x2 arithmetic with scalar-broadcast weights ---------------------------
__device__ __forceinline__ float vsub(float a, float b) { return a - b; }
__device__ __forceinline__ float2 vsub(float2 a, float2 b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
__device__ __forceinline__ float vmul(float a, float b) { return a * b; }
__device__ __forceinline__ float2 vmul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float vscale(float a, float m) { return a * m; }
__device__ __forceinline__ float2 vscale(float2 a, float m) {
  return __fmul2_rn(a, make_float2(m, m));
}
__device__ __forceinline__ float vfma(float a, float w, float c) { return fmaf(a, w, c); }
__device__ __forceinline__ float2 vfma(float2 a, float w, float2 c) {
  return __ffma2_rn(a, make_float2(w, w), c);
}
__device__ __forceinline__ float vfmav(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ float2 vfmav(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// edge masks as bit patterns (0 or ~0): a LOP3 on the ALU pipe instead of an FMUL by 0 / 1
__device__ __forceinline__ float vand(float a, uint32_t k) {
  return __uint_as_float(__float_as_uint(a) & k);
}
__device__ __forceinline__ float2 vand(float2 a, uint32_t k) {
  return make_float2(vand(a.x, k), vand(a.y, k));
}
__device__ __forceinline__ float vsplat(float w) { return w; }
__device__ __forceinline__ float2 vsplat2(float w) { return make_float2(w, w); }
__device__ __forceinline__ float vq(float dx) { return fmaf(dx, dx, 1.0f); }
__device__ __forceinline__ float2 vq(float2 dx) { return __ffma2_rn(dx, dx, make_float2(1.f, 1.f)); }
__device__ __forceinline__ float vqa(float dx, float al) { return fmaf(dx * al, dx, 1.0f); }
__device__ __forceinline__ float2 vqa(float2 dx, float al) {
  return __ffma2_rn(__fmul2_rn(dx, make_float2(al, al)), dx, make_float2(1.f, 1.f));
}
__device__ __forceinline__ float vrsq(float q) { return rsqrt_q(q); }
__device__ __forceinline__ float2 vrsq(float2 q) { return make_float2(rsqrt_q(q.x), rsqrt_q(q.y)); }

// Edge contribution to its origin node a (channel ca) and far node b (channel cb = -ca):
//   a: acc += dx*wL'_ca + s*(wN'_ca + dv*wD'_ca)
//   b: acc += dx*(-wL'_cb) + s*(dv*wD'_cb - wN'_cb)
// with dx = x_a - x_b, dv = v_a - v_b, s = dx * r, r = rsqrt(1 + alpha'_c dx^2) and the gains
// folded into the primed weights (wL' = g wL, wN' = g wN, wD' = g^2 wD, alpha' = alpha g^2).
// Evaluated folded, acc += dx * (wL' + r * (wN' + dv wD')): three FMAs per endpoint and no
// shared s = dx * r product. Invalid edges (an endpoint outside the grid) arrive with dx = 0
// and contribute exactly 0 whatever dv is (w stays finite), so only dx is masked.
template <bool ALPHA1, bool PA, bool PB, typename V>
__device__ __forceinline__ void edge(const FastNet& f, int ca, int cb, V dx, V dv, V& acc_a,
                                     V& acc_b) {
  const V q = ALPHA1 ? vq(dx) : vqa(dx, f.alpha[ca]);
  const V r = vrsq(q);
  if (PA) {
    const V t = vfma(dv, f.wd[ca], [&] {
      if constexpr (sizeof(V) == 8) return vsplat2(f.wn[ca]); else return vsplat(f.wn[ca]);
    }());
    const V w = vfmav(r, t, [&] {
      if constexpr (sizeof(V) == 8) return vsplat2(f.wl[ca]); else return vsplat(f.wl[ca]);
    }());
    acc_a = vfmav(dx, w, acc_a);
  }
  if (PB) {
    const V t = vfma(dv, f.wd[cb], [&] {
      if constexpr (sizeof(V) == 8) return vsplat2(f.nwn[cb]); else return vsplat(f.nwn[cb]);
    }());
    const V w = vfmav(r, t, [&] {
      if constexpr (sizeof(V) == 8) return vsplat2(f.nwl[cb]); else return vsplat(f.nwl[cb]);
    }());
    acc_b = vfmav(dx, w, acc_b);
  }
}

// Lane windows of a staged row: columns ix0-2 .. ix0+5 <-> box column 4*lane+2 .. 4*lane+9,
// columns ix0 .. ix0+3 <-> 4*lane+4 .. 4*lane+7. The (x, y) planes carry the xy_col swizzle
// (sc_device.cuh): box column j of a strip (x0 a multiple of 128, box from x0-4) sits at
// position xsw(j); a lane's four 2-column pieces are at xsw(4 lane + 2 + 2q), q = 0..3.
__device__ __forceinline__ int xsw(int j) { return j ^ (((j + 28) >> 3) & 2); }
// z planes: with the z_col swizzle (ZS, sc_device.cuh) box column j (global x0 - 4 + j) sits at
// zsw(j) and a lane reads its window as 8-byte pieces at zsw(4 lane + 2 + 2q), conflict-free per
// half-warp; on the plain layout it reads its own group in one 16-byte load
template <bool ZS>
__device__ __forceinline__ int zsw(int j) {
  return ZS ? j ^ (((j + 124) >> 4) & 2) : j;
}
template <bool ZS>
__device__ __forceinline__ float2 zpiece(const float* zplane, int j) {
  return *reinterpret_cast<const float2*>(zplane + zsw<ZS>(j));
}
// a lane's 4 z values in the stored order of its group (halves swapped when ZS and column bit 5)
template <bool ZS>
__device__ __forceinline__ float4 zgroup(int ix0, float a, float b, float c, float d) {
  return (ZS && ((ix0 >> 5) & 1)) ? make_float4(c, d, a, b) : make_float4(a, b, c, d);
}
template <bool ZS>
__device__ __forceinline__ void win4z(const float* zplane, int lane, float* o) {
  if constexpr (ZS) {
    const float2 a = zpiece<ZS>(zplane, FW * lane + 4), b = zpiece<ZS>(zplane, FW * lane + 6);
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
  } else {
    const float4 m = *reinterpret_cast<const float4*>(zplane + FW * lane + 4);
    o[0] = m.x; o[1] = m.y; o[2] = m.z; o[3] = m.w;
  }
}
__device__ __forceinline__ void win8(const float* xyplane, int lane, float2* o) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 m = *reinterpret_cast<const float4*>(xyplane + 2 * xsw(FW * lane + 2 + 2 * q));
    o[2 * q] = make_float2(m.x, m.y);
    o[2 * q + 1] = make_float2(m.z, m.w);
  }
}
__device__ __forceinline__ void win4(const float* xyplane, int lane, float2* o) {
  const float4 a = *reinterpret_cast<const float4*>(xyplane + 2 * xsw(FW * lane + 4));
  const float4 b = *reinterpret_cast<const float4*>(xyplane + 2 * xsw(FW * lane + 6));
  o[0] = make_float2(a.x, a.y); o[1] = make_float2(a.z, a.w);
  o[2] = make_float2(b.x, b.y); o[3] = make_float2(b.z, b.w);
}

// All edges of one component group (V = float2: x,y packed; V = float: z) whose upper
// endpoint lies on row R, pushed into the accumulators of rows R-2 (A0), R-1 (A1), R (A2).
// mL / mRt zero the edges that leave the grid through a strip's boundary lane; GENERAL applies
// the row masks of the first two rows of the cloth; TAIL (rows R >= y1, not owned) keeps only
// the pushes into rows R-1 and R-2.
template <bool ALPHA1, bool GENERAL, int TAIL, typename V>
__device__ __forceinline__ void comp_pass(const FastNet& f, const float* xR, const float* vR,
                                          const float* x1p, const float* v1p, const float* x2p,
                                          const float* v2p, int lane, uint32_t mL, uint32_t mRt,
                                          float m1, float m2, V (&A0)[4], V (&A1)[4], V (&A2)[4],
                                          V bias) {
  // windows are loaded right before their edge groups (rows R, R-2, R-1 in that order) so the
  // live register set stays small: R's window, then at most one of R-2 / R-1 beside it
  V xr[8], vr[8], x1[8], v1[8], x2[4], v2[4];
  V dummy{};
  if (TAIL == 2) {  // R = y1 + 1: row R-1 = y1 is not owned either, only N2 pushes into R-2
    win4(xR, lane, xr);
    win4(vR, lane, vr);
    win4(x2p, lane, x2);
    win4(v2p, lane, v2);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      edge<ALPHA1, true, false>(f, 9, 11, vsub(x2[k], xr[k]), vsub(v2[k], vr[k]), A0[k], dummy);
    return;
  }
  win8(xR, lane, xr);
  win8(vR, lane, vr);
  if (TAIL) {
    win8(x1p, lane, x1);
    win8(v1p, lane, v1);
    win4(x2p, lane, x2);
    win4(v2p, lane, v2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      edge<ALPHA1, true, false>(f, 1, 3, vsub(x1[k + 2], xr[k + 2]), vsub(v1[k + 2], vr[k + 2]),
                                A1[k], dummy);
      edge<ALPHA1, true, false>(f, 9, 11, vsub(x2[k], xr[k + 2]), vsub(v2[k], vr[k + 2]), A0[k],
                                dummy);
    }
#pragma unroll
    for (int e = 1; e < 5; ++e) {
      V dx = vsub(x1[e + 1], xr[e + 2]), dv = vsub(v1[e + 1], vr[e + 2]);
      if (e == 4) {
        dx = vand(dx, mRt);
      }
      edge<ALPHA1, true, false>(f, 4, 6, dx, dv, A1[e - 1], dummy);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      V dx = vsub(x1[e + 2], xr[e + 1]), dv = vsub(v1[e + 2], vr[e + 1]);
      if (e == 0) {
        dx = vand(dx, mL);
      }
      edge<ALPHA1, true, false>(f, 5, 7, dx, dv, A1[e], dummy);
    }
    return;
  }
  // init row R: b + v*wV
#pragma unroll
  for (int k = 0; k < 4; ++k) A2[k] = vfma(vr[k + 2], f.wv, bias);

  // E edges in row R: a = col ix0-1+e (j = e+1), b = col ix0+e (j = e+2)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    V dx = vsub(xr[e + 1], xr[e + 2]), dv = vsub(vr[e + 1], vr[e + 2]);
    if (e == 0 || e == 4) {
      dx = vand(dx, e == 0 ? mL : mRt);
    }
    if (e == 0) edge<ALPHA1, false, true>(f, 0, 2, dx, dv, dummy, A2[0]);
    else if (e == 4) edge<ALPHA1, true, false>(f, 0, 2, dx, dv, A2[3], dummy);
    else edge<ALPHA1, true, true>(f, 0, 2, dx, dv, A2[e - 1 < 0 ? 0 : e - 1], A2[e > 3 ? 3 : e]);
  }
  // E2 edges in row R: a = col ix0-2+e (j = e), b = col ix0+e (j = e+2)
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    V dx = vsub(xr[e], xr[e + 2]), dv = vsub(vr[e], vr[e + 2]);
    if (e <= 1 || e >= 4) {
      dx = vand(dx, e <= 1 ? mL : mRt);
    }
    if (e <= 1) edge<ALPHA1, false, true>(f, 8, 10, dx, dv, dummy, A2[e]);
    else if (e >= 4) edge<ALPHA1, true, false>(f, 8, 10, dx, dv, A2[e - 2], dummy);
    else edge<ALPHA1, true, true>(f, 8, 10, dx, dv, A2[e - 2], A2[e]);
  }
  // N2 edges (R-2 -> R), owned columns
  win4(x2p, lane, x2);
  win4(v2p, lane, v2);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    V dx2 = vsub(x2[k], xr[k + 2]), dv2 = vsub(v2[k], vr[k + 2]);
    if (GENERAL) {
      dx2 = vscale(dx2, m2);
    }
    edge<ALPHA1, true, true>(f, 9, 11, dx2, dv2, A0[k], A2[k]);
  }
  // N edges (R-1 -> R), owned columns
  win8(x1p, lane, x1);
  win8(v1p, lane, v1);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    V dx = vsub(x1[k + 2], xr[k + 2]), dv = vsub(v1[k + 2], vr[k + 2]);
    if (GENERAL) {
      dx = vscale(dx, m1);
    }
    edge<ALPHA1, true, true>(f, 1, 3, dx, dv, A1[k], A2[k]);
  }
  // NE edges: a = (ix0-1+e, R-1) (j = e+1), b = (ix0+e, R) (j = e+2)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    V dx = vsub(x1[e + 1], xr[e + 2]), dv = vsub(v1[e + 1], vr[e + 2]);
    if (GENERAL || e == 0 || e == 4) {
      if (e == 0 || e == 4) dx = vand(dx, e == 0 ? mL : mRt);
      if (GENERAL) dx = vscale(dx, m1);
    }
    if (e == 0) edge<ALPHA1, false, true>(f, 4, 6, dx, dv, dummy, A2[0]);
    else if (e == 4) edge<ALPHA1, true, false>(f, 4, 6, dx, dv, A1[3], dummy);
    else edge<ALPHA1, true, true>(f, 4, 6, dx, dv, A1[e - 1 < 0 ? 0 : e - 1], A2[e > 3 ? 3 : e]);
  }
  // NW edges: a = (ix0+e, R-1) (j = e+2), b = (ix0+e-1, R) (j = e+1)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    V dx = vsub(x1[e + 2], xr[e + 1]), dv = vsub(v1[e + 2], vr[e + 1]);
    if (GENERAL || e == 0 || e == 4) {
      if (e == 0 || e == 4) dx = vand(dx, e == 0 ? mL : mRt);
      if (GENERAL) dx = vscale(dx, m1);
    }
    if (e == 0) edge<ALPHA1, true, false>(f, 5, 7, dx, dv, A1[0], dummy);
    else if (e == 4) edge<ALPHA1, false, true>(f, 5, 7, dx, dv, dummy, A2[3]);
    else edge<ALPHA1, true, true>(f, 5, 7, dx, dv, A1[e > 3 ? 3 : e], A2[e - 1 < 0 ? 0 : e - 1]);
  }
}

// z component of column k (0..3) of a pair-packed accumulator row
__device__ __forceinline__ float& zc(float2 (&a)[2], int k) { return (k & 1) ? a[k >> 1].y : a[k >> 1].x; }
__device__ __forceinline__ float zc(const float2 (&a)[2], int k) {
  return (k & 1) ? a[k >> 1].y : a[k >> 1].x;
}

// z windows as register pairs: columns ix0-2 .. ix0+5 (w8) and ix0 .. ix0+3 (w4)
template <bool ZS>
__device__ __forceinline__ void win8p(const float* zplane, int lane, float2* o) {
  if constexpr (ZS) {
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = zpiece<ZS>(zplane, FW * lane + 2 + 2 * q);
  } else {
    o[0] = *reinterpret_cast<const float2*>(zplane + FW * lane + 2);
    const float4 m = *reinterpret_cast<const float4*>(zplane + FW * lane + 4);
    o[1] = make_float2(m.x, m.y);
    o[2] = make_float2(m.z, m.w);
    o[3] = *reinterpret_cast<const float2*>(zplane + FW * lane + 8);
  }
}
template <bool ZS>
__device__ __forceinline__ void win4p(const float* zplane, int lane, float2* o) {
  if constexpr (ZS) {
    o[0] = zpiece<ZS>(zplane, FW * lane + 4);
    o[1] = zpiece<ZS>(zplane, FW * lane + 6);
  } else {
    const float4 m = *reinterpret_cast<const float4*>(zplane + FW * lane + 4);
    o[0] = make_float2(m.x, m.y);
    o[1] = make_float2(m.z, m.w);
  }
}
__device__ __forceinline__ float zw(const float2* w, int i) { return (i & 1) ? w[i >> 1].y : w[i >> 1].x; }

// comp_pass for z with adjacent columns packed where the edge geometry keeps register pairs
// aligned: E2 edges (offset 2) and the vertical N / N2 edges run two columns per FFMA2 / MUFU
// pair; E, NE, NW (odd offsets) stay scalar on the pair halves.
template <bool ALPHA1, bool GENERAL, int TAIL, bool ZS>
__device__ __forceinline__ void comp_pass_z(const FastNet& f, const float* xR, const float* vR,
                                            const float* x1p, const float* v1p, const float* x2p,
                                            const float* v2p, int lane, uint32_t mL, uint32_t mRt,
                                            float m1, float m2, float2 (&A0)[2], float2 (&A1)[2],
                                            float2 (&A2)[2], float bias) {
  float2 xr[4], vr[4], x1[4], v1[4], x2[2], v2[2];
  float dummy = 0.f;
  float2 dummy2{};
  if (TAIL == 2) {  // N2 a-sides only (packed)
    win4p<ZS>(xR, lane, xr);
    win4p<ZS>(vR, lane, vr);
    win4p<ZS>(x2p, lane, x2);
    win4p<ZS>(v2p, lane, v2);
#pragma unroll
    for (int j = 0; j < 2; ++j)
      edge<ALPHA1, true, false>(f, 9, 11, vsub(x2[j], xr[j]), vsub(v2[j], vr[j]), A0[j], dummy2);
    return;
  }
  win8p<ZS>(xR, lane, xr);
  win8p<ZS>(vR, lane, vr);
  if (TAIL) {
    win8p<ZS>(x1p, lane, x1);
    win8p<ZS>(v1p, lane, v1);
    win4p<ZS>(x2p, lane, x2);
    win4p<ZS>(v2p, lane, v2);
    // N / N2 a-sides (packed), NE / NW a-sides (scalar)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      edge<ALPHA1, true, false>(f, 1, 3, vsub(x1[j + 1], xr[j + 1]), vsub(v1[j + 1], vr[j + 1]),
                                A1[j], dummy2);
      edge<ALPHA1, true, false>(f, 9, 11, vsub(x2[j], xr[j + 1]), vsub(v2[j], vr[j + 1]), A0[j],
                                dummy2);
    }
#pragma unroll
    for (int e = 1; e < 5; ++e) {
      float dx = zw(x1, e + 1) - zw(xr, e + 2), dv = zw(v1, e + 1) - zw(vr, e + 2);
      if (e == 4) {
        dx = vand(dx, mRt);
      }
      edge<ALPHA1, true, false>(f, 4, 6, dx, dv, zc(A1, e - 1), dummy);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float dx = zw(x1, e + 2) - zw(xr, e + 1), dv = zw(v1, e + 2) - zw(vr, e + 1);
      if (e == 0) {
        dx = vand(dx, mL);
      }
      edge<ALPHA1, true, false>(f, 5, 7, dx, dv, zc(A1, e), dummy);
    }
    return;
  }
  // init row R: b + v*wV
#pragma unroll
  for (int j = 0; j < 2; ++j) A2[j] = vfma(vr[j + 1], f.wv, make_float2(bias, bias));

  // E edges in row R (scalar): a = col ix0-1+e, b = col ix0+e
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = zw(xr, e + 1) - zw(xr, e + 2), dv = zw(vr, e + 1) - zw(vr, e + 2);
    if (e == 0 || e == 4) dx = vand(dx, e == 0 ? mL : mRt);
    if (e == 0) edge<ALPHA1, false, true>(f, 0, 2, dx, dv, dummy, zc(A2, 0));
    else if (e == 4) edge<ALPHA1, true, false>(f, 0, 2, dx, dv, zc(A2, 3), dummy);
    else edge<ALPHA1, true, true>(f, 0, 2, dx, dv, zc(A2, e - 1), zc(A2, e));
  }
  // E2 edges in row R, packed: pair j = edges e = 2j, 2j+1 (a = cols ix0-2+e, b = ix0+e)
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float2 dx = vsub(xr[j], xr[j + 1]), dv = vsub(vr[j], vr[j + 1]);
    if (j == 0 || j == 2) {
      dx = vand(dx, j == 0 ? mL : mRt);
    }
    if (j == 0) edge<ALPHA1, false, true>(f, 8, 10, dx, dv, dummy2, A2[0]);
    else if (j == 2) edge<ALPHA1, true, false>(f, 8, 10, dx, dv, A2[1], dummy2);
    else edge<ALPHA1, true, true>(f, 8, 10, dx, dv, A2[0], A2[1]);
  }
  // N2 edges (R-2 -> R), then N edges (R-1 -> R), packed column pairs
  win4p<ZS>(x2p, lane, x2);
  win4p<ZS>(v2p, lane, v2);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float2 dx2 = vsub(x2[j], xr[j + 1]), dv2 = vsub(v2[j], vr[j + 1]);
    if (GENERAL) {
      dx2 = vscale(dx2, m2);
    }
    edge<ALPHA1, true, true>(f, 9, 11, dx2, dv2, A0[j], A2[j]);
  }
  win8p<ZS>(x1p, lane, x1);
  win8p<ZS>(v1p, lane, v1);
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    float2 dx = vsub(x1[j + 1], xr[j + 1]), dv = vsub(v1[j + 1], vr[j + 1]);
    if (GENERAL) {
      dx = vscale(dx, m1);
    }
    edge<ALPHA1, true, true>(f, 1, 3, dx, dv, A1[j], A2[j]);
  }
  // NE edges (scalar): a = (ix0-1+e, R-1), b = (ix0+e, R)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = zw(x1, e + 1) - zw(xr, e + 2), dv = zw(v1, e + 1) - zw(vr, e + 2);
    if (GENERAL || e == 0 || e == 4) {
      if (e == 0 || e == 4) dx = vand(dx, e == 0 ? mL : mRt);
      if (GENERAL) dx *= m1;
    }
    if (e == 0) edge<ALPHA1, false, true>(f, 4, 6, dx, dv, dummy, zc(A2, 0));
    else if (e == 4) edge<ALPHA1, true, false>(f, 4, 6, dx, dv, zc(A1, 3), dummy);
    else edge<ALPHA1, true, true>(f, 4, 6, dx, dv, zc(A1, e - 1), zc(A2, e));
  }
  // NW edges (scalar): a = (ix0+e, R-1), b = (ix0+e-1, R)
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    float dx = zw(x1, e + 2) - zw(xr, e + 1), dv = zw(v1, e + 2) - zw(vr, e + 1);
    if (GENERAL || e == 0 || e == 4) {
      if (e == 0 || e == 4) dx = vand(dx, e == 0 ? mL : mRt);
      if (GENERAL) dx *= m1;
    }
    if (e == 0) edge<ALPHA1, true, false>(f, 5, 7, dx, dv, zc(A1, 0), dummy);
    else if (e == 4) edge<ALPHA1, false, true>(f, 5, 7, dx, dv, dummy, zc(A2, 3));
    else edge<ALPHA1, true, true>(f, 5, 7, dx, dv, zc(A1, e), zc(A2, e - 1));
  }
}

template <bool ALPHA1, bool GENERAL, int TAIL, bool ZS>
__device__ __forceinline__ void row_pass(const FastNet& f, const float* rowR, const float* row1,
                                         const float* row2, int lane, uint32_t mL, uint32_t mRt,
                                         float m1, float m2, float2 (&P0)[4], float2 (&P1)[4],
                                         float2 (&P2)[4], float2 (&Z0)[2], float2 (&Z1)[2],
                                         float2 (&Z2)[2]) {
  comp_pass<ALPHA1, GENERAL, TAIL, float2>(f, rowR + XY_X, rowR + XY_V, row1 + XY_X, row1 + XY_V,
                                           row2 + XY_X, row2 + XY_V, lane, mL, mRt, m1, m2, P0,
                                           P1, P2, make_float2(f.b[0], f.b[1]));
  comp_pass_z<ALPHA1, GENERAL, TAIL, ZS>(f, rowR + Z_X, rowR + Z_V, row1 + Z_X, row1 + Z_V,
                                     row2 + Z_X, row2 + Z_V, lane, mL, mRt, m1, m2, Z0, Z1, Z2,
                                     f.b[2]);
}

// component d of x (X = true) or v at box column j of a ring slot
template <bool ZS>
__device__ __forceinline__ float slot_val(const float* slot, bool X, int d, int j) {
  return d < 2 ? slot[(X ? XY_X : XY_V) + 2 * xsw(j) + d] : slot[(X ? Z_X : Z_V) + zsw<ZS>(j)];
}


// ---- finish of one completed row (row R-2 after the pass over row R): per lane, its 4 nodes --
// xs/vs/xz/vz: the old state of the lane's 4 nodes; P0/Z0: their cell impulses. k: step index
// (t_next = (k+1) dt, health keys), b: cloth.

// Lane's 4 old nodes from a staged row.
template <bool ZS>
__device__ __forceinline__ void finish_inputs(const float* row2, int lane, float2 (&xs)[4],
                                              float2 (&vs)[4], float (&xz)[4], float (&vz)[4]) {
  win4(row2 + XY_X, lane, xs);
  win4(row2 + XY_V, lane, vs);
  win4z<ZS>(row2 + Z_X, lane, xz);
  win4z<ZS>(row2 + Z_V, lane, vz);
}

// add_plug_impulse gravity/drag + advance without colliders (no mask, no contact decision
// depends on it): FMA-contracted and x,y packed — part of FAST mode's tolerance bar. Pins re-set
// with the reference's IEEE expression (kernels.hpp:245-251).
__device__ __forceinline__ void finish_simple(const StepArgs<float>& a, const ClothConst<float>& cc,
                                              int Rf, int ix0, float t_next,
                                              const float2 (&P0)[4], const float2 (&Z0)[2],
                                              const float2 (&xs)[4], const float2 (&vs)[4],
                                              const float (&xz)[4], const float (&vz)[4],
                                              float (&xo)[3][4], float (&vo)[3][4]) {
  const float dv_eff[3] = {cc.fin[0], cc.fin[1], cc.fin[2]};  // plugged gravity impulse or 0
  const float drag_eff = cc.fin[3];                            // plugged drag coefficient or 0
  const float2 dvxy = make_float2(dv_eff[0], dv_eff[1]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 imp = __fadd2_rn(P0[k], dvxy);
    imp = __ffma2_rn(vs[k], make_float2(-drag_eff, -drag_eff), imp);
    const float2 vv = __fadd2_rn(vs[k], imp);
    const float2 xx = __ffma2_rn(vv, make_float2(cc.dt, cc.dt), xs[k]);
    const float iz = fmaf(vz[k], -drag_eff, zc(Z0, k) + dv_eff[2]);
    const float vvz = vz[k] + iz;
    vo[0][k] = vv.x;
    vo[1][k] = vv.y;
    vo[2][k] = vvz;
    xo[0][k] = xx.x;
    xo[1][k] = xx.y;
    xo[2][k] = fmaf(vvz, cc.dt, xz[k]);
  }
  if (cc.n_pins > 0 && Rf >= cc.pin_row_lo && Rf <= cc.pin_row_hi) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t gnode = static_cast<int64_t>(Rf) * a.nx + ix0 + k;
      const int64_t w = cc.pin_word0 + (gnode >> 5);
      const uint32_t bits = __ldg(a.pin_bits + w);
      const uint32_t bit = 1u << (gnode & 31);
      if (bits & bit) {
        const int64_t slot = cc.anchor0 + __ldg(a.pin_rank + w) + __popc(bits & (bit - 1u));
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          vo[d][k] = cc.pin_u[d];
          xo[d][k] = __fadd_rn(__ldg(a.pin_anchors + 3 * slot + d), __fmul_rn(cc.pin_u[d], t_next));
        }
      }
    }
  }
}

// non-finite tracking of the simple finish (net.cpp:139-140, eval.cpp:98-99)
__device__ __forceinline__ void health_simple(Health* health, int b, int k, int Rf, int nx,
                                              int ix0, const float2 (&P0)[4],
                                              const float2 (&Z0)[2], const float (&xo)[3][4],
                                              const float (&vo)[3][4]) {
  bool fin_imp = true, fin = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    fin_imp = fin_imp && isfinite(P0[q].x) && isfinite(P0[q].y) && isfinite(zc(Z0, q));
#pragma unroll
    for (int d = 0; d < 3; ++d) fin = fin && isfinite(xo[d][q]) && isfinite(vo[d][q]);
  }
  if (!fin_imp) {
    for (int q = 0; q < 4; ++q)
      if (!(isfinite(P0[q].x) && isfinite(P0[q].y) && isfinite(zc(Z0, q)))) {
        const unsigned long long key = (static_cast<unsigned long long>(k + 1) << 32) |
                                       static_cast<unsigned long long>(Rf * nx + ix0 + q);
        atomicMin(&health[b].impulse_key, key);
        break;
      }
  }
  if (!fin) atomicMin(&health[b].state_frame, k + 1);
}

// The simple finish's outputs in the stored (xy_col / z_col swizzled) order of the lane's group:
// oxy / ovxy point at the group's first (x,y) pair of x / v, oz / ovz at its first z.
template <bool ZS>
__device__ __forceinline__ void store_simple(float* oxy, float* ovxy, float* oz, float* ovz,
                                             int ix0, const float (&xo)[3][4],
                                             const float (&vo)[3][4]) {
  const int sw = (ix0 >> 3) & 2;  // xy_col: this lane's group stores its halves swapped
  *reinterpret_cast<float4*>(oxy + 2 * sw) = make_float4(xo[0][0], xo[1][0], xo[0][1], xo[1][1]);
  *reinterpret_cast<float4*>(oxy + 2 * (2 ^ sw)) =
      make_float4(xo[0][2], xo[1][2], xo[0][3], xo[1][3]);
  *reinterpret_cast<float4*>(ovxy + 2 * sw) = make_float4(vo[0][0], vo[1][0], vo[0][1], vo[1][1]);
  *reinterpret_cast<float4*>(ovxy + 2 * (2 ^ sw)) =
      make_float4(vo[0][2], vo[1][2], vo[0][3], vo[1][3]);
  *reinterpret_cast<float4*>(oz) = zgroup<ZS>(ix0, xo[2][0], xo[2][1], xo[2][2], xo[2][3]);
  *reinterpret_cast<float4*>(ovz) = zgroup<ZS>(ix0, vo[2][0], vo[2][1], vo[2][2], vo[2][3]);
}

// The general finish's outputs (node-major) in the stored order of the lane's group.
template <bool ZS>
__device__ __forceinline__ void store_general(float* oxy, float* ovxy, float* oz, float* ovz,
                                              int ix0, const float (&xo)[4][3],
                                              const float (&vo)[4][3]) {
  const int sw = (ix0 >> 3) & 2;  // xy_col swizzle of this lane's group
  *reinterpret_cast<float4*>(oxy + 2 * sw) = make_float4(xo[0][0], xo[0][1], xo[1][0], xo[1][1]);
  *reinterpret_cast<float4*>(oxy + 2 * (2 ^ sw)) =
      make_float4(xo[2][0], xo[2][1], xo[3][0], xo[3][1]);
  *reinterpret_cast<float4*>(ovxy + 2 * sw) = make_float4(vo[0][0], vo[0][1], vo[1][0], vo[1][1]);
  *reinterpret_cast<float4*>(ovxy + 2 * (2 ^ sw)) =
      make_float4(vo[2][0], vo[2][1], vo[3][0], vo[3][1]);
  *reinterpret_cast<float4*>(oz) = zgroup<ZS>(ix0, xo[0][2], xo[1][2], xo[2][2], xo[3][2]);
  *reinterpret_cast<float4*>(ovz) = zgroup<ZS>(ix0, vo[0][2], vo[1][2], vo[2][2], vo[3][2]);
}

// The first sphere and plane of a cloth, loaded once per cloth (unit / item) instead of once
// per finished row; further colliders are read from the tables as they come.
struct Colliders {
  SphereConst<float> s0;
  PlaneConst<float> p0;
};
__device__ __forceinline__ Colliders load_colliders(const StepArgs<float>& a,
                                                    const ClothConst<float>& cc) {
  Colliders c{};
  if (cc.n_spheres > 0) c.s0 = a.spheres[cc.sphere0];
  if (cc.n_planes > 0) c.p0 = a.planes[cc.plane0];
  return c;
}

// Colliders and/or the contact mask: the lane's 4 nodes together, each node through the same
// IEEE round-to-nearest sequence as advance_with_impulse (sc_device.cuh: plug_tail, the
// velocity-level response on the old positions, x' = x + v' dt, the position-level projection,
// the re-pin), so contact decisions and masks match PARITY. The x and y components run as
// packed f32x2 RN operations (__fadd2_rn / __fmul2_rn: per-lane IEEE results, never
// contracted), which gives the same bits as the scalar sequence at half the instructions.
// CS: the cloth's collider set — COLL_ANY (table loops), or the shapes the BASELINE configs use,
// COLL_PLANE1 (one plane, no sphere: config 5) and COLL_SPHERE1 (one sphere, no plane: config 3),
// compiled as straight-line code. Same operations in the same order either way.
// COLL_PLANE1F: one frictionless plane and no sphere, finished by finish_plane_f.
constexpr int COLL_ANY = 0, COLL_PLANE1 = 1, COLL_SPHERE1 = 2, COLL_PLANE1F = 3;

// Broad phase of the one-sphere finish: true when some node of the warp's row may be within
// `lim` of the sphere (strict: dist <= lim counts; else dist < lim). A node is provably outside
// when one coordinate alone is: the reference's distance is sqrt_rn of a round-to-nearest sum of
// squares, each partial sum >= any of its terms (rounding is monotonic) and sqrt_rn(fl(r^2)) =
// |r|, so |r_d| > lim implies dist > lim (and |r_d| >= lim implies dist >= lim) — the response
// (kernels.hpp:213-225 / 229-244) is then a no-op for every node of the row, bit for bit, and the
// warp skips it (a uniform branch). Non-finite coordinates compare false and take the full path.
__device__ __forceinline__ bool sphere_near(const SphereConst<float>& sp, float lim, bool strict,
                                            const float (&px)[4], const float (&py)[4],
                                            const float (&pz)[4]) {
  bool far = true;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float r0 = fabsf(__fsub_rn(px[q], sp.c[0])), r1 = fabsf(__fsub_rn(py[q], sp.c[1])),
                r2 = fabsf(__fsub_rn(pz[q], sp.c[2]));
    far = far && (strict ? (r0 > lim || r1 > lim || r2 > lim)
                         : (r0 >= lim || r1 >= lim || r2 >= lim));
  }
  return __ballot_sync(__activemask(), !far) != 0u;
}
template <int CS = COLL_ANY>
__device__ __forceinline__ void finish_general(const StepArgs<float>& a, const ClothConst<float>& cc,
                                               const Colliders& col, int b, int k, int Rf,
                                               int ix0, float t_next, const float2 (&P0)[4],
                                               const float2 (&Z0)[2], const float2 (&xs)[4],
                                               const float2 (&vs)[4], const float (&xz)[4],
                                               const float (&vz)[4], float (&xo)[4][3],
                                               float (&vo)[4][3], uint8_t (&mk)[4]) {
  const int nx = a.nx;
  if (a.health) {  // non-finite cell impulse: first (step, node) (net.cpp:139-140)
    for (int q = 0; q < 4; ++q)
      if (!(isfinite(P0[q].x) && isfinite(P0[q].y) && isfinite(zc(Z0, q)))) {
        const unsigned long long key = (static_cast<unsigned long long>(k + 1) << 32) |
                                       static_cast<unsigned long long>(Rf * nx + ix0 + q);
        atomicMin(&a.health[b].impulse_key, key);
        break;
      }
  }
  // add_plug_impulse tail (kernels.hpp:188-195): gravity, then drag
  float2 ixy[4];
  float iz[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    ixy[q] = P0[q];
    iz[q] = zc(Z0, q);
  }
  if (cc.plug_gravity) {
    const float2 g = make_float2(cc.dv[0], cc.dv[1]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ixy[q] = __fadd2_rn(ixy[q], g);
      iz[q] = __fadd_rn(iz[q], cc.dv[2]);
    }
  }
  if (cc.plug_drag) {  // imp - v * drag_c (a subtraction is the addition of the exact negation)
    const float2 d = make_float2(cc.drag_c, cc.drag_c);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 m = __fmul2_rn(vs[q], d);
      ixy[q] = __fadd2_rn(ixy[q], make_float2(-m.x, -m.y));
      iz[q] = __fsub_rn(iz[q], __fmul_rn(vz[q], cc.drag_c));
    }
  }
  // vv = v + imp
  float2 vxy[4];
  float vzz[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    vxy[q] = __fadd2_rn(vs[q], ixy[q]);
    vzz[q] = __fadd_rn(vz[q], iz[q]);
    mk[q] = 0;
  }
  // velocity-level response on the OLD positions (kernels.hpp:213-225): spheres, then planes
  auto sphere_vel = [&](const SphereConst<float>& sp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float x[3] = {xs[q].x, xs[q].y, xz[q]};
      float vv[3] = {vxy[q].x, vxy[q].y, vzz[q]};
      sphere_velocity(sp, x, vv, mk[q]);
      vxy[q] = make_float2(vv[0], vv[1]);
      vzz[q] = vv[2];
    }
  };
  auto plane_vel = [&](const PlaneConst<float>& pl) {
    const float2 omf = make_float2(pl.omf, pl.omf);
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // plane_velocity, branch-free (selects, no divergence)
      const bool c = __fsub_rn(xz[q], pl.h) <= pl.band && vzz[q] < 0.f;
      const float2 d = __fmul2_rn(vxy[q], omf);
      const float dz = __fmul_rn(__fsub_rn(vzz[q], vzz[q]), pl.omf);
      vxy[q] = c ? d : vxy[q];
      vzz[q] = c ? dz : vzz[q];
      mk[q] = c ? 1 : mk[q];
    }
  };
  if constexpr (CS == COLL_SPHERE1) {
    const float ox[4] = {xs[0].x, xs[1].x, xs[2].x, xs[3].x};
    const float oy[4] = {xs[0].y, xs[1].y, xs[2].y, xs[3].y};
    if (sphere_near(col.s0, col.s0.Rband, true, ox, oy, xz)) sphere_vel(col.s0);
  } else if constexpr (CS == COLL_PLANE1) {
    plane_vel(col.p0);
  } else {
#pragma unroll 1
    for (int s = 0; s < cc.n_spheres; ++s) sphere_vel(s == 0 ? col.s0 : a.spheres[cc.sphere0 + s]);
#pragma unroll 1
    for (int s = 0; s < cc.n_planes; ++s) plane_vel(s == 0 ? col.p0 : a.planes[cc.plane0 + s]);
  }
  // x' = x + vv dt (kernels.hpp:226-227)
  float2 pxy[4];
  float pz[4];
  {
    const float2 dt2 = make_float2(cc.dt, cc.dt);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      pxy[q] = __fadd2_rn(xs[q], __fmul2_rn(vxy[q], dt2));
      pz[q] = __fadd_rn(xz[q], __fmul_rn(vzz[q], cc.dt));
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    xo[q][0] = pxy[q].x;
    xo[q][1] = pxy[q].y;
    xo[q][2] = pz[q];
    vo[q][0] = vxy[q].x;
    vo[q][1] = vxy[q].y;
    vo[q][2] = vzz[q];
  }
  // position-level intersection elimination (kernels.hpp:229-244): spheres, then planes
  auto sphere_pos = [&](const SphereConst<float>& sp) {
#pragma unroll
    for (int q = 0; q < 4; ++q) sphere_position(sp, xo[q], vo[q], mk[q]);
  };
  auto plane_pos = [&](const PlaneConst<float>& pl) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // plane_position, branch-free
      const bool below = xo[q][2] < pl.h;
      const float vn = vo[q][2];
      const bool damp = below && vn < 0.f;
      const float dx = __fmul_rn(vo[q][0], pl.omf), dy = __fmul_rn(vo[q][1], pl.omf);
      const float dz = __fmul_rn(__fsub_rn(vo[q][2], vn), pl.omf);
      xo[q][2] = below ? pl.h : xo[q][2];
      vo[q][0] = damp ? dx : vo[q][0];
      vo[q][1] = damp ? dy : vo[q][1];
      vo[q][2] = damp ? dz : vo[q][2];
      mk[q] = below ? 1 : mk[q];
    }
  };
  if constexpr (CS == COLL_SPHERE1) {
    const float nx4[4] = {xo[0][0], xo[1][0], xo[2][0], xo[3][0]};
    const float ny4[4] = {xo[0][1], xo[1][1], xo[2][1], xo[3][1]};
    const float nz4[4] = {xo[0][2], xo[1][2], xo[2][2], xo[3][2]};
    if (sphere_near(col.s0, col.s0.R, false, nx4, ny4, nz4)) sphere_pos(col.s0);
  } else if constexpr (CS == COLL_PLANE1) {
    plane_pos(col.p0);
  } else {
#pragma unroll 1
    for (int s = 0; s < cc.n_spheres; ++s) sphere_pos(s == 0 ? col.s0 : a.spheres[cc.sphere0 + s]);
#pragma unroll 1
    for (int s = 0; s < cc.n_planes; ++s) plane_pos(s == 0 ? col.p0 : a.planes[cc.plane0 + s]);
  }
  if (cc.n_pins > 0 && Rf >= cc.pin_row_lo && Rf <= cc.pin_row_hi) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      repin_t(a, cc, Rf, static_cast<int64_t>(Rf) * nx + ix0 + q, t_next, xo[q], vo[q], mk[q]);
  }
  if (a.health) {
    bool fin = true;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) fin = fin && isfinite(xo[q][d]) && isfinite(vo[q][d]);
    if (!fin) atomicMin(&a.health[b].state_frame, k + 1);
  }
}

// One frictionless plane (omf = 1 - friction == 1: config 5's free cloths), no sphere. Every
// contact decision and the mask depend on z alone (plane normal +z), so z keeps the IEEE
// round-to-nearest chain of advance_with_impulse (kernels.hpp:205-252, the plane following the
// sphere's ordering; the same decisions as PARITY) while x, y take the simple finish's contracted
// chain (FAST tolerance) and the velocity factors omf = 1 are identities, left out. 16 instead of
// ~35 instructions per node.
__device__ __forceinline__ void finish_plane_f(const StepArgs<float>& a, const ClothConst<float>& cc,
                                               const PlaneConst<float>& pl, int b, int k, int Rf,
                                               int ix0, float t_next, const float2 (&P0)[4],
                                               const float2 (&Z0)[2], const float2 (&xs)[4],
                                               const float2 (&vs)[4], const float (&xz)[4],
                                               const float (&vz)[4], float (&xo)[4][3],
                                               float (&vo)[4][3], uint8_t (&mk)[4]) {
  const int nx = a.nx;
  if (a.health) {  // non-finite cell impulse: first (step, node) (net.cpp:139-140)
    for (int q = 0; q < 4; ++q)
      if (!(isfinite(P0[q].x) && isfinite(P0[q].y) && isfinite(zc(Z0, q)))) {
        const unsigned long long key = (static_cast<unsigned long long>(k + 1) << 32) |
                                       static_cast<unsigned long long>(Rf * nx + ix0 + q);
        atomicMin(&a.health[b].impulse_key, key);
        break;
      }
  }
  const float2 dvxy = make_float2(cc.fin[0], cc.fin[1]);
  const float drag = cc.fin[3];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // x, y: plug (gravity, drag), integrate — contracted
    float2 imp = __fadd2_rn(P0[q], dvxy);
    imp = __ffma2_rn(vs[q], make_float2(-drag, -drag), imp);
    const float2 vv = __fadd2_rn(vs[q], imp);
    const float2 xx = __ffma2_rn(vv, make_float2(cc.dt, cc.dt), xs[q]);
    // z: add_plug_impulse tail (kernels.hpp:188-195), vv = v + imp, the velocity-level plane
    // response on the old position, x' = x + vv dt, the position-level projection — IEEE RN
    float iz = zc(Z0, q);
    if (cc.plug_gravity) iz = __fadd_rn(iz, cc.dv[2]);
    if (cc.plug_drag) iz = __fsub_rn(iz, __fmul_rn(vz[q], cc.drag_c));
    float vzz = __fadd_rn(vz[q], iz);
    const bool c = __fsub_rn(xz[q], pl.h) <= pl.band && vzz < 0.f;
    vzz = c ? __fsub_rn(vzz, vzz) : vzz;
    float pz = __fadd_rn(xz[q], __fmul_rn(vzz, cc.dt));
    const bool below = pz < pl.h;
    const bool damp = below && vzz < 0.f;
    pz = below ? pl.h : pz;
    vzz = damp ? __fsub_rn(vzz, vzz) : vzz;
    mk[q] = (c || below) ? 1 : 0;
    xo[q][0] = xx.x;
    xo[q][1] = xx.y;
    xo[q][2] = pz;
    vo[q][0] = vv.x;
    vo[q][1] = vv.y;
    vo[q][2] = vzz;
  }
  if (cc.n_pins > 0 && Rf >= cc.pin_row_lo && Rf <= cc.pin_row_hi) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      repin_t(a, cc, Rf, static_cast<int64_t>(Rf) * nx + ix0 + q, t_next, xo[q], vo[q], mk[q]);
  }
  if (a.health) {
    bool fin = true;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int d = 0; d < 3; ++d) fin = fin && isfinite(xo[q][d]) && isfinite(vo[q][d]);
    if (!fin) atomicMin(&a.health[b].state_frame, k + 1);
  }
}

// finish_general with the collider-set specialisation chosen per cloth (a uniform branch)
__device__ __forceinline__ int collider_shape(const ClothConst<float>& cc, const Colliders& col) {
  return cc.n_spheres == 0 && cc.n_planes == 1   ? (col.p0.omf == 1.0f ? COLL_PLANE1F : COLL_PLANE1)
         : cc.n_spheres == 1 && cc.n_planes == 0 ? COLL_SPHERE1
                                                 : COLL_ANY;
}

}  // namespace fastrow
}  // namespace scb
