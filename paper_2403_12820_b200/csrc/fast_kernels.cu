// FAST-mode fused step kernel (f32): forward_impulse -> add_plug_impulse -> advance_with_impulse
// in one pass over HBM (reference kernels.hpp:179-282 driven by eval.cpp:48-59).
//
// Design:
//  * Warp = one 128-column strip of one cloth, marching upward over a segment of rows. Each lane
//    owns 4 consecutive columns (float4 in every plane).
//  * Rows are staged in a 5-slot shared-memory ring by TMA (two cp.async.bulk.tensor.4d boxes per
//    row: the interleaved (x,y) pairs of x and v as 8-byte elements, and the z planes; 136
//    columns from the 16-byte-aligned column x0-4 — TMA rejects unaligned starts — with
//    negative / past-the-end coordinates zero-filled), one row ahead of use.
//  * x and y components are processed as packed f32x2 pairs (FADD2/FFMA2/FMUL2 with the channel
//    weights as scalar-broadcast operands), z as plain f32: two instruction streams for three
//    components.
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
#include <cstdlib>

#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

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

// One unit (cloth b, 128-column strip, rows [y0, y1)) of one step, reading a.in through the
// tensor maps and writing a.out. `phase` carries the ring barriers' parity bits across calls
// (the persistent kernel runs many units / steps on the same ring).
// GEN = false: no cloth of the launch takes the collider / pressure / mask finish, which is
// then compiled out (fewer live registers around the row loop)
template <bool ALPHA1, int RING, bool PEER = false, bool GEN = true, bool ZS = false>
__device__ __forceinline__ void run_unit(const CUtensorMap* tmap_xy, const CUtensorMap* tmap_z,
                                         const StepArgs<float>& a, const FastNet& f, int b,
                                         int strip, int y0, int y1, float* ring, uint64_t* full,
                                         float (*scratch)[13], uint32_t& phase) {
  const int lane = threadIdx.x;
  const int x0 = strip * STRIP;
  const int ix0 = x0 + FW * lane;
  const int nx = a.nx, ny = a.ny;

  // Rows y0-2 .. y1+1 pass through the ring; arithmetic starts at row y0 (the two rows below
  // only feed rows < y0) and the last two steps (rows y1, y1+1) only finish rows y1-2, y1-1.
  const int r_first = y0 - 2;
  const int r_last = y1 + 1;

  // the cloth's constants: loaded before the prologue's TMA waits so the two latencies overlap
  const ClothConst<float> cc = a.cloths[b];
  const bool simple = cc.n_spheres == 0 && cc.n_planes == 0 && !cc.plug_pressure &&
                      a.constrained == nullptr;
  const int64_t nodes = static_cast<int64_t>(nx) * ny;
  const float t_next = a.use_t_override ? a.t_override : __fmul_rn(float(a.k + 1), cc.dt);
  const float dv_eff[3] = {cc.fin[0], cc.fin[1], cc.fin[2]};  // plugged gravity impulse or 0
  const float drag_eff = cc.fin[3];                            // plugged drag coefficient or 0

  // ring slot t % RING of row r_first + t is tracked incrementally (no modulo in the loop); the
  // TMA operands are formed outside the lane-0 branch so they stay warp-uniform
  const uint32_t ring_s = smem_u32(ring), full_s = smem_u32(full);
  const int cx = x0 - 4, crow0 = r_first - a.g0;
  auto issue = [&](int t, int sl) {  // row r_first + t into slot sl
    const uint32_t dst = ring_s + static_cast<uint32_t>(sl) * (ROWF * 4);
    const uint32_t bar = full_s + static_cast<uint32_t>(sl) * 8;
    const int crow = crow0 + t;
    if (elect_one()) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "n"(ROW_BYTES)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(tmap_xy)), "r"(cx), "r"(crow), "r"(0), "r"(b), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst + Z_X * 4),
          "l"(reinterpret_cast<uint64_t>(tmap_z)), "r"(cx), "r"(crow), "r"(0), "r"(b), "r"(bar)
          : "memory");
    }
  };
  auto wait_slot = [&](int sl) {
    mbar_wait(&full[sl], (phase >> sl) & 1u);
    phase ^= 1u << sl;
  };
  auto nxt = [](int sl) { return sl + 1 == RING ? 0 : sl + 1; };
  __syncwarp();  // earlier generic reads of the ring are done before TMA refills it
  issue(0, 0);
  issue(1, 1);
  issue(2, 2);
  wait_slot(0);
  wait_slot(1);

  // nx % 4 == 0 (fast_supported): only a strip's outermost lanes own edges leaving the grid
  const uint32_t mL = ix0 >= 1 ? 0xffffffffu : 0u;
  const uint32_t mRt = ix0 + 4 < nx ? 0xffffffffu : 0u;
  const bool lane_live = ix0 < nx;


  // accumulators [column] for rows R-2 (P0/Z0), R-1 (P1/Z1), R (P2/Z2): P = (x,y), Z = z
  float2 P0[4], P1[4], P2[4];
  float2 Z0[2], Z1[2], Z2[2];  // column pairs (0,1), (2,3)
#pragma unroll
  for (int k = 0; k < 4; ++k) P0[k] = P1[k] = P2[k] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 2; ++j) Z0[j] = Z1[j] = Z2[j] = make_float2(0.f, 0.f);

  // slots of rows R, R-1, R-2 (R-3 for the pressure finish) and of the prefetched row R+1
  int sR = 2 % RING, s1 = 1, s2 = 0, s3 = RING - 1, sI = 3 % RING;
  // output row pointers (x.xy plane and x.z plane) of the finished row R-2, advanced per row
  const int64_t S = a.plane_stride;
  float* const out_b = a.out + static_cast<int64_t>(b) * 6 * S;
  float* oxy = out_b + 2 * (static_cast<int64_t>(y0 - 2 - a.g0) * a.pitch + ix0);
  float* oz = out_b + 4 * S + static_cast<int64_t>(y0 - 2 - a.g0) * a.pitch + ix0;

#pragma unroll 1
  for (int R = y0; R <= r_last; ++R) {
    const int t = R - r_first;
    __syncwarp();
    if (R + 1 <= r_last) issue(t + 1, sI);
    wait_slot(sR);

    const float* rowR = ring + sR * ROWF;
    const float* row1 = ring + s1 * ROWF;
    const float* row2 = ring + s2 * ROWF;
    if (R >= y1) {
      // the second tail row only feeds row y1 - 1 through N2 edges (simple-finish kernels; the
      // general-finish kernel measured faster with the one tail body)
      if (R < ny) {
        if (!GEN && R > y1)
          row_pass<ALPHA1, false, 2, ZS>(f, rowR, row1, row2, lane, mL, mRt, 1.f, 1.f, P0, P1,
                                         P2, Z0, Z1, Z2);
        else
          row_pass<ALPHA1, false, 1, ZS>(f, rowR, row1, row2, lane, mL, mRt, 1.f, 1.f, P0, P1,
                                         P2, Z0, Z1, Z2);
      }
    } else if (R >= 2) {
      row_pass<ALPHA1, false, 0, ZS>(f, rowR, row1, row2, lane, mL, mRt, 1.f, 1.f, P0, P1, P2, Z0,
                                     Z1, Z2);
    } else {
      row_pass<ALPHA1, true, 0, ZS>(f, rowR, row1, row2, lane, mL, mRt, R >= 1 ? 1.f : 0.f, 0.f,
                                    P0, P1, P2, Z0, Z1, Z2);
    }

    // row R-2 is complete: plug, integrate, collide, pin, store
    const int Rf = R - 2;
    if (Rf >= y0 && Rf < y1 && lane_live) {
      const int64_t lr = Rf - a.g0;
      if (!GEN || simple) {
        float2 xs[4], vs[4];
        float xz[4], vz[4];
        win4(row2 + XY_X, lane, xs);
        win4(row2 + XY_V, lane, vs);
        win4z<ZS>(row2 + Z_X, lane, xz);
        win4z<ZS>(row2 + Z_V, lane, vz);
        // add_plug_impulse gravity/drag + advance without colliders (no mask, no contact
        // decision depends on it): FMA-contracted and x,y packed — part of FAST mode's 1e-5 bar
        float xo[3][4], vo[3][4];
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
          for (int k = 0; k < 4; ++k) {
            fin_imp = fin_imp && isfinite(P0[k].x) && isfinite(P0[k].y) && isfinite(zc(Z0, k));
#pragma unroll
            for (int d = 0; d < 3; ++d) fin = fin && isfinite(xo[d][k]) && isfinite(vo[d][k]);
          }
          if (!fin_imp) {
            for (int k = 0; k < 4; ++k)
              if (!(isfinite(P0[k].x) && isfinite(P0[k].y) && isfinite(zc(Z0, k)))) {
                const unsigned long long key = (static_cast<unsigned long long>(a.k + 1) << 32) |
                                               static_cast<unsigned long long>(Rf * nx + ix0 + k);
                atomicMin(&a.health[b].impulse_key, key);
                break;
              }
          }
          if (!fin) atomicMin(&a.health[b].state_frame, a.k + 1);
        }
        float* ovxy = oxy + 2 * S;
        const int sw = (ix0 >> 3) & 2;  // xy_col: this lane's group stores its halves swapped
        *reinterpret_cast<float4*>(oxy + 2 * sw) =
            make_float4(xo[0][0], xo[1][0], xo[0][1], xo[1][1]);
        *reinterpret_cast<float4*>(oxy + 2 * (2 ^ sw)) =
            make_float4(xo[0][2], xo[1][2], xo[0][3], xo[1][3]);
        *reinterpret_cast<float4*>(ovxy + 2 * sw) =
            make_float4(vo[0][0], vo[1][0], vo[0][1], vo[1][1]);
        *reinterpret_cast<float4*>(ovxy + 2 * (2 ^ sw)) =
            make_float4(vo[0][2], vo[1][2], vo[0][3], vo[1][3]);
        *reinterpret_cast<float4*>(oz) = zgroup<ZS>(ix0, xo[2][0], xo[2][1], xo[2][2], xo[2][3]);
        *reinterpret_cast<float4*>(oz + S) = zgroup<ZS>(ix0, vo[2][0], vo[2][1], vo[2][2], vo[2][3]);
        // fused halo exchange: the two owned rows at a peer side also go into the neighbour's
        // ghost rows (its output buffer, remote over NVLink)
        if (PEER && (Rf < a.u0 + 2 || Rf >= a.u1 - 2))  // boundary rows only
#pragma unroll 1
        for (int side = 0; side < 2; ++side) {
          float* po = a.peer_out[side];
          if (po == nullptr) continue;
          if (side == 0 ? Rf >= a.u0 + 2 : Rf < a.u1 - 2) continue;
          const int64_t S2 = a.peer_S[side];
          const int64_t lr2 = Rf - a.peer_g0[side];
          float* pb = po + static_cast<int64_t>(b) * 6 * S2;
          float* pxy = pb + 2 * (lr2 * a.pitch + ix0);
          float* pz = pb + 4 * S2 + lr2 * a.pitch + ix0;
          const int sw2 = (ix0 >> 3) & 2;
          *reinterpret_cast<float4*>(pxy + 2 * sw2) =
              make_float4(xo[0][0], xo[1][0], xo[0][1], xo[1][1]);
          *reinterpret_cast<float4*>(pxy + 2 * (2 ^ sw2)) =
              make_float4(xo[0][2], xo[1][2], xo[0][3], xo[1][3]);
          *reinterpret_cast<float4*>(pxy + 2 * S2 + 2 * sw2) =
              make_float4(vo[0][0], vo[1][0], vo[0][1], vo[1][1]);
          *reinterpret_cast<float4*>(pxy + 2 * S2 + 2 * (2 ^ sw2)) =
              make_float4(vo[0][2], vo[1][2], vo[0][3], vo[1][3]);
          *reinterpret_cast<float4*>(pz) = zgroup<ZS>(ix0, xo[2][0], xo[2][1], xo[2][2], xo[2][3]);
          *reinterpret_cast<float4*>(pz + S2) = zgroup<ZS>(ix0, vo[2][0], vo[2][1], vo[2][2], vo[2][3]);
        }
      } else if (!cc.plug_pressure) {
        // colliders and/or the contact mask: the lane's 4 nodes together (collider outer, node
        // inner: each collider's constants are loaded once per row), each node through the
        // same IEEE-exact sequence as advance_with_impulse (sc_device.cuh), packed stores
        float2 xs[4], vs[4];
        float xz[4], vz[4];
        win4(row2 + XY_X, lane, xs);
        win4(row2 + XY_V, lane, vs);
        win4z<ZS>(row2 + Z_X, lane, xz);
        win4z<ZS>(row2 + Z_V, lane, vz);
        float x[4][3], vo[4][3], xo[4][3];
        uint8_t mk[4];
        bool fin_imp = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v[3] = {vs[k].x, vs[k].y, vz[k]};
          float imp[3] = {P0[k].x, P0[k].y, zc(Z0, k)};
          fin_imp = fin_imp && isfinite(imp[0]) && isfinite(imp[1]) && isfinite(imp[2]);
          plug_tail(cc, v, imp);
          x[k][0] = xs[k].x;
          x[k][1] = xs[k].y;
          x[k][2] = xz[k];
#pragma unroll
          for (int d = 0; d < 3; ++d) vo[k][d] = __fadd_rn(v[d], imp[d]);
          mk[k] = 0;
        }
        if (a.health && !fin_imp) {
          for (int k = 0; k < 4; ++k)
            if (!(isfinite(P0[k].x) && isfinite(P0[k].y) && isfinite(zc(Z0, k)))) {
              const unsigned long long key = (static_cast<unsigned long long>(a.k + 1) << 32) |
                                             static_cast<unsigned long long>(Rf * nx + ix0 + k);
              atomicMin(&a.health[b].impulse_key, key);
              break;
            }
        }
#pragma unroll 1
        for (int q = 0; q < cc.n_spheres; ++q) {
          const SphereConst<float> sp = a.spheres[cc.sphere0 + q];
#pragma unroll
          for (int k = 0; k < 4; ++k) sphere_velocity(sp, x[k], vo[k], mk[k]);
        }
#pragma unroll 1
        for (int q = 0; q < cc.n_planes; ++q) {
          const PlaneConst<float> pl = a.planes[cc.plane0 + q];
#pragma unroll
          for (int k = 0; k < 4; ++k) plane_velocity(pl, x[k], vo[k], mk[k]);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d) xo[k][d] = __fadd_rn(x[k][d], __fmul_rn(vo[k][d], cc.dt));
#pragma unroll 1
        for (int q = 0; q < cc.n_spheres; ++q) {
          const SphereConst<float> sp = a.spheres[cc.sphere0 + q];
#pragma unroll
          for (int k = 0; k < 4; ++k) sphere_position(sp, xo[k], vo[k], mk[k]);
        }
#pragma unroll 1
        for (int q = 0; q < cc.n_planes; ++q) {
          const PlaneConst<float> pl = a.planes[cc.plane0 + q];
#pragma unroll
          for (int k = 0; k < 4; ++k) plane_position(pl, xo[k], vo[k], mk[k]);
        }
        if (cc.n_pins > 0 && Rf >= cc.pin_row_lo && Rf <= cc.pin_row_hi) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            repin(a, cc, Rf, static_cast<int64_t>(Rf) * nx + ix0 + k, xo[k], vo[k], mk[k]);
        }
        if (a.health) {
          bool fin = true;
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int d = 0; d < 3; ++d) fin = fin && isfinite(xo[k][d]) && isfinite(vo[k][d]);
          if (!fin) atomicMin(&a.health[b].state_frame, a.k + 1);
        }
        const int sw = (ix0 >> 3) & 2;  // xy_col swizzle of this lane's group
        const float4 xy01 = make_float4(xo[0][0], xo[0][1], xo[1][0], xo[1][1]);
        const float4 xy23 = make_float4(xo[2][0], xo[2][1], xo[3][0], xo[3][1]);
        const float4 vxy01 = make_float4(vo[0][0], vo[0][1], vo[1][0], vo[1][1]);
        const float4 vxy23 = make_float4(vo[2][0], vo[2][1], vo[3][0], vo[3][1]);
        const float4 z4 = zgroup<ZS>(ix0, xo[0][2], xo[1][2], xo[2][2], xo[3][2]);
        const float4 vz4 = zgroup<ZS>(ix0, vo[0][2], vo[1][2], vo[2][2], vo[3][2]);
        float* ovxy = oxy + 2 * S;
        *reinterpret_cast<float4*>(oxy + 2 * sw) = xy01;
        *reinterpret_cast<float4*>(oxy + 2 * (2 ^ sw)) = xy23;
        *reinterpret_cast<float4*>(ovxy + 2 * sw) = vxy01;
        *reinterpret_cast<float4*>(ovxy + 2 * (2 ^ sw)) = vxy23;
        *reinterpret_cast<float4*>(oz) = z4;
        *reinterpret_cast<float4*>(oz + S) = vz4;
        if (PEER && (Rf < a.u0 + 2 || Rf >= a.u1 - 2))  // fused halo exchange, boundary rows
#pragma unroll 1
          for (int side = 0; side < 2; ++side) {
            float* po = a.peer_out[side];
            if (po == nullptr || (side == 0 ? Rf >= a.u0 + 2 : Rf < a.u1 - 2)) continue;
            const int64_t S2 = a.peer_S[side];
            const int64_t lr2 = Rf - a.peer_g0[side];
            float* pb = po + static_cast<int64_t>(b) * 6 * S2;
            float* pxy = pb + 2 * (lr2 * a.pitch + ix0);
            float* pz = pb + 4 * S2 + lr2 * a.pitch + ix0;
            *reinterpret_cast<float4*>(pxy + 2 * sw) = xy01;
            *reinterpret_cast<float4*>(pxy + 2 * (2 ^ sw)) = xy23;
            *reinterpret_cast<float4*>(pxy + 2 * S2 + 2 * sw) = vxy01;
            *reinterpret_cast<float4*>(pxy + 2 * S2 + 2 * (2 ^ sw)) = vxy23;
            *reinterpret_cast<float4*>(pz) = z4;
            *reinterpret_cast<float4*>(pz + S2) = vz4;
          }
        if (a.constrained)
          *reinterpret_cast<uchar4*>(a.constrained + b * nodes + static_cast<int64_t>(Rf) * nx +
                                     ix0) = make_uchar4(mk[0], mk[1], mk[2], mk[3]);
      } else {
        // pressure plug: one node at a time (compact code, same IEEE-exact chain)
        const float* rs = ring + s3 * ROWF;  // row Rf-1
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          scratch[lane][k] = P0[k].x;  // own row of the scratch only: no cross-lane sync
          scratch[lane][4 + k] = P0[k].y;
          scratch[lane][8 + k] = zc(Z0, k);
        }
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
          const int ix = ix0 + k;
          const int j = FW * lane + 4 + k;
          const int64_t gnode = static_cast<int64_t>(Rf) * nx + ix;
          float px[3], pv[3], imp[3], po[3], qo[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            px[d] = slot_val<ZS>(row2, true, d, j);
            pv[d] = slot_val<ZS>(row2, false, d, j);
            imp[d] = scratch[lane][4 * d + k];
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
              e[d] = __fsub_rn(px[d], slot_val<ZS>(row2, true, d, j + 1));
              n[d] = __fsub_rn(px[d], slot_val<ZS>(row1, true, d, j));
              w[d] = __fsub_rn(px[d], slot_val<ZS>(row2, true, d, j - 1));
              sv[d] = __fsub_rn(px[d], slot_val<ZS>(rs, true, d, j));
            }
            pressure_plug(cc, interior, e, n, w, sv, imp);
          }
          plug_tail(cc, pv, imp);
          uint8_t mk;
          advance_node(a, cc, Rf, gnode, px, pv, imp, po, qo, mk);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            out_b[elem_index(d, lr, ix, a.pitch, S, ZS)] = po[d];
            out_b[elem_index(3 + d, lr, ix, a.pitch, S, ZS)] = qo[d];
          }
          for (int side = 0; PEER && side < 2; ++side) {  // fused halo exchange (simple path)
            float* pp = a.peer_out[side];
            if (pp == nullptr || (side == 0 ? Rf >= a.u0 + 2 : Rf < a.u1 - 2)) continue;
            const int64_t S2 = a.peer_S[side];
            float* pb = pp + static_cast<int64_t>(b) * 6 * S2;
            const int64_t lr2 = Rf - a.peer_g0[side];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              pb[elem_index(d, lr2, ix, a.pitch, S2, ZS)] = po[d];
              pb[elem_index(3 + d, lr2, ix, a.pitch, S2, ZS)] = qo[d];
            }
          }
          if (a.constrained) a.constrained[b * nodes + gnode] = mk;
          if (a.health && !(isfinite(po[0]) && isfinite(po[1]) && isfinite(po[2]) &&
                            isfinite(qo[0]) && isfinite(qo[1]) && isfinite(qo[2])))
            atomicMin(&a.health[b].state_frame, a.k + 1);
        }
      }
    }
    // advance: slots, output rows, accumulator rows
    s3 = s2;
    s2 = s1;
    s1 = sR;
    sR = sI;
    sI = nxt(sI);
    oxy += 2 * a.pitch;
    oz += a.pitch;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      Z0[j] = Z1[j];
      Z1[j] = Z2[j];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      P0[k] = P1[k];
      P1[k] = P2[k];
    }
  }
}

__device__ unsigned long long* g_unit_times = nullptr;  // debug: [units][3] start, end, sm/warp

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Unit u -> (cloth b, strip, rows [y0, y1)); segment boundaries are spread evenly so no unit
// gets a runt remainder.
__device__ __forceinline__ void decode_unit(int unit, int n_strips, int n_segs, int u0, int rows,
                                            int& b, int& strip, int& y0, int& y1) {
  const int seg = unit % n_segs;
  strip = (unit / n_segs) % n_strips;
  b = unit / (n_segs * n_strips);
  y0 = u0 + static_cast<int>((static_cast<int64_t>(seg) * rows) / n_segs);
  y1 = u0 + static_cast<int>((static_cast<int64_t>(seg + 1) * rows) / n_segs);
}

#ifndef SC_FAST_MINB
#define SC_FAST_MINB 16
#endif
// MINB: resident CTAs per SM the register allocation targets. 16 (128 registers) suits short
// segments and single waves; 10 (160 registers, 12 CTAs/SM: more independent edges in flight)
// runs the row loop ~5% faster and wins on tall columns processed in several waves of long
// segments (config 4: 604 -> 571 us/step), but loses on short-segment problems (config 2, 5;
// MINB 8 = 206 registers is slower again: 631 us).
template <bool ALPHA1, int RING, bool PEER = false, bool GEN = true, int MINB = SC_FAST_MINB,
          bool ZS = false>
__global__ void __launch_bounds__(32, MINB) fast_step_kernel(const __grid_constant__ CUtensorMap tmap_xy,
                                                      const __grid_constant__ CUtensorMap tmap_z,
                                                      const StepArgs<float> a, const FastNet f,
                                                      const int n_strips, const int /*seg_rows*/,
                                                      const int n_segs) {
  // dynamic smem: [RING][ROWF] ring, then (RING = 5: some cloth plugs pressure) a [32][13]
  // per-lane impulse scratch for the pressure finish
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full[RING];
  float (*scratch)[13] = reinterpret_cast<float (*)[13]>(ring + RING * ROWF);
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int unit = blockIdx.x;
  int b, strip, y0, y1;
  decode_unit(unit, n_strips, n_segs, a.u0, a.u1 - a.u0, b, strip, y0, y1);
  b += a.b_off;
  // programmatic dependent launch: the setup above overlapped the previous step's tail; the
  // state it wrote is read from here on
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t phase = 0;
  unsigned long long* times = g_unit_times;
  if (times && threadIdx.x == 0) {
    unsigned smid, wid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    times[3 * unit] = gtimer();
    times[3 * unit + 2] = (static_cast<unsigned long long>(smid) << 32) | wid;
  }
  if (y0 < y1)
    run_unit<ALPHA1, RING, PEER, GEN, ZS>(&tmap_xy, &tmap_z, a, f, b, strip, y0, y1, ring, full, scratch,
                                 phase);
  if (times && threadIdx.x == 0) times[3 * unit + 1] = gtimer();
  // let the next step's grid launch once every CTA of this one is done with its work (an early
  // trigger would let waiting CTAs occupy SM slots a multi-wave grid still needs)
  asm volatile("griddepcontrol.launch_dependents;");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Persistent multi-step variant: one co-resident CTA per unit runs `steps` consecutive steps,
// ping-ponging between the two state buffers. Instead of a grid-wide barrier per step, a unit
// starts step k once its (up to 8) neighbour units — the only ones whose rows/columns lie within
// the stencil's 2-node reach — published completion of step k-1 (acquire/release flags in
// global memory). That covers both the read-after-write (halo rows of step k-1) and the
// write-after-read (neighbours done reading the buffer this step overwrites) hazards.
template <bool ALPHA1, int RING, bool GEN = true, bool ZS = false>
#ifndef SC_MULTI_MINB
#define SC_MULTI_MINB 12
#endif
__global__ void __launch_bounds__(32, GEN ? SC_MULTI_MINB : 16) fast_multi_kernel(
    const __grid_constant__ CUtensorMap txy0, const __grid_constant__ CUtensorMap tz0,
    const __grid_constant__ CUtensorMap txy1, const __grid_constant__ CUtensorMap tz1,
    const StepArgs<float> a0, const FastNet f, const int n_strips, const int seg_rows,
    const int n_segs, const int steps, int* __restrict__ done) {
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t full[RING];
  float (*scratch)[13] = reinterpret_cast<float (*)[13]>(ring + RING * ROWF);
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int unit = blockIdx.x;
  const int seg = unit % n_segs;
  int b, strip, y0, y1;
  decode_unit(unit, n_strips, n_segs, a0.u0, a0.u1 - a0.u0, b, strip, y0, y1);
  uint32_t phase = 0;
  StepArgs<float> a = a0;
  for (int s = 0; s < steps; ++s) {
    const int k = a0.k + s;
    if (s > 0) {
      // lanes 0..8 each watch one neighbour (all polled concurrently: one L2 round trip)
      if (threadIdx.x < 9 && threadIdx.x != 4) {
        const int dg = static_cast<int>(threadIdx.x) / 3 - 1, ds = static_cast<int>(threadIdx.x) % 3 - 1;
        const int g2 = seg + dg, s2 = strip + ds;
        if (g2 >= 0 && g2 < n_segs && s2 >= 0 && s2 < n_strips) {
          const int* flag = done + (b * n_strips + s2) * n_segs + g2;
          while (ld_acquire(flag) < k - 1) {
          }
        }
      }
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncwarp();
    const bool even = (s & 1) == 0;
    a.in = even ? a0.in : a0.out;
    a.out = even ? a0.out : const_cast<float*>(a0.in);
    a.k = k;
    if (y0 < y1)
      run_unit<ALPHA1, RING, false, GEN, ZS>(even ? &txy0 : &txy1, even ? &tz0 : &tz1, a, f, b, strip, y0, y1,
                             ring, full, scratch, phase);
    __syncwarp();  // orders every lane's stores before lane 0's (cumulative) release
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      st_release(done + unit, k);
    }
  }
}

__global__ void fill_done(int* done, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) done[i] = v;
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

template <bool ALPHA1, int RING>
void* kernel_ptr() {
  return reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING>);
}
template <bool ALPHA1, int RING>
void* simple_kernel_ptr() {
  return reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING, false, false>);
}
constexpr int kWideMinB = 10;
template <bool ALPHA1, int RING>
void* zs_kernel_ptr(bool peer) {
  return peer ? reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING, true, true, SC_FAST_MINB, true>)
              : reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING, false, true, SC_FAST_MINB, true>);
}
template <bool ALPHA1, int RING>
void* zs_multi_ptr() {
  return reinterpret_cast<void*>(fast_multi_kernel<ALPHA1, RING, true, true>);
}
template <bool ALPHA1, int RING>
void* wide_kernel_ptr() {
  return reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING, false, false, kWideMinB>);
}

void* pick_kernel(bool alpha1, int ring) {
  if (ring == 5) return alpha1 ? kernel_ptr<true, 5>() : kernel_ptr<false, 5>();
  return alpha1 ? kernel_ptr<true, 4>() : kernel_ptr<false, 4>();
}

template <bool ALPHA1, int RING>
void* peer_kernel_ptr() {
  return reinterpret_cast<void*>(fast_step_kernel<ALPHA1, RING, true>);
}

template <bool ALPHA1, int RING>
void* multi_ptr() {
  return reinterpret_cast<void*>(fast_multi_kernel<ALPHA1, RING>);
}
template <bool ALPHA1, int RING>
void* multi_simple_ptr() {
  return reinterpret_cast<void*>(fast_multi_kernel<ALPHA1, RING, false>);
}

void* pick_multi(bool alpha1, int ring, bool general = true) {
  if (!general) {
    if (ring == 5) return alpha1 ? multi_simple_ptr<true, 5>() : multi_simple_ptr<false, 5>();
    return alpha1 ? multi_simple_ptr<true, 4>() : multi_simple_ptr<false, 4>();
  }
  if (ring == 5) return alpha1 ? multi_ptr<true, 5>() : multi_ptr<false, 5>();
  return alpha1 ? multi_ptr<true, 4>() : multi_ptr<false, 4>();
}

size_t fast_smem_bytes(int ring, bool general) {
  size_t pad = 0;
  if (const char* env = std::getenv("SC_FAST_SMEM_PAD")) pad = std::strtoul(env, nullptr, 10);
  // the per-lane impulse scratch serves only the pressure finish (RING = 5); the collider / mask
  // finish keeps everything in registers, so `general` alone costs no shared memory
  (void)general;
  return sizeof(float) * (ring * ROWF + (ring == 5 ? 32 * 13 : 0)) + pad;  // pad: tuning knob
}

FastPlan plan_fast(int nx, int rows, int batch, int device, bool pressure, bool general) {
  FastPlan p{};
  p.ring = pressure ? 5 : 4;
  p.general = general;
  p.n_strips = (nx + STRIP - 1) / STRIP;
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t smem = fast_smem_bytes(p.ring, general);
  for (void* k : {pick_kernel(true, p.ring), pick_kernel(false, p.ring), pick_multi(true, p.ring),
                  p.ring == 5 ? simple_kernel_ptr<true, 5>() : simple_kernel_ptr<true, 4>(),
                  p.ring == 5 ? simple_kernel_ptr<false, 5>() : simple_kernel_ptr<false, 4>(),
                  p.ring == 5 ? wide_kernel_ptr<true, 5>() : wide_kernel_ptr<true, 4>(),
                  p.ring == 5 ? zs_kernel_ptr<true, 5>(false) : zs_kernel_ptr<true, 4>(false),
                  p.ring == 5 ? zs_kernel_ptr<false, 5>(false) : zs_kernel_ptr<false, 4>(false),
                  p.ring == 5 ? zs_kernel_ptr<true, 5>(true) : zs_kernel_ptr<true, 4>(true),
                  p.ring == 5 ? zs_kernel_ptr<false, 5>(true) : zs_kernel_ptr<false, 4>(true),
                  p.ring == 5 ? zs_multi_ptr<true, 5>() : zs_multi_ptr<true, 4>(),
                  p.ring == 5 ? zs_multi_ptr<false, 5>() : zs_multi_ptr<false, 4>(),
                  p.ring == 5 ? wide_kernel_ptr<false, 5>() : wide_kernel_ptr<false, 4>(),
                  pick_multi(false, p.ring), pick_multi(true, p.ring, false),
                  pick_multi(false, p.ring, false),
                  p.ring == 5 ? peer_kernel_ptr<true, 5>() : peer_kernel_ptr<true, 4>(),
                  p.ring == 5 ? peer_kernel_ptr<false, 5>() : peer_kernel_ptr<false, 4>()})
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pick_kernel(true, p.ring), 32, smem);
  if (occ < 1) occ = 1;
  const int64_t columns = static_cast<int64_t>(batch) * p.n_strips;
  const int max_segs = std::max(1, rows / 4);
  // choose the number of row segments maximising  fill x warm x balance:
  //  fill    — units / (waves x resident slots);
  //  warm    — seg / (seg + 1.5): each unit re-computes ~1.1 rows of edges below / above its
  //            segment and waits for its first three rows (measured, tools/batch_sweep.py);
  //  balance — 1 - 0.1 / waves: a single wave ends on its late warps (an SMSP issues its warp
  //            slots in a fixed order, so its warps finish in tiers), later waves refill freed
  //            slots;
  // with segments of at least 4 rows (small problems: many short units beat few long ones).
  auto segment = [&](int occupancy) {
    const int64_t slots = static_cast<int64_t>(sms) * occupancy;
    double best = -1.0;
    int best_segs = 1;
    for (int segs = 1; segs <= max_segs && segs <= 4096; ++segs) {
      // segments of floor/ceil(rows / segs) rows (decode_unit spreads the boundaries evenly)
      const double seg_rows = static_cast<double>(rows) / segs;
      const int64_t units = columns * segs;
      const int64_t waves = (units + slots - 1) / slots;
      const double fill = static_cast<double>(units) / static_cast<double>(waves * slots);
      const double warm = seg_rows / (seg_rows + 1.5);
      const double balance = 1.0 - 0.1 / static_cast<double>(waves);
      const double eff = fill * warm * balance;
      if (eff > best + 1e-9) {
        best = eff;
        best_segs = segs;
      }
    }
    return best_segs;
  };
  int best_segs = segment(occ);
  // simple-finish launches whose segments come out tall take the 12-CTA, wide-register kernel
  // (measured: config 4's 55-row segments gain 5%; config 2's 15-row single wave loses 1%)
  p.wide = false;
  if (!general) {
    int occ_w = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ_w, p.ring == 5 ? wide_kernel_ptr<true, 5>() : wide_kernel_ptr<true, 4>(), 32, smem);
    p.wide = occ_w > 0 && rows / best_segs >= 32;
    if (const char* env = std::getenv("SC_FAST_WIDE")) p.wide = occ_w > 0 && std::atoi(env) != 0;
    if (p.wide) {
      occ = occ_w;
      best_segs = segment(occ);
    }
  }
  p.seg_rows = (rows + best_segs - 1) / best_segs;
  if (const char* env = std::getenv("SC_FAST_SEG_ROWS")) {  // tuning knob for experiments
    const int v = std::atoi(env);
    if (v >= 2) best_segs = std::max(1, (rows + v - 1) / v);
    p.seg_rows = (rows + best_segs - 1) / best_segs;
  }
  p.n_segs = best_segs;
  p.units = columns * p.n_segs;
  // chunked stepping (capi.cu chunked_fast_steps: concurrent cloth-chunk streams fill each
  // other's launch ramps and tails): the longest segments that still give ~1.15 waves of units
  // (measured optimum: config 2 at 11-12 rows, config 5 at whole 128-row columns)
  {
    const int64_t slots = static_cast<int64_t>(sms) * occ;
    int cs = static_cast<int>((115 * slots + 100 * columns - 1) / (100 * columns));
    cs = std::max(1, std::min(cs, max_segs));
    if (const char* env = std::getenv("SC_CHUNK_SEG_ROWS")) {
      const int v = std::atoi(env);
      if (v >= 2) cs = std::max(1, (rows + v - 1) / v);
    }
    p.chunk_segs = cs;
  }
  p.smem = smem;
  p.occupancy = occ;
  int occ_multi = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_multi, pick_multi(true, p.ring, general), 32,
                                                smem);
  p.multi_ok = p.units <= static_cast<int64_t>(sms) * occ_multi;  // every unit co-resident
  if (!p.multi_ok && occ_multi > 0) {
    // the persistent kernel's own segmentation: one co-resident unit per slot
    const int64_t mslots = static_cast<int64_t>(sms) * occ_multi;
    const int msegs = static_cast<int>(std::max<int64_t>(1, mslots / columns));
    if (columns * std::min(msegs, max_segs) <= mslots) {
      p.multi_segs = std::min(msegs, max_segs);
      p.multi_ok = true;
    }
  } else {
    p.multi_segs = p.n_segs;
  }
  return p;
}

cudaError_t launch_fast(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tmap,
                        const FastPlan& p, cudaStream_t stream) {
  const int rows = a.u1 - a.u0;
  if (rows <= 0 || a.batch <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.units));
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const CUtensorMap& txy = tmap[0];
  const CUtensorMap& tz = tmap[1];
  const int ns = p.n_strips, sr = p.seg_rows, ng = p.n_segs;
  const bool peer = a.peer_out[0] != nullptr || a.peer_out[1] != nullptr;
#define SC_FK(A, R, P)                                                                     \
  (a.zs ? cudaLaunchKernelEx(&cfg, fast_step_kernel<A, R, P, true, SC_FAST_MINB, true>, txy, tz, a, \
                             f, ns, sr, ng)                                                    \
        : cudaLaunchKernelEx(&cfg, fast_step_kernel<A, R, P>, txy, tz, a, f, ns, sr, ng))
#define SC_FS(A, R) \
  cudaLaunchKernelEx(&cfg, fast_step_kernel<A, R, false, false>, txy, tz, a, f, ns, sr, ng)
#define SC_FW(A, R) \
  cudaLaunchKernelEx(&cfg, fast_step_kernel<A, R, false, false, kWideMinB>, txy, tz, a, f, ns, sr, ng)
  const bool simple = !peer && !p.general && a.constrained == nullptr && !a.zs;
  if (simple && p.wide) {
    if (p.ring == 5) return f.alpha1 ? SC_FW(true, 5) : SC_FW(false, 5);
    return f.alpha1 ? SC_FW(true, 4) : SC_FW(false, 4);
  }
#undef SC_FW
  if (simple) {  // simple finish only (plain z layout)
    if (p.ring == 5) return f.alpha1 ? SC_FS(true, 5) : SC_FS(false, 5);
    return f.alpha1 ? SC_FS(true, 4) : SC_FS(false, 4);
  }
#undef SC_FS
  if (peer) {  // fused halo exchange (strip contexts linked with sc_ctx_set_peer)
    if (p.ring == 5) return f.alpha1 ? SC_FK(true, 5, true) : SC_FK(false, 5, true);
    return f.alpha1 ? SC_FK(true, 4, true) : SC_FK(false, 4, true);
  }
  if (p.ring == 5) return f.alpha1 ? SC_FK(true, 5, false) : SC_FK(false, 5, false);
  return f.alpha1 ? SC_FK(true, 4, false) : SC_FK(false, 4, false);
#undef SC_FK
}

cudaError_t set_unit_timing(unsigned long long* dev_buf) {
  return cudaMemcpyToSymbol(g_unit_times, &dev_buf, sizeof(dev_buf));
}

cudaError_t launch_fast_multi(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tin,
                              const CUtensorMap* tout, const FastPlan& p, int steps, int* done,
                              cudaStream_t stream) {
  const int rows = a.u1 - a.u0;
  if (rows <= 0 || a.batch <= 0 || steps <= 0) return cudaSuccess;
  const int units = static_cast<int>(p.n_strips * static_cast<int64_t>(a.batch) * p.multi_segs);
  fill_done<<<(units + 255) / 256, 256, 0, stream>>>(done, units, a.k - 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(units));
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: units wait on each other
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int ns = p.n_strips, sr = p.seg_rows, ng = p.multi_segs;
#define SC_MZ(A, R)                                                                         \
  cudaLaunchKernelEx(&cfg, fast_multi_kernel<A, R, true, true>, tin[0], tin[1], tout[0], tout[1], \
                     a, f, ns, sr, ng, steps, done)
#define SC_MK(A, R, G)                                                                      \
  cudaLaunchKernelEx(&cfg, fast_multi_kernel<A, R, G>, tin[0], tin[1], tout[0], tout[1], a, f, \
                     ns, sr, ng, steps, done)
  if (!p.general && a.constrained == nullptr && !a.zs) {
    if (p.ring == 5) return f.alpha1 ? SC_MK(true, 5, false) : SC_MK(false, 5, false);
    return f.alpha1 ? SC_MK(true, 4, false) : SC_MK(false, 4, false);
  }
  if (a.zs) {
    if (p.ring == 5) return f.alpha1 ? SC_MZ(true, 5) : SC_MZ(false, 5);
    return f.alpha1 ? SC_MZ(true, 4) : SC_MZ(false, 4);
  }
  if (p.ring == 5) return f.alpha1 ? SC_MK(true, 5, true) : SC_MK(false, 5, true);
  return f.alpha1 ? SC_MK(true, 4, true) : SC_MK(false, 4, true);
#undef SC_MK
#undef SC_MZ
}

}  // namespace scb
