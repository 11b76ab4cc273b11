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

#include "fast_rowpass.cuh"
#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

using namespace fastrow;

constexpr int ONLY_PLANE_F = 1, ONLY_SPHERE = 2;

// One unit (cloth b, 128-column strip, rows [y0, y1)) of one step, reading a.in through the
// tensor maps and writing a.out. `phase` carries the ring barriers' parity bits across calls
// (the persistent kernel runs many units / steps on the same ring).
// GEN = false: no cloth of the launch takes the collider / pressure / mask finish, which is
// compiled out; ONLY (with GEN): every collider cloth has one collider of one kind and no
// pressure plug — the collider finish is that kind's alone (fewer live registers than the
// general dispatch): ONLY_PLANE_F finish_plane_f (one frictionless plane), ONLY_SPHERE
// finish_general<COLL_SPHERE1> (one sphere)
template <bool ALPHA1, int RING, bool PEER = false, bool GEN = true, bool ZS = false,
          int ONLY = 0>
__device__ __forceinline__ void run_unit(const CUtensorMap* tmap_xy, const CUtensorMap* tmap_z,
                                         const StepArgs<float>& a, const FastNet& f,
                                         const ClothConst<float>& cc, int b, int strip, int y0,
                                         int y1, float* ring, uint64_t* full,
                                         float (*scratch)[13], uint32_t& phase) {
  const int lane = threadIdx.x;
  const int x0 = strip * STRIP;
  const int ix0 = x0 + FW * lane;
  const int nx = a.nx, ny = a.ny;

  // Rows y0-2 .. y1+1 pass through the ring; arithmetic starts at row y0 (the two rows below
  // only feed rows < y0) and the last two steps (rows y1, y1+1) only finish rows y1-2, y1-1.
  const int r_first = y0 - 2;
  const int r_last = y1 + 1;

  const int64_t nodes = static_cast<int64_t>(nx) * ny;

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
  // the cloth's constants (their loads were issued before the grid dependency, fast_step_kernel)
  // are first consumed here, behind the TMA issue: the collider loads that depend on them and the
  // first rows' flight overlap instead of queueing one L2 round trip after the other
  const Colliders col = GEN ? load_colliders(a, cc) : Colliders{};
  const int shape = GEN && !ONLY ? collider_shape(cc, col) : COLL_ANY;
  const bool simple = cc.n_spheres == 0 && cc.n_planes == 0 && !cc.plug_pressure &&
                      a.constrained == nullptr;
  const float t_next = a.use_t_override ? a.t_override : __fmul_rn(float(a.k + 1), cc.dt);
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
        finish_inputs<ZS>(row2, lane, xs, vs, xz, vz);
        float xo[3][4], vo[3][4];
        finish_simple(a, cc, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo, vo);
        if (a.health) health_simple(a.health, b, a.k, Rf, nx, ix0, P0, Z0, xo, vo);
        store_simple<ZS>(oxy, oxy + 2 * S, oz, oz + S, ix0, xo, vo);
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
      } else if (ONLY || !cc.plug_pressure) {
        // colliders and/or the contact mask (finish_general), packed stores
        float2 xs[4], vs[4];
        float xz[4], vz[4];
        finish_inputs<ZS>(row2, lane, xs, vs, xz, vz);
        float vo[4][3], xo[4][3];
        uint8_t mk[4];
        if (ONLY == ONLY_SPHERE)
          finish_general<COLL_SPHERE1>(a, cc, col, b, a.k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz,
                                       xo, vo, mk);
        else if (ONLY == ONLY_PLANE_F || shape == COLL_PLANE1F)
          finish_plane_f(a, cc, col.p0, b, a.k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo, vo,
                         mk);
        else if (shape == COLL_PLANE1)
          finish_general<COLL_PLANE1>(a, cc, col, b, a.k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz,
                                      xo, vo, mk);
        else if (shape == COLL_SPHERE1)
          finish_general<COLL_SPHERE1>(a, cc, col, b, a.k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz,
                                       xo, vo, mk);
        else
          finish_general(a, cc, col, b, a.k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo, vo, mk);
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

// debug: [units][3] start, end, sm/warp. In constant memory: the pointer is tested at the top of
// every unit, and a global-memory variable put an L2 round trip (~0.4 us) in front of the first
// TMA issue (ncu: 4% of config 3's stall samples on that load and its consumers)
__constant__ unsigned long long* g_unit_times = nullptr;

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
          bool ZS = false, int ONLY = 0>
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
  if (a.ids) b = __ldg(a.ids + b);
  // the cloth's constants do not depend on the previous step: their loads go out before the
  // grid dependency (consumed in run_unit behind the first TMA issue)
  const ClothConst<float> cc = a.cloths[b];
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
    run_unit<ALPHA1, RING, PEER, GEN, ZS, ONLY>(&tmap_xy, &tmap_z, a, f, cc, b, strip, y0, y1, ring,
                                                full, scratch, phase);
  if (times && threadIdx.x == 0) times[3 * unit + 1] = gtimer();
  // let the next step's grid launch once every CTA of this one is done with its work (an early
  // trigger would let waiting CTAs occupy SM slots a multi-wave grid still needs)
  asm volatile("griddepcontrol.launch_dependents;");
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
  f.live = 0;
  for (int c = 0; c < kChannels; ++c)
    if (f.wl[c] != 0.0f || f.wn[c] != 0.0f || f.wd[c] != 0.0f) f.live |= 1u << c;
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



template <bool ALPHA1, bool ZS, int ONLY>
void* only_kernel_ptr() {
  return reinterpret_cast<void*>(fast_step_kernel<ALPHA1, 4, false, true, SC_FAST_MINB, ZS, ONLY>);
}

size_t fast_smem_bytes(int ring, bool general) {
  size_t pad = 0;
  if (const char* env = std::getenv("SC_FAST_SMEM_PAD")) pad = std::strtoul(env, nullptr, 10);
  // the per-lane impulse scratch serves only the pressure finish (RING = 5); the collider / mask
  // finish keeps everything in registers, so `general` alone costs no shared memory
  (void)general;
  return sizeof(float) * (ring * ROWF + (ring == 5 ? 32 * 13 : 0)) + pad;  // pad: tuning knob
}

FastPlan plan_fast(int nx, int rows, int batch, int device, bool pressure, bool general,
                   int max_sms) {
  FastPlan p{};
  p.ring = pressure ? 5 : 4;
  p.general = general;
  p.n_strips = (nx + STRIP - 1) / STRIP;
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (max_sms > 0) sms = std::min(sms, max_sms);
  const size_t smem = fast_smem_bytes(p.ring, general);
  for (void* k : {pick_kernel(true, p.ring), pick_kernel(false, p.ring),
                  p.ring == 5 ? simple_kernel_ptr<true, 5>() : simple_kernel_ptr<true, 4>(),
                  p.ring == 5 ? simple_kernel_ptr<false, 5>() : simple_kernel_ptr<false, 4>(),
                  p.ring == 5 ? wide_kernel_ptr<true, 5>() : wide_kernel_ptr<true, 4>(),
                  p.ring == 5 ? zs_kernel_ptr<true, 5>(false) : zs_kernel_ptr<true, 4>(false),
                  p.ring == 5 ? zs_kernel_ptr<false, 5>(false) : zs_kernel_ptr<false, 4>(false),
                  p.ring == 5 ? zs_kernel_ptr<true, 5>(true) : zs_kernel_ptr<true, 4>(true),
                  p.ring == 5 ? zs_kernel_ptr<false, 5>(true) : zs_kernel_ptr<false, 4>(true),
                  p.ring == 5 ? wide_kernel_ptr<false, 5>() : wide_kernel_ptr<false, 4>(),
                  p.ring == 5 ? peer_kernel_ptr<true, 5>() : peer_kernel_ptr<true, 4>(),
                  p.ring == 5 ? peer_kernel_ptr<false, 5>() : peer_kernel_ptr<false, 4>(),
                  only_kernel_ptr<true, false, 1>(), only_kernel_ptr<false, false, 1>(),
                  only_kernel_ptr<true, true, 1>(), only_kernel_ptr<false, true, 1>(),
                  only_kernel_ptr<true, false, 2>(), only_kernel_ptr<false, false, 2>(),
                  only_kernel_ptr<true, true, 2>(), only_kernel_ptr<false, true, 2>()})
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
      // a single wave needs ~70% of the slots to keep the SMSPs issuing (config 3: 4-row units
      // filling 86% of the slots 21.7 us per step, 5-row units filling 69% 21.0)
      const double fill = waves == 1 ? std::min(1.0, units / (0.7 * slots))
                                     : static_cast<double>(units) / static_cast<double>(waves * slots);
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
  p.chunk_wide = false;
  int occ_w = 0;
  if (!general) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ_w, p.ring == 5 ? wide_kernel_ptr<true, 5>() : wide_kernel_ptr<true, 4>(), 32, smem);
    p.wide = occ_w > 0 && rows / best_segs >= 32;
    // under chunked stepping the wide-register kernel wins even on short segments (config 2:
    // 39.3 -> 38.5 us per step; the concurrent chunks supply the occupancy the 12 CTAs per SM
    // lack)
    p.chunk_wide = occ_w > 0;
    if (const char* env = std::getenv("SC_FAST_WIDE")) p.wide = p.chunk_wide = occ_w > 0 && std::atoi(env) != 0;
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
    const int64_t slots = static_cast<int64_t>(sms) * (p.chunk_wide ? occ_w : occ);
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
  // every collider cloth has one collider of one kind, no mask output (a collider-free cloth
  // asked for its mask takes the general finish): that kind's finish alone
  if (!peer && p.general && p.only != 0 && p.ring == 4 && a.constrained == nullptr) {
#define SC_FO(A, Z, O)                                                                        \
  cudaLaunchKernelEx(&cfg, fast_step_kernel<A, 4, false, true, SC_FAST_MINB, Z, O>, txy, tz, a, f, \
                     ns, sr, ng)
    if (p.only == ONLY_PLANE_F)
      return a.zs ? (f.alpha1 ? SC_FO(true, true, 1) : SC_FO(false, true, 1))
                  : (f.alpha1 ? SC_FO(true, false, 1) : SC_FO(false, false, 1));
    return a.zs ? (f.alpha1 ? SC_FO(true, true, 2) : SC_FO(false, true, 2))
                : (f.alpha1 ? SC_FO(true, false, 2) : SC_FO(false, false, 2));
#undef SC_FO
  }
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

}  // namespace scb
