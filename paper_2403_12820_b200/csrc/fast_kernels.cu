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
constexpr int RING = 6;            // staged rows: R-3 .. R+2
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

// Edge contribution to its origin node a (channel ca) and far node b (channel cb = -ca):
//   a: acc += dx*wL'_ca + s*(wN'_ca + dv*wD'_ca)
//   b: acc += dx*(-wL'_cb) + s*(dv*wD'_cb - wN'_cb)
// with dx = x_a - x_b, dv = v_a - v_b, s = dx * rsqrt(1 + alpha'_c dx^2) and the gains folded
// into the primed weights (wL' = g wL, wN' = g wN, wD' = g^2 wD, alpha' = alpha g^2).
template <bool ALPHA1>
__device__ __forceinline__ void edge(const FastNet& f, int ca, int cb, float xa, float xb,
                                     float va, float vb, bool push_a, bool push_b, float& acc_a,
                                     float& acc_b) {
  const float dx = xa - xb;
  const float dv = va - vb;
  const float q = ALPHA1 ? fmaf(dx, dx, 1.0f) : fmaf(dx * f.alpha[ca], dx, 1.0f);
  const float s = dx * rsqrtf(q);
  if (push_a) {
    const float t = fmaf(dv, f.wd[ca], f.wn[ca]);
    acc_a = fmaf(dx, f.wl[ca], acc_a);
    acc_a = fmaf(s, t, acc_a);
  }
  if (push_b) {
    const float t = fmaf(dv, f.wd[cb], f.nwn[cb]);
    acc_b = fmaf(dx, f.nwl[cb], acc_b);
    acc_b = fmaf(s, t, acc_b);
  }
}

template <bool ALPHA1>
__global__ void __launch_bounds__(32) fast_step_kernel(const __grid_constant__ CUtensorMap tmap,
                                                      const StepArgs<float> a, const FastNet f,
                                                      const int n_strips, const int seg_rows,
                                                      const int n_segs) {
  extern __shared__ __align__(128) float ring[];  // [RING][6][BOXW]
  __shared__ __align__(8) uint64_t full[RING];

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

  const int r_first = y0 - 2;  // first row entering the window
  const int r_last = y1 + 1;   // last row entering the window (finishes row y1-1)

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
    if (r_first + 1 <= r_last) issue(r_first + 1);
  }

  // lane-constant edge validity (both endpoints inside the grid columns)
  bool vE[5], vE2[6], vNE[5], vNW[5];
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    const int c = ix0 - 1 + e;
    vE[e] = c >= 0 && c + 1 < nx;
    vNE[e] = c >= 0 && c + 1 < nx;
    const int cw = ix0 + e;
    vNW[e] = cw - 1 >= 0 && cw < nx;
  }
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    const int c = ix0 - 2 + e;
    vE2[e] = c >= 0 && c + 2 < nx;
  }
  bool vN[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) vN[k] = ix0 + k < nx;

  const ClothConst<float> cc = a.cloths[b];
  const int64_t nodes = static_cast<int64_t>(nx) * ny;
  float* out_b = a.out + static_cast<int64_t>(b) * 6 * a.plane_stride;

  float A0[4][3], A1[4][3], A2[4][3];  // rows R-2, R-1, R
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int d = 0; d < 3; ++d) A0[k][d] = A1[k][d] = A2[k][d] = 0.0f;

#pragma unroll 1
  for (int R = r_first; R <= r_last; ++R) {
    const int t = R - r_first;
    __syncwarp();
    if (lane == 0 && R + 2 <= r_last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(R + 2);
    }
    mbar_wait(&full[t % RING], (t / RING) & 1);

    const float* rowR = ring + (t % RING) * ROWF;
    const float* row1 = ring + ((t + RING - 1) % RING) * ROWF;
    const float* row2 = ring + ((t + RING - 2) % RING) * ROWF;
    const bool okR = R >= 0 && R < ny;
    const bool ok1 = okR && R - 1 >= 0;  // rows R-1 and R both in the grid
    const bool ok2 = okR && R - 2 >= 0;  // rows R-2 and R both in the grid
    const bool have1 = t >= 1, have2 = t >= 2;

#pragma unroll
    for (int d = 0; d < 3; ++d) {
      // row R and R-1: columns ix0-2 .. ix0+5 <-> box index 4*lane+2 .. 4*lane+9
      // (LDS.64 + LDS.128 + LDS.64); row R-2: columns ix0 .. ix0+3 (one LDS.128)
      float xr[8], vr[8], x1[8], v1[8], x2[8], v2[8];
      auto load8 = [&](const float* base, float* o) {
        const float2 l = *reinterpret_cast<const float2*>(base + FW * lane + 2);
        const float4 m = *reinterpret_cast<const float4*>(base + FW * lane + 4);
        const float2 r = *reinterpret_cast<const float2*>(base + FW * lane + 8);
        o[0] = l.x; o[1] = l.y; o[2] = m.x; o[3] = m.y; o[4] = m.z; o[5] = m.w; o[6] = r.x; o[7] = r.y;
      };
      load8(rowR + d * BOXW, xr);
      load8(rowR + (3 + d) * BOXW, vr);
      if (have1) {
        load8(row1 + d * BOXW, x1);
        load8(row1 + (3 + d) * BOXW, v1);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) x1[j] = v1[j] = 0.0f;
      }
      if (have2) {
        const float4 a0 = *reinterpret_cast<const float4*>(row2 + d * BOXW + FW * lane + 4);
        const float4 c0 = *reinterpret_cast<const float4*>(row2 + (3 + d) * BOXW + FW * lane + 4);
        x2[2] = a0.x; x2[3] = a0.y; x2[4] = a0.z; x2[5] = a0.w;
        v2[2] = c0.x; v2[3] = c0.y; v2[4] = c0.z; v2[5] = c0.w;
      } else {
#pragma unroll
        for (int j = 2; j < 6; ++j) x2[j] = v2[j] = 0.0f;
      }
      // init row R: b + v*wV
#pragma unroll
      for (int k = 0; k < 4; ++k) A2[k][d] = fmaf(vr[k + 2], f.wv, f.b[d]);

      float dummy = 0.0f;
      // E edges in row R: a = col ix0-1+e (box j = e+1), b = col ix0+e (j = e+2)
#pragma unroll
      for (int e = 0; e < 5; ++e) {
        float& acc_a = e >= 1 ? A2[e >= 1 ? e - 1 : 0][d] : dummy;
        float& acc_b = e <= 3 ? A2[e <= 3 ? e : 0][d] : dummy;
        edge<ALPHA1>(f, 0, 2, xr[e + 1], xr[e + 2], vr[e + 1], vr[e + 2], okR && vE[e] && e >= 1,
                     okR && vE[e] && e <= 3, acc_a, acc_b);
      }
      // E2 edges in row R: a = col ix0-2+e (j = e), b = col ix0+e (j = e+2)
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        float& acc_a = e >= 2 ? A2[e >= 2 ? e - 2 : 0][d] : dummy;
        float& acc_b = e <= 3 ? A2[e <= 3 ? e : 0][d] : dummy;
        edge<ALPHA1>(f, 8, 10, xr[e], xr[e + 2], vr[e], vr[e + 2], okR && vE2[e] && e >= 2,
                     okR && vE2[e] && e <= 3, acc_a, acc_b);
      }
      // N edges (R-1 -> R) and N2 edges (R-2 -> R), owned columns
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        edge<ALPHA1>(f, 1, 3, x1[k + 2], xr[k + 2], v1[k + 2], vr[k + 2], ok1 && vN[k],
                     ok1 && vN[k], A1[k][d], A2[k][d]);
        edge<ALPHA1>(f, 9, 11, x2[k + 2], xr[k + 2], v2[k + 2], vr[k + 2], ok2 && vN[k],
                     ok2 && vN[k], A0[k][d], A2[k][d]);
      }
      // NE edges: a = (ix0-1+e, R-1) (j = e+1), b = (ix0+e, R) (j = e+2)
#pragma unroll
      for (int e = 0; e < 5; ++e) {
        float& acc_a = e >= 1 ? A1[e >= 1 ? e - 1 : 0][d] : dummy;
        float& acc_b = e <= 3 ? A2[e <= 3 ? e : 0][d] : dummy;
        edge<ALPHA1>(f, 4, 6, x1[e + 1], xr[e + 2], v1[e + 1], vr[e + 2], ok1 && vNE[e] && e >= 1,
                     ok1 && vNE[e] && e <= 3, acc_a, acc_b);
      }
      // NW edges: a = (ix0+e, R-1) (j = e+2), b = (ix0+e-1, R) (j = e+1)
#pragma unroll
      for (int e = 0; e < 5; ++e) {
        float& acc_a = e <= 3 ? A1[e <= 3 ? e : 0][d] : dummy;
        float& acc_b = e >= 1 ? A2[e >= 1 ? e - 1 : 0][d] : dummy;
        edge<ALPHA1>(f, 5, 7, x1[e + 2], xr[e + 1], v1[e + 2], vr[e + 1], ok1 && vNW[e] && e <= 3,
                     ok1 && vNW[e] && e >= 1, acc_a, acc_b);
      }
    }

    // row R-2 is complete: plug, integrate, collide, pin, store
    const int Rf = R - 2;
    if (Rf >= y0 && Rf < y1) {
      const float* rowf = row2;
      float xs[4][3], vs[4][3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const float4 p = *reinterpret_cast<const float4*>(rowf + d * BOXW + FW * lane + 4);
        const float4 q = *reinterpret_cast<const float4*>(rowf + (3 + d) * BOXW + FW * lane + 4);
        xs[0][d] = p.x; xs[1][d] = p.y; xs[2][d] = p.z; xs[3][d] = p.w;
        vs[0][d] = q.x; vs[1][d] = q.y; vs[2][d] = q.z; vs[3][d] = q.w;
      }
      float xo[4][3], vo[4][3];
      uint8_t mk[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ix = ix0 + k;
        const int64_t gnode = static_cast<int64_t>(Rf) * nx + ix;
        float imp[3] = {A0[k][0], A0[k][1], A0[k][2]};
        if (a.health && ix < nx && !(isfinite(imp[0]) && isfinite(imp[1]) && isfinite(imp[2]))) {
          const unsigned long long key = (static_cast<unsigned long long>(a.k + 1) << 32) |
                                         static_cast<unsigned long long>(gnode);
          atomicMin(&a.health[b].impulse_key, key);
        }
        if (cc.plug_pressure) {
          const float* rs = ring + ((t + RING - 3) % RING) * ROWF;  // row Rf-1
          const float* rn = row1;                                   // row Rf+1
          const int j = FW * lane + 4 + k;
          const bool interior = ix >= 1 && ix <= nx - 2 && Rf >= 1 && Rf <= ny - 2;
          float e[3], n[3], w[3], s[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            e[d] = __fsub_rn(xs[k][d], rowf[d * BOXW + j + 1]);
            n[d] = __fsub_rn(xs[k][d], rn[d * BOXW + j]);
            w[d] = __fsub_rn(xs[k][d], rowf[d * BOXW + j - 1]);
            s[d] = __fsub_rn(xs[k][d], rs[d * BOXW + j]);
          }
          pressure_plug(cc, interior, e, n, w, s, imp);
        }
        plug_tail(cc, vs[k], imp);
        advance_node(a, cc, gnode, xs[k], vs[k], imp, xo[k], vo[k], mk[k]);
      }
      float* o = out_b + static_cast<int64_t>(Rf - a.g0) * a.pitch + ix0;
      if (ix0 + 3 < nx) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          *reinterpret_cast<float4*>(o + d * a.plane_stride) =
              make_float4(xo[0][d], xo[1][d], xo[2][d], xo[3][d]);
          *reinterpret_cast<float4*>(o + (3 + d) * a.plane_stride) =
              make_float4(vo[0][d], vo[1][d], vo[2][d], vo[3][d]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (ix0 + k >= nx) break;
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            o[d * a.plane_stride + k] = xo[k][d];
            o[(3 + d) * a.plane_stride + k] = vo[k][d];
          }
        }
      }
      if (a.constrained) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (ix0 + k < nx) a.constrained[b * nodes + static_cast<int64_t>(Rf) * nx + ix0 + k] = mk[k];
      }
      if (a.health) {
        bool fin = true;
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int d = 0; d < 3; ++d)
            fin = fin && (ix0 + k >= nx || (isfinite(xo[k][d]) && isfinite(vo[k][d])));
        if (!fin) atomicMin(&a.health[b].state_frame, a.k + 1);
      }
    }
    // rotate accumulator rows
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        A0[k][d] = A1[k][d];
        A1[k][d] = A2[k][d];
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

bool fast_supported(const NetConst<float>& net) {
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
