// Wavefront temporal blocking of the FAST step: several timesteps per HBM
// round trip for batches of narrow cloths (nx <= 128: one 128-column strip per row).
//
// The reference advances every cloth one timestep per pass over memory (run_steps<T>,
// eval.cpp:48-59: forward_impulse -> add_plug_impulse -> advance_with_impulse, kernels.hpp:
// 179-282). The cell's reach is two rows (grid.cpp:14-30), and the FAST row pass finishes row
// R-2 as soon as row R has been seen (fast_rowpass.cuh). So a row's new state can replace its
// old state in place once the sweep is two rows past it, and a second sweep for the next
// timestep can follow three rows behind the first, reading what the first one wrote. This kernel
// runs W such sweeps at once:
//
//  * One persistent CTA per SM owns a contiguous range of cloths and W warps; warp w performs
//    timestep w of every pass of W timesteps. Rows stream through a ring of shared-memory slots
//    in a fixed order (pass-major, then cloth, then row, plus the two zero "tail" rows that
//    separate consecutive cloths), so every warp walks the same sequence of slot positions.
//  * Warp 0 also loads: TMA brings row positions a few steps ahead into their slots (rows past
//    the cloth are zero-filled out of bounds, exactly like the streaming kernel's tails).
//  * Warp w < W-1 writes the finished row back into its slot (level w+1) and arrives on the
//    slot's level barrier; warp w+1 waits on it before its row pass. The last level stores the
//    row to HBM (in place: the cloth's next pass reloads it later) and frees the slot for the
//    loader. Every barrier is an mbarrier (hardware-suspended waits).
//  * HBM traffic: 48 B per node per pass of W timesteps (48/W B per node-update). The arithmetic
//    per step is the streaming kernel's row pass and finish called unchanged, so the results are
//    bit-identical to W launches of fast_step_kernel.
// Pressure plugs (whose finish reads the row below the finished one at the old level) and mask
// output take the streaming kernel.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "fast_rowpass.cuh"
#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

using namespace fastrow;

constexpr int kWavePrefetch = 4;  // row positions the loader runs ahead of warp 0

// barriers addressed by 32-bit shared-window offsets computed once (no per-use address
// conversion); waits ask the hardware to suspend the warp until the phase flips
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// A wait that never hangs the device: after 20 s without the phase completing (a protocol bug,
// never a legitimate wait) the kernel traps, so the host sees a launch error instead of a hung
// GPU. The timer is read only on the retry path.
// hint_ns: the retry's suspend-time hint. try_wait with a hint compiles to NANOSLEEP.SYNCS — the
// warp sleeps until the barrier's phase completes (or the hint elapses) instead of spinning, so
// a waiting level costs no issue slots; its SMSP's other warps (the producing level among them)
// keep issuing. Without it the retry loop spun ~9 times per row (~100 issue slots per row step,
// ncu); time-neutral on config 5 (the spins filled issue slots no other warp could use).
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity, uint32_t hint_ns) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      ".reg .u64 t0, t1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "mov.u64 t0, %%globaltimer;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@p bra DONE_%=;\n"
      "mov.u64 t1, %%globaltimer;\n"
      "sub.u64 t1, t1, t0;\n"
      "setp.gt.u64 p, t1, 20000000000;\n"
      "@p trap;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(bar),
      "r"(parity), "r"(hint_ns)
      : "memory");
}
// an opaque copy: the compiler keeps the value in a register instead of re-deriving it (the
// shared-window base needs an S2R of the CTA id, which it would otherwise repeat per row)
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// W warps, one CTA per SM. Dynamic smem: [slots][ROWF] ring, then the barriers
// full[slots] (TMA landed), freeb[slots] (last level done with the slot),
// lev[W-1][slots] (level w+1 of the slot's row written back).
// FIN: 0 = collider-free cloths only (the collider finish compiled out), 1 = any collider set,
// 2 = collider cloths with one frictionless plane only (finish_plane_f: a small register peak, so
// the collider cloths run at 16 levels too)
template <bool ALPHA1, int W, int FIN, bool ZS>
__global__ void __launch_bounds__(32 * W, 1)
    wave_kernel(const __grid_constant__ CUtensorMap tmap_xy, const __grid_constant__ CUtensorMap tmap_z,
                const __grid_constant__ CUtensorMap tout_xy, const __grid_constant__ CUtensorMap tout_z,
                const StepArgs<float> a, const FastNet f, const int steps, const int slots,
                const int rev, const uint32_t hint) {
  extern __shared__ __align__(128) float ring[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(slots) * ROWF);
  uint64_t* freeb = full + slots;
  uint64_t* lev = freeb + slots;
  const int warp = static_cast<int>(threadIdx.x) >> 5;
  const int lane = static_cast<int>(threadIdx.x) & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&freeb[s], 32);
      for (int w = 0; w + 1 < W; ++w) mbar_init(&lev[w * slots + s], 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // this CTA's cloths [c0, c0 + m)
  const int B = a.batch;  // cloths [a.b_off, a.b_off + B) of the context
  const int c0 = a.b_off + static_cast<int>(static_cast<int64_t>(blockIdx.x) * B / gridDim.x);
  const int m = a.b_off + static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * B / gridDim.x) - c0;
  if (m <= 0) return;
  const int nx = a.nx, ny = a.ny;
  const int L = ny + 2;  // positions per (cloth, pass): rows 0..ny-1 and two zero tail rows
  const int passes = (steps + W - 1) / W;
  // position 0, 1: zero rows in front of the first cloth; then item i (pass i / m, cloth
  // c0 + i % m) row R at position 2 + i L + R
  const int Q = 2 + passes * m * L;

  const uint32_t ring_s = opaque(smem_u32(ring)), full_s = opaque(smem_u32(full));
  const uint32_t free_s = opaque(smem_u32(freeb)), lev_s = opaque(smem_u32(lev));
  // level of this warp: warp w runs timestep w of every pass (rev: timestep W-1-w, so the
  // hardware's issue priority of low warp slots goes to the deep levels)
  const int lvl = rev ? W - 1 - warp : warp;

  // Loader (level 0): row `crow` of cloth `cb` into slot `slot` (ring cycle `cyc_t`); rows past
  // the cloth (the two tail rows, and the two rows in front of the first cloth) come out of
  // bounds and are zero-filled by TMA. Stateless: warp 0 derives each target from its own
  // position, so the other warps carry no loader registers.
  // pass 0 reads a.in (tmap_*), later passes what the previous pass stored in a.out (tout_*);
  // a.in == a.out updates in place
  auto issue = [&](int ci_t, int crow, int slot, uint32_t cyc_t, bool first_pass) {
    const int cb = a.ids ? __ldg(a.ids + c0 + ci_t) : c0 + ci_t;
    const CUtensorMap* mxy = first_pass ? &tmap_xy : &tout_xy;
    const CUtensorMap* mz = first_pass ? &tmap_z : &tout_z;
    if (cyc_t > 0)  // the slot's previous position (cycle cyc_t - 1) must be released
      bar_wait(free_s + 8u * static_cast<uint32_t>(slot), (cyc_t - 1u) & 1u, hint);
    const uint32_t dst = ring_s + static_cast<uint32_t>(slot) * (ROWF * 4);
    const uint32_t bar = full_s + static_cast<uint32_t>(slot) * 8;
    if (elect_one()) {
      // the row was last written by generic stores (HBM: the previous pass's last level; smem:
      // the levels of the slot's previous row): order them before the async-proxy copy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "n"(ROW_BYTES)
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(mxy)), "r"(-4), "r"(crow), "r"(0), "r"(cb), "r"(bar)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst + Z_X * 4),
          "l"(reinterpret_cast<uint64_t>(mz)), "r"(-4), "r"(crow), "r"(0), "r"(cb), "r"(bar)
          : "memory");
    }
  };

  // Every barrier completes exactly once per ring cycle of its slot: the loader fills every
  // position, each level arrives for every position q-2 at position q (finished row or zero
  // tail row), the last level frees every position. So the phase a wait needs is the parity of
  // the position's ring cycle (a waiter never runs a whole cycle ahead of its producer: the ring
  // bounds the distance between levels).
  if (lvl == 0) {
    // positions 0, 1: zero rows (read as rows -2, -1 of the first cloth); 2 .. 2 + D - 1: item
    // 0's first D rows (D <= L: a pass has at least 4 positions); the main loop then keeps the
    // loader D positions ahead of warp 0
    for (int d = 0; d < 2 + kWavePrefetch; ++d)
      issue(0, d < 2 ? ny + d : d - 2, d % slots, static_cast<uint32_t>(d / slots), true);
    bar_wait(full_s, 0, hint);
    bar_wait(full_s + 8, 0, hint);
  }

  const uint32_t mL = 0xffffffffu;  // the lane's left edge leaves the grid only in lane 0
  const int ix0 = FW * lane;
  const uint32_t mLl = ix0 >= 1 ? mL : 0u;
  const uint32_t mRt = ix0 + 4 < nx ? 0xffffffffu : 0u;
  const bool lane_live = ix0 < nx;
  const int64_t S = a.plane_stride;
  // this warp's level barriers: it waits on lev[warp-1][], arrives on lev[warp][]
  const uint32_t lev_wait = lev_s + 8u * static_cast<uint32_t>((lvl > 0 ? lvl - 1 : 0) * slots);
  const uint32_t lev_mine = lev_s + 8u * static_cast<uint32_t>(lvl * slots);

  int sl = 2 % slots, s1 = 1, s2 = 0;  // slots of positions q, q-1, q-2
  uint32_t cyc = 0;                     // ring cycle of position q
#pragma unroll 1
  for (int p = 0; p < passes; ++p) {
    const int nlev = min(W, steps - p * W);
    if (lvl >= nlev) break;  // the remaining passes are shorter still
    const bool last = lvl == nlev - 1;
    const int k = a.k + p * W + lvl;  // this warp's step index in this pass
#pragma unroll 1
    for (int ci = 0; ci < m; ++ci) {
      const int b = a.ids ? __ldg(a.ids + c0 + ci) : c0 + ci;
      const ClothConst<float> cc = a.cloths[b];
      const Colliders col = FIN ? load_colliders(a, cc) : Colliders{};
      const int shape = FIN == 1 ? collider_shape(cc, col) : COLL_ANY;
      const bool simple = cc.n_spheres == 0 && cc.n_planes == 0;
      const float t_next = __fmul_rn(float(k + 1), cc.dt);
      float* const out_b = a.out + static_cast<int64_t>(b) * 6 * S;
      float2 P0[4], P1[4], P2[4];
      float2 Z0[2], Z1[2], Z2[2];
#pragma unroll
      for (int j = 0; j < 4; ++j) P0[j] = P1[j] = P2[j] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 2; ++j) Z0[j] = Z1[j] = Z2[j] = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int R = 0; R < L; ++R) {
        if (lvl == 0) {
          // position q + kWavePrefetch: row R + D of this cloth, or of the next item
          int rt = R + kWavePrefetch, ct = ci, pt = p;
          if (rt >= L) {
            rt -= L;
            if (++ct == m) {
              ct = 0;
              ++pt;
            }
          }
          const int st = sl + kWavePrefetch;
          if (pt < passes)
            issue(ct, rt, st >= slots ? st - slots : st, cyc + (st >= slots ? 1u : 0u), pt == 0);
          bar_wait(full_s + 8u * static_cast<uint32_t>(sl), cyc & 1u, hint);
        } else if (R < ny) {
          // tail rows are zeros the loader wrote (seen through level 0's wait chain); their
          // barrier phases still complete (arrivals below), keeping the cycle parity
          bar_wait(lev_wait + 8u * static_cast<uint32_t>(sl), cyc & 1u, hint);
        }
        float* rowR = ring + static_cast<size_t>(sl) * ROWF;
        float* row1 = ring + static_cast<size_t>(s1) * ROWF;
        float* row2 = ring + static_cast<size_t>(s2) * ROWF;
        if (R >= 2 && R < ny) {
          row_pass<ALPHA1, false, 0, ZS>(f, rowR, row1, row2, lane, mLl, mRt, 1.f, 1.f, P0, P1,
                                         P2, Z0, Z1, Z2);
        } else if (R < 2) {
          row_pass<ALPHA1, true, 0, ZS>(f, rowR, row1, row2, lane, mLl, mRt, R >= 1 ? 1.f : 0.f,
                                        0.f, P0, P1, P2, Z0, Z1, Z2);
        }
        const int Rf = R - 2;
        if (Rf >= 0) {
          if (lane_live) {
            float2 xs[4], vs[4];
            float xz[4], vz[4];
            finish_inputs<ZS>(row2, lane, xs, vs, xz, vz);
            // in place (box column of node ix0 is ix0 + 4) or, at the last level, to HBM; the two
            // destinations in separate branches so each store stays in its own address space
            if (!FIN || simple) {
              float xo[3][4], vo[3][4];
              finish_simple(a, cc, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo, vo);
              if (a.health) health_simple(a.health, b, k, Rf, nx, ix0, P0, Z0, xo, vo);
              if (last) {
                float* gxy = out_b + 2 * (static_cast<int64_t>(Rf) * a.pitch + ix0);
                float* gz = out_b + 4 * S + static_cast<int64_t>(Rf) * a.pitch + ix0;
                store_simple<ZS>(gxy, gxy + 2 * S, gz, gz + S, ix0, xo, vo);
              } else
                store_simple<ZS>(row2 + XY_X + 2 * (ix0 + 4), row2 + XY_V + 2 * (ix0 + 4),
                                 row2 + Z_X + ix0 + 4, row2 + Z_V + ix0 + 4, ix0, xo, vo);
            } else {
              float vo[4][3], xo[4][3];
              uint8_t mk[4];
              if (FIN == 2 || shape == COLL_PLANE1F)
                finish_plane_f(a, cc, col.p0, b, k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo,
                               vo, mk);
              else if (shape == COLL_PLANE1)
                finish_general<COLL_PLANE1>(a, cc, col, b, k, Rf, ix0, t_next, P0, Z0, xs, vs, xz,
                                            vz, xo, vo, mk);
              else
                finish_general(a, cc, col, b, k, Rf, ix0, t_next, P0, Z0, xs, vs, xz, vz, xo, vo,
                               mk);
              if (last) {
                float* gxy = out_b + 2 * (static_cast<int64_t>(Rf) * a.pitch + ix0);
                float* gz = out_b + 4 * S + static_cast<int64_t>(Rf) * a.pitch + ix0;
                store_general<ZS>(gxy, gxy + 2 * S, gz, gz + S, ix0, xo, vo);
              } else
                store_general<ZS>(row2 + XY_X + 2 * (ix0 + 4), row2 + XY_V + 2 * (ix0 + 4),
                                  row2 + Z_X + ix0 + 4, row2 + Z_V + ix0 + 4, ix0, xo, vo);
            }
          }
        }
        // position q-2 (row Rf in place, or a zero tail row) is ready for the next level; in the
        // last pass the next level may be idle (its barrier then simply keeps completing)
        if (lvl + 1 < W) bar_arrive(lev_mine + 8u * static_cast<uint32_t>(s2));
        if (last) {
          // the slot of position q-2 (row Rf, or a tail row of the previous cloth) is done
          if (Rf >= 0) asm volatile("fence.proxy.async.global;" ::: "memory");
          bar_arrive(free_s + 8u * static_cast<uint32_t>(s2));
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          Z0[j] = Z1[j];
          Z1[j] = Z2[j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          P0[j] = P1[j];
          P1[j] = P2[j];
        }
        s2 = s1;
        s1 = sl;
        if (++sl == slots) {
          sl = 0;
          ++cyc;
        }
      }
    }
  }
  // warp 0 drains nothing: every issued load was consumed (the loader stops at Q)
}

template <bool ALPHA1, int W, int FIN, bool ZS>
void* wave_ptr() {
  return reinterpret_cast<void*>(wave_kernel<ALPHA1, W, FIN, ZS>);
}

template <int W, int FIN>
void* pick_wave_f(bool alpha1, bool zs) {
  return zs ? (alpha1 ? wave_ptr<true, W, FIN, true>() : wave_ptr<false, W, FIN, true>())
            : (alpha1 ? wave_ptr<true, W, FIN, false>() : wave_ptr<false, W, FIN, false>());
}

template <int W>
void* pick_wave_w(bool alpha1, int fin, bool zs) {
  return fin == 2 ? pick_wave_f<W, 2>(alpha1, zs)
         : fin == 1 ? pick_wave_f<W, 1>(alpha1, zs)
                    : pick_wave_f<W, 0>(alpha1, zs);
}

void* pick_wave(int levels, bool alpha1, int fin, bool zs) {
  switch (levels) {
    case 8: return pick_wave_w<8>(alpha1, fin, zs);
    case 12: return pick_wave_w<12>(alpha1, fin, zs);
    default: return pick_wave_w<16>(alpha1, fin, zs);
  }
}

}  // namespace

size_t wave_smem_bytes(int levels, int slots) {
  return sizeof(float) * static_cast<size_t>(slots) * ROWF +
         sizeof(uint64_t) * static_cast<size_t>(slots) * (2 + (levels - 1));
}

WavePlan plan_wave(int nx, int ny, int batch, int device, bool general, int max_ctas,
                   bool plane_only) {
  WavePlan p{};
  p.ok = false;
  if (nx > STRIP || ny < 2 || batch < 1) return p;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  // 8 levels when a cloth-pass is too short for the sweeps three rows apart
  const int fin = general ? (plane_only ? 2 : 1) : 0;
  // 12 levels (384 threads, up to 168 registers): measured faster than 16 for collider-free
  // batches (config 5's collider-free group 572.5 -> 561.7 us per class-grouped step; a batch of
  // collider-free cloths alone 570 -> 557) and required by the general collider finish (its
  // register peak spills at 128); 16 for the lean plane-only finish (605 us per 4096 plane cloths)
  int want = fin == 2 ? 16 : 12;
  if (const char* env = std::getenv("SC_WAVE_LEVELS")) want = std::atoi(env);
  p.ctas = std::min(batch, max_ctas > 0 ? std::min(max_ctas, sms) : sms);
  const int m_min = batch / p.ctas;  // cloths of the least-loaded CTA
  int slots = 0;
  for (int levels : {16, 12, 8}) {
    if (levels > want) continue;
    // ring: as many slots as fit (<= 64: the per-slot parity bits live in one 64-bit word), no
    // more than one cloth-pass of positions per CTA (a cloth's next pass must never load a row
    // before this pass stored it), and enough for W sweeps three rows apart plus prefetch
    int sl = 64;
    while (sl > 0 && wave_smem_bytes(levels, sl) > static_cast<size_t>(smem_optin)) --sl;
    sl = static_cast<int>(std::min<int64_t>(sl, static_cast<int64_t>(m_min) * (ny + 2)));
    if (sl >= 3 * levels + kWavePrefetch + 4) {
      p.levels = levels;
      slots = sl;
      break;
    }
  }
  if (slots == 0) return p;
  p.slots = slots;
  p.rev = 0;
  p.hint_ns = 1000000;  // 1 ms: a wait ends on the barrier, not on the hint
  if (const char* env = std::getenv("SC_WAVE_REV")) p.rev = std::atoi(env);
  if (const char* env = std::getenv("SC_WAVE_HINT")) p.hint_ns = static_cast<uint32_t>(std::atoi(env));
  p.smem = wave_smem_bytes(p.levels, slots);
  p.general = general;
  p.fin = fin;
  for (bool a1 : {true, false})
    for (bool zs : {true, false})
      cudaFuncSetAttribute(pick_wave(p.levels, a1, fin, zs),
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
  p.ok = true;
  return p;
}

cudaError_t launch_wave(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tmap,
                        const CUtensorMap* tmap_out, const WavePlan& p, int steps,
                        cudaStream_t stream) {
  if (steps <= 0 || a.batch <= 0) return cudaSuccess;
  void* fn = pick_wave(p.levels, f.alpha1 != 0, p.fin, a.zs != 0);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.ctas));
  cfg.blockDim = dim3(static_cast<unsigned>(32 * p.levels));
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = stream;
  cfg.numAttrs = 0;
  const int slots = p.slots;
  int rev = p.rev;
  uint32_t hint = p.hint_ns;
  void* args[] = {const_cast<CUtensorMap*>(&tmap[0]), const_cast<CUtensorMap*>(&tmap[1]),
                  const_cast<CUtensorMap*>(&tmap_out[0]), const_cast<CUtensorMap*>(&tmap_out[1]),
                  const_cast<StepArgs<float>*>(&a), const_cast<FastNet*>(&f),
                  const_cast<int*>(&steps), const_cast<int*>(&slots), &rev, &hint};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace scb
