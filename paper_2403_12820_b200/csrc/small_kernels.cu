// Small-cloth FAST stepping: cloths of at most 1024 nodes (BASELINE config 1,
// 32 x 32) advance all their timesteps in one launch, one CTA per cloth, one thread per node, the
// whole state double-buffered in shared memory.
//
// The row-pass kernels give a 1024-node cloth eight live lanes of one warp per row and a latency
// chain of 32 rows per timestep (the wavefront kernel: 6 us per step, 2.6x the reference's
// 16-thread CPU rollout). Here every node of the cloth is a thread: a timestep is one evaluation
// of the reference cell per node — the twelve channels in the reference order (forward_impulse<T>,
// kernels.hpp:265-282; neighbour offsets grid.cpp:14-30, masked channels skipped), FAST arithmetic
// (FMA, rsqrt.approx ISRU, gains folded into the weights as in fast_kernels.cu) — followed by the
// plug tail and advance (add_plug_impulse / advance_with_impulse, kernels.hpp:179-252: the simple
// finish's contracted chain for collider-free cloths, the IEEE chain of sc_device.cuh otherwise,
// so contact decisions match PARITY), and one CTA barrier. The per-node channel order is the
// reference's, not the edge-shared order of the row pass: results are within the FAST tolerance
// of the oracle (tests/test_gpu_small.py) but not bit-identical to the other FAST kernels.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "fast_rowpass.cuh"
#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

constexpr int kSmallMaxNodes = 1024;
// canonical channel order E,N,W,S,NE,NW,SW,SE,E2,N2,W2,S2 (grid.cpp:14-30)
__constant__ int kSmallDx[kChannels] = {1, 0, -1, 0, 1, -1, -1, 1, 2, 0, -2, 0};
__constant__ int kSmallDy[kChannels] = {0, 1, 0, -1, 1, 1, -1, -1, 0, 2, 0, -2};

template <bool ALPHA1, bool GEN>
__global__ void __launch_bounds__(kSmallMaxNodes, 1)
    small_kernel(const StepArgs<float> a, const FastNet f, const int steps) {
  extern __shared__ __align__(16) float sm[];  // [2 buffers][6 components][n nodes]
  const int nx = a.nx, ny = a.ny, n = nx * ny;
  const int b = a.b_off + static_cast<int>(blockIdx.x);
  const int64_t S = a.plane_stride;
  const bool zs = a.zs != 0;
  const float* in_b = a.in + static_cast<int64_t>(b) * 6 * S;
  float* out_b = a.out + static_cast<int64_t>(b) * 6 * S;
  for (int q = threadIdx.x; q < 6 * n; q += blockDim.x) {
    const int p = q / n, i = q - p * n;
    sm[q] = in_b[elem_index(p, i / nx, i % nx, a.pitch, S, zs)];
  }
  const ClothConst<float> cc = a.cloths[b];
  const bool simple = cc.n_spheres == 0 && cc.n_planes == 0;
  const int i = static_cast<int>(threadIdx.x);
  const bool live = i < n;
  const int ix = live ? i % nx : 0, iy = live ? i / nx : 0;
  uint32_t valid = 0;  // channel c's neighbour is inside the grid
  int nbr[kChannels];
#pragma unroll
  for (int c = 0; c < kChannels; ++c) {
    const int jx = ix + kSmallDx[c], jy = iy + kSmallDy[c];
    nbr[c] = jy * nx + jx;
    if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) valid |= 1u << c;
  }
  const int64_t gnode = static_cast<int64_t>(iy) * nx + ix;
  __syncthreads();

#pragma unroll 1
  for (int s = 0; s < steps; ++s) {
    const float* cur = sm + (s & 1) * 6 * n;
    float* nxt = sm + ((s & 1) ^ 1) * 6 * n;
    if (live) {
      const int k = a.k + s;
      const float t_next = __fmul_rn(float(k + 1), cc.dt);
      float x[3], v[3], acc[3];
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        x[d] = cur[d * n + i];
        v[d] = cur[(3 + d) * n + i];
        acc[d] = fmaf(v[d], f.wv, f.b[d]);  // b_L + v wV
      }
#pragma unroll
      for (int c = 0; c < kChannels; ++c) {
        if (!((valid >> c) & 1u)) continue;
        const int j = nbr[c];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float dx = x[d] - cur[d * n + j];
          const float dv = v[d] - cur[(3 + d) * n + j];
          const float q = ALPHA1 ? fmaf(dx, dx, 1.0f) : fmaf(dx * f.alpha[c], dx, 1.0f);
          const float r = fastrow::rsqrt_q(q);
          const float w = fmaf(r, fmaf(dv, f.wd[c], f.wn[c]), f.wl[c]);
          acc[d] = fmaf(dx, w, acc[d]);
        }
      }
      if (a.health) {  // non-finite cell impulse: first (step, node) (net.cpp:139-140)
        if (!(isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]))) {
          const unsigned long long key = (static_cast<unsigned long long>(k + 1) << 32) |
                                         static_cast<unsigned long long>(gnode);
          atomicMin(&a.health[b].impulse_key, key);
        }
      }
      float xo[3], vo[3];
      uint8_t mk = 0;
      if (!GEN || simple) {
        // plug gravity / drag and integrate, contracted (the simple finish of fast_rowpass.cuh)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const float imp = fmaf(v[d], -cc.fin[3], acc[d] + cc.fin[d]);
          vo[d] = v[d] + imp;
          xo[d] = fmaf(vo[d], cc.dt, x[d]);
        }
      } else {
        // plug tail, then advance_with_impulse in IEEE round-to-nearest operations
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
      repin_t(a, cc, iy, gnode, t_next, xo, vo, mk);  // Dirichlet re-pin last
      if (a.health && !(isfinite(xo[0]) && isfinite(xo[1]) && isfinite(xo[2]) &&
                        isfinite(vo[0]) && isfinite(vo[1]) && isfinite(vo[2])))
        atomicMin(&a.health[b].state_frame, k + 1);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        nxt[d * n + i] = xo[d];
        nxt[(3 + d) * n + i] = vo[d];
      }
    }
    __syncthreads();
  }
  const float* fin = sm + (steps & 1) * 6 * n;
  for (int q = threadIdx.x; q < 6 * n; q += blockDim.x) {
    const int p = q / n, j = q - p * n;
    out_b[elem_index(p, j / nx, j % nx, a.pitch, S, zs)] = fin[q];
  }
}

void* pick_small(bool alpha1, bool gen) {
  if (gen)
    return alpha1 ? reinterpret_cast<void*>(small_kernel<true, true>)
                  : reinterpret_cast<void*>(small_kernel<false, true>);
  return alpha1 ? reinterpret_cast<void*>(small_kernel<true, false>)
                : reinterpret_cast<void*>(small_kernel<false, false>);
}

}  // namespace

bool small_supported(int nx, int ny) {
  if (const char* env = std::getenv("SC_SMALL"))
    if (std::atoi(env) == 0) return false;
  return nx >= 1 && ny >= 1 && nx * ny <= kSmallMaxNodes;
}

cudaError_t launch_small(const StepArgs<float>& a, const FastNet& f, bool general, int steps,
                         cudaStream_t stream) {
  if (steps <= 0 || a.batch <= 0) return cudaSuccess;
  const int n = a.nx * a.ny;
  const size_t smem = sizeof(float) * 12 * static_cast<size_t>(n);
  void* fn = pick_small(f.alpha1 != 0, general);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(a.batch));
  cfg.blockDim = dim3(static_cast<unsigned>((n + 31) / 32 * 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.numAttrs = 0;
  void* args[] = {const_cast<StepArgs<float>*>(&a), const_cast<FastNet*>(&f), &steps};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace scb
