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

#include "node_cell.cuh"

namespace scb {

namespace {

constexpr int kSmallMaxNodes = 1024;

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
    const int jx = ix + nodecell::kDx(c), jy = iy + nodecell::kDy(c);
    nbr[c] = jy * nx + jx;
    if (jx >= 0 && jx < nx && jy >= 0 && jy < ny) valid |= 1u << c;
  }
  valid &= f.live;  // zero-weight channels (config 1's skip channels) contribute dx * 0: skipped
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
      }
      nodecell::cell<ALPHA1>(f, x, v, valid,
                             [&](int c, int d) { return cur[d * n + nbr[c]]; }, acc);
      float xo[3], vo[3];
      uint8_t mk;
      nodecell::finish<GEN>(a, cc, simple, b, k, iy, gnode, t_next, x, v, acc, xo, vo, mk);
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
