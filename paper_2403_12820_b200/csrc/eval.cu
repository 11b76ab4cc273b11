// evaluate_rollout's per-frame position error sums (reference eval.cpp:105-133):
//   sum_f = sum over nodes of |x_test - x_ref|, |d| = sqrt((dx*dx + dy*dy) + dz*dz)
// Each node's norm is the reference's IEEE double expression exactly (RN intrinsics, no FMA);
// only the order of the node sum differs (a fixed two-level tree, deterministic run to run).
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/stencilcloth_b200.h"

namespace {

constexpr int kThreads = 256;

__global__ void frame_partials(const double* __restrict__ a, const double* __restrict__ b,
                               int64_t nodes, int blocks_per_frame, int f0,
                               double* __restrict__ partial) {
  __shared__ double sm[kThreads];
  const int64_t f = static_cast<int64_t>(f0) + blockIdx.y;
  const int64_t per_block = (nodes + blocks_per_frame - 1) / blocks_per_frame;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * per_block;
  const int64_t i1 = i0 + per_block < nodes ? i0 + per_block : nodes;
  const double* A = a + f * nodes * 3;
  const double* B = b + f * nodes * 3;
  double acc = 0.0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kThreads) {
    const double dx = __dsub_rn(A[3 * i], B[3 * i]);
    const double dy = __dsub_rn(A[3 * i + 1], B[3 * i + 1]);
    const double dz = __dsub_rn(A[3 * i + 2], B[3 * i + 2]);
    acc = __dadd_rn(acc, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                              __dmul_rn(dz, dz))));
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] = __dadd_rn(sm[threadIdx.x], sm[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[f * blocks_per_frame + blockIdx.x] = sm[0];
}

__global__ void frame_totals(const double* __restrict__ partial, int frames, int blocks_per_frame,
                             double* __restrict__ sums) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= frames) return;
  double s = 0.0;
  for (int k = 0; k < blocks_per_frame; ++k)
    s = __dadd_rn(s, partial[static_cast<int64_t>(f) * blocks_per_frame + k]);
  sums[f] = s;
}

thread_local std::string g_eval_err;

}  // namespace

extern "C" {

const char* sc_eval_last_error(void) { return g_eval_err.c_str(); }

sc_status sc_evaluate_frames(int device, const double* test_x, const double* ref_x,
                             int32_t frames, int64_t nodes, double* frame_sums) {
  auto fail = [](const char* what, cudaError_t e) {
    g_eval_err = std::string(what) + ": " + cudaGetErrorString(e);
    return SC_ERR_CUDA;
  };
  if (frames < 1 || nodes < 1 || !test_x || !ref_x || !frame_sums) {
    g_eval_err = "evaluate: empty or null input";
    return SC_ERR_CONFIG;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail("cudaSetDevice", e);
  const size_t bytes = static_cast<size_t>(frames) * nodes * 3 * sizeof(double);
  const int bpf = static_cast<int>(nodes / (kThreads * 64) + 1 > 512 ? 512 : nodes / (kThreads * 64) + 1);
  double *da = nullptr, *db = nullptr, *dp = nullptr, *ds = nullptr;
  sc_status st = SC_OK;
  cudaStream_t s = nullptr;
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return fail("stream", e);
  if ((e = cudaMallocAsync(&da, bytes, s)) != cudaSuccess ||
      (e = cudaMallocAsync(&db, bytes, s)) != cudaSuccess ||
      (e = cudaMallocAsync(&dp, sizeof(double) * frames * bpf, s)) != cudaSuccess ||
      (e = cudaMallocAsync(&ds, sizeof(double) * frames, s)) != cudaSuccess) {
    st = fail("cudaMalloc", e);
  } else {
    if ((e = cudaMemcpyAsync(da, test_x, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(db, ref_x, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) {
      st = fail("H2D frames", e);
    } else {
      // gridDim.y is capped at 65535: frames go in chunks
      for (int f0 = 0; f0 < frames && st == SC_OK; f0 += 65535) {
        const int nf = frames - f0 < 65535 ? frames - f0 : 65535;
        frame_partials<<<dim3(bpf, nf), kThreads, 0, s>>>(da, db, nodes, bpf, f0, dp);
        if ((e = cudaGetLastError()) != cudaSuccess) st = fail("frame_partials launch", e);
      }
      if (st == SC_OK) {
        frame_totals<<<(frames + 127) / 128, 128, 0, s>>>(dp, frames, bpf, ds);
        if ((e = cudaGetLastError()) != cudaSuccess) st = fail("frame_totals launch", e);
      }
      if (st == SC_OK &&
          (e = cudaMemcpyAsync(frame_sums, ds, sizeof(double) * frames, cudaMemcpyDeviceToHost,
                               s)) != cudaSuccess)
        st = fail("D2H sums", e);
    }
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess && st == SC_OK) st = fail("evaluate", e);
  }
  cudaFreeAsync(da, s);
  cudaFreeAsync(db, s);
  cudaFreeAsync(dp, s);
  cudaFreeAsync(ds, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return st;
}

}  // extern "C"
