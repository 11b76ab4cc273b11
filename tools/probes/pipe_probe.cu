// Pipe-throughput probe on the B200: FFMA vs FFMA2 (packed f32x2) vs MUFU.RSQ, per SM per clock.
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int KIND>
__global__ void k(float* out, int iters, float s) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
  unsigned long long p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = ((unsigned long long)__float_as_uint(a[2 * i]) << 32) | __float_as_uint(a[2 * i + 1]);
  const unsigned long long ss = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
  for (int it = 0; it < iters; ++it) {
    if (KIND == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f * s);
    } else if (KIND == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], ss, ss);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = rsqrtf(a[i]);
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; cudaMalloc(&o, sizeof(float) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"FFMA (16 ops/iter)", "FFMA2 (8 instr = 16 fma/iter)", "MUFU.RSQ (16/iter)"};
  for (int kind = 0; kind < 3; ++kind) {
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k<0><<<sms * 8, 256>>>(o, iters, 0.999f);
      if (kind == 1) k<1><<<sms * 8, 256>>>(o, iters, 0.999f);
      if (kind == 2) k<2><<<sms * 8, 256>>>(o, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lanes_ops = (double)sms * 8 * 256 * iters * 16;
      if (rep == 1) printf("%-32s %.3e lane-ops/s = %.1f per SM per ns  (%.2f TFLOP-ish)\n", names[kind], lanes_ops / (ms * 1e-3),
                           lanes_ops / (ms * 1e-3) / sms / 1e9, lanes_ops * 2 / (ms * 1e-3) / 1e12);
    }
  }
  printf("sms %d, clock %d kHz\n", sms, clk);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
