// Pipe-mix probe on the B200: can scalar FFMA issue alongside packed FFMA2 (separate FMA pipes)?
// Reports fma lane-ops per SM per ns for pure and interleaved streams.
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int NF, int NP>  // NF scalar FFMA chains, NP packed FFMA2 chains per iteration
__global__ void k(float* out, int iters, float s) {
  float a[NF > 0 ? NF : 1];
  unsigned long long p[NP > 0 ? NP : 1];
#pragma unroll
  for (int i = 0; i < NF; ++i) a[i] = threadIdx.x * 0.001f + i;
#pragma unroll
  for (int i = 0; i < NP; ++i)
    p[i] = ((unsigned long long)__float_as_uint(0.5f + i) << 32) | __float_as_uint(0.25f * i);
  const unsigned long long ss = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (NF > NP ? NF : NP); ++i) {
      if (i < NF) a[i] = fmaf(a[i], s, 0.5f * s);
      if (i < NP) p[i] = ffma2(p[i], ss, ss);
    }
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < NF; ++i) r += a[i];
#pragma unroll
  for (int i = 0; i < NP; ++i) r += __uint_as_float((unsigned)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// warps alternate: even warps run scalar FFMA, odd warps packed FFMA2 (mixing across warps only)
__global__ void kx(float* out, int iters, float s) {
  const bool packed = (threadIdx.x >> 5) & 1;
  float a[16];
  unsigned long long p[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    p[i] = ((unsigned long long)__float_as_uint(0.5f + i) << 32) | __float_as_uint(0.25f * i);
  const unsigned long long ss = ((unsigned long long)__float_as_uint(s) << 32) | __float_as_uint(s);
  if (packed) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], ss, ss);
  } else {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], s, 0.5f * s);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) r += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) r += __uint_as_float((unsigned)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int NF, int NP>
void run(const char* name, int sms, float* o) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<NF, NP><<<sms * 8, 256>>>(o, iters, 0.999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double lane_ops = (double)sms * 8 * 256 * iters * (NF + 2 * NP);
    const double instr = (double)sms * 8 * 8 * iters * (NF + NP);  // warp-instructions
    if (rep == 1)
      printf("%-28s %.1f fma lane-ops per SM per ns, %.2f warp-instr per SM per ns\n", name,
             lane_ops / (ms * 1e-3) / sms / 1e9, instr / (ms * 1e-3) / sms / 1e9);
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, sizeof(float) * sms * 8 * 256);
  run<16, 0>("FFMA x16", sms, o);
  run<0, 8>("FFMA2 x8", sms, o);
  run<8, 4>("FFMA x8 + FFMA2 x4", sms, o);
  run<8, 8>("FFMA x8 + FFMA2 x8", sms, o);
  run<16, 8>("FFMA x16 + FFMA2 x8", sms, o);
  {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      kx<<<sms * 8, 256>>>(o, iters, 0.999f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double lane_ops = (double)sms * 8 * 256 * iters * 16;
      if (rep == 1)
        printf("%-28s %.1f fma lane-ops per SM per ns\n", "warps alternate FFMA / FFMA2",
               lane_ops / (ms * 1e-3) / sms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
