// Dependent-add latency probe: one thread, N dependent DADD (and FADD for comparison).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dchain(double* out, double a, int n) {
  double s = 0.0, t = 1e-300;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) { s = __dadd_rn(s, a); a = __dadd_rn(a, t); }
  long long c1 = clock64();
  out[0] = s; out[1] = (double)(c1 - c0) / n;
}
__global__ void dchain1(double* out, double a, int n) {
  double s = 0.0;
  long long c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, a);
  long long c1 = clock64();
  out[0] = s; out[1] = (double)(c1 - c0) / n;
}
__global__ void fchain1(double* out, float a, int n) {
  float s = 0.0f;
  long long c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) s = __fadd_rn(s, a);
  long long c1 = clock64();
  out[0] = s; out[1] = (double)(c1 - c0) / n;
}
int main() {
  double* d; cudaMalloc(&d, 16); double h[2];
  dchain1<<<1,1>>>(d, 1.0000001, 1 << 20); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DADD dependent: %.2f cycles/add\n", h[1]);
  fchain1<<<1,1>>>(d, 1.0001f, 1 << 20); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("FADD dependent: %.2f cycles/add\n", h[1]);
  dchain<<<1,1>>>(d, 1.0000001, 1 << 20); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("2 interleaved DADD chains: %.2f cycles/iter\n", h[1]);
  return 0;
}
