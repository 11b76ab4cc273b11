// Standalone probe: one 3-D TMA box load (the fast kernel's row fetch) into shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, float* out, int c0, int c1, int c2) {
  extern __shared__ __align__(128) float ring[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    if (VARIANT == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else if (VARIANT != 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(132 * 6 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(ring)), "l"(VARIANT == 2 ? reinterpret_cast<uint64_t>(gmap) : reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 132 * 6; i += 32) out[i] = ring[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#include <cstdlib>
int main(int argc, char** argv) {
  const int pitch = 256, rows = 64, planes = 6 * 2;
  std::vector<float> h((size_t)pitch * rows * planes);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  float* o; cudaMalloc(&o, 132 * 6 * 4);
  void* fp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {pitch, rows, planes};
  cuuint64_t str[2] = {pitch * 4, (cuuint64_t)pitch * rows * 4};
  cuuint32_t box[3] = {132, 1, 6}, es[3] = {1, 1, 1};
  CUresult r = ((Enc)fp)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap)); cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
  int c0 = argc > 2 ? atoi(argv[2]) : -2;
  for (int variant = atoi(argv[1]); variant <= atoi(argv[1]); ++variant) {
    if (variant == 0) probe<0><<<1, 32, 4096>>>(m, gm, o, c0, 3, 6);
    if (variant == 1) probe<1><<<1, 32, 4096>>>(m, gm, o, c0, 3, 6);
    if (variant == 2) probe<2><<<1, 32, 4096>>>(m, gm, o, c0, 3, 6);
    if (variant == 3) probe<3><<<1, 32, 4096>>>(m, gm, o, c0, 3, 6);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", variant, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> ho(132 * 6);
    cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
    // expect plane 6+p row 3 cols -2..129 (first two zero)
    int bad = 0;
    for (int p = 0; p < 6; ++p) for (int c = 0; c < 132; ++c) {
      int gc = c + c0; float want = gc < 0 ? 0.f : h[((size_t)(6 + p) * rows + 3) * pitch + gc];
      if (ho[p * 132 + c] != want) ++bad;
    }
    printf("  mismatches %d\n", bad);
  }
  return 0;
}
