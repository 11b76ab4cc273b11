// Layout conversion at the C-ABI edge: the reference's AoS VecT<T>[node] (vec3.hpp:9-59)
// <-> the xy-interleaved SoA device layout of the step kernels (sc_device.cuh). Only the API edges
// run these; device-resident stepping never converts.
#include "sc_kernels.h"

namespace scb {
namespace {

template <typename T>
__global__ void aos_to_planar(const T* __restrict__ x, const T* __restrict__ v, T* __restrict__ out,
                              int batch, int nx, int rows, int64_t plane_stride, int pitch,
                              bool zs, int row0) {
  const int64_t per = static_cast<int64_t>(rows) * nx;
  const int64_t total = per * batch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per;
    const int64_t node = i - b * per;
    const int64_t r = node / nx + row0;
    const int64_t c = node - (r - row0) * nx;
    T* o = out + b * 6 * plane_stride;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      o[elem_index(d, r, c, pitch, plane_stride, zs)] = x[3 * i + d];
      o[elem_index(3 + d, r, c, pitch, plane_stride, zs)] = v[3 * i + d];
    }
  }
}

template <typename T>
__global__ void planar_to_aos(const T* __restrict__ in, T* __restrict__ x, T* __restrict__ v,
                              int batch, int nx, int rows, int64_t plane_stride, int pitch,
                              bool zs, int row0) {
  const int64_t per = static_cast<int64_t>(rows) * nx;
  const int64_t total = per * batch;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / per;
    const int64_t node = i - b * per;
    const int64_t r = node / nx + row0;
    const int64_t c = node - (r - row0) * nx;
    const T* s = in + b * 6 * plane_stride;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      if (x) x[3 * i + d] = s[elem_index(d, r, c, pitch, plane_stride, zs)];
      if (v) v[3 * i + d] = s[elem_index(3 + d, r, c, pitch, plane_stride, zs)];
    }
  }
}

int grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 64) g = 148 * 64;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

template <typename T>
cudaError_t launch_aos_to_planar(const T* x, const T* v, T* planar, int batch, int nx, int rows,
                                 int64_t plane_stride, int pitch, bool zs, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(batch) * rows * nx;
  aos_to_planar<T><<<grid_for(total), 256, 0, stream>>>(x, v, planar, batch, nx, rows,
                                                       plane_stride, pitch, zs, 0);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_planar_to_aos(const T* planar, T* x, T* v, int batch, int nx, int rows,
                                 int64_t plane_stride, int pitch, bool zs, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(batch) * rows * nx;
  planar_to_aos<T><<<grid_for(total), 256, 0, stream>>>(planar, x, v, batch, nx, rows,
                                                       plane_stride, pitch, zs, 0);
  return cudaGetLastError();
}

// One band of rows [row0, row0 + rows) of a single cloth: x, v point at the band's first AoS
// node (the pipelined single-cloth rollout, capi.cu rollout_band_pipelined).
cudaError_t launch_aos_to_planar_rows(const float* x, const float* v, float* planar, int nx,
                                      int row0, int rows, int64_t plane_stride, int pitch, bool zs,
                                      cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(rows) * nx;
  aos_to_planar<float><<<grid_for(total), 256, 0, stream>>>(x, v, planar, 1, nx, rows,
                                                           plane_stride, pitch, zs, row0);
  return cudaGetLastError();
}

cudaError_t launch_planar_to_aos_rows(const float* planar, float* x, float* v, int nx, int row0,
                                      int rows, int64_t plane_stride, int pitch, bool zs,
                                      cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(rows) * nx;
  planar_to_aos<float><<<grid_for(total), 256, 0, stream>>>(planar, x, v, 1, nx, rows,
                                                           plane_stride, pitch, zs, row0);
  return cudaGetLastError();
}

template cudaError_t launch_aos_to_planar<float>(const float*, const float*, float*, int, int, int,
                                                 int64_t, int, bool, cudaStream_t);
template cudaError_t launch_aos_to_planar<double>(const double*, const double*, double*, int, int,
                                                  int, int64_t, int, bool, cudaStream_t);
template cudaError_t launch_planar_to_aos<float>(const float*, float*, float*, int, int, int,
                                                 int64_t, int, bool, cudaStream_t);
template cudaError_t launch_planar_to_aos<double>(const double*, double*, double*, int, int, int,
                                                  int64_t, int, bool, cudaStream_t);

}  // namespace scb
