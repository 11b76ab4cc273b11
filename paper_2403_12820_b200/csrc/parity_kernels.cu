// PARITY-mode kernels: bit-exact with the reference templates at T = float and T = double.
//
// One fused kernel per reference operator chain:
//   KIND_STEP    forward_impulse -> add_plug_impulse -> advance_with_impulse  (run_steps<T>
//                one_step, eval.cpp:48-59; nn_step net.cpp:242-248)
//   KIND_FORWARD forward_impulse only                    (kernels.hpp:265-282)
//   KIND_PLUG    add_plug_impulse on a zero field        (sim.cpp:100-106)
//   KIND_ADVANCE advance_with_impulse with a given field (kernels.hpp:205-252)
//   KIND_PBS     total_impulse -> advance_with_impulse: step_semi_implicit (sim.cpp:150-155),
//                the ground-truth mass-spring step
//   KIND_TOTAL   total_impulse only (kernels.hpp:165-175)
//   KIND_FORCE   total_force: the same four accumulations, unscaled (sim.cpp:84-96)
// Every floating-point operation is a non-contractible IEEE RN primitive in the reference's
// order; this TU is additionally compiled with --fmad=false.
//
// Work decomposition: a CTA owns a TX x TY tile of one cloth (grid.z = cloth), stages the
// (TX+4) x (TY+4) halo tile of all six planes in shared memory (stencil radius 2: the skip
// channels E2/N2/W2/S2, grid.cpp:24-27) and each thread evaluates TY/8 nodes of one column.
#include "sc_device.cuh"
#include "sc_kernels.h"

namespace scb {

namespace {

constexpr int TX = 32;
constexpr int TY = 16;
constexpr int BX = 32;
constexpr int BY = 8;
constexpr int HX = TX + 4;
constexpr int HY = TY + 4;

template <typename T, int KIND>
__global__ void __launch_bounds__(BX* BY) parity_kernel(const StepArgs<T> a) {
  using R = RN<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sm = reinterpret_cast<T*>(smem_raw);  // [6][HY][HX]

  const int b = blockIdx.z;
  const int cx0 = blockIdx.x * TX;
  const int gy0 = a.u0 + blockIdx.y * TY;
  const int rows_local = static_cast<int>(a.plane_stride / a.pitch);
  const T* in = a.in + static_cast<int64_t>(b) * 6 * a.plane_stride;
  const int tid = threadIdx.y * BX + threadIdx.x;

  const bool need_state = true;
  if (need_state) {
    for (int e = tid; e < 6 * HY * HX; e += BX * BY) {
      const int p = e / (HY * HX);
      const int rem = e - p * HY * HX;
      const int ly = rem / HX;
      const int lx = rem - ly * HX;
      const int gx = cx0 - 2 + lx;
      const int lr = gy0 - 2 + ly - a.g0;
      T val = T(0);
      if (gx >= 0 && gx < a.nx && lr >= 0 && lr < rows_local)
        val = in[elem_index(p, lr, gx, a.pitch, a.plane_stride, a.zs)];
      sm[e] = val;
    }
    __syncthreads();
  }

  const ClothConst<T> cc = a.cloths[b];
  const int ix = cx0 + threadIdx.x;
  if (ix >= a.nx) return;
  const int64_t nodes = static_cast<int64_t>(a.nx) * a.ny;
  auto S = [&](int p, int ly, int lx) -> T { return sm[(p * HY + ly) * HX + lx]; };

#pragma unroll 1
  for (int ry = threadIdx.y; ry < TY; ry += BY) {
    const int iy = gy0 + ry;
    if (iy >= a.u1) break;
    const int ly = ry + 2, lx = threadIdx.x + 2;
    const int64_t gnode = static_cast<int64_t>(iy) * a.nx + ix;
    T x[3], v[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      x[d] = S(d, ly, lx);
      v[d] = S(3 + d, ly, lx);
    }
    T imp[3];
    if (KIND == KIND_STEP || KIND == KIND_FORWARD) {
      // forward_impulse<T> (kernels.hpp:268-281)
#pragma unroll
      for (int d = 0; d < 3; ++d) imp[d] = R::add(a.net.b[d], R::mul(v[d], a.net.wv));
#pragma unroll
      for (int c = 0; c < kChannels; ++c) {
        const int jx = ix + off_dx(c), jy = iy + off_dy(c);
        if (jx < 0 || jx >= a.nx || jy < 0 || jy >= a.ny) continue;
        const T g = a.net.gain[c];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const T phi = R::mul(R::sub(x[d], S(d, ly + off_dy(c), lx + off_dx(c))), g);
          const T xi = R::mul(R::sub(v[d], S(3 + d, ly + off_dy(c), lx + off_dx(c))), g);
          const T s = R::div(phi, R::sqrt(R::add(T(1), R::mul(R::mul(a.net.alpha, phi), phi))));
          const T t = R::add(R::add(R::mul(phi, a.net.wl[c]), R::mul(s, a.net.wn[c])),
                             R::mul(R::mul(xi, s), a.net.wd[c]));
          imp[d] = R::add(imp[d], t);
        }
      }
      if (a.health && !(R::finite(imp[0]) && R::finite(imp[1]) && R::finite(imp[2]))) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.k + 1) << 32) | static_cast<unsigned long long>(gnode);
        atomicMin(&a.health[b].impulse_key, key);
      }
    } else if (KIND == KIND_PBS || KIND == KIND_TOTAL || KIND == KIND_FORCE) {
      // total_impulse<T> (kernels.hpp:165-175): elastic, damping, pressure, external, * dt/m
      T f[3] = {T(0), T(0), T(0)};
      bool singular = false;
      T lens[kChannels];  // |x_i - x_j| per channel: the damping loop reuses the elastic loop's
#pragma unroll
      for (int c = 0; c < kChannels; ++c) {  // accumulate_elastic (kernels.hpp:86-108)
        const int jx = ix + off_dx(c), jy = iy + off_dy(c);
        lens[c] = T(0);
        if (jx < 0 || jx >= a.nx || jy < 0 || jy >= a.ny) continue;
        T dd[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) dd[d] = R::sub(x[d], S(d, ly + off_dy(c), lx + off_dx(c)));
        const T len =
            R::sqrt(R::add(R::add(R::mul(dd[0], dd[0]), R::mul(dd[1], dd[1])), R::mul(dd[2], dd[2])));
        lens[c] = len;
        if (len == T(0)) {
          singular = true;
          continue;
        }
        const T sc = R::div(R::mul(cc.stiffness, R::sub(len, cc.rest[c])), len);
#pragma unroll
        for (int d = 0; d < 3; ++d) f[d] = R::sub(f[d], R::mul(dd[d], sc));
      }
#pragma unroll
      for (int c = 0; c < kChannels; ++c) {  // accumulate_damping (kernels.hpp:112-136)
        const int jx = ix + off_dx(c), jy = iy + off_dy(c);
        if (jx < 0 || jx >= a.nx || jy < 0 || jy >= a.ny) continue;
        T dd[3], dv[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          dd[d] = R::sub(x[d], S(d, ly + off_dy(c), lx + off_dx(c)));
          dv[d] = R::sub(v[d], S(3 + d, ly + off_dy(c), lx + off_dx(c)));
        }
        const T len = lens[c];  // the same IEEE sqrt of the same operands (kernels.hpp:120-122)
        if (len == T(0)) continue;
        T dir[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) dir[d] = R::div(dd[d], len);
        const T sc = R::mul(cc.damping, R::add(R::add(R::mul(dv[0], dir[0]), R::mul(dv[1], dir[1])),
                                               R::mul(dv[2], dir[2])));
#pragma unroll
        for (int d = 0; d < 3; ++d) f[d] = R::sub(f[d], R::mul(dir[d], sc));
      }
      if (cc.pressure != T(0) && ix >= 1 && ix <= a.nx - 2 && iy >= 1 && iy <= a.ny - 2) {
        // accumulate_pressure (kernels.hpp:142-155): interior nodes only, added into f
        T e[3], n[3], w[3], s[3], c1[3], c2[3], c3[3], c4[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          e[d] = R::sub(x[d], S(d, ly, lx + 1));
          n[d] = R::sub(x[d], S(d, ly + 1, lx));
          w[d] = R::sub(x[d], S(d, ly, lx - 1));
          s[d] = R::sub(x[d], S(d, ly - 1, lx));
        }
        auto cross = [](const T* p, const T* q, T* o) {
          o[0] = R::sub(R::mul(p[1], q[2]), R::mul(p[2], q[1]));
          o[1] = R::sub(R::mul(p[2], q[0]), R::mul(p[0], q[2]));
          o[2] = R::sub(R::mul(p[0], q[1]), R::mul(p[1], q[0]));
        };
        cross(e, n, c1);
        cross(n, w, c2);
        cross(w, s, c3);
        cross(s, e, c4);
#pragma unroll
        for (int d = 0; d < 3; ++d)
          f[d] = R::add(f[d], R::mul(R::add(R::add(R::add(c1[d], c2[d]), c3[d]), c4[d]), cc.pressure));
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) {  // accumulate_external (kernels.hpp:159-162), then * dt/m
        f[d] = R::add(f[d], R::sub(R::mul(cc.grav[d], cc.mass), R::mul(v[d], cc.drag)));
        imp[d] = KIND == KIND_FORCE ? f[d] : R::mul(f[d], cc.scale);
      }
      if (singular && a.health) {
        const unsigned long long key =
            (static_cast<unsigned long long>(a.k + 1) << 32) | static_cast<unsigned long long>(gnode);
        atomicMin(&a.health[b].impulse_key, key);
      }
    } else if (KIND == KIND_PLUG) {
#pragma unroll
      for (int d = 0; d < 3; ++d) imp[d] = T(0);
    } else {  // KIND_ADVANCE
      const T* ip = a.impulse + (static_cast<int64_t>(b) * nodes + gnode) * 3;
#pragma unroll
      for (int d = 0; d < 3; ++d) imp[d] = ip[d];
    }

    if (KIND == KIND_STEP || KIND == KIND_PLUG) {
      if (cc.plug_pressure) {
        const bool interior = ix >= 1 && ix <= a.nx - 2 && iy >= 1 && iy <= a.ny - 2;
        T e[3], n[3], w[3], s[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          e[d] = R::sub(x[d], S(d, ly, lx + 1));
          n[d] = R::sub(x[d], S(d, ly + 1, lx));
          w[d] = R::sub(x[d], S(d, ly, lx - 1));
          s[d] = R::sub(x[d], S(d, ly - 1, lx));
        }
        pressure_plug(cc, interior, e, n, w, s, imp);
      }
      plug_tail(cc, v, imp);
    }

    if (KIND == KIND_FORWARD || KIND == KIND_PLUG || KIND == KIND_TOTAL || KIND == KIND_FORCE) {
      T* op = a.impulse + (static_cast<int64_t>(b) * nodes + gnode) * 3;
#pragma unroll
      for (int d = 0; d < 3; ++d) op[d] = imp[d];
      continue;
    }

    T xo[3], vo[3];
    uint8_t mask;
    advance_node(a, cc, iy, gnode, x, v, imp, xo, vo, mask);
    T* out = a.out + static_cast<int64_t>(b) * 6 * a.plane_stride;
    const int64_t lr = iy - a.g0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      out[elem_index(d, lr, ix, a.pitch, a.plane_stride, a.zs)] = xo[d];
      out[elem_index(3 + d, lr, ix, a.pitch, a.plane_stride, a.zs)] = vo[d];
    }
    if (a.constrained) a.constrained[static_cast<int64_t>(b) * nodes + gnode] = mask;
    if (a.health && !(R::finite(xo[0]) && R::finite(xo[1]) && R::finite(xo[2]) &&
                      R::finite(vo[0]) && R::finite(vo[1]) && R::finite(vo[2])))
      atomicMin(&a.health[b].state_frame, a.k + 1);
  }
}

template <typename T, int KIND>
cudaError_t launch_parity_t(const StepArgs<T>& a, cudaStream_t stream) {
  const int rows = a.u1 - a.u0;
  if (rows <= 0 || a.batch <= 0) return cudaSuccess;
  const dim3 grid((a.nx + TX - 1) / TX, (rows + TY - 1) / TY, a.batch);
  const dim3 block(BX, BY);
  const size_t smem = sizeof(T) * 6 * HY * HX;
  parity_kernel<T, KIND><<<grid, block, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace

template <typename T>
cudaError_t launch_parity(const StepArgs<T>& a, int kind, cudaStream_t stream) {
  switch (kind) {
    case KIND_STEP:
      return launch_parity_t<T, KIND_STEP>(a, stream);
    case KIND_FORWARD:
      return launch_parity_t<T, KIND_FORWARD>(a, stream);
    case KIND_PLUG:
      return launch_parity_t<T, KIND_PLUG>(a, stream);
    case KIND_ADVANCE:
      return launch_parity_t<T, KIND_ADVANCE>(a, stream);
    case KIND_PBS:
      return launch_parity_t<T, KIND_PBS>(a, stream);
    case KIND_TOTAL:
      return launch_parity_t<T, KIND_TOTAL>(a, stream);
    case KIND_FORCE:
      return launch_parity_t<T, KIND_FORCE>(a, stream);
  }
  return cudaErrorInvalidValue;
}

template cudaError_t launch_parity<float>(const StepArgs<float>&, int, cudaStream_t);
template cudaError_t launch_parity<double>(const StepArgs<double>&, int, cudaStream_t);

}  // namespace scb
