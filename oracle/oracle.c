/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the network-cell rollout step.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2403.12820 reference, `stencilcloth`):
 *   detail::forward_impulse<T>      /root/reference/proj/include/cloth/detail/kernels.hpp:265-282
 *   detail::isru<T>                 kernels.hpp:30-33
 *   detail::add_plug_impulse<T>     kernels.hpp:179-196 (+ accumulate_pressure :142-155)
 *   detail::advance_with_impulse<T> kernels.hpp:205-252 (+ contact_band :23-28)
 *   make_net_kernel<T>              include/cloth/detail/net_kernel.hpp:8-22
 *   run_steps<T> step sequence      src/eval.cpp:48-65
 *   stencil channel order           src/grid.cpp:14-30
 * instantiated at float and double. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline/reference legs may load it — as the checker, never as the thing measured or
 * shipped. Its bit-exactness against the reference's own templates is pinned by
 * tests/test_oracle_golden.py against fixtures produced by oracle/_ref (the reference sources
 * compiled by oracle/Makefile) and by the reference's own known-answer tests restated in
 * tests/test_oracle_kats.py.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/stencilcloth_b200.h"

/* canonical channel order E,N,W,S,NE,NW,SW,SE,E2,N2,W2,S2 (grid.cpp:14-30) */
static const int ORC_OFF[12][2] = {{1, 0},  {0, 1},   {-1, 0}, {0, -1}, {1, 1},  {-1, 1},
                                   {-1, -1}, {1, -1}, {2, 0},  {0, 2},  {-2, 0}, {0, -2}};

/* VecT::cross (include/cloth/vec3.hpp:47-49) */
#define ORC_CROSS(o, a, b)                 \
  do {                                     \
    (o)[0] = (a)[1] * (b)[2] - (a)[2] * (b)[1]; \
    (o)[1] = (a)[2] * (b)[0] - (a)[0] * (b)[2]; \
    (o)[2] = (a)[0] * (b)[1] - (a)[1] * (b)[0]; \
  } while (0)

#define T float
#define SFX f32
#define SQRT sqrtf
#define EPS FLT_EPSILON
#include "oracle_body.inc"
#undef T
#undef SFX
#undef SQRT
#undef EPS

#define T double
#define SFX f64
#define SQRT sqrt
#define EPS DBL_EPSILON
#include "oracle_body.inc"
#undef T
#undef SFX
#undef SQRT
#undef EPS

int orc_abi_version(void) { return SC_ABI_VERSION; }

/* struct sizes as compiled from include/stencilcloth_b200.h, so tests can check the Python
 * ctypes mirror of the boundary types byte for byte */
size_t orc_sizeof(int which) {
  switch (which) {
    case 0: return sizeof(sc_params);
    case 1: return sizeof(sc_sphere);
    case 2: return sizeof(sc_plane);
    case 3: return sizeof(sc_cloth_desc);
    case 4: return sizeof(sc_scene_desc);
  }
  return 0;
}
