// Launch interface between the C-ABI layer (capi.cu) and the kernel translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>

#include "sc_device.cuh"

namespace scb {

enum {
  KIND_STEP = 0,
  KIND_FORWARD = 1,
  KIND_PLUG = 2,
  KIND_ADVANCE = 3,
  KIND_PBS = 4,
  KIND_TOTAL = 5,
  KIND_FORCE = 6
};

// parity_kernels.cu (compiled with --fmad=false)
template <typename T>
cudaError_t launch_parity(const StepArgs<T>& a, int kind, cudaStream_t stream);

// fast_kernels.cu: f32 FAST step (FMA, rsqrt ISRU, one ISRU per undirected edge).
// Gains folded into the weights: wL' = g wL, wN' = g wN, wD' = g^2 wD, alpha' = alpha g^2.
struct FastNet {
  float wl[kChannels], wn[kChannels], wd[kChannels];
  float nwl[kChannels], nwn[kChannels];  // negated, for the far endpoint of an edge
  float alpha[kChannels];
  float b[3];
  float wv;
  int alpha1;  // every alpha' == 1 (default gains and alpha): skips one multiply per edge
  // channels with a nonzero weight (bit c). A channel whose three weights are all zero
  // contributes dx * 0 to the cell: the small-cloth kernel skips it (config 1's
  // "hidden 8, 3x3" cell is the reference cell with the four skip channels zeroed; a non-finite
  // neighbour then no longer spreads through such a channel, which only PARITY mode reproduces)
  unsigned live;
};
struct FastPlan {
  int n_strips, seg_rows, n_segs;
  int chunk_segs;  // row segments per strip column under chunked stepping
  int64_t units;  // one single-warp CTA per (cloth, 128-column strip, row segment)
  size_t smem;
  int ring;       // staged rows (5 when a cloth plugs pressure, else 4)
  bool general;   // some cloth takes the collider / pressure / mask finish
  bool wide;      // simple finish on the wide-register kernel (160 registers, tall segments)
  bool chunk_wide;  // the same under chunked stepping (capi.cu chunked_fast_steps)
  int occupancy;  // resident CTAs per SM
  // every collider cloth: one frictionless plane (1) / one sphere (2), no pressure plug — the
  // launches without mask output take the kernel with that collider finish alone; 0: dispatch
  int only;
};
FastNet make_fast_net(const NetConst<float>& net);
// Channel-pair sharing needs gain[c] == gain[negated(c)] (grid.cpp:32-35).
bool fast_supported(const NetConst<float>& net, int nx);
// max_sms > 0: plan the segmentation for that many SMs (the rest run a concurrent launch)
FastPlan plan_fast(int nx, int rows, int batch, int device, bool pressure, bool general,
                   int max_sms = 0);
// tmap[0]: xy pairs of a.in as 8-byte elements, dims (pitch, rows, 2, batch), box (136,1,2,1);
// tmap[1]: z planes, dims (pitch, rows, 2, batch) from element 4S, box (136,1,2,1).
cudaError_t launch_fast(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tmap,
                        const FastPlan& plan, cudaStream_t stream);
// debug: record [unit][start, end] globaltimer ns of every fast_step_kernel unit (nullptr: off)
cudaError_t set_unit_timing(unsigned long long* dev_buf);

// wave_kernels.cu: wavefront temporal blocking of the FAST step for batches of narrow cloths
// (nx <= 128): `levels` timesteps per pass over HBM, one persistent CTA per SM, state updated in
// place (a.in == a.out), bit-identical to `levels` fast_step_kernel launches.
struct WavePlan {
  bool ok;        // the kernel applies to this grid / batch
  int levels;     // W: timesteps per pass (= warps per CTA)
  int slots;      // shared-memory ring slots (rows)
  int ctas;       // persistent CTAs (one per SM, at most one per cloth)
  size_t smem;
  bool general;   // some cloth takes the collider finish
  int fin;        // finish set compiled in: 0 none, 1 any collider, 2 frictionless planes only
  int rev;        // level order reversed across warp slots (issue priority to deep levels)
  uint32_t hint_ns;  // mbarrier try_wait suspend-time hint (0: the hardware default)
};
// max_ctas > 0: use at most that many SMs (the rest stay free for a concurrent launch)
// plane_only: every collider cloth has one frictionless plane and no sphere (the lean finish)
WavePlan plan_wave(int nx, int ny, int batch, int device, bool general, int max_ctas = 0,
                   bool plane_only = false);
size_t wave_smem_bytes(int levels, int slots);
// `steps` timesteps k = a.k .. a.k + steps - 1 of the launch's cloths (a.batch of them from
// a.b_off, through a.ids when set), from a.in (tensor maps tmap) into a.out (tmap_out); a.in ==
// a.out updates in place.
cudaError_t launch_wave(const StepArgs<float>& a, const FastNet& f, const CUtensorMap* tmap,
                        const CUtensorMap* tmap_out, const WavePlan& plan, int steps,
                        cudaStream_t stream);

// small_kernels.cu: cloths of at most 1024 nodes (config 1): one CTA per cloth, one thread per
// node, the state double-buffered in shared memory, all `steps` timesteps of a.k .. in one launch
// from a.in into a.out. Per-node cell evaluation in the reference's channel order (FAST
// arithmetic; within the FAST tolerance, not bit-identical to the row-pass kernels).
bool small_supported(int nx, int ny);
cudaError_t launch_small(const StepArgs<float>& a, const FastNet& f, bool general, int steps,
                         cudaStream_t stream);

// layout.cu: AoS [batch][node][3] <-> planar [batch][6][rows][pitch]
// (rows = the ctx's local rows; AoS arrays hold exactly those rows.)
template <typename T>
cudaError_t launch_aos_to_planar(const T* x_aos, const T* v_aos, T* planar, int batch, int nx,
                                 int rows, int64_t plane_stride, int pitch, bool zs,
                                 cudaStream_t stream);
template <typename T>
cudaError_t launch_planar_to_aos(const T* planar, T* x_aos, T* v_aos, int batch, int nx, int rows,
                                 int64_t plane_stride, int pitch, bool zs, cudaStream_t stream);
// one band of rows [row0, row0 + rows) of a single f32 cloth; x, v point at the band's first node
cudaError_t launch_aos_to_planar_rows(const float* x, const float* v, float* planar, int nx,
                                      int row0, int rows, int64_t plane_stride, int pitch, bool zs,
                                      cudaStream_t stream);
cudaError_t launch_planar_to_aos_rows(const float* planar, float* x, float* v, int nx, int row0,
                                      int rows, int64_t plane_stride, int pitch, bool zs,
                                      cudaStream_t stream);

}  // namespace scb
