/*
 * stencilcloth_b200.h — C-ABI drop-in boundary for the network-cell rollout step of the
 * arXiv 2403.12820 reference (`stencilcloth`), implemented as sm_100a CUDA kernels.
 *
 * The reference path this replaces (all paths relative to /root/reference/proj):
 *   detail::forward_impulse<T>       include/cloth/detail/kernels.hpp:265-282
 *   detail::add_plug_impulse<T>      include/cloth/detail/kernels.hpp:179-196
 *   detail::advance_with_impulse<T>  include/cloth/detail/kernels.hpp:205-252
 * driven by run_steps<T> (src/eval.cpp:35-67) and rollout (src/eval.cpp:86-103), and exposed
 * publicly as forward_impulse / nn_step (include/cloth/net.hpp:111-130), plug_impulse /
 * advance_with_impulse (include/cloth/sim.hpp:35,52-54), rollout / benchmark_net
 * (include/cloth/eval.hpp:14,47-48) and the pybind surface (python/bindings.cpp:147-164).
 *
 * Conventions
 *  - Plain C types only: pointers + sizes, no torch / C++ types cross this boundary.
 *  - Host state arrays are AoS [batch][node][3] in the context precision (float for SC_F32,
 *    double for SC_F64), node index iy*nx+ix (include/cloth/grid.hpp:35), i.e. exactly the
 *    memory layout of the reference's std::vector<VecT<T>>.
 *  - Scene and parameter descriptors are double, like the reference's Scene / NetworkParams;
 *    they are cast once to the compute precision, as make_scene_kernel<T> / make_net_kernel<T>
 *    do (kernels.hpp:58-81, net_kernel.hpp:8-22).
 *  - Every entry point returns an sc_status; on failure sc_last_error() holds a message that
 *    names the offending field, mirroring ConfigError / NumericsError (include/cloth/error.hpp).
 *  - Calls are synchronous at return unless documented otherwise. One context per host
 *    thread; a context owns its device buffers, which persist across calls.
 */
#ifndef STENCILCLOTH_B200_H
#define STENCILCLOTH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SC_ABI_VERSION 2
#define SC_CHANNELS 12 /* kChannels, include/cloth/grid.hpp:13 */

typedef enum {
  SC_OK = 0,
  SC_ERR_CONFIG = 1,   /* cloth::ConfigError   (error.hpp:17-21) -> Python ValueError      */
  SC_ERR_NUMERICS = 2, /* cloth::NumericsError (error.hpp:29-33) -> Python ArithmeticError */
  SC_ERR_CUDA = 3,     /* device / driver failure (no CPU fallback exists)                  */
  SC_ERR_STATE = 4     /* call order violated (e.g. stepping before a scene is bound)       */
} sc_status;

typedef enum { SC_F32 = 0, SC_F64 = 1 } sc_precision;

typedef enum {
  /* Bit-exact with the reference templates at the context precision: IEEE sqrt and divide,
   * no FMA contraction, the reference's per-channel accumulation order (kernels.hpp:268-281). */
  SC_MODE_PARITY = 0,
  /* f32 only: FMA, rsqrt ISRU, one ISRU per undirected stencil edge (channel-pair sharing).
   * Per-step outputs within 1e-5 relative of PARITY; collision/pin masks identical. */
  SC_MODE_FAST = 1
} sc_mode;

/* NetworkParams (include/cloth/net.hpp:35-54), 53 scalars in for_each_scalar order
 * (net.hpp:72-81). isru_alpha must be > 0 (src/net.cpp:23-26). */
typedef struct {
  double kernel_gain[SC_CHANNELS];
  double linear_w[SC_CHANNELS];
  double linear_b[3];
  double nonlinear_w[SC_CHANNELS];
  double deriv_w[SC_CHANNELS];
  double self_velocity_w;
  double isru_alpha;
} sc_params;

/* SphereCollider (include/cloth/scene.hpp:31-35). */
typedef struct {
  double center[3];
  double radius;   /* > 0 */
  double friction; /* in [0, 1]; tangential velocity scale is (1 - friction) */
} sc_sphere;

/* Extension, no reference counterpart: the plane z = height with normal +z, resolved with the
 * sphere chain's ordering (kernels.hpp:213-243) after all spheres. Parity for it is unpinned. */
typedef struct {
  double height;
  double friction; /* in [0, 1] */
} sc_plane;

/* One cloth's scene constants: the per-cloth part of cloth::Scene (scene.hpp:43-60) as seen by
 * SceneKernel<T> (kernels.hpp:41-56). Wind folds into `gravity` (a constant acceleration, applied
 * exactly like gravity by add_plug_impulse, kernels.hpp:188-191). Arrays are borrowed for the
 * duration of the call that receives them. */
typedef struct {
  double dt;         /* > 0 */
  double mass;       /* > 0 */
  double drag;       /* >= 0 */
  double pressure;   /* signed */
  double gravity[3]; /* acceleration (gravity + wind) */
  int32_t plug_pressure, plug_gravity, plug_drag; /* PlugForce flags (scene.hpp:38) */
  int32_t n_pins;
  const int32_t* pin_nodes;   /* [n_pins], strictly increasing node indices (scene.cpp:43-52) */
  const double* pin_anchors;  /* [n_pins][3], anchor positions at t = 0 */
  double pin_velocity[3];     /* BoundarySpec::pin_velocity() (scene.hpp:27) */
  int32_t n_spheres;
  const sc_sphere* spheres;
  int32_t n_planes;
  const sc_plane* planes;
  /* Material of the ground-truth mass-spring step (PBS); unused by the
   * network step: spring stiffness and damping (MaterialParams, grid.hpp:65-76) and the grid
   * spacing that sets the rest lengths (spacing * {1, sqrt2, 2}, grid.cpp:14-30,93-95). */
  double stiffness; /* >= 0 */
  double damping;   /* >= 0 */
  double spacing;   /* > 0 when stepping PBS */
} sc_cloth_desc;

/* A batch of cloths sharing one nx-by-ny grid topology (build_grid, src/grid.cpp:83-138). */
typedef struct {
  int32_t nx, ny; /* >= 2 each */
  int32_t batch;  /* >= 1 */
  const sc_cloth_desc* cloths; /* [batch] */
} sc_scene_desc;

typedef struct sc_ctx sc_ctx;

/* ---- lifecycle ------------------------------------------------------------------------ */
int sc_abi_version(void);
const char* sc_last_error(void); /* thread-local; valid until the next failing call */
/* device: CUDA ordinal. Fails with SC_ERR_CUDA when no device / kernel image is usable. */
sc_status sc_ctx_create(int device, sc_precision precision, sc_ctx** out);
void sc_ctx_destroy(sc_ctx* ctx);

/* Validates like Scene::validate (src/scene.cpp:23-61) and uploads the per-cloth constants
 * (the SceneKernel<T> cast happens here, once, as in run_steps<T> eval.cpp:37). Allocates the
 * ctx-owned device state for batch*nx*ny nodes. */
sc_status sc_ctx_set_scene(sc_ctx* ctx, const sc_scene_desc* scene);
/* make_net_kernel<T> (net_kernel.hpp:8-22); rejects isru_alpha <= 0 (net.cpp:23-26). */
sc_status sc_ctx_set_params(sc_ctx* ctx, const sc_params* params);

/* Host AoS state <-> ctx device state. */
sc_status sc_ctx_set_state(sc_ctx* ctx, const void* x, const void* v);
sc_status sc_ctx_get_state(sc_ctx* ctx, void* x, void* v);

/* Device-resident stepping: `steps` applications of the fused step (forward_impulse ->
 * add_plug_impulse -> advance_with_impulse, the run_steps<T> sequence eval.cpp:48-59) to the ctx
 * state, producing frames k0+1 .. k0+steps with t_next = T(k+1) * T(dt). Asynchronous on the
 * ctx stream; sc_ctx_sync() waits. */
sc_status sc_ctx_advance(sc_ctx* ctx, int32_t steps, int32_t k0, sc_mode mode);
sc_status sc_ctx_sync(sc_ctx* ctx);
/* After advance: per-cloth first frame whose impulse / state held a non-finite value (-1 if
 * none) and the flat node index of the first such impulse (for the NumericsError text of
 * net.cpp:30-51 and eval.cpp:98-99). Any of the outputs may be NULL. */
sc_status sc_ctx_get_health(sc_ctx* ctx, int32_t* first_bad_impulse_frame,
                            int32_t* first_bad_impulse_node, int32_t* first_bad_state_frame);
/* Non-finite tracking during device-resident stepping (sc_ctx_advance / sc_rollout*): on by
 * default for SC_F64 contexts (rollout's checks, eval.cpp:98-99, net.cpp:139-140), off for
 * SC_F32 (run_steps<float> checks nothing, eval.cpp:48-59). Per-operator calls always track. */
sc_status sc_ctx_set_health_checks(sc_ctx* ctx, int32_t on);
/* FAST mode runs multi-step advances of narrow-cloth batches (nx <= 128, no pressure plug) as
 * one persistent wavefront launch: W timesteps per pass over HBM, rows updated in place in
 * shared memory (wave_kernels.cu), bit-identical to one launch per step; cloths of at most 1024
 * nodes as one small-cloth launch (one thread per node, the state in shared memory,
 * small_kernels.cu; within the FAST tolerance; SC_SMALL=0 turns that one off). Off: one
 * streaming launch per step (programmatic dependent launch chains them). Default on; the
 * environment variable SC_WAVE=0 turns it off for contexts that never called this.
 * Mask-producing last steps and contexts outside the kernels' domains always take the streaming
 * kernel. */
sc_status sc_ctx_set_persistent(sc_ctx* ctx, int32_t on);

/* Host-to-host rollout: upload x0/v0, advance `steps`, download the final state. When
 * `constrained` is non-NULL it receives the mask of the LAST step ([batch][node] uint8, the
 * advance_with_impulse output of kernels.hpp:211-250). FAST mode with >= 8 whole cloths, no mask
 * and page-locked x0 / v0 / x_out / v_out (sc_host_alloc) overlaps the transfers with the stepping
 * (cloth chunks on concurrent streams; results identical to the plain path). */
sc_status sc_rollout(sc_ctx* ctx, const void* x0, const void* v0, int32_t steps, int32_t k0,
                     sc_mode mode, void* x_out, void* v_out, uint8_t* constrained);

/* rollout() with frame storage (eval.cpp:86-103): frames_x / frames_v receive
 * (steps / stride + 1) frames, frame 0 being the input state. */
sc_status sc_rollout_frames(sc_ctx* ctx, const void* x0, const void* v0, int32_t steps,
                            int32_t stride, sc_mode mode, void* frames_x, void* frames_v);

/* ---- single-operator entry points (the reference's public per-op API) -------------------- */
/* forward_impulse (net.hpp:111-112 / kernels.hpp:265-282): impulse [batch][node][3]. */
sc_status sc_forward_impulse(sc_ctx* ctx, const void* x, const void* v, void* impulse);
/* plug_impulse (sim.hpp:35 / kernels.hpp:179-196) on a zero field. */
sc_status sc_plug_impulse(sc_ctx* ctx, const void* x, const void* v, void* impulse);
/* advance_with_impulse (sim.hpp:52-54 / kernels.hpp:205-252) with a caller impulse. t_next in
 * the context precision's arithmetic (cast from double). */
sc_status sc_advance_with_impulse(sc_ctx* ctx, const void* x, const void* v, const void* impulse,
                                  double t_next, void* x_out, void* v_out, uint8_t* constrained);
/* nn_step (net.hpp:129-130 / net.cpp:242-248) fused, with the optional constrained mask. */
sc_status sc_nn_step(sc_ctx* ctx, const void* x, const void* v, double t_next, sc_mode mode,
                     void* x_out, void* v_out, uint8_t* constrained);

/* ---- ground-truth mass-spring step (PBS; §8(f2)), PARITY only ---------------------------- */
/* total_impulse (sim.hpp:32 / kernels.hpp:165-175): elastic + damping + pressure + external
 * forces scaled by dt/m, [batch][node][3]. A coincident connected pair is SC_ERR_NUMERICS
 * naming the first node ("elastic force: singular spring ...", kernels.hpp:105-107). */
sc_status sc_total_impulse(sc_ctx* ctx, const void* x, const void* v, void* impulse);
/* step_semi_implicit (sim.hpp:58 / sim.cpp:150-155) from host state to host state. */
/* total_force (sim.cpp:84-96; binding total_force, bindings.cpp:156-161): the four force terms
 * accumulated in the reference order, unscaled, [batch][node][3]. Same errors as
 * sc_total_impulse. */
sc_status sc_total_force(sc_ctx* ctx, const void* x, const void* v, void* force);
sc_status sc_pbs_step(sc_ctx* ctx, const void* x, const void* v, double t_next, void* x_out,
                      void* v_out, uint8_t* constrained);
/* simulate_scene's stepping (sim.cpp:157-175) with frame storage like sc_rollout_frames; after
 * it, sc_ctx_get_health reports the first frame whose state went non-finite (state frame) and
 * the first singular spring (impulse frame / node). */
sc_status sc_simulate_frames(sc_ctx* ctx, const void* x0, const void* v0, int32_t steps,
                             int32_t stride, void* frames_x, void* frames_v);
/* ---- evaluate_rollout (§8(f4), eval.cpp:105-133) ---------------------------------------- */
/* Per-frame sums over nodes of |x_test - x_ref| (double AoS [frames][nodes][3] host arrays);
 * the caller forms 100 * sum / (nodes * bbox diagonal of reference frame 0) like the reference.
 * Context-free (its own stream on `device`); errors via sc_eval_last_error(). */
sc_status sc_evaluate_frames(int device, const double* test_x, const double* ref_x,
                             int32_t frames, int64_t nodes, double* frame_sums);
const char* sc_eval_last_error(void);

/* ---- training forward + backward (§8(f1), train.hpp / train.cpp, net.cpp:144-201) --------- */
/* A trainer holds one scene (batch 1, f64) and its ground-truth trajectory resident on the GPU
 * ([frames][node][3] f64 host arrays, copied once). Results are bit-identical to the reference's
 * sample_batch / compute_loss / backward_gradients / train_loop (see csrc/train.cu). */
typedef struct sc_trainer sc_trainer;

/* TrainConfig (train.hpp:16-53); schedule_kind 0 = Step, 1 = Cosine; freeze_mask bit g freezes
 * ParamGroup g (kernel=0, linear, bias, nonlinear, deriv, self_velocity, alpha=6). */
typedef struct sc_train_config {
  double alpha;
  int32_t batch_size, epochs;
  int32_t schedule_kind;
  double lr0, gamma;
  int32_t interval;
  double floor;
  int32_t period;
  uint64_t seed;
  int32_t de_population, de_generations;
  double de_bound, de_cross_prob, de_diff_weight;
  int32_t de_probe_batch;
  int32_t checkpoint_interval;
  uint32_t freeze_mask;
} sc_train_config;

/* AdamState (train.hpp:118-123) over the flat 53 scalars. */
typedef struct sc_adam_state {
  double m[53];
  double v[53];
  int64_t step;
} sc_adam_state;

sc_status sc_trainer_create(int device, const sc_scene_desc* scene, int32_t frames,
                            const double* frames_x, const double* frames_v, sc_trainer** out);
void sc_trainer_destroy(sc_trainer* trainer);
/* sample_batch (train.cpp:91-127) with a fresh Rng(rng_seed): batch indices (nullable) and the
 * force-integration targets f_k*dt [batch][node][3] (nullable); the batch becomes current. */
sc_status sc_trainer_sample_batch(sc_trainer* trainer, int32_t batch_size, uint64_t rng_seed,
                                  int32_t* indices_out, double* force_dt_out);
/* The index draw of sample_batch alone (host only, no device): batch_size distinct transitions
 * of a frames-long trajectory from Rng(rng_seed). */
sc_status sc_sample_indices(int32_t frames, int32_t batch_size, uint64_t rng_seed,
                            int32_t* indices_out);
/* Explicit transition indices as the current batch (targets computed on the device). */
sc_status sc_trainer_set_batch(sc_trainer* trainer, const int32_t* indices, int32_t count);
/* compute_loss (train.cpp:129-209) on the current batch: loss_out = {total, physics, data};
 * grads_out (53, for_each_gradient order, nullable) = the ParamGradients. */
sc_status sc_trainer_compute_loss(sc_trainer* trainer, const sc_params* params, double alpha,
                                  double* loss_out, double* grads_out);
/* train_loop (train.cpp:343-375): DE pre-search + Adam epochs, or fine-tune from resume_params
 * (+ trainable flags, + the Adam state in opt_inout). history_out: epochs x {step, lr, physics,
 * data, total} (nullable); opt_inout (nullable) receives the final Adam state; brackets_out
 * (nullable, 14 doubles): the InitBracket {lo, hi} of each ParamGroup (net.hpp:28-31). */
sc_status sc_trainer_run(sc_trainer* trainer, const sc_train_config* cfg,
                         const sc_params* resume_params, const uint8_t* resume_trainable,
                         sc_adam_state* opt_inout, sc_params* params_out, uint8_t* trainable_out,
                         double* history_out, double* brackets_out);
/* Data-parallel compute_loss in parts (one rank's contiguous share [b0, b1) of the current
 * batch), exact when combined in transition order (see training.DistributedTrainer):
 *   part_forward : cell impulses, residuals and per-node loss terms of the part; the part's data
 *                  count; bad_out = {first transition with a non-finite impulse, its node} or -1
 *   part_chain   : the loss sums continued from sums_in = {phys_sq, data_sq} over the part;
 *                  bad_out = first transition after which a sum is non-finite, or -1
 *   part_backward: with the batch-wide data count and batch size, the per-transition gradient
 *                  totals per_b[(b - b0) * 53 + s] (sum them in transition order)
 *   diagnose_forward: the reference's "network impulse non-finite ..." text for (frame, node). */
sc_status sc_trainer_part_forward(sc_trainer* trainer, const sc_params* params, int32_t b0,
                                  int32_t b1, uint64_t* count_out, int32_t* bad_out);
sc_status sc_trainer_part_chain(sc_trainer* trainer, const double* sums_in, double* sums_out,
                                int32_t* bad_out);
sc_status sc_trainer_part_backward(sc_trainer* trainer, const sc_params* params, double alpha,
                                   uint64_t global_count, int32_t global_batch, double* per_b);
sc_status sc_trainer_diagnose_forward(sc_trainer* trainer, const sc_params* params, int32_t frame,
                                      int32_t node, char* msg, int32_t len);
/* backward_gradients (net.cpp:144-201) for one state and upstream cotangent [node][3]. */
sc_status sc_backward_gradients(int device, int32_t nx, int32_t ny, const double* x,
                                const double* v, const sc_params* params, const double* upstream,
                                double* grads_out);

/* benchmark_sim (eval.hpp:46 / eval.cpp:151-153): device-timed PBS steps from the ctx state. */
sc_status sc_benchmark_sim(sc_ctx* ctx, int32_t steps, int32_t warmup, double* seconds);

/* benchmark_net (eval.hpp:47-48 / eval.cpp:69-82,155-158): warmup untimed steps then `steps`
 * timed steps from the ctx state, timed with CUDA events on the ctx stream. */
sc_status sc_benchmark(sc_ctx* ctx, int32_t steps, int32_t warmup, sc_mode mode,
                       double* seconds);
/* Per-launch device time of `steps` consecutive fused steps (events between launches on the
 * ctx stream), for roofline accounting: launch_ms[steps]. */
sc_status sc_benchmark_launches(sc_ctx* ctx, int32_t steps, int32_t k0, sc_mode mode,
                                float* launch_ms);

/* ---- row-strip domain decomposition (one rank's strip of a tall cloth) ------------------ */
/* Restricts the ctx to global rows [row0, row0 + rows) of an ny-row cloth plus up to two ghost
 * rows on each side that exist in the cloth. Call before sc_ctx_set_scene; nx/ny in the scene
 * descriptor stay the GLOBAL sizes and pin / node indices stay global. batch must be 1. */
sc_status sc_ctx_set_strip(sc_ctx* ctx, int32_t row0, int32_t rows);
/* Halo exchange support for a collective layer (NCCL send/recv or peer copies over NVLink):
 * pack the two owned rows adjacent to `side` (0 = the strip's low rows row0, row0+1;
 * 1 = its high rows) of the BACK buffer (the one sc_ctx_strip_step just wrote) into a contiguous
 * device buffer [6][2][nx] of the ctx precision, and unpack a neighbour's rows into the ghost
 * rows on `side` of the back buffer. Rows that fall outside the cloth are skipped. */
int64_t sc_ctx_halo_elems(sc_ctx* ctx);
sc_status sc_ctx_halo_pack(sc_ctx* ctx, int32_t side, void* dev_dst, void* cuda_stream);
sc_status sc_ctx_halo_unpack(sc_ctx* ctx, int32_t side, const void* dev_src, void* cuda_stream);
/* One step of the strip, restricted to owned local rows [r_begin, r_end) (so boundary rows can
 * be computed first and shipped while the interior runs). The state swap happens in
 * sc_ctx_strip_commit after all row ranges of the step were issued. */
sc_status sc_ctx_strip_step(sc_ctx* ctx, int32_t k, int32_t r_begin, int32_t r_end,
                            sc_mode mode, void* cuda_stream);
sc_status sc_ctx_strip_commit(sc_ctx* ctx);

/* Stream of the context (cudaStream_t) for callers that overlap their own work. */
void* sc_ctx_stream(sc_ctx* ctx);
/* Device buffers of the ctx state (front = current, back = next) for zero-copy views. */
sc_status sc_ctx_state_buffers(sc_ctx* ctx, void** front, void** back, int64_t* plane_stride,
                               int32_t* pitch, int32_t* local_rows, int32_t* row_base);

/* ---- fused halo exchange over peer memory (§8(e), config 4 strips) ------------------------ */
/* A strip context exports its two state buffers and its completion flags (CUDA IPC handles and
 * raw pointers); a neighbour links them with sc_ctx_set_peer (side 0: the strip below, 1: above;
 * use_ipc = 0 for contexts in the same process). sc_ctx_peer_step then runs one FAST step of
 * the whole owned strip in which the two boundary rows at each linked side are also stored
 * straight into the neighbour's ghost rows (NVLink peer stores), bracketed by a wait on the
 * neighbours' completion flags and a system-scope release of ours: no NCCL call, no pack. */
typedef struct sc_peer_export {
  unsigned char state_handle[2][64]; /* cudaIpcMemHandle_t of state buffers 0 and 1 */
  unsigned char flags_handle[64];
  void* state_ptr[2]; /* raw device pointers (same-process linking) */
  void* flags_ptr;
  int64_t plane_stride;
  int32_t g0, u0, u1, nx, pitch, batch, cur, device;
} sc_peer_export;
sc_status sc_ctx_peer_export(sc_ctx* ctx, sc_peer_export* out);
sc_status sc_ctx_set_peer(sc_ctx* ctx, int32_t side, const sc_peer_export* neighbour,
                          int32_t use_ipc);
sc_status sc_ctx_peer_step(sc_ctx* ctx, int32_t k, sc_mode mode, void* stream);

/* Page-locked host buffers, so host<->device copies of rollout() run at full PCIe/C2C rate. */
sc_status sc_host_alloc(size_t bytes, void** out);
void sc_host_free(void* p);
/* Number of kernel launches this ctx issued so far (device-resident stepping included). */
int64_t sc_ctx_launch_count(sc_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* STENCILCLOTH_B200_H */
