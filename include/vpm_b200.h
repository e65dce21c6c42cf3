/*
 * vpm_b200.h -- C ABI of the B200-native VPM-MPPI stepping library
 * (paper_2509_16079_b200/lib/libvpm_b200.so, sources in paper_2509_16079_b200/csrc/).
 *
 * Plain pointers and sizes only; no torch types.  Two layers:
 *
 *  1. Reference-facing host-buffer entry points.  They are exactly what the
 *     reference's stepping-module FFI binds (perchsim/_accel/_core.pyx, which
 *     Python reaches through perchsim/_accel/__init__.py:47-48 backend_module()):
 *        vpm_step           replaces _core.pyx:536-576   step(...)
 *        vpm_rollout        replaces _core.pyx:609-661   rollout(...)
 *        vpm_batch_rollout  replaces _core.pyx:664-714   batch_rollout(...)
 *        vpm_threads        replaces _core.pyx:744-745   omp_threads()
 *     Arguments keep the reference meaning and layout (FP64, C-order, the
 *     flattened FluidState 11-tuple of rollout.py:59-62, the frozen
 *     iparams/fparams ABI of config.py:280-300).  Host buffers in, host buffers
 *     out; the library does the host<->device copies.
 *
 *  2. Device-resident planner entry points used by the MPPI engine
 *     (mppi.py:62-84 optimize, policy.py:66-91 perturbed rollouts): device
 *     pointers plus a cudaStream_t passed as void*.
 *
 * Error convention (mirrors the reference): numerical failures are status codes
 * (0 ok, 1+t failed at step t) in the outputs; configuration errors return a
 * negative code from the call and set a message readable by vpm_last_error().
 */
#ifndef VPM_B200_H
#define VPM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VPM_OK 0
#define VPM_ERR_CONFIG (-1) /* limits / argument errors (reference: ValueError) */
#define VPM_ERR_CUDA (-2)   /* CUDA runtime failure */
#define VPM_ERR_ALLFAIL (-3) /* every MPPI candidate failed (mppi.py:55-56) */
#define VPM_ERR_RANK (-4)    /* < 6 perturbed rollouts survived (policy.py:88-90) */
#define VPM_ERR_DIVERGED (-5) /* Riccati recursion non-finite (policy.py:231-232) */

/* Flattened FluidState (rollout.py:59-62 order), FP64 reference layout.
 * wake_pos is (n_wake, 2) C-order; buffers may be longer than n_wake. */
typedef struct vpm_fluid {
  const double *wake_pos;
  const double *wake_gamma;
  const int64_t *wake_age;
  int32_t n_wake, ring_a, ring_b;
  const double *prev_pos; /* (nb, 2) */
  const double *prev_gamma;
  int32_t n_prev;
  double prev_lev;
  const double *ema; /* (nb,) */
} vpm_fluid;

/* Output fluid buffers sized as the reference's _dump_fluid (_core.pyx:579-606):
 * wake_pos (cap+4, 2), wake_gamma/wake_age (cap+4), prev_pos (nb, 2),
 * prev_gamma/ema (nb).  scalars = {n_wake, ring_a, ring_b, n_prev}. */
typedef struct vpm_fluid_out {
  double *wake_pos;
  double *wake_gamma;
  int64_t *wake_age;
  int32_t *scalars;
  double *prev_pos;
  double *prev_gamma;
  double *prev_lev;
  double *ema;
} vpm_fluid_out;

/* ---- layer 1: reference-facing, host buffers -------------------------------- */

/* One coupled step (integrate=1: Engine.step, 0: Engine.fluid_step).  x is
 * in/out (7).  Returns the step rc (0 ok, 2 non-finite) or a negative error.  fw
 * (2) and mw (1) receive the wing loads.  _core.pyx:536-576.
 * The reference's rc 1 (zero LU pivot in the boundary solve, _core.pyx:315-317)
 * cannot occur here: the three boundary systems are pose-invariant (they couple
 * points on the chord line only), so they are factorised once when the parameters
 * are unpacked and a singular one is reported as VPM_ERR_CONFIG ("boundary system is
 * singular for this configuration") before any step runs -- the configuration for
 * which the reference would return rc 1 at its first shedding or attached step. */
int vpm_step(double *x, double u, const vpm_fluid *fluid, const int64_t *iparams,
             const double *fparams, int integrate, double *fw, double *mw, vpm_fluid_out *out);

/* Open-loop rollout of T controls; x in/out (7 = final state).  traj (T+1, 7)
 * may be NULL; out may be NULL (no fluid returned).  Returns status (0 or 1+t)
 * or a negative error.  _core.pyx:609-661 */
int64_t vpm_rollout(double *x, const double *controls, int T, const vpm_fluid *fluid,
                    const int64_t *iparams, const double *fparams, double *traj,
                    vpm_fluid_out *out);

/* B independent rollouts from a shared x0 (7) and fluid fork; controls (B, T).
 * status (B) int64, finals (B, 7), trajs (B, T+1, 7) or NULL.  workers is
 * accepted for signature parity and ignored (one CTA per rollout).
 * _core.pyx:664-714 */
int vpm_batch_rollout(const double *x0, const double *controls, int B, int T,
                      const vpm_fluid *fluid, const int64_t *iparams, const double *fparams,
                      int record, int workers, int64_t *status, double *finals, double *trajs);

/* batch_rollout with one start state per row (x0 is (B, 7)): the perturbed
 * cloud of policy.perturbed_rollouts (policy.py:66-91) in one launch. */
int vpm_batch_rollout_x0(const double *x0, const double *controls, int B, int T,
                         const vpm_fluid *fluid, const int64_t *iparams, const double *fparams,
                         int record, int64_t *status, double *finals, double *trajs);

/* omp_threads() analogue: concurrent rollouts resident on the device. */
int vpm_threads(void);

/* Message of the last negative return on this thread. */
const char *vpm_last_error(void);

/* ---- layer 2: device-resident planner ------------------------------------- */

typedef struct vpm_plan vpm_plan;

/* Create a plan bound to the frozen parameter ABI and a CUDA device: uploads the
 * inverse boundary-system matrices, sizes scratch for up to max_rows rollouts of
 * horizon H.  Returns NULL on error (see vpm_last_error). */
vpm_plan *vpm_plan_create(const int64_t *iparams, const double *fparams, int max_rows, int H,
                          int device);
void vpm_plan_destroy(vpm_plan *p);

/* Upload the fluid snapshot (host) that every rollout forks from. */
int vpm_plan_set_fluid(vpm_plan *p, const vpm_fluid *fluid);

/* The two halves of vpm_plan_set_fluid: pack the snapshot into the plan's pinned
 * mirror (after the device is idle), and queue the mirror's copy to the device on
 * a stream -- so a captured CUDA graph can contain the upload (replan.py). */
int vpm_plan_stage_fluid(vpm_plan *p, const vpm_fluid *fluid);
int vpm_plan_upload_fluid(vpm_plan *p, void *stream);

/* Per-rollout outputs of a device batch; any pointer may be NULL. */
typedef struct vpm_batch_out {
  int64_t *status;      /* (rows) */
  double *finals;       /* (rows, 7) */
  double *trajs;        /* (rows, T+1, 7) */
  double *cost;         /* (rows) terminal cost, +inf when failed (mppi.py:28-34) */
  uint64_t *shed_mask;  /* (rows) bit t set when step t shed */
  int32_t *n_final;     /* (rows) final wake size */
  int64_t *interactions;/* (rows) regularised Biot-Savart interactions evaluated */
  uint64_t *shed_mask_hi; /* (rows) bit t-64 set when step t (64 <= t < 128) shed */
  uint64_t *wake_hash;  /* (rows) wake-index signature: per-step (wake size, ring-core
                           indices, shed flag) chain + final (index, age) sum; parity
                           diagnostic of the shed / merge / ordered-removal bookkeeping
                           (_core.pyx:157-172, 322-373) */
} vpm_batch_out;

/* Device batch of rows [row_begin, row_end) of a B_total-row candidate set.
 * Controls: if d_controls != NULL, row r uses d_controls[(r - row_begin)*T ...];
 * else MPPI sampling: row 0 is d_ustar, row r>=1 is
 * clip(d_ustar + sigma * d_noise[(r-1)*T ...], +-u_limit) (mppi.py:37-43, :79).
 * d_x0 is (7) when x0_stride == 0 or (rows, 7) when x0_stride == 7.
 * d_q / d_xperch (7 each) enable the cost output.  Launches on stream. */
int vpm_plan_batch(vpm_plan *p, const double *d_x0, int x0_stride, const double *d_controls,
                   const double *d_ustar, const double *d_noise, double sigma, int row_begin,
                   int row_end, int T, const double *d_q, const double *d_xperch, int record,
                   const vpm_batch_out *d_out, void *stream);

/* Closed-loop projection (project_forward, nmpc.py:88-103): one rollout of T
 * Engine.step calls from d_x0 under the feedback policy
 * u = clip(-K_k (x - tau_k) + xi_k), k = rint((t - t_start)/dt) clamped to
 * [0, pol_h) (evaluate_policy, policy.py:236-244), t accumulated from t0.  With
 * write_snapshot the resulting fluid replaces the plan's snapshot on the device
 * (the MPPI / nominal / policy launches of a replan then fork from it with no host
 * round trip).  d_status: 0 or 1 + failing step; d_final (7). */
int vpm_plan_project(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                     const double *d_states, const double *d_inputs, int pol_h, double t_start,
                     double t0, int64_t *d_status, double *d_final, int write_snapshot,
                     void *stream);

/* vpm_plan_project with {t_start, t0} read from device memory d_times (2) at run
 * time -- for CUDA-graph replay, where by-value arguments are frozen at capture. */
int vpm_plan_project_dev(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                         const double *d_states, const double *d_inputs, int pol_h, const double *d_times,
                         int64_t *d_status, double *d_final, int write_snapshot, void *stream);

/* Device-resident single step: Engine.step (integrate=1) / Engine.fluid_step
 * (integrate=0) of rollout.py:81-98 (_core.pyx:536-576) on the plan's snapshot IN
 * PLACE -- the stepped fluid becomes the snapshot, no host round trip of the wake.
 * x (7, host) and u are passed by value; with sensor (host xz) the FP64 induced
 * velocity there (vpm.py:93-128, regularised, r_core) is evaluated on the stepped
 * wake (the NMPC pressure sensor, nmpc.py:73-85).  Queues the launch(es); the step
 * record lands in h_record (host, VPM_STEP_RECORD_BYTES) -- written by the kernels
 * directly when h_record is page-locked (pinned), else through one queued copy:
 *   double x[7] (new state), fw[3] {fw_x, fw_z, m_w}, q[2] (sensor velocity);
 *   int32 rc (0 ok, 2 non-finite), n_wake, ring_a, ring_b, n_prev.
 * Returns without synchronising (vpm_stream_sync).  The plant / observed-wake loop
 * of nmpc.py:314-315 keeps its two fluids on the device between ticks this way. */
#define VPM_STEP_RECORD_BYTES 128
int vpm_plan_step(vpm_plan *p, const double *x, double u, int integrate, const double *sensor,
                  double r_core, void *h_record, void *stream);

/* Induced velocity (FP64, regularised with r_core) at one host point from the
 * plan's current device wake, synchronous.  out (2). */
int vpm_plan_probe(vpm_plan *p, const double *target, double r_core, double *out);

/* cudaStreamSynchronize on a stream passed as void*. */
int vpm_stream_sync(void *stream);

/* Perturbed cloud (perturbed_rollouts, policy.py:66-91) in one launch: row r starts
 * at x0 + x0_noise[r] * x0_scale and applies clip(u* + u_noise[r] * sigma_u);
 * trajectories (rows, T+1, 7) recorded. */
int vpm_plan_cloud(vpm_plan *p, const double *d_x0, const double *d_x0_noise,
                   const double *d_x0_scale, const double *d_ustar, const double *d_u_noise,
                   double sigma_u, int rows, int T, int64_t *d_status, double *d_trajs,
                   void *stream);

/* Copy the plan's (device) snapshot to host buffers (reference _dump_fluid layout). */
int vpm_plan_download_fluid(vpm_plan *p, vpm_fluid_out *out);

/* MPPI weighted partial sums over rows [0, rows) of this shard
 * (mppi.py:46-59 split for sharding): d_partial (H+2) =
 * {J_min_r, Z_r = sum exp(-(J-J_min_r)/lambda), S_r[H] = sum w u}.  Row r uses
 * the same control formula as vpm_plan_batch with global index row_begin + r. */
int vpm_mppi_partial(vpm_plan *p, const double *d_cost, int rows, int row_begin,
                     const double *d_ustar, const double *d_noise, double sigma, int T,
                     double temperature, double *d_partial, void *stream);

/* Combine W gathered partials (W, H+2) in rank order into d_ustar (H).  Sets
 * *d_flag = 1 when every candidate failed (d_ustar untouched; the caller raises).
 * The flag is sticky: the kernel never clears it, callers zero it once per
 * optimisation, so a failed iteration is never masked by a later success. */
int vpm_mppi_combine(const double *d_partials, int W, int T, double temperature,
                     double *d_ustar, int32_t *d_flag, void *stream);

/* Performance mode (no reference counterpart): standard-normal
 * noise drawn on the device for rows [row_begin, row_begin + rows) of one
 * iteration's (K, T) noise matrix -- counter-based Philox4x32-10 keyed by seed,
 * subsequence = global noise row, offset fixed by iteration, so any sharding of the
 * rows draws the same numbers.  d_out: (rows, T) FP64.  The reference-parity path
 * keeps host-drawn numpy noise (mppi.py:42). */
int vpm_noise_philox(uint64_t seed, uint64_t iteration, int row_begin, int rows, int T,
                     double *d_out, void *stream);

/* vpm_noise_philox with {seed, iteration} read from device memory d_seed_iter (2)
 * at run time, iteration + offset used (CUDA-graph replay of a replan cycle). */
int vpm_noise_philox_dev(const uint64_t *d_seed_iter, uint64_t offset, int row_begin, int rows, int T,
                         double *d_out, void *stream);

/* Whole MPPI iteration on one device (batch + partial + combine): two kernel
 * launches on stream -- the rollouts, then the softmax partial whose finishing CTA
 * also applies the W = 1 combine (bitwise vpm_mppi_partial + vpm_mppi_combine; the
 * same sticky *d_flag).  use_graph is reserved and ignored (callers that want graph
 * replay capture the stream themselves, as replan.py does).
 * d_noise: (B_total - 1, T).  d_cost scratch (B_total) and d_partial (T+2), which
 * holds the partial record afterwards. */
int vpm_mppi_iteration(vpm_plan *p, const double *d_x0, double *d_ustar, const double *d_noise,
                       double sigma, int B_total, int T, double temperature, const double *d_q,
                       const double *d_xperch, double *d_cost, double *d_partial,
                       int32_t *d_flag, int use_graph, void *stream);

/* Host-buffer MPPI optimise (mppi.py:62-84) for iters iterations with
 * pre-generated noise (iters, K, T): host u_star in/out (T).  Includes every
 * host<->device copy.  Returns VPM_ERR_ALLFAIL when a whole batch failed. */
int vpm_mppi_optimize_host(vpm_plan *p, const double *x0, double *u_star, const double *noise,
                           int iters, int K, int T, double sigma, double temperature,
                           const double *q, const double *x_perch);

/* ---- sample-built tracking controller (policy.py:66-266) ---------------------- */

/* Device: per-step least-squares Jacobians of the acceleration rows over the
 * surviving perturbed rollouts (estimate_linear_sequence, policy.py:141-171) when
 * do_fit, then the backward Riccati gains (tvlqr_backward, policy.py:206-233) when
 * do_riccati.  Shapes: nom_x (H+1,7), nom_u (H), cloud_x (K,H+1,7), cloud_u (K,H),
 * status (K); a_cont (H,3,5), b_cont (H,3), a_disc (H,7,7), b_disc (H,7) (inputs
 * when !do_fit), gains (H,7); *d_flag = 1 + step where the recursion diverged. */
int vpm_policy_fit(const double *d_nom_x, const double *d_nom_u, const double *d_cloud_x,
                   const double *d_cloud_u, const int64_t *d_status, int K, int H, double dt,
                   const double *d_q_running, double r_running, const double *d_q_final,
                   double *d_a_cont, double *d_b_cont, double *d_a_disc, double *d_b_disc,
                   double *d_gains, int32_t *d_flag, int do_fit, int do_riccati, void *stream);

/* Host buffers: build_policy (policy.py:247-266) -- K perturbed rollouts from
 * x0s (K,7) with controls u_cloud (K,H) on plan p's fluid in one launch, then fit
 * and Riccati.  Returns VPM_ERR_RANK (< 6 survivors) / VPM_ERR_DIVERGED like the
 * reference's RankDeficientData / FloatingPointError.  Any output may be NULL. */
int vpm_build_policy_host(vpm_plan *p, const double *nom_x, const double *nom_u, int H,
                          const double *x0s, const double *u_cloud, int K, double dt,
                          const double *q_running, double r_running, const double *q_final,
                          double *a_cont, double *b_cont, double *a_disc, double *b_disc,
                          double *gains, int64_t *status_out, double *cloud_x_out);

/* Host buffers: estimate_linear_sequence alone (policy.py:141-171). */
int vpm_policy_fit_host(const double *nom_x, const double *nom_u, int H, const double *cloud_x,
                        const double *cloud_u, const int64_t *status, int K, double dt,
                        double *a_cont, double *b_cont, double *a_disc, double *b_disc);

/* Host buffers: tvlqr_backward alone (policy.py:206-233). */
int vpm_tvlqr_host(const double *a_disc, const double *b_disc, int H, const double *q_running,
                   double r_running, const double *q_final, double *gains);

/* Average duration (ms) of the rollout kernel over the launches recorded since
 * the last reset, timed with CUDA events on the launch stream. */
int vpm_plan_timing(vpm_plan *p, int reset, double *avg_ms, int64_t *launches);

/* Pipe throughput microbenchmark on the current device: mode 0 FFMA (GFLOP/s),
 * 1 packed FFMA2 (GFLOP/s), 2 MUFU.RSQ (G ops/s), 3 the direct Biot-Savart
 * instruction mix (8 FP32 lane-ops + 1 MUFU.RSQ per interaction) in algorithmic
 * GFLOP/s at 12 flop per interaction -- the formulation's pipe ceiling. */
double vpm_fp32_peak_probe(int iters, int mode);

/* Host-only: the inverses of the three pose-invariant boundary systems the solve
 * uses (attached nb x nb, shedding forward, shedding reversed; (nb+2)^2 doubles
 * each, row-major, the attached block with row stride nb).  out: 3 (nb+2)^2. */
int vpm_boundary_inverse(const int64_t *iparams, const double *fparams, double *out);

/* Launch configuration chosen for a particle cap and a batch of rows on the
 * current device: threads per rollout CTA, targets per thread, dynamic shared
 * memory bytes. */
int vpm_launch_shape(int cap, int nb, int rows, int *threads, int *targets, int *smem_bytes);

/* Host buffers: velocity induced by n point vortices (pos (n,2), gamma (n)) at m
 * target points (targets (m,2)) -> out (m,2), FP64 on the device.  kernel 0 is the
 * regularised kernel with core radius r_core, 1 the singular kernel (a coincident
 * source contributes 0).  Replaces vpm.induced_velocity_at (vpm.py:105-128), the
 * NMPC pressure sensor's flow model (nmpc.py:71-85). */
int vpm_induced_velocity_host(const double *pos, const double *gamma, int n, const double *targets,
                              int m, double r_core, int kernel, double *out);

#ifdef __cplusplus
}
#endif
#endif /* VPM_B200_H */
