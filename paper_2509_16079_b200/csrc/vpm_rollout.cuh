// vpm_rollout.cuh -- sm_100a kernels of the VPM-MPPI hot path.
//
// One CTA owns one rollout for all H steps.  The wake (<= cap+8 particles) lives
// in shared memory as float4 {x, z, Gamma/(2 pi), age}, double-buffered; the
// rigid-body state, the bound-vortex row, the unsteady-load filter and every
// discrete decision live in an FP64 control block in shared memory.  The O(N^2)
// regularised Biot-Savart sweeps run on the FP32 pipe (packed FFMA2/FADD2/FMUL2 +
// MUFU.RSQ); everything O(1) / O(nb) runs in FP64 on warp 0.
//
// Reference semantics (paths relative to /root/reference/pkg/src/perchsim/):
//   step_core         _accel/_core.pyx:175-462  (== vpm.py:635-669 + glider.py:104-122)
//   run_rollout       _accel/_core.pyx:465-491
//   batch_rollout     _accel/_core.pyx:664-741
//   terminal cost     mppi.py:28-34
//   MPPI update       mppi.py:46-59
//
// Per-step phase schedule inside the CTA (barriers B1..B4), iteration t:
//
//   P1  all warps, source-split: wake velocity at the panels of step t-1 (the
//       loads of step t-1, _core.pyx:385-389; the sources are the post-merge wake,
//       i.e. exactly the sources of the convection sweep of step t); the live wake
//       is copied, compacted, into buffer 1.
//   B1
//   P2  the control warp (warp 0; the last warp with the symmetric sweep) runs D
//       after its share of S1/A: unsteady-Bernoulli loads of step t-1
//       (_core.pyx:375-418), elevator + Euler integration (_core.pyx:423-461),
//       envelope check (_core.pyx:483-484), then the chord frame / collocation
//       geometry, gates and control of step t (_core.pyx:228-256).
//       All warps: S1 = velocity at every live wake particle from every wake
//       particle + the previous bound row (convection, _core.pyx:192-221) over the
//       compacted copy of the wake made before B1 (buffer 1) -- register-tiled
//       direct sums, or for caps above 256 the symmetric-pair tile schedule
//       (sym_sweep, with one barrier per tile round); then A = Euler advection,
//       dissipation, ageing (_core.pyx:222-226) written compacted into buffer 0
//       (this retires the ordered removals of step t-1); Kelvin block sums;
//       per-warp merge candidates.
//   B2
//   S2  all warps, source-split: wake velocity at the nb collocation rows
//       (_core.pyx:273-296).
//   B3
//   E   warp 0: right-hand side, bound-circulation solve with the precomputed
//       inverse of the pose-invariant system, shed LEV/TEV
//       (_core.pyx:322-334), merge of the oldest particles (_core.pyx:336-357)
//       as a top-(m+1) selection, ring termination (_core.pyx:359-373).  Removed
//       particles become zero-circulation holes until the next A compacts them.
//   B4
//
// The loads of step t are computed lazily at the top of iteration t+1 because
// they need exactly the sources of the next convection sweep.
//
// Determinism: every floating-point reduction has a canonical order that does not
// depend on the CTA shape, the batch size or the row range -- per-target sums run
// over sources in index order (packed and scalar paths are bitwise identical),
// cross-thread sums are taken over fixed 32-source blocks with a fixed butterfly
// and then accumulated block by block.  A rollout therefore produces the same
// bits whatever launch it is part of (the reference's "batch == sequential",
// _core.pyx:671-676), and every rank count of the sharded planner agrees bitwise.
#pragma once

#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <math.h>
#include <stdint.h>

namespace vpm {

constexpr int NB_MAX = 64;     // reference MAXNB (_core.pyx:23)
constexpr int NT_MAX = 512;    // threads per rollout CTA
constexpr int NW_MAX = NT_MAX / 32;
constexpr int MC = 8;          // merge candidates kept per warp
#ifndef VPM_NSEG
#define VPM_NSEG 12
#endif
constexpr int NSEG = VPM_NSEG;  // source segments of the split sweeps (fixed: canonical order)
constexpr int HOLES_MAX = 16;
constexpr int WAKE_PAD = 8;    // wake slots beyond cap (reference buffers hold cap+4)
#ifndef VPM_SWEEP_UNROLL
#define VPM_SWEEP_UNROLL 8
#endif
#ifndef VPM_SLOT_REV
#define VPM_SLOT_REV 1
#endif
#ifndef VPM_D_PASS
#define VPM_D_PASS 1
#endif
constexpr int SWEEP_UNROLL = VPM_SWEEP_UNROLL;  // sources per sweep-loop trip
constexpr int D_PASS = VPM_D_PASS;  // warp 0 runs its control phase after (1) / before (0) its sweep
constexpr bool SLOT_REV = VPM_SLOT_REV;  // last warp takes the odd 32-particle block, not warp 0

// Optional per-phase cycle accounting of rollout 0 (threads 0 and 32), for tuning
// builds only (-DVPM_PHASE_TIMING; read back with vpm_debug_phase_cycles).
#ifdef VPM_PHASE_TIMING
__device__ unsigned long long g_phase[2][12];
// cycles accumulate in registers (a global read-modify-write per mark would sit on
// the critical path); PHASE_FLUSH writes them once after the step loop
#define PHASE_INIT                  \
  long long ph_last_ = clock64();   \
  unsigned long long ph_acc_[12] = {}
#define PHASE_MARK(i)                                                   \
  do {                                                                  \
    const long long now_ = clock64();                                   \
    ph_acc_[i] += (unsigned long long)(now_ - ph_last_);                \
    ph_last_ = now_;                                                    \
  } while (0)
#define PHASE_FLUSH                                                                 \
  do {                                                                              \
    if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 32))                 \
      for (int i_ = 0; i_ < 12; ++i_) g_phase[threadIdx.x >> 5][i_] += ph_acc_[i_]; \
  } while (0)
#else
#define PHASE_INIT
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#define PHASE_FLUSH \
  do {              \
  } while (0)
#endif
constexpr double TWO_PI = 6.283185307179586476925286766559;
constexpr double INV_TWO_PI = 0.15915494309189533576888376337251;
constexpr double PI = 3.14159265358979323846264338327950288;

struct Phys {
  int nb, cap;
  double r_core, k_diss, shed_off, crit_aoa, rho, dt, m, inertia, g, l, l_w, l_e, l_chord, s_e,
      phi_lim, u_lim, lev_gain, eta;
  // derived on the host: reciprocals of the constant divisors of the per-step
  // chain, panel length, cos(critical aoa) (-2 when the gate can never open)
  double inv_dt, inv_m, inv_inertia, s_pan, inv_s, cos_crit;
  float rc4f;
};

struct Args {
  Phys P;
  const double *ainv;  // 3 variants x (nb+2)^2, row-major; variant 0 (attached) stride nb
  // fluid snapshot, FP64 reference layout
  const double *wpos, *wgam;
  const int64_t *wage;
  int n_wake, ring_a, ring_b;
  const double *ppos, *pgam;
  int n_prev;
  double prev_lev;
  const double *ema;
  // start state
  const double *x0;
  int x0_stride;
  // device copies of the snapshot scalars {n_wake, ring_a, ring_b, n_prev} and
  // prev_lev; when set they override the host values (device-resident snapshots)
  const int32_t *snap_scal;
  const double *snap_plev;
  // per-row start-state perturbation: x0 += x0_noise[row] * x0_scale (policy cloud)
  const double *x0_noise, *x0_scale;
  // controls: explicit rows, MPPI sampling from u* and noise, or feedback
  const double *controls;
  const double *ustar, *noise;
  double sigma;
  // feedback u = clip(-K_k (x - tau_k) + xi_k), k = rint((t - t_start)/dt) clamped
  // (project_forward, nmpc.py:88-103; evaluate_policy, policy.py:236-244)
  const double *pol_gains, *pol_states, *pol_inputs;
  int pol_h;
  double pol_t_start, pol_t0;
  const double *pol_times;  // optional device {t_start, t0} (graph replay) overriding the two above
  // single-step mode (vpm_plan_step): start state and control by value
  double u_const;
  int use_u_const;
  double x0v[7];
  int use_x0v;
  int T, row_begin, rows;
  int integrate, check_envelope, need_fluid, record;
  int sym;  // symmetric-pair convection sweep: NT = 32 T warps of 128-particle tiles
  // outputs (any may be null)
  int64_t *status;
  double *finals, *trajs, *cost;
  const double *q, *xp;
  uint64_t *shed_mask;     // steps 0..63
  uint64_t *shed_mask_hi;  // steps 64..127
  uint64_t *wake_hash;     // wake-index signature (wake_sig_* below)
  int32_t *n_final;
  int64_t *inter;
  int32_t *rc_out;
  double *fw_out;  // (rows, 3): fw_x, fw_z, m_w of the last completed step
  double *o_wpos, *o_wgam;
  int64_t *o_wage;
  int32_t *o_scal;
  double *o_ppos, *o_pgam, *o_plev, *o_ema;
  int32_t *o_scal2;  // optional second copy of the dumped scalars (single-step mode)
};

struct Ctl {
  double x[7];
  double u;
  double fx, fz, nx, nz, s;
  double lx, lz, tx, tz;
  double lev_cur, lev_prev;
  double fwx, fwz, mw;
  int shed, rev;
  int hp;       // has_prev for the pending step's loads (n_prev > 0 at its start)
  int n_prev;   // rows in the previous bound row (0 or nb)
  int pending;  // loads + integration of the last solved step not yet applied
  int n_raw, n_live, ring_a, ring_b, n_holes;
  int holes[HOLES_MAX];
  int mcnt;     // merge candidates each warp keeps this step
  int fail, status, rc;
  int cur;      // wake buffer of the output dump: 0, or 1 after a failure in D
  double tacc;  // feedback mode: simulation time, accumulated like nmpc.py:102
  // precomputed by warp 1 while warp 0 runs E of the previous step: the elevator
  // force of the pending step {Ex, Ez, xe_x, xe_z} and sincos(theta_t)
  double el[4];
  double th_sn, th_cs;
  long long inter;
  unsigned long long shed_mask, shed_hi;
  unsigned long long whash, hsum;  // wake-index signature: step chain, final age sum
};

// ---- shared-memory layout (host computes the same size) ----------------------
struct Layout {
  int capbuf, nb, S, RS, nw, nblk;
  int off_psrc, off_st, off_ctl, off_d, off_red, off_cand, total;
};

__host__ __device__ inline int align16(int v) { return (v + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int cap, int nb, int nt, bool sym = false) {
  Layout L;
  L.capbuf = cap + WAKE_PAD;
  // the symmetric sweep keeps its 2 x 128 T float2 reaction buffers in wake buffer 0
  if (sym && L.capbuf < 4 * nt) L.capbuf = 4 * nt;
  L.nb = nb;
  L.S = nb + 2;
  L.RS = 2 * nb;                      // floats per source segment in the split sweeps
  L.nw = nt / 32;
  L.nblk = (L.capbuf + 31) / 32;      // 32-source blocks
  int off = 2 * L.capbuf * 16;        // double-buffered wake
  L.off_psrc = off;
  off += nb * 16;
  L.off_st = off;
  off += nb * 8;
  off = align16(off);
  L.off_ctl = off;
  off += align16((int)sizeof(Ctl));
  L.off_d = off;
  // cx cz bx bz gam pgp pxp pzp ema bvec (10 S) + pf (3 S) + Kelvin block sums (nblk)
  off += (13 * L.S + L.nblk) * 8;
  off = align16(off);
  L.off_red = off;
  off += NSEG * L.RS * 4;
  off = align16(off);
  L.off_cand = off;
  off += L.nw * MC * 4;
  L.total = align16(off);
  return L;
}

// ---- device helpers ------------------------------------------------------------
__device__ __forceinline__ float rsqrt_mufu(float v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// Wake-index signature (parity diagnostic, oracle/vpm_oracle.c computes the same):
// a chain over the steps of (wake size, ring-core indices, shed flag) after each
// step's shed / merge / ring termination (_core.pyx:322-373), then the sum over the
// final wake of mix(index, age) -- equal signatures mean the same shed steps, the
// same merge count per step and the same final (index -> age) order.
__host__ __device__ __forceinline__ unsigned long long wake_sig_mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ unsigned long long wake_sig_step(unsigned long long h, int n, int ra,
                                                                     int rb, int shed) {
  const unsigned long long key = (unsigned long long)(unsigned)n | ((unsigned long long)(shed != 0) << 31) |
                                 ((unsigned long long)(unsigned short)(ra + 1) << 32) |
                                 ((unsigned long long)(unsigned short)(rb + 1) << 48);
  return wake_sig_mix(h ^ key);
}
__host__ __device__ __forceinline__ unsigned long long wake_sig_elem(int c, int age) {
  return wake_sig_mix(((unsigned long long)(unsigned)c << 32) | (unsigned long long)(unsigned)age);
}

// One regularised Biot-Savart interaction (_core.pyx:89-97) in the form every
// path shares bitwise: with d' = s - t and c = g' / sqrt(r^4 + rc^4),
//   ax += c d'_z   (u_x = -ax)      az += c d'_x   (u_z = +az)
__device__ __forceinline__ void bs_chain(float sx, float sz, float sg, float ntx, float ntz,
                                         float rc4, float &ax, float &az) {
  const float dx = sx + ntx;
  const float dz = sz + ntz;
  const float r2 = fmaf(dx, dx, dz * dz);
  const float c = sg * rsqrt_mufu(fmaf(r2, r2, rc4));
  ax = fmaf(c, dz, ax);
  az = fmaf(c, dx, az);
}

// Register-tiled sweep: K targets per thread against n sources in shared memory,
// accumulated into (ax, az).  Pairs of targets run on the sm_100 f32x2 path
// (FADD2 / FMUL2 / FFMA2 take one issue slot for two lanes' worth of FP32 work, so
// the FMA pipe and the MUFU pipe -- 8 FP32 ops and 1 RSQ per interaction -- can
// both run near their rates); an odd target uses the scalar twin of the same math.
template <int K>
__device__ __forceinline__ void sweep_tile(const float4 *__restrict__ src, int n,
                                           const float *ntx, const float *ntz, float *ax,
                                           float *az, float rc4) {
  constexpr int KP = K / 2;
  float2 px[KP > 0 ? KP : 1], pz[KP > 0 ? KP : 1], qx[KP > 0 ? KP : 1], qz[KP > 0 ? KP : 1];
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    px[p] = make_float2(ntx[2 * p], ntx[2 * p + 1]);
    pz[p] = make_float2(ntz[2 * p], ntz[2 * p + 1]);
    qx[p] = make_float2(ax[2 * p], ax[2 * p + 1]);
    qz[p] = make_float2(az[2 * p], az[2 * p + 1]);
  }
  const float2 rc = make_float2(rc4, rc4);
  float ox = (K & 1) ? ax[K - 1] : 0.f, oz = (K & 1) ? az[K - 1] : 0.f;
#pragma unroll SWEEP_UNROLL
  for (int j = 0; j < n; ++j) {
    const float4 s = src[j];
    const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
#pragma unroll
    for (int p = 0; p < KP; ++p) {
      const float2 dx = __fadd2_rn(sx, px[p]);
      const float2 dz = __fadd2_rn(sz, pz[p]);
      const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
      const float2 q = __ffma2_rn(r2, r2, rc);
      const float2 rs = make_float2(rsqrt_mufu(q.x), rsqrt_mufu(q.y));
      const float2 c = __fmul2_rn(sg, rs);
      qx[p] = __ffma2_rn(c, dz, qx[p]);
      qz[p] = __ffma2_rn(c, dx, qz[p]);
    }
    if constexpr (K & 1) bs_chain(s.x, s.y, s.z, ntx[K - 1], ntz[K - 1], rc4, ox, oz);
  }
#pragma unroll
  for (int p = 0; p < KP; ++p) {
    ax[2 * p] = qx[p].x;
    ax[2 * p + 1] = qx[p].y;
    az[2 * p] = qz[p].x;
    az[2 * p + 1] = qz[p].y;
  }
  if constexpr (K & 1) {
    ax[K - 1] = ox;
    az[K - 1] = oz;
  }
}

// kw = number of target slots with at least one live lane in this warp (uniform).
// Not inlined on purpose: the sweep loop then gets the whole register budget for
// its interleaved interaction chains instead of sharing it with the kernel's
// outer state (inlined, ptxas serialised the chains through one temporary pair
// and MUFU latency went exposed); the call costs a few spills per step.
template <int R>
__device__ __noinline__ void sweep_dispatch(int kw, const float4 *src, int n, const float *ntx,
                                               const float *ntz, float *ax, float *az, float rc4) {
  switch (kw) {
    case 8: if constexpr (R >= 8) sweep_tile<8>(src, n, ntx, ntz, ax, az, rc4); break;
    case 7: if constexpr (R >= 7) sweep_tile<7>(src, n, ntx, ntz, ax, az, rc4); break;
    case 6: if constexpr (R >= 6) sweep_tile<6>(src, n, ntx, ntz, ax, az, rc4); break;
    case 5: if constexpr (R >= 5) sweep_tile<5>(src, n, ntx, ntz, ax, az, rc4); break;
    case 4: if constexpr (R >= 4) sweep_tile<4>(src, n, ntx, ntz, ax, az, rc4); break;
    case 3: if constexpr (R >= 3) sweep_tile<3>(src, n, ntx, ntz, ax, az, rc4); break;
    case 2: if constexpr (R >= 2) sweep_tile<2>(src, n, ntx, ntz, ax, az, rc4); break;
    case 1: sweep_tile<1>(src, n, ntx, ntz, ax, az, rc4); break;
    default: break;
  }
}

// ---- symmetric-pair convection sweep (tile schedule) --------------------------------
// Each unordered particle pair is evaluated once for both directions (the CPU core
// does the same, _core.pyx:203-214): 11 FP32 lane-ops + 1 MUFU.RSQ per pair instead of
// 2 x (8 + 1) for the two directed interactions.  The CTA has T warps; warp w owns the
// tile of particles 128 w + 32 k + lane (slot k = 0..3, held as the packed slot pairs
// (0,1) and (2,3)).  Pairs are covered as
//   - the own tile (and the previous bound row): direct, all four slots per
//     shared-memory broadcast source (rotating the tile's slots 2,3 past slots 0,1
//     instead measured slower: with one target pair per step the shuffles bound it);
//   - tile pairs (w, w+d), d = 1..(T-1)/2: warp w rotates every 32-particle block of
//     tile w+d through its lanes; the reactions go to a shared-memory buffer that the
//     owning warp adds after a barrier; for even T the pair (w, w+T/2) is split by
//     target rows (warp w: its slots 0,1 x all of tile w+T/2; warp w+T/2: all its
//     slots x blocks 2,3 of tile w).
// Lane rotation: lane l loads source 32 J + l of a block as its "packet" and the packet
// (coordinates and the reaction accumulated on it) moves one lane per step; after 32
// steps each target met every source of the block and the packet is home.  No
// cross-lane reduction and no atomics: every sum runs in a fixed order that depends
// only on T and the particle indices, so a rollout's result is the same in every launch
// with the same tile count (the launcher fixes T by the particle cap).

// targets NP packed slot pairs vs sources [j0, j1) (broadcast)
template <int NP>
__device__ __forceinline__ void sym_direct(const float4 *__restrict__ src, int j0, int j1, const float2 *px,
                                           const float2 *pz, float2 *qx, float2 *qz, float2 rc) {
#pragma unroll 4
  for (int j = j0; j < j1; ++j) {
    const float4 s = src[j];
    const float2 sx = make_float2(s.x, s.x), sz = make_float2(s.y, s.y), sg = make_float2(s.z, s.z);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const float2 dx = __fadd2_rn(sx, px[p]);
      const float2 dz = __fadd2_rn(sz, pz[p]);
      const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
      const float2 q = __ffma2_rn(r2, r2, rc);
      const float2 rs = make_float2(rsqrt_mufu(q.x), rsqrt_mufu(q.y));
      const float2 c = __fmul2_rn(sg, rs);
      qx[p] = __ffma2_rn(c, dz, qx[p]);
      qz[p] = __ffma2_rn(c, dx, qz[p]);
    }
  }
}

// NK packets (sx, sz, sg) rotated together through the lanes against NP packed
// target pairs (px, pz = negated target coordinates, pg = negated target Gamma/2pi);
// per step every packet meets the targets in packet order.  Returns the reaction on
// the lane's own packet sources in the (ax, az) convention.
template <int NP, int NK>
__device__ __forceinline__ void sym_rotate(float *sx, float *sz, float *sg, const float2 *px, const float2 *pz,
                                           const float2 *pg, float2 *qx, float2 *qz, float2 rc, int nxt,
                                           float *rbx, float *rbz) {
  float2 bx[NK], bz[NK];
#pragma unroll
  for (int k = 0; k < NK; ++k) bx[k] = bz[k] = make_float2(0.f, 0.f);
#pragma unroll(NK == 1 ? 4 : 2)
  for (int r = 0; r < 32; ++r) {
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      const float2 sx2 = make_float2(sx[k], sx[k]), sz2 = make_float2(sz[k], sz[k]),
                   sg2 = make_float2(sg[k], sg[k]);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float2 dx = __fadd2_rn(sx2, px[p]);
        const float2 dz = __fadd2_rn(sz2, pz[p]);
        const float2 r2 = __ffma2_rn(dx, dx, __fmul2_rn(dz, dz));
        const float2 q = __ffma2_rn(r2, r2, rc);
        const float2 rs = make_float2(rsqrt_mufu(q.x), rsqrt_mufu(q.y));
        const float2 cj = __fmul2_rn(sg2, rs);
        qx[p] = __ffma2_rn(cj, dz, qx[p]);
        qz[p] = __ffma2_rn(cj, dx, qz[p]);
        const float2 ci = __fmul2_rn(pg[p], rs);  // -g_target rs: reaction (t - s = -d')
        bx[k] = __ffma2_rn(ci, dz, bx[k]);
        bz[k] = __ffma2_rn(ci, dx, bz[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NK; ++k) {
      sx[k] = __shfl_sync(0xffffffffu, sx[k], nxt);
      sz[k] = __shfl_sync(0xffffffffu, sz[k], nxt);
      sg[k] = __shfl_sync(0xffffffffu, sg[k], nxt);
      bx[k].x = __shfl_sync(0xffffffffu, bx[k].x, nxt);
      bx[k].y = __shfl_sync(0xffffffffu, bx[k].y, nxt);
      bz[k].x = __shfl_sync(0xffffffffu, bz[k].x, nxt);
      bz[k].y = __shfl_sync(0xffffffffu, bz[k].y, nxt);
    }
  }
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    rbx[k] = bx[k].x + bx[k].y;
    rbz[k] = bz[k].x + bz[k].y;
  }
}

__device__ __forceinline__ float &slot_ref(float2 *v, int k) { return (k & 1) ? v[k >> 1].y : v[k >> 1].x; }

// The whole convection sweep of warp w (all warps call it: it contains the round
// barriers).  wb = compacted wake (nl particles), rb = reaction buffers (2 x 128 T
// float2, tile v's entries in float2 [256 v, 256 v + 256) so that the later advection
// writes of warp v only overwrite entries warp v has already consumed), psrc = previous
// bound row.  Returns (ax, az) of the warp's 4 slots; u_x = -ax, u_z = az.
__device__ __noinline__ void sym_sweep(const float4 *__restrict__ wb, float2 *rb, int nl,
                                       const float4 *__restrict__ psrc, int n_prev, float rc4, int T, int w,
                                       float *ax4, float *az4) {
  const int lane = threadIdx.x & 31, nxt = (lane + 1) & 31;
  const float2 rc = make_float2(rc4, rc4);
  const int base = 128 * w;
  float2 px[2], pz[2], pg[2], qx[2], qz[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int c0 = base + 64 * p + lane, c1 = c0 + 32;
    const float4 v0 = c0 < nl ? wb[c0] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 v1 = c1 < nl ? wb[c1] : make_float4(0.f, 0.f, 0.f, 0.f);
    px[p] = make_float2(-v0.x, -v1.x);
    pz[p] = make_float2(-v0.y, -v1.y);
    pg[p] = make_float2(-v0.z, -v1.z);
    qx[p] = make_float2(0.f, 0.f);
    qz[p] = make_float2(0.f, 0.f);
  }
  const bool act0 = base < nl, act1 = base + 64 < nl;
  // previous bound row and the own tile, direct (all four slots per broadcast source)
  if (act1) {
    sym_direct<2>(psrc, 0, n_prev, px, pz, qx, qz, rc);
    sym_direct<2>(wb, base, min(base + 128, nl), px, pz, qx, qz, rc);
  } else if (act0) {
    sym_direct<1>(psrc, 0, n_prev, px, pz, qx, qz, rc);
    sym_direct<1>(wb, base, min(base + 64, nl), px, pz, qx, qz, rc);
  }
  // tile pairs (w, w+d): warp w rotates tile w+d's blocks, the owner adds the reactions.
  // Blocks m0..m1-1 of tile v against np target pairs; pairs of blocks go together
  // when only target pair 0 takes part (more independent chains per step).
  auto sweep_blocks = [&](int v, int m0, int m1, int np, float2 *dst) {
    int m = m0;
    while (m < m1 && 128 * v + 32 * m < nl) {
      const int j = 128 * v + 32 * m;
      if (np == 1 && m + 1 < m1 && j + 32 < nl) {
        const float4 s0 = j + lane < nl ? wb[j + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 s1 = j + 32 + lane < nl ? wb[j + 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        float sx[2] = {s0.x, s1.x}, sz[2] = {s0.y, s1.y}, sg[2] = {s0.z, s1.z};
        float rbx[2], rbz[2];
        sym_rotate<1, 2>(sx, sz, sg, px, pz, pg, qx, qz, rc, nxt, rbx, rbz);
        dst[32 * m + lane] = make_float2(rbx[0], rbz[0]);
        dst[32 * m + 32 + lane] = make_float2(rbx[1], rbz[1]);
        m += 2;
      } else {
        const float4 s0 = j + lane < nl ? wb[j + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        float sx[1] = {s0.x}, sz[1] = {s0.y}, sg[1] = {s0.z};
        float rbx[1], rbz[1];
        if (np == 2) sym_rotate<2, 1>(sx, sz, sg, px, pz, pg, qx, qz, rc, nxt, rbx, rbz);
        else sym_rotate<1, 1>(sx, sz, sg, px, pz, pg, qx, qz, rc, nxt, rbx, rbz);
        dst[32 * m + lane] = make_float2(rbx[0], rbz[0]);
        m += 1;
      }
    }
  };
  auto receive = [&](const float2 *src, int k0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < k0 || base + 32 * k >= nl) continue;
      const float2 r = src[32 * k + lane];
      slot_ref(qx, k) += r.x;
      slot_ref(qz, k) += r.y;
    }
  };
  const int np = act1 ? 2 : 1;
  const int D = (T - 1) >> 1;
  for (int d = 1; d <= D; ++d) {
    const int v = w + d < T ? w + d : w + d - T;
    if (act0) sweep_blocks(v, 0, 4, np, rb + 256 * v + 128 * (d & 1));
    __syncthreads();
    const int u = w - d >= 0 ? w - d : w - d + T;  // the warp that rotated this tile
    if (act0 && 128 * u < nl) receive(rb + 256 * w + 128 * (d & 1), 0);
  }
  if (T >= 2 && (T & 1) == 0) {
    const int d = T >> 1;
    if (w < d) {  // slots 0,1 x all of tile w+d
      if (act0) sweep_blocks(w + d, 0, 4, 1, rb + 256 * (w + d) + 128 * (d & 1));
    } else {  // all slots x blocks 2,3 of tile w-d
      if (act0) sweep_blocks(w - d, 2, 4, np, rb + 256 * (w - d) + 128 * (d & 1));
    }
    __syncthreads();
    if (w < d) {
      if (act1 && 128 * (w + d) < nl) receive(rb + 256 * w + 128 * (d & 1), 2);
    } else {
      if (act0 && 128 * (w - d) < nl) receive(rb + 256 * w + 128 * (d & 1), 0);
    }
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    ax4[k] = slot_ref(qx, k);
    az4[k] = slot_ref(qz, k);
  }
}

// Deterministic butterfly-transpose reduction of 8 floats across a warp:
// afterwards every lane holds the full sum of value index (lane >> 2).
__device__ __forceinline__ float warp_reduce8(float v[8], int lane) {
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = h16 ? v[i] : v[i + 4];
    const float keep = h16 ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = h8 ? v[i] : v[i + 2];
    const float keep = h8 ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const float send = h4 ? v[0] : v[1];
    const float keep = h4 ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// raw slot of the c-th live particle, skipping the sorted hole list
// ROLLED: keep the hole loop rolled (a few instructions instead of the unrolled copy).
// The small-tile kernels (R < 4) use it in the epilogue: with many short rollouts per
// SM (C5 N = 128: 16 CTAs per SM, 5 steps) they are instruction-fetch bound (ncu:
// no_instruction 26% of the stall samples) and the prologue / epilogue are a large
// part of every CTA's instruction stream -- C5 N = 128 -6.5%, C3 -0.8%.  In the
// large kernels the same edit shifted C4 by +0.7% (code layout), so they keep the
// unrolled form.
template <bool ROLLED = false>
__device__ __forceinline__ int raw_index(int c, const int *holes, int nh) {
  int r = c;
  if constexpr (ROLLED) {
#pragma unroll 1
    for (int h = 0; h < nh; ++h)
      if (holes[h] <= r) ++r;
  } else {
    for (int h = 0; h < nh; ++h)
      if (holes[h] <= r) ++r;
  }
  return r;
}

// Source-split sweep for a handful of targets tgt[0..nt) (the nb panel or
// collocation points): the sources are cut into NSEG fixed segments and every
// (target, segment) pair is one sequential chain on one thread, stored as
// red[(k NSEG + seg) 2 (+1)] = (sum c d'_z, sum c d'_x) -- target-major: consecutive
// tasks write consecutive float pairs, free of bank conflicts (the segment-major
// layout cost the 513-row shard 3.7%) -- and consumers add the segments in order.  The
// cut depends only on n, so the result does not depend on the CTA shape; no
// cross-lane reductions are needed.
__device__ __forceinline__ void split_sweep(const float4 *__restrict__ src, int n,
                                            const float2 *tgt, int nt, float rc4, float *red,
                                            int RS, int tid, int nthreads) {
  const int len = (n + NSEG - 1) / NSEG;
  for (int task = tid; task < nt * NSEG; task += nthreads) {
    const int k = task / NSEG, seg = task - k * NSEG;
    const float ntx = -tgt[k].x, ntz = -tgt[k].y;
    const int j1 = min(n, (seg + 1) * len);
    float ax = 0.f, az = 0.f;
#pragma unroll 4
    for (int j = seg * len; j < j1; ++j) {
      const float4 s = src[j];
      bs_chain(s.x, s.y, s.z, ntx, ntz, rc4, ax, az);
    }
    red[(k * NSEG + seg) * 2] = ax;
    red[(k * NSEG + seg) * 2 + 1] = az;
  }
}

// wake velocity at split target k from the per-segment partials (segment order)
__device__ __forceinline__ void split_result(const float *red, int k, double &ux, double &uz) {
  double sx = 0.0, sz = 0.0;
  for (int b = 0; b < NSEG; ++b) {
    sx += (double)red[(k * NSEG + b) * 2];
    sz += (double)red[(k * NSEG + b) * 2 + 1];
  }
  ux = -sx;
  uz = sz;
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v > hi ? hi : (v < lo ? lo : v);
}

// control of global candidate row g at step t (mppi.py:37-43, :79; _core.pyx:183-187)
__device__ __forceinline__ double control_at(const Args &a, int row, int t, const double *x,
                                             double tacc) {
  double u;
  if (a.use_u_const) {
    u = a.u_const;
  } else if (a.pol_gains) {
    // evaluate_policy (policy.py:236-244): Python round() is round-half-even = rint
    const double t_start = a.pol_times ? a.pol_times[0] : a.pol_t_start;
    int k = (int)rint((tacc - t_start) * a.P.inv_dt);
    k = k < 0 ? 0 : (k > a.pol_h - 1 ? a.pol_h - 1 : k);
    double dot = 0.0;
    for (int j = 0; j < 7; ++j) dot += a.pol_gains[k * 7 + j] * (x[j] - a.pol_states[k * 7 + j]);
    u = clampd(-dot + a.pol_inputs[k], -a.P.u_lim, a.P.u_lim);
  } else if (a.controls) {
    u = a.controls[(size_t)row * a.T + t];
  } else {
    const int g = a.row_begin + row;
    u = a.ustar[t];
    if (g > 0) u = clampd(u + a.noise[(size_t)(g - 1) * a.T + t] * a.sigma, -a.P.u_lim, a.P.u_lim);
  }
  return u;
}

// ---- the rollout kernel -------------------------------------------------------------
// R = register-tile target slots per thread; blockDim.x * R >= cap + 4 (host
// guarantees), so every live particle is a register target.  MAXREG = register
// budget per thread (64: 8 CTAs of 128 threads per SM, 72: 7, 80: 6).
template <int R, int MAXREG>
__global__ void __maxnreg__(MAXREG) rollout_kernel(const Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Phys &P = a.P;
  const int nb = P.nb;
  const int NT = blockDim.x, NW = NT >> 5;
  const Layout L = make_layout(P.cap, nb, NT, a.sym != 0);
  float4 *wbuf = reinterpret_cast<float4 *>(smem);  // two wake buffers of capbuf
  float4 *psrc = reinterpret_cast<float4 *>(smem + L.off_psrc);
  float2 *st = reinterpret_cast<float2 *>(smem + L.off_st);
  Ctl *ctl = reinterpret_cast<Ctl *>(smem + L.off_ctl);
  double *dsh = reinterpret_cast<double *>(smem + L.off_d);
  const int S = L.S, RS = L.RS;
  double *cx = dsh, *cz = dsh + S, *bx = dsh + 2 * S, *bz = dsh + 3 * S, *gam = dsh + 4 * S;
  double *pgp = dsh + 5 * S, *pxp = dsh + 6 * S, *pzp = dsh + 7 * S, *ema = dsh + 8 * S;
  double *bvec = dsh + 9 * S, *pf = dsh + 10 * S, *kblk = dsh + 13 * S;
  float *red = reinterpret_cast<float *>(smem + L.off_red);
  unsigned *cand = reinterpret_cast<unsigned *>(smem + L.off_cand);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row = blockIdx.x;
  const int T = a.T;
  const float rc4 = P.rc4f;
  const double dt = P.dt;
  PHASE_INIT;

  // ---- prologue: fork the snapshot into shared memory (_core.pyx:494-526)
  const int sn_wake = a.snap_scal ? a.snap_scal[0] : a.n_wake;
  const int sn_prev = a.snap_scal ? a.snap_scal[3] : a.n_prev;
  for (int i = tid; i < sn_wake; i += NT)
    wbuf[i] = make_float4((float)a.wpos[2 * i], (float)a.wpos[2 * i + 1],
                          (float)(a.wgam[i] * INV_TWO_PI), __int_as_float((int)a.wage[i]));
  for (int j = tid; j < sn_prev; j += NT)
    psrc[j] = make_float4((float)a.ppos[2 * j], (float)a.ppos[2 * j + 1],
                          (float)(a.pgam[j] * INV_TWO_PI), 0.f);
  if (warp == 0) {
    for (int j = lane; j < nb; j += 32) {
      const bool have = j < sn_prev;
      pgp[j] = have ? a.pgam[j] : 0.0;
      pxp[j] = have ? a.ppos[2 * j] : 0.0;
      pzp[j] = have ? a.ppos[2 * j + 1] : 0.0;
      ema[j] = a.ema[j];
    }
    const double *x0 = a.use_x0v ? a.x0v : a.x0 + (size_t)row * a.x0_stride;
    if (lane < 7) {
      double xv = x0[lane];
      if (a.x0_noise) xv += a.x0_noise[(size_t)row * 7 + lane] * a.x0_scale[lane];
      ctl->x[lane] = xv;
      if (a.record && a.trajs) a.trajs[(size_t)row * (T + 1) * 7 + lane] = xv;
    }
    if (lane == 0) {
      ctl->n_raw = sn_wake;
      ctl->n_live = sn_wake;
      ctl->n_holes = 0;
      ctl->ring_a = a.snap_scal ? a.snap_scal[1] : a.ring_a;
      ctl->ring_b = a.snap_scal ? a.snap_scal[2] : a.ring_b;
      ctl->n_prev = sn_prev;
      ctl->lev_prev = a.snap_plev ? a.snap_plev[0] : a.prev_lev;
      ctl->tacc = a.pol_times ? a.pol_times[1] : a.pol_t0;
      ctl->lev_cur = 0.0;
      ctl->pending = 0;
      ctl->mcnt = min(MC, max(0, sn_wake + 3 - P.cap));
      ctl->fail = 0;
      ctl->status = 0;
      ctl->rc = 0;
      ctl->inter = 0;
      ctl->shed_mask = 0ull;
      ctl->shed_hi = 0ull;
      ctl->whash = 0ull;
      ctl->hsum = 0ull;
      ctl->fwx = ctl->fwz = ctl->mw = 0.0;
      ctl->hp = 0;
      ctl->shed = ctl->rev = 0;
      ctl->cur = 0;
    }
  }
  __syncthreads();

  for (int t = 0;; ++t) {
    const bool conv = t < T;
    const bool pend = ctl->pending;
    const int n_raw = ctl->n_raw, n_live = ctl->n_live, nh = ctl->n_holes;
    const int n_prev = ctl->n_prev;
    // Buffer 0 holds the wake (raw: removed particles are zero-circulation holes until
    // the next advection compacts them); buffer 1 receives a compacted copy at the top
    // of every convecting iteration, which the convection sweep reads (sources and
    // targets), while the advection writes the new wake back into buffer 0.
    float4 *wake = wbuf;
    float4 *wcmp = wbuf + L.capbuf;
    const bool sym = R >= 4 && a.sym && conv && n_live <= 128 * NW;  // uniform over the CTA
    // the control phase D runs on warp 0, or with the symmetric sweep on the last warp
    // (warp 0 runs E)
    const int dwarp = sym ? NW - 1 : 0;

    // ---------------- P1: wake velocity at the panels of step t-1 (its loads),
    // source-split over all warps.  (Carrying the 10 panel targets in one warp's
    // register sweep instead costs that warp a whole extra 32-target slot -- +25%
    // on the critical path at N=512 -- so the split sweep stays.)
    if (pend) split_sweep(wake, n_raw, st, nb, rc4, red, RS, tid, NT);
    if (conv)
      for (int c = tid; c < n_live; c += NT) wcmp[c] = wake[nh ? raw_index(c, ctl->holes, nh) : c];
    PHASE_MARK(0);
    __syncthreads();  // B1
    PHASE_MARK(1);

    // P2 runs in two passes: pass D_PASS is warp 0's control work, the other the
    // sweep + advection of every warp.
    for (int pass = 0; pass < 2; ++pass) {
    // ---------------- P2, control warp: D = loads + integration of step t-1,
    //                  geometry / gates / control of step t
    if (pass == D_PASS && warp == dwarp) {
      // The elevator force of the pending step and sincos(theta_t) were computed by
      // warp 1 during the previous E (they depend only on x_{t-1}, u_{t-1}); lane 29
      // prefetches the next open-loop control value (a global load).
      double u_next = 0.0;
      const bool feedback = a.pol_gains != nullptr;
      if (conv && lane == 29 && !feedback) u_next = control_at(a, row, t, ctl->x, ctl->tacc);
      if (pend) {
        const double fx = ctl->fx, fz = ctl->fz, nx = ctl->nx, nz = ctl->nz, s = ctl->s;
        const double rx = ctl->x[0], rz = ctl->x[1], vx = ctl->x[4], vz = ctl->x[5], om = ctl->x[6];
        const double th = ctl->x[2], phi = ctl->x[3], u = ctl->u;
        const int hp = ctl->hp;
        const double xwx = rx - P.l_w * fx, xwz = rz - P.l_w * fz;
        const double dlev = hp ? (ctl->lev_cur - ctl->lev_prev) * P.inv_dt : 0.0;

        double Fx, Fz, M;
        if (nb <= 32) {
          // one panel per lane: the cumulative circulations by a warp scan and the
          // force / moment sums by a fixed butterfly instead of per-lane serial loops
          const int p = lane;
          const bool act = p < nb;
          double uxp = 0.0, uzp = 0.0;
          if (act) split_result(red, p, uxp, uzp);
          double cum = act ? gam[p] : 0.0, cum_prev = act ? pgp[p] : 0.0;
          for (int o = 1; o < nb; o <<= 1) {
            const double c1 = __shfl_up_sync(0xffffffffu, cum, o);
            const double c2 = __shfl_up_sync(0xffffffffu, cum_prev, o);
            if (lane >= o) {
              cum += c1;
              cum_prev += c2;
            }
          }
          double pfx = 0.0, pfz = 0.0, pm = 0.0;
          if (act) {
            const double rate = hp ? (cum - cum_prev) * P.inv_dt + dlev : 0.0;
            const double e = P.eta * rate + (1.0 - P.eta) * (hp ? ema[p] : 0.0);
            const double svx = vx + om * (-(bz[p] - rz)), svz = vz + om * (bx[p] - rx);
            const double beta = (uxp - svx) * fx + (uzp - svz) * fz;
            const double dp = P.rho * (beta * gam[p] * P.inv_s + e);
            pfx = dp * s * nx;
            pfz = dp * s * nz;
            pm = (bx[p] - xwx) * pfz - (bz[p] - xwz) * pfx;
            ema[p] = e;
          }
          Fx = warp_sum_d(pfx);
          Fz = warp_sum_d(pfz);
          M = warp_sum_d(pm);
          __syncwarp();
          PHASE_MARK(9);
          if (act) { pgp[p] = gam[p]; pxp[p] = bx[p]; pzp[p] = bz[p]; }
        } else {
          for (int p = lane; p < nb; p += 32) {
            double uxp, uzp;
            split_result(red, p, uxp, uzp);
            double cum = 0.0, cum_prev = 0.0;
            for (int i = 0; i <= p; ++i) { cum += gam[i]; cum_prev += pgp[i]; }
            const double rate = hp ? (cum - cum_prev) * P.inv_dt + dlev : 0.0;
            const double e = P.eta * rate + (1.0 - P.eta) * (hp ? ema[p] : 0.0);
            const double svx = vx + om * (-(bz[p] - rz)), svz = vz + om * (bx[p] - rx);
            const double beta = (uxp - svx) * fx + (uzp - svz) * fz;
            const double dp = P.rho * (beta * gam[p] * P.inv_s + e);
            const double pfx = dp * s * nx, pfz = dp * s * nz;
            pf[3 * p] = pfx;
            pf[3 * p + 1] = pfz;
            pf[3 * p + 2] = (bx[p] - xwx) * pfz - (bz[p] - xwz) * pfx;
            ema[p] = e;
          }
          __syncwarp();
          PHASE_MARK(9);
          for (int p = lane; p < nb; p += 32) { pgp[p] = gam[p]; pxp[p] = bx[p]; pzp[p] = bz[p]; }
          // wing force / moment sums, one component per lane, panel order as _core.pyx:404-406
          double fc = 0.0;
          if (lane < 3)
            for (int p = 0; p < nb; ++p) fc += pf[3 * p + lane];
          Fx = __shfl_sync(0xffffffffu, fc, 0);
          Fz = __shfl_sync(0xffffffffu, fc, 1);
          M = __shfl_sync(0xffffffffu, fc, 2);
        }
        if (lane == 0) {
          ctl->fwx = Fx; ctl->fwz = Fz; ctl->mw = M;
          ctl->lev_prev = ctl->lev_cur;
          ctl->pending = 0;
          ctl->tacc += dt;  // nmpc.py:102, t += dt after each step
        }
        if (a.integrate) {
          // accelerations + forward Euler (_core.pyx:439-461), uniform on every lane
          // (the three divisions are independent and pipeline); the elevator force
          // comes from warp 1 (ctl->el)
          const double Ex = ctl->el[0], Ez = ctl->el[1], xex = ctl->el[2], xez = ctl->el[3];
          const double ax = (Fx + Ex) * P.inv_m;
          const double az = (Fz + Ez) * P.inv_m - P.g;
          const double wd =
              (M + ((xwx - rx) * Fz - (xwz - rz) * Fx) + ((xex - rx) * Ez - (xez - rz) * Ex)) * P.inv_inertia;
          const double xn[7] = {rx + dt * vx, rz + dt * vz, th + dt * om,
                                clampd(phi + dt * u, -P.phi_lim, P.phi_lim), vx + dt * ax,
                                vz + dt * az, om + dt * wd};
          bool fin = true;
#pragma unroll
          for (int i = 0; i < 7; ++i) fin = fin && isfinite(xn[i]);
          // lane i stores component i: a select chain, not a 7-way divergent switch
          double xl = xn[0];
#pragma unroll
          for (int i = 1; i < 7; ++i) xl = lane == i ? xn[i] : xl;
          if (lane < 7) ctl->x[lane] = xl;
          if (lane == 0) {
            bool failed = false;
            if (!fin) {
              ctl->fail = 1; ctl->status = t; ctl->rc = 2; failed = true;
            } else if (a.check_envelope && (fabs(xn[6]) > 300.0 || fabs(xn[4]) > 80.0 || fabs(xn[5]) > 80.0)) {
              ctl->fail = 1; ctl->status = t; ctl->rc = 0; failed = true;
            }
            // the failure-time wake: this iteration's advection already rewrote
            // buffer 0, its compacted copy in buffer 1 is the wake of step t-1
            if (failed && conv) { ctl->cur = 1; ctl->n_raw = n_live; ctl->n_holes = 0; }
          }
        }
        __syncwarp();
        PHASE_MARK(10);
        if (a.record && a.trajs && lane < 7 && !ctl->fail)
          a.trajs[((size_t)row * (T + 1) + t) * 7 + lane] = ctl->x[lane];
      }
      PHASE_MARK(11);
      if (conv) u_next = __shfl_sync(0xffffffffu, u_next, 29);
      if (conv && !ctl->fail) {
        // chord frame, collocation points, gates of step t (_core.pyx:228-256)
        const double rx = ctl->x[0], rz = ctl->x[1], th = ctl->x[2];
        const double vx = ctl->x[4], vz = ctl->x[5], om = ctl->x[6];
        double sn = ctl->th_sn, cs = ctl->th_cs;  // sincos(theta_t) from warp 1
        if (!pend) sincos(th, &sn, &cs);
        const double fx = cs, fz = sn, nx = -sn, nz = cs;
        const double s = P.s_pan;
        for (int i = lane; i <= nb; i += 32) { cx[i] = rx - fx * s * i; cz[i] = rz - fz * s * i; }
        for (int j = lane; j < nb; j += 32) {
          const double c0x = rx - fx * s * j, c0z = rz - fz * s * j;
          bx[j] = c0x - 0.5 * s * fx;
          bz[j] = c0z - 0.5 * s * fz;
        }
        // gates on the effective angle of attack aoa = wrap(theta - atan2(vw)) of
        // _core.pyx:247-256, tested without the angle: cos(aoa) = f.vw / |vw|, so
        // |aoa| > crit  <=>  f.vw < cos(crit) |vw|  and  |aoa| > pi/2  <=>  f.vw < 0
        // (|aoa| in [0, pi]; a vanishing relative wind gives aoa = 0, no gate)
        bool g_shed = false, g_rev = false;
        const double vwx = vx - P.l_w * om * nx, vwz = vz - P.l_w * om * nz;
        const double vw2 = vwx * vwx + vwz * vwz;
        if (vw2 >= 1e-18) {
          const double dot = fx * vwx + fz * vwz;
          g_shed = dot < P.cos_crit * sqrt(vw2);
          g_rev = dot < 0.0;
        }
        if (lane == 0) {
          ctl->fx = fx; ctl->fz = fz; ctl->nx = nx; ctl->nz = nz; ctl->s = s;
          ctl->lx = rx + P.shed_off * fx;
          ctl->lz = rz + P.shed_off * fz;
          ctl->tx = (rx - fx * s * nb) - P.shed_off * fx;
          ctl->tz = (rz - fz * s * nb) - P.shed_off * fz;
          ctl->shed = g_shed;
          ctl->rev = g_rev;
          const double u = feedback ? control_at(a, row, t, ctl->x, ctl->tacc) : u_next;
          ctl->u = clampd(u, -P.u_lim, P.u_lim);
        }
        __syncwarp();
        // collocation rows of step t for S2: the upstream edge point is skipped
        // (_core.pyx:274-275)
        const int shed_rev = ctl->shed && ctl->rev;
        for (int i = lane; i < nb; i += 32) {
          const int ri = shed_rev ? i : i + 1;
          st[i] = make_float2((float)cx[ri], (float)cz[ri]);
        }
      }
      PHASE_MARK(2);
    }
    const int wslot = SLOT_REV ? NW - 1 - warp : warp;
    if (pass != D_PASS && conv && !sym && 32 * wslot >= n_live) {
      // a warp without live targets (small wakes) only clears its merge candidates
      if (lane == 0)
        for (int r = 0; r < ctl->mcnt; ++r) cand[warp * MC + r] = 0u;
    } else if (pass != D_PASS && conv) {
      // ---------------- P2, all warps: S1 convection sweep of step t over the
      // compacted copy, then A (advect into buffer 0).  Direct path: slot k of warp w
      // holds the particles c = 32 (NW k + NW-1-w) + lane (the odd block lands on the
      // last warp, not on warp 0, which runs D after its slots).  Symmetric path:
      // warp w holds c = 128 w + 32 k + lane, k < 4.
      const int kmax = sym ? (R < 4 ? R : 4) : R;
      auto slot_base = [&](int k) { return sym ? 128 * warp + 32 * k : 32 * (NW * k + wslot); };
      float ux[R], uz[R];
      if (sym) {
        float ax4[4], az4[4];
        sym_sweep(wcmp, reinterpret_cast<float2 *>(wake), n_live, psrc, n_prev, rc4, NW, warp, ax4, az4);
#pragma unroll
        for (int k = 0; k < R; ++k) {
          ux[k] = k < 4 ? -ax4[k < 4 ? k : 0] : 0.f;
          uz[k] = k < 4 ? az4[k < 4 ? k : 0] : 0.f;
        }
      } else {
        float ntx[R], ntz[R], bx_[R], bz_[R];
        int kw = 0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const int c = slot_base(k) + lane;
          ntx[k] = 0.f;
          ntz[k] = 0.f;
          if (c < n_live) {
            const float4 v = wcmp[c];
            ntx[k] = -v.x;
            ntz[k] = -v.y;
          }
          if (slot_base(k) < n_live) kw = k + 1;
          ux[k] = 0.f;
          uz[k] = 0.f;
          bx_[k] = 0.f;
          bz_[k] = 0.f;
        }
        if (kw > 0) {  // a warp without live targets skips the calls (and their spills)
          sweep_dispatch<R>(kw, wcmp, n_live, ntx, ntz, ux, uz, rc4);
          sweep_dispatch<R>(kw, psrc, n_prev, ntx, ntz, bx_, bz_, rc4);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          ux[k] = -ux[k] - bx_[k];  // u_x = -(wake chain) - (bound-row chain)
          uz[k] = uz[k] + bz_[k];
        }
      }
      // A: advect / dissipate / age into slot c of buffer 0 (_core.pyx:222-226)
      const int ra = ctl->ring_a, rb = ctl->ring_b;
      unsigned keys[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int c = slot_base(k) + lane;
        keys[k] = 0u;
        double g = 0.0;
        if (k < kmax && c < n_live) {
          const float4 v = wcmp[c];
          const float nxp = (float)((double)v.x + dt * (double)ux[k]);
          const float nzp = (float)((double)v.y + dt * (double)uz[k]);
          const float ng = (float)((double)v.z * P.k_diss);
          const int na = __float_as_int(v.w) + 1;
          wake[c] = make_float4(nxp, nzp, ng, __int_as_float(na));
          g = (double)ng;
          if (c != ra && c != rb) keys[k] = ((unsigned)(na + 1) << 12) | (unsigned)(4095 - c);
        }
        // Kelvin sum over the canonical 32-particle block c / 32
        if (k < kmax && slot_base(k) < n_live) {
          g = warp_sum_d(g);
          if (lane == 0) kblk[slot_base(k) >> 5] = g;
        }
      }
      // keys are unique (the particle index is in the low bits), so the winner is
      // cleared by value: predicated selects, not a divergent switch on its slot
      const int mc = ctl->mcnt;
      for (int r = 0; r < mc; ++r) {
        unsigned best = 0u;
#pragma unroll
        for (int k = 0; k < R; ++k) best = max(best, keys[k]);
        const unsigned w = __reduce_max_sync(0xffffffffu, best);
        if (lane == 0) cand[warp * MC + r] = w;
#pragma unroll
        for (int k = 0; k < R; ++k) keys[k] = (w != 0u && keys[k] == w) ? 0u : keys[k];
      }
    }
      PHASE_MARK(3);
    }  // passes
    __syncthreads();  // B2
    PHASE_MARK(4);
    if (!conv || ctl->fail) break;

    // ---------------- S2: wake velocity at the collocation rows of step t
    split_sweep(wake, n_live, st, nb, rc4, red, RS, tid, NT);
    PHASE_MARK(5);
    __syncthreads();  // B3
    PHASE_MARK(6);

    // ---------------- E': warp 1, concurrently with E: the elevator flat-plate force
    // of the step just solved (it depends only on x_t and u_t, _core.pyx:423-437) and
    // sincos(theta_{t+1}) for the next geometry -- both off warp 0's critical path
    if (warp == 1 && lane == 0) {
      const double rx = ctl->x[0], rz = ctl->x[1], th = ctl->x[2], phi = ctl->x[3];
      const double vx = ctl->x[4], vz = ctl->x[5], om = ctl->x[6], u = ctl->u;
      const double fx = ctl->fx, fz = ctl->fz, nx = ctl->nx, nz = ctl->nz;
      double Ex = 0.0, Ez = 0.0, xex = 0.0, xez = 0.0;
      if (a.integrate) {
        double se, ce;
        sincos(th + phi, &se, &ce);
        const double fex = ce, fez = se, nex = -se, nez = ce;
        xex = rx - P.l * fx - P.l_e * fex;
        xez = rz - P.l * fz - P.l_e * fez;
        const double vex = vx - P.l * om * nx - P.l_e * (om + u) * nex;
        const double vez = vz - P.l * om * nz - P.l_e * (om + u) * nez;
        const double sp2 = vex * vex + vez * vez;
        if (sp2 >= 1e-18) {
          const double ae = th + phi - atan2(vez, vex);
          const double cn = 0.5 * P.rho * sp2 * P.s_e * 2.0 * sin(ae);
          Ex = cn * nex;
          Ez = cn * nez;
        }
      }
      ctl->el[0] = Ex;
      ctl->el[1] = Ez;
      ctl->el[2] = xex;
      ctl->el[3] = xez;
      double sn, cs;
      sincos(a.integrate ? th + dt * om : th, &sn, &cs);
      ctl->th_sn = sn;
      ctl->th_cs = cs;
    }
    // ---------------- E: solve, shed, merge, ring termination (warp 0)
    if (warp == 0) {
      const int shed = ctl->shed, rev = ctl->rev;
      const int ns = shed ? nb + 2 : nb, r0 = shed ? 1 : 0;
      const int nl = n_live;
      const int nblk2 = (nl + 31) >> 5;
      const double rx = ctl->x[0], rz = ctl->x[1], vx = ctl->x[4], vz = ctl->x[5], om = ctl->x[6];
      const double nx = ctl->nx, nz = ctl->nz;
      for (int i = lane; i < nb; i += 32) {
        double uxw, uzw;
        split_result(red, i, uxw, uzw);
        const int ri = (shed && rev) ? i : i + 1;
        const double px = cx[ri], pz = cz[ri];
        const double svx = vx + om * (-(pz - rz)), svz = vz + om * (px - rx);
        bvec[r0 + i] = (svx - uxw) * nx + (svz - uzw) * nz;
      }
      if (shed && lane == 0) {
        const int epan = rev ? nb - 1 : 0;
        bvec[0] = P.lev_gain * (ctl->n_prev > 0 ? pgp[epan] : 0.0);
        double tot = 0.0;
        for (int b = 0; b < nblk2; ++b) tot += kblk[b];
        bvec[nb + 1] = -(tot * TWO_PI);
      }
      __syncwarp();
      const int var = shed ? (rev ? 2 : 1) : 0;
      const double *Ai = a.ainv + (size_t)var * S * S;
      bool ok = true;
      for (int i = lane; i < ns; i += 32) {
        double acc = 0.0;
        for (int j = 0; j < ns; ++j) acc += Ai[i * ns + j] * bvec[j];
        gam[i] = acc;
        ok = ok && isfinite(acc);
      }
      ok = __all_sync(0xffffffffu, ok);
      __syncwarp();
      if (!ok) {
        if (lane == 0) {
          ctl->fail = 1; ctl->status = t + 1; ctl->rc = 2;
          ctl->n_raw = nl; ctl->n_holes = 0;
        }
      } else {
        const double levg = shed ? gam[nb] : 0.0;
        int n_now = nl;
        if (shed) {
          if (lane == 0) wake[nl] = make_float4((float)ctl->lx, (float)ctl->lz, (float)(gam[nb] * INV_TWO_PI), __int_as_float(0));
          if (lane == 1) wake[nl + 1] = make_float4((float)ctl->tx, (float)ctl->tz, (float)(gam[nb + 1] * INV_TWO_PI), __int_as_float(0));
          n_now = nl + 2;
        }
        __syncwarp();
        // ---- merge the oldest down to the cap: top-(m+1) by (age desc, index asc)
        int nholes = 0;
        int hl[HOLES_MAX];
        const int m = n_now - P.cap;
        int ra = ctl->ring_a, rb = ctl->ring_b;
        if (m > 0) {
          // gather the per-warp candidate lists: lane l holds entries l + 32 s
          const int mcn = ctl->mcnt;
          unsigned kk[5];
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int idx = lane + 32 * s4;
            kk[s4] = (mcn > 0 && idx < NW * mcn) ? cand[(idx / mcn) * MC + idx % mcn] : 0u;
          }
          // the particles shed this step (age 0, indices nl, nl+1) are candidates too
          kk[4] = 0u;
          if (shed && lane < 2) {
            const int id = nl + lane;
            if (id != ra && id != rb) kk[4] = (1u << 12) | (unsigned)(4095 - id);
          }
          // Selection and blob of the merged particles; both forms give the same bits.
          // Small-cap kernels (R < 4: latency-bound, C2 / replan) keep the winners
          // lane-distributed (no local-memory array: C2 -11%); the large kernels keep
          // the array form, which measured faster there (C4 -0.8%, 513-row shard -6%).
          if constexpr (R < 4) {
          // selection round r leaves its winner on lane r
          unsigned my_sel = 0u;
          int nsel = 0;
          for (int r = 0; r <= m && r < MC; ++r) {
            unsigned mine = 0u;
#pragma unroll
            for (int s5 = 0; s5 < 5; ++s5) mine = max(mine, kk[s5]);
            const unsigned w = __reduce_max_sync(0xffffffffu, mine);
            if (w == 0u) break;
            if (lane == r) my_sel = w;
            ++nsel;
#pragma unroll
            for (int s5 = 0; s5 < 5; ++s5)
              if (kk[s5] == w) kk[s5] = 0u;
          }
          if (nsel >= 2) {
            const int merges = min(m, nsel - 1);
            const int my_id = 4095 - (int)(my_sel & 4095u);
            const int idx0 = __shfl_sync(0xffffffffu, my_id, 0);
            float4 blob = wake[idx0];
            int lo = idx0;
            for (int r = 1; r <= merges; ++r) {
              const int id = __shfl_sync(0xffffffffu, my_id, r);
              const float4 p = wake[id];
              blob.x = 0.5f * (blob.x + p.x);
              blob.y = 0.5f * (blob.y + p.y);
              blob.z = blob.z + p.z;
              lo = min(lo, id);
            }
            __syncwarp();
            if (lane == 0) wake[lo] = blob;
            for (int r = 0; r <= merges; ++r) {
              const int id = __shfl_sync(0xffffffffu, my_id, r);
              if (id != lo) hl[nholes++] = id;
            }
          }
          } else {
          unsigned sel[MC];
          int nsel = 0;
          for (int r = 0; r <= m && r < MC; ++r) {
            unsigned mine = 0u;
#pragma unroll
            for (int s5 = 0; s5 < 5; ++s5) mine = max(mine, kk[s5]);
            const unsigned w = __reduce_max_sync(0xffffffffu, mine);
            if (w == 0u) break;
            sel[nsel++] = w;
#pragma unroll
            for (int s5 = 0; s5 < 5; ++s5)
              if (kk[s5] == w) kk[s5] = 0u;
          }
          if (nsel >= 2) {
            const int merges = min(m, nsel - 1);
            const int idx0 = 4095 - (int)(sel[0] & 4095u);
            float4 blob = wake[idx0];
            int lo = idx0;
            int ids[MC];
            ids[0] = idx0;
            for (int r = 1; r <= merges; ++r) {
              const int id = 4095 - (int)(sel[r] & 4095u);
              ids[r] = id;
              const float4 p = wake[id];
              blob.x = 0.5f * (blob.x + p.x);
              blob.y = 0.5f * (blob.y + p.y);
              blob.z = blob.z + p.z;
              lo = min(lo, id);
            }
            __syncwarp();
            if (lane == 0) wake[lo] = blob;
            for (int r = 0; r <= merges; ++r)
              if (ids[r] != lo) hl[nholes++] = ids[r];
          }
          }
        }
        // ---- ring termination against the offset chord (_core.pyx:359-373)
        if (ra >= 0 && rb >= 0) {
          __syncwarp();
          const float4 A0 = wake[ra], A1 = wake[rb];
          const double fx = ctl->fx, fz = ctl->fz;
          const double ox = -0.02 * P.l_chord * nx, oz = -0.02 * P.l_chord * nz;
          const double ax0 = A0.x, az0 = A0.y, ax1 = A1.x, az1 = A1.y;
          const double bx0 = rx + ox, bz0 = rz + oz;
          const double bx1 = rx - P.l_chord * fx + ox, bz1 = rz - P.l_chord * fz + oz;
          const double d1x = ax1 - ax0, d1z = az1 - az0, d2x = bx1 - bx0, d2z = bz1 - bz0;
          const double den = d1x * d2z - d1z * d2x;
          bool hit = false;
          if (den != 0.0) {  // 0 <= num / den <= 1 for both parameters, without dividing
            const double ex = bx0 - ax0, ez = bz0 - az0;
            const double nt = ex * d2z - ez * d2x, nu = ex * d1z - ez * d1x;
            hit = den > 0.0 ? (nt >= 0.0 && nt <= den && nu >= 0.0 && nu <= den)
                            : (nt <= 0.0 && nt >= den && nu <= 0.0 && nu >= den);
          }
          if (hit) {
            hl[nholes++] = ra;
            hl[nholes++] = rb;
            ra = -1;
            rb = -1;
          }
        }
        // sort holes ascending, zero their circulation, remap the ring indices
        int ra2 = ra, rb2 = rb;
        if constexpr (R < 4) {
          // lane-distributed: lane j holds hole j, its rank among the (distinct) holes
          // is its sorted position (small-cap kernels; the array form below is kept for
          // the large ones, see the merge selection above)
          int hv = -1;
#pragma unroll
          for (int h = 0; h < HOLES_MAX; ++h)
            if (h < nholes && lane == h) hv = hl[h];
          int rank = 0;
          for (int k = 0; k < nholes; ++k) rank += __shfl_sync(0xffffffffu, hv, k) < hv;
          __syncwarp();
          if (lane < nholes) {
            wake[hv].z = 0.f;
            ctl->holes[rank] = hv;
          }
          if (ra >= 0) ra2 = ra - __popc(__ballot_sync(0xffffffffu, lane < nholes && hv < ra));
          if (rb >= 0) rb2 = rb - __popc(__ballot_sync(0xffffffffu, lane < nholes && hv < rb));
        } else {
          for (int i = 1; i < nholes; ++i) {
            const int v = hl[i];
            int j = i - 1;
            while (j >= 0 && hl[j] > v) { hl[j + 1] = hl[j]; --j; }
            hl[j + 1] = v;
          }
          __syncwarp();
          if (lane < nholes) wake[hl[lane]].z = 0.f;
          for (int h = 0; h < nholes; ++h) {
            if (ra >= 0 && hl[h] < ra) --ra2;
            if (rb >= 0 && hl[h] < rb) --rb2;
          }
        }
        const int n_live_next = n_now - nholes;
        // previous bound row: sources of the next convection sweep, and the
        // panels are the split targets of the next loads sweep
        for (int p = lane; p < nb; p += 32) {
          psrc[p] = make_float4((float)bx[p], (float)bz[p], (float)(gam[p] * INV_TWO_PI), 0.f);
          st[p] = make_float2((float)bx[p], (float)bz[p]);
        }
        if (lane == 0) {
          ctl->lev_cur = levg;
          ctl->hp = ctl->n_prev > 0;
          ctl->n_prev = nb;
          ctl->pending = 1;
          ctl->n_raw = n_now;
          ctl->n_live = n_live_next;
          ctl->n_holes = nholes;
          if constexpr (R >= 4)
            for (int h = 0; h < nholes; ++h) ctl->holes[h] = hl[h];
          ctl->ring_a = ra2;
          ctl->ring_b = rb2;
          ctl->mcnt = min(MC, max(0, n_live_next + 3 - P.cap));
          if (shed && t < 64) ctl->shed_mask |= 1ull << t;
          if (shed && t >= 64 && t < 128) ctl->shed_hi |= 1ull << (t - 64);
          ctl->whash = wake_sig_step(ctl->whash, n_live_next, ra2, rb2, shed);
          ctl->inter += (long long)nl * (nl - 1) + (long long)n_prev * nl + (long long)nb * nl +
                        (long long)nb * n_live_next;
        }
      }
    }
    PHASE_MARK(7);
    __syncthreads();  // B4
    PHASE_MARK(8);
    if (ctl->fail) break;
  }
  __syncthreads();
  PHASE_FLUSH;

  // ---- epilogue: outputs
  if (a.wake_hash) {
    // final (index, age) sum of the signature; integer sums are order-free
    const int nl = ctl->n_live, nh = ctl->n_holes;
    const float4 *wfin = wbuf + ctl->cur * L.capbuf;
    unsigned long long hs = 0ull;
    for (int c = tid; c < nl; c += NT) hs += wake_sig_elem(c, __float_as_int(wfin[raw_index<(R < 4)>(c, ctl->holes, nh)].w));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, o);
    if (lane == 0) atomicAdd(&ctl->hsum, hs);
    __syncthreads();
  }
  if (tid == 0) {
    if (a.status) a.status[row] = ctl->status;
    if (a.rc_out) a.rc_out[row] = ctl->rc;
    if (a.shed_mask) a.shed_mask[row] = ctl->shed_mask;
    if (a.shed_mask_hi) a.shed_mask_hi[row] = ctl->shed_hi;
    if (a.wake_hash) a.wake_hash[row] = wake_sig_mix(ctl->whash ^ ctl->hsum);
    if (a.n_final) a.n_final[row] = ctl->n_live;
    if (a.inter) a.inter[row] = ctl->inter;
    if (a.fw_out) { a.fw_out[3 * row] = ctl->fwx; a.fw_out[3 * row + 1] = ctl->fwz; a.fw_out[3 * row + 2] = ctl->mw; }
    if (a.cost) {
      // terminal cost (mppi.py:28-34): inf when failed or non-finite
      double J = 0.0;
      for (int i = 0; i < 7; ++i) { const double d = ctl->x[i] - a.xp[i]; J += d * a.q[i] * d; }
      a.cost[row] = (ctl->status != 0 || !isfinite(J)) ? INFINITY : J;
    }
  }
  if (a.finals && tid < 7) a.finals[(size_t)row * 7 + tid] = ctl->x[tid];
  if (a.need_fluid && row == 0) {
    const int cap4 = P.cap + 4;
    const int nl = ctl->n_live, nh = ctl->n_holes;
    const float4 *wfin = wbuf + ctl->cur * L.capbuf;
    for (int c = tid; c < cap4; c += NT) {
      if (c < nl) {
        const float4 v = wfin[raw_index<(R < 4)>(c, ctl->holes, nh)];
        a.o_wpos[2 * c] = v.x;
        a.o_wpos[2 * c + 1] = v.y;
        a.o_wgam[c] = (double)v.z * TWO_PI;
        a.o_wage[c] = __float_as_int(v.w);
      } else {
        a.o_wpos[2 * c] = 0.0;
        a.o_wpos[2 * c + 1] = 0.0;
        a.o_wgam[c] = 0.0;
        a.o_wage[c] = 0;
      }
    }
    for (int p = tid; p < nb; p += NT) {
      const bool have = p < ctl->n_prev;
      a.o_ppos[2 * p] = have ? pxp[p] : 0.0;
      a.o_ppos[2 * p + 1] = have ? pzp[p] : 0.0;
      a.o_pgam[p] = have ? pgp[p] : 0.0;
      a.o_ema[p] = ema[p];
    }
    if (tid == 0) {
      a.o_scal[0] = nl;
      a.o_scal[1] = ctl->ring_a;
      a.o_scal[2] = ctl->ring_b;
      a.o_scal[3] = ctl->n_prev;
      a.o_plev[0] = ctl->lev_prev;
      if (a.o_scal2) {
        a.o_scal2[0] = nl;
        a.o_scal2[1] = ctl->ring_a;
        a.o_scal2[2] = ctl->ring_b;
        a.o_scal2[3] = ctl->n_prev;
      }
    }
  }
}

// ---- MPPI reductions -----------------------------------------------------------------
// Softmax partial of one shard (mppi.py:46-59): part = {J_min, Z, S[T]} with weights
// exp(-(J - J_min)/lambda) of the shard's rows and S_t their weighted clipped controls
// clip(u* + sigma noise).  A latency-bound streaming kernel: CTA c owns rows
// [64 c, 64 c + 64) -- each warp 8 consecutive rows, whose control rows (coalesced over
// t; rows with zero weight load nothing) it loads all at once -- and writes the chunk
// partial {J_min_c, Z_c, S_c[T]} relative to its own minimum.  The last CTA to finish
// (ticket) combines the chunks in a fixed two-level order, rescaled to the shard
// minimum, and re-arms the ticket (a one-CTA grid writes its record as the partial).
// Every sum has a fixed order, so the result does not depend on scheduling.  With
// ustar_out set (the single-device iteration) the finishing CTA also applies the
// update u* = S/Z, or raises the sticky failure flag when every row failed -- bitwise
// what mppi_combine_kernel computes from part with W = 1 (its rescaling factor is
// exp(-0) = 1), one launch fewer.  Measured alternative: one CTA of 32 warps looping
// over the rows (no ticket) was slower at every size from 257 rows up -- one SM's
// FP64 pipe then carries every row's exp and division.
constexpr int PCH_WARPS = 8, PCH_ROWS = 8 * PCH_WARPS;  // 256 threads, 64 rows per CTA

// fixed-order sum of v[w * stride], w = 0..n-1: four interleaved chains, then
// (c0 + c1) + (c2 + c3) -- a quarter of the dependent shared-load latency
__device__ __forceinline__ double sum_strided4(const double *v, int n, int stride) {
  double c[4] = {0.0, 0.0, 0.0, 0.0};
  int w = 0;
  for (; w < n; w += 4) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (w + q < n) c[q] += v[(w + q) * stride];
  }
  return (c[0] + c[1]) + (c[2] + c[3]);
}

// lanes' minimum by an xor butterfly (every lane gets it; min is order-free)
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o >= 1; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(32 * PCH_WARPS) mppi_partial_chunked_kernel(
    const double *__restrict__ cost, int rows, int row_begin, const double *ustar,
    const double *__restrict__ noise, double sigma, double ulim, int T, double lambda,
    double *__restrict__ chunks, unsigned *__restrict__ ticket, double *__restrict__ part, double *ustar_out,
    int32_t *__restrict__ flag) {
  // [NW][T+1] control sums (then the last CTA's group sums) | NW + NW reductions |
  // T+1 totals
  extern __shared__ double sh[];
  constexpr int NW = PCH_WARPS;
  double *sacc = sh, *sred = sh + NW * (T + 1), *stot = sred + 2 * NW;
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ld = T + 2;
  const int rw = blockIdx.x * PCH_ROWS + warp * 8;  // this warp's first row
  // the CTA's cost minimum (exact, order-free); lane j < 8 holds row j
  double Jl = (lane < 8 && rw + lane < rows) ? cost[rw + lane] : INFINITY;
  Jl = isfinite(Jl) ? Jl : INFINITY;
  double jm = warp_min(Jl);
  if (lane == 0) sred[warp] = jm;
  __syncthreads();
  jm = warp_min(lane < NW ? sred[lane] : INFINITY);
  const bool any = isfinite(jm);
  const double wl = (any && isfinite(Jl)) ? exp(-(Jl - jm) / lambda) : 0.0;
  const double z = warp_sum_d(wl);  // lanes >= 8 hold 0: fixed butterfly over the 8 rows
  // bit j: row j carries weight and has a noise row (row 0 of the batch is the
  // incumbent u* itself)
  const unsigned live = __ballot_sync(0xffffffffu, wl != 0.0 && row_begin + rw + lane > 0);
  for (int tc = 0; tc < T; tc += 64) {
    const int t0 = tc + lane, t1 = tc + 32 + lane;
    const double us0 = t0 < T ? ustar[t0] : 0.0, us1 = t1 < T ? ustar[t1] : 0.0;
    double a0 = 0.0, a1 = 0.0;
    // all 16 noise loads in flight at once: load-only predicated bodies (a branch
    // around load + arithmetic made them one round trip per row)
    double n0[8], n1[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double *nz = noise + (size_t)max(row_begin + rw + j - 1, 0) * T;
      const bool lj = (live >> j) & 1u;
      n0[j] = 0.0;
      n1[j] = 0.0;
      if (lj && t0 < T) n0[j] = nz[t0];
      if (lj && t1 < T) n1[j] = nz[t1];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // row order
      const double w = __shfl_sync(0xffffffffu, wl, j);
      const bool lj = (live >> j) & 1u;
      const double u0 = (lj && t0 < T) ? clampd(us0 + n0[j] * sigma, -ulim, ulim) : us0;
      const double u1 = (lj && t1 < T) ? clampd(us1 + n1[j] * sigma, -ulim, ulim) : us1;
      a0 += w * u0;
      a1 += w * u1;
    }
    if (t0 < T) sacc[warp * T + t0] = a0;
    if (t1 < T) sacc[warp * T + t1] = a1;
  }
  if (lane == 0) sred[NW + warp] = z;
  __syncthreads();
  // the CTA's record {J_min, Z, S[T]}: warps added in a fixed order
  const double Z = warp_sum_d(lane < NW ? sred[NW + lane] : 0.0);
  const bool solo = gridDim.x == 1;  // one chunk: the record is the shard partial
  double *mine = solo ? part : chunks + (size_t)blockIdx.x * ld;
  if (threadIdx.x == 0) {
    mine[0] = jm;
    mine[1] = Z;
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const double S = sum_strided4(sacc + t, NW, T);
    mine[2 + t] = S;
    // the W = 1 combine (mppi_combine_kernel): Z = 0 + Z_0 * 1, S_t = 0 + S_t,0 * 1
    if (solo && ustar_out && any) ustar_out[t] = (0.0 + S) / (0.0 + Z);
  }
  if (solo) {
    if (ustar_out && !any && threadIdx.x == 0 && flag) *flag = 1;  // sticky failure flag
    return;
  }
  // chunked: the last CTA combines the chunks in chunk order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int G = gridDim.x;
  // chunk records were written by other SMs: read them through L2 (__ldcg)
  // global minimum: all chunk minima loaded in parallel (min is exact, order-free)
  double gm = INFINITY;
  for (int c = threadIdx.x; c < G; c += blockDim.x) gm = fmin(gm, __ldcg(chunks + (size_t)c * ld));
  gm = warp_min(gm);
  if (lane == 0) sred[warp] = gm;
  __syncthreads();
  gm = warp_min(lane < NW ? sred[lane] : INFINITY);
  // Z and S in a fixed two-level order: warp w sums the contiguous chunk group
  // [w G / NW, (w+1) G / NW) in chunk order (lanes over the T+1 columns
  // {Z, S_0..S_T-1}, coalesced chunk-row loads), then the group sums are added in
  // group order.  The order depends only on G.
  double *gsum = sacc;  // [NW][T+1], the chunk's control sums are no longer needed
  const int c_lo = (int)((long long)warp * G / NW), c_hi = (int)((long long)(warp + 1) * G / NW);
  for (int col0 = 0; col0 < T + 1; col0 += 32) {
    const int col = col0 + lane;
    double acc = 0.0;
    int c = c_lo;
    for (; c + 8 <= c_hi; c += 8) {  // eight chunk rows in flight per lane (same order)
      double v[8], jc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        jc[q] = __ldcg(chunks + (size_t)(c + q) * ld);
        v[q] = col <= T ? __ldcg(chunks + (size_t)(c + q) * ld + 1 + col) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double sc = (isfinite(gm) && isfinite(jc[q])) ? exp(-(jc[q] - gm) / lambda) : 0.0;
        acc += v[q] * sc;
      }
    }
    for (; c < c_hi; ++c) {
      const double jc = __ldcg(chunks + (size_t)c * ld);
      const double v = col <= T ? __ldcg(chunks + (size_t)c * ld + 1 + col) : 0.0;
      const double sc = (isfinite(gm) && isfinite(jc)) ? exp(-(jc - gm) / lambda) : 0.0;
      acc += v * sc;
    }
    if (col <= T) gsum[warp * (T + 1) + col] = acc;
  }
  __syncthreads();
  for (int col = threadIdx.x; col < T + 1; col += blockDim.x) {
    double tot = 0.0;
    for (int w = 0; w < NW; ++w) tot += gsum[w * (T + 1) + col];
    part[1 + col] = tot;  // part[1] = Z, part[2 + t] = S_t
    stot[col] = tot;
  }
  if (threadIdx.x == 0) {
    part[0] = gm;
    *ticket = 0u;
  }
  if (ustar_out) {  // the W = 1 combine, from the totals on chip
    __syncthreads();
    if (!isfinite(gm)) {
      if (threadIdx.x == 0 && flag) *flag = 1;
    } else {
      for (int t = threadIdx.x; t < T; t += blockDim.x) ustar_out[t] = (0.0 + stot[1 + t]) / (0.0 + stot[0]);
    }
  }
}

// Combine W gathered partials in rank order.  The failure flag is
// sticky: set to 1 when every candidate failed (u* left unchanged), never cleared
// here -- callers zero it when an optimisation starts.
__global__ void mppi_combine_kernel(const double *__restrict__ parts, int W, int T, double lambda,
                                    double *__restrict__ ustar, int32_t *__restrict__ flag) {
  const int ld = T + 2;
  double jm = INFINITY;
  for (int r = 0; r < W; ++r) jm = fmin(jm, parts[r * ld]);
  if (!isfinite(jm)) {
    if (threadIdx.x == 0 && flag) *flag = 1;
    return;
  }
  double Z = 0.0;
  for (int r = 0; r < W; ++r) {
    const double j = parts[r * ld];
    if (isfinite(j)) Z += parts[r * ld + 1] * exp(-(j - jm) / lambda);
  }
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    double S = 0.0;
    for (int r = 0; r < W; ++r) {
      const double j = parts[r * ld];
      if (isfinite(j)) S += parts[r * ld + 2 + t] * exp(-(j - jm) / lambda);
    }
    ustar[t] = S / Z;
  }
}

// ---- device noise (performance mode) ----------------------------------
// Standard normals for rows [row_begin, row_begin + rows) of one iteration's (K, T)
// MPPI noise matrix.  One thread per (row, pair of steps): counter-based
// Philox4x32-10 keyed by seed, subsequence = global noise row, offset = iteration
// x 2^32 + 4 per pair (iterations never overlap, whatever T), Box-Muller in FP64
// (curand_normal2_double).  The value at (g, t) depends only on (seed, iteration,
// g, t), so every sharding of the rows draws the same numbers; writes coalesce.
// seed_iter (optional, graph replay): {seed, iteration} read on the device, the
// iteration argument then being an offset added to it.
__global__ void noise_philox_kernel(unsigned long long seed, unsigned long long iteration,
                                    int row_begin, int rows, int T, double *__restrict__ out,
                                    const unsigned long long *__restrict__ seed_iter = nullptr) {
  if (seed_iter) {
    seed = seed_iter[0];
    iteration += seed_iter[1];
  }
  const int P = (T + 1) >> 1;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * P) return;
  const int r = (int)(idx / P), pr = (int)(idx - (long long)r * P);
  curandStatePhilox4_32_10_t st;
  curand_init(seed, (unsigned long long)(row_begin + r), (iteration << 32) + 4ull * (unsigned long long)pr,
              &st);
  const double2 v = curand_normal2_double(&st);
  double *o = out + (size_t)r * T + 2 * pr;
  o[0] = v.x;
  if (2 * pr + 1 < T) o[1] = v.y;
}

// ---- sample-built TVLQR tracking controller (policy.py:121-233) ----------------------
struct PolicyArgs {
  const double *nom_x, *nom_u;      // (H+1, 7), (H)
  const double *cx, *cu;            // perturbed cloud: (K, H+1, 7), (K, H)
  const int64_t *status;            // (K) 0 = survived
  int K, H;
  double dt;
  const double *qr, *qf;            // (7) diagonal running / final weights
  double r;
  double *a_cont, *b_cont;          // (H, 3, 5), (H, 3)
  double *a_disc, *b_disc;          // (H, 7, 7), (H, 7)  (inputs when !do_fit)
  double *gains;                    // (H, 7)
  int32_t *flag;                    // [0]: 1 + step where Riccati diverged, 0 ok
  int do_fit, do_riccati;
};

// regressor state columns theta, phi, v_x, v_z, omega = 2..6 (policy.py:28)
__device__ __forceinline__ int reg_col(int c) { return c + 2; }

__device__ __forceinline__ void cloud_row(const PolicyArgs &p, int i, int k, const double *nk,
                                          const double *nk1, double z[6], double y[3]) {
  const double *s0 = p.cx + ((size_t)i * (p.H + 1) + k) * 7;
  const double *s1 = s0 + 7;
#pragma unroll
  for (int c = 0; c < 5; ++c) z[c] = s0[reg_col(c)] - nk[reg_col(c)];
  z[5] = p.cu[(size_t)i * p.H + k] - p.nom_u[k];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    y[r] = (s1[4 + r] - s0[4 + r]) / p.dt - (nk1[4 + r] - nk[4 + r]) / p.dt;
}

// Phase 1, one warp per step k: least squares of the acceleration rows (v_x, v_z,
// omega derivatives) on the 6 regressors over the surviving rollouts
// (estimate_linear_sequence, policy.py:141-171).  Columns with norm <= 1e-10 x the
// largest are dropped (their Jacobian entries stay 0); the others are scaled to
// unit norm, the normal equations are accumulated with warp reductions in FP64 and
// solved by Cholesky (the scaling keeps the squared condition number small; SURVEY
// 7.3.6).  Euler discretisation with the analytic kinematic rows
// (assemble_discrete, policy.py:121-138).
// The steps are independent: they are spread over the whole GPU (PFIT_WARPS warps
// per CTA, ceil(H / PFIT_WARPS) CTAs) -- one CTA of 16 warps took 5 rounds on one SM.
// Phase 2 (riccati_kernel, one 64-thread CTA, launched after): backward Riccati recursion
// S_N = Q_f, h_k = (b'S A)/(r + b'S b), S <- Q + A'S A - (A'S b) h', symmetrised
// (tvlqr_backward, policy.py:206-233).
constexpr int PFIT_WARPS = 2;
__global__ void __launch_bounds__(32 * PFIT_WARPS) policy_fit_kernel(const PolicyArgs p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  {
    for (int k = blockIdx.x * NW + warp; k < p.H; k += gridDim.x * NW) {
      const double *nk = p.nom_x + (size_t)k * 7, *nk1 = nk + 7;
      double n2[6] = {0, 0, 0, 0, 0, 0};
      for (int i = lane; i < p.K; i += 32) {
        if (p.status[i] != 0) continue;
        double z[6], y[3];
        cloud_row(p, i, k, nk, nk1, z, y);
#pragma unroll
        for (int c = 0; c < 6; ++c) n2[c] += z[c] * z[c];
      }
      double nrm[6], mx = 0.0;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        nrm[c] = sqrt(warp_sum_d(n2[c]));
        mx = fmax(mx, nrm[c]);
      }
      const double thr = 1e-10 * fmax(mx, 1e-30);
      double G[21], Rg[18];
#pragma unroll
      for (int e = 0; e < 21; ++e) G[e] = 0.0;
#pragma unroll
      for (int e = 0; e < 18; ++e) Rg[e] = 0.0;
      for (int i = lane; i < p.K; i += 32) {
        if (p.status[i] != 0) continue;
        double z[6], y[3];
        cloud_row(p, i, k, nk, nk1, z, y);
#pragma unroll
        for (int c = 0; c < 6; ++c) z[c] = nrm[c] > thr ? z[c] / nrm[c] : 0.0;
        int e = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a) {
#pragma unroll
          for (int b = a; b < 6; ++b) G[e++] += z[a] * z[b];
#pragma unroll
          for (int r = 0; r < 3; ++r) Rg[a * 3 + r] += z[a] * y[r];
        }
      }
#pragma unroll
      for (int e = 0; e < 21; ++e) G[e] = warp_sum_d(G[e]);
#pragma unroll
      for (int e = 0; e < 18; ++e) Rg[e] = warp_sum_d(Rg[e]);
      if (lane == 0) {
        // Cholesky of the active block (inactive columns: unit diagonal, zero rhs)
        double L[36], x[18];
        int e = 0;
        for (int a = 0; a < 6; ++a)
          for (int b = a; b < 6; ++b, ++e) {
            const bool act = nrm[a] > thr && nrm[b] > thr;
            L[b * 6 + a] = L[a * 6 + b] = act ? G[e] : (a == b ? 1.0 : 0.0);
          }
        for (int a = 0; a < 6; ++a)
          for (int r = 0; r < 3; ++r) x[a * 3 + r] = nrm[a] > thr ? Rg[a * 3 + r] : 0.0;
        for (int j = 0; j < 6; ++j) {
          double d = L[j * 6 + j];
          for (int m = 0; m < j; ++m) d -= L[j * 6 + m] * L[j * 6 + m];
          const bool dep = !(d > 1e-24);  // collinear excitation: drop the column
          d = dep ? 1.0 : sqrt(d);
          L[j * 6 + j] = d;
          for (int i2 = j + 1; i2 < 6; ++i2) {
            double v = L[i2 * 6 + j];
            for (int m = 0; m < j; ++m) v -= L[i2 * 6 + m] * L[j * 6 + m];
            L[i2 * 6 + j] = dep ? 0.0 : v / d;
          }
          if (dep)
            for (int r = 0; r < 3; ++r) x[j * 3 + r] = 0.0;
        }
        for (int r = 0; r < 3; ++r) {  // forward then backward substitution
          for (int j = 0; j < 6; ++j) {
            double v = x[j * 3 + r];
            for (int m = 0; m < j; ++m) v -= L[j * 6 + m] * x[m * 3 + r];
            x[j * 3 + r] = v / L[j * 6 + j];
          }
          for (int j = 5; j >= 0; --j) {
            double v = x[j * 3 + r];
            for (int m = j + 1; m < 6; ++m) v -= L[m * 6 + j] * x[m * 3 + r];
            x[j * 3 + r] = v / L[j * 6 + j];
          }
        }
        double *ac = p.a_cont + (size_t)k * 15, *bc = p.b_cont + (size_t)k * 3;
        double *ad = p.a_disc + (size_t)k * 49, *bd = p.b_disc + (size_t)k * 7;
        for (int e2 = 0; e2 < 49; ++e2) ad[e2] = (e2 % 8 == 0) ? 1.0 : 0.0;
        for (int e2 = 0; e2 < 7; ++e2) bd[e2] = 0.0;
        ad[0 * 7 + 4] = p.dt;
        ad[1 * 7 + 5] = p.dt;
        ad[2 * 7 + 6] = p.dt;
        bd[3] = p.dt;
        for (int r = 0; r < 3; ++r) {
          for (int c = 0; c < 6; ++c) {
            const double jv = nrm[c] > thr ? x[c * 3 + r] / nrm[c] : 0.0;
            if (c < 5) {
              ac[r * 5 + c] = jv;
              ad[(4 + r) * 7 + reg_col(c)] += p.dt * jv;
            } else {
              bc[r] = jv;
              bd[4 + r] = p.dt * jv;
            }
          }
        }
      }
    }
  }
}

// One thread per entry of the 7x7 recursion (64 threads, 3 barriers per step).  S is
// kept exactly symmetric (the symmetrisation adds the same two numbers either way
// round), so b'S = (S b)' and one product serves both; every dot product runs over its
// index in order, as the one-warp form it replaces did (bitwise the same gains).
__device__ __forceinline__ double dot7(const double *x, int sx, const double *y, int sy) {
  double v = 0.0;
#pragma unroll
  for (int m = 0; m < 7; ++m) v += x[m * sx] * y[m * sy];
  return v;
}

__global__ void __launch_bounds__(64) riccati_kernel(const PolicyArgs p) {
  __shared__ double S[49], SA[49], A[49], Sn[49], bv[7], Sb[7];
  const int tid = threadIdx.x;
  const bool ent = tid < 49;  // thread e < 49 owns entry (i, j) = (e / 7, e % 7)
  const int i = ent ? tid / 7 : 0, j = ent ? tid % 7 : 0;
  if (ent) S[tid] = i == j ? p.qf[i] : 0.0;
  const double qd = (ent && i == j) ? p.qr[i] : 0.0;  // running-cost diagonal entry
  if (tid == 0) p.flag[0] = 0;
  // (A_k, b_k) of the next step are loaded into registers while step k+1 computes:
  // the recursion is serial, so an L2 round trip per step would sit on its path
  double an = 0.0, bn = 0.0;
  if (ent) an = p.a_disc[(size_t)(p.H - 1) * 49 + tid];
  if (tid < 7) bn = p.b_disc[(size_t)(p.H - 1) * 7 + tid];
  for (int k = p.H - 1; k >= 0; --k) {
    if (ent) A[tid] = an;
    if (tid < 7) bv[tid] = bn;
    if (k > 0) {
      if (ent) an = p.a_disc[(size_t)(k - 1) * 49 + tid];
      if (tid < 7) bn = p.b_disc[(size_t)(k - 1) * 7 + tid];
    }
    __syncthreads();  // A_k, b_k and S_{k+1} visible
    if (ent) SA[tid] = dot7(S + 7 * i, 1, A + j, 7);                              // (S A)_ij
    else if (tid < 56) Sb[tid - 49] = dot7(S + 7 * (tid - 49), 1, bv, 1);        // (S b)_i
    __syncthreads();
    if (ent) {
      double denom = p.r;
      for (int m = 0; m < 7; ++m) denom += bv[m] * Sb[m];
      const double gj = dot7(A + j, 7, Sb, 1), gi = dot7(A + i, 7, Sb, 1);  // (A' S b)_j, _i
      const double hj = gj / denom;
      if (i == 0) p.gains[(size_t)k * 7 + j] = hj;
      Sn[tid] = qd + dot7(A + i, 7, SA + j, 7) - gi * hj;
    }
    __syncthreads();
    bool fin = true;
    if (ent) {
      const double v = 0.5 * (Sn[tid] + Sn[7 * j + i]);
      S[tid] = v;
      fin = isfinite(v);
    }
    if (!__syncthreads_and(fin)) {
      if (tid == 0) p.flag[0] = 1 + k;
      return;
    }
  }
}

// Pipe throughput probes, 8 independent chains per thread.
//   MODE 0: FFMA (2 flop / lane / op)   MODE 1: FFMA2 packed f32x2 (4 flop / lane / op)
//   MODE 2: MUFU.RSQ (1 op / lane)
// Velocity induced by n point vortices at m target points, FP64 (vpm.py:93-128):
// kernel 0 regularised  Gamma [dz, -dx] / (2 pi sqrt(r^4 + rc^4)),  kernel 1 singular
// Gamma [dz, -dx] / (2 pi r^2) with a coincident source contributing 0.  One warp
// per target: lane-strided partial sums in source order, then a fixed butterfly,
// so the result does not depend on the launch.  Used by the NMPC pressure sensor.
__global__ void induced_velocity_kernel(const double *__restrict__ pos, const double *__restrict__ gam,
                                        int n, const double *__restrict__ tg, int m, double rc4,
                                        int singular, double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= m) return;
  const double tx = tg[2 * i], tz = tg[2 * i + 1];
  double ux = 0.0, uz = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double dx = tx - pos[2 * j], dz = tz - pos[2 * j + 1];
    const double r2 = dx * dx + dz * dz;
    double c;
    if (singular) c = r2 == 0.0 ? 0.0 : gam[j] / (TWO_PI * r2);
    else c = gam[j] / (TWO_PI * sqrt(r2 * r2 + rc4));
    ux += c * dz;
    uz -= c * dx;
  }
  ux = warp_sum_d(ux);
  uz = warp_sum_d(uz);
  if (lane == 0) {
    out[2 * i] = ux;
    out[2 * i + 1] = uz;
  }
}

// One target, source count from the device (a plan's snapshot): the sensor
// velocity of vpm_plan_step / vpm_plan_probe.  Same per-lane order and butterfly
// as induced_velocity_kernel, so both give the same bits.
__global__ void induced_velocity1_kernel(const double *__restrict__ pos, const double *__restrict__ gam,
                                         const int32_t *__restrict__ n_dev, double tx, double tz,
                                         double rc4, int singular, double *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int n = n_dev[0];
  double ux = 0.0, uz = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double dx = tx - pos[2 * j], dz = tz - pos[2 * j + 1];
    const double r2 = dx * dx + dz * dz;
    double c;
    if (singular) c = r2 == 0.0 ? 0.0 : gam[j] / (TWO_PI * r2);
    else c = gam[j] / (TWO_PI * sqrt(r2 * r2 + rc4));
    ux += c * dz;
    uz -= c * dx;
  }
  ux = warp_sum_d(ux);
  uz = warp_sum_d(uz);
  if (lane == 0) {
    out[0] = ux;
    out[1] = uz;
  }
}

template <int MODE>
__global__ void fp32_probe_kernel(float *out, int iters, float a, float b) {
  float s = 0.f;
  if constexpr (MODE == 3) {
    // the direct Biot-Savart mix: per packed pair of interactions 8 packed FP32 ops
    // and 2 MUFU.RSQ, 4 independent chains (the formulation's pipe ceiling)
    float2 v[4], w[4];
    const float2 A = make_float2(a, a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = make_float2(1.f + threadIdx.x * 1e-3f + i, 2.f + i);
      w[i] = make_float2(b, 0.5f * b);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float2 t = v[i];
#pragma unroll
        for (int f = 0; f < 7; ++f) t = __ffma2_rn(t, A, w[i]);
        t = make_float2(rsqrt_mufu(t.x), rsqrt_mufu(t.y));
        v[i] = __ffma2_rn(t, A, v[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) s += v[i].x + v[i].y;
  } else if constexpr (MODE == 1) {
    float2 v[8];
    const float2 A = make_float2(a, a), Bv = make_float2(b, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = make_float2(threadIdx.x * 1e-3f + i, 0.5f * i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ffma2_rn(v[i], A, Bv);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i].x + v[i].y;
  } else {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 1.0f + threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = MODE == 0 ? fmaf(v[i], a, b) : rsqrt_mufu(v[i]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
  }
  if (s == 1.2345f) out[blockIdx.x] = s;
}

}  // namespace vpm
