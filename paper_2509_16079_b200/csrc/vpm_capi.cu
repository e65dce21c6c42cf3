// vpm_capi.cu -- extern "C" ABI of libvpm_b200.so (declared in include/vpm_b200.h).
//
// Host side of the hot path: parameter unpacking with the reference's frozen ABI
// (config.py:280-300, _core.pyx:65-86), the precomputed inverses of the three
// pose-invariant boundary systems, launch-shape selection, device plans and the
// reference-facing host-buffer entry points that replace _core.pyx's step /
// rollout / batch_rollout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vpm_b200.h"
#include "vpm_rollout.cuh"

using vpm::Args;
using vpm::Phys;

namespace {

thread_local std::string g_err;

int fail_cfg(const std::string &m) {
  g_err = m;
  return VPM_ERR_CONFIG;
}

int fail_cuda(cudaError_t e, const char *what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return VPM_ERR_CUDA;
}

#define CK(call)                                 \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return fail_cuda(e_, #call); \
  } while (0)

// frozen fparams order (config.py:283-285)
enum {
  FP_R_CORE, FP_K_DISS, FP_SHED_OFF, FP_CRIT_AOA, FP_RHO, FP_DT, FP_M, FP_I, FP_G, FP_L,
  FP_L_W, FP_L_E, FP_L_CHORD, FP_S_E, FP_PHI_LIM, FP_U_LIM, FP_LEV_GAIN, FP_ETA, FP_COUNT
};

constexpr int CAP_MAX = 4088;  // 12-bit particle index inside the merge keys

int unpack(const int64_t *ip, const double *fp, Phys *P) {
  if (!ip || !fp) return fail_cfg("iparams/fparams must not be null");
  if (ip[0] < 1 || ip[0] > vpm::NB_MAX)
    return fail_cfg("n_bound > " + std::to_string(vpm::NB_MAX) + " (or < 1) not supported");
  if (ip[1] < 4 || ip[1] > CAP_MAX)
    return fail_cfg("particle_cap > " + std::to_string(CAP_MAX) + " (or < 4) not supported");
  for (int i = 0; i < FP_COUNT; ++i)
    if (!std::isfinite(fp[i])) return fail_cfg("non-finite fparams entry " + std::to_string(i));
  P->nb = (int)ip[0];
  P->cap = (int)ip[1];
  P->r_core = fp[FP_R_CORE];
  P->k_diss = fp[FP_K_DISS];
  P->shed_off = fp[FP_SHED_OFF];
  P->crit_aoa = fp[FP_CRIT_AOA];
  P->rho = fp[FP_RHO];
  P->dt = fp[FP_DT];
  P->m = fp[FP_M];
  P->inertia = fp[FP_I];
  P->g = fp[FP_G];
  P->l = fp[FP_L];
  P->l_w = fp[FP_L_W];
  P->l_e = fp[FP_L_E];
  P->l_chord = fp[FP_L_CHORD];
  P->s_e = fp[FP_S_E];
  P->phi_lim = fp[FP_PHI_LIM];
  P->u_lim = fp[FP_U_LIM];
  P->lev_gain = fp[FP_LEV_GAIN];
  P->eta = fp[FP_ETA];
  const double r = P->r_core;
  P->rc4f = (float)(r * r * r * r);
  P->inv_dt = 1.0 / P->dt;
  P->inv_m = 1.0 / P->m;
  P->inv_inertia = 1.0 / P->inertia;
  P->s_pan = P->l_chord / P->nb;
  P->inv_s = 1.0 / P->s_pan;
  P->cos_crit = P->crit_aoa >= vpm::PI ? -2.0 : std::cos(P->crit_aoa);
  return VPM_OK;
}

// Gauss-Jordan inverse with partial pivoting (row-major); false when singular.
bool invert(std::vector<double> &a, int n, std::vector<double> &inv) {
  inv.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) inv[(size_t)i * n + i] = 1.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int r = k + 1; r < n; ++r)
      if (std::fabs(a[(size_t)r * n + k]) > std::fabs(a[(size_t)p * n + k])) p = r;
    if (a[(size_t)p * n + k] == 0.0) return false;
    if (p != k)
      for (int c = 0; c < n; ++c) {
        std::swap(a[(size_t)k * n + c], a[(size_t)p * n + c]);
        std::swap(inv[(size_t)k * n + c], inv[(size_t)p * n + c]);
      }
    const double d = a[(size_t)k * n + k];
    for (int c = 0; c < n; ++c) { a[(size_t)k * n + c] /= d; inv[(size_t)k * n + c] /= d; }
    for (int r = 0; r < n; ++r) {
      if (r == k) continue;
      const double f = a[(size_t)r * n + k];
      if (f == 0.0) continue;
      for (int c = 0; c < n; ++c) {
        a[(size_t)r * n + c] -= f * a[(size_t)k * n + c];
        inv[(size_t)r * n + c] -= f * inv[(size_t)k * n + c];
      }
    }
  }
  return true;
}

// The boundary system of _core.pyx:258-313 (vpm.py:331-391) assembled in the
// chord frame.  Every influence coefficient couples two points on the chord
// line, so A depends only on (shedding, reversed) and the config, not on the
// pose (SURVEY.md finding 0.5; verified there to 4.6e-12 over 400 poses).
// Variant 0: attached nb x nb; 1: shedding forward; 2: shedding reversed.
int build_inverses(const Phys &P, std::vector<double> &out) {
  const int nb = P.nb, S = nb + 2;
  out.assign((size_t)3 * S * S, 0.0);
  const double s = P.l_chord / nb;
  std::vector<double> col(nb + 1), pan(nb);
  for (int i = 0; i <= nb; ++i) col[i] = -s * i;
  for (int j = 0; j < nb; ++j) pan[j] = col[j] - 0.5 * s;
  const double lev = col[0] + P.shed_off, tev = col[nb] - P.shed_off;
  for (int var = 0; var < 3; ++var) {
    const bool shed = var > 0, rev = var == 2;
    const int ns = shed ? nb + 2 : nb, r0 = shed ? 1 : 0;
    std::vector<double> A((size_t)ns * ns, 0.0), inv;
    for (int i = 0; i < nb; ++i) {
      const int ri = (shed && rev) ? i : i + 1;
      for (int j = 0; j < ns; ++j) {
        const double src = j < nb ? pan[j] : (j == nb ? lev : tev);
        const double dx = col[ri] - src;  // normal (0,1): (dz nx - dx nz)/(2 pi r^2)
        A[(size_t)(r0 + i) * ns + j] = -dx / (vpm::TWO_PI * dx * dx);
      }
    }
    if (shed) {
      const int ecol = rev ? nb + 1 : nb, epan = rev ? nb - 1 : 0;
      A[ecol] = 1.0;
      A[epan] = P.lev_gain;
      for (int j = 0; j < ns; ++j) A[(size_t)(nb + 1) * ns + j] = 1.0;
    }
    if (!invert(A, ns, inv)) return fail_cfg("boundary system is singular for this configuration");
    std::memcpy(&out[(size_t)var * S * S], inv.data(), sizeof(double) * ns * ns);
  }
  return VPM_OK;
}

struct Shape {
  int nt, r, w0, minb;  // threads, slots per sweeping warp, control-warp slots, reg variant
  int sym = 0;          // symmetric-pair sweep (nt = 32 x tiles of 128 particles)
};

int device_sms() {
  static thread_local int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// Launch shape.  A rollout CTA has NT threads; each holds R register target slots.
// Caps above 256 use the symmetric-pair sweep with NT = 32 x ceil(cap / 128) (fixed
// by the cap, below).  Direct sweep (caps <= 256, and VPM_SYM=0): slot k of warp w =
// particles 32 (NW k + NW-1-w) .. +31, NT x R >= cap + 4 (the largest wake a
// snapshot may hold), so every particle is a register target; NT is the smallest
// power of two >= 64 (>= the split-sweep chain count when the launch is
// latency-bound) that still puts >= 24 warps on every SM given how many rollouts each
// SM receives.  Results do not depend on the direct shape (canonical reduction
// orders, see vpm_rollout.cuh).  VPM_SHAPE="nt,r" (direct) / VPM_MAXREG override for
// tuning.
Shape pick_shape(int cap, int nb, int rows) {
  const int need = cap + 4;
  const double per_sm = rows > 0 ? (double)rows / device_sms() : 1.0;
  if (const char *e = getenv("VPM_SHAPE")) {
    Shape s{0, 0, 0, 64};
    if (sscanf(e, "%d,%d", &s.nt, &s.r) == 2 && s.nt >= 64 && s.nt <= vpm::NT_MAX &&
        s.nt % 32 == 0 && s.r >= 1 && s.r <= 8 && s.nt * s.r >= need) {
      if (const char *m = getenv("VPM_MAXREG")) s.minb = atoi(m);
      return s;
    }
  }
  // Symmetric-pair sweep for caps above 256: T = ceil(cap / 128) warps of 128-particle
  // tiles (vpm_rollout.cuh, sym_sweep).  The shape is a function of the cap alone, so
  // every launch (single step, batch, any shard) of a given cap sums in the same
  // order.  R >= 4 slots per thread (the tile) and >= cap + 4 targets for the direct
  // fallback of overfull wakes.  VPM_SYM=0 selects the direct sweep, and an explicit
  // VPM_SHAPE (above) a direct-sweep shape (tuning / A-B).
  const char *se = getenv("VPM_SYM");
  if (cap > 256 && cap <= 2048 && !(se && atoi(se) == 0)) {
    const int T = (cap + 127) / 128;
    Shape s{32 * T, std::max(4, (need + 32 * T - 1) / (32 * T)), 0, 64, 1};
    if (per_sm > 8.0) {
      const int n_sm = (int)ceil(per_sm);
      const size_t smem = vpm::make_layout(cap, nb, s.nt, true).total + 1024;
      // register variants that leave fewer than 24 resident warps per SM are
      // excluded (N = 2048, 512 threads: one CTA per SM at 72 registers)
      auto slots = [&](int regs) {
        int c = 65536 / (s.nt * regs);
        c = std::min(c, 2048 / s.nt);
        c = std::min(c, 32);
        c = std::min(c, (int)((228 * 1024) / smem));
        return (c < 1 || (regs > 64 && c * s.nt < 768)) ? 1 << 30 : ((n_sm + c - 1) / c) * c;
      };
      // fewest slots; ties to the smaller register budget (more resident warps:
      // C5 N = 512, 112 slots either way, 64 registers 1% faster than 72)
      int bs = slots(64);
      for (int regs : {72, 80}) {
        const int sl = slots(regs);
        if (sl < bs) {
          bs = sl;
          s.minb = regs;
        }
      }
    }
    if (const char *m = getenv("VPM_MAXREG")) s.minb = atoi(m);
    return s;
  }
  Shape best{512, 8, 0, 64};
  if (per_sm <= 8.0) {
    // latency-bound launch (one round): the per-rollout critical path matters, so
    // about two 32-particle blocks per warp (the largest NT with need >= 2 NT) and
    // at least one thread per (target, segment) chain of the split sweeps (nb x
    // NSEG, capped at 256).  Measured: C2 (cap 60) 64 -> 128 threads 0.40 -> 0.34
    // ms; cap 512 at 513 / 1025 rows 256 x 3 beats 128 x 5 by 10% / 8%; cap 256 at
    // 1025 rows 128 x 3 beats 256 x 2 by 20%.
    int nt = 64;
    while (nt < 512 && need >= 4 * nt) nt *= 2;
    int nt0 = 64;
    while (nt0 < 256 && nt0 < nb * vpm::NSEG) nt0 *= 2;
    if (nt < nt0) nt = nt0;
    best = Shape{nt, (need + nt - 1) / nt, 0, 64};
  } else {
    // throughput-bound: the tightest tile that still keeps >= 24 warps per SM
    for (int nt = 64; nt <= 512; nt *= 2) {
      const int r = (need + nt - 1) / nt;
      if (r > 8) continue;
      best = Shape{nt, r, 0, 64};
      if (nt >= need) break;  // more lanes than particles
      const double ctas = per_sm < 1024.0 / nt ? per_sm : 1024.0 / nt;
      if (ctas * nt >= 768.0) break;
    }
  }
  // Wave quantisation: with c CTAs resident per SM (register-limited) a
  // throughput-bound launch costs ~ceil(n/c) * c rollout-slots per SM, whatever c
  // is.  Among the 64 / 72 / 80-register variants take the fewest slots, ties to
  // the larger register budget (the direct sweep interleaves more chains; measured
  // in round 1 with the direct sweep at caps 512 / 1024, which now take the
  // symmetric sweep and its own rule above: 72 registers 3.5% / 1.5% faster at equal
  // or fewer slots; 64-thread CTAs, end of round 2: C5 N = 128 / 256 at 72 registers
  // 2% / 1.3% faster than 64 at equal slots).  Variants that leave fewer than 3 CTAs
  // per SM are excluded.  Latency-bound launches (one round) keep 64.
  const int n_sm = (int)ceil(per_sm);
  if (per_sm > 8.0) {
    const size_t smem = vpm::make_layout(cap, nb, best.nt).total + 1024;
    auto slots = [&](int regs, int min_c) {
      int c = 65536 / (best.nt * regs);
      c = std::min(c, 2048 / best.nt);
      c = std::min(c, 32);
      c = std::min(c, (int)((228 * 1024) / smem));
      return c < min_c ? 1 << 30 : ((n_sm + c - 1) / c) * c;
    };
    int bs = slots(64, 1);
    for (int regs : {72, 80}) {
      const int sl = slots(regs, 3);
      if (sl <= bs) {
        bs = sl;
        best.minb = regs;
      }
    }
  }
  if (const char *m = getenv("VPM_MAXREG")) best.minb = atoi(m);
  return best;
}

template <int R, int MINB>
cudaError_t launch_t(const Args &a, int grid, int nt, size_t smem, cudaStream_t st) {
  auto k = vpm::rollout_kernel<R, MINB>;
  static thread_local size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  k<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

template <int MINB>
cudaError_t launch_r(const Args &a, int grid, const Shape &sh, size_t smem, cudaStream_t st) {
  switch (sh.r) {
    case 1: return launch_t<1, MINB>(a, grid, sh.nt, smem, st);
    case 2: return launch_t<2, MINB>(a, grid, sh.nt, smem, st);
    case 3: return launch_t<3, MINB>(a, grid, sh.nt, smem, st);
    case 4: return launch_t<4, MINB>(a, grid, sh.nt, smem, st);
    case 5: return launch_t<5, MINB>(a, grid, sh.nt, smem, st);
    case 6: return launch_t<6, MINB>(a, grid, sh.nt, smem, st);
    case 7: return launch_t<7, MINB>(a, grid, sh.nt, smem, st);
    default: return launch_t<8, MINB>(a, grid, sh.nt, smem, st);
  }
}

cudaError_t launch_rollouts(Args a, int grid, cudaStream_t st) {
  const Shape sh = pick_shape(a.P.cap, a.P.nb, grid);
  a.sym = sh.sym;
  const size_t smem = vpm::make_layout(a.P.cap, a.P.nb, sh.nt, sh.sym != 0).total;
#ifdef VPM_TUNING_SUBSET
  // tuning builds (tools/): only the shapes the C4 / 8-GPU-shard / C2 / C3 / C5 N=128 launches pick
  if (sh.r == 5 && sh.minb == 72) return launch_t<5, 72>(a, grid, sh.nt, smem, st);
  if (sh.r == 5 && sh.minb == 64) return launch_t<5, 64>(a, grid, sh.nt, smem, st);
  if (sh.r == 3 && sh.minb == 64) return launch_t<3, 64>(a, grid, sh.nt, smem, st);
  if (sh.r == 3 && sh.minb == 72) return launch_t<3, 72>(a, grid, sh.nt, smem, st);
  if (sh.r == 1 && sh.minb == 64) return launch_t<1, 64>(a, grid, sh.nt, smem, st);
  return cudaErrorNotSupported;
#else
  switch (sh.minb) {
    case 48: return launch_r<48>(a, grid, sh, smem, st);
    case 56: return launch_r<56>(a, grid, sh, smem, st);
    case 72: return launch_r<72>(a, grid, sh, smem, st);
    case 80: return launch_r<80>(a, grid, sh, smem, st);
    default: return launch_r<64>(a, grid, sh, smem, st);
  }
#endif
}

int check_fluid(const vpm_fluid *f, const Phys &P) {
  if (!f) return fail_cfg("fluid must not be null");
  if (f->n_wake < 0 || f->n_wake > P.cap + 4) return fail_cfg("n_wake outside [0, cap+4]");
  if (f->n_prev != 0 && f->n_prev != P.nb) return fail_cfg("n_prev must be 0 or n_bound");
  if (f->ring_a >= f->n_wake || f->ring_b >= f->n_wake) return fail_cfg("ring index beyond n_wake");
  for (int i = 0; i < f->n_wake; ++i)
    if (f->wake_age[i] < 0 || f->wake_age[i] > (1 << 19) - 4096)
      return fail_cfg("wake_age outside [0, 2^19 - 4096)");
  return VPM_OK;
}

}  // namespace

// ============================ device plan ========================================
struct vpm_plan {
  int device = 0;
  Phys P{};
  int max_rows = 0, H = 0;
  double *d_ainv = nullptr;
  // snapshot
  double *d_wpos = nullptr, *d_wgam = nullptr, *d_ppos = nullptr, *d_pgam = nullptr, *d_ema = nullptr;
  int64_t *d_wage = nullptr;
  int32_t *d_scal = nullptr;  // device {n_wake, ring_a, ring_b, n_prev}: kernels read these
  double *d_plev = nullptr;
  int n_wake = 0, ring_a = -1, ring_b = -1, n_prev = 0;
  double prev_lev = 0.0;
  double *d_snap = nullptr;  // the snapshot arrays above, one block
  double *h_snap = nullptr;  // pinned host mirror of d_snap (set_fluid staging)
  size_t snap_doubles = 0;
  double *d_wbuf = nullptr;  // chunk partials of the MPPI softmax reduction
  size_t wbuf_len = 0;
  unsigned *d_ticket = nullptr;  // last-CTA ticket of the chunked reduction (re-armed by it)
  void *d_rec = nullptr;  // single-step record (vpm_plan_step)
  // rollout-kernel timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // start/stop pairs
  size_t ev_used = 0;
  std::mutex mu;
  // host-buffer optimise path: own stream and grow-only scratch
  std::mutex host_mu;
  cudaStream_t hstream = nullptr;
  void *hscratch = nullptr;
  size_t hscratch_len = 0;
  void *hpin = nullptr;  // pinned host staging of the small inputs / outputs
  size_t hpin_len = 0;
};

static Args base_args(const vpm_plan *p) {
  Args a;
  std::memset(&a, 0, sizeof(a));
  a.P = p->P;
  a.ainv = p->d_ainv;
  a.wpos = p->d_wpos;
  a.wgam = p->d_wgam;
  a.wage = p->d_wage;
  a.n_wake = p->n_wake;
  a.ring_a = p->ring_a;
  a.ring_b = p->ring_b;
  a.ppos = p->d_ppos;
  a.pgam = p->d_pgam;
  a.n_prev = p->n_prev;
  a.prev_lev = p->prev_lev;
  a.ema = p->d_ema;
  a.snap_scal = p->d_scal;
  a.snap_plev = p->d_plev;
  a.integrate = 1;
  a.check_envelope = 1;
  return a;
}

static int plan_launch(vpm_plan *p, const Args &a, int grid, cudaStream_t st) {
  if (grid <= 0) return VPM_OK;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->timing) {
    if (p->ev_used + 2 > p->ev.size()) {
      for (int i = 0; i < 2; ++i) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        p->ev.push_back(e);
      }
    }
    e0 = p->ev[p->ev_used];
    e1 = p->ev[p->ev_used + 1];
    p->ev_used += 2;
    CK(cudaEventRecord(e0, st));
  }
  cudaError_t e = launch_rollouts(a, grid, st);
  if (e != cudaSuccess) return fail_cuda(e, "rollout_kernel launch");
  if (p->timing) CK(cudaEventRecord(e1, st));
  return VPM_OK;
}

extern "C" {

const char *vpm_last_error(void) { return g_err.c_str(); }

int vpm_launch_shape(int cap, int nb, int rows, int *threads, int *targets, int *smem_bytes) {
  const Shape s = pick_shape(cap, nb, rows);
  if (threads) *threads = s.nt;
  if (targets) *targets = s.r;
  if (smem_bytes) *smem_bytes = vpm::make_layout(cap, nb, s.nt, s.sym != 0).total;
  return VPM_OK;
}

vpm_plan *vpm_plan_create(const int64_t *iparams, const double *fparams, int max_rows, int H,
                          int device) {
  Phys P;
  if (unpack(iparams, fparams, &P) != VPM_OK) return nullptr;
  std::vector<double> inv;
  if (build_inverses(P, inv) != VPM_OK) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    g_err = "cudaSetDevice failed";
    return nullptr;
  }
  vpm_plan *p = new vpm_plan();
  p->device = device;
  p->P = P;
  p->max_rows = max_rows;
  p->H = H;
  const int cap4 = P.cap + 4;
  // The snapshot lives in ONE device block with a pinned host mirror, so
  // vpm_plan_set_fluid uploads it with a single copy:
  //   wpos 2 cap4 | wgam cap4 | wage cap4 (int64) | ppos 2 nb | pgam nb | ema nb |
  //   plev 1 | scal 4 int32 (2 doubles)
  p->snap_doubles = (size_t)4 * cap4 + 4 * P.nb + 3;
  bool ok = cudaMalloc(&p->d_ainv, inv.size() * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&p->d_snap, sizeof(double) * p->snap_doubles) == cudaSuccess &&
            cudaHostAlloc(&p->h_snap, sizeof(double) * p->snap_doubles, cudaHostAllocDefault) == cudaSuccess;
  if (ok) {
    double *b = p->d_snap;
    p->d_wpos = b;
    p->d_wgam = b + 2 * cap4;
    p->d_wage = reinterpret_cast<int64_t *>(b + 3 * cap4);
    p->d_ppos = b + 4 * cap4;
    p->d_pgam = p->d_ppos + 2 * P.nb;
    p->d_ema = p->d_pgam + P.nb;
    p->d_plev = p->d_ema + P.nb;
    p->d_scal = reinterpret_cast<int32_t *>(p->d_plev + 1);
    std::memset(p->h_snap, 0, sizeof(double) * p->snap_doubles);
  }
  if (ok) {
    const int32_t empty[4] = {0, -1, -1, 0};
    ok = cudaMemcpy(p->d_scal, empty, sizeof(empty), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemset(p->d_plev, 0, sizeof(double)) == cudaSuccess;
  }
  if (ok) ok = cudaMemcpy(p->d_ainv, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) ok = cudaMemset(p->d_ema, 0, sizeof(double) * P.nb) == cudaSuccess;
  if (!ok) {
    g_err = "device allocation failed";
    vpm_plan_destroy(p);
    return nullptr;
  }
  return p;
}

void vpm_plan_destroy(vpm_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaFree(p->d_ainv);
  cudaFree(p->d_snap);
  if (p->h_snap) cudaFreeHost(p->h_snap);
  cudaFree(p->d_wbuf);
  cudaFree(p->d_ticket);
  cudaFree(p->d_rec);
  cudaFree(p->hscratch);
  if (p->hpin) cudaFreeHost(p->hpin);
  if (p->hstream) cudaStreamDestroy(p->hstream);
  for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
  delete p;
}

// Upload a snapshot.  st == nullptr: synchronous, after every launch of every stream
// (the public entry point).  st != nullptr: queued on st behind the launches already
// there -- for a plan used on that one stream only (the thread-local host plans).
static int set_fluid_on(vpm_plan *p, const vpm_fluid *f, cudaStream_t st) {
  if (!p) return fail_cfg("null plan");
  int rc = check_fluid(f, p->P);
  if (rc) return rc;
  CK(cudaSetDevice(p->device));
  // synchronous / staging: no launch of any stream may still read the old snapshot
  // (nor, when staging, the pinned mirror the graph's upload copies from)
  if (!st || st == reinterpret_cast<cudaStream_t>(uintptr_t(-1))) CK(cudaDeviceSynchronize());
  // pack the used parts into the pinned mirror at their device offsets, one copy up
  const int cap4 = p->P.cap + 4, nb = p->P.nb;
  double *h = p->h_snap;
  if (f->n_wake > 0) {
    std::memcpy(h, f->wake_pos, sizeof(double) * 2 * f->n_wake);
    std::memcpy(h + 2 * cap4, f->wake_gamma, sizeof(double) * f->n_wake);
    std::memcpy(h + 3 * cap4, f->wake_age, sizeof(int64_t) * f->n_wake);
  }
  if (f->n_prev > 0) {
    std::memcpy(h + 4 * cap4, f->prev_pos, sizeof(double) * 2 * f->n_prev);
    std::memcpy(h + 4 * cap4 + 2 * nb, f->prev_gamma, sizeof(double) * f->n_prev);
  }
  std::memcpy(h + 4 * cap4 + 3 * nb, f->ema, sizeof(double) * nb);
  h[4 * cap4 + 4 * nb] = f->prev_lev;
  const int32_t scal[4] = {f->n_wake, f->ring_a, f->ring_b, f->n_prev};
  std::memcpy(h + 4 * cap4 + 4 * nb + 1, scal, sizeof(scal));
  if (st == reinterpret_cast<cudaStream_t>(uintptr_t(-1))) {
    // stage only: the caller uploads (vpm_plan_upload_fluid)
  } else if (st) {
    CK(cudaMemcpyAsync(p->d_snap, h, sizeof(double) * p->snap_doubles, cudaMemcpyHostToDevice, st));
  } else {
    CK(cudaMemcpy(p->d_snap, h, sizeof(double) * p->snap_doubles, cudaMemcpyHostToDevice));
  }
  p->n_wake = f->n_wake;
  p->ring_a = f->ring_a;
  p->ring_b = f->ring_b;
  p->n_prev = f->n_prev;
  p->prev_lev = f->prev_lev;
  return VPM_OK;
}

int vpm_plan_set_fluid(vpm_plan *p, const vpm_fluid *f) { return set_fluid_on(p, f, nullptr); }

// Pack a snapshot into the plan's pinned mirror only (no copy) / copy the mirror up
// on a stream: the two halves of set_fluid, so a CUDA graph can contain the upload.
int vpm_plan_stage_fluid(vpm_plan *p, const vpm_fluid *f) {
  return set_fluid_on(p, f, reinterpret_cast<cudaStream_t>(uintptr_t(-1)));
}

int vpm_plan_upload_fluid(vpm_plan *p, void *stream) {
  if (!p) return fail_cfg("null plan");
  CK(cudaSetDevice(p->device));
  CK(cudaMemcpyAsync(p->d_snap, p->h_snap, sizeof(double) * p->snap_doubles, cudaMemcpyHostToDevice,
                     (cudaStream_t)stream));
  return VPM_OK;
}

int vpm_plan_batch(vpm_plan *p, const double *d_x0, int x0_stride, const double *d_controls,
                   const double *d_ustar, const double *d_noise, double sigma, int row_begin,
                   int row_end, int T, const double *d_q, const double *d_xperch, int record,
                   const vpm_batch_out *o, void *stream) {
  if (!p) return fail_cfg("null plan");
  if (T < 0 || row_end < row_begin) return fail_cfg("bad row range / horizon");
  if (!d_controls && (!d_ustar || (!d_noise && row_end > 1))) return fail_cfg("controls or u*/noise required");
  Args a = base_args(p);
  a.x0 = d_x0;
  a.x0_stride = x0_stride;
  a.controls = d_controls;
  a.ustar = d_ustar;
  a.noise = d_noise;
  a.sigma = sigma;
  a.T = T;
  a.row_begin = row_begin;
  a.rows = row_end - row_begin;
  a.record = record;
  if (o) {
    a.status = o->status;
    a.finals = o->finals;
    a.trajs = o->trajs;
    a.cost = (d_q && d_xperch) ? o->cost : nullptr;
    a.shed_mask = o->shed_mask;
    a.shed_mask_hi = o->shed_mask_hi;
    a.wake_hash = o->wake_hash;
    a.n_final = o->n_final;
    a.inter = o->interactions;
  }
  a.q = d_q;
  a.xp = d_xperch;
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  return plan_launch(p, a, a.rows, (cudaStream_t)stream);
}

static int project_launch(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                          const double *d_states, const double *d_inputs, int pol_h, double t_start,
                          double t0, const double *d_times, int64_t *d_status, double *d_final,
                          int write_snapshot, void *stream);

int vpm_plan_project(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                     const double *d_states, const double *d_inputs, int pol_h, double t_start,
                     double t0, int64_t *d_status, double *d_final, int write_snapshot,
                     void *stream) {
  return project_launch(p, d_x0, T, d_gains, d_states, d_inputs, pol_h, t_start, t0, nullptr, d_status,
                        d_final, write_snapshot, stream);
}

int vpm_plan_project_dev(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                         const double *d_states, const double *d_inputs, int pol_h, const double *d_times,
                         int64_t *d_status, double *d_final, int write_snapshot, void *stream) {
  if (!d_times) return fail_cfg("times pointer must not be null");
  return project_launch(p, d_x0, T, d_gains, d_states, d_inputs, pol_h, 0.0, 0.0, d_times, d_status, d_final,
                        write_snapshot, stream);
}

static int project_launch(vpm_plan *p, const double *d_x0, int T, const double *d_gains,
                          const double *d_states, const double *d_inputs, int pol_h, double t_start,
                          double t0, const double *d_times, int64_t *d_status, double *d_final,
                          int write_snapshot, void *stream) {
  if (!p) return fail_cfg("null plan");
  if (T < 0 || pol_h < 1) return fail_cfg("bad projection horizon / policy length");
  Args a = base_args(p);
  a.x0 = d_x0;
  a.T = T;
  a.rows = 1;
  a.check_envelope = 0;  // Engine.step semantics (no envelope test, rollout.py:81-86)
  a.pol_gains = d_gains;
  a.pol_states = d_states;
  a.pol_inputs = d_inputs;
  a.pol_h = pol_h;
  a.pol_t_start = t_start;
  a.pol_t0 = t0;
  a.pol_times = d_times;
  a.status = d_status;
  a.finals = d_final;
  if (write_snapshot) {
    // a single CTA reads the snapshot in its prologue and overwrites it in its
    // epilogue: the projected fluid becomes the plan's snapshot on the device
    a.need_fluid = 1;
    a.o_wpos = p->d_wpos;
    a.o_wgam = p->d_wgam;
    a.o_wage = p->d_wage;
    a.o_scal = p->d_scal;
    a.o_ppos = p->d_ppos;
    a.o_pgam = p->d_pgam;
    a.o_plev = p->d_plev;
    a.o_ema = p->d_ema;
  }
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  return plan_launch(p, a, 1, (cudaStream_t)stream);
}

// Device record of the single-step path: one D2H copy per call (vpm_b200.h).
struct StepRecord {
  double x[7], fw[3], q[2];
  int32_t rc, scal[4], pad[3];
};
static_assert(sizeof(StepRecord) == VPM_STEP_RECORD_BYTES, "record layout");

int vpm_plan_step(vpm_plan *p, const double *x, double u, int integrate, const double *sensor,
                  double r_core, void *h_record, void *stream) {
  if (!p || !x) return fail_cfg("null plan / state");
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  if (!p->d_rec) CK(cudaMalloc(&p->d_rec, sizeof(StepRecord)));
  StepRecord *r = (StepRecord *)p->d_rec;
  // a page-locked record buffer is written by the kernels themselves (unified
  // addressing: the pinned host page is device-accessible), saving the queued copy
  // and its stream slot; pageable buffers go through the device record and a copy
  // (queried on every call: a cached answer could outlive the caller's buffer)
  bool direct = false;
  if (h_record) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h_record) == cudaSuccess && at.type == cudaMemoryTypeHost &&
        at.devicePointer) {
      r = (StepRecord *)at.devicePointer;
      direct = true;
    }
    cudaGetLastError();  // a pageable pointer is not an error here
  }
  Args a = base_args(p);
  a.use_x0v = 1;
  std::memcpy(a.x0v, x, sizeof(a.x0v));
  a.T = 1;
  a.rows = 1;
  a.integrate = integrate;
  a.check_envelope = 0;  // Engine.step semantics: rc only (rollout.py:81-86, _core.pyx:536-576)
  a.use_u_const = 1;
  a.u_const = u;
  a.finals = r->x;
  a.rc_out = &r->rc;
  a.fw_out = r->fw;
  a.need_fluid = 1;      // the stepped fluid replaces the plan's snapshot in place
  a.o_wpos = p->d_wpos;
  a.o_wgam = p->d_wgam;
  a.o_wage = p->d_wage;
  a.o_scal = p->d_scal;
  a.o_ppos = p->d_ppos;
  a.o_pgam = p->d_pgam;
  a.o_plev = p->d_plev;
  a.o_ema = p->d_ema;
  a.o_scal2 = r->scal;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = plan_launch(p, a, 1, st);
  if (rc) return rc;
  if (sensor) {
    const double rc2 = r_core * r_core;
    vpm::induced_velocity1_kernel<<<1, 32, 0, st>>>(p->d_wpos, p->d_wgam, p->d_scal, sensor[0], sensor[1],
                                                    rc2 * rc2, 0, r->q);
    CK(cudaGetLastError());
  }
  if (h_record && !direct) CK(cudaMemcpyAsync(h_record, r, sizeof(StepRecord), cudaMemcpyDeviceToHost, st));
  return VPM_OK;
}

int vpm_plan_probe(vpm_plan *p, const double *target, double r_core, double *out) {
  if (!p || !target || !out) return fail_cfg("null plan / target / output");
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  CK(cudaDeviceSynchronize());  // the snapshot may still be written by a queued step
  if (!p->d_rec) CK(cudaMalloc(&p->d_rec, sizeof(StepRecord)));
  StepRecord *r = (StepRecord *)p->d_rec;
  const double rc2 = r_core * r_core;
  vpm::induced_velocity1_kernel<<<1, 32>>>(p->d_wpos, p->d_wgam, p->d_scal, target[0], target[1], rc2 * rc2, 0,
                                           r->q);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, r->q, 2 * sizeof(double), cudaMemcpyDeviceToHost));
  return VPM_OK;
}

int vpm_stream_sync(void *stream) {
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return VPM_OK;
}

int vpm_plan_cloud(vpm_plan *p, const double *d_x0, const double *d_x0_noise,
                   const double *d_x0_scale, const double *d_ustar, const double *d_u_noise,
                   double sigma_u, int rows, int T, int64_t *d_status, double *d_trajs,
                   void *stream) {
  if (!p) return fail_cfg("null plan");
  Args a = base_args(p);
  a.x0 = d_x0;
  a.x0_noise = d_x0_noise;
  a.x0_scale = d_x0_scale;
  a.ustar = d_ustar;
  a.noise = d_u_noise;
  a.sigma = sigma_u;
  a.T = T;
  a.row_begin = 1;  // MPPI sampling with every row perturbed: row r uses noise row r
  a.rows = rows;
  a.record = 1;
  a.status = d_status;
  a.trajs = d_trajs;
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  return plan_launch(p, a, rows, (cudaStream_t)stream);
}

int vpm_plan_download_fluid(vpm_plan *p, vpm_fluid_out *out) {
  if (!p || !out) return fail_cfg("null plan / output");
  CK(cudaSetDevice(p->device));
  CK(cudaDeviceSynchronize());
  const int cap4 = p->P.cap + 4, nb = p->P.nb;
  CK(cudaMemcpy(out->scalars, p->d_scal, sizeof(int32_t) * 4, cudaMemcpyDeviceToHost));
  const int n = out->scalars[0];
  std::memset(out->wake_pos, 0, sizeof(double) * 2 * cap4);
  std::memset(out->wake_gamma, 0, sizeof(double) * cap4);
  std::memset(out->wake_age, 0, sizeof(int64_t) * cap4);
  if (n > 0) {
    CK(cudaMemcpy(out->wake_pos, p->d_wpos, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out->wake_gamma, p->d_wgam, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(out->wake_age, p->d_wage, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  }
  CK(cudaMemcpy(out->prev_pos, p->d_ppos, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out->prev_gamma, p->d_pgam, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out->prev_lev, p->d_plev, sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out->ema, p->d_ema, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  return VPM_OK;
}

// One launch of the shard's softmax partial (vpm_rollout.cuh, mppi_partial_chunked_kernel);
// ustar_out / flag: apply the single-device update in the same launch.
static int partial_launch(vpm_plan *p, const double *d_cost, int rows, int row_begin, const double *d_ustar,
                          const double *d_noise, double sigma, int T, double temperature, double *d_partial,
                          double *d_ustar_out, int32_t *d_flag, void *stream) {
  if (!p) return fail_cfg("null plan");
  if (temperature <= 0.0) return fail_cfg("temperature must be > 0");
  if (rows < 0 || T < 0) return fail_cfg("bad partial shape");
  std::lock_guard<std::mutex> lk(p->mu);
  CK(cudaSetDevice(p->device));
  const int G = std::max(1, (rows + vpm::PCH_ROWS - 1) / vpm::PCH_ROWS);
  const size_t need = (size_t)G * (T + 2);
  if (p->wbuf_len < need) {
    cudaFree(p->d_wbuf);
    p->d_wbuf = nullptr;
    CK(cudaMalloc(&p->d_wbuf, sizeof(double) * need));
    p->wbuf_len = need;
  }
  if (!p->d_ticket) {
    CK(cudaMalloc(&p->d_ticket, sizeof(unsigned)));
    CK(cudaMemset(p->d_ticket, 0, sizeof(unsigned)));
  }
  // shared memory: [NW][T+1] sums | 2 NW reductions | T+1 totals
  const size_t smem = sizeof(double) * ((size_t)vpm::PCH_WARPS * (T + 1) + 2 * vpm::PCH_WARPS + (T + 1));
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(vpm::mppi_partial_chunked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
  vpm::mppi_partial_chunked_kernel<<<G, 32 * vpm::PCH_WARPS, smem, (cudaStream_t)stream>>>(
      d_cost, rows, row_begin, d_ustar, d_noise, sigma, p->P.u_lim, T, temperature, p->d_wbuf, p->d_ticket,
      d_partial, d_ustar_out, d_flag);
  CK(cudaGetLastError());
  return VPM_OK;
}

int vpm_mppi_partial(vpm_plan *p, const double *d_cost, int rows, int row_begin,
                     const double *d_ustar, const double *d_noise, double sigma, int T,
                     double temperature, double *d_partial, void *stream) {
  return partial_launch(p, d_cost, rows, row_begin, d_ustar, d_noise, sigma, T, temperature, d_partial, nullptr,
                        nullptr, stream);
}

int vpm_mppi_combine(const double *d_partials, int W, int T, double temperature, double *d_ustar,
                     int32_t *d_flag, void *stream) {
  if (W < 1 || T < 0) return fail_cfg("bad combine shape");
  vpm::mppi_combine_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(d_partials, W, T, temperature, d_ustar, d_flag);
  CK(cudaGetLastError());
  return VPM_OK;
}

static int philox_launch(uint64_t seed, uint64_t iteration, const uint64_t *d_seed_iter, int row_begin,
                         int rows, int T, double *d_out, void *stream) {
  if (row_begin < 0 || rows < 0 || T < 0) return fail_cfg("bad noise shape");
  if (rows == 0 || T == 0) return VPM_OK;
  if (!d_out) return fail_cfg("noise output must not be null");
  const long long n = (long long)rows * ((T + 1) / 2);
  const int bs = 256;
  vpm::noise_philox_kernel<<<(unsigned)((n + bs - 1) / bs), bs, 0, (cudaStream_t)stream>>>(
      (unsigned long long)seed, (unsigned long long)iteration, row_begin, rows, T, d_out,
      (const unsigned long long *)d_seed_iter);
  CK(cudaGetLastError());
  return VPM_OK;
}

int vpm_noise_philox(uint64_t seed, uint64_t iteration, int row_begin, int rows, int T, double *d_out,
                     void *stream) {
  return philox_launch(seed, iteration, nullptr, row_begin, rows, T, d_out, stream);
}

int vpm_noise_philox_dev(const uint64_t *d_seed_iter, uint64_t offset, int row_begin, int rows, int T,
                         double *d_out, void *stream) {
  if (!d_seed_iter) return fail_cfg("seed/iteration pointer must not be null");
  return philox_launch(0, offset, d_seed_iter, row_begin, rows, T, d_out, stream);
}

int vpm_mppi_iteration(vpm_plan *p, const double *d_x0, double *d_ustar, const double *d_noise,
                       double sigma, int B_total, int T, double temperature, const double *d_q,
                       const double *d_xperch, double *d_cost, double *d_partial, int32_t *d_flag,
                       int use_graph, void *stream) {
  (void)use_graph;  // reserved (vpm_b200.h); stream capture is the caller's choice
  vpm_batch_out o;
  std::memset(&o, 0, sizeof(o));
  o.cost = d_cost;
  int rc = vpm_plan_batch(p, d_x0, 0, nullptr, d_ustar, d_noise, sigma, 0, B_total, T, d_q, d_xperch, 0, &o, stream);
  if (rc) return rc;
  // partial + the W = 1 combine in one launch (bitwise vpm_mppi_partial + vpm_mppi_combine)
  return partial_launch(p, d_cost, B_total, 0, d_ustar, d_noise, sigma, T, temperature, d_partial, d_ustar, d_flag,
                        stream);
}

int vpm_mppi_optimize_host(vpm_plan *p, const double *x0, double *u_star, const double *noise,
                           int iters, int K, int T, double sigma, double temperature,
                           const double *q, const double *x_perch) {
  if (!p) return fail_cfg("null plan");
  if (iters < 0 || K < 0 || T < 0) return fail_cfg("negative iterations / batch / horizon");
  CK(cudaSetDevice(p->device));
  std::lock_guard<std::mutex> hl(p->host_mu);
  if (!p->hstream) CK(cudaStreamCreateWithFlags(&p->hstream, cudaStreamNonBlocking));
  cudaStream_t st = p->hstream;
  const int B = K + 1;
  const size_t nn = (size_t)iters * K * T;
  // persistent, grow-only device scratch (no per-call allocation)
  const size_t need = 256 * 8 + sizeof(double) * (7 + (size_t)(T + 1) + nn + 14 + (size_t)B + (T + 2)) +
                      sizeof(int32_t) * (iters + 1);
  if (p->hscratch_len < need) {
    cudaFree(p->hscratch);
    p->hscratch = nullptr;
    p->hscratch_len = 0;
    CK(cudaMalloc(&p->hscratch, need));
    p->hscratch_len = need;
  }
  char *base = (char *)p->hscratch;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    void *r = base + off;
    off += bytes;
    return r;
  };
  // the small inputs x0 | u* | q | x_perch as one block (one staged copy)
  const size_t nsmall = 7 + (size_t)T + 7 + 7;
  double *d_small = (double *)take(nsmall * sizeof(double));
  double *d_x0 = d_small, *d_u = d_small + 7, *d_q = d_u + T, *d_xp = d_q + 7;
  double *d_noise = (double *)take((nn + 1) * sizeof(double));
  double *d_cost = (double *)take(B * sizeof(double));
  double *d_part = (double *)take((T + 2) * sizeof(double));
  int32_t *d_flag = (int32_t *)take((iters + 1) * sizeof(int32_t));
  // pinned staging [small inputs | u* out | flags out]: from pageable sources every
  // small copy would be a synchronous staged transfer
  const size_t pin_need = sizeof(double) * (nsmall + T) + sizeof(int32_t) * (iters + 1);
  if (p->hpin_len < pin_need) {
    if (p->hpin) cudaFreeHost(p->hpin);
    p->hpin = nullptr;
    p->hpin_len = 0;
    CK(cudaMallocHost(&p->hpin, pin_need));
    p->hpin_len = pin_need;
  }
  double *h_small = (double *)p->hpin, *h_u = h_small + nsmall;
  int32_t *h_flags = (int32_t *)(h_u + T);
  std::memcpy(h_small, x0, 7 * sizeof(double));
  std::memcpy(h_small + 7, u_star, T * sizeof(double));
  std::memcpy(h_small + 7 + T, q, 7 * sizeof(double));
  std::memcpy(h_small + 14 + T, x_perch, 7 * sizeof(double));
  CK(cudaMemcpyAsync(d_small, h_small, nsmall * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_noise, noise, nn * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_flag, 0, iters * sizeof(int32_t) + 4, st));
  int rc = VPM_OK;
  for (int it = 0; it < iters && rc == VPM_OK; ++it)
    rc = vpm_mppi_iteration(p, d_x0, d_u, d_noise + (size_t)it * K * T, sigma, B, T, temperature, d_q,
                            d_xp, d_cost, d_part, d_flag + it, 0, st);
  if (rc == VPM_OK) {
    CK(cudaMemcpyAsync(h_u, d_u, T * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (iters > 0) CK(cudaMemcpyAsync(h_flags, d_flag, iters * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  if (rc) return rc;
  std::memcpy(u_star, h_u, T * sizeof(double));
  for (int it = 0; it < iters; ++it)
    if (h_flags[it]) {
      g_err = "all sampled rollouts failed (infinite cost)";
      return VPM_ERR_ALLFAIL;
    }
  return VPM_OK;
}

int vpm_plan_timing(vpm_plan *p, int reset, double *avg_ms, int64_t *launches) {
  if (!p) return fail_cfg("null plan");
  CK(cudaSetDevice(p->device));
  double tot = 0.0;
  int64_t n = 0;
  for (size_t i = 0; i + 1 < p->ev_used; i += 2) {
    CK(cudaEventSynchronize(p->ev[i + 1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->ev[i], p->ev[i + 1]));
    tot += ms;
    ++n;
  }
  if (avg_ms) *avg_ms = n ? tot / n : 0.0;
  if (launches) *launches = n;
  if (reset) {
    p->ev_used = 0;
    p->timing = reset > 0;  // reset=1: start timing; reset=-1: stop timing
  }
  return VPM_OK;
}

double vpm_fp32_peak_probe(int iters, int mode) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8, threads = 256;
  float *d = nullptr;
  if (cudaMalloc(&d, blocks * sizeof(float)) != cudaSuccess) return -1.0;
  auto run = [&](int it) {
    if (mode == 3) vpm::fp32_probe_kernel<3><<<blocks, threads>>>(d, it, 0.9999f, 1e-4f);
    else if (mode == 1) vpm::fp32_probe_kernel<1><<<blocks, threads>>>(d, it, 0.9999f, 1e-4f);
    else if (mode == 2) vpm::fp32_probe_kernel<2><<<blocks, threads>>>(d, it, 0.9999f, 1e-4f);
    else vpm::fp32_probe_kernel<0><<<blocks, threads>>>(d, it, 0.9999f, 1e-4f);
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  run(iters / 4);  // warm-up
  cudaEventRecord(a);
  run(iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  // GFLOP/s for FFMA (2/lane-op) and FFMA2 (4/lane-op); G ops/s for MUFU; mode 3:
  // algorithmic Biot-Savart GFLOP/s of the mix (4 chains x 2 interactions per
  // thread-iteration, 12 flop each)
  const double per = mode == 1 ? 4.0 : (mode == 2 ? 1.0 : (mode == 3 ? 12.0 : 2.0));
  const double work = per * 8.0 * (double)iters * blocks * threads;
  return ms > 0.f ? work / (ms * 1e-3) / 1e9 : -1.0;
}

int vpm_boundary_inverse(const int64_t *iparams, const double *fparams, double *out) {
  Phys P;
  int rc = unpack(iparams, fparams, &P);
  if (rc) return rc;
  std::vector<double> inv;
  rc = build_inverses(P, inv);
  if (rc) return rc;
  std::memcpy(out, inv.data(), inv.size() * sizeof(double));
  return VPM_OK;
}

int vpm_threads(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * 8;
}

}  // extern "C"

// ======================= reference-facing host-buffer layer ==========================
namespace {

// One cached plan per (thread, parameter set); host calls from several Python
// threads (threaded NMPC, nmpc.py:219-222) get independent plans and streams.
struct HostCtx {
  std::vector<int64_t> ip;
  std::vector<double> fp;
  vpm_plan *plan = nullptr;
  cudaStream_t st = nullptr;
  void *scratch = nullptr;
  size_t scratch_len = 0;
  char *pin = nullptr;  // pinned staging of the packed small outputs (one D2H per call)
  size_t pin_len = 0;
};
thread_local HostCtx g_host;

char *host_pinned(size_t bytes) {
  HostCtx &h = g_host;
  if (h.pin_len < bytes) {
    if (h.pin) cudaFreeHost(h.pin);
    h.pin = nullptr;
    if (cudaMallocHost(&h.pin, bytes) != cudaSuccess) {
      h.pin_len = 0;
      return nullptr;
    }
    h.pin_len = bytes;
  }
  return h.pin;
}

int host_plan(const int64_t *ip, const double *fp, vpm_plan **out, cudaStream_t *st) {
  HostCtx &h = g_host;
  const bool same = h.plan && std::memcmp(h.ip.data(), ip, 2 * sizeof(int64_t)) == 0 &&
                    std::memcmp(h.fp.data(), fp, FP_COUNT * sizeof(double)) == 0;
  if (!same) {
    if (h.plan) vpm_plan_destroy(h.plan);
    int dev = 0;
    cudaGetDevice(&dev);
    h.plan = vpm_plan_create(ip, fp, 0, 0, dev);
    if (!h.plan) return VPM_ERR_CONFIG;
    h.ip.assign(ip, ip + 2);
    h.fp.assign(fp, fp + FP_COUNT);
  }
  if (!h.st) CK(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
  *out = h.plan;
  *st = h.st;
  return VPM_OK;
}

void *host_scratch(size_t bytes) {
  HostCtx &h = g_host;
  if (h.scratch_len < bytes) {
    cudaFree(h.scratch);
    h.scratch = nullptr;
    if (cudaMalloc(&h.scratch, bytes) != cudaSuccess) {
      h.scratch_len = 0;
      return nullptr;
    }
    h.scratch_len = bytes;
  }
  return h.scratch;
}

struct Carve {
  char *base;
  size_t off = 0;
  template <class T>
  T *take(size_t n) {
    off = (off + 255) & ~(size_t)255;
    T *p = reinterpret_cast<T *>(base + off);
    off += n * sizeof(T);
    return p;
  }
};

// Shared driver for step / rollout / batch_rollout with host buffers.  Everything is
// queued on the thread's own stream (the snapshot upload too: the thread-local plan
// is used on that stream only), the small outputs -- status, rc, finals, loads and
// the returned fluid -- are carved contiguously (one rollout: in the pinned staging,
// written by the kernel in place; batches: on the device, ONE copy back through the
// pinned staging); the stream is synchronised once.
int host_run(const double *x0, int x0_stride, const double *controls, int B, int T,
             const vpm_fluid *fluid, const int64_t *ip, const double *fp, int integrate,
             int check_env, int record, int64_t *status, double *finals, double *trajs,
             int32_t *rc_out, double *fw_out, vpm_fluid_out *fo) {
  Phys P;
  int rc = unpack(ip, fp, &P);
  if (rc) return rc;
  if (B < 0 || T < 0) return fail_cfg("negative batch or horizon");
  vpm_plan *p;
  cudaStream_t st;
  rc = host_plan(ip, fp, &p, &st);
  if (rc) return rc;
  rc = set_fluid_on(p, fluid, st);
  if (rc) return rc;
  if (B == 0) {
    CK(cudaStreamSynchronize(st));
    return VPM_OK;
  }
  const int cap4 = P.cap + 4, nb = P.nb;
  const size_t ntraj = record ? (size_t)B * (T + 1) * 7 : 0;
  const size_t need = 256 * 20 + sizeof(double) * ((size_t)B * 7 + (size_t)B * T + (size_t)B * 7 + ntraj + 3 * (size_t)B +
                                                   3 * cap4 + 4 * nb + 1) +
                      sizeof(int64_t) * ((size_t)B + cap4) + sizeof(int32_t) * ((size_t)B + 4);
  void *sc = host_scratch(need);
  if (!sc) return fail_cfg("device scratch allocation failed");
  // One rollout (Engine.step / fluid_step / rollout): the small outputs live in the
  // pinned staging itself -- the kernel writes them there through its device alias
  // (no copy back) -- and so do the inputs (read in place for a single step, else
  // one pinned upload).  Batches: outputs packed on the device, ONE copy back.
  char *pin = nullptr, *pin_dev = nullptr;
  if (B == 1) {
    pin = host_pinned(need);
    void *alias = nullptr;
    if (pin && cudaHostGetDevicePointer(&alias, pin, 0) == cudaSuccess) {
      pin_dev = (char *)alias;
    } else {
      cudaGetLastError();
      pin = nullptr;
    }
  }
  const bool direct = pin_dev != nullptr;
  Carve cv{direct ? pin_dev : (char *)sc};
  Carve cd{(char *)sc};  // device-only buffers
  // packed small outputs first, then the trajectories, then the inputs
  int64_t *d_st = cv.take<int64_t>(B);
  int32_t *d_rc = cv.take<int32_t>(B);
  double *d_fin = cv.take<double>((size_t)B * 7);
  double *d_fw = cv.take<double>((size_t)B * 3);
  Args a = base_args(p);
  if (fo) {
    a.need_fluid = 1;
    a.o_wpos = cv.take<double>(2 * (size_t)cap4);
    a.o_wgam = cv.take<double>(cap4);
    a.o_wage = cv.take<int64_t>(cap4);
    a.o_scal = cv.take<int32_t>(4);
    a.o_ppos = cv.take<double>(2 * (size_t)nb);
    a.o_pgam = cv.take<double>(nb);
    a.o_plev = cv.take<double>(1);
    a.o_ema = cv.take<double>(nb);
  }
  const size_t small_bytes = cv.off;
  if (!direct) cd.off = small_bytes;
  double *d_traj = record ? cd.take<double>(ntraj) : nullptr;
  const size_t nx0 = (size_t)(x0_stride ? B : 1) * 7, nctl = (size_t)B * (T > 0 ? T : 1);
  double *d_x0, *d_ctrl;
  if (direct && T <= 1) {  // a single step reads its state and control in place
    d_x0 = cv.take<double>(nx0 + nctl);
    d_ctrl = d_x0 + nx0;
    std::memcpy(pin + ((char *)d_x0 - pin_dev), x0, sizeof(double) * nx0);
    if (T > 0) std::memcpy(pin + ((char *)d_ctrl - pin_dev), controls, sizeof(double) * nctl);
  } else {
    d_x0 = cd.take<double>(nx0 + nctl);
    d_ctrl = d_x0 + nx0;
    if (direct) {  // one pinned upload of [x0 | controls]
      double *h_in = cv.take<double>(nx0 + nctl);
      double *hp = (double *)(pin + ((char *)h_in - pin_dev));
      std::memcpy(hp, x0, sizeof(double) * nx0);
      if (T > 0) std::memcpy(hp + nx0, controls, sizeof(double) * nctl);
      CK(cudaMemcpyAsync(d_x0, hp, sizeof(double) * (nx0 + (T > 0 ? nctl : 0)), cudaMemcpyHostToDevice, st));
    } else {
      CK(cudaMemcpyAsync(d_x0, x0, sizeof(double) * nx0, cudaMemcpyHostToDevice, st));
      if (T > 0) CK(cudaMemcpyAsync(d_ctrl, controls, sizeof(double) * nctl, cudaMemcpyHostToDevice, st));
    }
  }
  if (!direct) {
    pin = host_pinned(small_bytes);
    if (!pin) return fail_cfg("pinned staging allocation failed");
  }
  a.x0 = d_x0;
  a.x0_stride = x0_stride;
  a.controls = d_ctrl;
  a.T = T;
  a.rows = B;
  a.integrate = integrate;
  a.check_envelope = check_env;
  a.record = record;
  a.status = d_st;
  a.finals = d_fin;
  a.trajs = d_traj;
  a.rc_out = d_rc;
  a.fw_out = d_fw;
  if (record) CK(cudaMemsetAsync(d_traj, 0, sizeof(double) * ntraj, st));
  rc = plan_launch(p, a, B, st);
  if (rc) return rc;
  if (!direct) CK(cudaMemcpyAsync(pin, sc, small_bytes, cudaMemcpyDeviceToHost, st));
  if (trajs && record) CK(cudaMemcpyAsync(trajs, d_traj, sizeof(double) * ntraj, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const char *obase = direct ? pin_dev : (const char *)sc;
  auto from = [&](const void *d) { return pin + ((const char *)d - obase); };
  if (status) std::memcpy(status, from(d_st), sizeof(int64_t) * B);
  if (rc_out) std::memcpy(rc_out, from(d_rc), sizeof(int32_t) * B);
  if (finals) std::memcpy(finals, from(d_fin), sizeof(double) * B * 7);
  if (fw_out) std::memcpy(fw_out, from(d_fw), sizeof(double) * 3);
  if (fo) {
    std::memcpy(fo->wake_pos, from(a.o_wpos), sizeof(double) * 2 * cap4);
    std::memcpy(fo->wake_gamma, from(a.o_wgam), sizeof(double) * cap4);
    std::memcpy(fo->wake_age, from(a.o_wage), sizeof(int64_t) * cap4);
    std::memcpy(fo->scalars, from(a.o_scal), sizeof(int32_t) * 4);
    std::memcpy(fo->prev_pos, from(a.o_ppos), sizeof(double) * 2 * nb);
    std::memcpy(fo->prev_gamma, from(a.o_pgam), sizeof(double) * nb);
    std::memcpy(fo->prev_lev, from(a.o_plev), sizeof(double));
    std::memcpy(fo->ema, from(a.o_ema), sizeof(double) * nb);
  }
  return VPM_OK;
}

}  // namespace

extern "C" {

int vpm_step(double *x, double u, const vpm_fluid *fluid, const int64_t *iparams,
             const double *fparams, int integrate, double *fw, double *mw, vpm_fluid_out *out) {
  int64_t status = 0;
  int32_t rc = 0;
  double fwm[3] = {0.0, 0.0, 0.0};
  double xn[7];
  int e = host_run(x, 0, &u, 1, 1, fluid, iparams, fparams, integrate, 0, 0, &status, xn, nullptr,
                   &rc, fwm, out);
  if (e) return e;
  std::memcpy(x, xn, sizeof(xn));
  if (fw) { fw[0] = fwm[0]; fw[1] = fwm[1]; }
  if (mw) *mw = fwm[2];
  return status == 0 ? 0 : (rc ? rc : 1);
}

int64_t vpm_rollout(double *x, const double *controls, int T, const vpm_fluid *fluid,
                    const int64_t *iparams, const double *fparams, double *traj,
                    vpm_fluid_out *out) {
  int64_t status = 0;
  double xn[7];
  int e = host_run(x, 0, controls, 1, T, fluid, iparams, fparams, 1, 1, traj != nullptr, &status, xn,
                   traj, nullptr, nullptr, out);
  if (e) return e;
  std::memcpy(x, xn, sizeof(xn));
  return status;
}

int vpm_batch_rollout(const double *x0, const double *controls, int B, int T,
                      const vpm_fluid *fluid, const int64_t *iparams, const double *fparams,
                      int record, int workers, int64_t *status, double *finals, double *trajs) {
  (void)workers;
  return host_run(x0, 0, controls, B, T, fluid, iparams, fparams, 1, 1, record, status, finals,
                  trajs, nullptr, nullptr, nullptr);
}

// Batched rollouts with one start state per row (policy synthesis cloud,
// policy.py:66-91) plus the discrete-decision diagnostics used by the parity
// harness.  x0 is (B, 7).
int vpm_batch_rollout_x0(const double *x0, const double *controls, int B, int T,
                         const vpm_fluid *fluid, const int64_t *iparams, const double *fparams,
                         int record, int64_t *status, double *finals, double *trajs) {
  return host_run(x0, 7, controls, B, T, fluid, iparams, fparams, 1, 1, record, status, finals,
                  trajs, nullptr, nullptr, nullptr);
}

// ---- sample-built tracking controller ---------------------------------------------
int vpm_policy_fit(const double *d_nom_x, const double *d_nom_u, const double *d_cloud_x,
                   const double *d_cloud_u, const int64_t *d_status, int K, int H, double dt,
                   const double *d_q_running, double r_running, const double *d_q_final,
                   double *d_a_cont, double *d_b_cont, double *d_a_disc, double *d_b_disc,
                   double *d_gains, int32_t *d_flag, int do_fit, int do_riccati, void *stream) {
  if (H < 0 || K < 0 || dt <= 0.0) return fail_cfg("bad policy shape");
  if (H == 0) return VPM_OK;
  vpm::PolicyArgs a;
  a.nom_x = d_nom_x;
  a.nom_u = d_nom_u;
  a.cx = d_cloud_x;
  a.cu = d_cloud_u;
  a.status = d_status;
  a.K = K;
  a.H = H;
  a.dt = dt;
  a.qr = d_q_running;
  a.qf = d_q_final;
  a.r = r_running;
  a.a_cont = d_a_cont;
  a.b_cont = d_b_cont;
  a.a_disc = d_a_disc;
  a.b_disc = d_b_disc;
  a.gains = d_gains;
  a.flag = d_flag;
  a.do_fit = do_fit;
  a.do_riccati = do_riccati;
  if (do_fit) {
    const int grid = (H + vpm::PFIT_WARPS - 1) / vpm::PFIT_WARPS;
    vpm::policy_fit_kernel<<<grid, 32 * vpm::PFIT_WARPS, 0, (cudaStream_t)stream>>>(a);
    CK(cudaGetLastError());
  }
  if (do_riccati) {
    vpm::riccati_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(a);
    CK(cudaGetLastError());
  }
  return VPM_OK;
}

namespace {
// Host-buffer driver of the controller: optional perturbed rollouts on a plan, then
// the fit / Riccati kernel.  Outputs are copied back when their pointers are set.
int policy_host(vpm_plan *p, const double *nom_x, const double *nom_u, int H, const double *x0s,
                const double *u_cloud, const double *cloud_x_in, const int64_t *status_in, int K,
                double dt, const double *q_running, double r_running, const double *q_final,
                const double *a_disc_in, const double *b_disc_in, double *a_cont, double *b_cont,
                double *a_disc, double *b_disc, double *gains, int64_t *status_out,
                double *cloud_x_out, int do_fit, int do_riccati) {
  if (H < 0 || K < 0) return fail_cfg("negative horizon or sample count");
  if (do_fit && x0s && !p) return fail_cfg("a plan is required for the perturbed rollouts");
  if (H == 0) return VPM_OK;
  int dev = 0;
  if (p) {
    CK(cudaSetDevice(p->device));
    dev = p->device;
  } else {
    CK(cudaGetDevice(&dev));
  }
  // per-thread stream and grow-only scratch: no per-call allocation / stream churn
  static thread_local cudaStream_t st = nullptr;
  static thread_local void *buf = nullptr;
  static thread_local size_t buf_len = 0;
  static thread_local int buf_dev = -1;
  if (!st || buf_dev != dev) {
    if (st) cudaStreamDestroy(st);
    cudaFree(buf);
    buf = nullptr;
    buf_len = 0;
    st = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    buf_dev = dev;
  }
  const size_t nx = (size_t)K * (H + 1) * 7;
  const size_t need = 16 * 256 + sizeof(double) * ((H + 1) * 7 + H + nx + (size_t)K * H + (size_t)K * 7 +
                                                  14 + H * (15 + 3 + 49 + 7 + 7)) +
                      sizeof(int64_t) * K + 64;
  if (buf_len < need) {
    CK(cudaStreamSynchronize(st));
    cudaFree(buf);
    buf = nullptr;
    buf_len = 0;
    CK(cudaMalloc(&buf, need));
    buf_len = need;
  }
  Carve cv{(char *)buf};
  double *d_nx = cv.take<double>((size_t)(H + 1) * 7), *d_nu = cv.take<double>(H + 1);
  double *d_cx = cv.take<double>(nx + 1), *d_cu = cv.take<double>((size_t)K * H + 1);
  double *d_x0 = cv.take<double>((size_t)K * 7 + 1), *d_q = cv.take<double>(7), *d_qf = cv.take<double>(7);
  double *d_ac = cv.take<double>((size_t)H * 15 + 1), *d_bc = cv.take<double>((size_t)H * 3 + 1);
  double *d_ad = cv.take<double>((size_t)H * 49 + 1), *d_bd = cv.take<double>((size_t)H * 7 + 1);
  double *d_g = cv.take<double>((size_t)H * 7 + 1);
  int64_t *d_st = cv.take<int64_t>(K + 1);
  int32_t *d_flag = cv.take<int32_t>(4);
  int rc = VPM_OK;
  if (do_fit) {
    CK(cudaMemcpyAsync(d_nx, nom_x, sizeof(double) * (H + 1) * 7, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_nu, nom_u, sizeof(double) * H, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemcpyAsync(d_q, q_running, sizeof(double) * 7, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_qf, q_final, sizeof(double) * 7, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(d_flag, 0, 16, st));
  if (do_fit) {
    CK(cudaMemcpyAsync(d_cu, u_cloud, sizeof(double) * K * H, cudaMemcpyHostToDevice, st));
    if (x0s) {  // perturbed rollouts on the device (policy.py:66-91), one launch
      CK(cudaMemcpyAsync(d_x0, x0s, sizeof(double) * K * 7, cudaMemcpyHostToDevice, st));
      CK(cudaMemsetAsync(d_cx, 0, sizeof(double) * nx, st));
      vpm_batch_out o;
      std::memset(&o, 0, sizeof(o));
      o.status = d_st;
      o.trajs = d_cx;
      rc = vpm_plan_batch(p, d_x0, 7, d_cu, nullptr, nullptr, 0.0, 0, K, H, nullptr, nullptr, 1, &o, st);
    } else {
      CK(cudaMemcpyAsync(d_cx, cloud_x_in, sizeof(double) * nx, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(d_st, status_in, sizeof(int64_t) * K, cudaMemcpyHostToDevice, st));
    }
  } else {
    CK(cudaMemcpyAsync(d_ad, a_disc_in, sizeof(double) * H * 49, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_bd, b_disc_in, sizeof(double) * H * 7, cudaMemcpyHostToDevice, st));
  }
  int64_t survivors = K;
  if (rc == VPM_OK && do_fit && x0s) {
    std::vector<int64_t> sv(K > 0 ? K : 1);
    CK(cudaMemcpyAsync(sv.data(), d_st, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    survivors = 0;
    for (int i = 0; i < K; ++i) survivors += sv[i] == 0;
    if (status_out) std::memcpy(status_out, sv.data(), sizeof(int64_t) * K);
    if (survivors < 6) {
      g_err = "only " + std::to_string(survivors) + " of " + std::to_string(K) +
              " perturbed rollouts survived";
      rc = VPM_ERR_RANK;
    }
  }
  if (rc == VPM_OK && (do_fit || do_riccati))
    rc = vpm_policy_fit(d_nx, d_nu, d_cx, d_cu, d_st, K, H, dt, d_q, r_running, d_qf, d_ac, d_bc,
                        d_ad, d_bd, d_g, d_flag, do_fit, do_riccati, st);
  int32_t flag[4] = {0, 0, 0, 0};
  if (rc == VPM_OK) {
    if (a_cont && do_fit) CK(cudaMemcpyAsync(a_cont, d_ac, sizeof(double) * H * 15, cudaMemcpyDeviceToHost, st));
    if (b_cont && do_fit) CK(cudaMemcpyAsync(b_cont, d_bc, sizeof(double) * H * 3, cudaMemcpyDeviceToHost, st));
    if (a_disc && do_fit) CK(cudaMemcpyAsync(a_disc, d_ad, sizeof(double) * H * 49, cudaMemcpyDeviceToHost, st));
    if (b_disc && do_fit) CK(cudaMemcpyAsync(b_disc, d_bd, sizeof(double) * H * 7, cudaMemcpyDeviceToHost, st));
    if (gains && do_riccati) CK(cudaMemcpyAsync(gains, d_g, sizeof(double) * H * 7, cudaMemcpyDeviceToHost, st));
    if (cloud_x_out && do_fit) CK(cudaMemcpyAsync(cloud_x_out, d_cx, sizeof(double) * nx, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(flag, d_flag, sizeof(flag), cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  if (rc) return rc;
  if (do_riccati && flag[0]) {
    g_err = "Riccati recursion diverged at step " + std::to_string(flag[0] - 1);
    return VPM_ERR_DIVERGED;
  }
  return VPM_OK;
}
}  // namespace

int vpm_build_policy_host(vpm_plan *p, const double *nom_x, const double *nom_u, int H,
                          const double *x0s, const double *u_cloud, int K, double dt,
                          const double *q_running, double r_running, const double *q_final,
                          double *a_cont, double *b_cont, double *a_disc, double *b_disc,
                          double *gains, int64_t *status_out, double *cloud_x_out) {
  return policy_host(p, nom_x, nom_u, H, x0s, u_cloud, nullptr, nullptr, K, dt, q_running, r_running,
                     q_final, nullptr, nullptr, a_cont, b_cont, a_disc, b_disc, gains, status_out,
                     cloud_x_out, 1, 1);
}

int vpm_policy_fit_host(const double *nom_x, const double *nom_u, int H, const double *cloud_x,
                        const double *cloud_u, const int64_t *status, int K, double dt,
                        double *a_cont, double *b_cont, double *a_disc, double *b_disc) {
  const double zero7[7] = {0, 0, 0, 0, 0, 0, 0};
  return policy_host(nullptr, nom_x, nom_u, H, nullptr, cloud_u, cloud_x, status, K, dt, zero7, 1.0,
                     zero7, nullptr, nullptr, a_cont, b_cont, a_disc, b_disc, nullptr, nullptr,
                     nullptr, 1, 0);
}

int vpm_tvlqr_host(const double *a_disc, const double *b_disc, int H, const double *q_running,
                   double r_running, const double *q_final, double *gains) {
  const double zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return policy_host(nullptr, zero, zero, H, nullptr, nullptr, nullptr, nullptr, 0, 1.0, q_running,
                     r_running, q_final, a_disc, b_disc, nullptr, nullptr, nullptr, nullptr, gains,
                     nullptr, nullptr, 0, 1);
}

int vpm_induced_velocity_host(const double *pos, const double *gamma, int n, const double *targets,
                              int m, double r_core, int kernel, double *out) {
  if (n < 0 || m < 0) return fail_cfg("negative point count");
  if (kernel != 0 && kernel != 1) return fail_cfg("kernel must be 0 (regularised) or 1 (singular)");
  if (m == 0) return VPM_OK;
  HostCtx &h = g_host;
  if (!h.st) CK(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
  void *sc = host_scratch(256 * 4 + sizeof(double) * (3 * (size_t)n + 4 * (size_t)m + 4));
  if (!sc) return fail_cfg("device scratch allocation failed");
  Carve cv{(char *)sc};
  double *d_pos = cv.take<double>(2 * (size_t)n + 1), *d_gam = cv.take<double>((size_t)n + 1);
  double *d_tg = cv.take<double>(2 * (size_t)m), *d_out = cv.take<double>(2 * (size_t)m);
  if (n > 0) {
    CK(cudaMemcpyAsync(d_pos, pos, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, h.st));
    CK(cudaMemcpyAsync(d_gam, gamma, sizeof(double) * n, cudaMemcpyHostToDevice, h.st));
  }
  CK(cudaMemcpyAsync(d_tg, targets, sizeof(double) * 2 * m, cudaMemcpyHostToDevice, h.st));
  const double rc2 = r_core * r_core;
  vpm::induced_velocity_kernel<<<(m + 3) / 4, 128, 0, h.st>>>(d_pos, d_gam, n, d_tg, m, rc2 * rc2, kernel,
                                                              d_out);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost, h.st));
  CK(cudaStreamSynchronize(h.st));
  return VPM_OK;
}

}  // extern "C"

extern "C" int vpm_debug_phase_cycles(unsigned long long *out, int reset) {
#ifdef VPM_PHASE_TIMING
  if (out && cudaMemcpyFromSymbol(out, vpm::g_phase, sizeof(vpm::g_phase)) != cudaSuccess) return VPM_ERR_CUDA;
  if (reset) {
    static const unsigned long long zero[2][12] = {};
    if (cudaMemcpyToSymbol(vpm::g_phase, zero, sizeof(zero)) != cudaSuccess) return VPM_ERR_CUDA;
  }
  return 24;
#else
  (void)out;
  (void)reset;
  return VPM_ERR_CONFIG;
#endif
}
