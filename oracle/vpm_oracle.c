/*
 * TEST INFRASTRUCTURE ONLY -- never linked into, loaded by, or called from the
 * product path (paper_2509_16079_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and only
 * as the checker.
 *
 * FP64 CPU restatement of the perchsim coupled glider + vortex-wake step, the
 * open-loop rollout and the batched rollout (the hot path the CUDA kernel in
 * paper_2509_16079_b200/csrc/ replaces).  Each phase cites the reference line
 * range it restates (paths relative to /root/reference/pkg/src/perchsim/):
 *
 *   _accel/_core.pyx:175-462  step_core        (vpm.py:635-669 + glider.py:104-122)
 *   _accel/_core.pyx:465-491  run_rollout      (_accel/reference.py:85-111)
 *   _accel/_core.pyx:664-741  batch_rollout    (_accel/reference.py:114-145)
 *
 * Beyond the reference outputs it records, per rollout, the discrete-decision
 * diagnostics the parity harness needs: the bitmask of
 * steps that shed, the final wake size, and the smallest margin seen at the
 * stall / reversed-flow gates and at the ring-termination test, so that
 * FP32-vs-FP64 near-ties can be told apart from real bugs.
 *
 * Parity pin: tests/test_oracle.py checks this file against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXNB 64
#define OR_TWO_PI 6.283185307179586476925286766559
#define OR_PI 3.14159265358979323846264338327950288
#define OR_BLOWUP_OMEGA 300.0 /* _core.pyx:35 */
#define OR_BLOWUP_SPEED 80.0  /* _core.pyx:36 */

/* frozen fparams order, config.py:283-285 */
enum {
  P_R_CORE, P_K_DISS, P_SHED_OFF, P_CRIT_AOA, P_RHO, P_DT, P_M, P_I, P_G, P_L,
  P_L_W, P_L_E, P_L_CHORD, P_S_E, P_PHI_LIM, P_U_LIM, P_LEV_GAIN, P_ETA, P_COUNT
};

typedef struct {
  int nb, cap;
  double fp[P_COUNT];
  double rc4;
} Cfg;

typedef struct {
  double *x, *z, *g, *age; /* wake SoA, capacity cap+6 */
  int n, ring_a, ring_b;
  double px[OR_MAXNB], pz[OR_MAXNB], pg[OR_MAXNB];
  int n_prev;
  double prev_lev;
  double ema[OR_MAXNB];
} Wake;

typedef struct {
  double gate_margin; /* min | |aoa| - crit |, | |aoa| - pi/2 | over steps */
  double ring_margin; /* min distance of the intersection parameters from 0/1 */
  uint64_t shed_mask; /* bit t set when step t shed (t < 64) */
  uint64_t shed_hi;   /* bit t-64 set when step t shed (64 <= t < 128) */
  uint64_t whash;     /* wake-index signature chain (sig_step) */
  int step;           /* step index inside the rollout */
} Diag;

/* Wake-index signature, the same function the CUDA kernel evaluates
 * (paper_2509_16079_b200/csrc/vpm_rollout.cuh wake_sig_*): after each step's shed,
 * merge and ring termination (_core.pyx:322-373) the chain absorbs (wake size,
 * ring-core indices, shed flag); at the end the sum over the final wake of
 * mix(index, age) is folded in.  Equal signatures = same shed steps, same merges
 * per step, same final index -> age order (the ordered-removal contract of
 * remove_particle, _core.pyx:157-172). */
static uint64_t sig_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t sig_step(uint64_t h, int n, int ra, int rb, int shed) {
  uint64_t key = (uint64_t)(uint32_t)n | ((uint64_t)(shed != 0) << 31) |
                 ((uint64_t)(uint16_t)(ra + 1) << 32) | ((uint64_t)(uint16_t)(rb + 1) << 48);
  return sig_mix(h ^ key);
}

static void cfg_load(Cfg *c, const int64_t *ip, const double *fp) {
  c->nb = (int)ip[0];
  c->cap = (int)ip[1];
  memcpy(c->fp, fp, sizeof(double) * P_COUNT);
  double r = fp[P_R_CORE];
  c->rc4 = r * r * r * r; /* _core.pyx:86 */
}

/* regularised kernel velocity of (sx,sz,g) at (tx,tz); _core.pyx:89-97, vpm.py:79-90 */
static inline void kern_reg(double sx, double sz, double g, double tx, double tz,
                            double rc4, double *ux, double *uz) {
  double dx = tx - sx, dz = tz - sz;
  double r2 = dx * dx + dz * dz;
  double c = g / (OR_TWO_PI * sqrt(r2 * r2 + rc4));
  *ux += c * dz;
  *uz -= c * dx;
}

/* unit point vortex at s, normal velocity at t; _core.pyx:135-141, vpm.py:64-76 */
static inline double kern_sing_n(double sx, double sz, double tx, double tz,
                                 double nx, double nz) {
  double dx = tx - sx, dz = tz - sz;
  return (dz * nx - dx * nz) / (OR_TWO_PI * (dx * dx + dz * dz));
}

/* Gaussian elimination with partial pivoting on a row-major n x n system.
 * _core.pyx:100-132 (column-major there); np.linalg.solve in vpm.py:399.
 * Returns 1 on an exactly vanishing pivot. */
static int dense_solve(double *a, double *b, int n) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(a[k * n + k]);
    for (int r = k + 1; r < n; ++r)
      if (fabs(a[r * n + k]) > best) { best = fabs(a[r * n + k]); p = r; }
    if (best == 0.0) return 1;
    if (p != k) {
      for (int c = 0; c < n; ++c) { double t = a[k * n + c]; a[k * n + c] = a[p * n + c]; a[p * n + c] = t; }
      double t = b[k]; b[k] = b[p]; b[p] = t;
    }
    for (int r = k + 1; r < n; ++r) {
      double f = a[r * n + k] / a[k * n + k];
      a[r * n + k] = f;
      for (int c = k + 1; c < n; ++c) a[r * n + c] -= f * a[k * n + c];
      b[r] -= f * b[k];
    }
  }
  for (int k = n - 1; k >= 0; --k) {
    for (int c = k + 1; c < n; ++c) b[k] -= a[k * n + c] * b[c];
    b[k] /= a[k * n + k];
  }
  return 0;
}

/* ordered removal with ring-index remap; _core.pyx:157-172, vpm.py:482-494 */
static void wake_remove(Wake *w, int idx) {
  for (int i = idx; i < w->n - 1; ++i) {
    w->x[i] = w->x[i + 1]; w->z[i] = w->z[i + 1];
    w->g[i] = w->g[i + 1]; w->age[i] = w->age[i + 1];
  }
  w->n -= 1;
  if (w->ring_a == idx) w->ring_a = -1; else if (w->ring_a > idx) w->ring_a -= 1;
  if (w->ring_b == idx) w->ring_b = -1; else if (w->ring_b > idx) w->ring_b -= 1;
}

/* wake self-advection + previous bound row, dissipation, ageing.
 * _core.pyx:192-226, vpm.py:408-428.  (Pairwise-symmetric accumulation order as
 * in the compiled core.) */
static void phase_convect(Wake *w, const Cfg *c, double *vx, double *vz) {
  int n = w->n;
  if (n <= 0) return;
  for (int i = 0; i < n; ++i) { vx[i] = 0.0; vz[i] = 0.0; }
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      double dx = w->x[j] - w->x[i], dz = w->z[j] - w->z[i];
      double r2 = dx * dx + dz * dz;
      double inv = 1.0 / (OR_TWO_PI * sqrt(r2 * r2 + c->rc4));
      double ci = w->g[i] * inv, cj = w->g[j] * inv;
      vx[j] += ci * dz; vz[j] -= ci * dx;
      vx[i] -= cj * dz; vz[i] += cj * dx;
    }
  }
  for (int i = 0; i < n; ++i) {
    double ux = 0.0, uz = 0.0;
    for (int j = 0; j < w->n_prev; ++j) kern_reg(w->px[j], w->pz[j], w->pg[j], w->x[i], w->z[i], c->rc4, &ux, &uz);
    vx[i] += ux; vz[i] += uz;
  }
  double dt = c->fp[P_DT], kd = c->fp[P_K_DISS];
  for (int i = 0; i < n; ++i) {
    w->x[i] += dt * vx[i];
    w->z[i] += dt * vz[i];
    w->g[i] *= kd;
    w->age[i] += 1.0;
  }
}

/* proper segment intersection, degenerate -> no; _core.pyx:144-154, vpm.py:576-587.
 * *margin receives min(|t|,|1-t|,|u|,|1-u|) when the parameters are defined. */
static int seg_cross(double ax0, double az0, double ax1, double az1, double bx0,
                     double bz0, double bx1, double bz1, double *margin) {
  double d1x = ax1 - ax0, d1z = az1 - az0, d2x = bx1 - bx0, d2z = bz1 - bz0;
  double den = d1x * d2z - d1z * d2x;
  if (den == 0.0) return 0;
  double fx = bx0 - ax0, fz = bz0 - az0;
  double t = (fx * d2z - fz * d2x) / den;
  double u = (fx * d1z - fz * d1x) / den;
  double m = fmin(fmin(fabs(t), fabs(1.0 - t)), fmin(fabs(u), fabs(1.0 - u)));
  if (m < *margin) *margin = m;
  return t >= 0.0 && t <= 1.0 && u >= 0.0 && u <= 1.0;
}

/* One coupled step.  Returns 0 ok, 1 singular solve, 2 non-finite.
 * Phase order: _core.pyx:175-462 == vpm.py:635-669 then glider.py:104-122. */
static int coupled_step(double *xs, double u, Wake *w, const Cfg *c, int integrate,
                        double *fw, double *mw, double *scratch_v, Diag *dg) {
  const double *fp = c->fp;
  const int nb = c->nb;
  const double dt = fp[P_DT];
  /* input clamp, _core.pyx:183-187 */
  if (u > fp[P_U_LIM]) u = fp[P_U_LIM];
  else if (u < -fp[P_U_LIM]) u = -fp[P_U_LIM];
  const double rx = xs[0], rz = xs[1], th = xs[2], phi = xs[3];
  const double vx = xs[4], vz = xs[5], om = xs[6];

  phase_convect(w, c, scratch_v, scratch_v + (c->cap + 6));

  /* chord frame and points, _core.pyx:228-245, vpm.py:290-315 */
  const double fx = cos(th), fz = sin(th), nx = -sin(th), nz = cos(th);
  const double s = fp[P_L_CHORD] / nb;
  double cx[OR_MAXNB + 1], cz[OR_MAXNB + 1], bx[OR_MAXNB], bz[OR_MAXNB];
  for (int i = 0; i <= nb; ++i) { cx[i] = rx - fx * s * i; cz[i] = rz - fz * s * i; }
  for (int j = 0; j < nb; ++j) { bx[j] = cx[j] - 0.5 * s * fx; bz[j] = cz[j] - 0.5 * s * fz; }
  const double lx = cx[0] + fp[P_SHED_OFF] * fx, lz = cz[0] + fp[P_SHED_OFF] * fz;
  const double tx = cx[nb] - fp[P_SHED_OFF] * fx, tz = cz[nb] - fp[P_SHED_OFF] * fz;

  /* effective wing AoA and gates, _core.pyx:247-256, vpm.py:318-328 */
  double aoa = 0.0;
  {
    double wx = vx - fp[P_L_W] * om * nx, wz = vz - fp[P_L_W] * om * nz;
    if (wx * wx + wz * wz >= 1e-18) {
      double raw = th - atan2(wz, wx);
      aoa = atan2(sin(raw), cos(raw));
    }
  }
  const int shed = fabs(aoa) > fp[P_CRIT_AOA];
  const int rev = fabs(aoa) > 0.5 * OR_PI;
  if (dg) {
    double m = fmin(fabs(fabs(aoa) - fp[P_CRIT_AOA]), fabs(fabs(aoa) - 0.5 * OR_PI));
    if (m < dg->gate_margin) dg->gate_margin = m;
  }

  /* boundary system, _core.pyx:258-313, vpm.py:331-391 (row-major here) */
  const int ns = shed ? nb + 2 : nb;
  const int r0 = shed ? 1 : 0;
  double A[(OR_MAXNB + 2) * (OR_MAXNB + 2)];
  double gam[OR_MAXNB + 2];
  memset(A, 0, sizeof(double) * ns * ns);
  memset(gam, 0, sizeof(double) * ns);
  for (int i = 0; i < nb; ++i) {
    const int ri = (shed && rev) ? i : i + 1; /* skip the upstream edge point */
    const double px = cx[ri], pz = cz[ri];
    double ux = 0.0, uz = 0.0;
    for (int j = 0; j < w->n; ++j) kern_reg(w->x[j], w->z[j], w->g[j], px, pz, c->rc4, &ux, &uz);
    for (int j = 0; j < ns; ++j) {
      double sx = j < nb ? bx[j] : (j == nb ? lx : tx);
      double sz = j < nb ? bz[j] : (j == nb ? lz : tz);
      A[(r0 + i) * ns + j] = kern_sing_n(sx, sz, px, pz, nx, nz);
    }
    const double svx = vx - om * (pz - rz), svz = vz + om * (px - rx);
    gam[r0 + i] = (svx - ux) * nx + (svz - uz) * nz;
  }
  if (shed) {
    const int ecol = rev ? nb + 1 : nb, epan = rev ? nb - 1 : 0;
    A[0 * ns + ecol] = 1.0;
    A[0 * ns + epan] = fp[P_LEV_GAIN];
    gam[0] = fp[P_LEV_GAIN] * (w->n_prev > 0 ? w->pg[epan] : 0.0);
    double tot = 0.0;
    for (int j = 0; j < ns; ++j) A[(nb + 1) * ns + j] = 1.0;
    for (int j = 0; j < w->n; ++j) tot += w->g[j];
    gam[nb + 1] = -tot;
  }
  if (dense_solve(A, gam, ns)) return 1;
  for (int i = 0; i < ns; ++i)
    if (!isfinite(gam[i])) return 2;

  /* shed LEV then TEV, _core.pyx:322-334, vpm.py:431-446 */
  const double lev_g = shed ? gam[nb] : 0.0;
  if (shed) {
    int k = w->n;
    w->x[k] = lx; w->z[k] = lz; w->g[k] = gam[nb]; w->age[k] = 0.0;
    w->x[k + 1] = tx; w->z[k + 1] = tz; w->g[k + 1] = gam[nb + 1]; w->age[k + 1] = 0.0;
    w->n = k + 2;
    if (dg && dg->step < 64) dg->shed_mask |= (uint64_t)1 << dg->step;
    if (dg && dg->step >= 64 && dg->step < 128) dg->shed_hi |= (uint64_t)1 << (dg->step - 64);
  }

  /* merge the two oldest non-ring particles until at cap, _core.pyx:336-357,
   * vpm.py:449-479; order key (age desc, index asc) */
  while (w->n > c->cap) {
    int first = -1, second = -1;
    for (int i = 0; i < w->n; ++i) {
      if (i == w->ring_a || i == w->ring_b) continue;
      if (first < 0 || w->age[i] > w->age[first]) { second = first; first = i; }
      else if (second < 0 || w->age[i] > w->age[second]) second = i;
    }
    if (first < 0 || second < 0) break;
    int lo = first < second ? first : second, hi = first < second ? second : first;
    w->x[lo] = 0.5 * (w->x[lo] + w->x[hi]);
    w->z[lo] = 0.5 * (w->z[lo] + w->z[hi]);
    w->g[lo] = w->g[lo] + w->g[hi];
    w->age[lo] = w->age[lo] > w->age[hi] ? w->age[lo] : w->age[hi];
    wake_remove(w, hi);
  }

  /* ring termination against the chord offset by -0.02 l n, _core.pyx:359-373,
   * vpm.py:539-573 */
  if (w->ring_a >= 0 && w->ring_b >= 0) {
    const double ox = -0.02 * fp[P_L_CHORD] * nx, oz = -0.02 * fp[P_L_CHORD] * nz;
    double mm = 1e300;
    int hit = seg_cross(w->x[w->ring_a], w->z[w->ring_a], w->x[w->ring_b], w->z[w->ring_b],
                        rx + ox, rz + oz, rx - fp[P_L_CHORD] * fx + ox,
                        rz - fp[P_L_CHORD] * fz + oz, &mm);
    if (dg && mm < dg->ring_margin) dg->ring_margin = mm;
    if (hit) {
      int hi = w->ring_a > w->ring_b ? w->ring_a : w->ring_b;
      int lo = w->ring_a > w->ring_b ? w->ring_b : w->ring_a;
      wake_remove(w, hi);
      wake_remove(w, lo);
      w->ring_a = -1;
      w->ring_b = -1;
    }
  }
  if (dg) dg->whash = sig_step(dg->whash, w->n, w->ring_a, w->ring_b, shed);

  /* unsteady-Bernoulli panel loads about the wing point, _core.pyx:375-410,
   * vpm.py:580-628 */
  {
    const double eta = fp[P_ETA], rho = fp[P_RHO];
    const double xwx = rx - fp[P_L_W] * fx, xwz = rz - fp[P_L_W] * fz;
    const int hp = w->n_prev > 0;
    const double dlev = hp ? (lev_g - w->prev_lev) / dt : 0.0;
    double cum = 0.0, cum_prev = 0.0, Fx = 0.0, Fz = 0.0, M = 0.0;
    for (int i = 0; i < nb; ++i) {
      double ux = 0.0, uz = 0.0;
      for (int j = 0; j < w->n; ++j) kern_reg(w->x[j], w->z[j], w->g[j], bx[i], bz[i], c->rc4, &ux, &uz);
      cum += gam[i];
      double rate = 0.0;
      if (hp) { cum_prev += w->pg[i]; rate = (cum - cum_prev) / dt + dlev; }
      const double e = eta * rate + (1.0 - eta) * (hp ? w->ema[i] : 0.0);
      w->ema[i] = e;
      const double svx = vx - om * (bz[i] - rz), svz = vz + om * (bx[i] - rx);
      const double beta = (ux - svx) * fx + (uz - svz) * fz;
      const double dp = rho * (beta * gam[i] / s + e);
      const double pfx = dp * s * nx, pfz = dp * s * nz;
      Fx += pfx; Fz += pfz;
      M += (bx[i] - xwx) * pfz - (bz[i] - xwz) * pfx;
    }
    fw[0] = Fx; fw[1] = Fz; *mw = M;
    for (int i = 0; i < nb; ++i) { w->px[i] = bx[i]; w->pz[i] = bz[i]; w->pg[i] = gam[i]; }
    w->n_prev = nb;
    w->prev_lev = lev_g;
  }
  if (!integrate) return 0;

  /* elevator flat-plate force, accelerations, forward Euler:
   * _core.pyx:423-461, glider.py:40-122 */
  const double ce = cos(th + phi), se = sin(th + phi);
  const double fex = ce, fez = se, nex = -se, nez = ce;
  const double L = fp[P_L], Le = fp[P_L_E];
  const double xex = rx - L * fx - Le * fex, xez = rz - L * fz - Le * fez;
  const double vex = vx - L * om * nx - Le * (om + u) * nex;
  const double vez = vz - L * om * nz - Le * (om + u) * nez;
  const double sp2 = vex * vex + vez * vez;
  double Ex = 0.0, Ez = 0.0;
  if (sp2 >= 1e-18) {
    const double ae = th + phi - atan2(vez, vex);
    const double cn = 0.5 * fp[P_RHO] * sp2 * fp[P_S_E] * 2.0 * sin(ae);
    Ex = cn * nex; Ez = cn * nez;
  }
  const double xwx = rx - fp[P_L_W] * fx, xwz = rz - fp[P_L_W] * fz;
  const double ax = (fw[0] + Ex) / fp[P_M];
  const double az = (fw[1] + Ez) / fp[P_M] - fp[P_G];
  const double tq = *mw + ((xwx - rx) * fw[1] - (xwz - rz) * fw[0]) + ((xex - rx) * Ez - (xez - rz) * Ex);
  const double wd = tq / fp[P_I];
  xs[0] = rx + dt * vx;
  xs[1] = rz + dt * vz;
  xs[2] = th + dt * om;
  double ph = phi + dt * u;
  if (ph > fp[P_PHI_LIM]) ph = fp[P_PHI_LIM];
  else if (ph < -fp[P_PHI_LIM]) ph = -fp[P_PHI_LIM];
  xs[3] = ph;
  xs[4] = vx + dt * ax;
  xs[5] = vz + dt * az;
  xs[6] = om + dt * wd;
  for (int i = 0; i < 7; ++i)
    if (!isfinite(xs[i])) return 2;
  return 0;
}

typedef struct {
  const double *wake_pos, *wake_gamma;
  const int64_t *wake_age;
  int n_wake, ring_a, ring_b;
  const double *prev_pos, *prev_gamma;
  int n_prev;
  double prev_lev;
  const double *ema;
} Snapshot;

static void wake_fork(Wake *w, const Snapshot *s, const Cfg *c, double *buf) {
  int capbuf = c->cap + 6;
  w->x = buf; w->z = buf + capbuf; w->g = buf + 2 * capbuf; w->age = buf + 3 * capbuf;
  for (int i = 0; i < s->n_wake; ++i) {
    w->x[i] = s->wake_pos[2 * i]; w->z[i] = s->wake_pos[2 * i + 1];
    w->g[i] = s->wake_gamma[i]; w->age[i] = (double)s->wake_age[i];
  }
  w->n = s->n_wake; w->ring_a = s->ring_a; w->ring_b = s->ring_b;
  for (int i = 0; i < s->n_prev; ++i) {
    w->px[i] = s->prev_pos[2 * i]; w->pz[i] = s->prev_pos[2 * i + 1]; w->pg[i] = s->prev_gamma[i];
  }
  w->n_prev = s->n_prev; w->prev_lev = s->prev_lev;
  for (int i = 0; i < c->nb; ++i) w->ema[i] = s->ema[i];
}

static void wake_dump(const Wake *w, const Cfg *c, double *wake_pos, double *wake_gamma,
                      int64_t *wake_age, int *scal, double *prev_pos, double *prev_gamma,
                      double *prev_lev, double *ema) {
  int capbuf = c->cap + 4;
  memset(wake_pos, 0, sizeof(double) * 2 * capbuf);
  memset(wake_gamma, 0, sizeof(double) * capbuf);
  memset(wake_age, 0, sizeof(int64_t) * capbuf);
  for (int i = 0; i < w->n && i < capbuf; ++i) {
    wake_pos[2 * i] = w->x[i]; wake_pos[2 * i + 1] = w->z[i];
    wake_gamma[i] = w->g[i]; wake_age[i] = (int64_t)w->age[i];
  }
  scal[0] = w->n; scal[1] = w->ring_a; scal[2] = w->ring_b; scal[3] = w->n_prev;
  memset(prev_pos, 0, sizeof(double) * 2 * c->nb);
  memset(prev_gamma, 0, sizeof(double) * c->nb);
  for (int i = 0; i < w->n_prev; ++i) {
    prev_pos[2 * i] = w->px[i]; prev_pos[2 * i + 1] = w->pz[i]; prev_gamma[i] = w->pg[i];
  }
  *prev_lev = w->prev_lev;
  for (int i = 0; i < c->nb; ++i) ema[i] = w->ema[i];
}

/* run_rollout, _core.pyx:465-491: status 0 or 1 + failing step */
static int64_t run_one(double *xs, const double *ctrl, int T, Wake *w, const Cfg *c,
                       double *traj, double *scratch_v, Diag *dg, int64_t *nw_steps) {
  double fw[2], mw;
  if (traj) memcpy(traj, xs, 7 * sizeof(double));
  for (int t = 0; t < T; ++t) {
    if (dg) dg->step = t;
    int rc = coupled_step(xs, ctrl[t], w, c, 1, fw, &mw, scratch_v, dg);
    if (nw_steps) nw_steps[t] = w->n;
    if (rc != 0) return 1 + t;
    if (fabs(xs[6]) > OR_BLOWUP_OMEGA || fabs(xs[4]) > OR_BLOWUP_SPEED || fabs(xs[5]) > OR_BLOWUP_SPEED)
      return 1 + t;
    if (traj) memcpy(traj + 7 * (t + 1), xs, 7 * sizeof(double));
  }
  return 0;
}

/* Exported: single step (Engine.step / Engine.fluid_step contract, _core.pyx:536-576). */
int oracle_step(double *x, double u, const double *wake_pos, const double *wake_gamma,
                const int64_t *wake_age, int n_wake, int ring_a, int ring_b,
                const double *prev_pos, const double *prev_gamma, int n_prev, double prev_lev,
                const double *ema, const int64_t *iparams, const double *fparams, int integrate,
                double *fw, double *mw, double *o_wake_pos, double *o_wake_gamma,
                int64_t *o_wake_age, int *o_scal, double *o_prev_pos, double *o_prev_gamma,
                double *o_prev_lev, double *o_ema) {
  Cfg c;
  cfg_load(&c, iparams, fparams);
  if (c.nb > OR_MAXNB) return -1;
  int capbuf = c.cap + 6;
  double *buf = (double *)calloc((size_t)6 * capbuf, sizeof(double));
  Snapshot s = {wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma, n_prev, prev_lev, ema};
  Wake w;
  wake_fork(&w, &s, &c, buf);
  *mw = 0.0; fw[0] = fw[1] = 0.0;
  int rc = coupled_step(x, u, &w, &c, integrate, fw, mw, buf + 4 * capbuf, NULL);
  wake_dump(&w, &c, o_wake_pos, o_wake_gamma, o_wake_age, o_scal, o_prev_pos, o_prev_gamma, o_prev_lev, o_ema);
  free(buf);
  return rc;
}

/* Exported: batched independent rollouts (batch_rollout, _core.pyx:664-741), with
 * optional per-rollout start states (x0_stride = 7) for the policy-synthesis cloud
 * (policy.py:66-91) and per-rollout diagnostics.  Any output pointer may be NULL. */
int oracle_batch_rollout(const double *x0, int x0_stride, const double *controls, int B, int T,
                         const double *wake_pos, const double *wake_gamma, const int64_t *wake_age,
                         int n_wake, int ring_a, int ring_b, const double *prev_pos,
                         const double *prev_gamma, int n_prev, double prev_lev, const double *ema,
                         const int64_t *iparams, const double *fparams, int64_t *status,
                         double *finals, double *trajs, uint64_t *shed_mask, int32_t *n_final,
                         double *gate_margin, double *ring_margin, int64_t *nw_steps,
                         uint64_t *shed_mask_hi, uint64_t *wake_hash, int threads) {
  Cfg c;
  cfg_load(&c, iparams, fparams);
  if (c.nb > OR_MAXNB) return -1;
  Snapshot s = {wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma, n_prev, prev_lev, ema};
  const int capbuf = c.cap + 6;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
  for (int b = 0; b < B; ++b) {
    double *buf = (double *)malloc(sizeof(double) * 6 * capbuf);
    Wake w;
    wake_fork(&w, &s, &c, buf);
    double xs[7];
    memcpy(xs, x0 + (size_t)b * x0_stride, 7 * sizeof(double));
    Diag dg = {1e300, 1e300, 0, 0, 0, 0};
    int64_t rc = run_one(xs, controls + (size_t)b * T, T, &w, &c,
                         trajs ? trajs + (size_t)b * (T + 1) * 7 : NULL, buf + 4 * capbuf, &dg,
                         nw_steps ? nw_steps + (size_t)b * T : NULL);
    if (status) status[b] = rc;
    if (finals) memcpy(finals + 7 * (size_t)b, xs, 7 * sizeof(double));
    if (shed_mask) shed_mask[b] = dg.shed_mask;
    if (shed_mask_hi) shed_mask_hi[b] = dg.shed_hi;
    if (wake_hash) {
      uint64_t hs = 0;
      for (int i = 0; i < w.n; ++i) hs += sig_mix(((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)(int64_t)w.age[i]);
      wake_hash[b] = sig_mix(dg.whash ^ hs);
    }
    if (n_final) n_final[b] = w.n;
    if (gate_margin) gate_margin[b] = dg.gate_margin;
    if (ring_margin) ring_margin[b] = dg.ring_margin;
    free(buf);
  }
  return 0;
}

/* Exported: single rollout returning the final fluid (rollout, _core.pyx:609-661). */
int64_t oracle_rollout(double *x, const double *controls, int T, const double *wake_pos,
                       const double *wake_gamma, const int64_t *wake_age, int n_wake, int ring_a,
                       int ring_b, const double *prev_pos, const double *prev_gamma, int n_prev,
                       double prev_lev, const double *ema, const int64_t *iparams,
                       const double *fparams, double *traj, double *o_wake_pos,
                       double *o_wake_gamma, int64_t *o_wake_age, int *o_scal, double *o_prev_pos,
                       double *o_prev_gamma, double *o_prev_lev, double *o_ema) {
  Cfg c;
  cfg_load(&c, iparams, fparams);
  if (c.nb > OR_MAXNB) return -1;
  const int capbuf = c.cap + 6;
  double *buf = (double *)calloc((size_t)6 * capbuf, sizeof(double));
  Snapshot s = {wake_pos, wake_gamma, wake_age, n_wake, ring_a, ring_b, prev_pos, prev_gamma, n_prev, prev_lev, ema};
  Wake w;
  wake_fork(&w, &s, &c, buf);
  int64_t rc = run_one(x, controls, T, &w, &c, traj, buf + 4 * capbuf, NULL, NULL);
  if (o_wake_pos)
    wake_dump(&w, &c, o_wake_pos, o_wake_gamma, o_wake_age, o_scal, o_prev_pos, o_prev_gamma, o_prev_lev, o_ema);
  free(buf);
  return rc;
}

int oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
