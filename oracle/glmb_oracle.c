/*
 * glmb_oracle.c -- plain, slow, fp64 CPU ORACLE for the GLMB step core.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2512_06230_b200/, libglmb.so) never links, loads
 * or calls it, and shares no code, header, table or constant generator with
 * it.  This file follows the paper's definitions written out directly, in
 * the paper's order and notation, with no blocking, fusion or reordering.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section named beside it);
 * DESIGN.md "Readings" R1..R22 = the ambiguity register.
 *
 * Precision: every float input (states, weights, z, R, P_D, kappa, gamma, dt,
 * sigmas) is the fp32 value the GPU sees, widened exactly to double; every
 * arithmetic step below is fp64 (libm sin/cos/exp/log, correctly rounded or
 * within 1 ulp).  Outputs are fp64.
 *
 * Functions and the passage each follows:
 *   O1 oracle_philox4x32_10  -- Philox4x32-10 (Salmon et al., SC'11), R9
 *   O2 keying                -- (seed; p, gid, step, tag) counter layout, R9
 *   O3 oracle_uniform_u32    -- u = (2*(r>>9)+1) * 2^-24, R9
 *   O4 Box-Muller            -- n0 = sqrt(-2 ln ua) cos(2 pi ub), n1 = ... sin, R9
 *   O5 oracle_ctrv / oracle_predict -- CTRV survival propagation, P:3, P:24 (§Approach), R7, R8
 *   O6 oracle_birth          -- LMB birth sampling, P:24 (§Approach), R10
 *   O7 oracle_compat         -- C_k equation, P:26-38 (§Approach), R1-R6, R12
 *   O8 oracle_reweight       -- particle update, P:53 (§Approach), R13, R14, R16
 *   O9 oracle_death_prob     -- posterior death probability, P:44 (§Approach), R23
 *   O10 oracle_compat_rows   -- row-wise (CSR) view of C_k, R26
 *   O11 oracle_assoc_sample  -- two-stage sampler + hypothesis weight, R24-R26, R28
 *   O12 oracle_dedup         -- unique successor hypotheses, R27
 *   O13 oracle_prune         -- normalise, tau threshold, H_max, R29
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846

int oracle_version(void) { return 1; }

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ O1 */
/* Philox4x32-10: ten rounds of
 *   (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0))
 * with the key bumped by the Weyl constants (W0,W1) between rounds.
 * Constants: Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
 * as 1, 2, 3", SC'11, Philox4x32 (M0=0xD2511F53, M1=0xCD9E8D57,
 * W0=0x9E3779B9, W1=0xBB67AE85). */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                          uint32_t out[4]) {
  const uint64_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = M0 * (uint64_t)c0;
    uint64_t p1 = M1 * (uint64_t)c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* batched form: key = (lo32(seed), hi32(seed)) (O2) */
void oracle_philox_batch(uint64_t seed, const uint32_t *ctr, int64_t n,
                         uint32_t *out) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int64_t i = 0; i < n; ++i) oracle_philox4x32_10(ctr + 4 * i, key, out + 4 * i);
}

/* ------------------------------------------------------------------ O3 */
/* u = (2*(r>>9) + 1) * 2^-24, an odd multiple of 2^-24 in [2^-24, 1-2^-24]. */
double oracle_uniform_u32(uint32_t r) {
  return (2.0 * (double)(r >> 9) + 1.0) * (1.0 / 16777216.0);
}

/* ------------------------------------------------------------------ O4 */
static void box_muller(uint32_t ra, uint32_t rb, double *n0, double *n1) {
  double ua = oracle_uniform_u32(ra);
  double ub = oracle_uniform_u32(rb);
  double rho = sqrt(-2.0 * log(ua));
  *n0 = rho * cos(2.0 * OR_PI * ub);
  *n1 = rho * sin(2.0 * OR_PI * ub);
}

/* four standard normals from one Philox block: words (0,1) -> (n0,n1),
 * words (2,3) -> (n2,n3). */
void oracle_normals4(uint64_t seed, const uint32_t ctr[4], double n[4]) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t r[4];
  oracle_philox4x32_10(ctr, key, r);
  box_muller(r[0], r[1], &n[0], &n[1]);
  box_muller(r[2], r[3], &n[2], &n[3]);
}

void oracle_normals_batch(uint64_t seed, const uint32_t *ctr, int64_t n,
                          double *out) {
  for (int64_t i = 0; i < n; ++i) oracle_normals4(seed, ctr + 4 * i, out + 4 * i);
}

/* ------------------------------------------------------------------ O5 */
/* wrap(a) = a - 2 pi * ceil((a - pi) / (2 pi)) in (-pi, pi] (R7). */
double oracle_wrap(double a) {
  return a - 2.0 * OR_PI * ceil((a - OR_PI) / (2.0 * OR_PI));
}

/* CTRV ("constant turn rate and velocity", P:3, §Approach) with the
 * acceleration / yaw-acceleration noise terms of R7:
 *   |omega| > 1e-4:  dx = (v/omega)(sin(psi+omega dt) - sin psi)
 *                    dy = (v/omega)(cos psi - cos(psi+omega dt))
 *   else (2nd-order Taylor of the same flow):
 *                    dx = v dt cos psi - 1/2 v omega dt^2 sin psi
 *                    dy = v dt sin psi + 1/2 v omega dt^2 cos psi
 *   x+ = x + dx + 1/2 dt^2 cos psi nu_a
 *   y+ = y + dy + 1/2 dt^2 sin psi nu_a
 *   v+ = v + dt nu_a
 *   psi+ = wrap(psi + omega dt + 1/2 dt^2 nu_w)
 *   omega+ = omega + dt nu_w
 * s_in/s_out: [x, y, v, psi, omega]. */
void oracle_ctrv(const double s_in[5], double dt, double nu_a, double nu_w,
                 double s_out[5]) {
  double x = s_in[0], y = s_in[1], v = s_in[2], psi = s_in[3], om = s_in[4];
  double dx, dy;
  if (fabs(om) > 1e-4) {
    dx = (v / om) * (sin(psi + om * dt) - sin(psi));
    dy = (v / om) * (cos(psi) - cos(psi + om * dt));
  } else {
    dx = v * dt * cos(psi) - 0.5 * v * om * dt * dt * sin(psi);
    dy = v * dt * sin(psi) + 0.5 * v * om * dt * dt * cos(psi);
  }
  s_out[0] = x + dx + 0.5 * dt * dt * cos(psi) * nu_a;
  s_out[1] = y + dy + 0.5 * dt * dt * sin(psi) * nu_a;
  s_out[2] = v + dt * nu_a;
  s_out[3] = oracle_wrap(psi + om * dt + 0.5 * dt * dt * nu_w);
  s_out[4] = om + dt * nu_w;
}

/* Survival prediction: "particles representing targets that have survived
 * from step k-1 are propagated forward using the constant turn rate and
 * velocity kinematics model ... as a batch operation over all particles and
 * surviving tracks" (§Approach).  Noise (O2, R9): Philox block with
 * counter (p/2, gid_j, step, tag=0) (domain 0 = predict); particle p takes
 * (n0, n1) if p is even, (n2, n3) if odd; nu_a = sigma_a n_a, nu_w = sigma_w n_w.
 * Element (j,p) at j*ld + p.  Outputs fp64 [T][ld]. */
void oracle_predict(int32_t T, int32_t P, int64_t ld, const float *x,
                    const float *y, const float *v, const float *psi,
                    const float *omega, const int32_t *gid, float dt,
                    float sigma_a, float sigma_w, uint64_t seed, uint32_t step,
                    double *ox, double *oy, double *ov, double *opsi,
                    double *oomega) {
#pragma omp parallel for schedule(dynamic)
  for (int32_t j = 0; j < T; ++j) {
    for (int32_t p = 0; p < P; ++p) {
      int64_t e = (int64_t)j * ld + p;
      /* one Philox block per particle pair (R9): counter (p/2, gid, step, 0);
       * the even particle takes normals (n0, n1), the odd one (n2, n3) */
      uint32_t ctr[4] = {(uint32_t)p / 2u, (uint32_t)gid[j], step, 0u};
      double n[4];
      oracle_normals4(seed, ctr, n);
      double na = (p % 2 == 0) ? n[0] : n[2];
      double nw = (p % 2 == 0) ? n[1] : n[3];
      double s[5] = {x[e], y[e], v[e], psi[e], omega[e]}, o[5];
      oracle_ctrv(s, (double)dt, (double)sigma_a * na, (double)sigma_w * nw, o);
      ox[e] = o[0]; oy[e] = o[1]; ov[e] = o[2]; opsi[e] = o[3]; oomega[e] = o[4];
    }
  }
}

/* ------------------------------------------------------------------ O6 */
/* LMB birth: "a set of particles is sampled from the birth probability
 * distribution for each new track" (§Approach); distribution
 * N(mu_b, L_b L_b^T) (R10).  Draws: block tag (1<<8|0) gives n0..n3, block
 * tag (1<<8|1) words (0,1) give n4.  x = mu_b + L_b n, psi wrapped, w = 1/P.
 * mean: [B][5]; chol: [B][15] row-major packed lower triangle. */
void oracle_birth(int32_t B, int32_t P, int64_t ld, const float *mean,
                  const float *chol, const int32_t *gid, uint64_t seed,
                  uint32_t step, double *ox, double *oy, double *ov,
                  double *opsi, double *oomega, double *ow) {
#pragma omp parallel for schedule(dynamic)
  for (int32_t b = 0; b < B; ++b) {
    for (int32_t p = 0; p < P; ++p) {
      int64_t e = (int64_t)b * ld + p;
      uint32_t c0[4] = {(uint32_t)p, (uint32_t)gid[b], step, (1u << 8) | 0u};
      uint32_t c1[4] = {(uint32_t)p, (uint32_t)gid[b], step, (1u << 8) | 1u};
      double na[4], nb[4];
      oracle_normals4(seed, c0, na);
      oracle_normals4(seed, c1, nb);
      double n[5] = {na[0], na[1], na[2], na[3], nb[0]};
      double s[5];
      int idx = 0;
      for (int r = 0; r < 5; ++r) {
        double acc = (double)mean[b * 5 + r];
        for (int c = 0; c <= r; ++c) acc += (double)chol[b * 15 + idx + c] * n[c];
        idx += r + 1;
        s[r] = acc;
      }
      ox[e] = s[0]; oy[e] = s[1]; ov[e] = s[2];
      opsi[e] = oracle_wrap(s[3]);
      oomega[e] = s[4];
      ow[e] = 1.0 / (double)P;
    }
  }
}

/* ------------------------------------------------------------------ O7 */
/* N(z; (px,py), R) for a 2x2 SPD R = [[Rxx,Rxy],[Rxy,Ryy]]:
 *   exp(-1/2 d^T R^-1 d) / (2 pi sqrt(det R)),  d = z - (px,py),
 *   R^-1 = [[Ryy, -Rxy], [-Rxy, Rxx]] / det R. */
double oracle_gauss2(double zx, double zy, double px, double py, double Rxx,
                     double Rxy, double Ryy) {
  double det = Rxx * Ryy - Rxy * Rxy;
  double dx = zx - px, dy = zy - py;
  double q = (Ryy * dx * dx - 2.0 * Rxy * dx * dy + Rxx * dy * dy) / det;
  return exp(-0.5 * q) / (2.0 * OR_PI * sqrt(det));
}

/* ln N(z; (px,py), R) = -1/2 d^T R^-1 d - ln(2 pi sqrt(det R)), the same
 * density in log form (no underflow for far-away particles). */
double oracle_loggauss2(double zx, double zy, double px, double py, double Rxx,
                        double Rxy, double Ryy) {
  double det = Rxx * Ryy - Rxy * Rxy;
  double dx = zx - px, dy = zy - py;
  double q = (Ryy * dx * dx - 2.0 * Rxy * dx * dy + Rxx * dy * dy) / det;
  return -0.5 * q - log(2.0 * OR_PI * sqrt(det));
}

/* Compatibility matrix, P:26-38 (§Approach, equation for C_k):
 *   C[i,j] = g_ij * P_D * L(z_i | x_j)   for j = 1..T_k   (R1: P_D factor)
 *   C[i,0] = kappa                                         (clutter, R5)
 *   g_ij   = [L(z_i | x_j) >= gamma]                       (R2)
 *   L(z | x_j) = sum_p w_jp N(z; H x_jp, R), H = [I2 0]    (R3)
 * Weights are used as supplied (R12).  Sum over p is sequential fp64.
 * Outputs: Lik [T][M] (L without P_D, for the gate band), C_clutter [M],
 * C_tracks [T][ldc] (column-major C: column j+1 of C is row j here),
 * gate [T][ldg] u32 words, bit (i%32) of word i/32. */
void oracle_compat(int32_t T, int32_t P, int64_t ld, const float *x,
                   const float *y, const float *w, int32_t M, const float *Z,
                   float Rxx, float Rxy, float Ryy, float p_d, float kappa,
                   float gamma, double *Lik, double *C_clutter,
                   double *C_tracks, int64_t ldc, uint32_t *gate,
                   int64_t ldg) {
  for (int32_t i = 0; i < M; ++i) C_clutter[i] = (double)kappa;
#pragma omp parallel for schedule(dynamic)
  for (int32_t j = 0; j < T; ++j) {
    for (int64_t k = 0; k < ldg; ++k) gate[(int64_t)j * ldg + k] = 0u;
    for (int32_t i = 0; i < M; ++i) {
      double L = 0.0;
      for (int32_t p = 0; p < P; ++p) {
        int64_t e = (int64_t)j * ld + p;
        L += (double)w[e] * oracle_gauss2(Z[2 * i], Z[2 * i + 1], x[e], y[e],
                                          Rxx, Rxy, Ryy);
      }
      int g = (L >= (double)gamma);
      Lik[(int64_t)j * M + i] = L;
      C_tracks[(int64_t)j * ldc + i] = g ? (double)p_d * L : 0.0;
      if (g) gate[(int64_t)j * ldg + i / 32] |= (1u << (i % 32));
    }
  }
}

/* ------------------------------------------------------------------ O8 */
/* Particle update, P:53 (§Approach): "The particle weights are updated
 * according to the measurement likelihood" -- Bayes' rule on the weights of
 * track j for every measurement the association map theta assigns to it
 * (R13, R14: theta[i] = 0 clutter, theta[i] = c >= 1 means C column c;
 * local track j is column col_offset + j + 1):
 *   S_j = {i : theta_i = col_offset + j + 1}
 *   S_j empty : w unchanged, logZ_j = ln sum_p w_p, flag 0
 *   otherwise : l_p = ln w_p + sum_{i in S_j} ln N(z_i; (x_p,y_p), R)
 *               (ln N via oracle_loggauss2, the log of the same density)
 *               m = max_p l_p ; m = -inf -> w' = 1/P, flag bit0 (R16)
 *               w'_p = exp(l_p - m) / sum_q exp(l_q - m)
 *               logZ_j = m + ln sum_q exp(l_q - m)
 * (logZ_j = ln sum_p w_p prod_i N(z_i; .), the log normaliser; the max
 * shift is only fp64 range safety). */
void oracle_reweight(int32_t T, int32_t P, int64_t ld, const float *x,
                     const float *y, const float *w, int32_t M, const float *Z,
                     float Rxx, float Rxy, float Ryy, const int32_t *theta,
                     int32_t col_offset, double *w_out, double *logZ,
                     uint32_t *flags) {
#pragma omp parallel for schedule(dynamic)
  for (int32_t j = 0; j < T; ++j) {
    int32_t col = col_offset + j + 1;
    int nS = 0;
    for (int32_t i = 0; i < M; ++i) nS += (theta[i] == col);
    int64_t base = (int64_t)j * ld;
    flags[j] = 0u;
    if (nS == 0) {
      double s = 0.0;
      for (int32_t p = 0; p < P; ++p) {
        w_out[base + p] = (double)w[base + p];
        s += (double)w[base + p];
      }
      logZ[j] = log(s);
      continue;
    }
    double *l = (double *)malloc(sizeof(double) * (size_t)(P > 0 ? P : 1));
    double m = -INFINITY;
    for (int32_t p = 0; p < P; ++p) {
      double lp = log((double)w[base + p]);
      for (int32_t i = 0; i < M; ++i)
        if (theta[i] == col)
          lp += oracle_loggauss2(Z[2 * i], Z[2 * i + 1], x[base + p],
                                 y[base + p], Rxx, Rxy, Ryy);
      l[p] = lp;
      if (lp > m) m = lp;
    }
    if (m == -INFINITY) {
      for (int32_t p = 0; p < P; ++p) w_out[base + p] = 1.0 / (double)P;
      logZ[j] = -INFINITY;
      flags[j] = 1u;
    } else {
      double s = 0.0;
      for (int32_t p = 0; p < P; ++p) s += exp(l[p] - m);
      for (int32_t p = 0; p < P; ++p) w_out[base + p] = exp(l[p] - m) / s;
      logZ[j] = m + log(s);
    }
    free(l);
  }
}

/* ==================================================================
 * Hypothesis machinery: death probability, the
 * row-wise view of C_k, the two-stage association sampler with de-duplication,
 * the successor hypothesis weight, and pruning.  P:44-53 (§Approach).
 * ================================================================== */

/* O9 Posterior death probability, P:44 (§Approach: "We compute a posterior
 * probability of track death for each track d_prob(x_j), balancing its prior
 * survival probability against the likelihood of it being detected"; the
 * formula is deferred to a citation -- reading R23):
 *   e_j = max_{i : g_ij} C[i,j] / (C[i,j] + kappa)     (0 if no gated i)
 *   d_j = (1 - P_S) / ((1 - P_S) + P_S ((1 - P_D) + P_D e_j)),  d_j = 0 if P_S = 1.
 * C_tracks fp32 [T][ldc] (column-major C, as glmb_compat writes it), gate
 * [T][ldg] bits. */
void oracle_death_prob(int32_t T, int32_t M, const float *C_tracks, int64_t ldc,
                       const uint32_t *gate, int64_t ldg, float p_d, float kappa,
                       const float *p_s, double *d_out) {
  for (int32_t j = 0; j < T; ++j) {
    double e = 0.0;
    for (int32_t i = 0; i < M; ++i) {
      if ((gate[(int64_t)j * ldg + i / 32] >> (i % 32)) & 1u) {
        double c = (double)C_tracks[(int64_t)j * ldc + i];
        double r = c / (c + (double)kappa);
        if (r > e) e = r;
      }
    }
    double ps = (double)p_s[j], pd = (double)p_d;
    if (ps == 1.0) {
      d_out[j] = 0.0;
    } else {
      d_out[j] = (1.0 - ps) / ((1.0 - ps) + ps * ((1.0 - pd) + pd * e));
    }
  }
}

/* O10 Row-wise (CSR) view of C_k: row i lists the gated track columns j
 * (ascending) with C[i, j+1] -- the rows the categorical of P:46 normalises.
 * row_ptr [M+1]; col [nnz] (0-based track index j, i.e. C column j+1);
 * val [nnz] (the fp32 entry, copied); ln_val [nnz] = ln(val) in fp64. */
void oracle_compat_rows(int32_t T, int32_t M, const float *C_tracks, int64_t ldc,
                        const uint32_t *gate, int64_t ldg, int32_t *row_ptr,
                        int32_t *col, float *val, double *ln_val) {
  int32_t n = 0;
  for (int32_t i = 0; i < M; ++i) {
    row_ptr[i] = n;
    for (int32_t j = 0; j < T; ++j) {
      if ((gate[(int64_t)j * ldg + i / 32] >> (i % 32)) & 1u) {
        col[n] = j;
        val[n] = C_tracks[(int64_t)j * ldc + i];
        ln_val[n] = log((double)val[n]);
        ++n;
      }
    }
  }
  row_ptr[M] = n;
}

/* one uniform for (index n, parent h, sample s, domain): Philox4x32-10 block
 * with counter (n/4, h, step, domain<<24 | s), word n%4, mapped by O3
 * (reading R24) */
static double sampler_uniform(uint64_t seed, uint32_t step, uint32_t domain,
                              int64_t n, int32_t h, int32_t s) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {(uint32_t)(n / 4), (uint32_t)h, step, (domain << 24) | (uint32_t)s};
  uint32_t r[4];
  oracle_philox4x32_10(ctr, key, r);
  return oracle_uniform_u32(r[n % 4]);
}

/* O11 Two-stage association sampler, P:44-48 (§Approach), one sample (h, s)
 * of parent hypothesis h:
 *  stage 1 ("Bernoulli sampling step using d_prob to determine which
 *   tracks survive"): track j of the parent survives iff u_j < 1 - d_j,
 *   decided in fp32 as the kernel does (R25);
 *  stage 2 ("for each measurement i, an association is sampled from a
 *   categorical distribution defined by normalizing the corresponding row in
 *   the modified matrix C'_k"; dead columns zeroed): theta_i = 0 with weight
 *   kappa, theta_i = j+1 with weight C[i, j+1] for surviving j -- inverse CDF
 *   in fp32 in ascending column order (R26): total = kappa + sum, t = u*total,
 *   first column whose running sum exceeds t (the last positive one if
 *   rounding leaves none).
 *  weight ("multiplying its parent's weight with the joint likelihood of
 *   the sampled survival/death events and data associations", R28):
 *   ln w = ln w_parent + sum_{j in parent} (alive ? ln P_S : ln(1 - P_S))
 *        + sum_i ln C'[i, theta_i] + sum_{alive j} lc(n_j),
 *   n_j = #{i : theta_i = j+1}; lc(0) = ln(1 - P_D), lc(n >= 1) = 0 by default;
 *   with a count table (n_count > 0) lc(n) = count_lp[min(n, n_count - 1)]:
 *   the cardinality prior on the number of measurements per object that the
 *   independent proposal ignores and the importance weight restores.
 * Outputs for sample q = h*H_up + s: alive [q][ldt] bits, theta [q][ldm],
 * logw [q]. */
void oracle_assoc_sample(int32_t H_old, int32_t H_up, int32_t T, int32_t M,
                         const uint32_t *parent_mask, int64_t ldt,
                         const double *parent_logw, const float *d_prob,
                         const float *p_s, float p_d, float kappa,
                         const int32_t *row_ptr, const int32_t *col,
                         const float *val, const double *ln_val,
                         const double *count_lp, int32_t n_count, uint64_t seed,
                         uint32_t step, uint32_t *alive, int32_t *theta,
                         int64_t ldm, double *logw) {
#pragma omp parallel for schedule(dynamic)
  for (int64_t q = 0; q < (int64_t)H_old * H_up; ++q) {
    int32_t h = (int32_t)(q / H_up), s = (int32_t)(q % H_up);
    const uint32_t *pm = parent_mask + (int64_t)h * ldt;
    uint32_t *al = alive + q * ldt;
    int32_t *th = theta + q * ldm;
    int *detected = (int *)calloc((size_t)(T > 0 ? T : 1), sizeof(int));
    double lw = parent_logw[h];
    for (int64_t k = 0; k < ldt; ++k) al[k] = 0u;
    /* stage 1 */
    for (int32_t j = 0; j < T; ++j) {
      if (!((pm[j / 32] >> (j % 32)) & 1u)) continue;
      float u = (float)sampler_uniform(seed, step, 2u, j, h, s);
      float thr = 1.0f - d_prob[j];
      int a = u < thr;
      if (a) al[j / 32] |= 1u << (j % 32);
      lw += a ? log((double)p_s[j]) : log(1.0 - (double)p_s[j]);
    }
    /* stage 2 */
    for (int32_t i = 0; i < M; ++i) {
      float u = (float)sampler_uniform(seed, step, 3u, i, h, s);
      float total = kappa;
      for (int32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e)
        if ((al[col[e] / 32] >> (col[e] % 32)) & 1u) total = total + val[e];
      float t = u * total;
      float acc = kappa;
      int32_t pick = -1, last = 0;
      double lpick = log((double)kappa), llast = lpick;
      if (t < acc) {
        pick = 0;
      } else {
        for (int32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
          if (!((al[col[e] / 32] >> (col[e] % 32)) & 1u)) continue;
          acc = acc + val[e];
          last = col[e] + 1;
          llast = ln_val[e];
          if (t < acc) {
            pick = col[e] + 1;
            lpick = ln_val[e];
            break;
          }
        }
        if (pick < 0) {
          pick = last;
          lpick = llast;
        }
      }
      th[i] = pick;
      lw += lpick;
      if (pick > 0) detected[pick - 1] += 1;
    }
    for (int32_t j = 0; j < T; ++j) {
      if (!((al[j / 32] >> (j % 32)) & 1u)) continue;
      if (n_count > 0)
        lw += count_lp[detected[j] < n_count ? detected[j] : n_count - 1];
      else if (detected[j] == 0)
        lw += log(1.0 - (double)p_d);
    }
    logw[q] = lw;
    free(detected);
  }
}

/* O12 De-duplication, P:46 ("yielding a large set of new assignment
 * hypotheses from which only the unique hypotheses are retained"): within a
 * parent, sample s is unique iff no earlier sample s' < s has the same
 * surviving-track set and the same association map (R27). */
void oracle_dedup(int32_t H_old, int32_t H_up, int32_t M, const uint32_t *alive,
                  int64_t ldt, const int32_t *theta, int64_t ldm, uint8_t *unique) {
#pragma omp parallel for schedule(dynamic)
  for (int32_t h = 0; h < H_old; ++h) {
    for (int32_t s = 0; s < H_up; ++s) {
      int64_t q = (int64_t)h * H_up + s;
      int dup = 0;
      for (int32_t s2 = 0; s2 < s && !dup; ++s2) {
        int64_t q2 = (int64_t)h * H_up + s2;
        int same = 1;
        for (int64_t k = 0; k < ldt && same; ++k) same = alive[q * ldt + k] == alive[q2 * ldt + k];
        for (int32_t i = 0; i < M && same; ++i) same = theta[q * ldm + i] == theta[q2 * ldm + i];
        dup = same;
      }
      unique[q] = (uint8_t)!dup;
    }
  }
}

/* O13 Normalisation and pruning, P:53 (§Approach: "hypotheses with weights
 * below a predefined threshold tau are discarded. Finally, the H_max most
 * likely hypotheses are retained"): over the unique candidates,
 * w_c = exp(lw_c - max) / sum; keep w_c >= tau (the largest is always kept);
 * order by (w descending, index ascending); keep the first h_max; renormalise
 * the kept weights to sum 1 (R29).  Returns the kept count. */
int32_t oracle_prune(int32_t n, const double *logw, const uint8_t *unique, double tau,
                     int32_t h_max, int32_t *keep_idx, double *keep_w) {
  double m = -INFINITY;
  int32_t arg = -1;
  for (int32_t c = 0; c < n; ++c)
    if (unique[c] && logw[c] > m) { m = logw[c]; arg = c; }
  if (arg < 0 || h_max <= 0) return 0;
  double s = 0.0;
  for (int32_t c = 0; c < n; ++c)
    if (unique[c]) s += exp(logw[c] - m);
  int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  double *w = (double *)malloc(sizeof(double) * (size_t)n);
  int32_t k = 0;
  for (int32_t c = 0; c < n; ++c) {
    if (!unique[c]) continue;
    double wc = exp(logw[c] - m) / s;
    if (wc >= tau || c == arg) { idx[k] = c; w[k] = wc; ++k; }
  }
  /* insertion sort by (w desc, index asc) */
  for (int32_t a = 1; a < k; ++a) {
    int32_t ia = idx[a];
    double wa = w[a];
    int32_t b = a - 1;
    while (b >= 0 && (w[b] < wa || (w[b] == wa && idx[b] > ia))) {
      idx[b + 1] = idx[b]; w[b + 1] = w[b]; --b;
    }
    idx[b + 1] = ia; w[b + 1] = wa;
  }
  int32_t nk = k < h_max ? k : h_max;
  double sk = 0.0;
  for (int32_t a = 0; a < nk; ++a) sk += w[a];
  for (int32_t a = 0; a < nk; ++a) { keep_idx[a] = idx[a]; keep_w[a] = w[a] / sk; }
  free(idx);
  free(w);
  return nk;
}

/* ==================================================================
 * Particle loop after the hypothesis update: unique
 * (track, measurement-set) pairs, the batched per-pair Bayes update with its
 * effective sample size, and systematic resampling.  P:53 (§Approach).
 * ================================================================== */

/* O14 Unique association pairs, P:53 ("we perform a batched particle update
 * for all unique (track, measurement) association pairs generated across the
 * new set of hypotheses"), reading R30: for r = 0..n_hyp-1 (the given order,
 * e.g. the pruned ranking) and hypothesis q = hyp_idx[r], every track j
 * (ascending) alive in q gets the set S = {i : theta_q[i] = j+1} (ascending
 * i).  The pair (j, S) is numbered on its first occurrence in that scan;
 * pair_of[r][j] = its number, -1 for tracks not alive in q.
 * Outputs: pair_track [n_pairs], pair_ptr [n_pairs+1], pair_meas [nnz]
 * (capacities n_hyp*T and n_hyp*M suffice).  Returns n_pairs. */
int32_t oracle_assoc_pairs(int32_t n_hyp, const int32_t *hyp_idx, const uint32_t *alive,
                           int64_t ldt, const int32_t *theta, int64_t ldm, int32_t T,
                           int32_t M, int32_t *pair_track, int32_t *pair_ptr,
                           int32_t *pair_meas, int32_t *pair_of) {
  int32_t K = 0, nnz = 0;
  int32_t *S = (int32_t *)malloc(sizeof(int32_t) * (size_t)(M > 0 ? M : 1));
  pair_ptr[0] = 0;
  for (int32_t r = 0; r < n_hyp; ++r) {
    int64_t q = hyp_idx[r];
    const uint32_t *al = alive + q * ldt;
    const int32_t *th = theta + q * ldm;
    for (int32_t j = 0; j < T; ++j) {
      if (!((al[j / 32] >> (j % 32)) & 1u)) {
        pair_of[(int64_t)r * T + j] = -1;
        continue;
      }
      int32_t n = 0;
      for (int32_t i = 0; i < M; ++i)
        if (th[i] == j + 1) S[n++] = i;
      int32_t found = -1;
      for (int32_t k = 0; k < K && found < 0; ++k) {
        if (pair_track[k] != j || pair_ptr[k + 1] - pair_ptr[k] != n) continue;
        int same = 1;
        for (int32_t e = 0; e < n && same; ++e) same = pair_meas[pair_ptr[k] + e] == S[e];
        if (same) found = k;
      }
      if (found < 0) {
        found = K;
        pair_track[K] = j;
        for (int32_t e = 0; e < n; ++e) pair_meas[nnz + e] = S[e];
        nnz += n;
        pair_ptr[K + 1] = nnz;
        ++K;
      }
      pair_of[(int64_t)r * T + j] = found;
    }
  }
  free(S);
  return K;
}

/* O15 Batched particle update over pairs, P:53 ("The particle weights are
 * updated according to the measurement likelihood"): pair k updates the
 * particles of track pair_track[k] with its set S_k exactly as O8 does for
 * S_j (Bayes' rule, log normaliser, uniform reset + flag when every weight
 * is zero; S_k empty: weights copied, logZ = ln sum w), and reports the
 * effective sample size ESS_k = (sum_p w'_p)^2 / sum_p w'_p^2 of the new
 * weights (Kong-Liu; reading R31).  w_out [K][P] fp64. */
void oracle_reweight_pairs(int32_t P, int64_t ld, const float *x, const float *y,
                           const float *w, const float *Z, float Rxx, float Rxy, float Ryy,
                           int32_t K, const int32_t *pair_track, const int32_t *pair_ptr,
                           const int32_t *pair_meas, double *w_out, double *logZ,
                           uint32_t *flags, double *ess) {
#pragma omp parallel for schedule(dynamic)
  for (int32_t k = 0; k < K; ++k) {
    int64_t base = (int64_t)pair_track[k] * ld;
    double *wo = w_out + (int64_t)k * P;
    int32_t e0 = pair_ptr[k], e1 = pair_ptr[k + 1];
    flags[k] = 0u;
    if (e1 == e0) {
      double s = 0.0;
      for (int32_t p = 0; p < P; ++p) {
        wo[p] = (double)w[base + p];
        s += wo[p];
      }
      logZ[k] = log(s);
    } else {
      double *l = (double *)malloc(sizeof(double) * (size_t)P);
      double m = -INFINITY;
      for (int32_t p = 0; p < P; ++p) {
        double lp = log((double)w[base + p]);
        for (int32_t e = e0; e < e1; ++e) {
          int32_t i = pair_meas[e];
          lp += oracle_loggauss2(Z[2 * i], Z[2 * i + 1], x[base + p], y[base + p], Rxx, Rxy, Ryy);
        }
        l[p] = lp;
        if (lp > m) m = lp;
      }
      if (m == -INFINITY) {
        for (int32_t p = 0; p < P; ++p) wo[p] = 1.0 / (double)P;
        logZ[k] = -INFINITY;
        flags[k] = 1u;
      } else {
        double s = 0.0;
        for (int32_t p = 0; p < P; ++p) s += exp(l[p] - m);
        for (int32_t p = 0; p < P; ++p) wo[p] = exp(l[p] - m) / s;
        logZ[k] = m + log(s);
      }
      free(l);
    }
    double s1 = 0.0, s2 = 0.0;
    for (int32_t p = 0; p < P; ++p) {
      s1 += wo[p];
      s2 += wo[p] * wo[p];
    }
    ess[k] = s2 > 0.0 ? s1 * s1 / s2 : 0.0;
  }
}

/* O16 Systematic resampling of one weight vector, P:53 ("a resampling step
 * is performed if necessary to prevent particle degeneracy"), readings R31,
 * R32.  Weights are taken in units of 2^-26: W_m = floor(w_m 2^26) (exact
 * for fp32 w in [0, 1]), S = sum W, Q = sum W^2 (exact integers).
 *  - resample iff 2 S^2 < P Q, i.e. ESS = S^2/Q < P/2 (S = 0: no resample);
 *  - U = 2 (r >> 9) + 1 with r = word 0 of Philox4x32-10(key(seed),
 *    counter (k, 0, step, 4 << 24)) -- the same odd 24-bit integer as O3's
 *    uniform u = U 2^-24 -- and V = floor(U S / 2^24);
 *  - position n = 0..P-1: t_n = floor((n S + V) / P), the systematic grid
 *    (u + n)/P of the total mass; ancestor a_n = min{m : W_0 + ... + W_m > t_n}.
 * Returns 1 and fills anc [P] when it resamples, else returns 0 (anc
 * untouched).  Requires P <= 2^14 (so every product fits 64 bits). */
int oracle_resample(int32_t P, const float *w, uint64_t seed, uint32_t step, int32_t k,
                    int32_t *anc) {
  unsigned __int128 S = 0, Q = 0;
  uint64_t *W = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)P);
  for (int32_t m = 0; m < P; ++m) {
    W[m] = (uint64_t)floor((double)w[m] * 67108864.0);
    S += W[m];
    Q += (unsigned __int128)W[m] * W[m];
  }
  int res = S > 0 && 2 * S * S < (unsigned __int128)P * Q;
  if (res) {
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)k, 0u, step, 4u << 24};
    uint32_t r[4];
    oracle_philox4x32_10(ctr, key, r);
    uint64_t U = 2ull * (r[0] >> 9) + 1ull;
    uint64_t V = (uint64_t)((U * S) >> 24);
    for (int32_t n = 0; n < P; ++n) {
      uint64_t t = (uint64_t)(((unsigned __int128)n * S + V) / (unsigned)P);
      uint64_t cum = 0;
      int32_t a = P - 1;
      for (int32_t m = 0; m < P; ++m) {
        cum += W[m];
        if (cum > t) { a = m; break; }
      }
      anc[n] = a;
    }
  }
  free(W);
  return res;
}

/* ==================================================================
 * Closing the tracker loop: the kept hypotheses become
 * the next step's parents, and the MAP hypothesis gives the state estimate.
 * ================================================================== */

/* O17 Next parents, P:44 ("For each of the H_old hypotheses from the
 * previous timestep k-1, a new set of H_up hypotheses is generated") with
 * P:24 (births are superposed on every hypothesis), reading R33: kept
 * hypothesis r (< n_kept, in pruned order) becomes parent r of the next
 * step; its tracks are the pairs it uses, pair_of[r][j] >= 0 (their rows in
 * the new particle set, < K_cap), plus the B birth columns birth_col0 ..
 * birth_col0+B-1; its log-weight is ln keep_w[r]. */
void oracle_next_parents(int32_t n_kept, const double *keep_w, const int32_t *pair_of,
                         int32_t T, int32_t K_cap, int32_t B, int32_t birth_col0,
                         int64_t ldt, uint32_t *mask, double *logw) {
  for (int32_t r = 0; r < n_kept; ++r) {
    uint32_t *m = mask + (int64_t)r * ldt;
    for (int64_t k = 0; k < ldt; ++k) m[k] = 0u;
    for (int32_t j = 0; j < T; ++j) {
      int32_t k = pair_of[(int64_t)r * T + j];
      if (k >= 0 && k < K_cap) m[k / 32] |= 1u << (k % 32);
    }
    for (int32_t b = 0; b < B; ++b) {
      int32_t c = birth_col0 + b;
      m[c / 32] |= 1u << (c % 32);
    }
    logw[r] = log(keep_w[r]);
  }
}

/* O18 State estimate of the most likely hypothesis (reading R34): for every
 * track j alive in kept hypothesis 0 (pair_of row 0 >= 0), the weighted mean
 * position of its updated particles, sum_p w_p (x_p, y_p) / sum_p w_p, of row
 * pair_of[0][j] of the new particle set; est [T][3] = (x, y, 1), or
 * (NaN, NaN, 0) for tracks not in the hypothesis. */
void oracle_map_estimate(int32_t n_kept, const int32_t *pair_of0, int32_t T, int32_t P,
                         int64_t ld, const float *x, const float *y, const float *w,
                         double *est) {
  for (int32_t j = 0; j < T; ++j) {
    int32_t k = n_kept > 0 ? pair_of0[j] : -1;
    if (k < 0) {
      est[3 * j] = NAN; est[3 * j + 1] = NAN; est[3 * j + 2] = 0.0;
      continue;
    }
    double sw = 0.0, sx = 0.0, sy = 0.0;
    for (int32_t p = 0; p < P; ++p) {
      double wp = (double)w[(int64_t)k * ld + p];
      sw += wp;
      sx += wp * (double)x[(int64_t)k * ld + p];
      sy += wp * (double)y[(int64_t)k * ld + p];
    }
    est[3 * j] = sx / sw; est[3 * j + 1] = sy / sw; est[3 * j + 2] = 1.0;
  }
}
