/*
 * glmb.h -- C ABI of the B200-native GLMB step core (arXiv 2512.06230).
 *
 * The library (paper_2512_06230_b200/libglmb.so, sm_100a) implements the
 * data-parallel core of one step of the paper's particle GLMB tracker:
 *
 *   glmb_predict   CTRV survival propagation of every particle of every
 *                  surviving track, with Philox4x32-10 process noise
 *                  (§Approach "propagated forward using the
 *                  constant turn rate and velocity kinematics model ... a
 *                  batch operation over all particles and surviving tracks").
 *   glmb_birth     LMB birth sampling, P particles per new track from
 *                  N(mu_b, L_b L_b^T)  ("a set of particles is sampled
 *                  from the birth probability distribution for each new track").
 *   glmb_compat    the M_k x (T_k+1) compatibility matrix C_k with gate bits
 *                  (equation for C_k; P:37 gate g = [L >= gamma];
 *                  P:39 "the entire construction ... can be performed in
 *                  parallel").
 *   glmb_reweight  per-track particle reweighting under a supplied
 *                  association map theta_k (P:42 theta_k; "The particle
 *                  weights are updated according to the measurement likelihood").
 *
 * Readings of the paper where it is silent or ambiguous (P_D factor in C,
 * gate on L without P_D, kappa as an intensity, the CTRV noise terms, the
 * Philox keying, theta encoding) are listed in DESIGN.md ("Readings").
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Every pointer argument is a DEVICE pointer (cudaMalloc / torch CUDA
 *    memory) owned by the caller, unless the parameter name ends in _host.
 *    The library never allocates, frees or retains a pointer.
 *  - Calls validate their arguments, enqueue kernels on `stream` and return
 *    without synchronising (except glmb_step_host, which is synchronous).
 *    Launch failures return GLMB_ERR_CUDA; execution faults surface at the
 *    caller's next synchronisation.  No call ever aborts the process.
 *  - `stream` is a cudaStream_t (ABI-compatible typedef below).  A non-NULL
 *    stream selects the device; NULL means the legacy default stream of the
 *    calling thread's current device.
 *  - Particle arrays are SoA, track-major fp32: element (j, p) of each array
 *    is at j*ld + p.  Requirements: n_particles >= 4 and a multiple of 4,
 *    ld >= n_particles and a multiple of 4, every array 16-byte aligned
 *    (GLMB_ERR_ALIGNMENT otherwise).  Elements p in [n_particles, ld) are
 *    never read or written.
 *  - M == 0 gives a 0-row C (glmb_compat writes nothing); glmb_reweight
 *    with M == 0 leaves every weight untouched and writes log_norm = ln sum w.
 *    n_tracks == 0 is a no-op for predict/birth/reweight; glmb_compat with
 *    n_tracks == 0 writes only C_clutter (the clutter-only matrix).
 *  - Coordinates are metres in a local frame; |x|,|y| <= 1e4 m keeps the
 *    fp32 contract of DESIGN.md (fp32 resolution 1e-3 m at 1e4 m).
 *  - NaN inputs are not flagged: a NaN likelihood compares false against
 *    gamma, so g = 0 and C = 0 for that entry.
 */
#ifndef GLMB_H_
#define GLMB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *glmb_stream_t; /* == cudaStream_t */

typedef enum {
  GLMB_OK = 0,
  GLMB_ERR_INVALID_ARG = -1,        /* a size, parameter or null pointer violates the contract */
  GLMB_ERR_ALIGNMENT = -2,          /* an array is not 16-B aligned or ld/P not multiples of 4 */
  GLMB_ERR_UNSUPPORTED_DEVICE = -3, /* device is not compute capability 10.0 (sm_100a) */
  GLMB_ERR_CUDA = -4                /* a CUDA runtime call or kernel launch failed */
} glmb_status;

/* Particle set: T tracks x P particles, SoA fp32 [T][ld] per array.
 * Pointers may alias none of each other.  `w` are the particle weights
 * w_j^p of P:21 (used as supplied: compat does not renormalise them). */
typedef struct {
  float *x, *y, *v, *psi, *omega, *w;
  int32_t n_tracks;    /* T >= 0                                 */
  int32_t n_particles; /* P >= 4, P % 4 == 0                      */
  int64_t ld;          /* >= P, ld % 4 == 0                       */
} glmb_particles;

/* Library version (major*10000 + minor*100 + patch). */
int glmb_version(void);

/* Human-readable text of a status code (static storage, never NULL). */
const char *glmb_status_string(glmb_status s);

/* Checks that `device` is compute capability 10.0 and caches its SM count.
 * Optional: every other call performs the same check lazily.
 * Returns GLMB_ERR_UNSUPPORTED_DEVICE on any other device. */
glmb_status glmb_init(int device);

/* Number of streaming multiprocessors of `device` (0 on error). */
int glmb_sm_count(int device);

/* ---------------------------------------------------------------------
 * glmb_predict -- CTRV survival propagation (P:3, §Approach).
 *
 * For every track j < in->n_tracks and particle p < P:
 *   (n0, n1, n2, n3) = Box-Muller normals of Philox4x32-10(
 *        key = (lo32 seed, hi32 seed), counter = (p / 2, gid[j], step, 0))
 *   (na, nw) = (n0, n1) for even p, (n2, n3) for odd p
 *   nu_a = sigma_a * na,  nu_w = sigma_w * nw
 *   h = omega dt / 2
 *   x'     = x + v dt sinc(h) cos(psi + h) + 1/2 dt^2 cos(psi) nu_a
 *   y'     = y + v dt sinc(h) sin(psi + h) + 1/2 dt^2 sin(psi) nu_a
 *   v'     = v + dt nu_a
 *   psi'   = wrap(psi + omega dt + 1/2 dt^2 nu_w)   in (-pi, pi]
 *   omega' = omega + dt nu_w
 * (the half-angle form of the CTRV flow; identical to
 *  (v/omega)(sin(psi+omega dt) - sin psi) etc., stable as omega -> 0.)
 * Weights are not touched.  `out` may equal `in` (in place); otherwise
 * in/out must not overlap and must have the same n_tracks / n_particles.
 * gid: [n_tracks] int32 global track ids (the Philox key word; makes the
 * draws independent of sharding and column position).
 * Errors: INVALID_ARG if dt <= 0, sigma_a < 0, sigma_w < 0, shape mismatch,
 * or a NULL pointer with n_tracks > 0.
 * --------------------------------------------------------------------- */
glmb_status glmb_predict(const glmb_particles *in, const glmb_particles *out,
                         const int32_t *gid, float dt, float sigma_a,
                         float sigma_w, uint64_t seed, uint32_t step,
                         glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_birth -- LMB birth sampling (§Approach).
 *
 * For every birth track b < out->n_tracks and particle p < P:
 *   n0..n3 = Box-Muller normals of Philox(counter = (p, gid[b], step, 0x100))
 *   n4     = first normal of Philox(counter = (p, gid[b], step, 0x101))
 *   s = mean[b] + L_b n          (L_b = chol[b], packed row-major lower
 *                                 triangle: L00, L10 L11, L20 L21 L22, ...)
 *   (x, y, v, psi, omega) = (s0, s1, s2, wrap(s3), s4),  w = 1/P
 * `out` describes the B birth rows (typically the particle arrays offset to
 * row T, so births follow the survivors: C column T+b+1).
 * mean: [B][5] fp32, chol: [B][15] fp32, gid: [B] int32 (device).
 * Errors: INVALID_ARG on NULL pointers with B > 0.
 * --------------------------------------------------------------------- */
glmb_status glmb_birth(const glmb_particles *out, const int32_t *gid,
                       const float *mean, const float *chol, uint64_t seed,
                       uint32_t step, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_compat -- compatibility matrix C_k (§Approach).
 *
 *   L_ij = sum_p w_jp N(z_i; (x_jp, y_jp), R)         (H = [I2 0])
 *   g_ij = [L_ij >= gamma]                             (inclusive)
 *   C[i, j+1] = g_ij ? p_d * L_ij : 0
 *   C[i, 0]   = kappa                                  (clutter)
 * for i < M, j < trk->n_tracks.  The sum is the dense mixture over all P
 * particles (the gate is applied after L).
 *
 * Z: [M][2] fp32 measurements z_i (x, y).
 * R = [[Rxx, Rxy], [Rxy, Ryy]] must be SPD.
 * Outputs (column-major C, each column contiguous over measurements):
 *   C_clutter [M] fp32      = kappa (may be NULL: not written)
 *   C_tracks  [T][ldc] fp32, entry (j, i) = C[i, j+1]; ldc >= M.
 *             Entries i in [M, ldc) are not written.
 *   gate      [T][ldg] u32, bit (i % 32) of word (j, i / 32) = g_ij;
 *             ldg >= ceil(M/32); bits i >= M of the last word are 0;
 *             words >= ceil(M/32) are not written.
 * Results are bit-identical for any n_tracks split (sharding) and any row
 * permutation of Z (each entry is computed independently, in a fixed
 * particle order).
 * Precondition for the 1e-4 fp32 contract: weights in [0, 1]
 * (P:21's particle weights); terms below 2^-126 flush to zero.
 * Errors: INVALID_ARG if R is not SPD, p_d not in (0,1], kappa < 0,
 * gamma < 1e-30 (the fp32 exactness precondition), ldc < M,
 * ldg < ceil(M/32), or NULL outputs with T > 0 and M > 0.
 * --------------------------------------------------------------------- */
glmb_status glmb_compat(const glmb_particles *trk, const float *Z, int32_t M,
                        float Rxx, float Rxy, float Ryy, float p_d,
                        float kappa, float gamma, float *C_clutter,
                        float *C_tracks, int64_t ldc, uint32_t *gate,
                        int64_t ldg, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_compat_skipping -- glmb_compat with exact zero-tile skipping (opt-in;
 * an optimisation of a4/a5, not the method's definition): a warp skips a
 * particle tile when every one of its measurements lies >= 200 whitened
 * units^2 (q' = 1/2 log2(e) d^T R^-1 d >= 200) from the tile's bounding box.
 * Every skipped pair's contribution is exactly +0 on both exp paths
 * (2^-200 flushes to zero in fp32), so C, the gate words and C_clutter are
 * bit-identical to glmb_compat's.  skipped_pairs (DEVICE uint64, may be NULL):
 * incremented by the number of particle-measurement pairs skipped (for
 * reporting evaluated pairs; the caller zeroes it).  Arguments, layout and
 * errors as glmb_compat.  (GLMB_COMPAT_SKIP=1 in the environment makes
 * glmb_compat itself skip, for A/B runs.)
 * --------------------------------------------------------------------- */
glmb_status glmb_compat_skipping(const glmb_particles *trk, const float *Z,
                                 int32_t M, float Rxx, float Rxy, float Ryy,
                                 float p_d, float kappa, float gamma,
                                 float *C_clutter, float *C_tracks, int64_t ldc,
                                 uint32_t *gate, int64_t ldg,
                                 uint64_t *skipped_pairs, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_compat_peers -- glmb_compat fused with the all-gather of C_k's column
 * blocks across ranks: the epilogue stores column j of this
 * rank's tracks to row row0 + j of EVERY peer_C[r] [.][ldc] and its gate words
 * to row row0 + j of every peer_G[r] [.][ldg], r < n_peers, instead of a local
 * C_tracks / gate -- e.g. the peers' symmetric-memory buffers mapped over
 * NVLink, so the transfer overlaps the likelihood tile by tile and no
 * collective runs afterwards (the caller orders the ranks with a barrier
 * before reading the gathered C).  peer_C / peer_G: DEVICE arrays of n_peers
 * device pointers (1 <= n_peers <= 64).  Same arithmetic as glmb_compat, so
 * the gathered C is bit-identical to the single-GPU C.  C_clutter is written
 * locally (may be NULL).  Errors as glmb_compat, plus INVALID_ARG on bad
 * n_peers / row0 / NULL pointer arrays.
 * --------------------------------------------------------------------- */
glmb_status glmb_compat_peers(const glmb_particles *trk, const float *Z,
                              int32_t M, float Rxx, float Rxy, float Ryy,
                              float p_d, float kappa, float gamma,
                              float *C_clutter, float *const *peer_C,
                              uint32_t *const *peer_G, int32_t n_peers,
                              int64_t row0, int64_t ldc, int64_t ldg,
                              glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_reweight -- particle update under theta_k (§Approach).
 *
 * theta: [M] int32, theta[i] = 0 means clutter, c >= 1 means C column c
 * (values outside [0, col_offset + T] are ignored).  Local track j is C
 * column col_offset + j + 1 (col_offset = global index of local track 0).
 *   S_j = { i : theta[i] == col_offset + j + 1 }
 *   S_j empty: w unchanged, log_norm[j] = ln sum_p w_p, flags[j] = 0
 *   else:      l_p = ln w_p + sum_{i in S_j} ln N(z_i; (x_p, y_p), R)
 *              w'_p = exp(l_p - m) / sum_q exp(l_q - m),  m = max_p l_p
 *              log_norm[j] = m + ln sum_q exp(l_q - m)
 *              if every w_p == 0: w'_p = 1/P, log_norm = -inf, flags[j] = 1
 * The new weights go to w_out ([T][ld], 16-B aligned, same layout as w):
 * w_out == trk->w updates in place; a separate buffer leaves trk->w intact
 * (so glmb_compat may read it concurrently on another stream; tracks with
 * S_j empty are then copied).  log_norm: [T] fp32, flags: [T] u32 (bit 0 =
 * degenerate track reset to uniform).
 * Errors: INVALID_ARG if R is not SPD or a needed pointer is NULL;
 * ALIGNMENT if w_out is not 16-B aligned.
 * --------------------------------------------------------------------- */
glmb_status glmb_reweight(const glmb_particles *trk, float *w_out,
                          const float *Z, int32_t M, float Rxx, float Rxy, float Ryy,
                          const int32_t *theta, int32_t col_offset,
                          float *log_norm, uint32_t *flags,
                          glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * One whole step: predict (rows [0, n_survivors)) -> birth (rows
 * [n_survivors, tracks.n_tracks)) -> compat (all rows) -> reweight (all
 * rows), enqueued on `stream`.  Exactly the four calls above, in order.
 * --------------------------------------------------------------------- */
typedef struct {
  glmb_particles tracks;   /* T_k = T + B rows: survivors then births   */
  int32_t n_survivors;     /* T                                          */
  const int32_t *gid;      /* [T_k] global ids (device)                  */
  const float *birth_mean; /* [B][5] (device)                            */
  const float *birth_chol; /* [B][15] (device)                           */
  float dt, sigma_a, sigma_w;
  uint64_t seed;
  uint32_t step;
  float Rxx, Rxy, Ryy, p_d, kappa, gamma;
  int32_t col_offset;      /* global column offset of local row 0        */
  float *w_out;            /* NULL: reweight in place; else [T_k][ld] spare
                              weight buffer the new weights go to (the
                              caller swaps buffers after the step)       */
} glmb_step_params;

glmb_status glmb_step(const glmb_step_params *prm, const float *Z, int32_t M,
                      const int32_t *theta, float *C_clutter, float *C_tracks,
                      int64_t ldc, uint32_t *gate, int64_t ldg,
                      float *log_norm, uint32_t *flags, glmb_stream_t stream);

/* End-to-end step with HOST inputs and outputs (synchronous).
 * Copies Z_host [M][2] and theta_host [M] (pinned host memory recommended)
 * into the device workspaces Z_dev / theta_dev (capacity >= M), runs
 * glmb_step, copies C_clutter, C_tracks ([T_k][ldc]), gate ([T_k][ldg]),
 * log_norm and flags back into the *_host buffers, then synchronises
 * `stream`.  The particle state stays resident on the device.
 * copy_stream (may be NULL; needs a non-NULL `stream`): a second stream for
 * the read-back -- C_k's columns and gate words are copied back on
 * copy_stream while reweight runs (environment GLMB_HOST_CHUNKS = 2..4 also
 * splits compat into track chunks so the read-back overlaps compat; results
 * are identical either way: C is bit-identical under any split of the
 * tracks). */
glmb_status glmb_step_host(const glmb_step_params *prm, const float *Z_host,
                           int32_t M, const int32_t *theta_host, float *Z_dev,
                           int32_t *theta_dev, float *C_clutter_dev,
                           float *C_tracks_dev, int64_t ldc, uint32_t *gate_dev,
                           int64_t ldg, float *log_norm_dev,
                           uint32_t *flags_dev, float *C_clutter_host,
                           float *C_tracks_host, uint32_t *gate_host,
                           float *log_norm_host, uint32_t *flags_host,
                           glmb_stream_t stream, glmb_stream_t copy_stream);

/* End-to-end step returning C_k in its row-wise sparse form (synchronous): the
 * step of glmb_step_host, then glmb_compat_rows on the device, and a read-back
 * of the CSR of the gated entries -- row_ptr [M+1], col / val [nnz] (as
 * glmb_compat_rows defines them; C[i][0] = kappa and every other entry is 0)
 * -- plus log_norm and flags.  C_k is ~0.1 % dense at the BASELINE scenes, so
 * this moves kilobytes over PCIe instead of T_k x ldc floats.  cap: device
 * capacity of col/val/ln_val; cap_host: host capacity of col_host/val_host;
 * first_host: how many entries to copy speculatively with row_ptr (before nnz
 * is known on the host).  The first min(first_host, cap_host, cap) entries come
 * back with row_ptr; the rest (when nnz exceeds that) in a second exact-size
 * copy after one synchronisation.  With prm->w_out set and an
 * aux_stream (and a non-NULL stream), reweight runs on aux_stream beside
 * compat (out of place: the caller swaps weight buffers afterwards); else the
 * four calls run in order on `stream`.  Errors: INVALID_ARG when nnz exceeds
 * cap or cap_host (the device or host arrays are too small). */
glmb_status glmb_step_host_csr(const glmb_step_params *prm, const float *Z_host,
                               int32_t M, const int32_t *theta_host,
                               float *Z_dev, int32_t *theta_dev,
                               float *C_tracks_dev, int64_t ldc,
                               uint32_t *gate_dev, int64_t ldg,
                               float *log_norm_dev, uint32_t *flags_dev,
                               int32_t *row_ptr_dev, int32_t *col_dev,
                               float *val_dev, double *ln_val_dev, int32_t cap,
                               int32_t *row_ptr_host, int32_t *col_host,
                               float *val_host, int32_t cap_host,
                               int32_t first_host, float *log_norm_host,
                               uint32_t *flags_host, glmb_stream_t stream,
                               glmb_stream_t aux_stream);

/* =====================================================================
 * Hypothesis machinery: the consumers of C_k.
 * P:44-53 §Approach.  Readings R23-R29 in DESIGN.md §3.
 * ===================================================================== */

/* ---------------------------------------------------------------------
 * glmb_death_prob -- posterior death probability d_prob(x_j) (P:44:
 * "balancing its prior survival probability against the likelihood of it
 * being detected"; the formula is deferred to a citation -- reading R23):
 *   e_j = max_{i : g_ij} C[i, j+1] / (C[i, j+1] + kappa)   (0 if no gated i)
 *   d_j = (1 - P_S,j) / ((1 - P_S,j) + P_S,j ((1 - P_D) + P_D e_j)),
 *   d_j = 0 when P_S,j == 1.
 * C_tracks [T][ldc] fp32 and gate [T][ldg] u32 exactly as glmb_compat writes
 * them; p_s [T] fp32 prior survival probabilities; d_out [T] fp32 (computed
 * in fp64, rounded once).
 * Errors: INVALID_ARG on T < 0, M < 0, p_d not in (0,1], kappa < 0, ldc < M,
 * ldg < ceil(M/32), NULL pointers with T > 0.
 * --------------------------------------------------------------------- */
glmb_status glmb_death_prob(int32_t T, int32_t M, const float *C_tracks,
                            int64_t ldc, const uint32_t *gate, int64_t ldg,
                            float p_d, float kappa, const float *p_s,
                            float *d_out, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_compat_rows -- row-wise (CSR) copy of the gated entries of C_k: the
 * rows that the categorical of P:44 ("normalizing the corresponding row in
 * the modified matrix C'_k") is drawn from.
 *   row_ptr [M+1] int32: row i's entries are [row_ptr[i], row_ptr[i+1]);
 *           row_ptr[M] = nnz = number of set gate bits (always written,
 *           even when nnz > cap)
 *   col [cap] int32   track index j (C column j+1), ascending within a row
 *   val [cap] fp32    C[i, j+1] copied bit-exactly
 *   ln_val [cap] fp64 ln(val) (used by the hypothesis weight)
 * Entries past `cap` are not written: the caller checks row_ptr[M] <= cap
 * after the stream synchronises and re-runs with a larger cap otherwise.
 * Errors: INVALID_ARG on negative sizes, NULL row_ptr, NULL outputs with
 * cap > 0, or bad ldc / ldg.
 * --------------------------------------------------------------------- */
glmb_status glmb_compat_rows(int32_t T, int32_t M, const float *C_tracks,
                             int64_t ldc, const uint32_t *gate, int64_t ldg,
                             int32_t *row_ptr, int32_t *col, float *val,
                             double *ln_val, int32_t cap, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_assoc_sample -- the two-stage association sampler and the
 * successor hypothesis weight, for H_old parents x H_up samples.
 * Sample q = h*H_up + s of parent h:
 *  stage 1 ("a Bernoulli sampling step using d_prob to determine which
 *   tracks survive"): for every track j set in parent_mask[h],
 *   u = uniform24(word j%4 of Philox4x32-10(key(seed),
 *                 counter (j/4, h, step, 2<<24 | s)))
 *   alive_j = (u < 1.0f - d_prob[j])              (fp32 compare, R24/R25)
 *  stage 2 ("for each measurement i, an association is sampled from a
 *   categorical distribution defined by normalizing the corresponding row in
 *   the modified matrix C'_k"): u_i from counter (i/4, h, step, 3<<24 | s),
 *   word i%4; in fp32 with round-to-nearest adds in ascending column order,
 *   total = kappa + sum_{alive gated j} C[i, j+1], t = u_i * total, theta_i =
 *   the first column whose running sum (starting at kappa for column 0)
 *   exceeds t; if rounding leaves none, the last alive gated column (R26).
 *  weight ("multiplying its parent's weight with the joint likelihood of
 *   the sampled survival/death events and data associations", R28), fp64:
 *   logw = parent_logw[h] + sum_{j in parent} (alive ? ln P_S,j : ln(1-P_S,j))
 *        + sum_i ln C'[i, theta_i] + sum_{alive j} lc(n_j)
 *   (ln C'[i, 0] = ln kappa; ln C'[i, j+1] = ln_val of the CSR entry;
 *   n_j = #{i : theta_i = j+1}).  lc: with n_count == 0 (count_lp may be
 *   NULL) lc(0) = ln(1-P_D), lc(n >= 1) = 0; with n_count > 0 (device
 *   count_lp [n_count] fp64, T <= 32768) lc(n) = count_lp[min(n, n_count-1)]:
 *   the prior on the number of measurements per object that the independent
 *   proposal ignores and the importance weight restores.
 * Inputs: parent_mask [H_old][ldt] u32 (bit j%32 of word j/32: track j is in
 * parent h), ldt >= ceil(T/32), 1 <= ldt <= 12288; parent_logw [H_old] fp64;
 * d_prob, p_s [T] fp32; the CSR of glmb_compat_rows (row_ptr [M+1], col,
 * val, ln_val).
 * Outputs: alive [H_old*H_up][ldt] u32 (bits of dead / absent tracks 0);
 *   theta [H_old*H_up][ldm] int32 (0 = clutter, c >= 1 = C column c;
 *   entries [M, ldm) not written; ldm % 4 == 0, theta 16-B aligned);
 *   logw [H_old*H_up] fp64; hash [H_old*H_up] u64 (optional, may be NULL): a
 *   64-bit fingerprint of (alive, theta) consumed by glmb_dedup.
 * n_parents (device int32, may be NULL): only parents h < *n_parents are
 * sampled (the rest of the H_old slots are skipped; their outputs untouched).
 * Results do not depend on the launch configuration (bit-exact integers).
 * Errors: INVALID_ARG on negative sizes, H_up >= 2^24, H_old*H_up >= 2^31,
 * p_d not in (0,1], kappa < 0, bad ldt / ldm, NULL pointers;
 * ALIGNMENT on ldm % 4 != 0 or a misaligned theta.
 * --------------------------------------------------------------------- */
glmb_status glmb_assoc_sample(int32_t H_old, const int32_t *n_parents,
                              int32_t H_up, int32_t T, int32_t M,
                              const uint32_t *parent_mask, int32_t ldt,
                              const double *parent_logw, const float *d_prob,
                              const float *p_s, float p_d, float kappa,
                              const int32_t *row_ptr, const int32_t *col,
                              const float *val, const double *ln_val,
                              const double *count_lp, int32_t n_count,
                              uint64_t seed, uint32_t step, uint32_t *alive,
                              int32_t *theta, int64_t ldm, double *logw,
                              uint64_t *hash, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_dedup -- unique successors ("only the unique hypotheses are
 * retained", R27): unique[q] = 1 iff no earlier sample s2 < s of the same
 * parent has identical alive words (ldt) and theta entries (M); exact (the
 * fingerprints from glmb_assoc_sample only select the pairs compared).
 * n_parents (device int32, may be NULL): samples of parents h >= *n_parents
 * get unique = 0.
 * Errors: INVALID_ARG on negative sizes, ldt < 1, ldm < M, NULL pointers.
 * --------------------------------------------------------------------- */
glmb_status glmb_dedup(int32_t H_old, const int32_t *n_parents, int32_t H_up,
                       int32_t M,
                       const uint32_t *alive, int32_t ldt, const int32_t *theta,
                       int64_t ldm, const uint64_t *hash, uint8_t *unique,
                       glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_prune -- normalisation and pruning ("hypotheses with weights
 * below a predefined threshold tau are discarded. Finally, the H_max most
 * likely hypotheses are retained", R29), over the n candidates with
 * unique[c] != 0:
 *   w_c = exp(logw_c - max) / sum_c' exp(logw_c' - max)      (fp64)
 *   keep w_c >= tau (the first maximiser is always kept); order by
 *   (w desc, index asc); keep the first h_max; renormalise to sum 1.
 * Outputs: keep_idx [h_max] int32 (candidate indices), keep_w [h_max] fp64,
 * *n_kept (device int32) = the kept count k <= h_max (entries >= k untouched).
 * workspace: [n] u64 device scratch.
 * Errors: INVALID_ARG on n < 0, tau < 0 or NaN, h_max < 0 or
 * h_max > GLMB_PRUNE_HMAX_LIMIT, NULL pointers.
 * --------------------------------------------------------------------- */
#define GLMB_PRUNE_HMAX_LIMIT 16384
glmb_status glmb_prune(int32_t n, const double *logw, const uint8_t *unique,
                       double tau, int32_t h_max, uint64_t *workspace,
                       int32_t *keep_idx, double *keep_w, int32_t *n_kept,
                       glmb_stream_t stream);

/* =====================================================================
 * Particle loop: unique association pairs, the batched
 * per-pair particle update, systematic resampling.  P:53 §Approach.
 * Readings R30-R32 in DESIGN.md §3.
 * ===================================================================== */
#define GLMB_PAIRS_PMAX 16384 /* particles per track for reweight_pairs / resample */

/* ---------------------------------------------------------------------
 * glmb_assoc_pairs -- the unique (track, measurement set) pairs of P:53 ("a
 * batched particle update for all unique (track, measurement) association
 * pairs generated across the new set of hypotheses", R30).
 * For r = 0..n_hyp-1, hypothesis q = hyp_idx[r] (rows of the sampler's alive
 * [.][ldt] / theta [.][ldm] outputs, e.g. glmb_prune's keep_idx), every track
 * j < T alive in q has S = {i < M : theta_q[i] == j+1} (ascending).  Pairs
 * are numbered by first occurrence in (r, j) order:
 *   pair_track [K] int32, pair_ptr [K+1] int32 (pair k's measurements are
 *   pair_meas[pair_ptr[k] .. pair_ptr[k+1])), pair_of [n_hyp][T] int32 (the
 *   pair of (r, j), -1 if j is not alive in q), *n_pairs = K (device int32).
 * Capacities: pair_track n_hyp*T, pair_ptr n_hyp*T + 1, pair_meas n_hyp*M.
 * n_hyp_dev (device int32, may be NULL): use only the first min(n_hyp,
 * *n_hyp_dev) hypotheses (e.g. glmb_prune's n_kept) -- no host round trip;
 * pair_of rows past it are not written.
 * workspace: device scratch of glmb_assoc_pairs_workspace_size(n_hyp, T, M)
 * bytes.  Exact (fingerprints only preselect the compared lists).
 * Errors: INVALID_ARG on negative sizes, T > 17066, bad ldt / ldm, NULL
 * pointers, a short workspace.
 * --------------------------------------------------------------------- */
size_t glmb_assoc_pairs_workspace_size(int32_t n_hyp, int32_t T, int32_t M);
glmb_status glmb_assoc_pairs(int32_t n_hyp, const int32_t *n_hyp_dev,
                             const int32_t *hyp_idx,
                             const uint32_t *alive, int32_t ldt,
                             const int32_t *theta, int64_t ldm, int32_t T,
                             int32_t M, int32_t *pair_track, int32_t *pair_ptr,
                             int32_t *pair_meas, int32_t *pair_of,
                             int32_t *n_pairs, void *workspace,
                             size_t workspace_bytes, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_reweight_pairs -- the batched particle update over pairs: pair
 * k updates the particles of source track pair_track[k] with S_k exactly as
 * glmb_reweight does for S_j, writing row k of w_out ([K][ld_out] fp32),
 * log_norm[k], flags[k] (bit 0: all weights zero, reset to uniform) and
 * ess[k] = (sum w')^2 / sum w'^2 (fp32; R31).  S_k empty: weights copied.
 * K is the capacity (grid size); n_pairs (device int32, may be NULL) limits
 * the work to the first *n_pairs pairs, so the call can follow
 * glmb_assoc_pairs without a host round trip.  src->n_particles <=
 * GLMB_PAIRS_PMAX.
 * Errors: INVALID_ARG (R not SPD, NULL pointers, P too large);
 * ALIGNMENT (w_out, ld_out).
 * --------------------------------------------------------------------- */
glmb_status glmb_reweight_pairs(const glmb_particles *src, const float *Z,
                                int32_t M, float Rxx, float Rxy, float Ryy,
                                int32_t K, const int32_t *n_pairs,
                                const int32_t *pair_track,
                                const int32_t *pair_ptr,
                                const int32_t *pair_meas, float *w_out,
                                int64_t ld_out, float *log_norm,
                                uint32_t *flags, float *ess,
                                glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_resample -- systematic resampling "if necessary" (R31/R32).
 * For pair k (< K, and < *n_pairs if n_pairs != NULL), weights w[k][.]
 * (fp32 in [0, 1], stride ldw) are taken as integers W_m = floor(w_m 2^26);
 * S = sum W, Q = sum W^2 (exact).  If S > 0 and 2 S^2 < P Q (ESS < P/2):
 *   U = 2 (r >> 9) + 1, r = word 0 of Philox4x32-10(key(seed), counter
 *   (k, 0, step, 4 << 24)); V = floor(U S / 2^24);
 *   slot n < P takes ancestor a_n = min{m : W_0 + ... + W_m > floor((n S + V) / P)}
 *   out row k: (x, y, v, psi, omega) of src row pair_track[k] at a_n, w = 1/P;
 *   flags[k] |= 2.
 * Otherwise out row k = the source particles with weights w[k] (flags bit 1
 * cleared).  `out` describes >= K rows (a new particle set, one row per pair);
 * flags may be NULL.  P <= GLMB_PAIRS_PMAX.
 * Errors: INVALID_ARG / ALIGNMENT as for the other particle calls.
 * --------------------------------------------------------------------- */
glmb_status glmb_resample(const glmb_particles *src, int32_t K,
                          const int32_t *n_pairs, const int32_t *pair_track,
                          const float *w, int64_t ldw,
                          const glmb_particles *out, uint64_t seed,
                          uint32_t step, uint32_t *flags, glmb_stream_t stream);

/* =====================================================================
 * Tracker loop: the kept hypotheses become the next
 * step's parents; the most likely hypothesis gives the state estimate.
 * Readings R33, R34 in DESIGN.md §3.
 * ===================================================================== */

/* glmb_next_parents -- P:44 ("For each of the H_old hypotheses from the
 * previous timestep ...") with P:24 (births superposed on every hypothesis):
 * for r < *n_kept (the kept hypotheses in pruned order, as glmb_prune and
 * glmb_assoc_pairs leave them): parent_mask[r] ([ldt] u32 words) = bits of
 * the pairs pair_of[r][j] >= 0 with index < K_cap (their rows in the new
 * particle set) and of the birth columns birth_col0 .. birth_col0+B-1;
 * parent_logw[r] = ln keep_w[r]; *n_parents = min(*n_kept, n_hyp_cap).
 * birth_col0_dev (optional, device): when non-NULL the birth columns start at
 * min(*birth_col0_dev, K_cap) instead (e.g. glmb_assoc_pairs' *n_pairs, so
 * the call can be enqueued before the host reads the pair count).
 * Rows r >= *n_kept are not written.  All pointers device memory.
 * Errors: INVALID_ARG on negative sizes, K_cap or birth columns beyond
 * 32*ldt, ldt > 12288, NULL pointers. */
glmb_status glmb_next_parents(int32_t n_hyp_cap, const int32_t *n_kept,
                              const double *keep_w, const int32_t *pair_of,
                              int32_t T, int32_t K_cap, int32_t B,
                              int32_t birth_col0, uint32_t *parent_mask,
                              int32_t ldt, double *parent_logw,
                              int32_t *n_parents,
                              const int32_t *birth_col0_dev,
                              glmb_stream_t stream);

/* glmb_map_estimate -- the state estimate of the most likely hypothesis
 * (R34): for every old track j < T with 0 <= k = pair_of0[j] < set->n_tracks
 * (row 0 of glmb_assoc_pairs' pair_of, i.e. the best kept hypothesis; a pair
 * past the set's rows -- a K_cap overflow -- counts as none) and *n_kept > 0,
 * est[j] = (sum_p w_p x_p / sum_p w_p, ... y ..., 1) over row k of `set` (the
 * new particle set); otherwise est[j] = (NaN, NaN, 0).  est: [T][3] fp64,
 * sums in fp64.  Errors: INVALID_ARG on NULL pointers / bad particle set. */
glmb_status glmb_map_estimate(const int32_t *n_kept, const int32_t *pair_of0,
                              int32_t T, const glmb_particles *set, double *est,
                              glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * glmb_update -- the whole update after C_k in one call: the
 * work of glmb_death_prob -> glmb_compat_rows -> glmb_assoc_sample ->
 * glmb_dedup -> glmb_prune -> glmb_assoc_pairs -> glmb_reweight_pairs ->
 * glmb_resample (-> glmb_map_estimate when est != NULL), enqueued in that
 * order on `stream` with the counts passed between them on the device (no
 * host round trip); the death probabilities and the CSR row counts share one
 * grid (identical outputs).  Each field has the meaning, layout and
 * requirements of the same argument of those calls; the first failing call's
 * status is returned (earlier calls stay enqueued).
 * --------------------------------------------------------------------- */
typedef struct {
  /* sizes and model */
  int32_t T, M, H_old, H_up, h_max, K_cap;
  float p_d, kappa, Rxx, Rxy, Ryy;
  double tau;
  uint64_t seed;
  uint32_t step;
  /* inputs (device) */
  glmb_particles tracks;         /* the T_k predicted tracks (x, y, w read; all read by resample) */
  const float *C_tracks;         /* [T][ldc] as glmb_compat writes it */
  int64_t ldc;
  const uint32_t *gate;          /* [T][ldg] */
  int64_t ldg;
  const float *Z;                /* [M][2] */
  const float *p_s;              /* [T] */
  const uint32_t *parent_mask;   /* [H_old][ldt] */
  int32_t ldt;
  const double *parent_logw;     /* [H_old] */
  const int32_t *n_parents;      /* device count or NULL */
  const double *count_lp;        /* [n_count] or NULL */
  int32_t n_count;
  /* workspaces and outputs (device) */
  float *d_prob;                 /* [T] */
  int32_t *row_ptr, *col;        /* [M+1], [rows_cap] */
  float *val;                    /* [rows_cap] */
  double *ln_val;                /* [rows_cap] */
  int32_t rows_cap;
  uint32_t *alive;               /* [H_old*H_up][ldt] */
  int32_t *theta;                /* [H_old*H_up][ldm] */
  int64_t ldm;
  double *logw;                  /* [H_old*H_up] */
  uint64_t *hash;                /* [H_old*H_up] */
  uint8_t *unique;               /* [H_old*H_up] */
  uint64_t *prune_ws;            /* [H_old*H_up] */
  int32_t *keep_idx;             /* [h_max] */
  double *keep_w;                /* [h_max] */
  int32_t *n_kept;               /* device int32 */
  int32_t *pair_track, *pair_ptr, *pair_meas, *pair_of, *n_pairs;  /* as glmb_assoc_pairs (n_hyp = h_max) */
  void *pairs_ws;
  size_t pairs_ws_bytes;
  float *w_new;                  /* [K_cap][ld_new] */
  int64_t ld_new;
  float *log_norm;               /* [K_cap] */
  uint32_t *flags;               /* [K_cap] */
  float *ess;                    /* [K_cap] */
  glmb_particles out;            /* the new particle set, >= K_cap rows */
  double *est;                   /* [T][3] MAP estimate, or NULL */
} glmb_update_params;

glmb_status glmb_update(const glmb_update_params *u, glmb_stream_t stream);

/* ---------------------------------------------------------------------
 * Test hooks (not on the hot path; same device code as predict/birth).
 * glmb_philox_dump: out[n] = Philox4x32-10(key(seed), ctr[n]) for n < N.
 * glmb_normals_dump: out[n] = the four Box-Muller normals of that block
 * (words (0,1) -> out[n][0..1], words (2,3) -> out[n][2..3]).
 * ctr, out: [N][4] device arrays.
 * --------------------------------------------------------------------- */
glmb_status glmb_philox_dump(uint64_t seed, const uint32_t *ctr, int32_t N,
                             uint32_t *out, glmb_stream_t stream);
glmb_status glmb_normals_dump(uint64_t seed, const uint32_t *ctr, int32_t N,
                              float *out, glmb_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* GLMB_H_ */
