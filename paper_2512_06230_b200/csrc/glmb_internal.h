// glmb_internal.h -- launcher interfaces between the C ABI (abi.cu) and the
// kernel translation units.  Arguments are already validated by abi.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace glmb {

// Kernel launch with programmatic stream serialization (the hypothesis chain: each
// kernel starts with grid_dep_wait(), so its launch overlaps the previous kernel's
// tail).  GLMB_PDL=0 launches plainly (A/B runs).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct PredictArgs {
  const float *x, *y, *v, *psi, *omega;
  float *ox, *oy, *ov, *opsi, *oomega;
  const int32_t *gid;
  int32_t T, P;
  int64_t ld;
  float dt, sigma_a, sigma_w;
  uint32_t key0, key1, step;
};

struct BirthArgs {
  float *x, *y, *v, *psi, *omega, *w;
  const int32_t *gid;
  const float *mean, *chol;
  int32_t B, P;
  int64_t ld;
  uint32_t key0, key1, step;
};

// Whitened, centred measurement geometry for compat:
//   X' = a1 (x - cx) + a2 (y - cy),  Y' = b2 (y - cy)
// so that  1/2 log2(e) d^T R^-1 d = |(dX', dY')|^2  and  L = norm * sum w 2^-|d'|^2.
struct CompatArgs {
  const float *x, *y, *w;
  int64_t ld;
  int32_t T, P;
  const float *Z;
  int32_t M;
  float a1, a2, b2, norm;
  float p_d, kappa, gamma;
  float *C_clutter, *C_tracks;
  int64_t ldc;
  uint32_t *gate;
  int64_t ldg;
  int32_t n_mtiles;  // measurement tiles per track
  int32_t K;         // measurements per thread (tile = 32 * NW * K)
  int32_t NW;        // warps per CTA
  int32_t CL;        // CTAs (particle chunks) per (track, measurement tile): cluster size
  int32_t track_major;  // unit order: 1 = a track's measurement tiles adjacent, 0 = tile-major
  int32_t lo_slot;      // 1: a warp whose only valid slot is the pair's low one evaluates it alone
  // fused all-gather (glmb_compat_peers): n_peers > 0 writes column j to row peer_row0 + j of
  // every peer_C[r] / peer_G[r] (device arrays of n_peers pointers, e.g. symmetric memory
  // mapped over NVLink) instead of C_tracks / gate
  float *const *peer_C;
  uint32_t *const *peer_G;
  int32_t n_peers;
  int64_t peer_row0;
  // exact zero-tile skipping (opt-in: glmb_compat_skipping, or GLMB_COMPAT_SKIP=1 for
  // glmb_compat): skip = 1 selects the skipping kernel; skip_count (optional) is a device
  // counter of the particle-measurement pairs skipped because their contribution is exactly +0
  int32_t skip;
  unsigned long long *skip_count;
};

struct ReweightArgs {
  const float *x, *y;
  const float *w;  // weights read
  float *w_out;    // weights written (may equal w: in place)
  int64_t ld;
  int32_t T, P;
  const float *Z;
  int32_t M;
  const int32_t *theta;
  int32_t col_offset;
  double qa, qb, qc;   // q' = qa dx^2 + qb dx dy + qc dy^2 = 1/2 log2(e) d^T R^-1 d
  double log_norm1;    // ln(2 pi sqrt(det R))
  float *log_norm;
  uint32_t *flags;
  // pair mode (glmb_reweight_pairs): unit k updates source row pair_track[k] with
  // S_k = pair_meas[pair_ptr[k] .. pair_ptr[k+1]) and writes row k of w_out (stride
  // ld_out), log_norm[k], flags[k], ess[k].  theta mode: pair_track == nullptr,
  // unit j = row j, ld_out = ld, ess == nullptr.
  const int32_t *pair_track, *pair_ptr, *pair_meas;
  const int32_t *n_units_dev;  // optional device count of valid units (<= T)
  int64_t ld_out;
  float *ess;
  int32_t units_cap;  // pair mode: > 0 caps the grid at this many units, each cluster looping
                      // over units u, u + grid, ... < min(T, *n_units_dev) (T is a capacity there)
};

// ---- hypothesis machinery (hyp.cu)
struct DeathArgs {
  int32_t T, M;
  const float *C_tracks;
  int64_t ldc;
  const uint32_t *gate;
  int64_t ldg;
  float p_d, kappa;
  const float *p_s;
  float *d_out;
};

struct RowsArgs {
  int32_t T, M;
  const uint32_t *gate;
  int64_t ldg;
  const float *C_tracks;
  int64_t ldc;
  int32_t *row_ptr, *col;
  float *val;
  double *ln_val;
  int32_t cap;
};

struct SampleArgs {
  int32_t H_old, H_up, T, M;
  const int32_t *n_parents;  // optional device count (<= H_old) of valid parents
  const uint32_t *parent_mask;
  int32_t ldt;
  const double *parent_logw;
  const float *d_prob, *p_s;
  float p_d, kappa;
  const int32_t *row_ptr, *col;
  const float *val;
  const double *ln_val;
  const double *count_lp;  // optional per-track measurement-count log prior (n_count entries)
  int32_t n_count;
  uint32_t key0, key1, step;
  uint32_t *alive;
  int32_t *theta;
  int64_t ldm;
  double *logw;
  unsigned long long *hash;
  int32_t spc;      // set by the launcher: samples per CTA
  int32_t pool;     // set by the launcher: shared-memory bytes the kernel carves at run time
};

struct DedupArgs {
  int32_t H_old, H_up, M, ldt;
  const int32_t *n_parents;  // optional device count of valid parents (others: unique = 0)
  int64_t ldm;
  const uint32_t *alive;
  const int32_t *theta;
  const unsigned long long *hash;
  uint8_t *unique;
};

struct PruneArgs {
  int32_t n;
  const double *logw;
  const uint8_t *unique;
  double tau;
  int32_t h_max, cap2;
  unsigned long long *keys;  // workspace [n]
  int32_t *keep_idx;
  double *keep_w;
  int32_t *n_kept;
};

cudaError_t launch_predict(const PredictArgs &a, int sm_count, cudaStream_t s);
cudaError_t launch_birth(const BirthArgs &a, int sm_count, cudaStream_t s);
cudaError_t launch_philox_dump(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, uint32_t *out,
                               cudaStream_t s);
cudaError_t launch_normals_dump(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, float *out,
                                cudaStream_t s);
// chooses K / n_mtiles from (M, P) only (never from T: bit-identical sharding)
void compat_plan(int32_t M, int32_t P, int32_t *K, int32_t *NW, int32_t *CL, int32_t *n_mtiles);
cudaError_t launch_compat(const CompatArgs &a, cudaStream_t s);
bool compat_skip_env();
cudaError_t launch_clutter_fill(float *C_clutter, int32_t M, float kappa, cudaStream_t s);
cudaError_t launch_reweight(const ReweightArgs &a, cudaStream_t s);
cudaError_t launch_death_prob(const DeathArgs &a, cudaStream_t s);
cudaError_t launch_compat_rows(const RowsArgs &a, int sm_count, cudaStream_t s);
// glmb_update: death_prob and the CSR row counts in one grid, then the scan and the fill
cudaError_t launch_death_and_rows(const DeathArgs &d, const RowsArgs &a, int sm_count, cudaStream_t s);
cudaError_t launch_assoc_sample(const SampleArgs &a, int sm_count, cudaStream_t s);
cudaError_t launch_dedup(const DedupArgs &a, cudaStream_t s);
int32_t prune_capacity(int32_t h_max);
cudaError_t launch_prune(const PruneArgs &a, cudaStream_t s);

// ---- particle loop (pairs.cu)
struct PairsArgs {
  int32_t n_hyp, T, M, ldt;
  int64_t ldm;
  const int32_t *n_hyp_dev;  // optional device count (<= n_hyp) of hypotheses to use
  const int32_t *hyp_idx;
  const uint32_t *alive;
  const int32_t *theta;
  int32_t *pair_track, *pair_ptr, *pair_meas, *pair_of, *n_pairs;
  // workspace (n_hyp*T entries each, and n_hyp*M for the lists)
  int32_t *cnt, *off, *first, *list, *row_k, *row_m;
  unsigned long long *fp;
};
size_t pairs_workspace_bytes(int32_t n_hyp, int32_t T, int32_t M);
cudaError_t launch_assoc_pairs(const PairsArgs &a, void *ws, cudaStream_t s);

struct ResampleArgs {
  const float *x, *y, *v, *psi, *omega;  // source particles [.][ld]
  int64_t ld;
  int32_t P;
  const int32_t *pair_track;
  const float *w;                        // reweighted weights [K][ldw]
  int64_t ldw;
  int32_t K;
  const int32_t *n_units_dev;
  float *ox, *oy, *ov, *opsi, *oomega, *ow;  // output particles [K][ld_out]
  int64_t ld_out;
  uint32_t key0, key1, step;
  uint32_t *flags;                       // bit 1 set when unit k was resampled
};
cudaError_t launch_resample(const ResampleArgs &a, int sm_count, cudaStream_t s);

// ---- tracker loop (pairs.cu)
struct NextParentsArgs {
  int32_t n_hyp_cap;
  const int32_t *n_kept;
  const double *keep_w;
  const int32_t *pair_of;  // [n_hyp_cap][T]
  int32_t T, K_cap, B, birth_col0, ldt;
  uint32_t *parent_mask;   // [n_hyp_cap][ldt]
  double *parent_logw;
  int32_t *n_parents;
  const int32_t *birth_col0_dev;  // optional: birth columns start at min(*birth_col0_dev, K_cap)
};
cudaError_t launch_next_parents(const NextParentsArgs &a, cudaStream_t s);

struct MapEstimateArgs {
  const int32_t *n_kept, *pair_of0;
  int32_t T, P;
  int32_t n_rows;  // rows of the particle set: a pair index k >= n_rows is treated like k < 0
  int64_t ld;
  const float *x, *y, *w;
  double *est;  // [T][3]
};
cudaError_t launch_map_estimate(const MapEstimateArgs &a, cudaStream_t s);

}  // namespace glmb
