// hyp.cu -- the hypothesis machinery that consumes C_k (
// PAPER.md P:44-53 §Approach):
//
//   death_prob     d_j from the best gated entry of column j        (reading R23)
//   compat_rows    row-wise (CSR) copy of the gated entries of C_k   (the rows P:46 normalises)
//   assoc_sample   two-stage sampler: Bernoulli survival, then one categorical
//                  per measurement row of C'_k; log-weight of each sample
//   dedup          first occurrence of each (alive set, theta) within a parent
//   prune          normalise, drop w < tau, keep the H_max most likely
//
// Integer outcomes (alive bits, theta) are decided in fp32 exactly as the
// readings R25/R26 state, so they are bit-identical to any implementation that
// follows them; log-weights accumulate in fp64.
#include <algorithm>
#include <cstdlib>

#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr uint32_t kDomainSurvive = 2u, kDomainAssoc = 3u;

// ------------------------------------------------------------------ death probability
// One warp per track column: e_j = max over gated i of r_i = C[i, j+1] / (C[i, j+1] + kappa),
// then d_j = (1 - P_S) / ((1 - P_S) + P_S ((1 - P_D) + P_D e_j)).  fp64 with explicitly
// rounded operations (no FMA contraction): IEEE-exact steps, so d_j is reproducible.
__device__ __forceinline__ void death_prob_warp(const DeathArgs &a, const int32_t j, const int lane) {
  if (j >= a.T) return;
  const float *col = a.C_tracks + static_cast<int64_t>(j) * a.ldc;
  const uint32_t *g = a.gate + static_cast<int64_t>(j) * a.ldg;
  const double kappa = static_cast<double>(a.kappa);
  double e = 0.0;
  // the column's gate words are loaded 32 at a time (one per lane), then only the nonzero
  // ones are visited (broadcast by shuffle): one L2 round trip per 1024 rows instead of a
  // dependent load per 32 rows; the max does not depend on the visiting order
  const int32_t nw = (a.M + 31) >> 5;
  for (int32_t w0 = 0; w0 < nw; w0 += 32) {
    const uint32_t mine = w0 + lane < nw ? __ldg(g + w0 + lane) : 0u;
    for (uint32_t nz = __ballot_sync(0xffffffffu, mine != 0u); nz != 0u; nz &= nz - 1u) {
      const int src = __ffs(nz) - 1;
      const uint32_t word = __shfl_sync(0xffffffffu, mine, src);
      const int32_t i = 32 * (w0 + src) + lane;
      if (i < a.M && ((word >> lane) & 1u)) {
        const double c = static_cast<double>(__ldg(col + i));
        e = fmax(e, __ddiv_rn(c, __dadd_rn(c, kappa)));
      }
    }
  }
  e = warp_max_d(e);
  if (lane == 0) {
    const double ps = static_cast<double>(__ldg(a.p_s + j)), pd = static_cast<double>(a.p_d);
    const double dead = __dsub_rn(1.0, ps);
    const double detect = __dadd_rn(__dsub_rn(1.0, pd), __dmul_rn(pd, e));
    a.d_out[j] = ps == 1.0 ? 0.0f : __double2float_rn(__ddiv_rn(dead, __dadd_rn(dead, __dmul_rn(ps, detect))));
  }
}

__global__ void __launch_bounds__(256) death_prob_kernel(DeathArgs a) {
  grid_dep_wait();
  death_prob_warp(a, blockIdx.x * 8 + (threadIdx.x >> 5), threadIdx.x & 31);
}

// ------------------------------------------------------------------ CSR of the gated entries
// CTA (w, c) = 32 consecutive rows (gate word column w) x the c-th of gridDim.y track
// chunks; warp k owns the contiguous sub-chunk k of it, so entries come out in
// ascending j.  Splitting the tracks over CTAs spreads the fill (and its fp64 logs)
// over the GPU: with a few word columns (M ~ 100) one CTA per column ran on 4 SMs.
constexpr int kRowWarps = 32;

__device__ __forceinline__ void range_part(int32_t lo, int32_t hi, int parts, int k, int32_t &j0, int32_t &j1) {
  const int32_t ch = (hi - lo + parts - 1) / parts;
  j0 = min(hi, lo + k * ch);
  j1 = min(hi, j0 + ch);
}


// row totals: each CTA adds its chunk's counts (row_ptr zeroed by the launcher)
__device__ __forceinline__ void rows_count_block(const RowsArgs &a, const int w, const int chunk, const int n_chunks) {
  __shared__ int32_t cnt[kRowWarps][32];
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  int32_t c0, c1, j0, j1;
  range_part(0, a.T, n_chunks, chunk, c0, c1);
  range_part(c0, c1, kRowWarps, k, j0, j1);
  int32_t c = 0;
  for (int32_t j = j0; j < j1; ++j) c += (__ldg(a.gate + static_cast<int64_t>(j) * a.ldg + w) >> lane) & 1u;
  cnt[k][lane] = c;
  __syncthreads();
  if (k == 0) {
    int32_t s = 0;
#pragma unroll
    for (int q = 0; q < kRowWarps; ++q) s += cnt[q][lane];
    const int32_t i = w * 32 + lane;
    if (i < a.M) {
      if (n_chunks == 1) a.row_ptr[i] = s;
      else if (s) atomicAdd(a.row_ptr + i, s);
    }
  }
}

__global__ void __launch_bounds__(kRowWarps * 32) rows_count_kernel(RowsArgs a) {
  grid_dep_wait();
  rows_count_block(a, blockIdx.x, blockIdx.y, gridDim.y);
}

// glmb_update's first launch: death probabilities (a warp per column, the first
// n_death_blocks CTAs) and the CSR row counts (the rest) read the same C_k and gate words
// and write disjoint outputs, so one grid does both
__global__ void __launch_bounds__(kRowWarps * 32) death_and_count_kernel(DeathArgs d, RowsArgs r, int n_death_blocks,
                                                                         int words, int n_chunks) {
  grid_dep_wait();
  if (static_cast<int>(blockIdx.x) < n_death_blocks) {
    death_prob_warp(d, static_cast<int32_t>(blockIdx.x) * kRowWarps + (threadIdx.x >> 5), threadIdx.x & 31);
    return;
  }
  const int b = static_cast<int>(blockIdx.x) - n_death_blocks;
  rows_count_block(r, b % words, b / words, n_chunks);
}

// exclusive scan of row_ptr[0..M) in place, row_ptr[M] = total (one CTA)
__global__ void __launch_bounds__(1024) rows_scan_kernel(int32_t *row_ptr, int32_t M) {
  grid_dep_wait();
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int32_t base = 0; base < M; base += 1024) {
    const int32_t i = base + threadIdx.x;
    const int32_t v = i < M ? row_ptr[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int32_t s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;  // inclusive warp-total prefix
    }
    __syncthreads();
    const int32_t carry = carry_s;
    const int32_t excl = carry + (wid ? wsum[wid - 1] : 0) + x - v;
    if (i < M) row_ptr[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) row_ptr[M] = carry_s;
}

__global__ void __launch_bounds__(kRowWarps * 32) rows_fill_kernel(RowsArgs a) {
  grid_dep_wait();
  __shared__ int32_t cnt[kRowWarps][32];
  __shared__ int32_t pre[kRowWarps][32];
  const int w = blockIdx.x, lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  int32_t c0, c1, j0, j1;
  range_part(0, a.T, gridDim.y, blockIdx.y, c0, c1);
  range_part(c0, c1, kRowWarps, k, j0, j1);
  // entries of this row in the tracks before the CTA's chunk (warp-strided count)
  int32_t p = 0;
  for (int32_t j = k; j < c0; j += kRowWarps) p += (__ldg(a.gate + static_cast<int64_t>(j) * a.ldg + w) >> lane) & 1u;
  int32_t c = 0;
  for (int32_t j = j0; j < j1; ++j) c += (__ldg(a.gate + static_cast<int64_t>(j) * a.ldg + w) >> lane) & 1u;
  cnt[k][lane] = c;
  pre[k][lane] = p;
  __syncthreads();
  const int32_t i = w * 32 + lane;
  if (i >= a.M) return;
  int32_t pos = a.row_ptr[i];
  for (int q = 0; q < kRowWarps; ++q) pos += pre[q][lane];
  for (int q = 0; q < k; ++q) pos += cnt[q][lane];
  for (int32_t j = j0; j < j1; ++j) {
    if ((__ldg(a.gate + static_cast<int64_t>(j) * a.ldg + w) >> lane) & 1u) {
      if (pos < a.cap) {
        const float v = __ldg(a.C_tracks + static_cast<int64_t>(j) * a.ldc + i);
        a.col[pos] = j;
        a.val[pos] = v;
        a.ln_val[pos] = log(static_cast<double>(v));
      }
      ++pos;
    }
  }
}

// ------------------------------------------------------------------ two-stage sampler
// CTA = (parent h, group of 32 samples): LANE l of every warp is sample s = 32 g + l, and
// the warps split the work items -- stage 1 the parent's track words, stage 2 the row
// quads holding a parent entry.  Every lane of a warp thus walks the same track quad or
// the same row at the same time (uniform control flow, the row's entries read from shared
// memory as broadcasts); only the uniforms, and hence the alive bits and picks, differ
// per lane.  The samples' alive / detected sets live in shared memory as [word][lane].
#ifndef GLMB_SAMP_DEBUG
#define GLMB_SAMP_DEBUG 0  // A/B timing builds only: 1 skips stage 1's Philox, 2 skips stage 2, 3 stamps phases
                           // (16 %globaltimer slots per CTA in the fingerprint output: profiles/sampler_phases.py)
#endif
#ifndef GLMB_SAMP_WARPS
#define GLMB_SAMP_WARPS 16
#endif
#ifndef GLMB_SAMP_BLOCKS
#define GLMB_SAMP_BLOCKS 3
#endif
constexpr int kSampWarps = GLMB_SAMP_WARPS;
constexpr int kSampThreads = 32 * kSampWarps;

// one fingerprint term (summed mod 2^64 over a sample's detected rows and alive words):
// any deterministic function works -- dedup compares the words exactly when two
// fingerprints agree -- so one multiply-xorshift round stands in for a full finaliser
__device__ __forceinline__ uint64_t fp_term(uint32_t v, uint64_t idx) {
  uint64_t z = ((idx << 32) | v) * 0xBF58476D1CE4E5B9ull;
  return z ^ (z >> 31);
}

// Block-wide exclusive scan of one int32 per thread (kSampThreads threads).
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t *red, int32_t &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[wid] = x;
  __syncthreads();
  int32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kSampWarps; ++w) {
    const int32_t r = red[w];
    before += w < wid ? r : 0;
    tot += r;
  }
  total = tot;
  __syncthreads();
  return before + x - v;
}

// Once per CTA: the parent's rows of C'_k -- the gated entries whose column is in the
// parent, in ascending column order -- are filtered into shared memory (when they fit,
// else the CTA walks the global CSR), the parent's track words are listed, and the row
// quads holding a parent entry are listed with the mask of their non-empty rows.  The
// other rows draw theta_i = 0 with ln kappa whatever their uniform (see draw_row) and are
// stored as zeros.  Same draws and the same fp32 operation order as a walk of the full
// rows (columns outside the parent are never alive), so the integer outcomes do not
// depend on any of this.
constexpr int kFilterBatch = 8;  // CSR words (32 entries) a warp loads per round of the row filter

__device__ __forceinline__ uint32_t word_of(const u32x4 &r, int e) {
  return e == 0 ? r.a : e == 1 ? r.b : e == 2 ? r.c : r.d;
}

// Row i's categorical draw for this lane's sample (R26): clutter kappa, then the
// alive gated columns in ascending order; inverse CDF in fp32 with the word's 24-bit
// uniform.  The entries are the same for every lane (broadcast reads); the walk visits
// all of them without an early exit, so the control flow stays uniform across the warp.
// Adds the picked entry's ln value to lw and returns theta_i (0 = clutter).  An empty
// row draws the clutter entry whatever u is.  al_of(j): bit j of this lane's alive set.
template <class AliveOf>
__device__ __forceinline__ int32_t draw_row(const int32_t *rp, const int32_t *cl, const float *vl,
                                            const double *lvl, const AliveOf &al_of, float kappa,
                                            double ln_kappa, int32_t i, uint32_t word, double &lw) {
  const int32_t e0 = rp[i], e1 = rp[i + 1];
  // the row is the same for every lane of the warp, so the entry count -- and every
  // branch on it below -- is warp-uniform
  if (e1 - e0 == 1) {
    // one gated parent entry (most rows): the walk reduces to pick = j + 1 iff track j is
    // alive and u (kappa + C) does not fall below kappa
    const int32_t j = cl[e0];
    const bool al = al_of(j);
    const float tot = al ? __fadd_rn(kappa, vl[e0]) : kappa;
    const bool hit = al && !(__fmul_rn(uniform24(word), tot) < kappa);
    lw += hit ? lvl[e0] : ln_kappa;
    return hit ? j + 1 : 0;
  }
  float total = kappa;
  for (int32_t x = e0; x < e1; ++x)
    if (al_of(cl[x])) total = __fadd_rn(total, vl[x]);
  const float tt = __fmul_rn(uniform24(word), total);
  // pick = the first alive column whose running sum (from kappa) exceeds tt; if rounding
  // leaves none although tt >= kappa, the last alive column; tt < kappa: clutter
  int32_t pick = 0, last = 0;
  double lpick = ln_kappa, llast = ln_kappa;
  bool found = !(tt >= kappa);
  float acc = kappa;
  for (int32_t x = e0; x < e1; ++x) {
    const int32_t j = cl[x];
    if (!al_of(j)) continue;
    acc = __fadd_rn(acc, vl[x]);
    last = j + 1;
    llast = lvl[x];
    if (!found && tt < acc) {
      pick = j + 1;
      lpick = llast;
      found = true;
    }
  }
  if (!found) {
    pick = last;
    lpick = llast;
  }
  lw += lpick;
  return pick;
}

__global__ void __launch_bounds__(kSampThreads, GLMB_SAMP_BLOCKS) assoc_sample_kernel(SampleArgs a) {
  grid_dep_wait();
  extern __shared__ __align__(16) unsigned char smraw[];
  // a.pool bytes at the front (the kept-entry bitmap, then the parent's rows), carved
  // at run time; fixed arrays after it
  unsigned char *pool = smraw;
  double *slc = reinterpret_cast<double *>(smraw + a.pool);            // [n_count] count prior
  double *red_lw = slc + max(a.n_count, 0);                             // [kSampWarps][32]
  unsigned long long *red_fp = reinterpret_cast<unsigned long long *>(red_lw + 32 * kSampWarps);  // [W][32]
  int32_t *red_ms = reinterpret_cast<int32_t *>(red_fp + 32 * kSampWarps);  // [W][32]
  const int32_t tw = (a.T + 31) >> 5;                                   // track words in use (<= ldt)
  uint32_t *alive = reinterpret_cast<uint32_t *>(red_ms + 32 * kSampWarps);  // [tw][32]
  uint32_t *det = alive + 32 * tw;                                      // [tw][32]
  // count prior: per (track, lane) counts packed 4 x u8 per word when M < 256 (a count never
  // exceeds M), else 2 x u16 -- [(T + per - 1) / per][32]
  const int cbits = a.M < 256 ? 8 : 16, cper = 32 / cbits;
  const uint32_t cmask = (1u << cbits) - 1u;
  const int32_t cwords = a.n_count > 0 ? (a.T + cper - 1) / cper : 0;
  uint32_t *cnt = det + 32 * tw;
  int32_t *frp = reinterpret_cast<int32_t *>(cnt + 32 * cwords);        // [M + 1]
  int32_t *nzq = frp + a.M + 1;                                         // [(M + 3) / 4]
  int32_t *pw = nzq + ((a.M + 3) >> 2);                                 // [ldt] parent words
  uint32_t *pmask = reinterpret_cast<uint32_t *>(pw + a.ldt);           // [ldt]
  int32_t *kthr = reinterpret_cast<int32_t *>(pmask + a.ldt);          // [T] survival thresholds
  __shared__ int32_t red_i[kSampWarps];
  __shared__ int32_t use_smem, n_pw, n_nzq, n_nzr;
  const int n_groups = (a.H_up + 31) >> 5;
  const int32_t h = static_cast<int32_t>(blockIdx.x / n_groups);
  const int32_t g = static_cast<int32_t>(blockIdx.x - static_cast<int64_t>(h) * n_groups);
  if (a.n_parents != nullptr && h >= __ldg(a.n_parents)) return;  // inactive parent slot
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t s = 32 * g + lane;          // this lane's sample
#if GLMB_SAMP_DEBUG == 3   // A/B timing build: %globaltimer per CTA phase into the fingerprint output
  auto stamp = [&](int k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.hash[16 * blockIdx.x + k] = t;
    }
  };
  stamp(0);
#else
  auto stamp = [](int) {};
#endif
  const bool valid = s < a.H_up;
  const uint32_t* pm = a.parent_mask + static_cast<int64_t>(h) * a.ldt;
  for (int32_t k = threadIdx.x; k < a.ldt; k += kSampThreads) pmask[k] = __ldg(pm + k);
  for (int32_t k = threadIdx.x; k < a.n_count; k += kSampThreads) slc[k] = __ldg(a.count_lp + k);
  // R25's fp32 decision u < 1 - d_j as an integer compare: u = k 2^-24 with k = 2 (r >> 9) + 1
  // exact, and (1 - d_j) 2^24 is exact too, so u < 1 - d_j  <=>  k < ceil((1 - d_j) 2^24)
  for (int32_t j = threadIdx.x; j < a.T; j += kSampThreads) {
    const float thr = __fsub_rn(1.0f, __ldg(a.d_prob + j));
    const float t = thr * 16777216.0f;
    kthr[j] = !(thr == thr) ? 0 : t <= 0.0f ? 0 : t >= 16777218.0f ? 16777218 : static_cast<int32_t>(ceilf(t));
  }
  for (int32_t k = threadIdx.x; k < 32 * tw; k += kSampThreads) {
    alive[k] = 0u;
    det[k] = 0u;
  }
  if (a.n_count > 0)
    for (int32_t k = threadIdx.x; k < 32 * cwords; k += kSampThreads) cnt[k] = 0u;
  __syncthreads();
  stamp(10);
  auto in_parent = [&](int32_t j) { return ((pmask[j >> 5] >> (j & 31)) & 1u) != 0u; };

  // ---- the parent's rows (pool), filtered in ascending column order.  A stable
  // compaction of the CSR's entry stream: a bitmap of the kept entries (coalesced, one
  // ballot per 32 entries) and its word prefix K give row i's start K(row_ptr[i]) and
  // entry x's slot K(x).  Rows too many for the bitmap: a count and a fill pass per row.
  const int32_t r0 = __ldg(a.row_ptr), r1 = __ldg(a.row_ptr + a.M);
  const int32_t nwords = (r1 - r0 + 31) >> 5;
  const int64_t avail = a.pool;
  size_t rows_at = 0;  // pool offset of the filtered rows
  int32_t kept = 0;
  if (8 * static_cast<int64_t>(nwords) <= avail / 2) {
    uint32_t *kb = reinterpret_cast<uint32_t *>(pool);
    int32_t *kbp = reinterpret_cast<int32_t *>(kb + nwords);
    // a warp takes kFilterBatch consecutive words per round, all loads issued first
    for (int32_t w0 = wid * kFilterBatch; w0 < nwords; w0 += kSampWarps * kFilterBatch) {
      int32_t jj[kFilterBatch];
#pragma unroll
      for (int u = 0; u < kFilterBatch; ++u) {
        const int32_t x = r0 + 32 * (w0 + u) + lane;
        jj[u] = x < r1 ? __ldg(a.col + x) : -1;
      }
#pragma unroll
      for (int u = 0; u < kFilterBatch; ++u) {
        const uint32_t word = __ballot_sync(0xffffffffu, jj[u] >= 0 && in_parent(jj[u]));
        if (lane == 0 && w0 + u < nwords) kb[w0 + u] = word;
      }
    }
    __syncthreads();
    stamp(11);
    for (int32_t w0 = 0; w0 < nwords; w0 += kSampThreads) {
      const int32_t w = w0 + threadIdx.x;
      int32_t tot;
      const int32_t ex = block_excl_scan(w < nwords ? __popc(kb[w]) : 0, red_i, tot);
      if (w < nwords) kbp[w] = kept + ex;
      kept += tot;
    }
    __syncthreads();
    stamp(12);
    const int32_t total = kept;
    auto K = [&](int32_t x) -> int32_t {
      const int32_t d = x - r0, w = d >> 5;
      return w < nwords ? kbp[w] + __popc(kb[w] & ((1u << (d & 31)) - 1u)) : total;
    };
    for (int32_t i = threadIdx.x; i <= a.M; i += kSampThreads) frp[i] = K(__ldg(a.row_ptr + i));
    rows_at = static_cast<size_t>(8) * nwords;
    if (static_cast<int64_t>(rows_at + 16 * static_cast<size_t>(kept)) <= avail) {
      double *flv = reinterpret_cast<double *>(pool + rows_at);
      float *fval = reinterpret_cast<float *>(flv + kept);
      int32_t *fcol = reinterpret_cast<int32_t *>(fval + kept);
      for (int32_t w = wid; w < nwords; w += kSampWarps) {
        const uint32_t word = kb[w];
        if (!((word >> lane) & 1u)) continue;
        const int32_t x = r0 + 32 * w + lane;
        const int32_t o = kbp[w] + __popc(word & ((1u << lane) - 1u));
        fcol[o] = __ldg(a.col + x);
        fval[o] = __ldg(a.val + x);
        flv[o] = __ldg(a.ln_val + x);
      }
    }
  } else {
    for (int32_t i0 = 0; i0 < a.M; i0 += kSampThreads) {
      const int32_t i = i0 + threadIdx.x;
      int32_t c = 0;
      if (i < a.M) {
        const int32_t e1 = __ldg(a.row_ptr + i + 1);
        for (int32_t x = __ldg(a.row_ptr + i); x < e1; ++x) c += in_parent(__ldg(a.col + x));
      }
      int32_t tot;
      const int32_t ex = block_excl_scan(c, red_i, tot);
      if (i < a.M) frp[i] = kept + ex;
      kept += tot;
    }
    if (threadIdx.x == 0) frp[a.M] = kept;
    __syncthreads();
    if (static_cast<int64_t>(16 * static_cast<size_t>(kept)) <= avail) {
      double *flv = reinterpret_cast<double *>(pool);
      float *fval = reinterpret_cast<float *>(flv + kept);
      int32_t *fcol = reinterpret_cast<int32_t *>(fval + kept);
      for (int32_t i = threadIdx.x; i < a.M; i += kSampThreads) {
        int32_t o = frp[i];
        const int32_t e1 = __ldg(a.row_ptr + i + 1);
        for (int32_t x = __ldg(a.row_ptr + i); x < e1; ++x) {
          const int32_t j = __ldg(a.col + x);
          if (in_parent(j)) {
            fcol[o] = j;
            fval[o] = __ldg(a.val + x);
            flv[o] = __ldg(a.ln_val + x);
            ++o;
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) use_smem = static_cast<int64_t>(rows_at + 16 * static_cast<size_t>(kept)) <= avail;
  __syncthreads();
  stamp(13);

  const bool sm_rows = use_smem;
  const double *flv = reinterpret_cast<const double *>(pool + rows_at);
  const float *fval = reinterpret_cast<const float *>(flv + kept);
  const int32_t *fcol = reinterpret_cast<const int32_t *>(fval + kept);
  const int32_t *rp = sm_rows ? frp : a.row_ptr;
  const int32_t *cl = sm_rows ? fcol : a.col;
  const float *vl = sm_rows ? fval : a.val;
  const double *lvl = sm_rows ? flv : a.ln_val;
  const double ln_kappa = log(static_cast<double>(a.kappa));
  const double ln_miss = log(1.0 - static_cast<double>(a.p_d));
  const int32_t rquads = (a.M + 3) >> 2;
  // ---- the parent's track words (ascending) and the row quads holding a parent entry
  // (quad << 4 | mask of its non-empty rows)
  {
    int32_t cw = 0;
    for (int32_t w0 = 0; w0 < tw; w0 += kSampThreads) {
      const int32_t w = w0 + threadIdx.x;
      const bool any = w < tw && pmask[w] != 0u;
      int32_t tot;
      const int32_t ex = block_excl_scan(any, red_i, tot);
      if (any) pw[cw + ex] = w;
      cw += tot;
    }
    int32_t cq = 0, cr = 0;
    for (int32_t t0 = 0; t0 < rquads; t0 += kSampThreads) {
      const int32_t t = t0 + threadIdx.x;
      uint32_t mask = 0u;
      if (t < rquads) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int32_t i = 4 * t + e;
          if (i < a.M && rp[i + 1] > rp[i]) mask |= 1u << e;
        }
      }
      int32_t tq, tr;
      const int32_t exq = block_excl_scan(mask != 0u, red_i, tq);
      const int32_t exr = block_excl_scan(__popc(mask), red_i, tr);
      (void)exr;
      if (mask != 0u) nzq[cq + exq] = static_cast<int32_t>((static_cast<uint32_t>(t) << 4) | mask);
      cq += tq;
      cr += tr;
    }
    if (threadIdx.x == 0) {
      n_pw = cw;
      n_nzq = cq;
      n_nzr = cr;
    }
  }
  stamp(14);
  // ---- theta rows of the CTA's samples zero-filled (coalesced); stage 2 stores the picks
  const bool vec_store = ((a.ldm & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.theta) & 15) == 0);
  const int32_t n_s = min(32, a.H_up - 32 * g);
  {
    int32_t *th0 = a.theta + (static_cast<int64_t>(h) * a.H_up + 32 * g) * a.ldm;
    for (int32_t ss = wid; ss < n_s; ss += kSampWarps) {   // a warp per sample row
      int32_t *th = th0 + static_cast<int64_t>(ss) * a.ldm;
      if (vec_store) {
        for (int32_t t = lane; t < rquads; t += 32) {
          if (4 * t + 3 < a.M) *reinterpret_cast<int4 *>(th + 4 * t) = make_int4(0, 0, 0, 0);
          else for (int32_t i = 4 * t; i < a.M; ++i) th[i] = 0;
        }
      } else {
        for (int32_t i = lane; i < a.M; i += 32) th[i] = 0;
      }
    }
  }
  __syncthreads();
  const int32_t npw = n_pw, nzq_n = n_nzq, nzr_n = n_nzr;
  stamp(1);

  // ---- stage 1: track j of the parent survives iff u_j < 1 - d_j (fp32, R25);
  // Philox block (j/4, h, step, 2<<24 | s), word j%4.  A warp per parent word (8 quads):
  // the word's alive bits of every lane's sample are stored once, no atomics.
  double lw = 0.0;
  float memo_ps = -1.0f;              // P_S of the memoised logs (none yet)
  double memo_ls = 0.0, memo_ld = 0.0;
  int32_t n_al = 0, n_dd = 0;
  for (int32_t v = wid; v < npw; v += kSampWarps) {
    const int32_t w = pw[v];
    const uint32_t pbits = pmask[w];
    uint32_t abits = 0u;
    for (int32_t qq = 0; qq < 8; ++qq) {
      const uint32_t qbits = (pbits >> (4 * qq)) & 0xFu;
      if (qbits == 0u) continue;
      const int32_t t = 8 * w + qq;
#if GLMB_SAMP_DEBUG == 1
      const u32x4 r{0u, 0u, 0u, 0u};
#else
      const u32x4 r = philox4x32_10(
          u32x4{static_cast<uint32_t>(t), static_cast<uint32_t>(h), a.step, (kDomainSurvive << 24) | static_cast<uint32_t>(s)},
          a.key0, a.key1);
#endif
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!((qbits >> e) & 1u)) continue;
        const int32_t j = 4 * t + e;
        const bool al = static_cast<int32_t>(((word_of(r, e) >> 9) << 1) | 1u) < kthr[j];
        const float ps = __ldg(a.p_s + j);
        if (ps != memo_ps) {  // tracks mostly share a few P_S values: logs memoised (warp-uniform),
          lw += static_cast<double>(n_al) * memo_ls + static_cast<double>(n_dd) * memo_ld;
          n_al = n_dd = 0;    // the survival terms counted per memo and folded in when it changes
          memo_ps = ps;
          memo_ls = log(static_cast<double>(ps));
          memo_ld = log(1.0 - static_cast<double>(ps));
        }
        n_al += al;
        n_dd += !al;
        abits |= static_cast<uint32_t>(al) << (4 * qq + e);
      }
    }
    alive[32 * w + lane] = abits;
  }
  lw += static_cast<double>(n_al) * memo_ls + static_cast<double>(n_dd) * memo_ld;
  __syncthreads();   // every sample's alive set is complete
  stamp(2);

  // ---- stage 2: each row i draws theta_i from the row of C'_k (clutter kappa,
  // surviving gated columns in ascending order), inverse CDF in fp32 (R26);
  // Philox block (i/4, h, step, 3<<24 | s), word i%4.  A warp per non-empty row quad.
  uint64_t fp = 0ull;
  auto al_of = [&](int32_t j) { return ((alive[32 * (j >> 5) + lane] >> (j & 31)) & 1u) != 0u; };
  int32_t *th = a.theta + (static_cast<int64_t>(h) * a.H_up + s) * a.ldm;
#if GLMB_SAMP_DEBUG == 2
  if (nzq_n > 0 && a.M < 0)
#endif
  for (int32_t v = wid; v < nzq_n; v += kSampWarps) {
    const uint32_t ent = static_cast<uint32_t>(nzq[v]);
    const int32_t t = static_cast<int32_t>(ent >> 4);
    const u32x4 r = philox4x32_10(u32x4{static_cast<uint32_t>(t), static_cast<uint32_t>(h), a.step,
                                        (kDomainAssoc << 24) | static_cast<uint32_t>(s)},
                                  a.key0, a.key1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (!((ent >> e) & 1u)) continue;
      const int32_t i = 4 * t + e;
      const int32_t pick = draw_row(rp, cl, vl, lvl, al_of, a.kappa, ln_kappa, i, word_of(r, e), lw);
      if (pick > 0) {
        atomicOr(det + 32 * ((pick - 1) >> 5) + lane, 1u << ((pick - 1) & 31));
        if (a.n_count > 0) atomicAdd(cnt + 32 * ((pick - 1) / cper) + lane, 1u << (cbits * ((pick - 1) % cper)));
        // fingerprint over the detected rows only (theta is 0 elsewhere)
        fp += fp_term(static_cast<uint32_t>(pick), static_cast<uint64_t>(a.ldt) + i);
        if (valid) th[i] = pick;
      }
    }
  }
  __syncthreads();   // det / cnt complete
  stamp(3);

  // ---- missed detections (alive tracks with no measurement) or, with a count prior,
  // lc(n_j) for every alive track; fingerprint of the alive words; alive words out
  int32_t missed = 0;
  uint32_t *al_out = a.alive + (static_cast<int64_t>(h) * a.H_up + s) * a.ldt;
  for (int32_t k = wid; k < a.ldt; k += kSampWarps) {
    const uint32_t av = k < tw ? alive[32 * k + lane] : 0u;   // words past the tracks: 0
    if (valid) al_out[k] = av;
    fp += fp_term(av, static_cast<uint64_t>(k));
    if (a.n_count == 0) {
      if (k < tw) missed += __popc(av & ~det[32 * k + lane]);
    } else {
      for (uint32_t rest = av; rest != 0u; rest &= rest - 1u) {
        const int32_t j = 32 * k + __ffs(rest) - 1;
        const uint32_t n = (cnt[32 * (j / cper) + lane] >> (cbits * (j % cper))) & cmask;
        lw += slc[min(static_cast<int32_t>(n), a.n_count - 1)];
      }
    }
  }
  red_lw[32 * wid + lane] = lw;
  red_fp[32 * wid + lane] = static_cast<unsigned long long>(fp);
  red_ms[32 * wid + lane] = missed;
  __syncthreads();
  if (wid == 0 && valid) {
    double lws = 0.0;
    unsigned long long fps = 0ull;
    int32_t ms = 0;
#pragma unroll
    for (int w = 0; w < kSampWarps; ++w) {
      lws += red_lw[32 * w + lane];
      fps += red_fp[32 * w + lane];
      ms += red_ms[32 * w + lane];
    }
    // rows without a parent entry: theta_i = 0 with ln kappa each
    const int32_t n_empty = a.M - nzr_n;
    const double l_empty = n_empty > 0 ? static_cast<double>(n_empty) * ln_kappa : 0.0;
    const int64_t q = static_cast<int64_t>(h) * a.H_up + s;
    a.logw[q] = __ldg(a.parent_logw + h) + (lws + l_empty) + static_cast<double>(ms) * ln_miss;
#if GLMB_SAMP_DEBUG != 3
    if (a.hash) a.hash[q] = fps;
#endif
  }
  stamp(4);
}

// ------------------------------------------------------------------ dedup
// One CTA per parent: sample s is a duplicate iff some s2 < s of the same parent
// has the same fingerprint and the same (alive, theta) words.  Per chunk of 256
// samples: each thread finds its sample's first earlier sample with an equal
// fingerprint (hashes tiled through shared memory), the warps then compare those
// pairs word by word (coalesced), and only a fingerprint collision (equal hash,
// different sample) sends its thread on to the later candidates.
constexpr int kDedupThreads = 256, kDedupTile = 2048;

__device__ bool same_sample(const DedupArgs &a, int64_t q1, int64_t q2) {
  const uint32_t *A1 = a.alive + q1 * a.ldt, *A2 = a.alive + q2 * a.ldt;
  for (int32_t k = 0; k < a.ldt; ++k)
    if (A1[k] != A2[k]) return false;
  const int32_t *T1 = a.theta + q1 * a.ldm, *T2 = a.theta + q2 * a.ldm;
  for (int32_t i = 0; i < a.M; ++i)
    if (T1[i] != T2[i]) return false;
  return true;
}

__global__ void __launch_bounds__(kDedupThreads) dedup_kernel(DedupArgs a) {
  grid_dep_wait();
  __shared__ unsigned long long hs[kDedupTile];
  __shared__ int32_t cand[kDedupThreads];
  __shared__ uint8_t same[kDedupThreads];
  const int32_t h = blockIdx.x;
  const int64_t base = static_cast<int64_t>(h) * a.H_up;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (a.n_parents != nullptr && h >= __ldg(a.n_parents)) {  // inactive parent slot: no candidates
    for (int32_t s = threadIdx.x; s < a.H_up; s += kDedupThreads) a.unique[base + s] = 0;
    return;
  }
  for (int32_t s0 = 0; s0 < a.H_up; s0 += kDedupThreads) {
    const int32_t s = s0 + threadIdx.x;
    const unsigned long long mine = s < a.H_up ? a.hash[base + s] : 0ull;
    int32_t c = -1;
    const int32_t s_hi = min(a.H_up, s0 + kDedupThreads);  // largest s of this chunk + 1
    for (int32_t t0 = 0; t0 < s_hi; t0 += kDedupTile) {
      __syncthreads();
      for (int32_t k = threadIdx.x; k < kDedupTile && t0 + k < s_hi; k += kDedupThreads) hs[k] = a.hash[base + t0 + k];
      __syncthreads();
      if (s < a.H_up && c < 0) {
        const int32_t lim = min(kDedupTile, s - t0);
        for (int32_t k = 0; k < lim; ++k) {
          if (hs[k] == mine) {
            c = t0 + k;
            break;
          }
        }
      }
    }
    cand[threadIdx.x] = s < a.H_up ? c : -1;
    __syncthreads();
    for (int r = wid; r < kDedupThreads; r += kDedupThreads / 32) {
      const int32_t k = cand[r];
      if (k < 0) continue;
      const int64_t q1 = base + s0 + r, q2 = base + k;
      const uint32_t *A1 = a.alive + q1 * a.ldt, *A2 = a.alive + q2 * a.ldt;
      const int32_t *T1 = a.theta + q1 * a.ldm, *T2 = a.theta + q2 * a.ldm;
      bool diff = false;
      for (int32_t w = lane; w < a.ldt; w += 32) diff |= A1[w] != A2[w];
      for (int32_t i = lane; i < a.M; i += 32) diff |= T1[i] != T2[i];
      const bool any = __any_sync(0xffffffffu, diff);
      if (lane == 0) same[r] = !any;
    }
    __syncthreads();
    if (s < a.H_up) {
      bool dup = false;
      if (c >= 0) {
        dup = same[threadIdx.x];
        for (int32_t k = c + 1; !dup && k < s; ++k)  // fingerprint collision: later candidates
          dup = a.hash[base + k] == mine && same_sample(a, base + s, base + k);
      }
      a.unique[base + s] = dup ? 0 : 1;
    }
  }
}

// ------------------------------------------------------------------ prune
// One CTA.  Keys: candidate c gets key = bits(w_c) + 1 (w_c >= 0, so the IEEE
// bit pattern orders like the value), 0 otherwise.  The H_max largest keys are
// found by an MSB-first radix select; ties at the threshold are taken in index
// order; the kept set is bitonic-sorted by (w desc, index asc) in shared memory.
constexpr int kPruneThreads = 1024;

struct MaxArg {
  double v;
  int32_t i;
};
__device__ __forceinline__ MaxArg better(MaxArg x, MaxArg y) {
  if (y.i < 0) return x;
  if (x.i < 0) return y;
  if (y.v > x.v || (y.v == x.v && y.i < x.i)) return y;
  return x;
}

__global__ void __launch_bounds__(kPruneThreads) prune_kernel(PruneArgs a) {
  grid_dep_wait();
  extern __shared__ unsigned char psm[];
  unsigned long long *skey = reinterpret_cast<unsigned long long *>(psm);  // [cap2]
  int32_t *sidx = reinterpret_cast<int32_t *>(skey + a.cap2);              // [cap2]
  __shared__ double sd[32];
  __shared__ int32_t si[32];
  __shared__ uint32_t hist[256];
  __shared__ unsigned long long prefix_s;
  __shared__ int32_t need_s, done_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t n = a.n;

  // (1) max / first argmax over unique candidates
  MaxArg m{-INFINITY, -1};
  for (int32_t c = threadIdx.x; c < n; c += kPruneThreads)
    if (a.unique[c]) m = better(m, MaxArg{a.logw[c], c});
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MaxArg y{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
    m = better(m, y);
  }
  if (lane == 0) { sd[wid] = m.v; si[wid] = m.i; }
  __syncthreads();
  if (wid == 0) {
    m = MaxArg{sd[lane], si[lane]};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      MaxArg y{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
      m = better(m, y);
    }
    if (lane == 0) { sd[0] = m.v; si[0] = m.i; }
  }
  __syncthreads();
  const double mx = sd[0];
  const int32_t arg = si[0];
  __syncthreads();
  if (arg < 0 || a.h_max <= 0) {
    if (threadIdx.x == 0) *a.n_kept = 0;
    return;
  }
  // (2) s = sum exp(lw - max), fixed order
  // (the exponentials are parked in the key buffer for (3))
  double acc = 0.0;
  for (int32_t c = threadIdx.x; c < n; c += kPruneThreads) {
    const double e = a.unique[c] ? exp(a.logw[c] - mx) : 0.0;
    a.keys[c] = static_cast<unsigned long long>(__double_as_longlong(e));
    acc += e;
  }
  acc = warp_sum_d(acc);
  if (lane == 0) sd[wid] = acc;
  __syncthreads();
  if (wid == 0) {
    acc = warp_sum_d(sd[lane]);
    if (lane == 0) sd[0] = acc;
  }
  __syncthreads();
  const double ssum = sd[0];
  // (3) keys
  int32_t cnt = 0;
  for (int32_t c = threadIdx.x; c < n; c += kPruneThreads) {
    unsigned long long key = 0ull;
    if (a.unique[c]) {
      const double w = __longlong_as_double(static_cast<long long>(a.keys[c])) / ssum;
      if (w >= a.tau || c == arg) key = static_cast<unsigned long long>(__double_as_longlong(w)) + 1ull;
    }
    a.keys[c] = key;
    cnt += key != 0ull;
  }
  __syncthreads();
  // total candidates
  {
    int32_t v = cnt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) si[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t t = 0;
      for (int q = 0; q < 32; ++q) t += si[q];
      need_s = t;
    }
    __syncthreads();
  }
  const int32_t K = need_s;
  const int32_t nk = min(K, a.h_max);
  // (4) radix select of the nk-th largest key (threshold thr: keep key > thr, plus
  //     the first `ties` keys == thr in index order)
  unsigned long long thr = 1ull;  // K <= h_max: keep every key >= 1
  int32_t ties = 0;
  bool select = K > a.h_max;
  if (select) {
    if (threadIdx.x == 0) { prefix_s = 0ull; need_s = a.h_max; done_s = 0; }
    __syncthreads();
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int b = threadIdx.x; b < 256; b += kPruneThreads) hist[b] = 0u;
      __syncthreads();
      const unsigned long long pre = prefix_s;
      const unsigned long long hmask = shift == 56 ? 0ull : (~0ull << (shift + 8));
      for (int32_t c = threadIdx.x; c < n; c += kPruneThreads) {
        const unsigned long long key = a.keys[c];
        if ((key & hmask) == pre) atomicAdd(&hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // warp 0: the largest bin b whose count reaches the remaining need
        const int l = threadIdx.x;
        const int32_t need = need_s;
        int32_t hb[8], sl = 0;  // lane l holds bins 255 - 8l - k, k = 0..7 (descending)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          hb[k] = static_cast<int32_t>(hist[255 - 8 * l - k]);
          sl += hb[k];
        }
        int32_t incl = sl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
          if (l >= o) incl += y;
        }
        const uint32_t hit = __ballot_sync(0xffffffffu, incl >= need);
        const int L = hit ? __ffs(hit) - 1 : 31;
        if (l == L) {
          int32_t above = incl - sl;  // bins above this lane's first bin
          int b = 255 - 8 * l - 7;
          int32_t rem = need - above;
          int32_t hbb = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (hb[k] >= need - above) {
              b = 255 - 8 * l - k;
              rem = need - above;
              hbb = hb[k];
              break;
            }
            above += hb[k];
            rem = need - above;
          }
          const unsigned long long pb = pre | (static_cast<unsigned long long>(b) << shift);
          if (hbb == rem && shift > 0) {
            // the whole bin is kept: every key >= pb (its lowest possible value) and none
            // below -- threshold pb - 1 with no ties, the remaining digits need no pass
            need_s = 0;
            prefix_s = pb - 1ull;
            done_s = 1;
          } else {
            need_s = rem;
            prefix_s = pb;
          }
        }
      }
      __syncthreads();
      if (done_s) break;
    }
    thr = prefix_s;
    ties = need_s;  // how many keys == thr to keep
    __syncthreads();
  }
  // (5) compaction in index order: kept = key > thr (select) or key >= thr (no select),
  // plus the first `ties` keys == thr.  Slot = (# gt before) + min(# ties before, ties);
  // both counts from one per-warp round (packed in 16-bit halves), scanned by every warp.
  {
    int32_t carry_gt = 0, carry_tie = 0;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int32_t base = 0; base < n; base += kPruneThreads) {
      const int32_t c = base + threadIdx.x;
      const unsigned long long key = c < n ? a.keys[c] : 0ull;
      const bool gt = select ? key > thr : key >= thr;
      const bool tie = select && key == thr;
      const uint32_t gtb = __ballot_sync(0xffffffffu, gt), tb = __ballot_sync(0xffffffffu, tie);
      if (lane == 0) si[wid] = __popc(gtb) | (__popc(tb) << 16);
      __syncthreads();
      const int32_t v = si[lane];
      int32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const int32_t before = __shfl_sync(0xffffffffu, incl - v, wid);
      const int32_t gt_before = carry_gt + (before & 0xffff) + __popc(gtb & lt_mask);
      const int32_t tie_before = carry_tie + (before >> 16) + __popc(tb & lt_mask);
      const bool keep = gt || (tie && tie_before < ties);
      const int32_t pos = gt_before + min(tie_before, ties);
      if (keep && pos < a.cap2) {
        skey[pos] = key;
        sidx[pos] = c;
      }
      carry_gt += total & 0xffff;
      carry_tie += total >> 16;
      __syncthreads();
    }
  }
  // pad to cap2 with sentinels (key 0 sorts last)
  for (int32_t p = nk + threadIdx.x; p < a.cap2; p += kPruneThreads) {
    skey[p] = 0ull;
    sidx[p] = 0x7fffffff;
  }
  __syncthreads();
  // (6) bitonic sort, descending by key, ascending by index
  for (int32_t size = 2; size <= a.cap2; size <<= 1) {
    for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int32_t p = threadIdx.x; p < a.cap2; p += kPruneThreads) {
        const int32_t o = p ^ stride;
        if (o > p) {
          const bool desc = (p & size) == 0;
          const unsigned long long k1 = skey[p], k2 = skey[o];
          const int32_t i1 = sidx[p], i2 = sidx[o];
          // "p before o" in the target order (key desc, idx asc)
          const bool before = k1 > k2 || (k1 == k2 && i1 < i2);
          if (before != desc) {
            skey[p] = k2; skey[o] = k1;
            sidx[p] = i2; sidx[o] = i1;
          }
        }
      }
      __syncthreads();
    }
  }
  // (7) renormalise the kept weights
  double ws = 0.0;
  for (int32_t p = threadIdx.x; p < nk; p += kPruneThreads)
    ws += __longlong_as_double(static_cast<long long>(skey[p] - 1ull));
  ws = warp_sum_d(ws);
  if (lane == 0) sd[wid] = ws;
  __syncthreads();
  if (wid == 0) {
    ws = warp_sum_d(sd[lane]);
    if (lane == 0) sd[0] = ws;
  }
  __syncthreads();
  const double wsum = sd[0];
  for (int32_t p = threadIdx.x; p < nk; p += kPruneThreads) {
    a.keep_idx[p] = sidx[p];
    a.keep_w[p] = __longlong_as_double(static_cast<long long>(skey[p] - 1ull)) / wsum;
  }
  if (threadIdx.x == 0) *a.n_kept = nk;
}

}  // namespace

cudaError_t launch_death_prob(const DeathArgs &a, cudaStream_t s) {
  cudaError_t e0 = launch_pdl(death_prob_kernel, dim3((a.T + 7) / 8), dim3(256), 0, s, a);
  if (e0 != cudaSuccess) return e0;
  return cudaGetLastError();
}

cudaError_t launch_death_and_rows(const DeathArgs &d, const RowsArgs &a, int sm_count, cudaStream_t s) {
  const int32_t words = (a.M + 31) / 32;
  const int sms = sm_count > 0 ? sm_count : 148;
  const int32_t chunks = std::max<int32_t>(1, std::min<int32_t>((sms + words - 1) / std::max<int32_t>(words, 1),
                                                                (a.T + 63) / 64));
  if (a.M > 0 && (chunks > 1 || a.T == 0)) {
    cudaError_t e = cudaMemsetAsync(a.row_ptr, 0, sizeof(int32_t) * a.M, s);
    if (e != cudaSuccess) return e;
  }
  const int n_death = (d.T + kRowWarps - 1) / kRowWarps;
  const int n_count = (a.T > 0 && words > 0) ? words * chunks : 0;
  cudaError_t e = cudaSuccess;
  if (n_death + n_count > 0)
    e = launch_pdl(death_and_count_kernel, dim3(n_death + n_count), dim3(kRowWarps * 32), 0, s, d, a, n_death,
                   std::max<int32_t>(words, 1), chunks);
  if (e == cudaSuccess) e = launch_pdl(rows_scan_kernel, dim3(1), dim3(1024), 0, s, a.row_ptr, a.M);
  if (e == cudaSuccess && n_count > 0)
    e = launch_pdl(rows_fill_kernel, dim3(words, chunks), dim3(kRowWarps * 32), 0, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_compat_rows(const RowsArgs &a, int sm_count, cudaStream_t s) {
  const int32_t words = (a.M + 31) / 32;
  // track chunks per word column: ~1 CTA per SM in all, >= 64 tracks per chunk
  const int sms = sm_count > 0 ? sm_count : 148;
  const int32_t chunks = std::max<int32_t>(1, std::min<int32_t>((sms + words - 1) / std::max<int32_t>(words, 1),
                                                                (a.T + 63) / 64));
  if (a.M > 0 && (chunks > 1 || a.T == 0)) {  // chunked counts accumulate atomically
    cudaError_t e = cudaMemsetAsync(a.row_ptr, 0, sizeof(int32_t) * a.M, s);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid(static_cast<unsigned>(words), static_cast<unsigned>(chunks));
  cudaError_t e = cudaSuccess;
  if (a.T > 0 && words > 0) e = launch_pdl(rows_count_kernel, grid, dim3(kRowWarps * 32), 0, s, a);
  if (e == cudaSuccess) e = launch_pdl(rows_scan_kernel, dim3(1), dim3(1024), 0, s, a.row_ptr, a.M);
  if (e == cudaSuccess && a.T > 0 && words > 0) e = launch_pdl(rows_fill_kernel, grid, dim3(kRowWarps * 32), 0, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool pdl_enabled() {
  static const bool v = [] {
    const char *e = std::getenv("GLMB_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

cudaError_t launch_assoc_sample(const SampleArgs &a, int sm_count, cudaStream_t s) {
  SampleArgs b = a;
  b.spc = 32;   // samples per CTA: one per lane
  const int64_t groups = (a.H_up + 31) / 32;
  const int64_t n = static_cast<int64_t>(a.H_old) * groups;
  const size_t fixed =
      sizeof(double) * static_cast<size_t>(max(a.n_count, 0)) +
      (sizeof(double) + sizeof(unsigned long long) + sizeof(int32_t)) * 32 * kSampWarps +
      sizeof(uint32_t) * 32 * 2 * ((static_cast<size_t>(a.T) + 31) / 32) +
      (a.n_count > 0 ? sizeof(uint32_t) * 32 * ((static_cast<size_t>(a.T) + (a.M < 256 ? 3 : 1)) / (a.M < 256 ? 4 : 2))
                     : 0) +
      sizeof(int32_t) * (static_cast<size_t>(a.M) + 1) + sizeof(int32_t) * ((static_cast<size_t>(a.M) + 3) / 4) +
      2 * sizeof(uint32_t) * static_cast<size_t>(a.ldt) + sizeof(int32_t) * static_cast<size_t>(a.T) + 16;
  if (fixed + 1024 > 220 * 1024) return cudaErrorInvalidValue;
  // shared memory per CTA sized so the grid runs in one wave where it can; the pool
  // beyond the fixed arrays holds the kept-entry bitmap and the parent's rows
  const int64_t sms = sm_count > 0 ? sm_count : 148;
  int64_t per_sm = std::min<int64_t>(8, std::max<int64_t>(1, (n + sms - 1) / sms));
  // fewer CTAs per SM rather than a pool too small for the parent's rows (the fallback
  // walks the whole global CSR)
  while (per_sm > 1 && (227 * 1024) / per_sm - 2048 < fixed + 24 * 1024) --per_sm;
  const size_t target = std::min<size_t>(220 * 1024, (227 * 1024) / per_sm - 2048);
  static const int pool_env = [] {  // test hook: force a small pool (every fallback path)
    const char *e = std::getenv("GLMB_SAMPLER_POOL");
    return e ? std::atoi(e) : 0;
  }();
  size_t pool = target > fixed + 1024 ? (target - fixed) & ~static_cast<size_t>(15) : 1024;
  if (pool_env > 0) pool = static_cast<size_t>(pool_env) & ~static_cast<size_t>(15);
  b.pool = static_cast<int32_t>(pool);
  const size_t smem = pool + fixed;
  cudaError_t e = cudaFuncSetAttribute(assoc_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  e = launch_pdl(assoc_sample_kernel, dim3(static_cast<unsigned>(n)), dim3(kSampThreads), smem, s, b);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_dedup(const DedupArgs &a, cudaStream_t s) {
  cudaError_t e = launch_pdl(dedup_kernel, dim3(a.H_old), dim3(kDedupThreads), 0, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int32_t prune_capacity(int32_t h_max) {
  int32_t c = 1;
  while (c < h_max) c <<= 1;
  return c;
}

cudaError_t launch_prune(const PruneArgs &a, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(a.cap2) * (sizeof(unsigned long long) + sizeof(int32_t));
  if (smem > 40 * 1024) {  // dynamic + static shared memory past the 48 KB default
    cudaError_t e =
        cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  {
    cudaError_t e = launch_pdl(prune_kernel, dim3(1), dim3(kPruneThreads), smem, s, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace glmb
