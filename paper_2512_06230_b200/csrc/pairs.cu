// pairs.cu -- the particle loop after the hypothesis update (
// PAPER.md P:53 §Approach):
//
//   assoc_pairs   unique (track, measurement set) pairs over the kept hypotheses
//                 ("a batched particle update for all unique (track, measurement)
//                 association pairs", reading R30)
//   resample      systematic resampling of each pair's reweighted particles when
//                 ESS < P/2 ("a resampling step is performed if necessary", R31, R32)
//
// (the per-pair Bayes update itself is reweight.cu's cluster kernel in pair mode.)
// The resampling CDF is built from integer weights W = floor(w 2^26), so the
// prefix sums, the ESS decision and the ancestors are exact integers: the same
// on any hardware and in any summation order.
#include <algorithm>
#include <cstdlib>

#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

__device__ __forceinline__ unsigned long long mix64p(unsigned long long z) {  // SplitMix64 finaliser
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// block-wide exclusive scan of one int per thread (blockDim.x == 1024 or less, multiple of 32)
template <typename Ti>
__device__ Ti block_excl_scan(Ti v, Ti *wsum /* [32] */, Ti &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Ti x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const Ti y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    Ti s = lane < nw ? wsum[lane] : Ti(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const Ti y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  total = wsum[nw - 1];
  const Ti r = (wid ? wsum[wid - 1] : Ti(0)) + x - v;
  __syncthreads();
  return r;
}

// ------------------------------------------------------------------ per-hypothesis inversion of theta
// One CTA per kept hypothesis r: |S| and a fingerprint of S for every track,
// the per-track offsets, and the lists S (ascending i) in list[r][0..M).
constexpr int kInvThreads = 256;
constexpr int kInvSortMax = 32;  // rows per track sorted by one thread; more: the warp walk

__global__ void __launch_bounds__(kInvThreads) invert_kernel(PairsArgs a) {
  grid_dep_wait();
  extern __shared__ unsigned char smraw[];
  unsigned long long *fp = reinterpret_cast<unsigned long long *>(smraw);  // [T]
  int32_t *cnt = reinterpret_cast<int32_t *>(fp + a.T);                   // [T]
  __shared__ int32_t wsum[32];
  const int32_t r = blockIdx.x;
  if (a.n_hyp_dev != nullptr && r >= __ldg(a.n_hyp_dev)) return;
  const int64_t q = __ldg(a.hyp_idx + r);
  const uint32_t *al = a.alive + q * a.ldt;
  const int32_t *th = a.theta + q * a.ldm;
  for (int32_t j = threadIdx.x; j < a.T; j += kInvThreads) {
    cnt[j] = 0;
    fp[j] = 0ull;
  }
  __syncthreads();
  for (int32_t i = threadIdx.x; i < a.M; i += kInvThreads) {
    const int32_t c = __ldg(th + i);
    if (c >= 1 && c <= a.T) {
      const int32_t j = c - 1;
      if ((__ldg(al + (j >> 5)) >> (j & 31)) & 1u) {
        atomicAdd(cnt + j, 1);
        atomicAdd(fp + j, mix64p(static_cast<unsigned long long>(i) + 0x632BE59BD9B4E019ull));
      }
    }
  }
  __syncthreads();
  // per-track outputs and the exclusive scan of the counts (offsets into list[r])
  int32_t carry = 0;
  bool big = false;  // some track holds more than kInvSortMax rows
  const int64_t rb = static_cast<int64_t>(r) * a.T;
  int32_t *start = reinterpret_cast<int32_t *>(fp);  // [T] list starts (fp is consumed)
  for (int32_t j0 = 0; j0 < a.T; j0 += kInvThreads) {
    const int32_t j = j0 + threadIdx.x;
    int32_t c = 0;
    unsigned long long f = 0ull;
    if (j < a.T) {
      const bool alive = (__ldg(al + (j >> 5)) >> (j & 31)) & 1u;
      c = cnt[j];
      f = fp[j];
      a.cnt[rb + j] = alive ? c : -1;
      a.fp[rb + j] = mix64p(f ^ (static_cast<unsigned long long>(c) << 40));
      big |= c > kInvSortMax;
    }
    int32_t tot;
    const int32_t ex = block_excl_scan(c, wsum, tot);  // (its barriers order fp reads before start writes)
    if (j < a.T) {
      a.off[rb + j] = carry + ex;
      cnt[j] = carry + ex;  // becomes the list cursor of track j
      start[j] = carry + ex;
    }
    carry += tot;
  }
  int32_t *list = a.list + static_cast<int64_t>(r) * a.M;
  if (!__syncthreads_or(big)) {
    // lists in ascending i: every listed row takes a slot of its track by an atomic
    // cursor (any order), then each track sorts its few rows -- the same ascending list
    // whatever order the atomics ran in
    for (int32_t i = threadIdx.x; i < a.M; i += kInvThreads) {
      const int32_t c = __ldg(th + i);
      if (c >= 1 && c <= a.T && ((__ldg(al + ((c - 1) >> 5)) >> ((c - 1) & 31)) & 1u))
        list[atomicAdd(cnt + c - 1, 1)] = i;
    }
    __syncthreads();
    for (int32_t j = threadIdx.x; j < a.T; j += kInvThreads) {
      const int32_t b = start[j], e = cnt[j];
      for (int32_t x = b + 1; x < e; ++x) {  // insertion sort (<= kInvSortMax rows)
        const int32_t v = list[x];
        int32_t y = x - 1;
        while (y >= b && list[y] > v) {
          list[y + 1] = list[y];
          --y;
        }
        list[y + 1] = v;
      }
    }
    return;
  }
  // a track with many rows: warp 0 walks the rows 32 at a time; lanes with the same
  // track are ranked by lane, and the group's leader advances the cursor
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int32_t i0 = 0; i0 < a.M; i0 += 32) {
      const int32_t i = i0 + lane;
      int32_t key = -1 - lane;  // unique per lane when the row is not listed
      if (i < a.M) {
        const int32_t c = __ldg(th + i);
        if (c >= 1 && c <= a.T && ((__ldg(al + ((c - 1) >> 5)) >> ((c - 1) & 31)) & 1u)) key = c - 1;
      }
      const uint32_t grp = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(grp) - 1;
      int32_t b = 0;
      if (key >= 0 && lane == leader) {
        b = cnt[key];
        cnt[key] = b + __popc(grp);
      }
      b = __shfl_sync(0xffffffffu, b, leader);
      if (key >= 0) list[b + __popc(grp & ((1u << lane) - 1u))] = i;
    }
  }
}

// first occurrence of each (j, S): the earliest r' <= r with the same list
__global__ void __launch_bounds__(256) first_kernel(PairsArgs a) {
  grid_dep_wait();
  const int32_t r = blockIdx.y;
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.T || (a.n_hyp_dev != nullptr && r >= __ldg(a.n_hyp_dev))) return;
  const int64_t e = static_cast<int64_t>(r) * a.T + j;
  const int32_t c = a.cnt[e];
  if (c < 0) {
    a.first[e] = -1;
    return;
  }
  const unsigned long long f = a.fp[e];
  const int32_t *mine = a.list + static_cast<int64_t>(r) * a.M + a.off[e];
  // earlier rows checked kFirstBatch at a time: their (count, fingerprint) loads are issued
  // together (one dependent L2 round trip per earlier row was the limiter), then compared
  // in row order, so the first match is still the smallest r2
  constexpr int kFirstBatch = 8;
  int32_t first = r;
  for (int32_t rb = 0; rb < r && first == r; rb += kFirstBatch) {
    int32_t cc[kFirstBatch];
    unsigned long long ff[kFirstBatch];
#pragma unroll
    for (int u = 0; u < kFirstBatch; ++u) {
      const int64_t e2 = static_cast<int64_t>(rb + u) * a.T + j;
      cc[u] = rb + u < r ? a.cnt[e2] : -2;
      ff[u] = rb + u < r ? a.fp[e2] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kFirstBatch; ++u) {
      if (first != r || cc[u] != c || ff[u] != f) continue;
      const int32_t r2 = rb + u;
      const int32_t *other = a.list + static_cast<int64_t>(r2) * a.M + a.off[static_cast<int64_t>(r2) * a.T + j];
      bool same = true;
      for (int32_t k = 0; k < c && same; ++k) same = mine[k] == other[k];
      if (same) first = r2;
    }
  }
  a.first[e] = first;
}

// numbering in (r, j) order: pair index and list offset of each first occurrence.
// (1) per hypothesis row: how many new pairs and list entries; (2) one small CTA
// scans the rows; (3) per row: a block scan places the row's new pairs.
__device__ __forceinline__ int32_t n_hyp_used(const PairsArgs &a) {
  return a.n_hyp_dev != nullptr ? min(a.n_hyp, __ldg(a.n_hyp_dev)) : a.n_hyp;
}

__global__ void __launch_bounds__(256) row_count_kernel(PairsArgs a) {
  grid_dep_wait();
  __shared__ int32_t rk[8], rm[8];
  const int32_t r = blockIdx.x;
  int32_t k = 0, m = 0;
  if (r < n_hyp_used(a)) {
    const int64_t rb = static_cast<int64_t>(r) * a.T;
    for (int32_t j = threadIdx.x; j < a.T; j += blockDim.x) {
      const bool isnew = a.first[rb + j] == r;
      k += isnew;
      m += isnew ? a.cnt[rb + j] : 0;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    k += __shfl_xor_sync(0xffffffffu, k, o);
    m += __shfl_xor_sync(0xffffffffu, m, o);
  }
  if ((threadIdx.x & 31) == 0) {
    rk[threadIdx.x >> 5] = k;
    rm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t tk = 0, tm = 0;
    for (int q = 0; q < 8; ++q) {
      tk += rk[q];
      tm += rm[q];
    }
    a.row_k[r] = tk;
    a.row_m[r] = tm;
  }
}

__global__ void __launch_bounds__(1024) row_scan_kernel(PairsArgs a) {
  grid_dep_wait();
  __shared__ int32_t wsum[32];
  int32_t kc = 0, mc = 0;
  for (int32_t r0 = 0; r0 < a.n_hyp; r0 += 1024) {
    const int32_t r = r0 + threadIdx.x;
    const int32_t k = r < a.n_hyp ? a.row_k[r] : 0, m = r < a.n_hyp ? a.row_m[r] : 0;
    int32_t ktot, mtot;
    const int32_t ko = kc + block_excl_scan(k, wsum, ktot);
    const int32_t mo = mc + block_excl_scan(m, wsum, mtot);
    if (r < a.n_hyp) {
      a.row_k[r] = ko;  // in place: becomes the row's first pair index / list offset
      a.row_m[r] = mo;
    }
    kc += ktot;
    mc += mtot;
  }
  if (threadIdx.x == 0) {
    a.pair_ptr[kc] = mc;
    *a.n_pairs = kc;
  }
}

__global__ void __launch_bounds__(256) number_kernel(PairsArgs a) {
  grid_dep_wait();
  __shared__ int32_t wsum[32];
  const int32_t r = blockIdx.x;
  if (r >= n_hyp_used(a)) return;
  const int64_t rb = static_cast<int64_t>(r) * a.T;
  int32_t kc = a.row_k[r], mc = a.row_m[r];
  for (int32_t j0 = 0; j0 < a.T; j0 += blockDim.x) {
    const int32_t j = j0 + threadIdx.x;
    int32_t isnew = 0, c = 0;
    if (j < a.T) {
      isnew = a.first[rb + j] == r;
      c = isnew ? a.cnt[rb + j] : 0;
    }
    int32_t ktot, mtot;
    const int32_t k = kc + block_excl_scan(isnew, wsum, ktot);
    const int32_t m = mc + block_excl_scan(c, wsum, mtot);
    if (isnew) {
      a.pair_track[k] = j;
      a.pair_ptr[k] = m;
      a.pair_of[rb + j] = k;
    }
    kc += ktot;
    mc += mtot;
  }
}

// pair_of for repeats and the measurement lists of the new pairs
__global__ void __launch_bounds__(256) finish_kernel(PairsArgs a) {
  grid_dep_wait();
  const int32_t r = blockIdx.y;
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.T || (a.n_hyp_dev != nullptr && r >= __ldg(a.n_hyp_dev))) return;
  const int64_t e = static_cast<int64_t>(r) * a.T + j;
  const int32_t f = a.first[e];
  if (f < 0) {
    a.pair_of[e] = -1;
    return;
  }
  if (f != r) {
    a.pair_of[e] = a.pair_of[static_cast<int64_t>(f) * a.T + j];
    return;
  }
  const int32_t k = a.pair_of[e];
  const int32_t c = a.cnt[e];
  const int32_t *src = a.list + static_cast<int64_t>(r) * a.M + a.off[e];
  int32_t *dst = a.pair_meas + a.pair_ptr[k];
  for (int32_t t = 0; t < c; ++t) dst[t] = src[t];
}

// ------------------------------------------------------------------ systematic resampling
// One CTA per pair k.  W_m = floor(w_m 2^26) in shared memory, cum_m = W_0 + ...
// + W_m (u64, exact, one block scan of per-thread chunk sums), S = cum_{P-1}, Q =
// sum W_m^2 (u128, exact).  Resample iff 2 S^2 < P Q (ESS < P/2).  Output slot n
// takes ancestor a_n = min{m : cum_m > t_n}, t_n = floor((n S + V) / P), V =
// floor(U S 2^-24), U = 2 (r >> 9) + 1 from Philox(counter (k, 0, step, 4 << 24))
// word 0 -- found particle-parallel (range starts marked, then a prefix max; see
// below).  Ancestors are non-decreasing in n, so the gathers of consecutive slots
// hit neighbouring addresses.  NT threads per pair: 256 for P <= 2048 (short CTAs),
// 512 above, three CTAs per SM at 40 registers (a 1024-thread CTA at 64 registers held a
// whole SM's register file).
// nf(c) = min{n >= 0 : n S + V >= c P}, capped at P; exact (fp64 estimate, integer
// fix-up; c P, n S <= 2^55 for S <= P 2^26, P <= 2^14)
__device__ __forceinline__ int res_first_slot(unsigned long long c, unsigned long long P, unsigned long long V,
                                              unsigned long long S, double inv_s) {
  const unsigned long long cp = c * P;
  if (cp <= V) return 0;
  const unsigned long long num = cp - V;
  unsigned long long n = static_cast<unsigned long long>(static_cast<double>(num) * inv_s);
  while (n * S < num) ++n;
  while (n > 0 && (n - 1) * S >= num) --n;
  return static_cast<int>(n < P ? n : P);
}

template <int kResThreads>
__device__ __forceinline__ void resample_unit(const ResampleArgs &a, const int k) {
  extern __shared__ __align__(16) unsigned char rs[];
  uint32_t *Wsm = reinterpret_cast<uint32_t *>(rs);          // [P] integer weights
  int *anc = reinterpret_cast<int *>(Wsm + a.P);              // [P] ancestor of each slot
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long qlo[kResThreads / 32], qhi[kResThreads / 32];
  __shared__ int do_res;
  const int j = __ldg(a.pair_track + k);
  const int64_t src = static_cast<int64_t>(j) * a.ld, dst = static_cast<int64_t>(k) * a.ld_out;
  const float *wk = a.w + static_cast<int64_t>(k) * a.ldw;
  const int quads = a.P >> 2;
  // integer weights (2^26 scaling of an fp32 in [0, 1] is exact; floor by conversion)
  unsigned __int128 qsum = 0;
  for (int g = threadIdx.x; g < quads; g += kResThreads) {
    const float4 w4 = __ldg(reinterpret_cast<const float4 *>(wk) + g);
    const uint32_t W0 = __float2uint_rd(w4.x * 67108864.0f), W1 = __float2uint_rd(w4.y * 67108864.0f),
                   W2 = __float2uint_rd(w4.z * 67108864.0f), W3 = __float2uint_rd(w4.w * 67108864.0f);
    reinterpret_cast<uint4 *>(Wsm)[g] = make_uint4(W0, W1, W2, W3);
    qsum += static_cast<unsigned long long>(W0) * W0 + static_cast<unsigned long long>(W1) * W1 +
            static_cast<unsigned long long>(W2) * W2 + static_cast<unsigned long long>(W3) * W3;
  }
  __syncthreads();
  // contiguous chunk of quads per thread (16-B shared loads) -> local sums -> block
  // exclusive scan -> cum before the chunk
  const int qper = (quads + kResThreads - 1) / kResThreads;
  const int g0 = min(quads, static_cast<int>(threadIdx.x) * qper), g1 = min(quads, g0 + qper);
  const uint4 *W4 = reinterpret_cast<const uint4 *>(Wsm);
  unsigned long long loc = 0;
  for (int g = g0; g < g1; ++g) {
    const uint4 w = W4[g];
    loc += (static_cast<unsigned long long>(w.x) + w.y) + (static_cast<unsigned long long>(w.z) + w.w);
  }
  unsigned long long S;
  const unsigned long long run0 = block_excl_scan(loc, wsum, S);  // cum before this thread's chunk
  // Q: exact 128-bit sum (lo/hi halves reduced with carries by one thread)
  {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long lo = static_cast<unsigned long long>(qsum), hi = static_cast<unsigned long long>(qsum >> 64);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o), hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
      const unsigned long long s = lo + lo2;
      hi += hi2 + (s < lo);
      lo = s;
    }
    if (lane == 0) {
      qlo[wid] = lo;
      qhi[wid] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned __int128 Q = 0;
      for (int w = 0; w < kResThreads / 32; ++w) Q += (static_cast<unsigned __int128>(qhi[w]) << 64) | qlo[w];
      const unsigned __int128 S2 = static_cast<unsigned __int128>(S) * S;
      do_res = S > 0 && 2 * S2 < static_cast<unsigned __int128>(a.P) * Q;
      if (a.flags != nullptr) a.flags[k] = (a.flags[k] & ~2u) | (do_res ? 2u : 0u);
    }
    __syncthreads();
  }
  float4 *ox = reinterpret_cast<float4 *>(a.ox + dst), *oy = reinterpret_cast<float4 *>(a.oy + dst),
         *ov = reinterpret_cast<float4 *>(a.ov + dst), *op = reinterpret_cast<float4 *>(a.opsi + dst),
         *oo = reinterpret_cast<float4 *>(a.oomega + dst), *ow = reinterpret_cast<float4 *>(a.ow + dst);
  if (!do_res) {  // keep the particles with their new weights
    for (int g = threadIdx.x; g < quads; g += kResThreads) {
      __stcs(ox + g, __ldg(reinterpret_cast<const float4 *>(a.x + src) + g));
      __stcs(oy + g, __ldg(reinterpret_cast<const float4 *>(a.y + src) + g));
      __stcs(ov + g, __ldg(reinterpret_cast<const float4 *>(a.v + src) + g));
      __stcs(op + g, __ldg(reinterpret_cast<const float4 *>(a.psi + src) + g));
      __stcs(oo + g, __ldg(reinterpret_cast<const float4 *>(a.omega + src) + g));
      __stcs(ow + g, __ldg(reinterpret_cast<const float4 *>(wk) + g));
    }
    return;
  }
  const u32x4 r = philox4x32_10(u32x4{static_cast<uint32_t>(k), 0u, a.step, 4u << 24}, a.key0, a.key1);
  const unsigned long long U = 2ull * (r.a >> 9) + 1ull;
  const unsigned long long V = (U * S) >> 24;  // U < 2^24, S <= 2^40: no overflow
  const float inv_p = 1.0f / static_cast<float>(a.P);
  // ancestors, particle-parallel: a_n = m exactly for n in [nf(cum_{m-1}), nf(cum_m)),
  // nf(c) = min{n : t_n >= c} = ceil((c P - V) / S) (t_n = floor((n S + V) / P) is
  // non-decreasing and t_n >= c <=> n S + V >= c P).  Each particle with offspring marks
  // the first slot of its range; a block prefix-max over the slots then gives every slot
  // its ancestor (ranges are ordered, so the last mark at or before n is a_n) -- no
  // search, and a heavy particle's long range costs one write, not one per slot.
  for (int n = threadIdx.x; n < a.P; n += kResThreads) anc[n] = -1;
  __syncthreads();
  {
    const unsigned long long Pl = static_cast<unsigned long long>(a.P);
    const double inv_s = 1.0 / static_cast<double>(S);
    unsigned long long c = run0;
    int lo = res_first_slot(c, Pl, V, S, inv_s);
    for (int g = g0; g < g1; ++g) {
      const uint4 w = W4[g];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t Wm = (&w.x)[e];
        if (Wm == 0u) continue;
        c += Wm;
        const int hi = res_first_slot(c, Pl, V, S, inv_s);
        if (hi > lo) anc[lo] = 4 * g + e;
        lo = hi;
      }
    }
  }
  __syncthreads();
  {  // inclusive prefix max over the slots: contiguous chunk per thread, warp + block scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int4 *A4 = reinterpret_cast<int4 *>(anc);
    int cmax = -1;
    for (int g = g0; g < g1; ++g) {
      const int4 v = A4[g];
      cmax = max(max(cmax, max(v.x, v.y)), max(v.z, v.w));
    }
    int x = cmax;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = max(x, y);
    }
    __shared__ int wmax[kResThreads / 32];
    if (lane == 31) wmax[wid] = x;
    __syncthreads();
    // exclusive max over the warps before this one: a shuffle scan of wmax[]
    int wv = lane < kResThreads / 32 ? wmax[lane] : -1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv = max(wv, y);
    }
    const int before = wid > 0 ? __shfl_sync(0xffffffffu, wv, wid - 1) : -1;
    const int xprev = __shfl_up_sync(0xffffffffu, x, 1);
    int run = max(before, lane > 0 ? xprev : -1);
    for (int g = g0; g < g1; ++g) {
      int4 v = A4[g];
      run = max(run, v.x);
      v.x = run;
      run = max(run, v.y);
      v.y = run;
      run = max(run, v.z);
      v.z = run;
      run = max(run, v.w);
      v.w = run;
      A4[g] = v;
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < quads; g += kResThreads) {
    const int4 an = reinterpret_cast<const int4 *>(anc)[g];
    float4 X, Y, Vv, Ps, Om;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t m = src + (&an.x)[e];
      (&X.x)[e] = __ldg(a.x + m);
      (&Y.x)[e] = __ldg(a.y + m);
      (&Vv.x)[e] = __ldg(a.v + m);
      (&Ps.x)[e] = __ldg(a.psi + m);
      (&Om.x)[e] = __ldg(a.omega + m);
    }
    __stcs(ox + g, X);
    __stcs(oy + g, Y);
    __stcs(ov + g, Vv);
    __stcs(op + g, Ps);
    __stcs(oo + g, Om);
    __stcs(ow + g, make_float4(inv_p, inv_p, inv_p, inv_p));
  }
}

// Grid-stride over the device count of pairs (the grid is capped near the resident
// CTA count: a capacity-sized grid of mostly empty 1024-thread CTAs cost ~0.1 ms).
template <int kResThreads>
__global__ void __launch_bounds__(kResThreads, kResThreads == 512 ? 3 : (kResThreads == 256 ? 4 : 1)) resample_kernel(ResampleArgs a) {
  grid_dep_wait();
  const int n = a.n_units_dev != nullptr ? min(a.K, __ldg(a.n_units_dev)) : a.K;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    resample_unit<kResThreads>(a, k);
    __syncthreads();  // shared memory is reused by the next unit
  }
}

// ------------------------------------------------------------------ tracker loop (f4)
// Kept hypothesis r -> parent r of the next step: bits of the pairs it uses
// (rows of the new particle set) plus the birth columns; ln of its weight.
__global__ void __launch_bounds__(128) next_parents_kernel(NextParentsArgs a) {
  grid_dep_wait();
  extern __shared__ uint32_t msk[];  // [ldt]
  const int32_t r = blockIdx.x;
  const int32_t nk = __ldg(a.n_kept);
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.n_parents = min(nk, a.n_hyp_cap);
  if (r >= nk) return;
  for (int32_t k = threadIdx.x; k < a.ldt; k += blockDim.x) msk[k] = 0u;
  __syncthreads();
  const int32_t *po = a.pair_of + static_cast<int64_t>(r) * a.T;
  for (int32_t j = threadIdx.x; j < a.T; j += blockDim.x) {
    const int32_t k = __ldg(po + j);
    if (k >= 0 && k < a.K_cap) atomicOr(msk + (k >> 5), 1u << (k & 31));
  }
  const int32_t col0 = a.birth_col0_dev != nullptr ? min(__ldg(a.birth_col0_dev), a.K_cap) : a.birth_col0;
  for (int32_t b = threadIdx.x; b < a.B; b += blockDim.x) {
    const int32_t c = col0 + b;
    atomicOr(msk + (c >> 5), 1u << (c & 31));
  }
  __syncthreads();
  uint32_t *out = a.parent_mask + static_cast<int64_t>(r) * a.ldt;
  for (int32_t k = threadIdx.x; k < a.ldt; k += blockDim.x) out[k] = msk[k];
  if (threadIdx.x == 0) a.parent_logw[r] = log(__ldg(a.keep_w + r));
}

// MAP estimate: weighted mean position of each track of kept hypothesis 0 (fp64 sums)
__global__ void __launch_bounds__(256) map_estimate_kernel(MapEstimateArgs a) {
  grid_dep_wait();
  __shared__ double red[3][8];
  const int32_t j = blockIdx.x;
  const int32_t k = __ldg(a.n_kept) > 0 ? __ldg(a.pair_of0 + j) : -1;
  double *e = a.est + 3 * static_cast<int64_t>(j);
  if (k < 0 || k >= a.n_rows) {  // no pair, or a pair past the set's rows (K_cap overflow)
    if (threadIdx.x == 0) {
      e[0] = __longlong_as_double(0x7ff8000000000000ll);
      e[1] = e[0];
      e[2] = 0.0;
    }
    return;
  }
  const int64_t base = static_cast<int64_t>(k) * a.ld;
  double sw = 0.0, sx = 0.0, sy = 0.0;
  for (int32_t p = threadIdx.x; p < a.P; p += blockDim.x) {
    const double w = __ldg(a.w + base + p);
    sw += w;
    sx += w * static_cast<double>(__ldg(a.x + base + p));
    sy += w * static_cast<double>(__ldg(a.y + base + p));
  }
  sw = warp_sum_d(sw);
  sx = warp_sum_d(sx);
  sy = warp_sum_d(sy);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][wid] = sw;
    red[1][wid] = sx;
    red[2][wid] = sy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tw = 0.0, tx = 0.0, ty = 0.0;
    for (int q = 0; q < 8; ++q) {
      tw += red[0][q];
      tx += red[1][q];
      ty += red[2][q];
    }
    e[0] = tx / tw;
    e[1] = ty / tw;
    e[2] = 1.0;
  }
}

}  // namespace

size_t pairs_workspace_bytes(int32_t n_hyp, int32_t T, int32_t M) {
  const size_t nt = static_cast<size_t>(n_hyp) * T;
  return nt * (3 * sizeof(int32_t) + sizeof(unsigned long long)) + static_cast<size_t>(n_hyp) * M * sizeof(int32_t) +
         2 * static_cast<size_t>(n_hyp) * sizeof(int32_t) + 64;
}

cudaError_t launch_assoc_pairs(const PairsArgs &in, void *ws, cudaStream_t s) {
  PairsArgs a = in;
  const size_t nt = static_cast<size_t>(a.n_hyp) * a.T;
  unsigned char *p = static_cast<unsigned char *>(ws);
  p = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  a.fp = reinterpret_cast<unsigned long long *>(p);
  a.cnt = reinterpret_cast<int32_t *>(a.fp + nt);
  a.off = a.cnt + nt;
  a.first = a.off + nt;
  a.list = a.first + nt;
  a.row_k = a.list + static_cast<size_t>(a.n_hyp) * a.M;
  a.row_m = a.row_k + a.n_hyp;
  if (a.n_hyp == 0 || a.T == 0) {
    cudaError_t e = cudaMemsetAsync(a.n_pairs, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
    return cudaMemsetAsync(a.pair_ptr, 0, sizeof(int32_t), s);
  }
  const size_t smem = static_cast<size_t>(a.T) * (sizeof(unsigned long long) + sizeof(int32_t));
  if (smem > 40 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_pdl(invert_kernel, dim3(a.n_hyp), dim3(kInvThreads), smem, s, a);
  const dim3 g2((a.T + 255) / 256, a.n_hyp);
  if (e == cudaSuccess) e = launch_pdl(first_kernel, g2, dim3(256), 0, s, a);
  if (e == cudaSuccess) e = launch_pdl(row_count_kernel, dim3(a.n_hyp), dim3(256), 0, s, a);
  if (e == cudaSuccess) e = launch_pdl(row_scan_kernel, dim3(1), dim3(1024), 0, s, a);
  if (e == cudaSuccess) e = launch_pdl(number_kernel, dim3(a.n_hyp), dim3(256), 0, s, a);
  if (e == cudaSuccess) e = launch_pdl(finish_kernel, g2, dim3(256), 0, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_resample(const ResampleArgs &a, int sm_count, cudaStream_t s) {
  if (a.K == 0) return cudaSuccess;
  const size_t smem = static_cast<size_t>(a.P) * (sizeof(uint32_t) + sizeof(int));
  // about two waves of resident CTAs (shared memory bounds residency at large P)
  const int sms = sm_count > 0 ? sm_count : 148;
  const int per_sm = a.P <= 2048 ? std::max(1, std::min(8, static_cast<int>((200 * 1024) / (smem + 1024))))
                                 : std::max(1, std::min(3, static_cast<int>((200 * 1024) / (smem + 1024))));
  const int grid = std::min(a.K, 2 * sms * per_sm);
  // threads per pair above P = 2048: 512 (three CTAs per SM at 40 registers;
  // a 1024-thread CTA held a whole SM's register file) unless GLMB_RESAMPLE_NT=1024
  static const int res_nt = [] {
    const char *e = std::getenv("GLMB_RESAMPLE_NT");
    return e && std::atoi(e) == 1024 ? 1024 : 512;
  }();
  if (smem > 40 * 1024) {
    cudaError_t e = a.P <= 2048 ? cudaFuncSetAttribute(resample_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(smem))
                    : res_nt == 512 ? cudaFuncSetAttribute(resample_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(smem))
                                : cudaFuncSetAttribute(resample_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  cudaError_t e2 = a.P <= 2048  ? launch_pdl(resample_kernel<256>, dim3(grid), dim3(256), smem, s, a)
                   : res_nt == 512 ? launch_pdl(resample_kernel<512>, dim3(grid), dim3(512), smem, s, a)
                                   : launch_pdl(resample_kernel<1024>, dim3(grid), dim3(1024), smem, s, a);
  if (e2 != cudaSuccess) return e2;
  return cudaGetLastError();
}

}  // namespace glmb

namespace glmb {

cudaError_t launch_next_parents(const NextParentsArgs &a, cudaStream_t s) {
  if (a.n_hyp_cap == 0) return cudaMemsetAsync(a.n_parents, 0, sizeof(int32_t), s);
  cudaError_t e = launch_pdl(next_parents_kernel, dim3(a.n_hyp_cap), dim3(128), sizeof(uint32_t) * a.ldt, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_map_estimate(const MapEstimateArgs &a, cudaStream_t s) {
  if (a.T == 0) return cudaSuccess;
  cudaError_t e = launch_pdl(map_estimate_kernel, dim3(a.T), dim3(256), 0, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace glmb
