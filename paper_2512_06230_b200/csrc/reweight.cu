// reweight.cu -- glmb_reweight: Bayes update of each track's particle weights
// under the supplied association map theta_k (§Approach).
//
//   S_j = {i : theta_i = col_offset + j + 1}
//   l_p = log2 w_p - sum_{i in S_j} 1/2 log2(e) d_ip^T R^-1 d_ip      (log2 domain)
//   m = max_p l_p,  s = sum_p 2^(l_p - m),  w'_p = 2^(l_p - m) / s
//   log_norm_j = (m + log2 s) ln 2 - |S_j| ln(2 pi sqrt(det R))
//
// HBM-bound: x, y, w are read once and w written once (16 B per particle).
// Launch variants by P (shape depends on P only: shard-invariant results):
//  * 2048 <= P <= 25600: the e-cache kernel (reweight_ecache_unit below): the
//    centred quadratic form (O(1) per particle for any |S_j|), an fp32 pass with
//    a checked error budget and an fp64 rerun otherwise, e_p parked in shared
//    memory between the two passes;
//  * smaller P: thread-block clusters holding the particles in registers;
//  * larger P: the generic path recomputing l_p (fp64) in the second pass.
// Where l_p is fp64 the max shift l_p - m keeps full relative accuracy even when
// the assigned measurement is far from the cloud; 2^(l-m) itself is fp32 MUFU.
// Block reductions run in a fixed order -> deterministic, shard-invariant.
#include <cfloat>
#include <cstdlib>

#include <cooperative_groups.h>

#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef GLMB_RW_DEBUG
#define GLMB_RW_DEBUG 0   // A/B timing builds only: 3 stamps the e-cache kernel's phases into w_out
#endif
#ifndef GLMB_RW_ECACHE_BLOCKS
#define GLMB_RW_ECACHE_BLOCKS 4
#endif
constexpr int kSCap = 256;   // assigned measurements held in shared memory (more: global rescan)

struct SList {
  double2 z[kSCap];
  int n;           // |S_j|
  int in_smem;     // 1 if all of S_j fits in z[]
  int e0;          // pair mode: first index of S_k in pair_meas
};

// Pair mode: S_k is given explicitly (ascending i) -- fetch its measurements.
__device__ void collect_S_pair(const ReweightArgs &a, int k, SList &S) {
  const int e0 = __ldg(a.pair_ptr + k), n = __ldg(a.pair_ptr + k + 1) - e0;
  const float2 *Z2 = reinterpret_cast<const float2 *>(a.Z);
  for (int e = threadIdx.x; e < n && e < kSCap; e += blockDim.x) {
    const float2 z = __ldg(Z2 + __ldg(a.pair_meas + e0 + e));
    S.z[e] = make_double2(z.x, z.y);
  }
  if (threadIdx.x == 0) {
    S.n = n;
    S.in_smem = n <= kSCap;
    S.e0 = e0;
  }
  __syncthreads();
}

// Collect S_j in ascending i.  Chunks of 8 * kThreads indices: every thread
// issues its 8 theta loads at once (one L2 round trip per chunk, not one per
// 32 indices), each warp ballots per row, and warp 0 turns the 64 (row, warp)
// masks -- already in ascending-i order -- into list positions with a
// warp-shuffle prefix sum and fetches the hit measurements.
constexpr int kRows = 8;
template <int NT = kThreads>
__device__ void collect_S(const ReweightArgs &a, int col, SList &S, uint32_t *masks /* [64] */) {
  constexpr int kW = NT / 32, kR = 64 / kW;  // kR rows of NT indices per chunk: 64 (row, warp) masks
  static_assert(kR * kW == 64, "warp 0 scans two masks per lane");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int total = 0;  // maintained by warp 0
  for (int base = 0; base < a.M; base += kR * NT) {
    int th[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int i = base + r * NT + threadIdx.x;
      th[r] = i < a.M ? __ldg(a.theta + i) : -1;
    }
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const uint32_t m = __ballot_sync(0xffffffffu, th[r] == col);
      if (lane == 0) masks[r * kW + warp] = m;
    }
    __syncthreads();
    if (warp == 0) {
      uint32_t m0 = masks[lane], m1 = masks[lane + 32];  // mask k covers i = base + 32 k + bit
      const int c0 = __popc(m0), c1 = __popc(m1);
      int s0 = c0, s1 = c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t0 = __shfl_up_sync(0xffffffffu, s0, o), t1 = __shfl_up_sync(0xffffffffu, s1, o);
        if (lane >= o) {
          s0 += t0;
          s1 += t1;
        }
      }
      const int tot0 = __shfl_sync(0xffffffffu, s0, 31), tot1 = __shfl_sync(0xffffffffu, s1, 31);
      int off0 = total + s0 - c0, off1 = total + tot0 + s1 - c1;
      const float2 *Z2 = reinterpret_cast<const float2 *>(a.Z);
      while (m0) {
        const int i = base + 32 * lane + __ffs(m0) - 1;
        m0 &= m0 - 1;
        if (off0 < kSCap) {
          const float2 z = __ldg(Z2 + i);
          S.z[off0] = make_double2(z.x, z.y);
        }
        ++off0;
      }
      while (m1) {
        const int i = base + 32 * (lane + 32) + __ffs(m1) - 1;
        m1 &= m1 - 1;
        if (off1 < kSCap) {
          const float2 z = __ldg(Z2 + i);
          S.z[off1] = make_double2(z.x, z.y);
        }
        ++off1;
      }
      total += tot0 + tot1;
    }
    __syncthreads();  // masks are rewritten by the next chunk
  }
  if (threadIdx.x == 0) {
    S.n = total;
    S.in_smem = total <= kSCap;
  }
  __syncthreads();
}

__device__ __forceinline__ double qform(const ReweightArgs &a, double zx, double zy, double px, double py) {
  const double dx = zx - px, dy = zy - py;
  return fma(dx, fma(a.qa, dx, a.qb * dy), a.qc * dy * dy);
}

// l_p for one particle (fp64 accumulation in ascending i).
__device__ __forceinline__ double log_weight(const ReweightArgs &a, const SList &S, int col, float px, float py,
                                             float w) {
  // MUFU.LG2: abs. error ~2^-22 in log2 w = rel. error ~1.7e-7 in w'
  double l = w > 0.f ? static_cast<double>(__log2f(w)) : -INFINITY;
  const double dpx = px, dpy = py;
  if (S.in_smem) {
    for (int s = 0; s < S.n; ++s) l -= qform(a, S.z[s].x, S.z[s].y, dpx, dpy);
  } else if (a.pair_meas != nullptr) {
    for (int e = S.e0; e < S.e0 + S.n; ++e) {
      const float2 z = __ldg(reinterpret_cast<const float2 *>(a.Z) + __ldg(a.pair_meas + e));
      l -= qform(a, z.x, z.y, dpx, dpy);
    }
  } else {
    for (int i = 0; i < a.M; ++i)
      if (__ldg(a.theta + i) == col) {
        const float2 z = __ldg(reinterpret_cast<const float2 *>(a.Z) + i);
        l -= qform(a, z.x, z.y, dpx, dpy);
      }
  }
  return l;
}

__device__ double block_max(double v, double *red) {
  v = warp_max_d(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int k = 1; k < kWarps; ++k) r = fmax(r, red[k]);
  __syncthreads();
  return r;
}

__device__ double block_sum(double v, double *red) {
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
#pragma unroll
  for (int k = 1; k < kWarps; ++k) r += red[k];
  __syncthreads();
  return r;
}

__device__ __forceinline__ float &q4(float4 &v, int q) { return (&v.x)[q]; }

// CACHED: l_p (fp64) cached in dynamic shared memory (P * 8 bytes), so the
// particles are read from HBM once; otherwise l_p is recomputed per pass.
template <bool CACHED>
__global__ void __launch_bounds__(kThreads) reweight_kernel(const ReweightArgs a) {
  extern __shared__ __align__(16) double lcache[];
  __shared__ SList S;
  __shared__ double red[kWarps];
  __shared__ uint32_t masks[kRows * kWarps];
  const int j = blockIdx.x;
  const int col = a.col_offset + j + 1;
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float4 *xs = reinterpret_cast<const float4 *>(a.x + base);
  const float4 *ys = reinterpret_cast<const float4 *>(a.y + base);
  const float4 *ws = reinterpret_cast<const float4 *>(a.w + base);
  float4 *wo = reinterpret_cast<float4 *>(a.w_out + base);
  const bool copy_out = a.w_out != a.w;
  const int quads = a.P >> 2;

  collect_S(a, col, S, masks);
  const int nS = S.n;

  if (nS == 0) {  // untouched; log_norm = ln sum w
    double s = 0.0;
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      const float4 w4 = __ldcs(ws + g);
      if (copy_out) __stcs(wo + g, w4);
      s += (static_cast<double>(w4.x) + w4.y) + (static_cast<double>(w4.z) + w4.w);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      a.log_norm[j] = static_cast<float>(log(s));
      a.flags[j] = 0u;
    }
    return;
  }

  // pass 1: l_p and the block max
  double lm = -INFINITY;
#pragma unroll 4
  for (int g = threadIdx.x; g < quads; g += kThreads) {
    float4 X = __ldcs(xs + g), Y = __ldcs(ys + g), Wv = __ldcs(ws + g);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double l = log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q));
      if constexpr (CACHED) lcache[4 * g + q] = l;
      lm = fmax(lm, l);
    }
  }
  const double m = block_max(lm, red);

  if (m == -INFINITY) {  // every weight zero: uniform reset, flagged (never abort)
    const float u = 1.0f / static_cast<float>(a.P);
    for (int g = threadIdx.x; g < quads; g += kThreads) __stcs(wo + g, make_float4(u, u, u, u));
    if (threadIdx.x == 0) {
      a.log_norm[j] = -INFINITY;
      a.flags[j] = 1u;
    }
    return;
  }

  // pass 2: e_p = 2^(l_p - m) (kept in place of l_p) and s = sum e_p
  double s = 0.0;
  for (int g = threadIdx.x; g < quads; g += kThreads) {
    float4 X, Y, Wv;
    if constexpr (!CACHED) {
      X = __ldcs(xs + g);
      Y = __ldcs(ys + g);
      Wv = __ldcs(ws + g);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double l;
      if constexpr (CACHED) l = lcache[4 * g + q];
      else l = log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q));
      const float e = ex2_approx(static_cast<float>(l - m));
      if constexpr (CACHED) lcache[4 * g + q] = e;
      s += e;
    }
  }
  s = block_sum(s, red);
  const float inv_s = static_cast<float>(1.0 / s);

  // pass 3: w'_p = e_p / s
  for (int g = threadIdx.x; g < quads; g += kThreads) {
    float4 o;
    if constexpr (CACHED) {
#pragma unroll
      for (int q = 0; q < 4; ++q) q4(o, q) = static_cast<float>(lcache[4 * g + q]) * inv_s;
    } else {
      float4 X = __ldcs(xs + g), Y = __ldcs(ys + g), Wv = __ldcs(ws + g);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        q4(o, q) = ex2_approx(static_cast<float>(log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q)) - m)) * inv_s;
    }
    __stcs(wo + g, o);
  }
  if (threadIdx.x == 0) {
    const double ln2 = 0.69314718055994530942;
    a.log_norm[j] = static_cast<float>((m + log2(s)) * ln2 - nS * a.log_norm1);
    a.flags[j] = 0u;
  }
}

// Split cluster barrier: arrive without a release fence, wait at exit.
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// (max, sum) pairs combined exactly as one pass over all terms would give up
// to rounding: (m, s) + (m', s') = (M, s 2^(m-M) + s' 2^(m'-M)), M = max(m, m').
// Applied by one thread in a fixed order, so the reduction is deterministic.
__device__ __forceinline__ void ms_merge(double &m, double &s, double &s2, double m2, double t, double t2) {
  const double M = fmax(m, m2);
  if (M == -INFINITY) {
    s = 0.0;
    s2 = 0.0;
    return;
  }
  const double f1 = ex2_approx(static_cast<float>(m - M)), f2 = ex2_approx(static_cast<float>(m2 - M));
  s = s * f1 + t * f2;
  s2 = s2 * (f1 * f1) + t2 * (f2 * f2);
  m = M;
}

// Thread-block-cluster variant (P <= 8 * 1024 * R): the CL CTAs of a cluster
// split one track's particles and keep them in registers.  One pass computes
// l_p, each warp's (max m_w, sum 2^(l - m_w)) by shuffles, and one thread per
// CTA merges the warps and then the cluster's CTAs (DSMEM, rank order:
// deterministic) -- one reduction and one cluster barrier instead of a max
// pass and a sum pass, and no per-thread rescaling.  w'_p = 2^(l_p - m_w) *
// 2^(m_w - m) / s.  Particle loads are issued
// before the theta scan so the two latencies overlap.
// One unit (track j in theta mode, pair k in pair mode) by the whole cluster; every
// path ends with a cluster barrier, so the shared memory is free for the next unit.
template <int CL, int R>
__device__ __forceinline__ void reweight_unit(const ReweightArgs &a, const int u) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ SList S;
  __shared__ double red[3][kWarps];
  __shared__ uint32_t masks[kRows * kWarps];
  __shared__ double part[3];  // this CTA's (max, sum, sum of squares), read by the peers
  const int crank = static_cast<int>(cluster.block_rank());
  const bool pairs = a.pair_track != nullptr;
  const int j = pairs ? __ldg(a.pair_track + u) : u;
  const int col = a.col_offset + j + 1;
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float4 *xs = reinterpret_cast<const float4 *>(a.x + base);
  const float4 *ys = reinterpret_cast<const float4 *>(a.y + base);
  const float4 *ws = reinterpret_cast<const float4 *>(a.w + base);
  float4 *wo = reinterpret_cast<float4 *>(a.w_out + static_cast<int64_t>(u) * a.ld_out);
  const bool copy_out = pairs || a.w_out != a.w;
  const int quads = a.P >> 2;
  const int per = (quads + CL - 1) / CL;
  const int q0 = crank * per, q1 = min(quads, q0 + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  float4 X[R], Y[R], W[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int g = q0 + threadIdx.x + r * kThreads;
    if (g < q1) {
      X[r] = __ldcs(xs + g);
      Y[r] = __ldcs(ys + g);
      W[r] = __ldcs(ws + g);
    }
  }
  if (pairs) collect_S_pair(a, u, S);
  else collect_S(a, col, S, masks);
  const int nS = S.n;

  if (nS == 0) {  // untouched; log_norm = ln sum w; ESS = (sum w)^2 / sum w^2
    double sw = 0.0, sw2 = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = q0 + threadIdx.x + r * kThreads;
      if (g < q1) {
        sw += (static_cast<double>(W[r].x) + W[r].y) + (static_cast<double>(W[r].z) + W[r].w);
        sw2 += (static_cast<double>(W[r].x) * W[r].x + static_cast<double>(W[r].y) * W[r].y) +
               (static_cast<double>(W[r].z) * W[r].z + static_cast<double>(W[r].w) * W[r].w);
      }
    }
    sw = block_sum(sw, red[0]);
    if (a.ess != nullptr) sw2 = block_sum(sw2, red[1]);
    if (threadIdx.x == 0) {
      part[1] = sw;
      part[2] = sw2;
    }
    cluster.sync();
    if (copy_out) {  // after the barrier: the copy does not sit behind its release fence
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int g = q0 + threadIdx.x + r * kThreads;
        if (g < q1) __stcs(wo + g, W[r]);
      }
    }
    if (crank == 0 && threadIdx.x == 0) {
      double tot = 0.0, tot2 = 0.0;
#pragma unroll
      for (int r = 0; r < CL; ++r) {
        const double *pr = cluster.map_shared_rank(part, r);
        tot += pr[1];
        tot2 += pr[2];
      }
      a.log_norm[u] = static_cast<float>(log(tot));
      a.flags[u] = 0u;
      if (a.ess != nullptr) a.ess[u] = tot2 > 0.0 ? static_cast<float>(tot * tot / tot2) : 0.0f;
    }
    if (crank == 0) __syncthreads();
    cluster_arrive_relaxed();  // done with the peers' shared memory
    cluster_wait();            // ... and they with ours
    return;
  }

  double l[4 * R];
  double mw = -INFINITY;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const bool ok = q0 + threadIdx.x + r * kThreads < q1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      l[4 * r + q] = ok ? log_weight(a, S, col, q4(X[r], q), q4(Y[r], q), q4(W[r], q)) : -INFINITY;
      mw = fmax(mw, l[4 * r + q]);
    }
  }
  // warp max (fp64 shuffles, no conversions), then terms relative to it
  mw = warp_max_d(mw);
  float e[4 * R];
  float sw = 0.0f, sw2 = 0.0f;
#pragma unroll
  for (int k = 0; k < 4 * R; ++k) {
    e[k] = mw == -INFINITY ? 0.0f : ex2_approx(static_cast<float>(l[k] - mw));
    sw += e[k];
    sw2 = fmaf(e[k], e[k], sw2);
  }
  sw = warp_sum(sw);
  if (a.ess != nullptr) sw2 = warp_sum(sw2);
  // block: thread 0 merges the warps in order; cluster: thread 0 of every CTA
  // merges the CL parts in rank order (all CTAs get the same (m, s))
  __shared__ double bc[3];
  if (lane == 0) {
    red[0][warp] = mw;
    red[1][warp] = sw;
    red[2][warp] = sw2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mb = red[0][0], sb = red[1][0], s2b = red[2][0];
#pragma unroll
    for (int k = 1; k < kWarps; ++k) ms_merge(mb, sb, s2b, red[0][k], red[1][k], red[2][k]);
    part[0] = mb;
    part[1] = sb;
    part[2] = s2b;
  }
  cluster.sync();
  if (threadIdx.x == 0) {
    double mc = -INFINITY, sc = 0.0, s2c = 0.0;
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      const double *pr = cluster.map_shared_rank(part, r);
      ms_merge(mc, sc, s2c, pr[0], pr[1], pr[2]);
    }
    bc[0] = mc;
    bc[1] = sc;
    bc[2] = s2c;
  }
  __syncthreads();
  const double mc = bc[0], sc = bc[1], s2c = bc[2];
  // every read of a peer's shared memory is done: arrive now (relaxed: no
  // memory ordering needed), wait only at exit so the stores below do not
  // sit behind a release fence
  cluster_arrive_relaxed();

  if (mc == -INFINITY) {  // every weight zero: uniform reset, flagged (never abort)
    const float uw = 1.0f / static_cast<float>(a.P);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = q0 + threadIdx.x + r * kThreads;
      if (g < q1) __stcs(wo + g, make_float4(uw, uw, uw, uw));
    }
    if (crank == 0 && threadIdx.x == 0) {
      a.log_norm[u] = -INFINITY;
      a.flags[u] = 1u;
      if (a.ess != nullptr) a.ess[u] = static_cast<float>(a.P);
    }
    cluster_wait();
    return;
  }
  // w'_p = 2^(l_p - m_w) 2^(m_w - m) / s; a factor below FLT_MIN flushes only
  // weights whose exact value is below FLT_MIN as well
  const float f = mw == -INFINITY ? 0.0f : ex2_approx(static_cast<float>(mw - mc)) * static_cast<float>(1.0 / sc);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int g = q0 + threadIdx.x + r * kThreads;
    if (g < q1) __stcs(wo + g, make_float4(e[4 * r] * f, e[4 * r + 1] * f, e[4 * r + 2] * f, e[4 * r + 3] * f));
  }
  if (crank == 0 && threadIdx.x == 0) {
    const double ln2 = 0.69314718055994530942;
    a.log_norm[u] = static_cast<float>((mc + log2(sc)) * ln2 - nS * a.log_norm1);
    a.flags[u] = 0u;
    if (a.ess != nullptr) a.ess[u] = static_cast<float>(sc * sc / s2c);  // (sum w')^2 / sum w'^2
  }
  cluster_wait();
}

template <int CL, int R>
__global__ void __launch_bounds__(kThreads, R == 1 ? 5 : (R == 2 ? 3 : 2)) reweight_cluster_kernel(const ReweightArgs a) {
  grid_dep_wait();  // pair mode is launched with programmatic serialization (hypothesis chain)
  // units u = cluster index, + clusters in the grid, ... (one pass unless the grid is capped)
  const int n_units = a.n_units_dev != nullptr ? min(a.T, __ldg(a.n_units_dev)) : a.T;
  const int stride = static_cast<int>(gridDim.x) / CL;
  for (int u = static_cast<int>(blockIdx.x) / CL; u < n_units; u += stride) reweight_unit<CL, R>(a, u);
}

// Flat two-pass variant: one 256-thread CTA per unit, no cluster.  Pass 1 streams the
// unit's particles once from HBM and keeps a per-thread online (m, s, s2) -- s relative to
// the thread's running max, rescaled when the max moves; the warps' and then the CTA's
// triples merge in a fixed order.  Pass 2 re-reads x, y, w (L2-resident by then),
// recomputes l_p bit for bit and writes w'_p = 2^(l_p - m) / s.  Nothing waits at a
// cluster barrier holding registers, so ~8 CTAs per SM stream concurrently.
// The per-thread sums stay fp32 (at most P / 256 terms of at most 1 each, rel. error
// ~1e-6); the conversions fp32 <-> fp64 run on the XU pipe beside MUFU, so keeping the
// running sums out of fp64 halves them per particle.
__device__ __forceinline__ void online_add(double l, double &m, float &s, float &s2) {
  if (l == -INFINITY) return;
  if (l > m) {
    const float f = m == -INFINITY ? 0.0f : ex2_approx(static_cast<float>(m - l));
    s = fmaf(s, f, 1.0f);
    s2 = fmaf(s2, f * f, 1.0f);
    m = l;
  } else {
    const float e = ex2_approx(static_cast<float>(l - m));
    s += e;
    s2 = fmaf(e, e, s2);
  }
}

template <bool LC>
__device__ __forceinline__ void reweight_flat_unit(const ReweightArgs &a, const int u) {
  extern __shared__ __align__(16) double lc[];  // [P] l_p when LC
  __shared__ SList S;
  __shared__ double red[3][kWarps];
  __shared__ uint32_t masks[kRows * kWarps];
  __shared__ double bc[3];
  const bool pairs = a.pair_track != nullptr;
  const int j = pairs ? __ldg(a.pair_track + u) : u;
  const int col = a.col_offset + j + 1;
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float4 *xs = reinterpret_cast<const float4 *>(a.x + base);
  const float4 *ys = reinterpret_cast<const float4 *>(a.y + base);
  const float4 *ws = reinterpret_cast<const float4 *>(a.w + base);
  float4 *wo = reinterpret_cast<float4 *>(a.w_out + static_cast<int64_t>(u) * a.ld_out);
  const bool copy_out = pairs || a.w_out != a.w;
  const int quads = a.P >> 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the first quad's loads are issued before the S scan, so the two latencies overlap
  float4 X0, Y0, W0;
  if (static_cast<int>(threadIdx.x) < quads) {
    X0 = __ldg(xs + threadIdx.x);
    Y0 = __ldg(ys + threadIdx.x);
    W0 = __ldg(ws + threadIdx.x);
  }
  if (pairs) collect_S_pair(a, u, S);
  else collect_S(a, col, S, masks);
  const int nS = S.n;

  if (nS == 0) {  // untouched; log_norm = ln sum w; ESS = (sum w)^2 / sum w^2
    double sw = 0.0, sw2 = 0.0;
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      const float4 w4 = __ldcs(ws + g);
      if (copy_out) __stcs(wo + g, w4);
      sw += (static_cast<double>(w4.x) + w4.y) + (static_cast<double>(w4.z) + w4.w);
      sw2 += (static_cast<double>(w4.x) * w4.x + static_cast<double>(w4.y) * w4.y) +
             (static_cast<double>(w4.z) * w4.z + static_cast<double>(w4.w) * w4.w);
    }
    sw = block_sum(sw, red[0]);
    if (a.ess != nullptr) sw2 = block_sum(sw2, red[1]);
    if (threadIdx.x == 0) {
      a.log_norm[u] = static_cast<float>(log(sw));
      a.flags[u] = 0u;
      if (a.ess != nullptr) a.ess[u] = sw2 > 0.0 ? static_cast<float>(sw * sw / sw2) : 0.0f;
    }
    __syncthreads();
    return;
  }

  // pass 1: online (m, s, s2) per thread; the next quad's loads are issued before this
  // quad's arithmetic
  double m = -INFINITY;
  float sm = 0.0f, sm2 = 0.0f;
  {
    int g = threadIdx.x;
    float4 X = X0, Y = Y0, W = W0;
#pragma unroll 1
    for (; g < quads; g += kThreads) {
      const int gn = g + kThreads;
      float4 Xn, Yn, Wn;
      if (gn < quads) {
        Xn = __ldg(xs + gn);
        Yn = __ldg(ys + gn);
        Wn = __ldg(ws + gn);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double l = log_weight(a, S, col, q4(X, q), q4(Y, q), q4(W, q));
        if constexpr (LC) lc[4 * g + q] = l;
        online_add(l, m, sm, sm2);
      }
      X = Xn;
      Y = Yn;
      W = Wn;
    }
  }
  // warp: max by shuffles, the lanes' sums rescaled to it; CTA: thread 0 merges the warps
  const double mw = warp_max_d(m);
  const double f = mw == -INFINITY || m == -INFINITY ? 0.0 : static_cast<double>(ex2_approx(static_cast<float>(m - mw)));
  double sw = warp_sum_d(static_cast<double>(sm) * f),
         sw2 = a.ess != nullptr ? warp_sum_d(static_cast<double>(sm2) * (f * f)) : 0.0;
  if (lane == 0) {
    red[0][warp] = mw;
    red[1][warp] = sw;
    red[2][warp] = sw2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mb = red[0][0], sb = red[1][0], s2b = red[2][0];
#pragma unroll
    for (int k = 1; k < kWarps; ++k) ms_merge(mb, sb, s2b, red[0][k], red[1][k], red[2][k]);
    bc[0] = mb;
    bc[1] = sb;
    bc[2] = s2b;
  }
  __syncthreads();
  const double mc = bc[0], sc = bc[1], s2c = bc[2];
  if (mc == -INFINITY) {  // every weight zero: uniform reset, flagged (never abort)
    const float uw = 1.0f / static_cast<float>(a.P);
    for (int g = threadIdx.x; g < quads; g += kThreads) __stcs(wo + g, make_float4(uw, uw, uw, uw));
    if (threadIdx.x == 0) {
      a.log_norm[u] = -INFINITY;
      a.flags[u] = 1u;
      if (a.ess != nullptr) a.ess[u] = static_cast<float>(a.P);
    }
    __syncthreads();
    return;
  }
  // pass 2: w'_p = 2^(l_p - m) / s (l_p recomputed from the L2-resident particles)
  const float inv_s = static_cast<float>(1.0 / sc);
  if constexpr (LC) {
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      float4 o;
#pragma unroll
      for (int q = 0; q < 4; ++q) q4(o, q) = ex2_approx(static_cast<float>(lc[4 * g + q] - mc)) * inv_s;
      __stcs(wo + g, o);
    }
  } else {
    int g = threadIdx.x;
    float4 X, Y, W;
    if (g < quads) {
      X = __ldcs(xs + g);
      Y = __ldcs(ys + g);
      W = __ldcs(ws + g);
    }
#pragma unroll 1
    for (; g < quads; g += kThreads) {
      const int gn = g + kThreads;
      float4 Xn, Yn, Wn;
      if (gn < quads) {
        Xn = __ldcs(xs + gn);
        Yn = __ldcs(ys + gn);
        Wn = __ldcs(ws + gn);
      }
      float4 o;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        q4(o, q) = ex2_approx(static_cast<float>(log_weight(a, S, col, q4(X, q), q4(Y, q), q4(W, q)) - mc)) * inv_s;
      __stcs(wo + g, o);
      X = Xn;
      Y = Yn;
      W = Wn;
    }
  }
  if (threadIdx.x == 0) {
    const double ln2 = 0.69314718055994530942;
    a.log_norm[u] = static_cast<float>((mc + log2(sc)) * ln2 - nS * a.log_norm1);
    a.flags[u] = 0u;
    if (a.ess != nullptr) a.ess[u] = static_cast<float>(sc * sc / s2c);
  }
  __syncthreads();  // S, red and bc are reused by the next unit
}

template <bool LC>
__global__ void __launch_bounds__(kThreads, 3) reweight_flat_kernel(const ReweightArgs a) {
  grid_dep_wait();
  const int n_units = a.n_units_dev != nullptr ? min(a.T, __ldg(a.n_units_dev)) : a.T;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) reweight_flat_unit<LC>(a, u);
}

// E-cache variant (the default for 2048 <= P <= 25600): one 256-thread CTA per unit, 4
// per SM (62 registers: the fp32 pass keeps two quads of loads in flight).  (1) When S_j fits in shared memory, sum_{s in S} q'(z_s - p) is evaluated as
// C0 + n q'(zbar - p) (zbar the mean of S_j's measurements, C0 = sum q'(z_s - zbar): the
// cross terms vanish), so every particle costs one fp64 quadratic form whatever |S_j| is;
// C0 is added back into log_norm only.  (2) Pass 1 parks e_p = 2^(l_p - m_t) in fp32 in
// shared memory (4 B per particle), m_t being the thread's running max (fp64), and
// rescales the thread's parked entries whenever a quad raises it; pass 2 writes
// w'_p = e_p 2^(m_t - m) / s from shared memory.  Pass 1 runs in fp32 (ecache_pass1_f32)
// and is kept when the unit's max shows every weight that matters is inside the fp32
// error budget; otherwise (far measurements, tiny weights, S_j past shared memory) it is
// rerun with l_p in fp64, so the max shift keeps full accuracy.
//
// Pass 1 of the e-cache variant: per quad l_p (fp64; CENTRED: the centred quadratic form,
// else the general per-measurement loop); the thread's running max m rises to the quad's
// max (its parked e's, s and s2 rescaled by 2^(m_old - m_new)); e_p parked in shared memory.
template <bool CENTRED>
__device__ __forceinline__ void ecache_pass1(const ReweightArgs &a, const SList &S, int col, const float4 *xs,
                                             const float4 *ys, const float4 *ws, float4 *e4, int quads, float4 X,
                                             float4 Y, float4 W, const double *cq, double &m, float &sm,
                                             float &sm2) {
  int g = threadIdx.x;
#pragma unroll 1
  for (; g < quads; g += kThreads) {
    if (g != static_cast<int>(threadIdx.x)) {   // the first quad was loaded before the S scan
      X = __ldg(xs + g);
      Y = __ldg(ys + g);
      W = __ldg(ws + g);
    }
    double l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float px = q4(X, q), py = q4(Y, q), w = q4(W, q);
      if constexpr (CENTRED) {   // the unit's constants re-read from shared memory (registers are scarce)
        const double dx = cq[0] - static_cast<double>(px), dy = cq[1] - static_cast<double>(py);
        const double lw = w > 0.f ? static_cast<double>(__log2f(w)) : -INFINITY;
        l[q] = lw - fma(dx, fma(cq[2], dx, cq[3] * dy), cq[4] * dy * dy);
      } else {
        l[q] = log_weight(a, S, col, px, py, w);
      }
    }
    const double lq = fmax(fmax(l[0], l[1]), fmax(l[2], l[3]));
    if (lq > m) {
      if (m != -INFINITY) {
        const float f = ex2_approx(static_cast<float>(m - lq));
        sm *= f;
        sm2 *= f * f;
        for (int gp = threadIdx.x; gp < g; gp += kThreads) {
          float4 e = e4[gp];
          e.x *= f;
          e.y *= f;
          e.z *= f;
          e.w *= f;
          e4[gp] = e;
        }
      }
      m = lq;
    }
    float4 e;
#pragma unroll
    for (int q = 0; q < 4; ++q) q4(e, q) = l[q] == -INFINITY ? 0.0f : ex2_approx(static_cast<float>(l[q] - m));
    sm += (e.x + e.y) + (e.z + e.w);
    sm2 = fmaf(e.x, e.x, fmaf(e.y, e.y, fmaf(e.z, e.z, fmaf(e.w, e.w, sm2))));
    e4[g] = e;
  }
}

// Fast pass 1 of the e-cache variant, all fp32 (MUFU.LG2 + MUFU.EX2 per particle, no
// fp64 conversions): d = (p - zhi) - zlo with zbar = zhi + zlo split into two floats
// (p - zhi is exact by Sterbenz for nearby coordinates), q' = n d^T A d in fp32.  Its
// error is ~q' 2^-22; a weight matters only if l_p >= m - 100 (below that 2^(l - m) <
// 1e-30, the absolute tolerance), i.e. q' <= 100 - m, so once the unit's max m >= -300
// every weight that matters has q' <= 400 and a relative error <= 1e-4 / 2 -- the caller
// checks that and otherwise reruns pass 1 in fp64 (far measurements, tiny weights).
// The thread's running max starts at the warp's max over the first quads.
__device__ __forceinline__ void ecache_pass1_f32(const float4 *xs, const float4 *ys, const float4 *ws, float4 *e4,
                                                 int quads, float4 X, float4 Y, float4 W, const float *c32,
                                                 float &m, float &sm, float &sm2) {
  const float zhx = c32[0], zlx = c32[1], zhy = c32[2], zly = c32[3], na = c32[4], nb = c32[5], nc = c32[6];
  bool first = true;   // quads >= kThreads (P >= 1024): every lane has a first quad
  // two quads in flight ahead of the one computed (the loads of one thread are a serial
  // chain otherwise: one quad of prefetch left each iteration waiting on memory latency)
  float4 Xn, Yn, Wn, Xm, Ym, Wm;
  if (static_cast<int>(threadIdx.x) + kThreads < quads) {
    Xn = __ldg(xs + threadIdx.x + kThreads);
    Yn = __ldg(ys + threadIdx.x + kThreads);
    Wn = __ldg(ws + threadIdx.x + kThreads);
  }
#pragma unroll 1
  for (int g = threadIdx.x; g < quads; g += kThreads) {
    const int gm = g + 2 * kThreads;
    if (gm < quads) {
      Xm = __ldg(xs + gm);
      Ym = __ldg(ys + gm);
      Wm = __ldg(ws + gm);
    }
    float l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float dx = (q4(X, q) - zhx) - zlx, dy = (q4(Y, q) - zhy) - zly;
      const float w = q4(W, q);
      l[q] = w > 0.f ? __log2f(w) - fmaf(dx, fmaf(na, dx, nb * dy), nc * dy * dy) : -INFINITY;
    }
    const float lq = fmaxf(fmaxf(l[0], l[1]), fmaxf(l[2], l[3]));
    if (first) {
      float wm = lq;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
      m = wm;
      first = false;
    }
    if (lq > m) {
      if (m != -INFINITY) {
        const float f = ex2_approx(m - lq);
        sm *= f;
        sm2 *= f * f;
        for (int gp = threadIdx.x; gp < g; gp += kThreads) {
          float4 e = e4[gp];
          e.x *= f;
          e.y *= f;
          e.z *= f;
          e.w *= f;
          e4[gp] = e;
        }
      }
      m = lq;
    }
    float4 e;
#pragma unroll
    for (int q = 0; q < 4; ++q) q4(e, q) = l[q] == -INFINITY ? 0.0f : ex2_approx(l[q] - m);
    sm += (e.x + e.y) + (e.z + e.w);
    sm2 = fmaf(e.x, e.x, fmaf(e.y, e.y, fmaf(e.z, e.z, fmaf(e.w, e.w, sm2))));
    e4[g] = e;
    X = Xn;
    Y = Yn;
    W = Wn;
    Xn = Xm;
    Yn = Ym;
    Wn = Wm;
  }
}

__device__ __forceinline__ void reweight_ecache_unit(const ReweightArgs &a, const int u) {
  extern __shared__ __align__(16) float ec[];  // [P] e_p
  __shared__ SList S;
  __shared__ double red[3][kWarps];
  __shared__ uint32_t masks[kRows * kWarps];
  __shared__ double cq[6];   // zbar x, y; n qa, n qb, n qc; C0
  __shared__ float c32[7];   // zbar split into (hi, lo) floats for x and y; n qa, n qb, n qc
  const bool pairs = a.pair_track != nullptr;
  const int j = pairs ? __ldg(a.pair_track + u) : u;
  const int col = a.col_offset + j + 1;
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float4 *xs = reinterpret_cast<const float4 *>(a.x + base);
  const float4 *ys = reinterpret_cast<const float4 *>(a.y + base);
  const float4 *ws = reinterpret_cast<const float4 *>(a.w + base);
  float4 *wo = reinterpret_cast<float4 *>(a.w_out + static_cast<int64_t>(u) * a.ld_out);
  float4 *e4 = reinterpret_cast<float4 *>(ec);
  const bool copy_out = pairs || a.w_out != a.w;
  const int quads = a.P >> 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if GLMB_RW_DEBUG == 3   // A/B timing build: %globaltimer per phase, stored over the unit's first weights at the end
  __shared__ unsigned long long tst[8];
  auto stamp = [&](int k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tst[k] = t;
    }
  };
  stamp(0);
#else
  auto stamp = [](int) {};
#endif
  // the first quad's loads are issued before the S scan, so the two latencies overlap
  float4 X0, Y0, W0;
  if (static_cast<int>(threadIdx.x) < quads) {
    X0 = __ldg(xs + threadIdx.x);
    Y0 = __ldg(ys + threadIdx.x);
    W0 = __ldg(ws + threadIdx.x);
  }
  if (pairs) collect_S_pair(a, u, S);
  else collect_S(a, col, S, masks);
  const int nS = S.n;

  if (nS == 0) {  // untouched; log_norm = ln sum w; ESS = (sum w)^2 / sum w^2
    double sw = 0.0, sw2 = 0.0;
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      const float4 w4 = __ldcs(ws + g);
      if (copy_out) __stcs(wo + g, w4);
      sw += (static_cast<double>(w4.x) + w4.y) + (static_cast<double>(w4.z) + w4.w);
      sw2 += (static_cast<double>(w4.x) * w4.x + static_cast<double>(w4.y) * w4.y) +
             (static_cast<double>(w4.z) * w4.z + static_cast<double>(w4.w) * w4.w);
    }
    sw = block_sum(sw, red[0]);
    if (a.ess != nullptr) sw2 = block_sum(sw2, red[1]);
    if (threadIdx.x == 0) {
      a.log_norm[u] = static_cast<float>(log(sw));
      a.flags[u] = 0u;
      if (a.ess != nullptr) a.ess[u] = sw2 > 0.0 ? static_cast<float>(sw * sw / sw2) : 0.0f;
    }
    return;
  }
  const bool centred = S.in_smem;
  if (centred && threadIdx.x == 0) {
    double sx = 0.0, sy = 0.0;
    for (int k = 0; k < nS; ++k) {
      sx += S.z[k].x;
      sy += S.z[k].y;
    }
    const double zx = sx / nS, zy = sy / nS;
    double c0 = 0.0;
    for (int k = 0; k < nS; ++k) c0 += qform(a, S.z[k].x, S.z[k].y, zx, zy);
    cq[0] = zx;
    cq[1] = zy;
    cq[2] = nS * a.qa;
    cq[3] = nS * a.qb;
    cq[4] = nS * a.qc;
    cq[5] = c0;
    const float hx = static_cast<float>(zx), hy = static_cast<float>(zy);
    c32[0] = hx;
    c32[1] = static_cast<float>(zx - hx);
    c32[2] = hy;
    c32[3] = static_cast<float>(zy - hy);
    c32[4] = static_cast<float>(cq[2]);
    c32[5] = static_cast<float>(cq[3]);
    c32[6] = static_cast<float>(cq[4]);
  }
  __syncthreads();
  stamp(1);
  // warp: max by shuffles, the lanes' sums rescaled to it; CTA: after one barrier every
  // thread merges the warps' partials itself (same order everywhere: identical results)
  double mc = -INFINITY, sc = 0.0, s2c = 0.0;
  auto merge = [&](double m, float sm, float sm2) {
    const double mw = warp_max_d(m);
    const double f = mw == -INFINITY || m == -INFINITY ? 0.0 : static_cast<double>(ex2_approx(static_cast<float>(m - mw)));
    double sw = warp_sum_d(static_cast<double>(sm) * f),
           sw2 = a.ess != nullptr ? warp_sum_d(static_cast<double>(sm2) * (f * f)) : 0.0;
    if (lane == 0) {
      red[0][warp] = mw;
      red[1][warp] = sw;
      red[2][warp] = sw2;
    }
    __syncthreads();
    mc = red[0][0];
    sc = red[1][0];
    s2c = red[2][0];
#pragma unroll
    for (int k = 1; k < kWarps; ++k) ms_merge(mc, sc, s2c, red[0][k], red[1][k], red[2][k]);
  };
  // pass 1: fp32 when the centred form applies, kept when the unit's max shows every weight
  // that matters is within the fp32 error budget (see ecache_pass1_f32); else fp64
  double m = -INFINITY;
  float sm = 0.0f, sm2 = 0.0f;
  bool fp64 = !centred;
  if (centred) {
    float m32 = -INFINITY;
    ecache_pass1_f32(xs, ys, ws, e4, quads, X0, Y0, W0, c32, m32, sm, sm2);
    m = m32;
    stamp(2);
    merge(m, sm, sm2);
    stamp(3);
    fp64 = mc != -INFINITY && mc < -300.0;   // CTA-uniform
    if (fp64) __syncthreads();   // every thread has read red before the rerun's merge overwrites it
  }
  if (fp64) {
    m = -INFINITY;
    sm = sm2 = 0.0f;
    if (static_cast<int>(threadIdx.x) < quads) {
      X0 = __ldg(xs + threadIdx.x);
      Y0 = __ldg(ys + threadIdx.x);
      W0 = __ldg(ws + threadIdx.x);
    }
    if (centred) ecache_pass1<true>(a, S, col, xs, ys, ws, e4, quads, X0, Y0, W0, cq, m, sm, sm2);
    else ecache_pass1<false>(a, S, col, xs, ys, ws, e4, quads, X0, Y0, W0, cq, m, sm, sm2);
    merge(m, sm, sm2);
  }
  if (mc == -INFINITY) {  // every weight zero: uniform reset, flagged (never abort)
    const float uw = 1.0f / static_cast<float>(a.P);
    for (int g = threadIdx.x; g < quads; g += kThreads) __stcs(wo + g, make_float4(uw, uw, uw, uw));
    if (threadIdx.x == 0) {
      a.log_norm[u] = -INFINITY;
      a.flags[u] = 1u;
      if (a.ess != nullptr) a.ess[u] = static_cast<float>(a.P);
    }
    return;
  }
  // pass 2: w'_p = e_p 2^(m_t - m) / s from the thread's own parked entries
  const float ft = m == -INFINITY ? 0.0f : ex2_approx(static_cast<float>(m - mc)) * static_cast<float>(1.0 / sc);
  for (int g = threadIdx.x; g < quads; g += kThreads) {
    const float4 e = e4[g];
    __stcs(wo + g, make_float4(e.x * ft, e.y * ft, e.z * ft, e.w * ft));
  }
#if GLMB_RW_DEBUG == 3
  stamp(4);
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tst[5] = smid;
    tst[6] = fp64 ? 1ull : 0ull;
    for (int k = 0; k < 7; ++k) reinterpret_cast<unsigned long long *>(wo)[k] = tst[k];
  }
#endif
  if (threadIdx.x == 0) {
    const double ln2 = 0.69314718055994530942;
    const double c0 = centred ? cq[5] : 0.0;   // the centred form's constant term
    a.log_norm[u] = static_cast<float>((mc - c0 + log2(sc)) * ln2 - nS * a.log_norm1);
    a.flags[u] = 0u;
    if (a.ess != nullptr) a.ess[u] = static_cast<float>(sc * sc / s2c);
  }
}

__global__ void __launch_bounds__(kThreads, GLMB_RW_ECACHE_BLOCKS) reweight_ecache_kernel(const ReweightArgs a) {
  grid_dep_wait();
  const int n_units = a.n_units_dev != nullptr ? min(a.T, __ldg(a.n_units_dev)) : a.T;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    if (u != static_cast<int>(blockIdx.x)) __syncthreads();   // S, red, cq reused by the next unit
    reweight_ecache_unit(a, u);
  }
}

template <int CL, int R>
cudaError_t launch_cluster(const ReweightArgs &a, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  const int units = a.units_cap > 0 ? min(a.T, a.units_cap) : a.T;
  cfg.gridDim = dim3(static_cast<unsigned>(units) * CL);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (a.pair_track != nullptr && pdl_enabled()) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, reweight_cluster_kernel<CL, R>, a);
}

constexpr int kMaxCacheBytes = 100 * 1024;

}  // namespace

cudaError_t launch_reweight(const ReweightArgs &a, cudaStream_t s) {
  if (a.T == 0) return cudaSuccess;
  // default: the flat kernel with l_p cached in shared memory for 2048 <= P <= 12800
  // (measured at cfg3: 78 -> 51 us standalone; the cluster kernel stays best for small P).
  // GLMB_REWEIGHT_FLAT: 0 = cluster kernel, 1 = flat recompute, 2 = flat cached (A/B).
  static const int flat_env = [] {
    const char *e = std::getenv("GLMB_REWEIGHT_FLAT");
    return e ? std::atoi(e) : -1;
  }();
  const bool ecache_ok = a.P >= 4 * kThreads && static_cast<size_t>(a.P) * 4 <= kMaxCacheBytes;
  const bool ecache_default = flat_env < 0 && a.P >= 2048 && ecache_ok;
  if ((flat_env == 3 && ecache_ok) || ecache_default) {
    const int units = a.units_cap > 0 ? min(a.T, a.units_cap) : a.T;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(units));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cfg.dynamicSmemBytes = static_cast<size_t>(a.P) * 4;
    cudaError_t e = cudaFuncSetAttribute(reweight_ecache_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kMaxCacheBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (a.pair_track != nullptr && pdl_enabled()) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, reweight_ecache_kernel, a);
  }
  if (flat_env == 1 || flat_env == 2) {
    const int units = a.units_cap > 0 ? min(a.T, a.units_cap) : a.T;
    const bool lcache = flat_env != 1 && static_cast<size_t>(a.P) * 8 <= kMaxCacheBytes;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(units));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = s;
    cfg.dynamicSmemBytes = lcache ? static_cast<size_t>(a.P) * 8 : 0;
    if (lcache) {
      cudaError_t e = cudaFuncSetAttribute(reweight_flat_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kMaxCacheBytes);
      if (e != cudaSuccess) return e;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = (a.pair_track != nullptr && pdl_enabled()) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return lcache ? cudaLaunchKernelEx(&cfg, reweight_flat_kernel<true>, a)
                  : cudaLaunchKernelEx(&cfg, reweight_flat_kernel<false>, a);
  }
  // Launch shape depends on P only (never on T): shard-invariant results.
  const int quads = a.P >> 2;
  static const int rw_r = [] {  // quads per thread: 1 (more, lighter CTAs) or 2; A-B knob
    const char *e = std::getenv("GLMB_REWEIGHT_R");
    return e ? std::atoi(e) : 1;
  }();
  if (rw_r == 1) {
    if (quads <= 1 * kThreads) return launch_cluster<1, 1>(a, s);
    if (quads <= 2 * kThreads) return launch_cluster<2, 1>(a, s);
    if (quads <= 4 * kThreads) return launch_cluster<4, 1>(a, s);
    if (quads <= 8 * kThreads) return launch_cluster<8, 1>(a, s);
  }
  if (rw_r != 4) {
    if (quads <= 1 * kThreads * 2) return launch_cluster<1, 2>(a, s);
    if (quads <= 2 * kThreads * 2) return launch_cluster<2, 2>(a, s);
    if (quads <= 4 * kThreads * 2) return launch_cluster<4, 2>(a, s);
    if (quads <= 8 * kThreads * 2) return launch_cluster<8, 2>(a, s);
  }
  if (quads <= 1 * kThreads * 4) return launch_cluster<1, 4>(a, s);
  if (quads <= 2 * kThreads * 4) return launch_cluster<2, 4>(a, s);
  if (quads <= 4 * kThreads * 4) return launch_cluster<4, 4>(a, s);
  if (quads <= 8 * kThreads * 4) return launch_cluster<8, 4>(a, s);
  const size_t cache = static_cast<size_t>(a.P) * sizeof(double);
  if (cache <= kMaxCacheBytes) {
    static bool attr_set[64] = {};  // per device; benign race: idempotent attribute
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaError_t e = cudaFuncSetAttribute(reweight_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kMaxCacheBytes);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
    reweight_kernel<true><<<a.T, kThreads, cache, s>>>(a);
  } else {
    reweight_kernel<false><<<a.T, kThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace glmb
