// reweight.cu -- glmb_reweight: Bayes update of each track's particle weights
// under the supplied association map theta_k (§Approach).
//
//   S_j = {i : theta_i = col_offset + j + 1}
//   l_p = log2 w_p - sum_{i in S_j} 1/2 log2(e) d_ip^T R^-1 d_ip      (log2 domain)
//   m = max_p l_p,  s = sum_p 2^(l_p - m),  w'_p = 2^(l_p - m) / s
//   log_norm_j = (m + log2 s) ln 2 - |S_j| ln(2 pi sqrt(det R))
//
// One CTA (256 threads) per track.  HBM-bound: x, y, w are read once and w
// written once (16 B per particle).  The exponent l_p is accumulated in fp64
// (a handful of DFMA per particle-measurement, negligible next to the HBM
// time) so the max-shift l_p - m keeps full relative accuracy even when the
// assigned measurement is far from the cloud; 2^(l-m) itself is fp32 MUFU.
// Particles are cached in registers (R float4 quads per thread, P <= 1024 R)
// so the two passes (block max, then block sum) read HBM once; larger P uses
// the generic path that recomputes l_p in the second pass.
// Block reductions run in a fixed order -> deterministic, shard-invariant.
#include <cfloat>

#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSCap = 1024;  // assigned measurements held in shared memory

struct SList {
  double2 z[kSCap];
  int n;           // |S_j|
  int in_smem;     // 1 if all of S_j fits in z[]
};

// Collect S_j in ascending i with warp 0 (ballot + popc prefix).
__device__ void collect_S(const ReweightArgs &a, int col, SList &S) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int n = 0;
    for (int base = 0; base < a.M; base += 32) {
      const int i = base + lane;
      const bool hit = (i < a.M) && (__ldg(a.theta + i) == col);
      const uint32_t mask = __ballot_sync(0xffffffffu, hit);
      if (hit) {
        const int pos = n + __popc(mask & ((1u << lane) - 1u));
        if (pos < kSCap) {
          const float2 z = __ldg(reinterpret_cast<const float2 *>(a.Z) + i);
          S.z[pos] = make_double2(z.x, z.y);
        }
      }
      n += __popc(mask);
    }
    if (lane == 0) {
      S.n = n;
      S.in_smem = n <= kSCap;
    }
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
  double l = w > 0.f ? static_cast<double>(log2f(w)) : -INFINITY;
  const double dpx = px, dpy = py;
  if (S.in_smem) {
    for (int s = 0; s < S.n; ++s) l -= qform(a, S.z[s].x, S.z[s].y, dpx, dpy);
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

// R > 0: register-cached path (P <= 1024 R).  R == 0: generic recompute path.
template <int R>
__global__ void __launch_bounds__(kThreads) reweight_kernel(const ReweightArgs a) {
  __shared__ SList S;
  __shared__ double red[kWarps];
  const int j = blockIdx.x;
  const int col = a.col_offset + j + 1;
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float *xs = a.x + base, *ys = a.y + base;
  float *ws = a.w + base;
  const int quads = a.P >> 2;

  collect_S(a, col, S);
  const int nS = S.n;

  if (nS == 0) {  // untouched; log_norm = ln sum w
    double s = 0.0;
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      const float4 w4 = __ldcs(reinterpret_cast<const float4 *>(ws) + g);
      s += (static_cast<double>(w4.x) + w4.y) + (static_cast<double>(w4.z) + w4.w);
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      a.log_norm[j] = static_cast<float>(log(s));
      a.flags[j] = 0u;
    }
    return;
  }

  double m;
  double lc[R > 0 ? 4 * R : 1];
  if constexpr (R > 0) {
    double lm = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = threadIdx.x + r * kThreads;
      if (g < quads) {
        float4 X = __ldcs(reinterpret_cast<const float4 *>(xs) + g);
        float4 Y = __ldcs(reinterpret_cast<const float4 *>(ys) + g);
        float4 Wv = __ldcs(reinterpret_cast<const float4 *>(ws) + g);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          lc[4 * r + q] = log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q));
          lm = fmax(lm, lc[4 * r + q]);
        }
      }
    }
    m = block_max(lm, red);
  } else {
    double lm = -INFINITY;
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      float4 X = __ldcs(reinterpret_cast<const float4 *>(xs) + g);
      float4 Y = __ldcs(reinterpret_cast<const float4 *>(ys) + g);
      float4 Wv = __ldcs(reinterpret_cast<const float4 *>(ws) + g);
#pragma unroll
      for (int q = 0; q < 4; ++q) lm = fmax(lm, log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q)));
    }
    m = block_max(lm, red);
  }

  if (m == -INFINITY) {  // every weight zero: uniform reset, flagged (never abort)
    const float u = 1.0f / static_cast<float>(a.P);
    for (int g = threadIdx.x; g < quads; g += kThreads)
      __stcs(reinterpret_cast<float4 *>(ws) + g, make_float4(u, u, u, u));
    if (threadIdx.x == 0) {
      a.log_norm[j] = -INFINITY;
      a.flags[j] = 1u;
    }
    return;
  }

  // pass 2: s = sum 2^(l - m)
  double s = 0.0;
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = threadIdx.x + r * kThreads;
      if (g < quads) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float e = ex2_approx(static_cast<float>(lc[4 * r + q] - m));
          lc[4 * r + q] = e;
          s += e;
        }
      }
    }
  } else {
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      float4 X = __ldcs(reinterpret_cast<const float4 *>(xs) + g);
      float4 Y = __ldcs(reinterpret_cast<const float4 *>(ys) + g);
      float4 Wv = __ldcs(reinterpret_cast<const float4 *>(ws) + g);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        s += ex2_approx(static_cast<float>(log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q)) - m));
    }
  }
  s = block_sum(s, red);
  const float inv_s = static_cast<float>(1.0 / s);

  // pass 3: write w'
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int g = threadIdx.x + r * kThreads;
      if (g < quads) {
        float4 o;
#pragma unroll
        for (int q = 0; q < 4; ++q) q4(o, q) = static_cast<float>(lc[4 * r + q]) * inv_s;
        __stcs(reinterpret_cast<float4 *>(ws) + g, o);
      }
    }
  } else {
    for (int g = threadIdx.x; g < quads; g += kThreads) {
      float4 X = __ldcs(reinterpret_cast<const float4 *>(xs) + g);
      float4 Y = __ldcs(reinterpret_cast<const float4 *>(ys) + g);
      float4 Wv = __ldcs(reinterpret_cast<const float4 *>(ws) + g);
      float4 o;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        q4(o, q) = ex2_approx(static_cast<float>(log_weight(a, S, col, q4(X, q), q4(Y, q), q4(Wv, q)) - m)) * inv_s;
      __stcs(reinterpret_cast<float4 *>(ws) + g, o);
    }
  }
  if (threadIdx.x == 0) {
    const double ln2 = 0.69314718055994530942;
    a.log_norm[j] = static_cast<float>((m + log2(s)) * ln2 - nS * a.log_norm1);
    a.flags[j] = 0u;
  }
}

template <int R>
cudaError_t launch_r(const ReweightArgs &a, cudaStream_t s) {
  reweight_kernel<R><<<a.T, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reweight(const ReweightArgs &a, cudaStream_t s) {
  if (a.T == 0) return cudaSuccess;
  const int quads_per_thread = ((a.P >> 2) + kThreads - 1) / kThreads;
  if (quads_per_thread <= 1) return launch_r<1>(a, s);
  if (quads_per_thread <= 2) return launch_r<2>(a, s);
  if (quads_per_thread <= 4) return launch_r<4>(a, s);
  if (quads_per_thread <= 8) return launch_r<8>(a, s);
  return launch_r<0>(a, s);
}

}  // namespace glmb
