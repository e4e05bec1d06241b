// compat.cu -- glmb_compat: fused particle-mixture likelihood, gate and C_k.
//
//   L_ij = sum_p w_jp N(z_i; (x_jp, y_jp), R),  g_ij = [L_ij >= gamma],
//   C[i, j+1] = g_ij P_D L_ij,  C[i, 0] = kappa          (§Approach)
//
// Design: the work is M*T*P independent Gaussian
// evaluations -- one exp per pair, bound by the SFU (MUFU.EX2) pipe, not by
// HBM and not a dense contraction (no tensor cores).
//  * One CTA (4 warps) = one (track j, measurement tile of 128*K) unit; warp w
//    owns the contiguous measurements m0 + 32Kw + 32k + lane (k < K) in
//    registers, so every measurement's sum over the particles is completed by
//    one thread in a fixed order -- no cross-thread reduction, and C is
//    bit-identical for any sharding of the tracks and any permutation of Z's
//    rows.  Warps past M skip the arithmetic; the ragged last measurement
//    tiles are scheduled last (unit = mt*T + j) to fill the tail.
//  * The track's particles stream through shared memory in tiles of
//    kTileP, moved by the TMA bulk-copy engine (cp.async.bulk + mbarrier,
//    kStages-deep ring) and reused by all 128*K measurements of the CTA.
//  * Each tile is whitened once in place (X' = a1(x-cx) + a2(y-cy),
//    Y' = b2(y-cy), centred on the track's first particle so the fp32
//    subtraction of large coordinates is exact), which turns
//    1/2 log2(e) d^T R^-1 d into |d'|^2 for any SPD R.  Per pair the inner
//    loop is then FADD2 dx, FADD2 dy, FMUL2, FFMA2, MUFU.EX2, FFMA2 acc on
//    packed fp32x2 (two particles per instruction).
//  * Two-level summation (per tile, then across tiles) keeps the fp32 sum
//    error ~kTileP/2*eps instead of P/2*eps.
//  * Epilogue: L = norm*sum, gate bit via __ballot_sync (32 consecutive
//    measurements of a warp = one gate word), coalesced C stores.
#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr int kThreads = 128;
constexpr int kTileP = 512;   // particles per shared-memory stage (fixed: sets the sum order)
constexpr int kStages = 4;    // TMA ring depth
constexpr int kMaxK = 4;
constexpr int kSmemBytes = kStages * 3 * kTileP * 4;

__device__ __forceinline__ void issue_tile(const CompatArgs &a, const float *xs, const float *ys, const float *ws,
                                           float *stage, uint64_t *bar, int t) {
  const int p0 = t * kTileP;
  const int np = min(kTileP, a.P - p0);
  const uint32_t bytes = static_cast<uint32_t>(np) * 4u;  // P % 4 == 0 -> multiple of 16
  mbar_arrive_expect_tx(bar, 3u * bytes);
  bulk_g2s(stage, xs + p0, bytes, bar);
  bulk_g2s(stage + kTileP, ys + p0, bytes, bar);
  bulk_g2s(stage + 2 * kTileP, ws + p0, bytes, bar);
}

// Sum over one shared-memory tile for this warp's first KV measurement slices.
template <int K, int KV>
__device__ __forceinline__ void tile_pairs(const float2 *__restrict__ X2, const float2 *__restrict__ Y2,
                                           const float2 *__restrict__ W2, int npairs, const float (&zx)[K],
                                           const float (&zy)[K], float (&tot)[K]) {
  f2 acc[KV];
#pragma unroll
  for (int k = 0; k < KV; ++k) acc[k] = 0ull;
#pragma unroll 2
  for (int q = 0; q < npairs; ++q) {
    const float2 xv = X2[q], yv = Y2[q], wv = W2[q];
    const f2 px = f2_pack(xv.x, xv.y), py = f2_pack(yv.x, yv.y), pw = f2_pack(wv.x, wv.y);
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const f2 dx = f2_sub(f2_pack(zx[k], zx[k]), px);
      const f2 dy = f2_sub(f2_pack(zy[k], zy[k]), py);
      const f2 qq = f2_fma(dy, dy, f2_mul(dx, dx));
      float q0, q1;
      f2_unpack(qq, q0, q1);
      acc[k] = f2_fma(pw, f2_pack(ex2_approx(-q0), ex2_approx(-q1)), acc[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    float lo, hi;
    f2_unpack(acc[k], lo, hi);
    tot[k] += lo + hi;
  }
}

template <int K>
__device__ __forceinline__ void tile_dispatch(int kv, const float *X, const float *Y, const float *W, int npairs,
                                              const float (&zx)[K], const float (&zy)[K], float (&tot)[K]) {
  const float2 *X2 = reinterpret_cast<const float2 *>(X);
  const float2 *Y2 = reinterpret_cast<const float2 *>(Y);
  const float2 *W2 = reinterpret_cast<const float2 *>(W);
  if (kv == K) {
    tile_pairs<K, K>(X2, Y2, W2, npairs, zx, zy, tot);
  } else {
    if constexpr (K > 1) if (kv == 1) tile_pairs<K, 1>(X2, Y2, W2, npairs, zx, zy, tot);
    if constexpr (K > 2) if (kv == 2) tile_pairs<K, (K > 2 ? 2 : 1)>(X2, Y2, W2, npairs, zx, zy, tot);
    if constexpr (K > 3) if (kv == 3) tile_pairs<K, (K > 3 ? 3 : 1)>(X2, Y2, W2, npairs, zx, zy, tot);
    if constexpr (K > 4) {
      if (kv == 4) tile_pairs<K, 4>(X2, Y2, W2, npairs, zx, zy, tot);
      if (kv == 5) tile_pairs<K, (K > 5 ? 5 : 4)>(X2, Y2, W2, npairs, zx, zy, tot);
      if (kv == 6) tile_pairs<K, (K > 6 ? 6 : 4)>(X2, Y2, W2, npairs, zx, zy, tot);
      if (kv == 7) tile_pairs<K, (K > 7 ? 7 : 4)>(X2, Y2, W2, npairs, zx, zy, tot);
    }
  }
}

// Unit u = mt * T + j (all full measurement tiles first, the ragged last tiles
// at the end of the grid, so the short units fill the tail of the schedule).
// Warp w owns the contiguous measurements m0 + w*32K + k*32 + lane, k < K.
template <int K>
__global__ void __launch_bounds__(kThreads) compat_kernel(const CompatArgs a) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[kStages];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mt = blockIdx.x / a.T;
  const int j = blockIdx.x - mt * a.T;
  const int wbase = mt * (kThreads * K) + warp * (32 * K);  // first measurement of this warp
  const int kv = min(K, max(0, (a.M - wbase + 31) >> 5));   // measurement slices with any valid lane
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float *xs = a.x + base, *ys = a.y + base, *ws = a.w + base;
  const int ntiles = (a.P + kTileP - 1) / kTileP;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < kStages && s < ntiles; ++s) issue_tile(a, xs, ys, ws, smem + s * 3 * kTileP, &bars[s], s);
  }

  const float cx = __ldg(xs), cy = __ldg(ys);  // centre: the track's first particle
  float zx[K], zy[K], tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = wbase + k * 32 + lane;
    zx[k] = 0.f;
    zy[k] = 0.f;
    if (i < a.M) {
      const float2 z = __ldg(reinterpret_cast<const float2 *>(a.Z) + i);
      const float lx = z.x - cx, ly = z.y - cy;
      zx[k] = fmaf(a.a2, ly, a.a1 * lx);
      zy[k] = a.b2 * ly;
    }
    tot[k] = 0.f;
  }

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % kStages;
    float *X = smem + s * 3 * kTileP;
    float *Y = X + kTileP;
    const float *W = Y + kTileP;
    const int np = min(kTileP, a.P - t * kTileP);
    mbar_wait_parity(&bars[s], static_cast<uint32_t>(t / kStages) & 1u);
    for (int idx = tid; idx < np; idx += kThreads) {  // whiten in place
      const float lx = X[idx] - cx, ly = Y[idx] - cy;
      X[idx] = fmaf(a.a2, ly, a.a1 * lx);
      Y[idx] = a.b2 * ly;
    }
    __syncthreads();
    if (kv > 0) tile_dispatch<K>(kv, X, Y, W, np >> 1, zx, zy, tot);
    fence_proxy_async_smem();  // order this CTA's generic smem accesses before the next TMA write
    __syncthreads();
    if (tid == 0 && t + kStages < ntiles) issue_tile(a, xs, ys, ws, X, &bars[s], t + kStages);
  }

  // epilogue: likelihood, gate bit, C entry, clutter column
  if (kv == 0) return;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < kv) {
      const int i = wbase + k * 32 + lane;
      const bool valid = i < a.M;
      const float L = tot[k] * a.norm;
      const bool g = valid && (L >= a.gamma);
      if (valid) a.C_tracks[static_cast<int64_t>(j) * a.ldc + i] = g ? a.p_d * L : 0.0f;
      const uint32_t word = __ballot_sync(0xffffffffu, g);
      if (lane == 0) a.gate[static_cast<int64_t>(j) * a.ldg + ((wbase + k * 32) >> 5)] = word;
      if (j == 0 && a.C_clutter != nullptr && valid) a.C_clutter[i] = a.kappa;
    }
  }
}

__global__ void clutter_fill_kernel(float *c, int32_t M, float kappa) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) c[i] = kappa;
}

template <int K>
cudaError_t launch_k(const CompatArgs &a, cudaStream_t s) {
  const int64_t grid = static_cast<int64_t>(a.T) * a.n_mtiles;
  compat_kernel<K><<<static_cast<unsigned>(grid), kThreads, kSmemBytes, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

void compat_plan(int32_t M, int32_t P, int32_t *K, int32_t *n_mtiles) {
  // Depends on (M, P) only -- never on T -- so any sharding of the tracks runs
  // the same per-column code (bit-identical C).  Measurements per thread K = 4
  // (tile of 512) for large M; small M uses the smallest K covering M.
  (void)P;
  int32_t k = kMaxK;
  const int32_t warps_needed = (M + 31) / 32;
  while (k > 1 && warps_needed <= (kThreads / 32) * (k / 2)) k /= 2;
  *K = k;
  *n_mtiles = (M + kThreads * k - 1) / (kThreads * k);
}

cudaError_t launch_compat(const CompatArgs &a, cudaStream_t s) {
  switch (a.K) {
    case 1: return launch_k<1>(a, s);
    case 2: return launch_k<2>(a, s);
    case 4: return launch_k<4>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_clutter_fill(float *C_clutter, int32_t M, float kappa, cudaStream_t s) {
  if (M == 0 || C_clutter == nullptr) return cudaSuccess;
  clutter_fill_kernel<<<(M + 255) / 256, 256, 0, s>>>(C_clutter, M, kappa);
  return cudaGetLastError();
}

}  // namespace glmb
