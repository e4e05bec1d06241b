// compat.cu -- glmb_compat: fused particle-mixture likelihood, gate and C_k.
//
//   L_ij = sum_p w_jp N(z_i; (x_jp, y_jp), R),  g_ij = [L_ij >= gamma],
//   C[i, j+1] = g_ij P_D L_ij,  C[i, 0] = kappa          (§Approach)
//
// Design: the work is M*T*P independent Gaussian
// evaluations -- one exp per pair, bound by the SFU (MUFU.EX2) pipe, not by
// HBM and not a dense contraction (no tensor cores).
//  * One CTA = one (track j, measurement tile of 128*K) unit; each thread
//    owns K measurements (i = m0 + k*128 + tid) in registers, so every
//    measurement's sum over the particles is completed by one thread in a
//    fixed order -- no cross-thread reduction, and C is bit-identical for any
//    sharding of the tracks and any permutation of Z's rows.
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
constexpr int kMaxK = 8;
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

template <int K>
__global__ void __launch_bounds__(kThreads) compat_kernel(const CompatArgs a) {
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[kStages];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = blockIdx.x / a.n_mtiles;
  const int mt = blockIdx.x - j * a.n_mtiles;
  const int m0 = mt * (kThreads * K);
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
  f2 zx2[K], zy2[K];
  float tot[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = m0 + k * kThreads + tid;
    float zx = 0.f, zy = 0.f;
    if (i < a.M) {
      const float2 z = __ldg(reinterpret_cast<const float2 *>(a.Z) + i);
      const float lx = z.x - cx, ly = z.y - cy;
      zx = fmaf(a.a2, ly, a.a1 * lx);
      zy = a.b2 * ly;
    }
    zx2[k] = f2_pack(zx, zx);
    zy2[k] = f2_pack(zy, zy);
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

    f2 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0ull;
    const float2 *X2 = reinterpret_cast<const float2 *>(X);
    const float2 *Y2 = reinterpret_cast<const float2 *>(Y);
    const float2 *W2 = reinterpret_cast<const float2 *>(W);
    const int npairs = np >> 1;
#pragma unroll 2
    for (int q = 0; q < npairs; ++q) {
      const float2 xv = X2[q], yv = Y2[q], wv = W2[q];
      const f2 px = f2_pack(xv.x, xv.y), py = f2_pack(yv.x, yv.y), pw = f2_pack(wv.x, wv.y);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const f2 dx = f2_sub(zx2[k], px);
        const f2 dy = f2_sub(zy2[k], py);
        const f2 qq = f2_fma(dy, dy, f2_mul(dx, dx));
        float q0, q1;
        f2_unpack(qq, q0, q1);
        acc[k] = f2_fma(pw, f2_pack(ex2_approx(-q0), ex2_approx(-q1)), acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float lo, hi;
      f2_unpack(acc[k], lo, hi);
      tot[k] += lo + hi;
    }
    fence_proxy_async_smem();  // order this CTA's generic smem accesses before the next TMA write
    __syncthreads();
    if (tid == 0 && t + kStages < ntiles) issue_tile(a, xs, ys, ws, X, &bars[s], t + kStages);
  }

  // epilogue: likelihood, gate bit, C entry, clutter column
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int i = m0 + k * kThreads + tid;
    const bool valid = i < a.M;
    const float L = tot[k] * a.norm;
    const bool g = valid && (L >= a.gamma);
    if (valid) a.C_tracks[static_cast<int64_t>(j) * a.ldc + i] = g ? a.p_d * L : 0.0f;
    const uint32_t word = __ballot_sync(0xffffffffu, g);
    const int wi = (m0 + k * kThreads + warp * 32) >> 5;
    if (lane == 0 && wi * 32 < a.M) a.gate[static_cast<int64_t>(j) * a.ldg + wi] = word;
    if (j == 0 && a.C_clutter != nullptr && valid) a.C_clutter[i] = a.kappa;
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
  (void)P;
  const int32_t per_tile_max = kThreads * kMaxK;
  int32_t nt = (M + per_tile_max - 1) / per_tile_max;
  if (nt < 1) nt = 1;
  const int32_t per_tile = (M + nt - 1) / nt;
  int32_t k = (per_tile + kThreads - 1) / kThreads;
  if (k < 1) k = 1;
  *K = k;
  *n_mtiles = (M + kThreads * k - 1) / (kThreads * k);
}

cudaError_t launch_compat(const CompatArgs &a, cudaStream_t s) {
  switch (a.K) {
    case 1: return launch_k<1>(a, s);
    case 2: return launch_k<2>(a, s);
    case 3: return launch_k<3>(a, s);
    case 4: return launch_k<4>(a, s);
    case 5: return launch_k<5>(a, s);
    case 6: return launch_k<6>(a, s);
    case 7: return launch_k<7>(a, s);
    case 8: return launch_k<8>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_clutter_fill(float *C_clutter, int32_t M, float kappa, cudaStream_t s) {
  if (M == 0 || C_clutter == nullptr) return cudaSuccess;
  clutter_fill_kernel<<<(M + 255) / 256, 256, 0, s>>>(C_clutter, M, kappa);
  return cudaGetLastError();
}

}  // namespace glmb
