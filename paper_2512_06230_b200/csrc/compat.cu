// compat.cu -- glmb_compat: fused particle-mixture likelihood, gate and C_k.
//
//   L_ij = sum_p w_jp N(z_i; (x_jp, y_jp), R),  g_ij = [L_ij >= gamma],
//   C[i, j+1] = g_ij P_D L_ij,  C[i, 0] = kappa          (§Approach)
//
// Design: the work is M*T*P independent Gaussian
// evaluations -- one exp per pair.  It is bound by the exp throughput of the
// SM (MUFU.EX2, 16/clk/SM measured), not by HBM and not a dense contraction
// (no tensor cores: see DESIGN.md for why q = |z|^2 - 2 z.p + |p|^2 as a
// K=4 GEMM would not survive tf32/bf16 at these coordinates).
//  * One CTA (4 warps) = one (track j, measurement tile of 128*K) unit; warp w
//    owns the contiguous measurements m0 + 32Kw + 32k + lane (k < K) in
//    registers, so every measurement's sum over the particles is completed by
//    one thread in a fixed particle order -- no cross-thread reduction, and C
//    is bit-identical for any sharding of the tracks and any permutation of
//    Z's rows.  Warps past M skip the arithmetic; the ragged last measurement
//    tiles are scheduled last (unit = mt*T + j) to fill the tail.  K = 2 and
//    40 registers give 12 resident CTAs (48 warps) per SM.
//  * The track's particles stream through shared memory in tiles of kTileP,
//    moved by the TMA bulk-copy engine (cp.async.bulk + mbarrier) and reused
//    by all 128*K measurements of the CTA; one tile of arithmetic (~50 us per
//    CTA) hides the next tile's copy, so a single raw stage suffices.
//  * Whitening: with U' the scaled Cholesky factor of R^-1,
//    1/2 log2(e) d^T R^-1 d = |U'(z - c) - U'(p - c)|^2 for any SPD R, where c
//    is the mean of the track's first tile (so p - c and z - c are exact or
//    small even at 4 km coordinates).  Each raw tile is whitened once into an
//    AoS float4 tile (X', Y', -, w), double buffered so one __syncthreads per
//    tile suffices.
//  * Inner loop: one LDS.128 per particle; the thread's measurements are
//    packed in pairs (fp32x2), the particle's values are scalar operands that
//    FFMA2 broadcasts: dx, dy = z' - p' exactly as in the definition (no
//    |z|^2 - 2z.p + |p|^2 expansion, whose cancellation grows with the cloud
//    width), q = dx^2 + dy^2, acc += w 2^-q.  One particle in 10 (default;
//    GLMB_COMPAT_EMU) evaluates its exps on the FMA pipe instead of MUFU
//    (round-to-nearest range reduction with the 1.5*2^23 trick, degree-4
//    near-minimax polynomial, rel. error 2.7e-6, exponent added with an integer shift-add, scaled by 2^64 so
//    tiny results flush to zero like MUFU.EX2.FTZ), which offloads the MUFU
//    pipe.  The choice is by particle index, so
//    every measurement sees the same arithmetic (row-permutation bit-exact).
//  * Two-level summation (per tile, then across tiles) keeps the fp32 sum
//    error ~kTileP*eps instead of P*eps.
//  * Epilogue: L = norm*sum, gate bit via __ballot_sync (32 consecutive
//    measurements of a warp = one gate word), coalesced C stores.
#include <cstdlib>

#include <cooperative_groups.h>

#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr int kVWarps = 4;  // the centre sum is defined over 4 (virtual) warps of 32 threads
constexpr int kTileP = 256;          // particles per shared-memory tile (fixed: sets the sum order)
constexpr int kStages = 1;           // raw tiles (x, y, w) in flight: one tile of compute (~50 us) hides a TMA
constexpr int kMaxK = 8;
// resident CTAs per SM the register allocation must allow (4 warps each)
template <int NW, int K>
constexpr int min_blocks() { return NW == 4 ? (K <= 2 ? 12 : 8) : (NW == 2 ? 20 : 28); }
constexpr int kRawFloats = 3 * kTileP;
constexpr int kSmemBytes = kStages * kRawFloats * 4 + 2 * kTileP * 16;  // raw ring + 2 AoS tiles

// degree-4 near-minimax fit of 2^f on [-1/2, 1/2] (max rel. error 2.6e-6, 2.7e-6 in fp32
// Horner): one FFMA2 fewer than degree 5 on the FMA pipe; the polynomial covers 1 particle in
// 10, so C's relative error from it is <= 2.7e-6 (the contract is 1e-4)
constexpr float kC0 = 0.999999261416315f, kC1 = 0.6931218155360352f, kC2 = 0.24024745060218355f,
                kC3 = 0.05591785367459349f, kC4 = 0.009570086922274257f;
constexpr float kRound64 = 12582976.0f;  // 1.5 * 2^23 + 64: x + kRound64 = round(x) + 64 in the low bits
constexpr float kTwoM64 = 5.42101086242752217e-20f;  // 2^-64

// 2^-q for a packed pair on the FMA + ALU pipes (no MUFU), returned scaled by
// 2^64 (the caller folds 2^-64 into the weight, so results below 2^-126 flush
// to zero exactly as MUFU.EX2.FTZ does).  q >= 0 is clamped at 189 so the
// integer exponent 64 - round(q) >= -125 stays a valid float exponent.
__device__ __forceinline__ f2 exp2_poly2_x64_neg(f2 q) {
  float q0, q1;
  f2_unpack(q, q0, q1);
  const f2 e = f2_pack(-fminf(q0, 189.0f), -fminf(q1, 189.0f));
  const f2 rnd = f2_pack(kRound64, kRound64);
  const f2 t = f2_add(e, rnd);             // low mantissa bits of t = round(e) + 64
  const f2 f = f2_sub(e, f2_sub(t, rnd));  // f = e - round(e) in [-1/2, 1/2]
  f2 p = f2_fma(f2_pack(kC4, kC4), f, f2_pack(kC3, kC3));
  p = f2_fma(p, f, f2_pack(kC2, kC2));
  p = f2_fma(p, f, f2_pack(kC1, kC1));
  p = f2_fma(p, f, f2_pack(kC0, kC0));
  float p0, p1, t0, t1;
  f2_unpack(p, p0, p1);
  f2_unpack(t, t0, t1);
  // << 23 moves round(e) + 64 into the exponent field of p in [2^-1/2, 2^1/2]
  p0 = __uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23));
  p1 = __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23));
  return f2_pack(p0, p1);
}

// Scalar mirrors of the packed ops (the same PTX rounding, no contraction): one lane of a
// packed pair computed alone gives the packed result's bits for that lane.
__device__ __forceinline__ float f1_add(float a, float b) {
  float r;
  asm("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float f1_sub(float a, float b) {
  float r;
  asm("sub.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float f1_mul(float a, float b) {
  float r;
  asm("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float f1_fma(float a, float b, float c) {
  float r;
  asm("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// exp2_poly2_x64_neg for one lane
__device__ __forceinline__ float exp2_poly1_x64_neg(float q) {
  const float e = -fminf(q, 189.0f);
  const float t = f1_add(e, kRound64);
  const float f = f1_sub(e, f1_sub(t, kRound64));
  float p = f1_fma(kC4, f, kC3);
  p = f1_fma(p, f, kC2);
  p = f1_fma(p, f, kC1);
  p = f1_fma(p, f, kC0);
  return __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23));
}

// 2^-q on MUFU.EX2 (the negation is an operand modifier)
__device__ __forceinline__ f2 exp2_mufu2_neg(f2 q) {
  float q0, q1;
  f2_unpack(q, q0, q1);
  return f2_pack(ex2_approx(-q0), ex2_approx(-q1));
}

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

// Per-thread measurements, packed in pairs (slot 2h, 2h+1 -> lane halves).
template <int K>
struct Meas {
  static constexpr int H = (K + 1) / 2;
  f2 zx2[H], zy2[H];         // 2 z'x, 2 z'y
  float tot[2 * H];          // running sums per measurement slot
};

// One particle against the thread's HV measurement pairs.  POLY_MASK bit h:
// pair h takes 2^e from the FMA-pipe polynomial instead of MUFU.
// AoS entry p = (X', Y', w 2^-64, w).  e = -|z' - p'|^2 from the exact difference
// (z' = zx2 / 2 exactly): dx, dy by FFMA2, q by FMUL2 + FFMA2; the sign of -q is
// an operand modifier of MUFU / the polynomial's adds.
template <int H, int POLY_MASK, bool LO = false>
__device__ __forceinline__ void particle_step(const float4 p, const f2 (&zx2)[H], const f2 (&zy2)[H],
                                              f2 (&acc)[H], int hv) {
  if constexpr (LO) {   // H == 1 and only the pair's low slot holds measurements: that lane alone
    float zx, zxh, zy, zyh, a0, a1;
    f2_unpack(zx2[0], zx, zxh);
    f2_unpack(zy2[0], zy, zyh);
    f2_unpack(acc[0], a0, a1);
    const float dx = f1_fma(zx, 0.5f, -p.x), dy = f1_fma(zy, 0.5f, -p.y);
    const float q = f1_fma(dy, dy, f1_mul(dx, dx));
    if (POLY_MASK & 1) a0 = f1_fma(p.z, exp2_poly1_x64_neg(q), a0);
    else a0 = f1_fma(p.w, ex2_approx(-q), a0);
    acc[0] = f2_pack(a0, a1);
    return;
  }
  const f2 pw = f2_pack(p.w, p.w);
  const f2 half = f2_pack(0.5f, 0.5f);
  const f2 npx = f2_pack(-p.x, -p.x), npy = f2_pack(-p.y, -p.y);
#pragma unroll
  for (int h = 0; h < H; ++h) {
    if (h < hv) {
      const f2 dx = f2_fma(zx2[h], half, npx);  // z'x - p'x
      const f2 dy = f2_fma(zy2[h], half, npy);
      const f2 q = f2_fma(dy, dy, f2_mul(dx, dx));
      if ((POLY_MASK >> h) & 1) {
        const f2 pw64 = f2_pack(p.z, p.z);  // w 2^-64, precomputed in the tile
        acc[h] = f2_fma(pw64, exp2_poly2_x64_neg(q), acc[h]);
      } else {
        acc[h] = f2_fma(pw, exp2_mufu2_neg(q), acc[h]);
      }
    }
  }
}

// Mask of the pairs that use the polynomial for particle u of an EMU_PERIOD group:
// pair h is emulated when (u + 2h) % EMU_PERIOD == EMU_PERIOD - 1, so the
// polynomial work is spread over the group instead of bunched on one particle.
template <int EMU_PERIOD, int H>
constexpr int poly_mask(int u) {
  int m = 0;
  if (EMU_PERIOD < 0) {  // bunched: every pair of particle |P|-1 (pair-independent choice)
    if (u == -EMU_PERIOD - 1) m = (1 << H) - 1;
    return m;
  }
  for (int h = 0; h < H; ++h)
    if (EMU_PERIOD > 0 && (u + 2 * h) % EMU_PERIOD == EMU_PERIOD - 1) m |= 1 << h;
  return m;
}

template <int H, int EMU_PERIOD, bool LO, int U = 0>
__device__ __forceinline__ void step_u(int u, const float4 p, const f2 (&zx2)[H], const f2 (&zy2)[H],
                                       f2 (&acc)[H], int hv) {
  // u is a compile-time constant after unrolling; recurse to turn it into a template argument
  if constexpr (U < (EMU_PERIOD > 0 ? EMU_PERIOD : -EMU_PERIOD)) {
    if (u == U) particle_step<H, poly_mask<EMU_PERIOD, H>(U), LO>(p, zx2, zy2, acc, hv);
    else step_u<H, EMU_PERIOD, LO, U + 1>(u, p, zx2, zy2, acc, hv);
  }
}

// Sum over one AoS tile for this warp's first HV measurement pairs.
template <int K, int HV, int EMU_PERIOD, bool LO = false>
__device__ __forceinline__ void tile_sum(const float4 *__restrict__ A, int np, Meas<K> &m) {
  constexpr int H = Meas<K>::H;
  f2 acc[H];
#pragma unroll
  for (int h = 0; h < H; ++h) acc[h] = 0ull;
  int p = 0;
  if constexpr (EMU_PERIOD != 0) {
    constexpr int PER = EMU_PERIOD > 0 ? EMU_PERIOD : -EMU_PERIOD;
#pragma unroll 1
    for (; p + PER <= np; p += PER) {
#pragma unroll
      for (int u = 0; u < PER; ++u) step_u<H, EMU_PERIOD, LO>(u, A[p + u], m.zx2, m.zy2, acc, HV);
    }
  }
#pragma unroll 4
  for (; p < np; ++p) particle_step<H, 0, LO>(A[p], m.zx2, m.zy2, acc, HV);
#pragma unroll
  for (int h = 0; h < H; ++h) {
    float lo, hi;
    f2_unpack(acc[h], lo, hi);
    m.tot[2 * h] += lo;
    m.tot[2 * h + 1] += hi;
  }
}

// kv: measurement slots with a valid lane.  K = 2 with only the first slot valid (the
// ragged last warp of a tile when M mod 64 <= 32) evaluates that slot alone: half the exps,
// bit-identical sums (the packed ops lane for lane).
template <int K, int EMU_PERIOD>
__device__ __forceinline__ void tile_dispatch(int kv, bool lo, const float4 *A, int np, Meas<K> &m) {
  constexpr int H = Meas<K>::H;
  const int hv = (kv + 1) >> 1;
  if constexpr (K == 2) {
    if (kv == 1 && lo) {
      tile_sum<K, 1, EMU_PERIOD, true>(A, np, m);
      return;
    }
  }
  if (hv == H) tile_sum<K, H, EMU_PERIOD>(A, np, m);
  else if constexpr (H > 1) {
    if (hv == 1) tile_sum<K, 1, EMU_PERIOD>(A, np, m);
    if constexpr (H > 2) {
      if (hv == 2) tile_sum<K, 2, EMU_PERIOD>(A, np, m);
      if (hv == 3) tile_sum<K, (H > 3 ? 3 : 2), EMU_PERIOD>(A, np, m);
    }
  }
}

// Units: every track's full measurement tiles (track-major), then the ragged
// last tiles of all tracks (so the short units fill the tail of the schedule).
// CL > 1: a thread-block cluster of CL CTAs shares one (track, measurement tile)
// unit, CTA rank c summing the particle tiles [c tpc, (c+1) tpc); rank 0 adds the
// ranks' partial sums in rank order through DSMEM and writes the epilogue.  Each
// CTA does 1/CL of the unit's work, so the last wave of the grid is CL times
// shorter (the tail of a 2.2-wave grid cost ~12 % of the launch).
// SKIP (opt-in, GLMB_COMPAT_SKIP=1): a warp skips a particle tile when every one of its
// measurements lies >= kSkipD2 whitened units^2 from the tile's bounding box.  Every pair
// it skips has q >= 200, where both exp paths give exactly +0 (MUFU.EX2.FTZ flushes below
// 2^-126; the polynomial clamps at q = 189 and w 2^-64 * p 2^-125 rounds to 0 below
// 2^-150), so C and the gate words are bit-identical to the dense pass.
constexpr float kSkipD2 = 200.0f;

template <int NW, int K, int EMU_PERIOD, int CL, bool SKIP = false>
__global__ void __launch_bounds__(32 * NW, min_blocks<NW, K>()) compat_kernel(const CompatArgs a) {
  grid_dep_wait();  // launched with programmatic serialization after predict / birth
  constexpr int H = Meas<K>::H;
  constexpr int kThreads = 32 * NW;
  constexpr int kTileM = 32 * NW;  // measurements per tile per K
  __shared__ float part[CL > 1 ? K : 1][CL > 1 ? kThreads : 1];  // this CTA's partial sums
  extern __shared__ __align__(128) float smem[];
  float4 *aos = reinterpret_cast<float4 *>(smem + kStages * kRawFloats);  // 2 AoS tiles
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ float red[2][kVWarps];
  __shared__ float tbox[SKIP ? 2 : 1][SKIP ? NW : 1][4];  // per tile parity and warp: min/max X', Y'

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int unit = blockIdx.x / CL;
  const int crank = CL > 1 ? static_cast<int>(blockIdx.x - unit * CL) : 0;
  // unit order: a track's full measurement tiles are adjacent (they run concurrently and
  // share the particle tiles through L2: one HBM read of the state instead of one per tile),
  // the ragged last tiles of all tracks come last (short units fill the tail of the grid)
  const int n_full = a.M % (kTileM * K) == 0 ? a.n_mtiles : a.n_mtiles - 1;
  int mt, j;
  if (a.track_major == 0) {  // GLMB_COMPAT_ORDER=0: tile-major (A/B runs)
    mt = unit / a.T;
    j = unit - mt * a.T;
  } else if (unit < a.T * n_full) {
    j = unit / n_full;
    mt = unit - j * n_full;
  } else {
    j = unit - a.T * n_full;
    mt = a.n_mtiles - 1;
  }
  const int wbase = mt * (kTileM * K) + warp * (32 * K);   // first measurement of this warp
  const int kv = min(K, max(0, (a.M - wbase + 31) >> 5));  // measurement slots with any valid lane
  const int hv = (kv + 1) >> 1;                            // packed pairs with any valid slot
  const int64_t base = static_cast<int64_t>(j) * a.ld;
  const float *xs = a.x + base, *ys = a.y + base, *ws = a.w + base;
  const int ntiles = (a.P + kTileP - 1) / kTileP;
  const int tpc = (ntiles + CL - 1) / CL;                 // tiles per cluster rank
  const int t_begin = min(ntiles, crank * tpc), t_end = min(ntiles, t_begin + tpc);
  static_assert(kStages == 1, "the chunked tile schedule below assumes one raw stage");
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // the first tile is always tile 0 (the centre); ranks > 0 then jump to their own chunk
  if (tid == 0) issue_tile(a, xs, ys, ws, smem, &bars[0], 0);
  uint32_t phase = 0;
  float2 zr[2 * H];
#pragma unroll
  for (int k = 0; k < 2 * H; ++k) {
    const int i = wbase + k * 32 + lane;
    zr[k] = (k < K && i < a.M) ? __ldg(reinterpret_cast<const float2 *>(a.Z) + i) : make_float2(0.f, 0.f);
  }

  Meas<K> m;
  float cx = 0.f, cy = 0.f;
  // ranks > 0: tile 0 only for the centre, then the rank's first tile
  int t = crank == 0 ? 0 : -1;
  for (; t < t_end; ++t) {
    const float *X = smem;
    const float *Y = X + kTileP;
    const float *W = Y + kTileP;
    float4 *A = aos + (t & 1) * kTileP;
    const int tt = t < 0 ? 0 : t;                         // the tile in the raw stage
    const int np = min(kTileP, a.P - tt * kTileP);
    mbar_wait_parity(&bars[0], phase);
    phase ^= 1u;
    if (tt == 0 && (t == 0 || t < 0)) {  // centre c = mean position of the first tile (fixed order -> deterministic)
      // summed as 128 virtual threads in 4 virtual warps whatever NW is, so the centre
      // (and hence C) is the same for every launch shape
#pragma unroll
      for (int v = 0; v < kVWarps / NW; ++v) {
        const int vt = tid + v * kThreads;
        float sx = 0.f, sy = 0.f;
        for (int idx = vt; idx < np; idx += 32 * kVWarps) {
          sx += X[idx];
          sy += Y[idx];
        }
        sx = warp_sum(sx);
        sy = warp_sum(sy);
        if (lane == 0) {
          red[0][vt >> 5] = sx;
          red[1][vt >> 5] = sy;
        }
      }
      __syncthreads();
      cx = ((red[0][0] + red[0][1]) + (red[0][2] + red[0][3])) / static_cast<float>(np);
      cy = ((red[1][0] + red[1][1]) + (red[1][2] + red[1][3])) / static_cast<float>(np);
#pragma unroll
      for (int h = 0; h < H; ++h) {
        float zx[2], zy[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float lx = zr[2 * h + u].x - cx, ly = zr[2 * h + u].y - cy;
          zx[u] = fmaf(a.a2, ly, a.a1 * lx);
          zy[u] = a.b2 * ly;
        }
        m.zx2[h] = f2_pack(2.0f * zx[0], 2.0f * zx[1]);
        m.zy2[h] = f2_pack(2.0f * zy[0], 2.0f * zy[1]);
        m.tot[2 * h] = 0.f;
        m.tot[2 * h + 1] = 0.f;
      }
    }
    if (t < 0) {  // centre only: load the rank's first own tile next
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0 && t_begin < t_end) issue_tile(a, xs, ys, ws, smem, &bars[0], t_begin);
      t = t_begin - 1;
      continue;
    }
    // whiten raw tile -> AoS (X', Y', w 2^-64, w)
    if constexpr (!SKIP) {
      for (int idx = tid; idx < np; idx += kThreads) {
        const float lx = X[idx] - cx, ly = Y[idx] - cy;
        A[idx] = make_float4(fmaf(a.a2, ly, a.a1 * lx), a.b2 * ly, W[idx] * kTwoM64, W[idx]);
      }
    } else {
      float bx0 = INFINITY, bx1 = -INFINITY, by0 = INFINITY, by1 = -INFINITY;
      for (int idx = tid; idx < np; idx += kThreads) {
        const float lx = X[idx] - cx, ly = Y[idx] - cy;
        const float qx = fmaf(a.a2, ly, a.a1 * lx), qy = a.b2 * ly;
        A[idx] = make_float4(qx, qy, W[idx] * kTwoM64, W[idx]);
        bx0 = fminf(bx0, qx);
        bx1 = fmaxf(bx1, qx);
        by0 = fminf(by0, qy);
        by1 = fmaxf(by1, qy);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        bx0 = fminf(bx0, __shfl_xor_sync(0xffffffffu, bx0, o));
        bx1 = fmaxf(bx1, __shfl_xor_sync(0xffffffffu, bx1, o));
        by0 = fminf(by0, __shfl_xor_sync(0xffffffffu, by0, o));
        by1 = fmaxf(by1, __shfl_xor_sync(0xffffffffu, by1, o));
      }
      if (lane == 0) {
        tbox[t & 1][warp][0] = bx0;
        tbox[t & 1][warp][1] = bx1;
        tbox[t & 1][warp][2] = by0;
        tbox[t & 1][warp][3] = by1;
      }
    }
    fence_proxy_async_smem();  // the raw stage was read through the generic proxy; TMA rewrites it next
    __syncthreads();           // AoS tile t complete; every warp is done with tile t-1
    if (tid == 0 && t + 1 < t_end) issue_tile(a, xs, ys, ws, smem, &bars[0], t + 1);
    if constexpr (!SKIP) {
      if (hv > 0) tile_dispatch<K, EMU_PERIOD>(kv, a.lo_slot != 0, A, np, m);
    } else if (hv > 0) {
      {
        float x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          x0 = fminf(x0, tbox[t & 1][w][0]);
          x1 = fmaxf(x1, tbox[t & 1][w][1]);
          y0 = fminf(y0, tbox[t & 1][w][2]);
          y1 = fmaxf(y1, tbox[t & 1][w][3]);
        }
        bool far = true;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int i = wbase + k * 32 + lane;
          if (i < a.M) {
            float zx, zy, z1x, z1y;
            f2_unpack(m.zx2[k >> 1], zx, z1x);
            f2_unpack(m.zy2[k >> 1], zy, z1y);
            if (k & 1) {
              zx = z1x;
              zy = z1y;
            }
            zx *= 0.5f;
            zy *= 0.5f;
            const float dx = fmaxf(0.0f, fmaxf(x0 - zx, zx - x1)), dy = fmaxf(0.0f, fmaxf(y0 - zy, zy - y1));
            far &= fmaf(dx, dx, dy * dy) >= kSkipD2;
          }
        }
        const bool skip = __all_sync(0xffffffffu, far);
        if (skip && lane == 0 && a.skip_count != nullptr)
          atomicAdd(a.skip_count, static_cast<unsigned long long>(np) * static_cast<unsigned long long>(min(32 * K, a.M - wbase)));
        if (!skip) tile_dispatch<K, EMU_PERIOD>(kv, a.lo_slot != 0, A, np, m);
      }
    }
  }

  if constexpr (CL > 1) {  // rank 0 adds the ranks' partial sums in rank order (DSMEM)
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
#pragma unroll
    for (int k = 0; k < K; ++k) part[k][tid] = m.tot[k];
    cluster.sync();
    if (crank == 0) {
#pragma unroll
      for (int r = 1; r < CL; ++r) {
        const float(*pp)[kThreads] = reinterpret_cast<const float(*)[kThreads]>(cluster.map_shared_rank(&part[0][0], r));
#pragma unroll
        for (int k = 0; k < K; ++k) m.tot[k] += pp[k][tid];
      }
    }
    cluster.sync();  // peers keep their shared memory until rank 0 has read it
    if (crank != 0) return;
  }

  // epilogue: likelihood, gate bit, C entry, clutter column
  if (kv == 0) return;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < kv) {
      const int i = wbase + k * 32 + lane;
      const bool valid = i < a.M;
      const float L = m.tot[k] * a.norm;
      const bool g = valid && (L >= a.gamma);
      const float c = g ? a.p_d * L : 0.0f;
      const uint32_t word = __ballot_sync(0xffffffffu, g);
      if (a.n_peers == 0) {
        if (valid) a.C_tracks[static_cast<int64_t>(j) * a.ldc + i] = c;
        if (lane == 0) a.gate[static_cast<int64_t>(j) * a.ldg + ((wbase + k * 32) >> 5)] = word;
      } else {  // fused all-gather: this column goes straight into every rank's copy of C_k
        const int64_t row = a.peer_row0 + j;
        for (int r = 0; r < a.n_peers; ++r) {
          if (valid) a.peer_C[r][row * a.ldc + i] = c;
          if (lane == 0) a.peer_G[r][row * a.ldg + ((wbase + k * 32) >> 5)] = word;
        }
      }
      if (j == 0 && a.C_clutter != nullptr && valid) a.C_clutter[i] = a.kappa;
    }
  }
}

__global__ void clutter_fill_kernel(float *c, int32_t M, float kappa) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < M) c[i] = kappa;
}

template <int NW, int K, int EMU_PERIOD, int CL, bool SKIP>
cudaError_t launch_kc(const CompatArgs &a, cudaStream_t s) {
  const int64_t grid = static_cast<int64_t>(a.T) * a.n_mtiles * CL;
  if (CL == 1)
    return launch_pdl(compat_kernel<NW, K, EMU_PERIOD, CL, SKIP>, dim3(static_cast<unsigned>(grid)), dim3(32 * NW),
                      kSmemBytes, s, a);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, compat_kernel<NW, K, EMU_PERIOD, CL, SKIP>, a);
}

template <int NW, int K, int EMU_PERIOD>
cudaError_t launch_k(const CompatArgs &a, cudaStream_t s) {
  // exact zero-tile skipping (a.skip, opt-in; the dense pass is the default and the measured
  // headline).  Built for the default exp split only.
  if constexpr (EMU_PERIOD == -10) {
    if (a.skip)
      return a.CL == 4 ? launch_kc<NW, K, EMU_PERIOD, 4, true>(a, s)
             : a.CL == 2 ? launch_kc<NW, K, EMU_PERIOD, 2, true>(a, s) : launch_kc<NW, K, EMU_PERIOD, 1, true>(a, s);
  }
  if (a.CL == 4) return launch_kc<NW, K, EMU_PERIOD, 4, false>(a, s);
  return a.CL == 2 ? launch_kc<NW, K, EMU_PERIOD, 2, false>(a, s) : launch_kc<NW, K, EMU_PERIOD, 1, false>(a, s);
}

// Share of the exps evaluated on the FMA pipe: one particle in |EMU| (negative:
// every measurement pair of that particle, so each measurement sees the same
// MUFU/polynomial mix and C stays bit-exact under row permutations of Z;
// positive: pair h of particle u when (u + 2h) % EMU == EMU - 1, spread; 0:
// all MUFU).  Default -10 (measured best bit-exact setting on B200, see
// profiles/README.md).  GLMB_COMPAT_EMU overrides it (diagnostics / A-B runs).
int emu_period() {
  static int v = [] {
    const char *e = std::getenv("GLMB_COMPAT_EMU");
    return e ? std::atoi(e) : -10;
  }();
  return v;
}

template <int NW, int K>
cudaError_t launch_e(const CompatArgs &a, cudaStream_t s) {
  switch (emu_period()) {  // the measured neighbourhood of the default (profiles/README.md)
    case 0: return launch_k<NW, K, 0>(a, s);
    case -8: return launch_k<NW, K, -8>(a, s);
    case -12: return launch_k<NW, K, -12>(a, s);
    default: return launch_k<NW, K, -10>(a, s);
  }
}

}  // namespace

void compat_plan(int32_t M, int32_t P, int32_t *K, int32_t *NW, int32_t *CL, int32_t *n_mtiles) {
  // Depends on (M, P) only -- never on T -- so any sharding of the tracks runs
  // the same per-column code (bit-identical C).  A warp holds 32 K measurements;
  // K = 2 (one packed pair per thread) wherever M allows, NW warps per CTA:
  //   M > 128: NW = 4, K = kDefaultK (GLMB_COMPAT_K overrides: A/B runs)
  //   64 < M <= 128: NW = 2, K = 2;  32 < M <= 64: NW = 1, K = 2;  M <= 32: NW = 1, K = 1
  // CL: particle chunks per (track, measurement tile), a thread-block cluster (>= 8
  // particle tiles per CTA, or one each at P = 1024); GLMB_COMPAT_CL overrides (A/B runs)
  static const int32_t cl_env = [] {
    const char *e = std::getenv("GLMB_COMPAT_CL");
    return e ? std::atoi(e) : 0;
  }();
  const int32_t ptiles = (P + kTileP - 1) / kTileP;
  // measured (cfg3): CL = 1 14.5, 2 15.3, 4 14.9 pairs/clk/SM; at P = 1024 (4 tiles) a tile per
  // rank: cfg1 (T_k = 68) 34 -> 23 us, the convoy (T_k ~ 800) unchanged -- small grids fill more SMs
  int32_t cl = ptiles >= 16 ? 2 : ptiles == 4 ? 4 : 1;
  if (cl_env == 1 || cl_env == 2 || cl_env == 4) cl = cl_env;
  *CL = cl;
  static const int32_t kmax = [] {
    const char *e = std::getenv("GLMB_COMPAT_K");
    const int v = e ? std::atoi(e) : 2;
    return (v == 1 || v == 2) ? v : 2;
  }();
  int32_t k = kmax, nw = 4;
  if (M <= 32) {
    k = 1;
    nw = 1;
  } else if (M <= 64) {
    k = 2;
    nw = 1;
  } else if (M <= 128) {
    k = 2;
    nw = 2;
  } else {
    const int32_t warps_needed = (M + 31) / 32;
    while (k > 2 && warps_needed <= 4 * (k / 2)) k /= 2;
  }
  *K = k;
  *NW = nw;
  *n_mtiles = (M + 32 * nw * k - 1) / (32 * nw * k);
}

cudaError_t launch_compat(const CompatArgs &a_in, cudaStream_t s) {
  static const int order_env = [] {
    const char *e = std::getenv("GLMB_COMPAT_ORDER");
    return e ? std::atoi(e) : 1;
  }();
  CompatArgs a = a_in;
  a.track_major = order_env;
  static const int lo_env = [] {   // GLMB_COMPAT_LO=0: the packed pair always (A/B; same C bits)
    const char *e = std::getenv("GLMB_COMPAT_LO");
    return e ? std::atoi(e) : 1;
  }();
  a.lo_slot = lo_env != 0;
  if (a.NW == 1) return a.K == 1 ? launch_e<1, 1>(a, s) : launch_e<1, 2>(a, s);
  if (a.NW == 2) return launch_e<2, 2>(a, s);
  switch (a.K) {
    case 1: return launch_e<4, 1>(a, s);
    case 2: return launch_e<4, 2>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

// GLMB_COMPAT_SKIP=1 turns glmb_compat into the skipping variant (A/B runs and tests)
bool compat_skip_env() {
  static const bool v = [] {
    const char *e = std::getenv("GLMB_COMPAT_SKIP");
    return e && std::atoi(e) == 1;
  }();
  return v;
}

cudaError_t launch_clutter_fill(float *C_clutter, int32_t M, float kappa, cudaStream_t s) {
  if (M == 0 || C_clutter == nullptr) return cudaSuccess;
  clutter_fill_kernel<<<(M + 255) / 256, 256, 0, s>>>(C_clutter, M, kappa);
  return cudaGetLastError();
}

}  // namespace glmb
