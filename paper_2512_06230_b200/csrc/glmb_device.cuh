// glmb_device.cuh -- device primitives of the GLMB step core (sm_100a).
//
// Philox4x32-10 counter-based generator, the exact 24-bit uniform map,
// Box-Muller normals, packed fp32x2 arithmetic, and the mbarrier /
// cp.async.bulk (TMA bulk-copy engine) wrappers used by glmb_compat.
// Nothing here is shared with oracle/ (see DESIGN.md "Oracle independence").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace glmb {

// ---------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11): round (c0,c1,c2,c3) ->
// (hi(B*c2)^c1^k0, lo(B*c2), hi(A*c0)^c3^k1, lo(A*c0)), Weyl key bump.
struct u32x4 {
  uint32_t a, b, c, d;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 ctr, uint32_t k0, uint32_t k1) {
  constexpr uint32_t kMulA = 0xD2511F53u, kMulB = 0xCD9E8D57u;
  constexpr uint32_t kWeylA = 0x9E3779B9u, kWeylB = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hiA = __umulhi(kMulA, ctr.a), loA = kMulA * ctr.a;
    const uint32_t hiB = __umulhi(kMulB, ctr.c), loB = kMulB * ctr.c;
    ctr = u32x4{hiB ^ ctr.b ^ k0, loB, hiA ^ ctr.d ^ k1, loA};
    k0 += kWeylA;
    k1 += kWeylB;
  }
  return ctr;
}

// Exact uniform in (0,1): (2*(r>>9)+1) * 2^-24 (the integer < 2^24 converts exactly).
__device__ __forceinline__ float uniform24(uint32_t r) {
  return __uint2float_rn(((r >> 9) << 1) | 1u) * 5.9604644775390625e-8f;
}

// Box-Muller pair from two raw words: rho = sqrt(-2 ln ua), (rho cos 2pi ub, rho sin 2pi ub).
// logf / sqrtf are the accurate libdevice versions (ln ua near 1 needs them);
// the angle goes to MUFU sin/cos as 2 pi ub - pi in (-pi, pi) (abs. error ~2^-21,
// i.e. < 3e-6 on n) with cos(t + pi) = -cos t, sin(t + pi) = -sin t.
__device__ __forceinline__ void box_muller(uint32_t ra, uint32_t rb, float &n0, float &n1) {
  const float ua = uniform24(ra), ub = uniform24(rb);
  const float rho = sqrtf(-2.0f * logf(ua));
  float s, c;
  __sincosf(fmaf(6.28318530717958647692f, ub, -3.14159265358979323846f), &s, &c);
  n0 = -rho * c;
  n1 = -rho * s;
}

// wrap(a) = a - 2 pi ceil((a - pi) / 2 pi)  -> (-pi, pi]
__device__ __forceinline__ float wrap_angle(float a) {
  constexpr float kPi = 3.14159265358979323846f, kTwoPi = 6.28318530717958647692f;
  if (a > -kPi && a <= kPi) return a;
  return a - kTwoPi * ceilf((a - kPi) * (1.0f / kTwoPi));
}

// ---------------------------------------------------------------- f32x2
// Packed fp32 pairs (SASS FADD2 / FMUL2 / FFMA2 on sm_100a).
typedef unsigned long long f2;

__device__ __forceinline__ f2 f2_pack(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(f2 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
  f2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// MUFU.EX2 (ex2.approx.ftz.f32): rel. error ~2^-22, flushes subnormals.
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// ---------------------------------------------------------------- programmatic dependent launch
// First statement of every kernel of the hypothesis chain: with the launch attribute
// set (launch_pdl), the kernel's CTAs may start while the previous kernel drains and
// wait here until its writes are visible; launched without it, this is a no-op.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier / TMA bulk
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine, completion counted
// on `bar` in bytes.  dst/src 16-B aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace glmb
