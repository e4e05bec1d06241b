// kernels_rng.cu -- glmb_predict and glmb_birth kernels (+ Philox test hooks).
//
// Both passes are HBM-bound streams over SoA fp32 particle arrays: each
// thread owns 4 consecutive particles of one track (one 128-bit load / store
// per array), draws their process noise from Philox4x32-10 keyed by
// (seed; counter, gid, step, tag) and writes the result.  Predict uses one
// Philox block per particle pair (counter p >> 1, words (0,1) / (2,3)).  Grid: grid-stride over
// the T*P/4 particle quads with 256-thread blocks, sized to 148 SMs x 8.
#include "glmb_device.cuh"
#include "glmb_internal.h"

namespace glmb {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float4 ld_stream(const float *p) { return __ldcs(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ void st_stream(float *p, float4 v) { __stcs(reinterpret_cast<float4 *>(p), v); }
__device__ __forceinline__ float &at(float4 &v, int q) { return (&v.x)[q]; }

// CTRV survival propagation (§Approach), half-angle form:
//   dx = v dt sinc(h) cos(psi + h), dy = v dt sinc(h) sin(psi + h), h = omega dt / 2
__global__ void __launch_bounds__(kThreads) predict_kernel(const PredictArgs a) {
  grid_dep_wait();
  const int32_t quads = a.P >> 2;
  const int64_t total = static_cast<int64_t>(a.T) * quads;
  const float half_dt = 0.5f * a.dt;
  const float half_dt2 = 0.5f * a.dt * a.dt;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t j = static_cast<int32_t>(g / quads);
    const int32_t p0 = static_cast<int32_t>(g - static_cast<int64_t>(j) * quads) << 2;
    const int64_t e = static_cast<int64_t>(j) * a.ld + p0;
    float4 X = ld_stream(a.x + e), Y = ld_stream(a.y + e), V = ld_stream(a.v + e);
    float4 PS = ld_stream(a.psi + e), OM = ld_stream(a.omega + e);
    const uint32_t gid = static_cast<uint32_t>(__ldg(a.gid + j));
    // one Philox block per particle pair: counter (p >> 1, gid, step, 0);
    // words (0,1) drive the even particle, words (2,3) the odd one
    const u32x4 r01 = philox4x32_10(u32x4{static_cast<uint32_t>(p0 >> 1), gid, a.step, 0u}, a.key0, a.key1);
    const u32x4 r23 = philox4x32_10(u32x4{static_cast<uint32_t>((p0 >> 1) + 1), gid, a.step, 0u}, a.key0, a.key1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32x4 &r = q < 2 ? r01 : r23;
      float n0, n1;
      if (q & 1) box_muller(r.c, r.d, n0, n1);
      else box_muller(r.a, r.b, n0, n1);
      const float nu_a = a.sigma_a * n0, nu_w = a.sigma_w * n1;
      const float x = at(X, q), y = at(Y, q), v = at(V, q), psi = at(PS, q), om = at(OM, q);
      const float h = om * half_dt;
      // MUFU sin/cos (abs. error ~2^-21 on |arg| <~ pi): contributes < 3e-6 m to x, y
      float sp, cp, sph, cph;
      __sincosf(psi, &sp, &cp);
      __sincosf(psi + h, &sph, &cph);  // sin / cos (psi + h)
      const float h2 = h * h;
      // sinc(h) = sin h / h: Taylor to h^8 (error < 3e-11 for |h| < 0.5), else libdevice sinf
      const float sinc = fabsf(h) < 0.5f
                             ? fmaf(h2, fmaf(h2, fmaf(h2, fmaf(h2, 1.0f / 362880.0f, -1.0f / 5040.0f),
                                                        1.0f / 120.0f), -1.0f / 6.0f), 1.0f)
                             : sinf(h) / h;
      const float vds = v * a.dt * sinc;
      const float an = half_dt2 * nu_a;
      at(X, q) = fmaf(an, cp, fmaf(vds, cph, x));
      at(Y, q) = fmaf(an, sp, fmaf(vds, sph, y));
      at(V, q) = fmaf(a.dt, nu_a, v);
      at(PS, q) = wrap_angle(fmaf(half_dt2, nu_w, fmaf(om, a.dt, psi)));
      at(OM, q) = fmaf(a.dt, nu_w, om);
    }
    st_stream(a.ox + e, X);
    st_stream(a.oy + e, Y);
    st_stream(a.ov + e, V);
    st_stream(a.opsi + e, PS);
    st_stream(a.oomega + e, OM);
  }
}

// LMB birth: s = mu_b + L_b n, n0..n3 from tag 0x100, n4 from tag 0x101.
__global__ void __launch_bounds__(kThreads) birth_kernel(const BirthArgs a) {
  grid_dep_wait();
  const int32_t quads = a.P >> 2;
  const int64_t total = static_cast<int64_t>(a.B) * quads;
  const float winit = 1.0f / static_cast<float>(a.P);
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t b = static_cast<int32_t>(g / quads);
    const int32_t p0 = static_cast<int32_t>(g - static_cast<int64_t>(b) * quads) << 2;
    const int64_t e = static_cast<int64_t>(b) * a.ld + p0;
    const uint32_t gid = static_cast<uint32_t>(__ldg(a.gid + b));
    float mu[5], L[15];
#pragma unroll
    for (int r = 0; r < 5; ++r) mu[r] = __ldg(a.mean + 5 * b + r);
#pragma unroll
    for (int r = 0; r < 15; ++r) L[r] = __ldg(a.chol + 15 * b + r);
    float4 out[5];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t p = static_cast<uint32_t>(p0 + q);
      const u32x4 r0 = philox4x32_10(u32x4{p, gid, a.step, 0x100u}, a.key0, a.key1);
      const u32x4 r1 = philox4x32_10(u32x4{p, gid, a.step, 0x101u}, a.key0, a.key1);
      float n[6];
      box_muller(r0.a, r0.b, n[0], n[1]);
      box_muller(r0.c, r0.d, n[2], n[3]);
      box_muller(r1.a, r1.b, n[4], n[5]);
      int idx = 0;
#pragma unroll
      for (int row = 0; row < 5; ++row) {
        float acc = mu[row];
#pragma unroll
        for (int c = 0; c <= row; ++c) acc = fmaf(L[idx + c], n[c], acc);
        idx += row + 1;
        at(out[row], q) = acc;
      }
      at(out[3], q) = wrap_angle(at(out[3], q));
    }
    st_stream(a.x + e, out[0]);
    st_stream(a.y + e, out[1]);
    st_stream(a.v + e, out[2]);
    st_stream(a.psi + e, out[3]);
    st_stream(a.omega + e, out[4]);
    st_stream(a.w + e, make_float4(winit, winit, winit, winit));
  }
}

__global__ void philox_dump_kernel(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, uint32_t *out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u32x4 r = philox4x32_10(u32x4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, k0, k1);
  out[4 * i] = r.a;
  out[4 * i + 1] = r.b;
  out[4 * i + 2] = r.c;
  out[4 * i + 3] = r.d;
}

__global__ void normals_dump_kernel(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, float *out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u32x4 r = philox4x32_10(u32x4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, k0, k1);
  box_muller(r.a, r.b, out[4 * i], out[4 * i + 1]);
  box_muller(r.c, r.d, out[4 * i + 2], out[4 * i + 3]);
}

int grid_for(int64_t quads, int sm_count) {
  const int64_t need = (quads + kThreads - 1) / kThreads;
  const int64_t cap = static_cast<int64_t>(sm_count > 0 ? sm_count : 148) * 8;
  return static_cast<int>(need < cap ? need : cap);
}

}  // namespace

cudaError_t launch_predict(const PredictArgs &a, int sm_count, cudaStream_t s) {
  const int64_t quads = static_cast<int64_t>(a.T) * (a.P >> 2);
  if (quads == 0) return cudaSuccess;
  {
    cudaError_t e = launch_pdl(predict_kernel, dim3(grid_for(quads, sm_count)), dim3(kThreads), 0, s, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_birth(const BirthArgs &a, int sm_count, cudaStream_t s) {
  const int64_t quads = static_cast<int64_t>(a.B) * (a.P >> 2);
  if (quads == 0) return cudaSuccess;
  {
    cudaError_t e = launch_pdl(birth_kernel, dim3(grid_for(quads, sm_count)), dim3(kThreads), 0, s, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_philox_dump(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, uint32_t *out,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  philox_dump_kernel<<<(n + 255) / 256, 256, 0, s>>>(k0, k1, ctr, n, out);
  return cudaGetLastError();
}

cudaError_t launch_normals_dump(uint32_t k0, uint32_t k1, const uint32_t *ctr, int32_t n, float *out,
                                cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  normals_dump_kernel<<<(n + 255) / 256, 256, 0, s>>>(k0, k1, ctr, n, out);
  return cudaGetLastError();
}

}  // namespace glmb
