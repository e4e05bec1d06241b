// peaks.cu -- micro-benchmark of the issue pipes the GLMB kernels are bound by
// (standalone executable, not part of libglmb.so).  Prints one JSON object:
// MUFU.EX2, FFMA2 (packed fp32x2), FFMA throughput per SM per clock and the
// SM count / clock seen, so every roofline in bench.py uses measured numbers.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void ex2_kernel(float *out, int iters, float seed, long long *cyc) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed * (c + 1) * 1e-3f - 0.5f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void ffma2_kernel(float *out, int iters, float seed, long long *cyc) {
  unsigned long long v[kChains], m, a;
  asm("mov.b64 %0, {%1, %1};" : "=l"(m) : "f"(0.999f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(seed * 1e-3f));
#pragma unroll
  for (int c = 0; c < kChains; ++c) asm("mov.b64 %0, {%1, %2};" : "=l"(v[c]) : "f"(seed + c), "f"(seed - c));
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(m), "l"(a));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v[c]));
    s += lo + hi;
  }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void ffma_kernel(float *out, int iters, float seed, long long *cyc) {
  float v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = seed + c;
  const float m = 0.999f, a = seed * 1e-3f;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[c]) : "f"(m), "f"(a));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

// NM independent MUFU.EX2 and NF independent FFMA2 per iteration (8 chains each):
// tells whether the SFU and FMA pipes overlap at full rate.
template <int NM, int NF>
__global__ void mix_kernel(float *out, int iters, float seed, long long *cyc) {
  float v[NM > 0 ? NM : 1];
  unsigned long long u[NF > 0 ? NF : 1], m, a;
  asm("mov.b64 %0, {%1, %1};" : "=l"(m) : "f"(0.999f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(a) : "f"(seed * 1e-3f));
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = seed * (c + 1) * 1e-3f - 0.5f;
#pragma unroll
  for (int c = 0; c < NF; ++c) asm("mov.b64 %0, {%1, %2};" : "=l"(u[c]) : "f"(seed + c), "f"(seed - c));
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < (NM > NF ? NM : NF); ++c) {
      if (c < NM) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
      if (c < NF) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(u[c]) : "l"(m), "l"(a));
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NM; ++c) s += v[c];
#pragma unroll
  for (int c = 0; c < NF; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(u[c]));
    s += lo + hi;
  }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

// NM MUFU.EX2 per LDS.128 broadcast (all lanes read the same 16 B of shared memory).
template <int NM>
__global__ void mufu_lds_kernel(float *out, int iters, float seed, long long *cyc) {
  __shared__ float4 buf[64];
  if (threadIdx.x < 64) buf[threadIdx.x] = make_float4(seed, seed * 0.5f, seed * 0.25f, seed * 0.125f);
  __syncthreads();
  float v[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) v[c] = seed * (c + 1) * 1e-3f - 0.5f;
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    const float4 p = buf[i & 63];
    acc += p.x + p.w;
#pragma unroll
    for (int c = 0; c < NM; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
  }
  float s = acc;
#pragma unroll
  for (int c = 0; c < NM; ++c) s += v[c];
  if (s == 12345.f) out[0] = s;
}

template <int NM>
void run_mufu_lds(int sms, float *out, long long *cyc) {
  const int threads = 256, blocks = sms * 8, iters = 4096;
  mufu_lds_kernel<NM><<<blocks, threads>>>(out, 16, 1.0f, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mufu_lds_kernel<NM><<<blocks, threads>>>(out, iters, 1.0f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double th = double(blocks) * threads * iters;
  printf("  \"mufu%d_per_lds128\": {\"ex2_per_s\": %.6e, \"ms\": %.4f},\n", NM, th * NM / (ms * 1e-3), ms);
}

template <int NM, int NF>
void run_mix(int sms, float *out, long long *cyc) {
  const int threads = 256, blocks = sms * 8, iters = 2048;
  mix_kernel<NM, NF><<<blocks, threads>>>(out, 16, 1.0f, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mix_kernel<NM, NF><<<blocks, threads>>>(out, iters, 1.0f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double th = double(blocks) * threads * iters;
  printf("  \"mix_m%d_f%d\": {\"ex2_per_s\": %.6e, \"ffma2_per_s\": %.6e, \"ms\": %.4f},\n", NM, NF,
         th * NM / (ms * 1e-3), th * NF / (ms * 1e-3), ms);
}

template <typename F>
void run(const char *name, F kern, int sms, int clk_khz, float *out, long long *cyc, bool last) {
  const int threads = 256, blocks_per_sm = 8, iters = 4096;
  const int blocks = sms * blocks_per_sm;
  kern<<<blocks, threads>>>(out, 16, 1.0f, cyc);  // warm up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters, 1.0f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = double(blocks) * threads * iters * kChains;  // thread-level instructions
  const double per_s = ops / (ms * 1e-3);
  // thread-level instructions per clock per SM at the attribute (max) clock: an FFMA2 is one
  // instruction doing two FP32 lanes, MUFU.EX2 / FFMA one
  printf("  \"%s\": {\"ops_per_s\": %.6e, \"ms\": %.4f, \"thread_instr_per_clk_per_sm\": %.3f}%s\n", name, per_s,
         ms, per_s / sms / (clk_khz * 1e3), last ? "" : ",");
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float *out;
  long long *cyc;
  cudaMalloc(&out, 16);
  cudaMalloc(&cyc, 16);
  printf("{\n  \"sm_count\": %d,\n  \"attr_clock_mhz\": %.1f,\n", sms, clk_khz / 1e3);
  run_mufu_lds<2>(sms, out, cyc);
  run_mufu_lds<4>(sms, out, cyc);
  run_mufu_lds<8>(sms, out, cyc);
  run_mix<8, 8>(sms, out, cyc);
  run_mix<8, 12>(sms, out, cyc);
  run_mix<8, 16>(sms, out, cyc);
  run_mix<4, 16>(sms, out, cyc);
  run("mufu_ex2", ex2_kernel, sms, clk_khz, out, cyc, false);
  run("ffma2_f32x2", ffma2_kernel, sms, clk_khz, out, cyc, false);
  run("ffma", ffma_kernel, sms, clk_khz, out, cyc, true);
  printf("}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
