// stream_pattern.cu -- standalone diagnostic (not part of libglmb): what HBM bandwidth the
// reweight's access pattern can reach with no arithmetic and no phases.  Three [T][P] fp32
// arrays (x, y, w) read and one (w_out) written, 16 B per particle, at cfg3's shape, in
//   (a) row-per-CTA order: CTA u streams row u of each array (what reweight does: 1040 rows,
//       4 CTAs of 256 threads resident per SM, 3 quads in flight per thread), and
//   (b) grid-stride order: the same bytes as one flat stream per array (what an elementwise
//       kernel does).
// Build + run on the box:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/stream_pattern.cu
//                          -o /tmp/sp && /tmp/sp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) rows_kernel(const float4 *x, const float4 *y, const float4 *w, float4 *o,
                                                       int quads_per_row, int rows) {
  for (int u = blockIdx.x; u < rows; u += gridDim.x) {
    const size_t base = static_cast<size_t>(u) * quads_per_row;
    float acc = 0.f;
    for (int g = threadIdx.x; g < quads_per_row; g += blockDim.x) {
      const float4 a = __ldg(x + base + g), b = __ldg(y + base + g), c = __ldg(w + base + g);
      float4 r;
      r.x = a.x + b.x + c.x;
      r.y = a.y + b.y + c.y;
      r.z = a.z + b.z + c.z;
      r.w = a.w + b.w + c.w;
      acc += r.x;
      __stcs(o + base + g, r);
    }
    if (acc == 1.2345f) o[0] = make_float4(acc, 0, 0, 0);
  }
}

__global__ void flat_kernel(const float4 *x, const float4 *y, const float4 *w, float4 *o, size_t n) {
  for (size_t g = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; g < n;
       g += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldg(x + g), b = __ldg(y + g), c = __ldg(w + g);
    float4 r;
    r.x = a.x + b.x + c.x;
    r.y = a.y + b.y + c.y;
    r.z = a.z + b.z + c.z;
    r.w = a.w + b.w + c.w;
    __stcs(o + g, r);
  }
}

int main() {
  const int T = 1040, P = 8192, Q = P / 4;
  const size_t n = static_cast<size_t>(T) * Q;
  float4 *d;
  cudaMalloc(&d, 6 * n * sizeof(float4));   // x y v psi omega w as in the particle store, + w_out
  float4 *x = d, *y = d + n, *w = d + 5 * n, *o;
  cudaMalloc(&o, n * sizeof(float4));
  cudaMemset(d, 0, 6 * n * sizeof(float4));
  cudaMemset(o, 0, n * sizeof(float4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 16.0 * n * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / 20;
    printf("%-40s %7.1f us  %7.1f GB/s\n", name, us, bytes / us / 1e3);
  };
  timeit("rows: grid = T (1040 CTAs x 256)", [&] { rows_kernel<<<T, 256>>>(x, y, w, o, Q, T); });
  timeit("rows: grid = 4 x SMs (persistent)", [&] { rows_kernel<<<4 * sms, 256>>>(x, y, w, o, Q, T); });
  timeit("rows: grid = T, 1024 threads", [&] { rows_kernel<<<T, 1024>>>(x, y, w, o, Q, T); });
  timeit("flat: grid-stride, 8 x SMs x 256", [&] { flat_kernel<<<8 * sms, 256>>>(x, y, w, o, n); });
  timeit("flat: grid-stride, 32 x SMs x 256", [&] { flat_kernel<<<32 * sms, 256>>>(x, y, w, o, n); });
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
