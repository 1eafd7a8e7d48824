// MEASUREMENT INFRASTRUCTURE (not the product): on-chip bandwidth peaks of this B200 for the
// roofline bench.py reports.  MEASURED_PEAKS.json (driver-written) carries the HBM copy
// bandwidth; the sweeps' binding units are on chip (the gathered C rows are L2 / L1 hits), so
// their roofline needs these denominators too:
//   ftp_l2_read_gbs   : L2 -> SM read bandwidth, 16-B ld.global.cg (L1 bypassed) over a
//                       24 MB buffer that stays L2-resident, every SM busy
//   ftp_l1_read_gbs   : L1 hit bandwidth, 16-B ld.global.ca over a 32 KB per-CTA window
//   ftp_smem_read_gbs : shared-memory read bandwidth, conflict-free LDS.128
// Each is the best of `reps` timed launches (CUDA events) after a warm-up launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__global__ void __launch_bounds__(512) l2_read(const float4 *__restrict__ buf, int64_t n4,
                                               int iters, float *sink) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int it = 0; it < iters; ++it)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v;
      asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(buf + i));
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 123.456f) *sink = acc.x;
}

__global__ void __launch_bounds__(512) l1_read(const float4 *__restrict__ buf, int win4,
                                               int iters, float *sink) {
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *w = buf + (int64_t)(blockIdx.x % 64) * win4;
  for (int it = 0; it < iters; ++it)
#pragma unroll 4
    for (int i = threadIdx.x; i < win4; i += blockDim.x) {
      float4 v;
      asm volatile("ld.global.ca.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(w + i));
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 123.456f) *sink = acc.x;
}

__global__ void __launch_bounds__(512) smem_read(int iters, float *sink) {
  __shared__ float4 s[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    s[i] = make_float4((float)i, 1.f, 2.f, 3.f);
  __syncthreads();
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = s[(threadIdx.x + k * 512 + it) & 2047];
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 123.456f) *sink = acc.x;
}

int sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

template <class F>
double best_ms(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

}  // namespace

extern "C" {

int ftp_l2_read_gbs(int reps, double *out) {
  const int64_t bytes = 24ll << 20;
  const int64_t n4 = bytes / 16;
  float4 *buf = nullptr;
  float *sink = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess) return 1;
  cudaMemset(buf, 0, bytes);
  const int iters = 20, grid = sms() * 4;
  const double ms = best_ms([&] { l2_read<<<grid, 512>>>(buf, n4, iters, sink); }, reps);
  *out = (double)bytes * iters / (ms * 1e-3) / 1e9;
  cudaFree(buf);
  cudaFree(sink);
  return cudaGetLastError() != cudaSuccess;
}

int ftp_l1_read_gbs(int reps, double *out) {
  const int win4 = 2048;  // 32 KB per CTA window (64 distinct windows)
  float4 *buf = nullptr;
  float *sink = nullptr;
  if (cudaMalloc(&buf, (size_t)64 * win4 * 16) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess)
    return 1;
  cudaMemset(buf, 0, (size_t)64 * win4 * 16);
  const int iters = 400, grid = sms() * 2;
  const double ms = best_ms([&] { l1_read<<<grid, 512>>>(buf, win4, iters, sink); }, reps);
  *out = (double)grid * win4 * 16.0 * iters / (ms * 1e-3) / 1e9;
  cudaFree(buf);
  cudaFree(sink);
  return cudaGetLastError() != cudaSuccess;
}

int ftp_smem_read_gbs(int reps, double *out) {
  float *sink = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return 1;
  const int iters = 4000, grid = sms() * 4;
  const double ms = best_ms([&] { smem_read<<<grid, 512>>>(iters, sink); }, reps);
  *out = (double)grid * 512 * 16.0 * 4 * iters / (ms * 1e-3) / 1e9;
  cudaFree(sink);
  return cudaGetLastError() != cudaSuccess;
}

}  // extern "C"
