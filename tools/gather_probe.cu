// MEASUREMENT INFRASTRUCTURE (not the product): how fast can one B200 gather random 128-B rows
// (the C^(n) rows of the sweeps) and read per-slot metadata streams, for the access patterns the
// K3b designs use.  Prints one line per pattern: G rows/s and the on-chip GB/s they imply.
//   coop8   : 8 lanes per row, 4 rows per LDG.128 warp instruction (coalesced per row)
//   quad4   : 4 lanes per row, 2 LDG.128 per lane (quadr DIRECT)
//   thread  : one thread per row, 8 LDG.128 per thread (lane-per-row consumer)
//   meta_div: each thread walks its own 4-B stream (32 different lines per instruction)
//   meta_coal: the same bytes read coalesced
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

constexpr int ITERS = 64;  // rows per lane-group per launch pass

__global__ void __launch_bounds__(256) coop8(const float4 *__restrict__ C, const int *__restrict__ idx,
                                             int64_t nidx, float *sink) {
  const int lane = threadIdx.x & 31, gs = lane >> 3, gc = lane & 7;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t b = warp * 32; b + 32 <= nidx; b += nw * 32) {
    const int my = __ldg(idx + b + lane);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = __shfl_sync(0xffffffffu, my, 4 * it + gs);
      const float4 v = __ldg(C + (int64_t)r * 8 + gc);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) *sink = acc.x;
}

__global__ void __launch_bounds__(256) quad4(const float4 *__restrict__ C, const int *__restrict__ idx,
                                             int64_t nidx, float *sink) {
  const int lane = threadIdx.x & 31, gs = lane >> 2, gc = lane & 3;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t b = warp * 32; b + 32 <= nidx; b += nw * 32) {
    const int my = __ldg(idx + b + lane);
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int r = __shfl_sync(0xffffffffu, my, 8 * it + gs);
      const float4 v = __ldg(C + (int64_t)r * 8 + 2 * gc);
      const float4 w = __ldg(C + (int64_t)r * 8 + 2 * gc + 1);
      acc.x += v.x + w.x, acc.y += v.y + w.y, acc.z += v.z + w.z, acc.w += v.w + w.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) *sink = acc.x;
}

__global__ void __launch_bounds__(256) thread_row(const float4 *__restrict__ C, const int *__restrict__ idx,
                                                  int64_t nidx, float *sink) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int64_t b = t; b < nidx; b += nt) {
    const int r = __ldg(idx + b);
    const float4 *row = C + (int64_t)r * 8;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 v = __ldg(row + c);
      acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 1.2345f) *sink = acc.x;
}

// each thread: its own stream of `len` consecutive ints at stream * len
__global__ void __launch_bounds__(256) meta_div(const int *__restrict__ m, int len, float *sink) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int *s = m + t * len;
  int acc = 0;
#pragma unroll 8
  for (int k = 0; k < len; ++k) acc += __ldg(s + k);
  if (acc == 12345) *sink = (float)acc;
}
__global__ void __launch_bounds__(256) meta_coal(const int *__restrict__ m, int len, float *sink) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int *s = m + warp * 32 * len;
  int acc = 0;
#pragma unroll 8
  for (int k = 0; k < len; ++k) acc += __ldg(s + 32 * k + lane);
  if (acc == 12345) *sink = (float)acc;
}

template <class F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t nidx = 1 << 25;  // 33.5 M rows gathered per launch
  std::vector<int> h(nidx);
  float *sink;
  CK(cudaMalloc(&sink, 4));
  int *idx;
  CK(cudaMalloc(&idx, nidx * 4));
  const int64_t table_rows[3] = {2048, 17770, 480189};  // 256 KB, 2.3 MB, 61 MB of 128-B rows
  float4 *C;
  CK(cudaMalloc(&C, table_rows[2] * 128));
  CK(cudaMemset(C, 0, table_rows[2] * 128));
  for (int ti = 0; ti < 3; ++ti) {
    uint64_t s = 88172645463325252ull;
    for (int64_t i = 0; i < nidx; ++i) {
      s ^= s << 13, s ^= s >> 7, s ^= s << 17;
      h[i] = (int)(s % (uint64_t)table_rows[ti]);
    }
    CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
    for (int bps : {4, 8}) {
      const int grid = sms * bps;
      float t1 = time_it([&] { coop8<<<grid, 256>>>(C, idx, nidx, sink); });
      float t2 = time_it([&] { quad4<<<grid, 256>>>(C, idx, nidx, sink); });
      float t3 = time_it([&] { thread_row<<<grid, 256>>>(C, idx, nidx, sink); });
      printf("table %7lld rows, %d blocks/SM x 256 thr: coop8 %.2f G rows/s (%.0f GB/s)  quad4 %.2f (%.0f)  "
             "thread %.2f (%.0f)\n",
             (long long)table_rows[ti], bps, nidx / t1 / 1e6, nidx * 128.0 / t1 / 1e6,
             nidx / t2 / 1e6, nidx * 128.0 / t2 / 1e6, nidx / t3 / 1e6, nidx * 128.0 / t3 / 1e6);
    }
  }
  // metadata streams: 256 threads x sms*8 blocks, len ints each
  {
    const int grid = sms * 8, len = 256;
    const int64_t n = (int64_t)grid * 256 * len;
    int *m;
    CK(cudaMalloc(&m, n * 4));
    CK(cudaMemset(m, 0, n * 4));
    float t1 = time_it([&] { meta_div<<<grid, 256>>>(m, len, sink); });
    float t2 = time_it([&] { meta_coal<<<grid, 256>>>(m, len, sink); });
    printf("meta streams (%lld MB): divergent %.0f GB/s (%.2f G words/s)  coalesced %.0f GB/s\n",
           (long long)(n * 4 >> 20), n * 4.0 / t1 / 1e6, n / t1 / 1e6, n * 4.0 / t2 / 1e6);
    CK(cudaFree(m));
  }
  return 0;
}
