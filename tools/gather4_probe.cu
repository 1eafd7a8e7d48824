// MEASUREMENT INFRASTRUCTURE (not the product): TMA tile::gather4 of 128-B rows of a C matrix
// (rows x R fp32) into a 128-B-swizzled shared-memory ring -- the K3c producers' gather, issued by
// the TMA unit instead of 16-B cp.async per lane.  Checks the landed bytes against the expected
// swizzled layout for box heights 1 and 4 and R = 32 / 24 (columns past R must read 0), then
// times a gather4 stream against the cp.async form.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W_%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap *m, int c0, int r0, int r1, int r2,
                                   int r3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}

// one CTA: gather rows idx[0..31] (8 gather4) into a 4 KB swizzled tile, copy it out raw
__global__ void check_kernel(const __grid_constant__ CUtensorMap m, const int *idx, float *out) {
  __shared__ __align__(1024) uint8_t tile[4096 + 1024];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t t = (su32(tile) + 1023) & ~1023u, b = su32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(4096) : "memory");
    for (int k = 0; k < 8; ++k)
      g4(t + 512 * k, &m, 0, idx[4 * k], idx[4 * k + 1], idx[4 * k + 2], idx[4 * k + 3], b);
  }
  wait(b, 0);
  const uint8_t *base = tile + (t - su32(tile));
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) out[e] = reinterpret_cast<const float *>(base)[e];
}

// throughput: every CTA streams `iters` batches of 128 rows (32 gather4 from 32 lanes of warp 0)
__global__ void __launch_bounds__(128) stream_g4(const __grid_constant__ CUtensorMap m, const int *idx,
                                                 int64_t nidx, int iters, float *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (su32(sm) + 1023) & ~1023u;
  __shared__ __align__(8) uint64_t bars[4];
  if (threadIdx.x == 0) {
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(bars + k)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int st = it & 3;
    const uint32_t bar = su32(bars + st), dst = base + st * 16384;
    if (it >= 4) {
      wait(su32(bars + st), ((it >> 2) - 1) & 1);
    }
    if (threadIdx.x < 32) {
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(16384) : "memory");
      __syncwarp();
      const int64_t o = ((int64_t)(blockIdx.x * iters + it) * 128 + 4 * lane) % (nidx - 4);
      const int4 r = *reinterpret_cast<const int4 *>(idx + (o & ~3ll));
      g4(dst + 512 * lane, &m, 0, r.x, r.y, r.z, r.w, bar);
    }
    if (it >= 3) {  // consume stage it - 3
      const int cs = (it - 3) & 3;
      wait(su32(bars + cs), ((it - 3) >> 2) & 1);
      const uint8_t *p = sm + (base - su32(sm)) + cs * 16384;
      acc += reinterpret_cast<const float *>(p)[threadIdx.x * 32];
      __syncthreads();
    }
  }
  if (acc == 1.2345f) *sink = acc;
}

__global__ void __launch_bounds__(128) stream_cp(const float4 *C, const int *idx, int64_t nidx, int iters,
                                                 float *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (su32(sm) + 1023) & ~1023u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, gc = lane & 7, gs = lane >> 3;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int st = it & 3;
    const int64_t o = ((int64_t)(blockIdx.x * iters + it) * 128 + 32 * w) % (nidx - 32);
    const int my = idx[o + lane];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int s = 4 * k + gs, r = __shfl_sync(0xffffffffu, my, s);
      const uint32_t dst = base + st * 16384 + (32 * w + s) * 128 + ((gc ^ (s & 7)) << 4);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(C + (int64_t)r * 8 + gc));
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (it >= 3) {
      asm volatile("cp.async.wait_group 3;\n" ::: "memory");
      __syncthreads();
      const uint8_t *p = sm + (base - su32(sm)) + ((it - 3) & 3) * 16384;
      acc += reinterpret_cast<const float *>(p)[threadIdx.x * 32];
      __syncthreads();
    }
  }
  if (acc == 1.2345f) *sink = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
  const int64_t rows = 480189;
  auto enc = encoder();
  int *idx;
  float *out, *sink;
  const int64_t nidx = 1 << 24;
  std::vector<int> h(nidx);
  uint64_t s = 88172645463325252ull;
  for (auto &v : h) {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    v = (int)(s % (uint64_t)rows);
  }
  CK(cudaMalloc(&idx, nidx * 4));
  CK(cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, 4096));
  CK(cudaMalloc(&sink, 4));
  for (int R : {32, 24}) {
    std::vector<float> hc(rows * R);
    for (int64_t i = 0; i < rows * R; ++i) hc[i] = (float)(i % 100003) + 0.25f;
    float *C;
    CK(cudaMalloc(&C, rows * R * 4));
    CK(cudaMemcpy(C, hc.data(), rows * R * 4, cudaMemcpyHostToDevice));
    for (int bh : {1}) {  // gather4 needs box height 1 (4: illegal instruction)
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)rows};
      cuuint64_t strides[1] = {(cuuint64_t)R * 4};
      cuuint32_t box[2] = {32, (cuuint32_t)bh};
      cuuint32_t es[2] = {1, 1};
      CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (rc != CUDA_SUCCESS) {
        printf("R=%d box height %d: encode failed %d\n", R, bh, (int)rc);
        continue;
      }
      check_kernel<<<1, 128>>>(m, idx, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("R=%d box height %d: %s\n", R, bh, cudaGetErrorString(e));
        return 1;
      }
      std::vector<float> ho(1024);
      CK(cudaMemcpy(ho.data(), out, 4096, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int t = 0; t < 32; ++t)
        for (int c = 0; c < 32; ++c) {
          const int chunk = c >> 2, pos = ((chunk ^ (t & 7)) << 2) + (c & 3);
          const float want = c < R ? hc[(int64_t)h[t] * R + c] : 0.f;
          if (ho[t * 32 + pos] != want) ++bad;
        }
      printf("R=%d box height %d: %d mismatches of 1024 (swizzled layout, zero past R)\n", R, bh, bad);
    }
    CK(cudaFree(C));
  }
  // throughput (R = 32)
  {
    float *C;
    CK(cudaMalloc(&C, rows * 128));
    CK(cudaMemset(C, 0, rows * 128));
    CUtensorMap m;
    cuuint64_t dims[2] = {32, (cuuint64_t)rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t smem = 4 * 16384 + 1024;
    CK(cudaFuncSetAttribute(stream_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(stream_cp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int iters = 2000;
    for (int bps : {1, 2, 3}) {
      cudaEvent_t a, b;
      cudaEventCreate(&a), cudaEventCreate(&b);
      float t1 = 0, t2 = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        stream_g4<<<sms * bps, 128, smem>>>(m, idx, nidx, iters, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&t1, a, b);
        cudaEventRecord(a);
        stream_cp<<<sms * bps, 128, smem>>>(reinterpret_cast<const float4 *>(C), idx, nidx, iters, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&t2, a, b);
      }
      const double nrows = (double)sms * bps * iters * 128;
      printf("%d CTA/SM: gather4 %.1f G rows/s, cp.async %.1f G rows/s\n", bps, nrows / t1 / 1e6,
             nrows / t2 / 1e6);
    }
  }
  return 0;
}
