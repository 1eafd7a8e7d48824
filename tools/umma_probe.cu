// MEASUREMENT INFRASTRUCTURE (not the product): latency of one K3c combine (a batch of
// tcgen05.mma kind::tf32, M = 128, N = 32 or 64, K = 8 per instruction) from issue to the
// commit's mbarrier arrive, for the schedules the factor sweep could use:
//   dep12   : 12 MMAs into one accumulator (3xTF32 over 4 k-steps)
//   split2  : 4 x (N = 64: A_hi [Bt_hi | Bt_lo]) + 4 x (N = 32: A_lo Bt_hi), two accumulators
//   ss12    : dep12 with A from shared memory instead of TMEM
//   batch4  : four dep12 batches (four accumulators) issued back to back, one commit
// One CTA per SM, every SM busy; clock64 cycles per batch, averaged.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W_%=;\n}\n" ::"r"(su32(bar)), "r"(ph) : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(int mode, int iters, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t *base = (uint8_t *)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t *bar = (uint64_t *)(base + 3 * 16384 + 32768);
  uint32_t *slot = (uint32_t *)(bar + 1);
  for (int i = threadIdx.x; i < (3 * 16384 + 32768) / 4; i += 128) ((float *)base)[i] = 0.001f * (i & 63);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *slot;
  const uint32_t i32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t i64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const uint32_t bh = su32(base), bl = bh + 4096, asm_ = su32(base + 16384);
  long long t0 = 0;
  uint32_t ph = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (mode == 0) {
        const uint32_t ah = tmem, al = tmem + 32, d = tmem + 64;
        for (int k = 0; k < 4; ++k) {
          mma_ts(d, al + 8 * k, sw128(bh + 32 * k), i32, k > 0);
          mma_ts(d, ah + 8 * k, sw128(bl + 32 * k), i32, 1);
          mma_ts(d, ah + 8 * k, sw128(bh + 32 * k), i32, 1);
        }
      } else if (mode == 1) {
        const uint32_t ah = tmem, al = tmem + 32, d1 = tmem + 64, d2 = tmem + 128;
        for (int k = 0; k < 4; ++k) {
          mma_ts(d1, ah + 8 * k, sw128(bh + 32 * k), i64, k > 0);  // B rows 0-63 = [hi; lo]
          mma_ts(d2, al + 8 * k, sw128(bh + 32 * k), i32, k > 0);
        }
      } else if (mode == 2) {
        const uint32_t d = tmem + 64;
        for (int k = 0; k < 4; ++k) {
          mma_ss(d, sw128(asm_ + 32 * k), sw128(bh + 32 * k), i32, k > 0);
          mma_ss(d, sw128(asm_ + 32 * k), sw128(bl + 32 * k), i32, 1);
          mma_ss(d, sw128(asm_ + 32 * k), sw128(bh + 32 * k), i32, 1);
        }
      } else if (mode >= 4) {  // 12 dependent MMAs at N = 64 / 128 / 256
        const uint32_t nN = mode == 4 ? 64u : mode == 5 ? 128u : 256u;
        const uint32_t iN = (1u << 4) | (2u << 7) | (2u << 10) | ((nN >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t ah = tmem, d = tmem + 256;
        for (int k = 0; k < 12; ++k) mma_ts(d, ah + 8 * (k & 3), sw128(bh + 32 * (k & 3)), iN, k > 0);
      } else {
        for (int bb = 0; bb < 4; ++bb) {
          const uint32_t ah = tmem + 96 * bb, al = ah + 32, d = ah + 64;
          for (int k = 0; k < 4; ++k) {
            mma_ts(d, al + 8 * k, sw128(bh + 32 * k), i32, k > 0);
            mma_ts(d, ah + 8 * k, sw128(bl + 32 * k), i32, 1);
            mma_ts(d, ah + 8 * k, sw128(bh + 32 * k), i32, 1);
          }
        }
      }
      commit(bar);
      wait(bar, ph);
      ph ^= 1;
    }
    t0 = clock64() - t0;
    out[blockIdx.x] = t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *out;
  cudaMalloc(&out, sizeof(long long) * sms);
  const size_t smem = 3 * 16384 + 32768 + 1024 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char *names[7] = {"dep12 (TS, one accumulator)", "split2 (N=64 hi|lo + N=32 lo)",
                          "ss12 (A from smem)", "batch4 (4 x dep12, one commit)",
                          "12 x N=64", "12 x N=128", "12 x N=256"};
  const int iters = 2000;
  for (int mode = 0; mode < 7; ++mode) {
    probe<<<sms, 128, smem>>>(mode, 10, out);
    probe<<<sms, 128, smem>>>(mode, iters, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: CUDA error %s\n", names[mode], cudaGetErrorString(e));
      return 1;
    }
    long long h[1024];
    cudaMemcpy(h, out, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("%-34s %8.1f cycles per commit round\n", names[mode], avg / iters);
  }
  return 0;
}
