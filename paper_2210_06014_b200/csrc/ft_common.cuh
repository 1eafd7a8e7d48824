// Shared helpers for the sm_100a FasterTucker kernels (libft_b200.so).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "ft_b200.h"

namespace ft {

void set_error(const char *fmt, ...);
int fail(ft_status st, const char *fmt, ...);
int check_launch(const char *what);
int sm_count();
void keep_pool();

constexpr unsigned FULL = 0xffffffffu;

#define FT_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      return ::ft::fail(FT_ERR_CUDA, "%s:%d %s -> %s", __FILE__, __LINE__, #call,        \
                        cudaGetErrorString(_e));                                         \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// |x| as ordered uint bits: for non-negative floats, uint order == float order, and NaN
// (0x7fc00000+) sorts above +inf (0x7f800000).  Used by the fused divergence guards.
__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

__device__ __forceinline__ void guard_max(uint32_t *guard, uint32_t bits) {
  // warp-aggregate then one atomic per warp
  bits = __reduce_max_sync(FULL, bits);
  if ((threadIdx.x & 31) == 0 && guard) atomicMax(guard, bits);
}

// Streaming (read-once) loads: do not pollute L1; the gathered C rows use the default path.
__device__ __forceinline__ int ld_stream(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float *p) { return __ldcs(p); }

}  // namespace ft
