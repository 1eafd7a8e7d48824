// K2  C^(u) = A^(u) B^(u): refresh_dot_mode (_ckern.pyx:21-33 / _pykern.py:16-26) with the
// divergence guard of train.py:101-110 fused into the same pass over A.
//
// HBM-bound (8 flop/B at fp32 for J = R = 32): each warp streams a contiguous 32-row tile of A
// through shared memory with coalesced 128-bit loads, computes the 32 x R outputs with the
// reference's sequential-j accumulation order, and writes C back through shared memory as one
// contiguous, coalesced store.
#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int WARPS = 4;
constexpr int TILE = 32;  // rows per warp

struct Dsts {
  float *p[FT_MAX_PEERS];
  int n;
};

__global__ void __launch_bounds__(WARPS * 32)
    refresh_kernel(int64_t I, int J, int R, const float *__restrict__ A,
                   const float *__restrict__ Bt, Dsts dst, uint32_t *guard) {
  __shared__ float bts[FT_MAX_RANK][FT_MAX_RANK + 1];
  __shared__ float tile[WARPS][TILE][FT_MAX_RANK + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < R * J; k += blockDim.x) bts[k / J][k % J] = Bt[k];
  __syncthreads();
  const int64_t row0 = ((int64_t)blockIdx.x * WARPS + w) * TILE;
  if (row0 >= I) return;
  const int rows = (int)(I - row0 < TILE ? I - row0 : TILE);
  const int nA = rows * J;
  const float *src = A + row0 * J;
  uint32_t gmax = 0;
  for (int k = lane; k < nA; k += 32) {
    float v = __ldcs(src + k);
    gmax = max(gmax, abs_bits(v));
    tile[w][k / J][k % J] = v;
  }
  if (guard) guard_max(guard, gmax);
  __syncwarp();
  float out[FT_MAX_RANK];
  if (lane < rows) {
    float a[FT_MAX_RANK];
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j) a[j] = j < J ? tile[w][lane][j] : 0.f;
#pragma unroll
    for (int r = 0; r < FT_MAX_RANK; ++r) {
      float s = 0.f;
      if (r < R) {
        // sequential j, as the reference (padded j >= J contribute exact zeros at the end)
#pragma unroll
        for (int j = 0; j < FT_MAX_RANK; ++j)
          if (j < J) s = __fmaf_rn(a[j], bts[r][j], s);
      }
      out[r] = s;
    }
  }
  __syncwarp();
  if (lane < rows) {
#pragma unroll
    for (int r = 0; r < FT_MAX_RANK; ++r)
      if (r < R) tile[w][lane][r] = out[r];
  }
  __syncwarp();
  // the tile goes to every destination: the local C_u and, for the fused refresh + all-gather,
  // each peer rank's C_u through its CUDA-IPC-mapped pointer (NVLink stores on a multi-GPU node)
  const int nC = rows * R;
  for (int d = 0; d < dst.n; ++d) {
    float *out = dst.p[d] + row0 * R;
    for (int k = lane; k < nC; k += 32) __stcs(out + k, tile[w][k / R][k % R]);
  }
}

}  // namespace
}  // namespace ft

extern "C" int ft_refresh(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt,
                          float *C, uint32_t *guard, void *stream) {
  using namespace ft;
  if (I < 0 || J < 1 || R < 1 || J > FT_MAX_RANK || R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ft_refresh: I=%lld J=%d R=%d outside kernel cover",
                (long long)I, J, R);
  if (I == 0) return FT_OK;
  if (!A || !Bt || !C) return fail(FT_ERR_ARG, "ft_refresh: null pointer");
  const int64_t blocks = (I + WARPS * TILE - 1) / (WARPS * TILE);
  Dsts d{};
  d.p[0] = C;
  d.n = 1;
  refresh_kernel<<<(unsigned)blocks, WARPS * 32, 0, as_stream(stream)>>>(I, J, R, A, Bt, d, guard);
  return check_launch("ft_refresh");
}

extern "C" int ft_refresh_scatter(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt,
                                  float *const *dsts, int32_t ndst, uint32_t *guard,
                                  void *stream) {
  using namespace ft;
  if (I < 0 || J < 1 || R < 1 || J > FT_MAX_RANK || R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ft_refresh_scatter: I=%lld J=%d R=%d outside kernel cover",
                (long long)I, J, R);
  if (!dsts || ndst < 1 || ndst > FT_MAX_PEERS)
    return fail(FT_ERR_ARG, "ft_refresh_scatter: 1..%d destinations required", FT_MAX_PEERS);
  if (I == 0) return FT_OK;
  if (!A || !Bt) return fail(FT_ERR_ARG, "ft_refresh_scatter: null pointer");
  Dsts d{};
  for (int k = 0; k < ndst; ++k) {
    if (!dsts[k]) return fail(FT_ERR_ARG, "ft_refresh_scatter: null destination %d", k);
    d.p[k] = dsts[k];
  }
  d.n = ndst;
  const int64_t blocks = (I + WARPS * TILE - 1) / (WARPS * TILE);
  refresh_kernel<<<(unsigned)blocks, WARPS * 32, 0, as_stream(stream)>>>(I, J, R, A, Bt, d, guard);
  return check_launch("ft_refresh_scatter");
}
