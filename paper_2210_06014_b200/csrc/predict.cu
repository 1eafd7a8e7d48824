// K6  predict_batch / evaluate (model.py:219-230, train.py:91-98) from the coherent C^(n) cache.
//
// xhat = sum_r prod_n C_n[i_n, r], products in mode order as the reference.
// SSE / SAE accumulate in fp64 and reduce in a fixed order (per-block partials, then one block).
#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int PTHREADS = 256;

// One warp scores 32 entries per step: lane k loads entry k's coordinates (coalesced), then for
// each mode the warp issues 32 independent row gathers (lane r reads element r of the entry's
// C_n row -- one 128-B request per row), so 32 x N loads are in flight per warp; the products
// are reduced over r for all 32 entries at once by recursive halving (31 shuffles), leaving
// entry k's prediction in lane k.
template <int RP>
__global__ void __launch_bounds__(PTHREADS)
    predict_kernel(const ft_model_t m, int64_t M, const int32_t *__restrict__ idx,
                   const float *__restrict__ vals, float *__restrict__ out,
                   double *__restrict__ partials) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * PTHREADS + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * PTHREADS) >> 5;
  const int N = m.order, R = m.core_rank;
  const bool rl = lane < R;
  double sse = 0.0, sae = 0.0;
  for (int64_t base = warp * 32; base < M; base += nwarp * 32) {
    const int64_t e = base + lane;
    const bool ok = e < M;
    float t[32];
    for (int n = 0; n < N; ++n) {
      const int c = ok ? __ldcs(idx + e * N + n) : 0;
      const float *Cn = m.dots[n];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const int ck = __shfl_sync(FULL, c, k);
        const float v = rl ? __ldg(Cn + (int64_t)ck * R + lane) : 0.f;
        t[k] = n == 0 ? v : t[k] * v;
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const bool upper = lane & off;
#pragma unroll
      for (int k = 0; k < off; ++k) {
        const float send = upper ? t[k] : t[k + off];
        const float keep = upper ? t[k + off] : t[k];
        t[k] = keep + __shfl_xor_sync(FULL, send, off);
      }
    }
    if (ok) {
      const float s = t[0];  // lane k: prediction of entry base + k
      if (out) out[e] = s;
      if (vals) {
        const double res = (double)__ldcs(vals + e) - (double)s;
        sse += res * res;
        sae += fabs(res);
      }
    }
  }
  if (!partials) return;
  // block reduction (fixed order) -> partials[2*block]
  __shared__ double red[2][PTHREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sse += __shfl_xor_sync(FULL, sse, o);
    sae += __shfl_xor_sync(FULL, sae, o);
  }
  if (lane == 0) {
    red[0][threadIdx.x >> 5] = sse;
    red[1][threadIdx.x >> 5] = sae;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < PTHREADS / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
    }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
  }
}

__global__ void sum_partials(const double *__restrict__ partials, int nblocks, double *out2) {
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < nblocks; ++k) {
      a += partials[2 * k];
      b += partials[2 * k + 1];
    }
    out2[0] = a;
    out2[1] = b;
  }
}

int check_model(const ft_model_t *m) {
  if (!m || m->order < 2 || m->order > FT_MAX_ORDER) return fail(FT_ERR_ARG, "bad model");
  if (m->core_rank < 1 || m->core_rank > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "core rank %d outside kernel cover", m->core_rank);
  for (int n = 0; n < m->order; ++n)
    if (!m->dots[n]) return fail(FT_ERR_ARG, "dots[%d] null", n);
  return FT_OK;
}

int launch(const ft_model_t *m, int64_t M, const int32_t *idx, const float *vals, float *out,
           double *partials, int grid, cudaStream_t s) {
  const int R = m->core_rank;
  if (R <= 8)
    predict_kernel<8><<<grid, PTHREADS, 0, s>>>(*m, M, idx, vals, out, partials);
  else if (R <= 16)
    predict_kernel<16><<<grid, PTHREADS, 0, s>>>(*m, M, idx, vals, out, partials);
  else
    predict_kernel<32><<<grid, PTHREADS, 0, s>>>(*m, M, idx, vals, out, partials);
  return check_launch("predict_kernel");
}

}  // namespace
}  // namespace ft

using namespace ft;

extern "C" int ft_predict(const ft_model_t *model, int64_t M, const int32_t *idx, float *out,
                          void *stream) {
  if (int rc = check_model(model)) return rc;
  if (M == 0) return FT_OK;
  if (!idx || !out) return fail(FT_ERR_ARG, "ft_predict: null pointer");
  return launch(model, M, idx, nullptr, out, nullptr, sm_count() * 8, as_stream(stream));
}

extern "C" int ft_sse(const ft_model_t *model, int64_t M, const int32_t *idx, const float *vals,
                      double *out2, void *stream) {
  if (int rc = check_model(model)) return rc;
  if (!idx || !vals || !out2) return fail(FT_ERR_ARG, "ft_sse: null pointer");
  keep_pool();
  cudaStream_t s = as_stream(stream);
  const int grid = sm_count() * 8;
  double *partials = nullptr;
  FT_CUDA(cudaMallocAsync(&partials, sizeof(double) * 2 * grid, s));
  int rc = launch(model, M, idx, vals, nullptr, partials, grid, s);
  if (rc == FT_OK) {
    sum_partials<<<1, 32, 0, s>>>(partials, grid, out2);
    rc = check_launch("sum_partials");
  }
  cudaFreeAsync(partials, s);
  return rc;
}
