// K7  Synthetic COO generator: the distribution of coo.generate_synthetic (coo.py:164-213) --
// nnz DISTINCT cells uniform without replacement, values U[lo, hi] -- produced on the GPU
// (counter-based hashing, not numpy's PCG64 stream; parity inputs come from the reference).
//
//   1. draw m > nnz i.i.d. uniform cells as packed keys (one 64-bit hash per mode, exact
//      multiply-high range reduction), radix-sort, drop duplicates; top up until >= nnz remain;
//   2. give every distinct cell a random 64-bit priority and keep the nnz smallest -- a uniform
//      subset of a uniform i.i.d. sample, i.e. sampling without replacement;
//   3. decode the kept keys (in priority order = a random entry order) and draw values.
#include <cub/cub.cuh>

#include "ft_common.cuh"

namespace ft {
namespace {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct KeyLayout {
  int N;
  int shift[FT_MAX_ORDER];
  int bits[FT_MAX_ORDER];
  uint64_t dims[FT_MAX_ORDER];
};

__global__ void draw_keys(KeyLayout L, uint64_t seed, uint64_t ctr0, int64_t m,
                          uint64_t *__restrict__ keys) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  uint64_t key = 0;
  const uint64_t base = mix64(seed ^ 0x5851f42d4c957f2dull) ^ ((ctr0 + (uint64_t)k) * L.N);
  for (int n = 0; n < L.N; ++n) {
    const uint64_t h = mix64(base + (uint64_t)n * 0xd1b54a32d192ed03ull);
    key |= __umul64hi(h, L.dims[n]) << L.shift[n];
  }
  keys[k] = key;
}

__global__ void priorities(const uint64_t *__restrict__ keys, int64_t m, uint64_t seed,
                           uint64_t *__restrict__ pri) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  pri[k] = mix64(keys[k] ^ mix64(seed + 0x632be59bd9b4e019ull));
}

__global__ void decode(KeyLayout L, const uint64_t *__restrict__ keys, int64_t nnz,
                       uint64_t seed, float lo, float hi, int32_t *__restrict__ idx,
                       float *__restrict__ vals) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const uint64_t key = keys[k];
  for (int n = 0; n < L.N; ++n)
    idx[k * L.N + n] = (int32_t)((key >> L.shift[n]) & ((1ull << L.bits[n]) - 1ull));
  const uint64_t h = mix64(mix64(seed ^ 0x2545f4914f6cdd1dull) + (uint64_t)k);
  const float u = (float)((h >> 40) * (1.0 / 16777216.0));  // [0, 1), 24 bits
  vals[k] = lo + (hi - lo) * u;
}

// Index spaces wider than 64 bits (order 6 / 10 at 10 K per mode: 84 / 140 bits): i.i.d. uniform
// cells without a dedup pass -- the expected number of repeated cells, nnz^2 / (2 * capacity), is
// < 1e-7 at 200 M entries in 10^24 cells, and the B-CSF builder rejects any duplicate anyway.
__global__ void draw_iid(KeyLayout L, uint64_t seed, int64_t nnz, float lo, float hi,
                         int32_t *__restrict__ idx, float *__restrict__ vals) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const uint64_t base = mix64(seed ^ 0x5851f42d4c957f2dull) ^ ((uint64_t)k * L.N);
  for (int n = 0; n < L.N; ++n) {
    const uint64_t h = mix64(base + (uint64_t)n * 0xd1b54a32d192ed03ull);
    idx[k * L.N + n] = (int32_t)__umul64hi(h, L.dims[n]);
  }
  const uint64_t h = mix64(mix64(seed ^ 0x2545f4914f6cdd1dull) + (uint64_t)k);
  vals[k] = lo + (hi - lo) * (float)((h >> 40) * (1.0 / 16777216.0));
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace
}  // namespace ft

using namespace ft;

extern "C" int ft_generate_coo(int32_t N, const int64_t *dims, int64_t nnz, uint64_t seed,
                               float lo, float hi, int32_t *idx, float *vals, void *stream) {
  if (N < 2 || N > FT_MAX_ORDER || !dims || !idx || !vals)
    return fail(FT_ERR_ARG, "ft_generate_coo: bad arguments");
  if (nnz < 1) return fail(FT_ERR_ARG, "nnz must be positive");
  if (!(lo < hi)) return fail(FT_ERR_ARG, "value range must satisfy lo < hi");
  KeyLayout L{};
  L.N = N;
  int total = 0;
  double cap = 1.0;
  for (int n = N - 1; n >= 0; --n) {
    if (dims[n] < 1 || dims[n] > INT32_MAX) return fail(FT_ERR_ARG, "bad dim");
    const int b = dims[n] <= 1 ? 0 : 64 - __builtin_clzll((unsigned long long)(dims[n] - 1));
    L.shift[n] = total;
    L.bits[n] = b;
    L.dims[n] = (uint64_t)dims[n];
    total += b;
    cap *= (double)dims[n];
  }
  if ((double)nnz > cap) return fail(FT_ERR_ARG, "nnz exceeds capacity");
  if (total > 64) {
    if ((double)nnz * (double)nnz / (2.0 * cap) > 1e-6)
      return fail(FT_ERR_UNSUPPORTED, "key needs %d > 64 bits and the space is not sparse", total);
    draw_iid<<<nblk(nnz), 256, 0, as_stream(stream)>>>(L, seed, nnz, lo, hi, idx, vals);
    if (int rc = check_launch("ft_generate_coo(iid)")) return rc;
    FT_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return FT_OK;
  }
  if ((double)nnz > 0.5 * cap)
    return fail(FT_ERR_UNSUPPORTED, "dense request (nnz > capacity/2) not supported on device");
  keep_pool();
  cudaStream_t s = as_stream(stream);
  // expected duplicates ~ m^2 / (2 cap): draw with a margin, top up if short
  const double dup = (double)nnz * (double)nnz / (2.0 * cap);
  int64_t m = nnz + (int64_t)(2.0 * dup) + nnz / 100 + 1024;
  uint64_t *keys = nullptr, *tmpk = nullptr, *pri = nullptr, *prio_out = nullptr;
  int64_t *d_count = nullptr;
  int64_t have = 0;       // distinct keys currently in `keys`
  uint64_t ctr = 0;
  int rc = FT_OK;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  for (int round = 0; round < 16; ++round) {
    const int64_t draw = (round == 0) ? m : (nnz - have) * 2 + 1024;
    const int64_t tot = have + draw;
    uint64_t *nk = nullptr, *nk2 = nullptr;
    FT_CUDA(cudaMallocAsync(&nk, tot * 8, s));
    FT_CUDA(cudaMallocAsync(&nk2, tot * 8, s));
    if (have) FT_CUDA(cudaMemcpyAsync(nk, keys, have * 8, cudaMemcpyDeviceToDevice, s));
    draw_keys<<<nblk(draw), 256, 0, s>>>(L, seed, ctr, draw, nk + have);
    ctr += (uint64_t)draw;
    if (keys) cudaFreeAsync(keys, s);
    size_t b1 = 0, b2 = 0;
    if (!d_count) FT_CUDA(cudaMallocAsync(&d_count, 8, s));
    cub::DeviceRadixSort::SortKeys(nullptr, b1, nk, nk2, tot, 0, total > 0 ? total : 1, s);
    cub::DeviceSelect::Unique(nullptr, b2, nk2, nk, d_count, tot, s);
    size_t need = b1 > b2 ? b1 : b2;
    if (need > tmp_bytes) {
      if (tmp) cudaFreeAsync(tmp, s);
      FT_CUDA(cudaMallocAsync(&tmp, need, s));
      tmp_bytes = need;
    }
    b1 = tmp_bytes;
    FT_CUDA(cub::DeviceRadixSort::SortKeys(tmp, b1, nk, nk2, tot, 0, total > 0 ? total : 1, s));
    b2 = tmp_bytes;
    FT_CUDA(cub::DeviceSelect::Unique(tmp, b2, nk2, nk, d_count, tot, s));
    FT_CUDA(cudaMemcpyAsync(&have, d_count, 8, cudaMemcpyDeviceToHost, s));
    FT_CUDA(cudaStreamSynchronize(s));
    cudaFreeAsync(nk2, s);
    keys = nk;
    if (have >= nnz) break;
  }
  if (have < nnz) {
    rc = fail(FT_ERR_CUDA, "generator could not draw enough distinct cells");
  } else {
    FT_CUDA(cudaMallocAsync(&pri, have * 8, s));
    FT_CUDA(cudaMallocAsync(&prio_out, have * 8, s));
    FT_CUDA(cudaMallocAsync(&tmpk, have * 8, s));
    priorities<<<nblk(have), 256, 0, s>>>(keys, have, seed, pri);
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, pri, prio_out, keys, tmpk, have, 0, 64, s);
    void *t2 = nullptr;
    FT_CUDA(cudaMallocAsync(&t2, b, s));
    FT_CUDA(cub::DeviceRadixSort::SortPairs(t2, b, pri, prio_out, keys, tmpk, have, 0, 64, s));
    decode<<<nblk(nnz), 256, 0, s>>>(L, tmpk, nnz, seed, lo, hi, idx, vals);
    rc = check_launch("ft_generate_coo");
    cudaFreeAsync(t2, s);
  }
  if (keys) cudaFreeAsync(keys, s);
  if (pri) cudaFreeAsync(pri, s);
  if (prio_out) cudaFreeAsync(prio_out, s);
  if (tmpk) cudaFreeAsync(tmpk, s);
  if (tmp) cudaFreeAsync(tmp, s);
  if (d_count) cudaFreeAsync(d_count, s);
  FT_CUDA(cudaStreamSynchronize(s));
  return rc;
}
