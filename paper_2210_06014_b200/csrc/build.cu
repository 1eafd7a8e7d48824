// K1  B-CSF builder on the GPU (replaces csf.build_tree, csf.py:101-196).
//
// Pipeline (every step a data-parallel device primitive; no host loop over entries):
//   1. pack the coordinates in cyclic level order (root, root+1, ...) into <=64-bit keys;
//      > 64 key bits run several stable LSD radix passes (least significant level chunk first),
//      which is exactly np.lexsort's order (csf.py:120-124).  Coordinates are unique
//      (coo.py:56-59), so any correct sort is bit-exact.
//   2. gather the sorted level columns K_d and values; first-differing-level per entry (fdl).
//   3. fiber starts = fdl <= N-2 (csf.py:126-133); root runs over fibers; greedy split of each
//      run into ceil(len/thr) chunks of whole fibers (csf.py:136-148).
//   4. node starts per depth = (fdl <= d) | subtensor start (csf.py:157-166); inds / ptrs by
//      compaction and an exclusive scan of the next depth's starts (csf.py:168-178).
//   5. fiber_coord, sub_leaf_ptr (csf.py:180-183) and the row (root slice) index the exact
//      row-owner kernels walk.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <vector>

#include "ft_common.cuh"

namespace ft {
namespace {

struct Scratch {
  cudaStream_t s;
  std::vector<void *> ptrs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void *p : ptrs) cudaFreeAsync(p, s);
  }
  template <class T>
  T *get(size_t n) {
    void *p = nullptr;
    if (cudaMallocAsync(&p, n * sizeof(T) + 16, s) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T *>(p);
  }
};

struct LevelChunk {
  int d0, d1;  // levels [d0, d1)
  int shift[FT_MAX_ORDER];
  int bits;
};

struct PackArgs {
  int N;
  int lm[FT_MAX_ORDER];  // level -> mode
  int d0, d1;
  int shift[FT_MAX_ORDER];
};

__global__ void pack_keys(const int32_t *__restrict__ idx, const int32_t *__restrict__ perm,
                          int64_t nnz, PackArgs a, uint64_t *__restrict__ keys,
                          int32_t *__restrict__ iota_out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  int64_t e = perm ? perm[p] : p;
  if (iota_out) iota_out[p] = (int32_t)p;
  const int32_t *row = idx + e * a.N;
  uint64_t k = 0;
  for (int d = a.d0; d < a.d1; ++d) k |= (uint64_t)(uint32_t)row[a.lm[d]] << a.shift[d];
  keys[p] = k;
}

struct GatherArgs {
  int N;
  int lm[FT_MAX_ORDER];
  int32_t *K[FT_MAX_ORDER];
};

// K_d[p] = idx[perm[p], lm[d]] and vals (one random read of each entry's row, coalesced writes)
__global__ void gather_levels(const int32_t *__restrict__ idx, const float *__restrict__ vals,
                              const int32_t *__restrict__ perm, int64_t nnz, GatherArgs a,
                              float *__restrict__ vout) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int64_t e = perm[p];
  const int32_t *row = idx + e * a.N;
  for (int d = 0; d < a.N; ++d) a.K[d][p] = row[a.lm[d]];
  vout[p] = vals[e];
}

// fdl[p] = first level where sorted entry p differs from p-1 (coalesced reads of the K_d);
// N means an exact duplicate of its predecessor -> the smallest such original entry index
__global__ void first_diff_level(const int32_t *__restrict__ perm, int64_t nnz, GatherArgs a,
                                 uint8_t *__restrict__ fdl, unsigned long long *__restrict__ dup_min) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  int first = 0;
  if (p > 0) {
    first = a.N;
    for (int d = 0; d < a.N; ++d)
      if (a.K[d][p] != a.K[d][p - 1]) {
        first = d;
        break;
      }
  }
  fdl[p] = (uint8_t)first;
  if (first == a.N) atomicMin(dup_min, (unsigned long long)perm[p]);
}

// Single-chunk keys (sum of level bits <= 64: orders 3 / 4 at the BASELINE shapes): the sorted
// key IS the level-ordered coordinate tuple, so the levels, values (carried as the sort
// payload) and first-differing level decode from the sorted arrays with coalesced reads -- no
// random gather of idx[perm[p]] (was ~5 ms per Netflix tree).  An equal key pair (duplicate)
// sets *dup_flag; the caller then reruns the perm-based path for the reference's error report.
struct DecodeArgs {
  int N;
  int shift[FT_MAX_ORDER];
  uint64_t mask[FT_MAX_ORDER];
  int32_t *K[FT_MAX_ORDER];
};

__global__ void decode_levels(const uint64_t *__restrict__ keys, const uint32_t *__restrict__ vbits,
                              int64_t nnz, DecodeArgs a, float *__restrict__ vout,
                              uint8_t *__restrict__ fdl, int *__restrict__ dup_flag) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint64_t k = keys[p];
  for (int d = 0; d < a.N; ++d) a.K[d][p] = (int32_t)((k >> a.shift[d]) & a.mask[d]);
  vout[p] = __uint_as_float(vbits[p]);
  int first = 0;
  if (p > 0) {
    const uint64_t x = k ^ keys[p - 1];
    if (x == 0) {
      first = a.N;
      *dup_flag = 1;
    } else {
      const int hb = 63 - __clzll((long long)x);  // highest differing bit -> its level
      first = a.N - 1;
      for (int d = 0; d < a.N; ++d)
        if (a.mask[d] && hb >= a.shift[d] && hb < a.shift[d] + 64 - __clzll((long long)a.mask[d])) {
          first = d;
          break;
        }
    }
  }
  fdl[p] = (uint8_t)first;
}

__global__ void pack_keys_vals(const int32_t *__restrict__ idx, const float *__restrict__ vals,
                               int64_t nnz, PackArgs a, uint64_t *__restrict__ keys,
                               uint32_t *__restrict__ vbits) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int32_t *row = idx + p * a.N;
  uint64_t k = 0;
  for (int d = a.d0; d < a.d1; ++d) k |= (uint64_t)(uint32_t)row[a.lm[d]] << a.shift[d];
  keys[p] = k;
  vbits[p] = __float_as_uint(vals[p]);
}

__global__ void flags_le(const uint8_t *__restrict__ fdl, const uint8_t *__restrict__ extra,
                         int64_t n, int lim, uint8_t *__restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  out[p] = (fdl[p] <= lim) || (extra && extra[p]);
}

// select predicates over positions (DeviceSelect::If, no flag pass): a fiber starts where the
// first differing level is <= N-2; a fiber starts a root slice where level 0 changed
struct FdlLe {
  const uint8_t *fdl;
  int lim;
  __device__ __forceinline__ bool operator()(int32_t i) const { return fdl[i] <= lim; }
};
struct RunStart {
  const int32_t *fiber_ptr;
  const uint8_t *fdl;
  __device__ __forceinline__ bool operator()(int32_t f) const { return fdl[fiber_ptr[f]] == 0; }
};

__global__ void chunk_counts(const int32_t *__restrict__ run_start, int64_t nruns, int64_t F,
                             int64_t thr, int32_t *__restrict__ nch) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  int64_t len = (r + 1 < nruns ? run_start[r + 1] : F) - run_start[r];
  nch[r] = thr > 0 ? (int32_t)((len + thr - 1) / thr) : 1;
}

__global__ void write_chunks(const int32_t *__restrict__ run_start,
                             const int32_t *__restrict__ nch, const int32_t *__restrict__ off,
                             int64_t nruns, int64_t thr, const int32_t *__restrict__ fiber_ptr,
                             int32_t *__restrict__ sub_fiber_ptr,
                             int32_t *__restrict__ sub_leaf_ptr, uint8_t *__restrict__ subflag) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= nruns) return;
  int32_t n = nch[r], o = off[r], s0 = run_start[r];
  for (int32_t c = 0; c < n; ++c) {
    int32_t f = s0 + (int32_t)(c * (thr > 0 ? thr : 0));
    int32_t leaf = fiber_ptr[f];
    sub_fiber_ptr[o + c] = f;
    sub_leaf_ptr[o + c] = leaf;
    subflag[leaf] = 1;
  }
}

__global__ void gather_i32(const int32_t *__restrict__ src, const int32_t *__restrict__ pos,
                           int64_t n, int32_t *__restrict__ dst, int64_t dst_stride) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  dst[k * dst_stride] = src[pos[k]];
}

__global__ void set_i32(int32_t *p, int32_t v) { *p = v; }

inline unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// K1b: leaf-major index.  One warp per 32 fibers: lane f owns fiber f's leaf range; the warp
// then writes the ranges cooperatively (consecutive lanes -> consecutive leaves), so the store
// stream is coalesced even when fibers hold one leaf each (Netflix tree 0: 1.006 leaves/fiber).
__global__ void leaf_pc_kernel(const int32_t *__restrict__ fiber_ptr,
                               const int32_t *__restrict__ fiber_coord, int64_t F, int N,
                               int32_t *__restrict__ leaf_pc) {
  const int NP = N - 2;  // prefix levels 1..N-2 per leaf (<= 4)
  const int lane = threadIdx.x & 31;
  const int64_t f0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~(int64_t)31;
  const int64_t f = f0 + lane;
  int lb = 0, le = 0, pc[4] = {0, 0, 0, 0};
  if (f < F) {
    lb = __ldg(fiber_ptr + f);
    le = __ldg(fiber_ptr + f + 1);
#pragma unroll
    for (int d = 0; d < 4; ++d)
      if (d < NP) pc[d] = __ldg(fiber_coord + f * (N - 1) + 1 + d);
  }
  const int first = __shfl_sync(0xffffffffu, lb, 0);
  int last = le;
  for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
  // leaves [first, last) of this warp's fibers: each leaf finds its fiber among the 32 ranges
  // (warp-uniform trip count: every lane takes part in the shuffles)
  for (int base = first; base < last; base += 32) {
    const int L = base + lane;
    int lo = 0;  // largest k with lb_k <= L among the warp's real fibers (5 halving steps)
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
      const int lbm = __shfl_sync(0xffffffffu, lb, lo + step);
      if (lbm <= L && f0 + lo + step < F) lo += step;
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int v = __shfl_sync(0xffffffffu, pc[d], lo);
      if (d < NP && L < last) leaf_pc[(int64_t)L * NP + d] = v;
    }
  }
}

__global__ void seg_count_kernel(const int32_t *__restrict__ rlp, int64_t rows, int max_len,
                                 int32_t *__restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) cnt[r] = (__ldg(rlp + r + 1) - __ldg(rlp + r) + max_len - 1) / max_len;
}

__global__ void seg_fill_kernel(const int32_t *__restrict__ rlp, const int32_t *__restrict__ rc,
                                const int32_t *__restrict__ off, int64_t rows, int max_len,
                                int32_t *__restrict__ seg_coord, int32_t *__restrict__ seg_ptr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const int lb = __ldg(rlp + r), le = __ldg(rlp + r + 1), c = __ldg(rc + r);
  int o = __ldg(off + r);
  for (int L = lb; L < le; L += max_len, ++o) {
    seg_coord[o] = c;
    seg_ptr[o] = L;
  }
  if (r == rows - 1) seg_ptr[o] = le;
}

__global__ void row_leaf_ptr_kernel(const int32_t *__restrict__ fiber_ptr,
                                    const int32_t *__restrict__ row_fiber_ptr, int64_t rows,
                                    int32_t *__restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= rows) out[r] = __ldg(fiber_ptr + __ldg(row_fiber_ptr + r));
}

// Compaction of the positions whose flag is set: out[k] = k-th set position; returns count.
struct Compactor {
  cudaStream_t s;
  Scratch &sc;
  int64_t *d_count;
  int64_t n_max;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  Compactor(cudaStream_t st, Scratch &scr, int64_t nmax) : s(st), sc(scr), n_max(nmax) {
    d_count = sc.get<int64_t>(1);
    thrust::counting_iterator<int32_t> it(0);
    size_t b1 = 0, b2 = 0, b3 = 0;
    cub::DeviceSelect::Flagged(nullptr, b1, it, (const uint8_t *)nullptr, (int32_t *)nullptr,
                               d_count, nmax, s);
    cub::DeviceSelect::If(nullptr, b2, it, (int32_t *)nullptr, d_count, nmax, FdlLe{nullptr, 0}, s);
    cub::DeviceSelect::If(nullptr, b3, it, (int32_t *)nullptr, d_count, nmax, RunStart{nullptr, nullptr}, s);
    tmp_bytes = b1 > b2 ? b1 : b2;
    tmp_bytes = tmp_bytes > b3 ? tmp_bytes : b3;
    tmp = sc.get<uint8_t>(tmp_bytes);
  }
  int run(const uint8_t *flags, int64_t n, int32_t *out, int64_t *host_count) {
    thrust::counting_iterator<int32_t> it(0);
    size_t b = tmp_bytes;
    FT_CUDA(cub::DeviceSelect::Flagged(tmp, b, it, flags, out, d_count, n, s));
    return fetch(host_count);
  }
  // positions i < n with pred(i), no flag array (the predicate reads fdl directly)
  template <class Pred>
  int run_if(Pred pred, int64_t n, int32_t *out, int64_t *host_count) {
    thrust::counting_iterator<int32_t> it(0);
    size_t b = tmp_bytes;
    FT_CUDA(cub::DeviceSelect::If(tmp, b, it, out, d_count, n, pred, s));
    return fetch(host_count);
  }
  int fetch(int64_t *host_count) {
    FT_CUDA(cudaMemcpyAsync(host_count, d_count, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FT_CUDA(cudaStreamSynchronize(s));
    return FT_OK;
  }
};

// ---- derived build: tree (t+1) from tree t's leaf order -------------------------------------
// Tree t holds the entries sorted by (i_t, i_{t+1}, ..., i_{t+N-1}); a STABLE sort of that
// sequence by (i_{t+1}, ..., i_{t+N-1}) alone gives (i_{t+1}, ..., i_{t+N-1}, i_t) -- tree t+1's
// order -- because equal keys keep their i_t-ascending order.  The key drops tree t's root
// level, so at the BASELINE shapes it fits 32 bits (Netflix: 27 / 31 bits, 4 radix passes of
// 4-byte keys instead of 6 of 8-byte keys); the payload carries (i_t, value).
__global__ void row_start_mark(const int32_t *__restrict__ row_leaf_ptr, int64_t rows,
                               uint32_t *__restrict__ mark) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) mark[__ldg(row_leaf_ptr + r)] = (uint32_t)r;
}

struct DerivedArgs {
  int N;
  int shift[FT_MAX_ORDER];  // new level d (< N-1) -> bit shift in the key
};

// N is a template parameter: the level loops unroll and the shift / mask / column tables stay in
// registers (with a runtime N the parameter structs were copied to the stack per thread)
template <int N>
__global__ void pack_derived(const uint32_t *__restrict__ leaf_row, const int32_t *__restrict__ row_coord,
                             const int32_t *__restrict__ leaf_pc, const int32_t *__restrict__ leaf_coord,
                             const float *__restrict__ vals, int64_t nnz, DerivedArgs a,
                             uint32_t *__restrict__ keys, unsigned long long *__restrict__ pay) {
  const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= nnz) return;
  constexpr int NP = N - 2;
  uint32_t k = 0;
  // new level d = old level d + 1: old levels 1..N-2 from leaf_pc, old level N-1 = leaf_coord
#pragma unroll
  for (int d = 0; d < NP; ++d) k |= (uint32_t)__ldg(leaf_pc + L * NP + d) << a.shift[d];
  k |= (uint32_t)__ldg(leaf_coord + L) << a.shift[N - 2];
  keys[L] = k;
  const uint32_t root = (uint32_t)__ldg(row_coord + __ldg(leaf_row + L));
  pay[L] = ((unsigned long long)root << 32) | __float_as_uint(__ldg(vals + L));
}

template <int N>
__global__ void decode_derived(const uint32_t *__restrict__ keys,
                               const unsigned long long *__restrict__ pay, int64_t nnz,
                               DerivedArgs a, DecodeArgs da, float *__restrict__ vout,
                               uint8_t *__restrict__ fdl) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const uint32_t k = keys[p];
  const unsigned long long q = pay[p];
#pragma unroll
  for (int d = 0; d < N - 1; ++d) da.K[d][p] = (int32_t)((k >> a.shift[d]) & (uint32_t)da.mask[d]);
  da.K[N - 1][p] = (int32_t)(q >> 32);
  vout[p] = __uint_as_float((uint32_t)q);
  int first = 0;
  if (p > 0) {
    const uint32_t x = k ^ keys[p - 1];
    if (x == 0) {
      first = N - 1;  // same prefix: the entries differ in the (old root) leaf level
    } else {
      // the most significant differing bit lies in the first (most significant) level whose
      // field it falls in; levels are laid out from level 0 (top) down
      const int hb = 31 - __clz((int)x);
      first = N - 2;
#pragma unroll
      for (int d = N - 2; d >= 0; --d)
        if (da.mask[d] && hb >= a.shift[d]) first = d < first ? d : first;
    }
  }
  fdl[p] = (uint8_t)first;
}

struct LeafPcArgs {
  const int32_t *K[4];
};
template <int NP>
__global__ void leaf_pc_from_levels(LeafPcArgs a, int64_t nnz, int32_t *__restrict__ out) {
  const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= nnz) return;
#pragma unroll
  for (int d = 0; d < NP; ++d) out[L * NP + d] = __ldg(a.K[d] + L);
}

// Everything after the level columns K_d (sorted, level order) and first-differing levels are
// known: fibers, root slices, subtensor split, fiber_coord, per-depth inds / ptrs (csf.py:126-183).
int finish_tree(cudaStream_t s, Scratch &sc, int N, int64_t nnz, int64_t thr, bool compact,
                int32_t *const *K, const uint8_t *fdl, int32_t *const *inds, int32_t *const *ptrs,
                int32_t *fiber_ptr, int32_t *fiber_coord, int32_t *sub_fiber_ptr,
                int32_t *sub_leaf_ptr, int32_t *row_fiber_ptr, int32_t *row_coord,
                int64_t *counts_out, int32_t *leaf_pc) {
  const unsigned nb = blocks_for(nnz);
  // every leaf carries its fiber's levels 1..N-2 in K_d; at order 3 K_1 IS the leaf_pc buffer
  // (the builders alias it), at orders 4-6 the columns are interleaved into it
  if (leaf_pc && N >= 4 && N <= 6) {
    LeafPcArgs la{};
    for (int d = 0; d < N - 2; ++d) la.K[d] = K[d + 1];
    if (N == 4) leaf_pc_from_levels<2><<<nb, 256, 0, s>>>(la, nnz, leaf_pc);
    if (N == 5) leaf_pc_from_levels<3><<<nb, 256, 0, s>>>(la, nnz, leaf_pc);
    if (N == 6) leaf_pc_from_levels<4><<<nb, 256, 0, s>>>(la, nnz, leaf_pc);
    if (int rc = check_launch("leaf_pc_from_levels")) return rc;
  }
  GatherArgs ga{};
  ga.N = N;
  for (int d = 0; d < N; ++d) ga.K[d] = K[d];
  Compactor comp(s, sc, nnz + 1);
  uint8_t *flagA = sc.get<uint8_t>(nnz), *flagB = sc.get<uint8_t>(nnz);
  uint8_t *subflag = sc.get<uint8_t>(nnz);
  int32_t *scan = sc.get<int32_t>(nnz + 1);
  int32_t *pos = sc.get<int32_t>(nnz + 1);
  if (!flagA || !flagB || !subflag || !scan || !pos)
    return fail(FT_ERR_CUDA, "ft_build_tree: out of device memory (flags)");

  // fibers: runs of equal first N-1 levels
  int64_t F = 0;
  if (int rc = comp.run_if(FdlLe{fdl, N - 2}, nnz, fiber_ptr, &F)) return rc;
  set_i32<<<1, 1, 0, s>>>(fiber_ptr + F, (int32_t)nnz);

  // root slices over fibers
  int64_t nruns = 0;
  if (int rc = comp.run_if(RunStart{fiber_ptr, fdl}, F, row_fiber_ptr, &nruns)) return rc;
  set_i32<<<1, 1, 0, s>>>(row_fiber_ptr + nruns, (int32_t)F);
  // row_coord[r] = K_0[fiber_ptr[row_fiber_ptr[r]]]
  {
    int32_t *first_leaf = sc.get<int32_t>(nruns);
    gather_i32<<<blocks_for(nruns), 256, 0, s>>>(fiber_ptr, row_fiber_ptr, nruns, first_leaf, 1);
    gather_i32<<<blocks_for(nruns), 256, 0, s>>>(ga.K[0], first_leaf, nruns, row_coord, 1);
  }

  // greedy split of each root slice into <= thr whole fibers (csf.py:136-148)
  int32_t *nch = sc.get<int32_t>(nruns), *off = sc.get<int32_t>(nruns + 1);
  chunk_counts<<<blocks_for(nruns), 256, 0, s>>>(row_fiber_ptr, nruns, F, thr, nch);
  {
    size_t b = 0;
    FT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, nch, off, nruns + 1, s));
    void *t = sc.get<uint8_t>(b);
    // off has nruns+1 entries: scan over nch padded with a trailing read is unsafe, so scan
    // nruns entries and compute the total separately.
    FT_CUDA(cub::DeviceScan::ExclusiveSum(t, b, nch, off, nruns, s));
  }
  int32_t hlast[2] = {0, 0};
  FT_CUDA(cudaMemcpyAsync(&hlast[0], off + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FT_CUDA(cudaMemcpyAsync(&hlast[1], nch + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FT_CUDA(cudaStreamSynchronize(s));
  const int64_t S = (int64_t)hlast[0] + hlast[1];
  if (!compact) {
    FT_CUDA(cudaMemsetAsync(subflag, 0, nnz, s));
    write_chunks<<<blocks_for(nruns), 256, 0, s>>>(row_fiber_ptr, nch, off, nruns, thr, fiber_ptr,
                                                   sub_fiber_ptr, sub_leaf_ptr, subflag);
    if (int rc = check_launch("write_chunks")) return rc;
    set_i32<<<1, 1, 0, s>>>(sub_fiber_ptr + S, (int32_t)F);
    set_i32<<<1, 1, 0, s>>>(sub_leaf_ptr + S, (int32_t)nnz);
  }

  // fiber_coord[f, d] = K_d[fiber_ptr[f]] (NULL: a compact tree without fiber coordinates --
  // build_forest(keep_fibers=False); the row-owner sweeps read the leaf-major index instead)
  if (fiber_coord)
    for (int d = 0; d < N - 1; ++d)
      gather_i32<<<blocks_for(F), 256, 0, s>>>(ga.K[d], fiber_ptr, F, fiber_coord + d, N - 1);

  // per-depth node starts; inds / ptrs.  Depth N-1: every leaf (inds[N-1] already written).
  counts_out[4 + N - 1] = nnz;
  int64_t n_next = nnz;
  uint8_t *flag_next = nullptr;  // flags of depth d+1 (null => all ones)
  size_t scan_bytes = 0;
  FT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, flagA, scan, nnz, s));
  void *scan_tmp = sc.get<uint8_t>(scan_bytes);
  uint8_t *fl[2] = {flagA, flagB};
  for (int d = N - 2; d >= 0 && !compact; --d) {
    uint8_t *flag_d = fl[d & 1];
    flags_le<<<nb, 256, 0, s>>>(fdl, subflag, nnz, d, flag_d);
    int64_t n_d = 0;
    if (int rc = comp.run(flag_d, nnz, pos, &n_d)) return rc;
    gather_i32<<<blocks_for(n_d), 256, 0, s>>>(ga.K[d], pos, n_d, inds[d], 1);
    if (flag_next == nullptr) {
      // child id of a start at position p is p itself
      FT_CUDA(cudaMemcpyAsync(ptrs[d], pos, n_d * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    } else {
      size_t b = scan_bytes;
      FT_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, b, flag_next, scan, nnz, s));
      gather_i32<<<blocks_for(n_d), 256, 0, s>>>(scan, pos, n_d, ptrs[d], 1);
    }
    set_i32<<<1, 1, 0, s>>>(ptrs[d] + n_d, (int32_t)n_next);
    counts_out[4 + d] = n_d;
    n_next = n_d;
    flag_next = flag_d;
  }
  if (int rc = check_launch("build_tree")) return rc;
  FT_CUDA(cudaStreamSynchronize(s));
  counts_out[0] = F;
  counts_out[1] = S;
  counts_out[2] = nruns;
  return FT_OK;
}

}  // namespace
}  // namespace ft

using namespace ft;

extern "C" int ft_build_tree(int32_t N, int64_t nnz, const int64_t *dims, const int32_t *idx,
                             const float *vals, int32_t root_mode, int64_t thr, float *leaf_vals,
                             int32_t *const *inds, int32_t *const *ptrs, int32_t *fiber_ptr,
                             int32_t *fiber_coord, int32_t *sub_fiber_ptr, int32_t *sub_leaf_ptr,
                             int32_t *row_fiber_ptr, int32_t *row_coord, int64_t *counts_out,
                             int32_t *leaf_pc, void *stream) {
  if (N < 2 || N > FT_MAX_ORDER) return fail(FT_ERR_ARG, "ft_build_tree: order %d unsupported", N);
  if (nnz <= 0) return fail(FT_ERR_EMPTY, "cannot index an empty tensor");
  if (nnz >= (int64_t)INT32_MAX) return fail(FT_ERR_UNSUPPORTED, "nnz %lld >= 2^31", (long long)nnz);
  if (root_mode < 0 || root_mode >= N) return fail(FT_ERR_ARG, "root_mode out of range");
  // compact build (ptrs == NULL): only what the sweep kernels read -- leaf coordinates, values,
  // fiber_ptr / fiber_coord and the rows; the per-depth inds[d < N-1] / ptrs and the subtensor
  // arrays (reference-format fields) are neither computed nor stored
  const bool compact = ptrs == nullptr;
  if (!dims || !idx || !vals || !leaf_vals || !inds || !inds[N - 1] || !fiber_ptr ||
      (!fiber_coord && !compact) || !row_fiber_ptr || !row_coord || !counts_out ||
      (!compact && (!sub_fiber_ptr || !sub_leaf_ptr)))
    return fail(FT_ERR_ARG, "ft_build_tree: null argument");
  keep_pool();
  cudaStream_t s = as_stream(stream);
  Scratch sc(s);

  int lm[FT_MAX_ORDER], bits[FT_MAX_ORDER];
  for (int d = 0; d < N; ++d) {
    lm[d] = (root_mode + d) % N;
    int64_t I = dims[lm[d]];
    if (I < 1 || I > (int64_t)INT32_MAX) return fail(FT_ERR_ARG, "dim %lld unsupported", (long long)I);
    bits[d] = I <= 1 ? 0 : 64 - __builtin_clzll((unsigned long long)(I - 1));
  }
  // level chunks of <= 64 bits, built from the last level backwards (LSD order)
  std::vector<LevelChunk> chunks;
  {
    int d1 = N;
    while (d1 > 0) {
      LevelChunk c{};
      c.d1 = d1;
      int tot = 0, d = d1;
      while (d > 0 && tot + bits[d - 1] <= 64) {
        tot += bits[d - 1];
        --d;
      }
      c.d0 = d;
      int sh = 0;
      for (int k = d1 - 1; k >= d; --k) {
        c.shift[k] = sh;
        sh += bits[k];
      }
      c.bits = tot;
      chunks.push_back(c);
      d1 = d;
    }
  }

  uint64_t *k0 = sc.get<uint64_t>(nnz), *k1 = sc.get<uint64_t>(nnz);
  int32_t *p0 = sc.get<int32_t>(nnz), *p1 = sc.get<int32_t>(nnz);
  if (!k0 || !k1 || !p0 || !p1) return fail(FT_ERR_CUDA, "ft_build_tree: out of device memory");
  size_t sort_bytes = 0;
  FT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, k0, k1, p0, p1, nnz, 0, 64, s));
  void *sort_tmp = sc.get<uint8_t>(sort_bytes);
  if (!sort_tmp) return fail(FT_ERR_CUDA, "ft_build_tree: out of device memory (sort)");

  const unsigned nb = blocks_for(nnz);
  // level columns (the leaf level goes straight to inds[N-1] = leaf_coord)
  GatherArgs ga{};
  ga.N = N;
  for (int d = 0; d < N; ++d) {
    ga.lm[d] = lm[d];
    ga.K[d] = (d == N - 1) ? inds[N - 1] : (d == 1 && N == 3 && leaf_pc) ? leaf_pc : sc.get<int32_t>(nnz);
    if (!ga.K[d]) return fail(FT_ERR_CUDA, "ft_build_tree: out of device memory (levels)");
  }
  uint8_t *fdl = sc.get<uint8_t>(nnz);
  bool decoded = false;
  if (chunks.size() == 1 && chunks[0].bits > 0) {
    // fast path: sort (key, value) pairs and decode (see decode_levels)
    const LevelChunk &c = chunks[0];
    PackArgs pa{};
    pa.N = N;
    for (int d = 0; d < N; ++d) pa.lm[d] = lm[d];
    pa.d0 = c.d0;
    pa.d1 = c.d1;
    for (int d = c.d0; d < c.d1; ++d) pa.shift[d] = c.shift[d];
    uint32_t *v0 = reinterpret_cast<uint32_t *>(p0), *v1 = reinterpret_cast<uint32_t *>(p1);
    pack_keys_vals<<<nb, 256, 0, s>>>(idx, vals, nnz, pa, k0, v0);
    if (int rc = check_launch("pack_keys_vals")) return rc;
    size_t b = sort_bytes;
    FT_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, b, k0, k1, v0, v1, nnz, 0, c.bits, s));
    DecodeArgs da{};
    da.N = N;
    for (int d = 0; d < N; ++d) {
      da.shift[d] = c.shift[d];
      da.mask[d] = bits[d] >= 64 ? ~0ull : ((1ull << bits[d]) - 1);
      da.K[d] = ga.K[d];
    }
    int *dflag = sc.get<int>(1);
    FT_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), s));
    decode_levels<<<nb, 256, 0, s>>>(k1, v1, nnz, da, leaf_vals, fdl, dflag);
    if (int rc = check_launch("decode_levels")) return rc;
    int hflag = 0;
    FT_CUDA(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s));
    FT_CUDA(cudaStreamSynchronize(s));
    decoded = hflag == 0;  // a duplicate: redo with the permutation to report its entry
  }
  int32_t *perm = nullptr;  // current permutation (sorted position -> entry)
  for (size_t ci = 0; ci < chunks.size() && !decoded; ++ci) {
    const LevelChunk &c = chunks[ci];
    PackArgs pa{};
    pa.N = N;
    for (int d = 0; d < N; ++d) pa.lm[d] = lm[d];
    pa.d0 = c.d0;
    pa.d1 = c.d1;
    for (int d = c.d0; d < c.d1; ++d) pa.shift[d] = c.shift[d];
    int32_t *vin = (ci == 0) ? p0 : perm;
    int32_t *vout = (vin == p0) ? p1 : p0;
    pack_keys<<<nb, 256, 0, s>>>(idx, ci == 0 ? nullptr : perm, nnz, pa, k0,
                                 ci == 0 ? p0 : nullptr);
    if (int rc = check_launch("pack_keys")) return rc;
    if (c.bits > 0) {
      size_t b = sort_bytes;
      FT_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp, b, k0, k1, vin, vout, nnz, 0, c.bits, s));
      perm = vout;
    } else {
      perm = vin;
    }
  }

  // sorted level columns via the permutation (multi-chunk keys, or the duplicate report)
  unsigned long long hdup = ~0ull;
  if (!decoded) {
    unsigned long long *dup = sc.get<unsigned long long>(1);
    FT_CUDA(cudaMemsetAsync(dup, 0xff, sizeof(unsigned long long), s));
    gather_levels<<<nb, 256, 0, s>>>(idx, vals, perm, nnz, ga, leaf_vals);
    first_diff_level<<<nb, 256, 0, s>>>(perm, nnz, ga, fdl, dup);
    if (int rc = check_launch("gather_levels")) return rc;
    FT_CUDA(cudaMemcpyAsync(&hdup, dup, sizeof(hdup), cudaMemcpyDeviceToHost, s));
    FT_CUDA(cudaStreamSynchronize(s));
  }
  for (int k = 0; k < 4 + N; ++k) counts_out[k] = 0;
  counts_out[3] = -1;
  if (hdup != ~0ull) {
    counts_out[3] = (int64_t)hdup;
    return fail(FT_ERR_DUPLICATE, "duplicate coordinate at entry %lld", (long long)hdup);
  }

  return finish_tree(s, sc, N, nnz, thr, compact, ga.K, fdl, inds, ptrs, fiber_ptr, fiber_coord,
                     sub_fiber_ptr, sub_leaf_ptr, row_fiber_ptr, row_coord, counts_out, leaf_pc);
}

extern "C" int ft_tree_leaf_index(const ft_tree_t *tree, int32_t *leaf_pc, int32_t *row_leaf_ptr,
                                  void *stream) {
  if (!tree) return fail(FT_ERR_ARG, "null tree");
  if (tree->order < 3) return fail(FT_ERR_ARG, "order %d < 3", tree->order);
  cudaStream_t s = as_stream(stream);
  const int64_t F = tree->num_fibers, rows = tree->num_rows;
  if (leaf_pc && F > 0) {
    if (!tree->fiber_ptr || !tree->fiber_coord) return fail(FT_ERR_ARG, "null fiber arrays");
    if (tree->order > 6) return fail(FT_ERR_UNSUPPORTED, "leaf index: order %d > 6", tree->order);
    leaf_pc_kernel<<<blocks_for(F), 256, 0, s>>>(tree->fiber_ptr, tree->fiber_coord, F,
                                                 tree->order, leaf_pc);
    if (int rc = check_launch("ft_tree_leaf_index(leaf_pc)")) return rc;
  }
  if (row_leaf_ptr) {
    if (!tree->fiber_ptr || !tree->row_fiber_ptr) return fail(FT_ERR_ARG, "null row arrays");
    row_leaf_ptr_kernel<<<blocks_for(rows + 1), 256, 0, s>>>(tree->fiber_ptr,
                                                             tree->row_fiber_ptr, rows,
                                                             row_leaf_ptr);
    if (int rc = check_launch("ft_tree_leaf_index(row_leaf_ptr)")) return rc;
  }
  return FT_OK;
}

extern "C" int ft_tree_row_segments(const ft_tree_t *tree, int32_t max_len, int32_t *seg_coord,
                                    int32_t *seg_leaf_ptr, int64_t *nseg_out, void *stream) {
  if (!tree || !seg_coord || !seg_leaf_ptr || !nseg_out) return fail(FT_ERR_ARG, "null argument");
  if (max_len < 1) return fail(FT_ERR_ARG, "max_len %d < 1", max_len);
  if (!tree->row_leaf_ptr || !tree->row_coord) return fail(FT_ERR_ARG, "tree has no row index");
  cudaStream_t s = as_stream(stream);
  const int64_t rows = tree->num_rows;
  if (rows == 0) {
    *nseg_out = 0;
    FT_CUDA(cudaMemsetAsync(seg_leaf_ptr, 0, sizeof(int32_t), s));
    FT_CUDA(cudaStreamSynchronize(s));
    return FT_OK;
  }
  Scratch sc(s);
  int32_t *cnt = sc.get<int32_t>(rows + 1), *off = sc.get<int32_t>(rows + 1);
  if (!cnt || !off) return fail(FT_ERR_CUDA, "scratch allocation failed");
  seg_count_kernel<<<blocks_for(rows), 256, 0, s>>>(tree->row_leaf_ptr, rows, max_len, cnt);
  if (int rc = check_launch("ft_tree_row_segments(count)")) return rc;
  FT_CUDA(cudaMemsetAsync(cnt + rows, 0, sizeof(int32_t), s));
  size_t tb = 0;
  FT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, rows + 1, s));
  void *tmp = sc.get<uint8_t>(tb);
  if (!tmp) return fail(FT_ERR_CUDA, "scratch allocation failed");
  FT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, rows + 1, s));
  seg_fill_kernel<<<blocks_for(rows), 256, 0, s>>>(tree->row_leaf_ptr, tree->row_coord, off, rows,
                                                   max_len, seg_coord, seg_leaf_ptr);
  if (int rc = check_launch("ft_tree_row_segments(fill)")) return rc;
  int32_t total = 0;
  FT_CUDA(cudaMemcpyAsync(&total, off + rows, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FT_CUDA(cudaStreamSynchronize(s));
  *nseg_out = total;
  return FT_OK;
}

extern "C" int ft_build_tree_derived(const ft_tree_t *prev, const int64_t *dims, int64_t thr,
                                     float *leaf_vals, int32_t *const *inds, int32_t *const *ptrs,
                                     int32_t *fiber_ptr, int32_t *fiber_coord,
                                     int32_t *sub_fiber_ptr, int32_t *sub_leaf_ptr,
                                     int32_t *row_fiber_ptr, int32_t *row_coord,
                                     int64_t *counts_out, int32_t *leaf_pc, void *stream) {
  if (!prev || !dims) return fail(FT_ERR_ARG, "ft_build_tree_derived: null argument");
  const int N = prev->order;
  const int64_t nnz = prev->nnz;
  if (N < 3 || N > 6) return fail(FT_ERR_UNSUPPORTED, "ft_build_tree_derived: order %d", N);
  if (!prev->leaf_pc || !prev->row_leaf_ptr || !prev->row_coord || !prev->leaf_coord || !prev->vals)
    return fail(FT_ERR_UNSUPPORTED, "ft_build_tree_derived: previous tree lacks the leaf index");
  if (nnz <= 0) return fail(FT_ERR_EMPTY, "cannot index an empty tensor");
  const bool compact = ptrs == nullptr;
  if (!leaf_vals || !inds || !inds[N - 1] || !fiber_ptr || (!fiber_coord && !compact) ||
      !row_fiber_ptr || !row_coord || !counts_out || (!compact && (!sub_fiber_ptr || !sub_leaf_ptr)))
    return fail(FT_ERR_ARG, "ft_build_tree_derived: null argument");
  const int root = (prev->root_mode + 1) % N;
  int lm[FT_MAX_ORDER], bits[FT_MAX_ORDER];
  for (int d = 0; d < N; ++d) {
    lm[d] = (root + d) % N;
    const int64_t I = dims[lm[d]];
    bits[d] = I <= 1 ? 0 : 64 - __builtin_clzll((unsigned long long)(I - 1));
  }
  int key_bits = 0;
  for (int d = 0; d < N - 1; ++d) key_bits += bits[d];
  if (key_bits > 32 || bits[N - 1] > 32)
    return fail(FT_ERR_UNSUPPORTED, "ft_build_tree_derived: %d key bits > 32", key_bits);
  keep_pool();
  cudaStream_t s = as_stream(stream);
  Scratch sc(s);
  DerivedArgs a{};
  a.N = N;
  {
    int sh = 0;
    for (int d = N - 2; d >= 0; --d) {  // level 0 most significant
      a.shift[d] = sh;
      sh += bits[d];
    }
  }
  const int64_t rows = prev->num_rows;
  const unsigned nb = blocks_for(nnz);
  // row index of every leaf of the previous tree: mark row starts, inclusive max-scan
  uint32_t *mark = sc.get<uint32_t>(nnz), *leaf_row = sc.get<uint32_t>(nnz);
  uint32_t *k0 = sc.get<uint32_t>(nnz), *k1 = sc.get<uint32_t>(nnz);
  unsigned long long *q0 = sc.get<unsigned long long>(nnz), *q1 = sc.get<unsigned long long>(nnz);
  if (!mark || !leaf_row || !k0 || !k1 || !q0 || !q1)
    return fail(FT_ERR_CUDA, "ft_build_tree_derived: out of device memory");
  FT_CUDA(cudaMemsetAsync(mark, 0, nnz * sizeof(uint32_t), s));
  row_start_mark<<<blocks_for(rows), 256, 0, s>>>(prev->row_leaf_ptr, rows, mark);
  {
    size_t b = 0;
    FT_CUDA(cub::DeviceScan::InclusiveScan(nullptr, b, mark, leaf_row, cub::Max(), nnz, s));
    void *t = sc.get<uint8_t>(b);
    if (!t) return fail(FT_ERR_CUDA, "ft_build_tree_derived: out of device memory (scan)");
    FT_CUDA(cub::DeviceScan::InclusiveScan(t, b, mark, leaf_row, cub::Max(), nnz, s));
  }
  switch (N) {
#define FT_PACK(n)                                                                               \
  case n:                                                                                        \
    pack_derived<n><<<nb, 256, 0, s>>>(leaf_row, prev->row_coord, prev->leaf_pc, prev->leaf_coord, \
                                       prev->vals, nnz, a, k0, q0);                              \
    break;
    FT_PACK(3) FT_PACK(4) FT_PACK(5) FT_PACK(6)
#undef FT_PACK
  }
  if (int rc = check_launch("pack_derived")) return rc;
  {
    size_t b = 0;
    FT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, k0, k1, q0, q1, nnz, 0, key_bits, s));
    void *t = sc.get<uint8_t>(b);
    if (!t) return fail(FT_ERR_CUDA, "ft_build_tree_derived: out of device memory (sort)");
    FT_CUDA(cub::DeviceRadixSort::SortPairs(t, b, k0, k1, q0, q1, nnz, 0, key_bits, s));
  }
  int32_t *K[FT_MAX_ORDER];
  DecodeArgs da{};
  da.N = N;
  for (int d = 0; d < N; ++d) {
    K[d] = (d == N - 1) ? inds[N - 1] : (d == 1 && N == 3 && leaf_pc) ? leaf_pc : sc.get<int32_t>(nnz);
    if (!K[d]) return fail(FT_ERR_CUDA, "ft_build_tree_derived: out of device memory (levels)");
    da.K[d] = K[d];
    da.mask[d] = bits[d] >= 64 ? ~0ull : ((1ull << bits[d]) - 1);
  }
  uint8_t *fdl = sc.get<uint8_t>(nnz);
  switch (N) {
#define FT_DECODE(n)                                                                   \
  case n:                                                                              \
    decode_derived<n><<<nb, 256, 0, s>>>(k1, q1, nnz, a, da, leaf_vals, fdl);          \
    break;
    FT_DECODE(3) FT_DECODE(4) FT_DECODE(5) FT_DECODE(6)
#undef FT_DECODE
  }
  if (int rc = check_launch("decode_derived")) return rc;
  for (int k = 0; k < 4 + N; ++k) counts_out[k] = 0;
  counts_out[3] = -1;
  return finish_tree(s, sc, N, nnz, thr, compact, K, fdl, inds, ptrs, fiber_ptr, fiber_coord,
                     sub_fiber_ptr, sub_leaf_ptr, row_fiber_ptr, row_coord, counts_out, leaf_pc);
}
