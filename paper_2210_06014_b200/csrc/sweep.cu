// K3b / K4 / K3a / K5: the FasterTucker factor and core SGD sweeps on sm_100a.
//
// Reference semantics (paths under /root/reference/pkg/src/fastertucker/):
//   factor_sweep  _ckern.pyx:132-199 (_pykern.py:69-137): for each fiber f of the tree rooted at
//     t = (u+1) mod N, cross[r] = prod_d C_{p_d}[fiber_coord[f,d], r] (left to right),
//     vec[j] = sum_r cross[r] Bt_u[r,j]; for each leaf: s = A_u[i].vec, e = x - s,
//     A_u[i,j] -= lr (reg A_u[i,j] - e vec[j]).
//   core_sweep    _ckern.pyx:202-269: same cross / s / e; acc[r,j] -= e cross[r] A_u[i,j].
//   apply_core_update _ckern.pyx:272-282: Bt_u -= lr (acc / omega + reg Bt_u).
//
// B200 design:
//   * K3b walks the tree ROOTED AT u.  Its root slice i is exactly the set of updates row i of
//     A_u receives, already in the reference's serial order (the tree-t order restricted to
//     i_u = i), and every other operand (C_m, m != u, and Bt_u) is frozen during the sweep.
//     So one warp owns one row: the row lives in registers (lane j holds A_u[i,j]) for the
//     whole slice, is read and written once, and no two warps ever touch the same row -- an
//     exact, deterministic, lock-free schedule.
//   * Leaves are processed in batches of 32.  The gather phase runs lanes-over-r: 32
//     independent coalesced 128-B row loads per prefix level are in flight per warp; the
//     rank products (cross) are staged in shared memory.  The combine phase runs
//     lanes-over-j: vec for all 32 leaves (J x R FMAs each) reads cross as shared-memory
//     broadcasts and Bt_u's column from registers.  Only the s -> e -> row update chain is
//     serial.
//   * K4 uses the row form of the core gradient: A_u and Bt_u are frozen during the core sweep
//     and C_u = A_u Bt_u^T is coherent, so s = A_u[i].vec = C_u[i].cross (an R-dot, no J x R
//     combine per leaf), g_i = sum_leaves e cross, and acc = -sum_i g_i (x) A_u[i], accumulated
//     per lane in registers, reduced per block in shared memory in a fixed order, and across
//     blocks by K5 -- no global atomics.
//   * K3a is the reference's own traversal (warp per fiber batch over tree t) with hogwild
//     (racing, lock-free) row updates, used for the workers>1 semantics.
#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int WPB = 8;    // warps per block
constexpr int BATCH = 32; // leaves per batch

struct SweepParams {
  int N;
  int npre;          // N-2 prefix levels (tree levels 1..N-2)
  int64_t nrows;
  const int32_t *leaf_coord;
  const float *vals;
  const int32_t *fiber_ptr;
  const int32_t *fiber_coord;
  const int32_t *row_fiber_ptr;
  const int32_t *row_coord;
  float *A;          // A_u  (I_u x J)
  const float *Bt;   // Bt_u (R x J)
  const float *Cu;   // C_u  (core sweep)
  const float *Cpre[FT_MAX_ORDER];  // C of tree levels 1..N-2 (modes u+1 .. u-2)
  const float *Cleaf;               // C_{u-1}
  int J, R;
  float lr, reg;
  float *partials;   // core: [grid][R*J]
};

// Fiber index of each of the batch's leaves (lane k -> leaf L0+k), given fcur = fiber holding
// leaf L0-1 (or L0).  At most 32 fibers can start inside a 32-leaf window.
__device__ __forceinline__ int batch_fibers(const int32_t *__restrict__ fiber_ptr, int fcur,
                                            int fend, int L0, int nb, int lane, int *fnext) {
  const int fidx = fcur + 1 + lane;
  const int fs = fidx < fend ? __ldg(fiber_ptr + fidx) : INT32_MAX;
  const unsigned bit = (fs < L0 + nb) ? (1u << (fs - L0)) : 0u;
  const unsigned mask = __reduce_or_sync(FULL, bit);
  *fnext = fcur + __popc(mask);
  return fcur + __popc(mask & (FULL >> (31 - lane)));
}

// ---- cp.async gathers ---------------------------------------------------------------------
// The gathered C rows land in shared memory without passing through registers, so a warp keeps
// 32 leaves x (N-1) rows in flight at ~60 registers (the v1 register-array gather needed 155
// registers and capped the SM at 8 warps).  .ca keeps the lines in L1: consecutive leaves of
// one fiber share their prefix rows.
__device__ __forceinline__ void cp_async4(float *dst, const float *src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async16(float *dst, const float *src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Row stride of a staged [BATCH][RS] tile: RS = RP + 4 keeps 16-B alignment for the vector
// copies and makes lane-k row reads (float4) bank-conflict free.
template <int RP>
struct Tile {
  static constexpr int RS = RP + 4;
  static constexpr int FLOATS = BATCH * RS;
};

// Stage rows C[coord_k, 0:R) of the batch's leaves k < nb into dst[k][0:R).  coord_lane holds
// leaf lane's row index.  R % 4 == 0 uses 16-B copies (R/4 lanes per row).
template <int RP>
__device__ __forceinline__ void gather_level(float *dst, const float *__restrict__ C, int R,
                                             int coord_lane, int nb, int lane) {
  constexpr int RS = Tile<RP>::RS;
  if ((R & 3) == 0) {
    const int R4 = R >> 2, total = nb * R4;
#pragma unroll
    for (int it = 0; it < RP / 4; ++it) {
      const int c = lane + 32 * it;
      const int k = c / R4, part = c - k * R4;
      const int coord = __shfl_sync(FULL, coord_lane, k & 31);
      if (c < total) cp_async16(dst + k * RS + part * 4, C + (int64_t)coord * R + part * 4);
    }
  } else {
#pragma unroll 4
    for (int k = 0; k < BATCH; ++k) {
      const int coord = __shfl_sync(FULL, coord_lane, k);
      if (k < nb && lane < R) cp_async4(dst + k * RS + lane, C + (int64_t)coord * R + lane);
    }
  }
}

// cross[k][r] = prod_levels C_level[coord][r] for the batch's leaves, left to right in the
// reference's prefix order (tree levels 1..N-2, then the leaf level), accumulated in X using Y
// as the landing buffer of the next level.
template <int RP>
__device__ __forceinline__ void stage_cross(const SweepParams &p, float *X, float *Y, int myfib,
                                            int lc, int nb, int lane) {
  constexpr int RS = Tile<RP>::RS;
  const int nlev = p.N - 1;  // N-2 prefix levels + the leaf level
  for (int lvl = 0; lvl < nlev; ++lvl) {
    const bool leaf = lvl == nlev - 1;
    const int coord =
        leaf ? lc : (lane < nb ? __ldg(p.fiber_coord + (int64_t)myfib * (p.N - 1) + 1 + lvl) : 0);
    gather_level<RP>(lvl == 0 ? X : Y, leaf ? p.Cleaf : p.Cpre[lvl], p.R, coord, nb, lane);
    if (lvl >= 1) {
      cp_async_wait_all();
      __syncwarp();
      if (lane < RP) {
        for (int k = 0; k < nb; ++k) X[k * RS + lane] *= Y[k * RS + lane];
      }
      __syncwarp();
    }
  }
}

// ------------------------------------------------------------------------------------------
// K3b: exact row-owner factor sweep
// ------------------------------------------------------------------------------------------
constexpr int WPB_R = 4;  // warps per block of the row kernels

template <int RP>
__global__ void __launch_bounds__(WPB_R * 32)
    factor_rows_kernel(const SweepParams p) {
  extern __shared__ float4 smem4[];
  constexpr int RS = Tile<RP>::RS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float *X = reinterpret_cast<float *>(smem4) + w * 2 * Tile<RP>::FLOATS;
  float *Y = X + Tile<RP>::FLOATS;
  for (int k = lane; k < 2 * Tile<RP>::FLOATS; k += 32) X[k] = 0.f;  // pads stay zero
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * WPB_R + w, nw = (int64_t)gridDim.x * WPB_R;
  const bool jl = lane < p.J;
  float bt[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) bt[r] = (jl && r < p.R) ? __ldg(p.Bt + r * p.J + lane) : 0.f;

  for (int64_t row = gw; row < p.nrows; row += nw) {
    const int i = __ldg(p.row_coord + row);
    const int fb = __ldg(p.row_fiber_ptr + row), fe = __ldg(p.row_fiber_ptr + row + 1);
    const int Lb = __ldg(p.fiber_ptr + fb), Le = __ldg(p.fiber_ptr + fe);
    float *arow = p.A + (int64_t)i * p.J;
    float a = jl ? arow[lane] : 0.f;
    int fcur = fb;
    for (int L0 = Lb; L0 < Le; L0 += BATCH) {
      const int nb = min(BATCH, Le - L0);
      const int lc = lane < nb ? __ldcs(p.leaf_coord + L0 + lane) : 0;
      const float x = lane < nb ? __ldcs(p.vals + L0 + lane) : 0.f;
      int fnext;
      const int myfib = batch_fibers(p.fiber_ptr, fcur, fe, L0, nb, lane, &fnext);
      stage_cross<RP>(p, X, Y, myfib, lc, nb, lane);
      // serial chain; vec_k = sum_r cross[k][r] Bt[r][j] (sequential r, broadcast reads) is
      // independent of the row, so it overlaps the previous leaf's reduction latency
#pragma unroll 4
      for (int k = 0; k < nb; ++k) {
        const float4 *xr = reinterpret_cast<const float4 *>(X + k * RS);
        float v = 0.f;
#pragma unroll
        for (int r4 = 0; r4 < RP / 4; ++r4) {
          const float4 c4 = xr[r4];
          v = __fmaf_rn(c4.x, bt[4 * r4], v);
          v = __fmaf_rn(c4.y, bt[4 * r4 + 1], v);
          v = __fmaf_rn(c4.z, bt[4 * r4 + 2], v);
          v = __fmaf_rn(c4.w, bt[4 * r4 + 3], v);
        }
        const float s = warp_sum(a * v);
        const float e = __shfl_sync(FULL, x, k) - s;
        const float g = p.reg * a - e * v;
        a = a - p.lr * g;
      }
      __syncwarp();
      fcur = fnext;
    }
    if (jl) arow[lane] = a;
  }
}

// ------------------------------------------------------------------------------------------
// K4: core-gradient row sweep; per-block partials of G^T A_u (acc = -partials summed)
// ------------------------------------------------------------------------------------------
template <int RP>
__global__ void __launch_bounds__(WPB_R * 32)
    core_rows_kernel(const SweepParams p) {
  extern __shared__ float4 smem4[];
  constexpr int RS = Tile<RP>::RS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float *X = reinterpret_cast<float *>(smem4) + w * (2 * Tile<RP>::FLOATS + RS);
  float *Y = X + Tile<RP>::FLOATS;
  float *cus = Y + Tile<RP>::FLOATS;  // C_u[i, :] of the current row
  for (int k = lane; k < 2 * Tile<RP>::FLOATS + RS; k += 32) X[k] = 0.f;
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * WPB_R + w, nw = (int64_t)gridDim.x * WPB_R;
  const bool rl = lane < p.R;
  float acc[FT_MAX_RANK];  // lane r: acc[j] = sum_i g_i[r] A_u[i, j]
#pragma unroll
  for (int j = 0; j < FT_MAX_RANK; ++j) acc[j] = 0.f;

  for (int64_t row = gw; row < p.nrows; row += nw) {
    const int i = __ldg(p.row_coord + row);
    const int fb = __ldg(p.row_fiber_ptr + row), fe = __ldg(p.row_fiber_ptr + row + 1);
    const int Lb = __ldg(p.fiber_ptr + fb), Le = __ldg(p.fiber_ptr + fe);
    if (rl) cus[lane] = __ldg(p.Cu + (int64_t)i * p.R + lane);
    float g = 0.f;
    int fcur = fb;
    for (int L0 = Lb; L0 < Le; L0 += BATCH) {
      const int nb = min(BATCH, Le - L0);
      const int lc = lane < nb ? __ldcs(p.leaf_coord + L0 + lane) : 0;
      const float x = lane < nb ? __ldcs(p.vals + L0 + lane) : 0.f;
      int fnext;
      const int myfib = batch_fibers(p.fiber_ptr, fcur, fe, L0, nb, lane, &fnext);
      stage_cross<RP>(p, X, Y, myfib, lc, nb, lane);
      // lane k: s_k = C_u[i] . cross_k  (= A_u[i] . vec_k, since C_u = A_u Bt_u^T is coherent)
      float s = 0.f;
      {
        const float4 *xr = reinterpret_cast<const float4 *>(X + (lane & 31) * RS);
        const float4 *cr = reinterpret_cast<const float4 *>(cus);
#pragma unroll
        for (int r4 = 0; r4 < RP / 4; ++r4) {
          const float4 a4 = xr[r4], c4 = cr[r4];
          s = __fmaf_rn(a4.x, c4.x, s);
          s = __fmaf_rn(a4.y, c4.y, s);
          s = __fmaf_rn(a4.z, c4.z, s);
          s = __fmaf_rn(a4.w, c4.w, s);
        }
      }
      const float e = lane < nb ? x - s : 0.f;
      // lane r: g_i[r] += sum_k e_k cross_k[r]
#pragma unroll 4
      for (int k = 0; k < nb; ++k) {
        const float ek = __shfl_sync(FULL, e, k);
        if (lane < RP) g = __fmaf_rn(ek, X[k * RS + lane], g);
      }
      __syncwarp();
      fcur = fnext;
    }
    // acc[r][j] += g[r] * A_u[i][j]  (row broadcast to all lanes)
    const float *arow = p.A + (int64_t)i * p.J;
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j)
      if (j < p.J) acc[j] = __fmaf_rn(g, __ldg(arow + j), acc[j]);
    __syncwarp();
  }
  // block reduction in fixed warp order -> partials[block]; reuses the staging tiles
  __syncthreads();
  const int RJ = p.R * p.J;
  float *red = reinterpret_cast<float *>(smem4);
  const int wstride = 2 * Tile<RP>::FLOATS + RS;
  if (rl) {
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j)
      if (j < p.J) red[w * wstride + lane * p.J + j] = acc[j];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < RJ; k += blockDim.x) {
    float s = 0.f;
    for (int ww = 0; ww < WPB_R; ++ww) s += red[ww * wstride + k];
    p.partials[(int64_t)blockIdx.x * RJ + k] = s;
  }
}

template <int RP>
constexpr size_t factor_smem() {
  return (size_t)WPB_R * 2 * Tile<RP>::FLOATS * sizeof(float);
}
template <int RP>
constexpr size_t core_smem() {
  return (size_t)WPB_R * (2 * Tile<RP>::FLOATS + Tile<RP>::RS) * sizeof(float);
}

// ------------------------------------------------------------------------------------------
// K3a: hogwild factor sweep over fibers of tree t (the reference's traversal)
// ------------------------------------------------------------------------------------------
struct FiberParams {
  int N;
  int64_t fib_lo, fib_hi;
  const int32_t *leaf_coord;
  const float *vals;
  const int32_t *fiber_ptr;
  const int32_t *fiber_coord;
  float *A;
  const float *Bt;
  const float *Cpre[FT_MAX_ORDER];  // C of tree levels 0..N-2 (prefix modes)
  int J, R;
  float lr, reg;
};

template <int RP>
__global__ void __launch_bounds__(WPB * 32)
    factor_fibers_kernel(const FiberParams p) {
  // one buffer per warp: first the rank products (cross, stride RP), then the batch's vecs
  __shared__ __align__(16) float buf_s[WPB][BATCH * (FT_MAX_RANK + 4)];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + w, nw = (int64_t)gridDim.x * wpb;
  const bool jl = lane < p.J, rl = lane < p.R;
  float bt[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) bt[r] = (jl && r < p.R) ? __ldg(p.Bt + r * p.J + lane) : 0.f;
  float(&cs)[BATCH][RP] = *reinterpret_cast<float(*)[BATCH][RP]>(buf_s[w]);
  float(&vec_s)[BATCH][FT_MAX_RANK + 1] =
      *reinterpret_cast<float(*)[BATCH][FT_MAX_RANK + 1]>(buf_s[w]);

  for (int64_t base = p.fib_lo + gw * BATCH; base < p.fib_hi; base += nw * BATCH) {
    const int nf = (int)(p.fib_hi - base < BATCH ? p.fib_hi - base : BATCH);
    float t[BATCH];
    for (int d = 0; d < p.N - 1; ++d) {
      const int fc = lane < nf ? __ldg(p.fiber_coord + (base + lane) * (p.N - 1) + d) : 0;
      const float *Cd = p.Cpre[d];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int c = __shfl_sync(FULL, fc, k);
        const float v = (rl && k < nf) ? __ldg(Cd + (int64_t)c * p.R + lane) : 0.f;
        t[k] = d == 0 ? v : t[k] * v;
      }
    }
    if (lane < RP) {
#pragma unroll
      for (int k = 0; k < BATCH; ++k) cs[k][lane] = t[k];
    }
    __syncwarp();
    float vk[BATCH];
#pragma unroll
    for (int k = 0; k < BATCH; ++k) {
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < RP; r += 4) {
        const float4 c4 = *reinterpret_cast<const float4 *>(&cs[k][r]);
        acc = __fmaf_rn(c4.x, bt[r], acc);
        acc = __fmaf_rn(c4.y, bt[r + 1], acc);
        acc = __fmaf_rn(c4.z, bt[r + 2], acc);
        acc = __fmaf_rn(c4.w, bt[r + 3], acc);
      }
      vk[k] = acc;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < BATCH; ++k) vec_s[k][lane] = vk[k];
    __syncwarp();
    // leaves of the batch's fibers form one contiguous range; 32 at a time, in parallel
    const int Lb = __ldg(p.fiber_ptr + base), Le = __ldg(p.fiber_ptr + base + nf);
    int fcur = (int)base;
    const int fend = (int)(base + nf);
    for (int L0 = Lb; L0 < Le; L0 += BATCH) {
      const int nb = min(BATCH, Le - L0);
      const int lc = lane < nb ? __ldcs(p.leaf_coord + L0 + lane) : 0;
      const float x = lane < nb ? __ldcs(p.vals + L0 + lane) : 0.f;
      int fnext;
      const int myfib = batch_fibers(p.fiber_ptr, fcur, fend, L0, nb, lane, &fnext);
      const int slot = myfib - (int)base;
      float a[BATCH];
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        const int i = __shfl_sync(FULL, lc, k);
        a[k] = (jl && k < nb) ? p.A[(int64_t)i * p.J + lane] : 0.f;
      }
#pragma unroll
      for (int k = 0; k < BATCH; ++k) {
        if (k < nb) {
          const int sl = __shfl_sync(FULL, slot, k);
          const float vj = vec_s[sl][lane];
          const float s = warp_sum(a[k] * vj);
          const float e = __shfl_sync(FULL, x, k) - s;
          const float g = p.reg * a[k] - e * vj;
          const int i = __shfl_sync(FULL, lc, k);
          // lock-free: the step is computed from a possibly stale row (hogwild) but is never
          // lost -- concurrent writers of one row accumulate through L2 atomics (RED.ADD)
          if (jl) atomicAdd(p.A + (int64_t)i * p.J + lane, -p.lr * g);
        }
      }
      fcur = fnext;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// K5: fixed-order reduction of the per-block partials + apply_core_update + guard
// ------------------------------------------------------------------------------------------
__global__ void core_apply_kernel(int RJ, float *Bt, const float *__restrict__ partials,
                                  int nparts, int negated, double omega, float lr, float reg,
                                  float *acc_out, uint32_t *guard, int apply) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t bits = 0;
  if (k < RJ) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += (double)partials[(int64_t)b * RJ + k];
    const float acc = (float)(negated ? -s : s);
    if (acc_out) acc_out[k] = acc;
    if (apply) {
      const float b = Bt[k];
      const float nb = b - lr * ((float)((double)acc / omega) + reg * b);
      Bt[k] = nb;
      bits = abs_bits(nb);
    }
  }
  if (apply && guard) guard_max(guard, bits);
}

// Persistent grid: as many blocks as can be co-resident (occupancy API), capped by the work.
template <class Kern>
inline int grid_for(Kern kern, int64_t work_warps, int wpb = WPB, size_t smem = 0) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wpb * 32, smem) !=
          cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = (work_warps + wpb - 1) / wpb;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <int RP>
int launch_factor_rows(const SweepParams &p, cudaStream_t s) {
  const size_t sm = factor_smem<RP>();
  const int g = grid_for(factor_rows_kernel<RP>, p.nrows, WPB_R, sm);
  factor_rows_kernel<RP><<<g, WPB_R * 32, sm, s>>>(p);
  return check_launch("ft_factor_sweep_rows");
}

template <int RP>
int core_rows_grid(const SweepParams &p) {
  return grid_for(core_rows_kernel<RP>, p.nrows, WPB_R, core_smem<RP>());
}

template <int RP>
int launch_core_rows(const SweepParams &p, int g, cudaStream_t s) {
  core_rows_kernel<RP><<<g, WPB_R * 32, core_smem<RP>(), s>>>(p);
  return check_launch("ft_core_sweep_rows");
}

int fill_rows_params(SweepParams &p, const ft_tree_t *tree, const ft_model_t *m) {
  if (!tree || !m) return fail(FT_ERR_ARG, "null tree/model");
  const int N = tree->order;
  if (N < 3 || N > FT_MAX_ORDER || m->order != N)
    return fail(FT_ERR_ARG, "order mismatch (tree %d, model %d)", N, m->order);
  const int u = tree->root_mode;
  if (u < 0 || u >= N) return fail(FT_ERR_ARG, "root_mode out of range");
  p.N = N;
  p.npre = N - 2;
  p.nrows = tree->num_rows;
  p.leaf_coord = tree->leaf_coord;
  p.vals = tree->vals;
  p.fiber_ptr = tree->fiber_ptr;
  p.fiber_coord = tree->fiber_coord;
  p.row_fiber_ptr = tree->row_fiber_ptr;
  p.row_coord = tree->row_coord;
  p.A = m->factors[u];
  p.Bt = m->cores_t[u];
  p.Cu = m->dots[u];
  for (int d = 1; d <= N - 2; ++d) p.Cpre[d - 1] = m->dots[(u + d) % N];
  p.Cleaf = m->dots[(u + N - 1) % N];
  p.J = m->ranks[u];
  p.R = m->core_rank;
  if (p.J < 1 || p.J > FT_MAX_RANK || p.R < 1 || p.R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ranks J=%d R=%d outside kernel cover (<= %d)", p.J, p.R,
                FT_MAX_RANK);
  for (int d = 0; d < N; ++d)
    if (d != u && !m->dots[d]) return fail(FT_ERR_ARG, "dots[%d] is null", d);
  if (!p.A || !p.Bt) return fail(FT_ERR_ARG, "null factor/core");
  return FT_OK;
}

}  // namespace
}  // namespace ft

using namespace ft;

extern "C" int ft_factor_sweep_rows(const ft_tree_t *tree, const ft_model_t *model, float lr,
                                    float reg, void *stream) {
  SweepParams p{};
  if (int rc = fill_rows_params(p, tree, model)) return rc;
  p.lr = lr;
  p.reg = reg;
  if (p.nrows == 0) return FT_OK;
  cudaStream_t s = as_stream(stream);
  if (p.R <= 8) return launch_factor_rows<8>(p, s);
  if (p.R <= 16) return launch_factor_rows<16>(p, s);
  return launch_factor_rows<32>(p, s);
}

extern "C" int64_t ft_core_partials_size(int32_t R, int32_t J) {
  return (int64_t)ft::sm_count() * 32 * R * J;  // >= any co-resident grid of core_rows_kernel
}

extern "C" int ft_core_sweep_rows(const ft_tree_t *tree, const ft_model_t *model,
                                  float *partials, int64_t partials_cap, int32_t *nblocks_out,
                                  void *stream) {
  SweepParams p{};
  if (int rc = fill_rows_params(p, tree, model)) return rc;
  if (!p.Cu) return fail(FT_ERR_ARG, "core sweep needs dots[u] (coherent cache)");
  if (!partials || !nblocks_out) return fail(FT_ERR_ARG, "null partials");
  p.partials = partials;
  const int g = p.R <= 8 ? core_rows_grid<8>(p) : p.R <= 16 ? core_rows_grid<16>(p)
                                                            : core_rows_grid<32>(p);
  if ((int64_t)g * p.R * p.J > partials_cap)
    return fail(FT_ERR_ARG, "partials buffer too small (%lld < %lld)", (long long)partials_cap,
                (long long)g * p.R * p.J);
  cudaStream_t s = as_stream(stream);
  *nblocks_out = g;
  if (p.R <= 8) return launch_core_rows<8>(p, g, s);
  if (p.R <= 16) return launch_core_rows<16>(p, g, s);
  return launch_core_rows<32>(p, g, s);
}

extern "C" int ft_factor_sweep_fibers(const ft_tree_t *tree, const ft_model_t *m, int64_t fib_lo,
                                      int64_t fib_hi, float lr, float reg, int32_t max_warps,
                                      void *stream) {
  if (!tree || !m) return fail(FT_ERR_ARG, "null tree/model");
  const int N = tree->order;
  if (N < 3 || N > FT_MAX_ORDER || m->order != N) return fail(FT_ERR_ARG, "order mismatch");
  const int t = tree->root_mode, u = (t + N - 1) % N;
  FiberParams p{};
  p.N = N;
  p.fib_lo = fib_lo;
  p.fib_hi = fib_hi;
  p.leaf_coord = tree->leaf_coord;
  p.vals = tree->vals;
  p.fiber_ptr = tree->fiber_ptr;
  p.fiber_coord = tree->fiber_coord;
  p.A = m->factors[u];
  p.Bt = m->cores_t[u];
  for (int d = 0; d < N - 1; ++d) p.Cpre[d] = m->dots[(t + d) % N];
  p.J = m->ranks[u];
  p.R = m->core_rank;
  p.lr = lr;
  p.reg = reg;
  if (p.J < 1 || p.J > FT_MAX_RANK || p.R < 1 || p.R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ranks outside kernel cover");
  if (fib_lo < 0 || fib_hi > tree->num_fibers || fib_lo > fib_hi)
    return fail(FT_ERR_ARG, "fiber range [%lld, %lld) invalid", (long long)fib_lo,
                (long long)fib_hi);
  if (fib_hi == fib_lo) return FT_OK;
  int64_t work = (fib_hi - fib_lo + BATCH - 1) / BATCH;
  if (max_warps > 0 && work > max_warps) work = max_warps;
  const int wpb = work < WPB ? (int)work : WPB;
  cudaStream_t s = as_stream(stream);
  if (p.R <= 8)
    factor_fibers_kernel<8><<<grid_for(factor_fibers_kernel<8>, work), wpb * 32, 0, s>>>(p);
  else if (p.R <= 16)
    factor_fibers_kernel<16><<<grid_for(factor_fibers_kernel<16>, work), wpb * 32, 0, s>>>(p);
  else
    factor_fibers_kernel<32><<<grid_for(factor_fibers_kernel<32>, work), wpb * 32, 0, s>>>(p);
  return check_launch("ft_factor_sweep_fibers");
}

extern "C" int ft_core_apply(int32_t R, int32_t J, float *Bt, const float *partials,
                             int32_t nparts, int32_t acc_is_negated, double omega, float lr,
                             float reg, float *acc_out, uint32_t *guard, void *stream) {
  if (R < 1 || J < 1 || R * J > 4096 || !Bt || !partials || nparts < 1 || !(omega > 0))
    return fail(FT_ERR_ARG, "ft_core_apply: bad arguments");
  const int RJ = R * J;
  core_apply_kernel<<<(RJ + 255) / 256, 256, 0, as_stream(stream)>>>(
      RJ, Bt, partials, nparts, acc_is_negated, omega, lr, reg, acc_out, guard, 1);
  return check_launch("ft_core_apply");
}

extern "C" int ft_core_reduce(int32_t R, int32_t J, const float *partials, int32_t nparts,
                              float *out, void *stream) {
  if (R < 1 || J < 1 || !partials || !out || nparts < 1)
    return fail(FT_ERR_ARG, "ft_core_reduce: bad arguments");
  const int RJ = R * J;
  core_apply_kernel<<<(RJ + 255) / 256, 256, 0, as_stream(stream)>>>(
      RJ, nullptr, partials, nparts, 0, 1.0, 0.f, 0.f, out, nullptr, 0);
  return check_launch("ft_core_reduce");
}
