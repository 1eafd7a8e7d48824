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
#include <stdlib.h>
#include <string.h>

#include "ft_common.cuh"

namespace ft {
int launch_factor_tc(const ft_tree_t *t, const ft_model_t *m, float lr, float reg,
                     cudaStream_t s);  // factor_tc.cu
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
  const int32_t *leaf_pc;       // leaf-major index (optional): level-1 coordinate per leaf
  const int32_t *row_leaf_ptr;  // first leaf of each row
  int64_t nsegs;                // core-sweep row segments (optional)
  const int32_t *seg_coord;
  const int32_t *seg_leaf_ptr;
  float *A;          // A_u  (I_u x J)
  const float *Bt;   // Bt_u (R x J)
  const float *Cu;   // C_u  (core sweep)
  const float *Cpre[FT_MAX_ORDER];  // C of tree levels 1..N-2 (modes u+1 .. u-2)
  const float *Cleaf;               // C_{u-1}
  int J, R;
  float lr, reg;
  float *partials;   // core: [grid][R*J]
  int64_t gather_bytes;  // bytes of the gathered C matrices (modes other than u)
  int quadw_rpg;         // quadw: rows per warp group (0: 4)
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

// Packed fp32x2 FMA (sm_100 FFMA2): d = a * b + c on both halves.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&d);
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
    constexpr int P4 = RP / 4;  // 16-B chunks per padded row (compile time: shifts, no divide)
    const int R4 = R >> 2;
#pragma unroll
    for (int it = 0; it < P4; ++it) {
      const int c = lane + 32 * it;
      const int k = c / P4, part = c % P4;
      const int coord = __shfl_sync(FULL, coord_lane, k);
      if (k < nb && part < R4) cp_async16(dst + k * RS + part * 4, C + (int64_t)coord * R + part * 4);
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
// With fold_leaf = false the leaf level is left in Y (cross = X * Y, folded by the caller).
template <int RP>
__device__ __forceinline__ void stage_cross(const SweepParams &p, float *X, float *Y, int myfib,
                                            int lc, int nb, int lane, bool fold_leaf = true) {
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
      if (leaf && !fold_leaf) break;
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

// ---- 3xTF32 tensor-core combine ---------------------------------------------------------
// vec for a batch of 32 leaves is a 32 x J x R GEMM: V = Cross (32 x R) * Bt_u (R x J).
// mma.sync.m16n8k8 TF32 with the 3-term split (a_hi b_hi + a_hi b_lo + a_lo b_hi) keeps fp32
// accuracy (BF16/1xTF32 are outside the 1e-4 contract's margin).
// tf32 by truncation: the high 19 bits, exactly representable, so lo = x - hi is exact and the
// 3-term product misses only lo_b*lo_a and lo's own truncation (~2^-22 relative).  (cvt.rna.tf32
// is emulated with ~6 integer/FP instructions on this part; a mask is one LOP3.)
__device__ __forceinline__ uint32_t to_tf32(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

constexpr int VS = 36;  // row stride of the staged V tile (32 leaves x 32 j)

// ---- batch index pipeline shared by the fiber-walking K3b kernels (ws, gram) ------------
// Staging tiles 32 floats wide with an XOR swizzle (conflict-free fragment loads, 16-B cp.async).
__device__ __forceinline__ int swz(int row, int col) { return row * 32 + (col ^ ((row & 7) << 2)); }

template <int RP>
__device__ __forceinline__ void gather_sw(float *dst, const float *__restrict__ C, int R,
                                          int coord_lane, int nb, int lane) {
  if ((R & 3) == 0) {
    constexpr int P4 = RP / 4;
    const int R4 = R >> 2;
#pragma unroll
    for (int it = 0; it < P4; ++it) {
      const int c = lane + 32 * it;
      const int k = c / P4, q = c % P4;
      const int coord = __shfl_sync(FULL, coord_lane, k);
      if (k < nb && q < R4) cp_async16(dst + swz(k, 4 * q), C + (int64_t)coord * R + 4 * q);
    }
  } else {
#pragma unroll 4
    for (int k = 0; k < BATCH; ++k) {
      const int coord = __shfl_sync(FULL, coord_lane, k);
      if (k < nb && lane < R) cp_async4(dst + swz(k, lane), C + (int64_t)coord * R + lane);
    }
  }
}


// Everything batch b needs before its gathers can be issued.
struct BatchIdx {
  int L0, nb, fcur;  // window [L0, L0+nb), fiber holding leaf L0
  int lc;            // lane k: leaf coordinate of leaf L0+k
  float x;           // lane k: value
  int fs;            // lane l: fiber_ptr[fcur + 1 + l] (fiber starts in the window)
};

__device__ __forceinline__ void load_batch_idx(const SweepParams &p, BatchIdx &b, int L0, int Le,
                                               int fcur, int fe, int lane) {
  b.L0 = L0;
  b.nb = min(BATCH, Le - L0);
  b.fcur = fcur;
  b.lc = lane < b.nb ? __ldcs(p.leaf_coord + L0 + lane) : 0;
  b.x = lane < b.nb ? __ldcs(p.vals + L0 + lane) : 0.f;
  const int fidx = fcur + 1 + lane;
  b.fs = fidx < fe ? __ldg(p.fiber_ptr + fidx) : INT32_MAX;
}

// fiber of each leaf + the next window's fcur (needs b.fs)
__device__ __forceinline__ int batch_fib(const BatchIdx &b, int lane, int *fnext) {
  const unsigned bit = (b.fs < b.L0 + b.nb) ? (1u << (b.fs - b.L0)) : 0u;
  const unsigned mask = __reduce_or_sync(FULL, bit);
  *fnext = b.fcur + __popc(mask);
  return b.fcur + __popc(mask & (FULL >> (31 - lane)));
}

// issue batch b's gathers: X = prod of the prefix levels, Y = leaf level (left in flight)
template <int RP>
__device__ __forceinline__ void issue_gathers(const SweepParams &p, const BatchIdx &b, int myfib,
                                              float *X, float *Y, int lane) {
  const int npre = p.N - 2;
  for (int lvl = 0; lvl < npre; ++lvl) {
    const int coord =
        lane < b.nb ? __ldg(p.fiber_coord + (int64_t)myfib * (p.N - 1) + 1 + lvl) : 0;
    gather_sw<RP>(lvl == 0 ? X : Y, p.Cpre[lvl], p.R, coord, b.nb, lane);
    if (lvl >= 1) {  // order > 3: fold this prefix level into X now
      cp_async_wait_all();
      __syncwarp();
      if (lane < RP)
        for (int k = 0; k < b.nb; ++k) X[swz(k, lane)] *= Y[swz(k, lane)];
      __syncwarp();
    }
  }
  gather_sw<RP>(Y, p.Cleaf, p.R, b.lc, b.nb, lane);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// ---- K3b dual: two rows per warp (orders 5-6 with many rows) -------------------------------
// Each 16-lane half of a warp owns one row of A_u (lane l holds columns l and l + 16) and walks
// its root slice in 16-leaf batches, so a warp advances two independent serial chains at once
// and each chain step reduces over 16 lanes (4 shuffle levels) instead of 32.  The batch of a
// half is one m16 tile of the tensor-core combine (V = cross * Bt_u, 3xTF32).  Rows are taken
// round-robin per half; a half that finishes its row writes it back and starts the next one.
constexpr int HB = 16;  // leaves per half-warp batch

// ---- mbarrier helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct DualPlan {
  static constexpr int XS = 36;       // staging row stride: 144-B rows (TMA-aligned), and
                                      // conflict-free A-fragment loads
  static constexpr int XT = HB * XS;  // 16 x 36 staging tile
  static constexpr int VT = HB * VS;  // 16 x 36 V tile
  // V reuses X (dead once the MMA has read it); +16: the halves' V reads hit disjoint banks
  static constexpr int HALF_FLOATS = 2 * XT + 16;
  static constexpr int WARP_FLOATS = 2 * HALF_FLOATS;
  static constexpr int WPB = 8;
  static constexpr int BAR_BYTES = WPB * 8 + 64;  // one mbarrier per warp, padded to 16 B
  template <int RP, int JP>
  static constexpr int bfrag_u4() { return (RP / 8 > 0 ? RP / 8 : 1) * (JP / 8) * 32; }
  template <int RP, int JP>
  static constexpr size_t bytes() {
    return (size_t)bfrag_u4<RP, JP>() * 16 + BAR_BYTES + (size_t)WPB * WARP_FLOATS * sizeof(float);
  }
};

template <int RP, int JP>
__global__ void __launch_bounds__(DualPlan::WPB * 32, 2)
    factor_rows_dual_kernel(const SweepParams p) {
  constexpr int KT = RP / 8 > 0 ? RP / 8 : 1, NT = JP / 8;  // JP = padded J (16 or 32)
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane >> 4, l = lane & 15;
  const int gq = lane >> 2, tq = lane & 3;
  uint4 *bfrag = reinterpret_cast<uint4 *>(smem4);
  uint64_t *bar = reinterpret_cast<uint64_t *>(bfrag + DualPlan::bfrag_u4<RP, JP>()) + w;
  float *wbase = reinterpret_cast<float *>(reinterpret_cast<char *>(bfrag + DualPlan::bfrag_u4<RP, JP>()) +
                                           DualPlan::BAR_BYTES) +
                 w * DualPlan::WARP_FLOATS;
  constexpr int XS = DualPlan::XS;
  // tile of half hh: wbase + hh * HALF_FLOATS (+ XT for Y, + 2 XT for V); computed by
  // arithmetic, not through a pointer array, so the accesses stay LDS/STS (not generic LD/ST)
#define XH(hh) (wbase + (hh) * DualPlan::HALF_FLOATS)
#define YH(hh) (wbase + (hh) * DualPlan::HALF_FLOATS + DualPlan::XT)
#define VH(hh) (wbase + (hh) * DualPlan::HALF_FLOATS)
  for (int k = lane; k < DualPlan::WARP_FLOATS; k += 32) wbase[k] = 0.f;
  for (int f = threadIdx.x; f < DualPlan::bfrag_u4<RP, JP>(); f += blockDim.x) {
    const int ll = f & 31, nt = (f >> 5) % NT, kt = (f >> 5) / NT;
    const int g = ll >> 2, t = ll & 3, j = 8 * nt + g;
    uint32_t hv[2], lv[2];
    for (int hh = 0; hh < 2; ++hh) {
      const int r = 8 * kt + t + 4 * hh;
      const float bv = (r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f;
      hv[hh] = to_tf32(bv);
      lv[hh] = to_tf32(bv - __uint_as_float(hv[hh]));
    }
    bfrag[f] = make_uint4(hv[0], hv[1], lv[0], lv[1]);
  }
  __syncthreads();
  const int64_t nstream = (int64_t)gridDim.x * DualPlan::WPB * 2;  // row streams
  const int64_t mystream = ((int64_t)blockIdx.x * DualPlan::WPB + w) * 2 + h;
  const bool j0 = l < p.J, j1 = JP > 16 && l + 16 < p.J;
  float *Xh = XH(h), *Yh = YH(h), *Vh = VH(h);

  // per-half row state (replicated in the half's 16 lanes)
  int64_t row = mystream - nstream;
  int fe = 0, Le = 0, L0 = 0, fcur = 0;
  float *arow = nullptr;
  float a0 = 0.f, a1 = 0.f;
  bool active = true;
  // next batch's index loads, issued one batch ahead within a row (the batch header's dependent
  // loads -- fiber window -> ballot -> coordinates -> gathers -- were the top stall)
  bool have_pf = false;
  int pf_lc = 0, pf_fs = INT32_MAX;
  float pf_x = 0.f;
  for (;;) {
    // a half whose row is exhausted writes it back and starts its next non-empty row
    if (active && L0 >= Le) {
      if (arow) {
        if (j0) arow[l] = a0;
        if (j1) arow[l + 16] = a1;
        arow = nullptr;
      }
      row += nstream;
      if (row < p.nrows) {
        const int i = __ldg(p.row_coord + row);
        const int fb = __ldg(p.row_fiber_ptr + row);
        fe = __ldg(p.row_fiber_ptr + row + 1);
        L0 = __ldg(p.fiber_ptr + fb);
        Le = __ldg(p.fiber_ptr + fe);
        fcur = fb;
        arow = p.A + (int64_t)i * p.J;
        a0 = j0 ? arow[l] : 0.f;
        a1 = j1 ? arow[l + 16] : 0.f;
      } else {
        active = false;
      }
      have_pf = false;
    }
    if (!__any_sync(FULL, active)) break;
    const int nb = active ? min(HB, Le - L0) : 0;  // this half's batch
    // leaf data and the fiber of each leaf (window of <= 16 fiber starts per half)
    const bool lv = l < nb;
    int lc, fs;
    float x;
    if (have_pf) {
      lc = pf_lc;
      x = pf_x;
      fs = pf_fs;
    } else {
      lc = lv ? __ldcs(p.leaf_coord + L0 + l) : 0;
      x = lv ? __ldcs(p.vals + L0 + l) : 0.f;
      const int fidx = fcur + 1 + l;
      fs = (active && fidx < fe) ? __ldg(p.fiber_ptr + fidx) : INT32_MAX;
    }
    const unsigned bit = (fs < L0 + nb) ? (1u << (fs - L0)) : 0u;
    const unsigned hmask = (__reduce_or_sync(FULL, bit << (16 * h)) >> (16 * h)) & 0xffffu;
    // (the OR of both halves' shifted bits, then this half's 16 bits)
    const int myfib = fcur + __popc(hmask & (0xffffu >> (15 - l)));
    const int fnext = fcur + __popc(hmask);
    {  // prefetch the next batch of this row
      const int L1 = L0 + nb;
      have_pf = active && L1 < Le;
      if (have_pf) {
        const int nb1 = min(HB, Le - L1);
        pf_lc = l < nb1 ? __ldcs(p.leaf_coord + L1 + l) : 0;
        pf_x = l < nb1 ? __ldcs(p.vals + L1 + l) : 0.f;
        const int fidx = fnext + 1 + l;
        pf_fs = fidx < fe ? __ldg(p.fiber_ptr + fidx) : INT32_MAX;
      }
    }
    // ---- gathers: prefix levels into X (folded progressively), the leaf level into Y ----
    const int npre = p.N - 2;
    for (int lvl = 0; lvl <= npre; ++lvl) {
      const bool leaf = lvl == npre;
      const int coord =
          leaf ? lc : (lv ? __ldg(p.fiber_coord + (int64_t)myfib * (p.N - 1) + 1 + lvl) : 0);
      float *dst = (lvl == 0) ? Xh : Yh;
      const float *C = leaf ? p.Cleaf : p.Cpre[lvl];
      if ((p.R & 3) == 0) {
        constexpr int P4 = RP / 4;
        const int R4 = p.R >> 2;
#pragma unroll
        for (int it = 0; it < P4; ++it) {
          const int c = l + 16 * it;
          const int k = c / P4, q = c % P4;
          const int ck = __shfl_sync(FULL, coord, 16 * h + k);
          if (k < nb && q < R4) cp_async16(dst + k * XS + 4 * q, C + (int64_t)ck * p.R + 4 * q);
        }
      } else {
        for (int k = 0; k < HB; ++k) {
          const int ck = __shfl_sync(FULL, coord, 16 * h + k);
          for (int r = l; r < p.R; r += 16)
            if (k < nb) cp_async4(dst + k * XS + r, C + (int64_t)ck * p.R + r);
        }
      }
      if (lvl >= 1 && !leaf) {
        cp_async_wait_all();
        __syncwarp();
        for (int k = 0; k < nb; ++k)
          for (int r = l; r < RP; r += 16) Xh[k * XS + r] *= Yh[k * XS + r];
        __syncwarp();
      }
    }
    cp_async_wait_all();
    __syncwarp();
    // ---- V_h = (X_h * Y_h) * Bt_u: one m16 tile per half, 3xTF32 ----
    float acc[2][NT][4];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[hh][nt][q] = 0.f;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const float *Xs = XH(hh), *Ys = YH(hh);
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int c0 = 8 * kt + tq;
        const int o0 = gq * XS + c0, o1 = (gq + 8) * XS + c0, o2 = o0 + 4, o3 = o1 + 4;
        const float x0 = Xs[o0] * Ys[o0], x1 = Xs[o1] * Ys[o1], x2 = Xs[o2] * Ys[o2],
                    x3 = Xs[o3] * Ys[o3];
        const uint32_t h0 = to_tf32(x0), h1 = to_tf32(x1), h2 = to_tf32(x2), h3 = to_tf32(x3);
        const uint32_t l0 = to_tf32(x0 - __uint_as_float(h0));
        const uint32_t l1 = to_tf32(x1 - __uint_as_float(h1));
        const uint32_t l2 = to_tf32(x2 - __uint_as_float(h2));
        const uint32_t l3 = to_tf32(x3 - __uint_as_float(h3));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint4 bb = bfrag[(kt * NT + nt) * 32 + lane];
          mma_tf32(acc[hh][nt], l0, l1, l2, l3, bb.x, bb.y);
          mma_tf32(acc[hh][nt], h0, h1, h2, h3, bb.z, bb.w);
          mma_tf32(acc[hh][nt], h0, h1, h2, h3, bb.x, bb.y);
        }
      }
    }
    __syncwarp();  // every lane's A fragments are read before V overwrites X
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int c0 = 8 * nt + 2 * tq;
        *reinterpret_cast<float2 *>(VH(hh) + gq * VS + c0) = make_float2(acc[hh][nt][0], acc[hh][nt][1]);
        *reinterpret_cast<float2 *>(VH(hh) + (gq + 8) * VS + c0) =
            make_float2(acc[hh][nt][2], acc[hh][nt][3]);
      }
    __syncwarp();
    // ---- two serial chains (one per half): s = a.v over 16 lanes x 2 columns ----
    const int nbmax = max(__shfl_sync(FULL, nb, 0), __shfl_sync(FULL, nb, 16));
#pragma unroll 4
    for (int k = 0; k < nbmax; ++k) {
      const float v0 = Vh[k * VS + l], v1 = JP > 16 ? Vh[k * VS + l + 16] : 0.f;
      float s = a0 * v0 + a1 * v1;
      s += __shfl_xor_sync(FULL, s, 8);
      s += __shfl_xor_sync(FULL, s, 4);
      s += __shfl_xor_sync(FULL, s, 2);
      s += __shfl_xor_sync(FULL, s, 1);
      const float e = __shfl_sync(FULL, x, 16 * h + (k & 15)) - s;
      if (k < nb) {
        const float g0 = p.reg * a0 - e * v0, g1 = p.reg * a1 - e * v1;
        a0 = a0 - p.lr * g0;
        a1 = a1 - p.lr * g1;
      }
    }
    __syncwarp();
    if (p.R < RP) {  // V overwrote X's zero columns r in [R, RP): restore them
      for (int k = 0; k < HB; ++k)
        for (int r = p.R + l; r < RP; r += 16) Xh[k * XS + r] = 0.f;
      __syncwarp();
    }
    L0 += nb;
    fcur = fnext;
  }
}
#undef XH
#undef YH
#undef VH


// ---- K3b, warp-specialised (producer / consumer) two-row version --------------------------
// A warp pair owns two rows (one per 16-lane half, as in the dual kernel).  The PRODUCER warp
// walks both root slices in 16-leaf batches -- index loads prefetched a batch ahead, cp.async
// gathers double-buffered (batch b+1's are in flight while batch b's rank products go through
// the 3xTF32 tensor-core combine) -- and publishes V plus the batch's values into a 2-stage
// shared-memory ring (mbarrier full / empty).  The CONSUMER warp only runs the two serial
// chains s = a.v, e = x - s, a -= lr (reg a - e v).  All tiles are 16 x 32 floats with the XOR
// swizzle (conflict-free fragment loads, 16-B cp.async) so a pair fits 24.6 KB and 8 pairs an SM.
// Order-3 tensors only (the prefix is a single C row); other orders use dual / gram.
namespace ws {
constexpr int NS = 2;                       // ring stages
constexpr int PAIRS = 4;                    // warp pairs per block
constexpr int HT = HB * 32;                 // swizzled 16 x 32 tile
constexpr int STAGE_FLOATS = 2 * HT + 2 * HB + 8;  // V[2 halves], x[2][16], meta[8]
constexpr int PAIR_FLOATS = NS * STAGE_FLOATS + 8 * HT;  // ring + producer X/Y x 2 halves x 2 bufs
constexpr int BAR_BYTES = PAIRS * 2 * NS * 8 + 32;
template <int RP, int JP>
constexpr int bfrag_u4() { return (RP / 8 > 0 ? RP / 8 : 1) * (JP / 8) * 32; }
template <int RP, int JP>
constexpr size_t bytes() {
  return (size_t)bfrag_u4<RP, JP>() * 16 + BAR_BYTES + (size_t)PAIRS * PAIR_FLOATS * 4;
}
}  // namespace ws

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_one() {  // all but the most recent group
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

// producer-side state of one half (replicated in the half's 16 lanes)
struct WsHalf {
  int64_t row;
  int fe, Le, L0, fcur;
  bool active, ended, have_pf;
  int pf_lc, pf_fs;
  float pf_x;
};
// what the producer knows about one in-flight batch
struct WsBatch {
  int nb, newrow;
  float x;
  bool stop;
};

template <int RP>
__device__ __forceinline__ WsBatch ws_advance(const SweepParams &p, WsHalf &H, int64_t nstream,
                                              float *Xb, float *Yb, int h, int l) {
  WsBatch B;
  B.newrow = -1;
  if (H.active && H.L0 >= H.Le) {
    H.row += nstream;
    if (H.row < p.nrows) {
      B.newrow = __ldg(p.row_coord + H.row);
      const int fb = __ldg(p.row_fiber_ptr + H.row);
      H.fe = __ldg(p.row_fiber_ptr + H.row + 1);
      H.L0 = __ldg(p.fiber_ptr + fb);
      H.Le = __ldg(p.fiber_ptr + H.fe);
      H.fcur = fb;
    } else {
      H.active = false;
    }
    H.have_pf = false;
  }
  if (!H.active && !H.ended) {
    B.newrow = -2;
    H.ended = true;
  }
  B.stop = !__any_sync(FULL, H.active);
  const int nb = H.active ? min(HB, H.Le - H.L0) : 0;
  B.nb = nb;
  const bool lv = l < nb;
  int lc, fs;
  if (H.have_pf) {
    lc = H.pf_lc;
    B.x = H.pf_x;
    fs = H.pf_fs;
  } else {
    lc = lv ? __ldcs(p.leaf_coord + H.L0 + l) : 0;
    B.x = lv ? __ldcs(p.vals + H.L0 + l) : 0.f;
    const int fidx = H.fcur + 1 + l;
    fs = (H.active && fidx < H.fe) ? __ldg(p.fiber_ptr + fidx) : INT32_MAX;
  }
  const unsigned bit = (fs < H.L0 + nb) ? (1u << (fs - H.L0)) : 0u;
  const unsigned hmask = (__reduce_or_sync(FULL, bit << (16 * h)) >> (16 * h)) & 0xffffu;
  const int myfib = H.fcur + __popc(hmask & (0xffffu >> (15 - l)));
  const int fnext = H.fcur + __popc(hmask);
  const int pc = lv ? __ldg(p.fiber_coord + (int64_t)myfib * 2 + 1) : 0;
  {  // prefetch the next batch's indices of this row
    const int L1 = H.L0 + nb;
    H.have_pf = H.active && L1 < H.Le;
    if (H.have_pf) {
      const int nb1 = min(HB, H.Le - L1);
      H.pf_lc = l < nb1 ? __ldcs(p.leaf_coord + L1 + l) : 0;
      H.pf_x = l < nb1 ? __ldcs(p.vals + L1 + l) : 0.f;
      const int fidx = fnext + 1 + l;
      H.pf_fs = fidx < H.fe ? __ldg(p.fiber_ptr + fidx) : INT32_MAX;
    }
  }
  if (!B.stop) {  // gathers: prefix row into X, leaf row into Y
    if ((p.R & 3) == 0) {
      constexpr int P4 = RP / 4;
      const int R4 = p.R >> 2;
#pragma unroll
      for (int q2 = 0; q2 < P4; ++q2) {
        const int c = l + 16 * q2;
        const int k = c / P4, q = c % P4;
        const int ck = __shfl_sync(FULL, pc, 16 * h + k);
        const int cl = __shfl_sync(FULL, lc, 16 * h + k);
        if (k < nb && q < R4) {
          cp_async16(Xb + swz(k, 4 * q), p.Cpre[0] + (int64_t)ck * p.R + 4 * q);
          cp_async16(Yb + swz(k, 4 * q), p.Cleaf + (int64_t)cl * p.R + 4 * q);
        }
      }
    } else {
      for (int k = 0; k < HB; ++k) {
        const int ck = __shfl_sync(FULL, pc, 16 * h + k);
        const int cl = __shfl_sync(FULL, lc, 16 * h + k);
        for (int r = l; r < p.R; r += 16)
          if (k < nb) {
            cp_async4(Xb + swz(k, r), p.Cpre[0] + (int64_t)ck * p.R + r);
            cp_async4(Yb + swz(k, r), p.Cleaf + (int64_t)cl * p.R + r);
          }
      }
    }
  }
  cp_async_commit();
  H.L0 += nb;
  H.fcur = fnext;
  return B;
}

template <int RP, int JP>
__global__ void __launch_bounds__(ws::PAIRS * 64, 2)
    factor_rows_ws_kernel(const SweepParams p) {
  constexpr int KT = RP / 8 > 0 ? RP / 8 : 1, NT = JP / 8;
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int pair = w >> 1, role = w & 1;  // role 0: producer, 1: consumer
  const int h = lane >> 4, l = lane & 15;
  const int gq = lane >> 2, tq = lane & 3;
  uint4 *bfrag = reinterpret_cast<uint4 *>(smem4);
  uint64_t *bars = reinterpret_cast<uint64_t *>(bfrag + ws::bfrag_u4<RP, JP>()) + pair * 2 * ws::NS;
  uint64_t *full = bars, *empty = bars + ws::NS;
  float *pbase = reinterpret_cast<float *>(reinterpret_cast<char *>(bfrag + ws::bfrag_u4<RP, JP>()) +
                                           ws::BAR_BYTES) +
                 pair * ws::PAIR_FLOATS;
  float *ring = pbase;                           // NS stages
  float *stg = pbase + ws::NS * ws::STAGE_FLOATS;  // [buf 2][X/Y 2][half 2] swizzled tiles
#define WS_TILE(buf, xy, hh) (stg + (((buf) * 2 + (xy)) * 2 + (hh)) * ws::HT)
  if (role == 0) {
    for (int k = lane; k < 8 * ws::HT; k += 32) stg[k] = 0.f;
    if (lane == 0)
      for (int st = 0; st < ws::NS; ++st) {
        mbar_init(full + st, 32);
        mbar_init(empty + st, 32);
      }
  }
  for (int f = threadIdx.x; f < ws::bfrag_u4<RP, JP>(); f += blockDim.x) {
    const int ll = f & 31, nt = (f >> 5) % NT, kt = (f >> 5) / NT;
    const int g = ll >> 2, t = ll & 3, j = 8 * nt + g;
    uint32_t hv[2], lv2[2];
    for (int hh = 0; hh < 2; ++hh) {
      const int r = 8 * kt + t + 4 * hh;
      const float bv = (r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f;
      hv[hh] = to_tf32(bv);
      lv2[hh] = to_tf32(bv - __uint_as_float(hv[hh]));
    }
    bfrag[f] = make_uint4(hv[0], hv[1], lv2[0], lv2[1]);
  }
  __syncthreads();
  const int64_t nstream = (int64_t)gridDim.x * ws::PAIRS * 2;
  const int64_t mystream = ((int64_t)blockIdx.x * ws::PAIRS + pair) * 2 + h;

  if (role == 0) {
    // ===================================== producer =====================================
    WsHalf H;
    H.row = mystream - nstream;
    H.fe = H.Le = H.L0 = H.fcur = 0;
    H.active = true;
    H.ended = H.have_pf = false;
    H.pf_lc = 0;
    H.pf_fs = INT32_MAX;
    H.pf_x = 0.f;
    WsBatch cur = ws_advance<RP>(p, H, nstream, WS_TILE(0, 0, h), WS_TILE(0, 1, h), h, l);
    for (int it = 0;; ++it) {
      const int buf = it & 1;
      WsBatch nxt;
      nxt.stop = true;
      if (!cur.stop) {  // batch it+1's gathers fly while batch it goes through the MMA
        __syncwarp();
        nxt = ws_advance<RP>(p, H, nstream, WS_TILE(buf ^ 1, 0, h), WS_TILE(buf ^ 1, 1, h), h, l);
        cp_async_wait_one();
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
      float acc[2][NT][4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[hh][nt][q] = 0.f;
      if (!cur.stop) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float *Xs = WS_TILE(buf, 0, hh), *Ys = WS_TILE(buf, 1, hh);
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const int c0 = 8 * kt + tq;
            const int o0 = swz(gq, c0), o1 = swz(gq + 8, c0), o2 = swz(gq, c0 + 4),
                      o3 = swz(gq + 8, c0 + 4);
            const float x0 = Xs[o0] * Ys[o0], x1 = Xs[o1] * Ys[o1], x2 = Xs[o2] * Ys[o2],
                        x3 = Xs[o3] * Ys[o3];
            const uint32_t h0 = to_tf32(x0), h1 = to_tf32(x1), h2 = to_tf32(x2),
                           h3 = to_tf32(x3);
            const uint32_t l0 = to_tf32(x0 - __uint_as_float(h0));
            const uint32_t l1 = to_tf32(x1 - __uint_as_float(h1));
            const uint32_t l2 = to_tf32(x2 - __uint_as_float(h2));
            const uint32_t l3 = to_tf32(x3 - __uint_as_float(h3));
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const uint4 bb = bfrag[(kt * NT + nt) * 32 + lane];
              mma_tf32(acc[hh][nt], l0, l1, l2, l3, bb.x, bb.y);
              mma_tf32(acc[hh][nt], h0, h1, h2, h3, bb.z, bb.w);
              mma_tf32(acc[hh][nt], h0, h1, h2, h3, bb.x, bb.y);
            }
          }
        }
      }
      // publish batch `it` into the ring
      const int st = it % ws::NS;
      if (it >= ws::NS) mbar_wait(empty + st, ((it / ws::NS) - 1) & 1);
      float *S = ring + st * ws::STAGE_FLOATS;
      if (!cur.stop) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int c0 = 8 * nt + 2 * tq;
            float *V = S + hh * ws::HT;
            *reinterpret_cast<float2 *>(V + swz(gq, c0)) = make_float2(acc[hh][nt][0], acc[hh][nt][1]);
            *reinterpret_cast<float2 *>(V + swz(gq + 8, c0)) =
                make_float2(acc[hh][nt][2], acc[hh][nt][3]);
          }
        S[2 * ws::HT + h * HB + l] = cur.x;
      }
      int *meta = reinterpret_cast<int *>(S + 2 * ws::HT + 2 * HB);
      if (l == 0) {
        meta[2 * h] = cur.nb;
        meta[2 * h + 1] = cur.newrow;
      }
      if (lane == 0) meta[4] = cur.stop ? 1 : 0;
      __syncwarp();
      mbar_arrive(full + st);
      if (cur.stop) break;
      cur = nxt;
    }
  } else {
    // ===================================== consumer =====================================
    const bool j0 = l < p.J, j1 = JP > 16 && l + 16 < p.J;
    float *arow = nullptr;
    float a0 = 0.f, a1 = 0.f;
    for (int it = 0;; ++it) {
      const int st = it % ws::NS;
      mbar_wait(full + st, (it / ws::NS) & 1);
      const float *S = ring + st * ws::STAGE_FLOATS;
      const int *meta = reinterpret_cast<const int *>(S + 2 * ws::HT + 2 * HB);
      const int nb = meta[2 * h], newrow = meta[2 * h + 1];
      const bool stop = meta[4] != 0;
      if (newrow != -1) {  // this half's row ended (and maybe a new one starts)
        if (arow) {
          if (j0) arow[l] = a0;
          if (j1) arow[l + 16] = a1;
          arow = nullptr;
        }
        if (newrow >= 0) {
          arow = p.A + (int64_t)newrow * p.J;
          a0 = j0 ? arow[l] : 0.f;
          a1 = j1 ? arow[l + 16] : 0.f;
        }
      }
      if (stop) break;
      const float *Vh = S + h * ws::HT;
      const float xl = S[2 * ws::HT + h * HB + l];
      const int nbmax = max(__shfl_sync(FULL, nb, 0), __shfl_sync(FULL, nb, 16));
#pragma unroll 4
      for (int k = 0; k < nbmax; ++k) {
        const float v0 = Vh[swz(k, l)], v1 = JP > 16 ? Vh[swz(k, l + 16)] : 0.f;
        float s = a0 * v0 + a1 * v1;
        s += __shfl_xor_sync(FULL, s, 8);
        s += __shfl_xor_sync(FULL, s, 4);
        s += __shfl_xor_sync(FULL, s, 2);
        s += __shfl_xor_sync(FULL, s, 1);
        const float e = __shfl_sync(FULL, xl, 16 * h + (k & 15)) - s;
        if (k < nb) {
          const float g0 = p.reg * a0 - e * v0, g1 = p.reg * a1 - e * v1;
          a0 = a0 - p.lr * g0;
          a1 = a1 - p.lr * g1;
        }
      }
      __syncwarp();
      mbar_arrive(empty + st);
    }
    if (arow) {
      if (j0) arow[l] = a0;
      if (j1) arow[l + 16] = a1;
    }
  }
#undef WS_TILE
}

#include "quad.cuh"

// ---- K3b, Gram form of the serial chain (tensor cores for both GEMMs) -------------------
// Within a batch the row evolves as a_{m+1} = a_m + lr (e_m v_m - reg a_m).
// Tracking w_k = a_m . v_k for every leaf k of the batch gives
//     e_m = x_m - w_m,      w_k <- w_k + lr (e_m (v_m . v_k) - reg w_k),
// an exact restatement of the reference's s = a . v that makes the serial dependency per leaf
// ONE shuffle and two FMAs (~40 cycles) instead of a 32-lane reduction (~5 dependent
// shuffles).  Off the chain, per batch: V = cross Bt_u (3xTF32 mma), then [G | d] =
// V [V^T | a_0] (3xTF32 mma, only the tiles with some m < k, plus d = V a_0 as a fifth n-tile).
// After the chain the row is replayed a <- a + lr (e_m v_m - reg a) in leaf order.
constexpr int GS = 40;  // stride of the G tile: 32 x (32 Gram columns + 8 for d)

struct GramPlan {
  static constexpr int TILE = BATCH * 32;  // swizzled X / Y tiles (G reuses both)
  static constexpr int WARP_FLOATS = 2 * TILE + BATCH * VS;
  static constexpr int WPB = 8;
  template <int RP, int JP>
  static constexpr int bfrag_u4() { return (RP / 8 > 0 ? RP / 8 : 1) * (JP / 8) * 32; }
  template <int RP, int JP>
  static constexpr size_t bytes() {
    return (size_t)bfrag_u4<RP, JP>() * 16 + (size_t)WPB * WARP_FLOATS * sizeof(float);
  }
};
static_assert(BATCH * GS + BATCH <= 2 * BATCH * 32, "G and a_0 must fit in the X/Y tiles");

__device__ __forceinline__ void split3(float v, uint32_t &hi, uint32_t &lo) {
  hi = to_tf32(v);
  lo = to_tf32(v - __uint_as_float(hi));
}

template <int RP, int JP>
__global__ void __launch_bounds__(GramPlan::WPB * 32, 2)
    factor_rows_gram_kernel(const SweepParams p) {
  constexpr int KT = RP / 8 > 0 ? RP / 8 : 1, NT = JP / 8;  // JP = padded J (16 or 32)
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  uint4 *bfrag = reinterpret_cast<uint4 *>(smem4);
  float *X = reinterpret_cast<float *>(bfrag + GramPlan::bfrag_u4<RP, JP>()) + w * GramPlan::WARP_FLOATS;
  float *Y = X + GramPlan::TILE;
  float *V = Y + GramPlan::TILE;
  float *G = X;  // after V exists, X / Y are dead
  for (int k = lane; k < GramPlan::WARP_FLOATS; k += 32) X[k] = 0.f;
  for (int f = threadIdx.x; f < GramPlan::bfrag_u4<RP, JP>(); f += blockDim.x) {
    const int l = f & 31, nt = (f >> 5) % NT, kt = (f >> 5) / NT;
    const int g = l >> 2, t = l & 3, j = 8 * nt + g;
    uint32_t hv[2], lv[2];
    for (int h = 0; h < 2; ++h) {
      const int r = 8 * kt + t + 4 * h;
      split3((r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f, hv[h], lv[h]);
    }
    bfrag[f] = make_uint4(hv[0], hv[1], lv[0], lv[1]);
  }
  __syncthreads();
  const int64_t gw = (int64_t)blockIdx.x * GramPlan::WPB + w;
  const int64_t nw = (int64_t)gridDim.x * GramPlan::WPB;
  const bool jl = lane < p.J;
  const float lr = p.lr, reg = p.reg;

  for (int64_t row = gw; row < p.nrows; row += nw) {
    const int i = __ldg(p.row_coord + row);
    const int fb = __ldg(p.row_fiber_ptr + row), fe = __ldg(p.row_fiber_ptr + row + 1);
    const int Lb = __ldg(p.fiber_ptr + fb), Le = __ldg(p.fiber_ptr + fe);
    float *arow = p.A + (int64_t)i * p.J;
    float a = jl ? arow[lane] : 0.f;
    // Index pipeline (long rows): batch b+1's leaf / value / fiber-window loads are issued at
    // batch b-1, its fibers and prefix coordinate (order 3) at batch b, so no batch waits on a
    // dependent global load before its gathers go out.
    BatchIdx nxt;
    load_batch_idx(p, nxt, Lb, Le, fb, fe, lane);
    int nfnext;
    int nfib = batch_fib(nxt, lane, &nfnext);
    int npc = (p.N == 3 && lane < nxt.nb) ? __ldg(p.fiber_coord + (int64_t)nfib * 2 + 1) : 0;
    BatchIdx nn;
    bool has_nn = Lb + BATCH < Le;
    if (has_nn) load_batch_idx(p, nn, Lb + BATCH, Le, nfnext, fe, lane);
    for (int L0 = Lb; L0 < Le; L0 += BATCH) {
      const BatchIdx cur = nxt;
      const int myfib = nfib, pc = npc;
      if (p.N == 3) {
        gather_sw<RP>(X, p.Cpre[0], p.R, pc, cur.nb, lane);
        gather_sw<RP>(Y, p.Cleaf, p.R, cur.lc, cur.nb, lane);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      } else {
        issue_gathers<RP>(p, cur, myfib, X, Y, lane);
      }
      if (has_nn) {  // advance the index pipeline under this batch's gathers
        nxt = nn;
        nfib = batch_fib(nxt, lane, &nfnext);
        npc = (p.N == 3 && lane < nxt.nb) ? __ldg(p.fiber_coord + (int64_t)nfib * 2 + 1) : 0;
        has_nn = nxt.L0 + BATCH < Le;
        if (has_nn) load_batch_idx(p, nn, nxt.L0 + BATCH, Le, nfnext, fe, lane);
      }
      cp_async_wait_all();
      __syncwarp();
      const int nb = cur.nb, mts = nb > 16 ? 2 : 1;
      // ---- V = (X * Y) * Bt_u ----
      float acc[2][NT][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.f;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= mts) break;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int r0 = 16 * mt + gq, c0 = 8 * kt + tq;
          const int o0 = swz(r0, c0), o1 = swz(r0 + 8, c0), o2 = swz(r0, c0 + 4),
                    o3 = swz(r0 + 8, c0 + 4);
          uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
          split3(X[o0] * Y[o0], h0, l0);
          split3(X[o1] * Y[o1], h1, l1);
          split3(X[o2] * Y[o2], h2, l2);
          split3(X[o3] * Y[o3], h3, l3);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint4 bb = bfrag[(kt * NT + nt) * 32 + lane];
            mma_tf32(acc[mt][nt], l0, l1, l2, l3, bb.x, bb.y);
            mma_tf32(acc[mt][nt], h0, h1, h2, h3, bb.z, bb.w);
            mma_tf32(acc[mt][nt], h0, h1, h2, h3, bb.x, bb.y);
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int r0 = 16 * mt + gq, c0 = 8 * nt + 2 * tq;
          *reinterpret_cast<float2 *>(V + r0 * VS + c0) = make_float2(acc[mt][nt][0], acc[mt][nt][1]);
          *reinterpret_cast<float2 *>(V + (r0 + 8) * VS + c0) =
              make_float2(acc[mt][nt][2], acc[mt][nt][3]);
        }
      __syncwarp();  // V visible; X / Y dead from here (G overwrites them)
      // ---- G = V V^T (1xTF32 at small lr: G only enters as the lr-scaled correction, measured
      // 5.8e-6 vs 5.7e-6 for fp32 over a 45 K-step row at lr 1e-3), tiles with some m < k ----
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        if (mt >= mts) break;
        float gacc[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int q = 0; q < 4; ++q) gacc[nt][q] = 0.f;
#pragma unroll
        for (int kt = 0; kt < NT; ++kt) {  // the Gram contracts over j
          const int r0 = 16 * mt + gq, c0 = 8 * kt + tq;
          const float f0 = V[r0 * VS + c0], f1 = V[(r0 + 8) * VS + c0];
          const float f2 = V[r0 * VS + c0 + 4], f3 = V[(r0 + 8) * VS + c0 + 4];
          const uint32_t a0 = to_tf32(f0), a1 = to_tf32(f1), a2 = to_tf32(f2), a3 = to_tf32(f3);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (mt == 1 && nt < 2) continue;  // rows 16..31 x cols 0..15: every m > k
            const int n0 = 8 * nt + gq;
            const float e0 = V[n0 * VS + c0], e1 = V[n0 * VS + c0 + 4];
            const uint32_t b0 = to_tf32(e0), b1 = to_tf32(e1);
            // G in 3xTF32 like every other contraction (its error enters the chain as lr e dG)
            mma_tf32(gacc[nt], to_tf32(f0 - __uint_as_float(a0)), to_tf32(f1 - __uint_as_float(a1)),
                     to_tf32(f2 - __uint_as_float(a2)), to_tf32(f3 - __uint_as_float(a3)), b0, b1);
            mma_tf32(gacc[nt], a0, a1, a2, a3, to_tf32(e0 - __uint_as_float(b0)),
                     to_tf32(e1 - __uint_as_float(b1)));
            mma_tf32(gacc[nt], a0, a1, a2, a3, b0, b1);
          }
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          if (mt == 1 && nt < 2) continue;
          const int r0 = 16 * mt + gq, c0 = 8 * nt + 2 * tq;
          *reinterpret_cast<float2 *>(G + r0 * GS + c0) = make_float2(gacc[nt][0], gacc[nt][1]);
          *reinterpret_cast<float2 *>(G + (r0 + 8) * GS + c0) = make_float2(gacc[nt][2], gacc[nt][3]);
        }
      }
      // ---- d_k = a_0 . v_k in fp32 (lane k; a_0 broadcast from smem) ----
      float *as = G + BATCH * GS;  // 32 floats after the G tile
      as[lane] = a;
      __syncwarp();
      float dk = 0.f;
      {
        const float4 *vr = reinterpret_cast<const float4 *>(V + lane * VS);
        const float4 *ar = reinterpret_cast<const float4 *>(as);
#pragma unroll
        for (int j4 = 0; j4 < JP / 4; ++j4) {
          const float4 v4 = vr[j4], a4 = ar[j4];
          dk = __fmaf_rn(v4.x, a4.x, dk);
          dk = __fmaf_rn(v4.y, a4.y, dk);
          dk = __fmaf_rn(v4.z, a4.z, dk);
          dk = __fmaf_rn(v4.w, a4.w, dk);
        }
      }
      __syncwarp();
      // ---- the serial chain, scalar per leaf (lane k tracks w_k = a_m . v_k) ----
      float wk = dk;
      float e_mine = 0.f;
#pragma unroll 8
      for (int m = 0; m < nb; ++m) {
        const float gmk = G[m * GS + lane];
        const float em = __shfl_sync(FULL, cur.x - wk, m);
        e_mine = lane == m ? em : e_mine;
        // w += lr (e_m G[m][k] - reg w): the decay is applied as -lr reg w, never through a
        // rounded alpha = 1 - lr reg (its fp32 rounding would compound over long rows)
        wk = __fmaf_rn(lr, __fmaf_rn(em, gmk, -reg * wk), wk);
      }
      // ---- replay the row in leaf order: a += lr (e_m v_m - reg a) ----
#pragma unroll 8
      for (int m = 0; m < nb; ++m) {
        const float em = __shfl_sync(FULL, e_mine, m);
        a = __fmaf_rn(lr, __fmaf_rn(em, V[m * VS + lane], -reg * a), a);
      }
      __syncwarp();
      // G overwrote X / Y: restore their zero columns r in [R, RP) before the next gathers
      if (p.R < RP && lane >= p.R && lane < RP)
        for (int k = 0; k < BATCH; ++k) {
          X[swz(k, lane)] = 0.f;
          Y[swz(k, lane)] = 0.f;
        }
      __syncwarp();
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
  float *X = reinterpret_cast<float *>(smem4) + w * (2 * Tile<RP>::FLOATS + RS + BATCH);
  float *Y = X + Tile<RP>::FLOATS;
  float *cus = Y + Tile<RP>::FLOATS;  // C_u[i, :] of the current row
  float *es = cus + RS;               // the batch's residuals e_k
  for (int k = lane; k < 2 * Tile<RP>::FLOATS + RS + BATCH; k += 32) X[k] = 0.f;
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
    // index pipeline: the next batch's leaf / value / fiber-window loads fly under this batch
    BatchIdx nxt;
    load_batch_idx(p, nxt, Lb, Le, fb, fe, lane);
    for (int L0 = Lb; L0 < Le; L0 += BATCH) {
      const BatchIdx cur = nxt;
      const int nb = cur.nb, lc = cur.lc;
      const float x = cur.x;
      int fnext;
      const int myfib = batch_fib(cur, lane, &fnext);
      if (L0 + BATCH < Le) load_batch_idx(p, nxt, L0 + BATCH, Le, fnext, fe, lane);
      // cross = X * Y is folded into both consumers below (no separate product pass)
      stage_cross<RP>(p, X, Y, myfib, lc, nb, lane, /*fold_leaf=*/false);
      // lane k: s_k = C_u[i] . cross_k  (= A_u[i] . vec_k, since C_u = A_u Bt_u^T is coherent)
      float s = 0.f;
      {
        const float4 *xr = reinterpret_cast<const float4 *>(X + lane * RS);
        const float4 *yr = reinterpret_cast<const float4 *>(Y + lane * RS);
        const float4 *cr = reinterpret_cast<const float4 *>(cus);
#pragma unroll
        for (int r4 = 0; r4 < RP / 4; ++r4) {
          const float4 a4 = xr[r4], b4 = yr[r4], c4 = cr[r4];
          s = __fmaf_rn(a4.x * b4.x, c4.x, s);
          s = __fmaf_rn(a4.y * b4.y, c4.y, s);
          s = __fmaf_rn(a4.z * b4.z, c4.z, s);
          s = __fmaf_rn(a4.w * b4.w, c4.w, s);
        }
      }
      es[lane] = lane < nb ? x - s : 0.f;
      __syncwarp();
      // lane r: g_i[r] += sum_k e_k cross_k[r]  (e_k as float4 broadcasts; e_k = 0 past nb)
      if (lane < RP) {
        const float4 *e4p = reinterpret_cast<const float4 *>(es);
#pragma unroll
        for (int k4 = 0; k4 < BATCH / 4; ++k4) {
          if (4 * k4 < nb) {
            const float4 e4 = e4p[k4];
            const int b = 4 * k4 * RS + lane;
            g = __fmaf_rn(e4.x, X[b] * Y[b], g);
            g = __fmaf_rn(e4.y, X[b + RS] * Y[b + RS], g);
            g = __fmaf_rn(e4.z, X[b + 2 * RS] * Y[b + 2 * RS], g);
            g = __fmaf_rn(e4.w, X[b + 3 * RS] * Y[b + 3 * RS], g);
          }
        }
      }
      __syncwarp();
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
  const int wstride = 2 * Tile<RP>::FLOATS + RS + BATCH;
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
  return (size_t)WPB_R * (2 * Tile<RP>::FLOATS + Tile<RP>::RS + BATCH) * sizeof(float);
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
      // a warp is one serial hogwild worker: each leaf reads its row just before stepping it
      // (different warps race, exactly as the reference's worker threads do)
      for (int k = 0; k < nb; ++k) {
        const int i = __shfl_sync(FULL, lc, k);
        const int sl = __shfl_sync(FULL, slot, k);
        float *ap = p.A + (int64_t)i * p.J + lane;
        const float ak = jl ? *reinterpret_cast<volatile float *>(ap) : 0.f;
        const float vj = vec_s[sl][lane];
        const float s = warp_sum(ak * vj);
        const float e = __shfl_sync(FULL, x, k) - s;
        const float g = p.reg * ak - e * vj;
        // lock-free: the step is never lost -- concurrent writers of one row accumulate
        // through L2 atomics (RED.ADD)
        if (jl) atomicAdd(ap, -p.lr * g);
        __syncwarp();
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

template <int RP, int JP>
int launch_dual(const SweepParams &q, cudaStream_t s) {
  const size_t sm = DualPlan::bytes<RP, JP>();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_dual_kernel<RP, JP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  const int g = grid_for(factor_rows_dual_kernel<RP, JP>, (q.nrows + 1) / 2, DualPlan::WPB, sm);
  factor_rows_dual_kernel<RP, JP><<<g, DualPlan::WPB * 32, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(dual)");
}

template <int RP, int JP>
int launch_ws(const SweepParams &q, cudaStream_t s) {
  const size_t sm = ws::bytes<RP, JP>();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_ws_kernel<RP, JP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_rows_ws_kernel<RP, JP>,
                                                    ws::PAIRS * 64, sm) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  int64_t g = (q.nrows + 2 * ws::PAIRS - 1) / (2 * ws::PAIRS);
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  factor_rows_ws_kernel<RP, JP><<<(int)g, ws::PAIRS * 64, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(ws)");
}

template <int RP, int JP>
int launch_gram(const SweepParams &p, cudaStream_t s) {
  const size_t sm = GramPlan::bytes<RP, JP>();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_gram_kernel<RP, JP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  const int g = grid_for(factor_rows_gram_kernel<RP, JP>, p.nrows, GramPlan::WPB, sm);
  factor_rows_gram_kernel<RP, JP><<<g, GramPlan::WPB * 32, sm, s>>>(p);
  return check_launch("ft_factor_sweep_rows(gram)");
}

template <int RP>
int launch_factor_rows(const SweepParams &p, cudaStream_t s) {
  // FT_FACTOR_KERNEL forces one warp-level K3b for A/B measurement (it also skips K3c):
  // quadr, quadw, dual, ws, gram.  auto: quadr for many rows at orders 3-4 (K3c takes most of
  // these when the slot layout is present), quadw for few long rows at orders 3-4, dual for
  // many rows at orders 5-6, gram for few rows at orders 5-6.
  static const int chosen = [] {
    const char *e = getenv("FT_FACTOR_KERNEL");
    if (!e) return 0;
    if (strcmp(e, "quadr") == 0) return 1;
    if (strcmp(e, "quadw") == 0) return 2;
    if (strcmp(e, "dual") == 0) return 3;
    if (strcmp(e, "ws") == 0) return 4;
    if (strcmp(e, "gram") == 0) return 5;
    return 0;
  }();
  int v = chosen;
  if ((v == 1 || v == 2) && !quad_ok(p)) v = 0;
  if ((v == 1 && p.N > 4) || (v == 2 && p.N > 4) || (v == 4 && p.N != 3)) v = 0;
  if (v == 0) {
    // quadr from 4 (order 3) / 2 (order 4) rows per warp slot of the whole GPU up, quadw
    // below: tools/time_shards.py on the row-sharded sweeps (Netflix mode 1 at 8.9 K / 4.4 K /
    // 2.2 K rows: quadr 2.20 / 1.49 / 1.50 ms, quadw 2.86 / 1.45 / 0.74; Yahoo mode 2 at 3.1 K
    // rows: 23.6 / 21.1; order-4 10 K^4 at 2.5 K / 1.25 K rows: quadr 12.4 / 12.6, quadw
    // 16.4 / 8.2 -- its quadw producers gather two prefix levels)
    const bool many = p.nrows >= (int64_t)sm_count() * quad::WPB * (p.N == 4 ? 2 : 4);
    if (quad_ok(p) && many && p.N <= 4)
      v = 1;
    else if (quad_ok(p) && p.N <= 4)
      v = 2;
    else
      v = p.nrows >= (int64_t)2 * sm_count() * 16 ? 3 : (p.N == 3 ? 4 : 5);
  }
  if (v >= 3 && !p.fiber_ptr)
    return fail(FT_ERR_UNSUPPORTED, "this tree has no fiber arrays (drop_fibers): the fiber-walking "
                "K3b kernels cannot run it");
  switch (v) {
    case 1: return launch_quadr(p, s);
    case 2: return launch_quadw(p, s);
    case 3: return p.J <= 16 ? launch_dual<RP, 16>(p, s) : launch_dual<RP, 32>(p, s);
    case 4: return p.J <= 16 ? launch_ws<RP, 16>(p, s) : launch_ws<RP, 32>(p, s);
    default: return p.J <= 16 ? launch_gram<RP, 16>(p, s) : launch_gram<RP, 32>(p, s);
  }
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
  p.leaf_pc = tree->leaf_pc;
  p.row_leaf_ptr = tree->row_leaf_ptr;
  p.nsegs = tree->seg_coord && tree->seg_leaf_ptr ? tree->num_segs : 0;
  p.seg_coord = tree->seg_coord;
  p.seg_leaf_ptr = tree->seg_leaf_ptr;
  p.A = m->factors[u];
  p.Bt = m->cores_t[u];
  p.Cu = m->dots[u];
  for (int d = 1; d <= N - 2; ++d) p.Cpre[d - 1] = m->dots[(u + d) % N];
  p.Cleaf = m->dots[(u + N - 1) % N];
  p.J = m->ranks[u];
  p.R = m->core_rank;
  p.gather_bytes = 0;
  for (int d = 0; d < N; ++d)
    if (d != u) p.gather_bytes += (int64_t)m->dims[d] * m->core_rank * 4;
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
  // K3c (factor_tc.cu): tcgen05 combine, one thread per row, when the tree carries the slot
  // layout and no warp-level variant is forced; -1 = does not apply
  if (!getenv("FT_FACTOR_KERNEL")) {
    const int rc = launch_factor_tc(tree, model, lr, reg, s);
    if (rc >= 0) return rc;
  }
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
  // FT_CORE_KERNEL=rows forces the one-row-per-warp kernel (the simple reference form);
  // default: K4 quad over the row segments when it applies
  static const bool core_rows_forced = [] {
    const char *e = getenv("FT_CORE_KERNEL");
    return e && strcmp(e, "rows") == 0;
  }();
  // quad walks the row SEGMENTS (rows cut at <= 512 leaves: the core gradient is a sum over a
  // row's leaves), so few long rows fill the GPU too (Netflix mode 2: 2,182 rows -> 89 K
  // segments); without segments it needs rows to fill its 4-rows-per-warp slots
  const int64_t fill = (int64_t)2 * sm_count() * cquad::WPB * 4;
  // (a tree without fiber arrays can only run quad: the fill rule is a speed choice only)
  const bool use_quad = !core_rows_forced && core_quad_ok(p) &&
                        ((p.nsegs > 0 ? p.nsegs : p.nrows) >= fill || !p.fiber_ptr);
  if (use_quad && p.nsegs > 0) {  // the quad kernel reads segments through the row fields
    p.nrows = p.nsegs;
    p.row_coord = p.seg_coord;
    p.row_leaf_ptr = p.seg_leaf_ptr;
  }
  if (!use_quad && !p.fiber_ptr)
    return fail(FT_ERR_UNSUPPORTED, "this tree has no fiber arrays (drop_fibers): K4 needs quad");
  const int g = use_quad ? core_quad_grid(p)
                : p.R <= 8 ? core_rows_grid<8>(p) : p.R <= 16 ? core_rows_grid<16>(p)
                                                              : core_rows_grid<32>(p);
  if ((int64_t)g * p.R * p.J > partials_cap)
    return fail(FT_ERR_ARG, "partials buffer too small (%lld < %lld)", (long long)partials_cap,
                (long long)g * p.R * p.J);
  cudaStream_t s = as_stream(stream);
  *nblocks_out = g;
  if (use_quad) return launch_core_quad(p, g, s);
  if (p.R <= 8) return launch_core_rows<8>(p, g, s);
  if (p.R <= 16) return launch_core_rows<16>(p, g, s);
  return launch_core_rows<32>(p, g, s);
}

extern "C" int ft_factor_sweep_fibers(const ft_tree_t *tree, const ft_model_t *m, int64_t fib_lo,
                                      int64_t fib_hi, float lr, float reg, int32_t max_warps,
                                      void *stream) {
  if (tree && !tree->fiber_ptr)
    return ft::fail(FT_ERR_UNSUPPORTED, "ft_factor_sweep_fibers: the tree's fiber arrays were dropped");
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

extern "C" int ft_sse_tree(const ft_tree_t *tree, const ft_model_t *model, double *out2,
                           void *stream) {
  SweepParams p{};
  if (int rc = fill_rows_params(p, tree, model)) return rc;
  if (!out2) return fail(FT_ERR_ARG, "ft_sse_tree: null out2");
  if (!p.Cu) return fail(FT_ERR_ARG, "ft_sse_tree needs dots[u] (coherent cache)");
  if (!core_quad_ok(p) || p.nsegs <= 0)
    return fail(FT_ERR_UNSUPPORTED, "ft_sse_tree: needs order 3-6, R %% 4 == 0 and the leaf index");
  keep_pool();
  cudaStream_t s = as_stream(stream);
  p.nrows = p.nsegs;
  p.row_coord = p.seg_coord;
  p.row_leaf_ptr = p.seg_leaf_ptr;
  const int g = core_quad_grid<true>(p);
  double *partials = nullptr;
  FT_CUDA(cudaMallocAsync(&partials, sizeof(double) * 2 * g, s));
  p.partials = reinterpret_cast<float *>(partials);
  int rc = launch_core_quad_t<true>(p, g, s);
  if (rc == FT_OK) {
    sum_pairs_f64<<<1, 32, 0, s>>>(partials, g, out2);
    rc = check_launch("ft_sse_tree(sum)");
  }
  cudaFreeAsync(partials, s);
  return rc;
}
