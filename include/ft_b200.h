/* ft_b200.h -- C ABI of the B200-native FasterTucker hot path (libft_b200.so).
 *
 * The reference (arXiv 2210.06014 package `fastertucker` 0.1.0) binds its hot path through the
 * kernel-plugin module `fastertucker._kernels.impl` (pkg/src/fastertucker/_kernels/__init__.py:11-65),
 * whose four entry points are Cython functions over numpy buffers (_kernels/_ckern.pyx:21-282).
 * This library is the sm_100a replacement for those entry points plus the B-CSF builder the
 * reference runs in numpy (csf.py:101-196) and the predict/RMSE reduction (model.py:219-230,
 * train.py:91-98).  Each declaration below cites the reference interface it replaces.
 *
 * Conventions
 *   - Every pointer argument named d_* or held in ft_tree_t / ft_model_t is DEVICE memory owned
 *     by the caller (the Python host layer allocates it as torch tensors).  The library never
 *     frees caller memory; it allocates its own scratch stream-ordered (cudaMallocAsync).
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *     default stream) unless documented as synchronous.
 *   - Every call returns an ft_status; on failure ft_last_error() returns a thread-local message.
 *   - Values are fp32, indices int32 (the reference uses fp64 / int64; see DESIGN.md for the
 *     precision contract: rel 1e-4 per sweep against the fp64 reference).
 *   - Matrices are row-major: A_n is I_n x J_n, Bt_n (= B_n^T, the reference's cores_t) is
 *     R x J_n, C_n (the reference's DotCache.arrays[n]) is I_n x R.
 */
#ifndef FT_B200_H
#define FT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FT_API __attribute__((visibility("default")))
#else
#define FT_API
#endif

#define FT_MAX_ORDER 16
#define FT_MAX_RANK 32
#define FT_MAX_PEERS 16

typedef enum {
  FT_OK = 0,
  FT_ERR_ARG = 1,         /* invalid argument (shape, order, rank > FT_MAX_RANK, ...)       */
  FT_ERR_CUDA = 2,        /* a CUDA runtime / launch error                                 */
  FT_ERR_DUPLICATE = 3,   /* duplicate coordinate found while building (coo.py:56-59)       */
  FT_ERR_EMPTY = 4,       /* empty tensor (csf.py:108-109 BuildError)                      */
  FT_ERR_UNSUPPORTED = 5  /* shape outside what the compiled kernels cover                 */
} ft_status;

/* One B-CSF tree as the sweep kernels read it (a view; all arrays device, caller-owned).
 * Mirrors csf.CsfTree (csf.py:32-80): level_modes = (root, root+1, ..., root+N-1) mod N.
 * row_fiber_ptr / row_coord are NOT reference fields: they are the runs of equal root
 * coordinate over fibers (the unsplit root slices), which the exact row-owner kernels walk. */
typedef struct {
  int32_t order;                /* N >= 3                                                    */
  int32_t root_mode;            /* level-0 mode t; leaf mode is (t+N-1) mod N               */
  int64_t nnz;                  /* leaves                                                    */
  int64_t num_fibers;           /* F                                                         */
  int64_t num_rows;             /* root slices (distinct level-0 coordinates)                */
  const int32_t *leaf_coord;    /* [nnz]   csf inds[N-1]                                     */
  const float *vals;            /* [nnz]   csf vals (level order)                            */
  const int32_t *fiber_ptr;     /* [F+1]   csf fiber_ptr                                     */
  const int32_t *fiber_coord;   /* [F*(N-1)] csf fiber_coord, row-major                      */
  const int32_t *row_fiber_ptr; /* [rows+1] fiber index where each root slice starts         */
  const int32_t *row_coord;     /* [rows]  level-0 coordinate of each root slice             */
  /* Leaf-major index (optional, NULL = absent; filled by ft_tree_leaf_index).  Not reference
   * fields: derived once per tree so the row-owner kernels read every per-leaf operand with
   * plain coalesced loads instead of the fiber-window ballot -> fiber_coord dependent chain. */
  const int32_t *leaf_pc;       /* [nnz x (N-2)] levels 1..N-2 of each leaf's fiber (N <= 6) */
  const int32_t *row_leaf_ptr;  /* [rows+1] first leaf of each root slice                    */
  /* Row segments for the core sweep (optional): every root slice cut into pieces of at most
   * `max_len` leaves (ft_tree_row_segments).  The core gradient is a sum over a row's leaves,
   * so pieces of one row may run on different warps; the factor sweep never uses them. */
  int64_t num_segs;
  const int32_t *seg_coord;     /* [segs]  row coordinate of each segment                    */
  const int32_t *seg_leaf_ptr;  /* [segs+1] first leaf of each segment                       */
  /* Slot layout for the tcgen05 factor sweep (optional, slot_grid = 0 = absent; K1d,
   * ft_tree_slot_plan / ft_tree_slot_fill).  Slot q = c + G s (CTA c < G, slot s < 128) owns rows
   * q, q + 128 G, ... and walks their leaves one per batch; entry [batch][s] of CTA c holds that
   * leaf's coordinates and value, so each batch's operands are coalesced loads. */
  int32_t slot_grid;            /* G (CTAs the layout was built for)                         */
  int32_t slot_kb;              /* leaves of one row slot per batch: 1 or 8 (128/KB rows/CTA) */
  const int32_t *slot_batch_ptr;/* [G+1] first batch of each CTA                             */
  const int32_t *slot_lc;       /* [batches x 128] leaf coordinate | 0x80000000 on the first
                                   leaf of a row; -1 = padding (the slot's stream ended)      */
  const int32_t *slot_pc;       /* [batches x (N-2) x 128] levels 1..N-2                      */
  const float *slot_x;          /* [batches x 128] values                                    */
} ft_tree_t;

/* Model parameters and the C^(n) cache (model.py:45-103, cache.py:28-57). */
typedef struct {
  int32_t order;
  int32_t core_rank;                /* R                                                    */
  int64_t dims[FT_MAX_ORDER];       /* I_n                                                  */
  int32_t ranks[FT_MAX_ORDER];      /* J_n                                                  */
  float *factors[FT_MAX_ORDER];     /* A_n  [I_n x J_n]                                     */
  float *cores_t[FT_MAX_ORDER];     /* Bt_n [R x J_n]                                       */
  float *dots[FT_MAX_ORDER];        /* C_n  [I_n x R]                                       */
} ft_model_t;

/* ---------------------------------------------------------------------------------------- */
FT_API const char *ft_last_error(void);
FT_API int ft_abi_version(void);
/* number of SMs of the current device (sizes persistent grids and partial buffers) */
FT_API int ft_sm_count(int32_t *out);

/* K1  B-CSF builder.  Replaces csf.build_tree (csf.py:101-196): lexicographic sort in the
 * cyclic level order, fiber runs, greedy split of root slices at `thr` whole fibers
 * (thr <= 0 means fiber_threshold=None), per-depth inds/ptrs.  Output arrays are bit-identical
 * to the reference's (as int32).  idx: device int32 [nnz x N] row-major, 0-based, unique.
 * dims: HOST int64[N].  Output buffers are device, caller-allocated with capacity:
 *   leaf_vals[nnz], inds[d][nnz] (d < N), ptrs[d][nnz+1] (d < N-1), fiber_ptr[nnz+1],
 *   fiber_coord[nnz*(N-1)], sub_fiber_ptr[nnz+1], sub_leaf_ptr[nnz+1],
 *   row_fiber_ptr[nnz+1], row_coord[nnz].   inds / ptrs are HOST arrays of device pointers.
 * counts_out (HOST int64[4+N]): F, S, rows, first duplicate position (-1 if none),
 *   then node count per depth.  SYNCHRONOUS (sizes are data dependent).
 * Compact build: ptrs == NULL (and inds[d < N-1], sub_fiber_ptr, sub_leaf_ptr may be NULL)
 *   skips the reference-format per-depth arrays and subtensors, producing only what the sweep
 *   kernels read (leaf coordinates, values, fiber_ptr / fiber_coord, rows); a compact build may
 *   also pass fiber_coord == NULL (no fiber coordinates: the row-owner sweeps read leaf_pc).
 * leaf_pc (optional, device int32 [nnz x (N-2)], 3 <= N <= 6): the leaf-major prefix index of
 *   ft_tree_leaf_index, written from the sorted level columns at no extra pass (order 3: the
 *   builder sorts straight into it).
 * Returns FT_ERR_DUPLICATE (with counts_out[3] set) if two entries share a coordinate. */
FT_API int ft_build_tree(int32_t N, int64_t nnz, const int64_t *dims, const int32_t *idx,
                  const float *vals, int32_t root_mode, int64_t thr, float *leaf_vals,
                  int32_t *const *inds, int32_t *const *ptrs, int32_t *fiber_ptr,
                  int32_t *fiber_coord, int32_t *sub_fiber_ptr, int32_t *sub_leaf_ptr,
                  int32_t *row_fiber_ptr, int32_t *row_coord, int64_t *counts_out,
                  int32_t *leaf_pc, void *stream);

/* K1  derived build: the tree rooted at (prev->root_mode + 1) mod N from the tree `prev`
 * (which must carry the leaf-major index, ft_tree_leaf_index): a stable 32-bit-key radix sort
 * of prev's leaf order by its levels 1..N-1 gives the new tree's order (prev's root level
 * becomes the new leaf level), then the same fiber / root-slice / split / per-depth steps as
 * ft_build_tree.  Output arrays, capacities and counts_out as ft_build_tree (dims: HOST
 * int64[N]); bit-identical to building from the COO.  FT_ERR_UNSUPPORTED when the key would
 * exceed 32 bits or prev lacks the index (build from the COO instead).  SYNCHRONOUS. */
FT_API int ft_build_tree_derived(const ft_tree_t *prev, const int64_t *dims, int64_t thr,
                                 float *leaf_vals, int32_t *const *inds, int32_t *const *ptrs,
                                 int32_t *fiber_ptr, int32_t *fiber_coord, int32_t *sub_fiber_ptr,
                                 int32_t *sub_leaf_ptr, int32_t *row_fiber_ptr,
                                 int32_t *row_coord, int64_t *counts_out, int32_t *leaf_pc,
                                 void *stream);
/* K1b Leaf-major index of a built tree (reads tree->fiber_ptr / fiber_coord / row_fiber_ptr):
 *   leaf_pc[L * (N-2) + d] = fiber_coord[f(L) * (N-1) + 1 + d], d < N-2, for every leaf L of
 *   fiber f(L) (the prefix levels 1..N-2 expanded to the leaves; orders 3-6 only), and
 *   row_leaf_ptr[r] = fiber_ptr[row_fiber_ptr[r]] for r <= rows.
 * Either output may be NULL.  Asynchronous. */
FT_API int ft_tree_leaf_index(const ft_tree_t *tree, int32_t *leaf_pc, int32_t *row_leaf_ptr,
                              void *stream);
/* K1c Row segments (reads tree->row_coord / row_leaf_ptr): root slice r becomes
 * ceil(len_r / max_len) consecutive segments of <= max_len leaves.  Output capacity: rows +
 * nnz / max_len + 1 entries for seg_coord, one more for seg_leaf_ptr.  *nseg_out (HOST) gets the
 * segment count.  SYNCHRONOUS (the count is read back). */
FT_API int ft_tree_row_segments(const ft_tree_t *tree, int32_t max_len, int32_t *seg_coord,
                                int32_t *seg_leaf_ptr, int64_t *nseg_out, void *stream);
/* K1d Slot layout for the tcgen05 factor sweep (reads tree->row_leaf_ptr / leaf_coord /
 * leaf_pc / vals).  Not a reference structure: it re-orders the tree's leaves so that the
 * sweep over the tree rooted at u (factor_sweep, _ckern.pyx:132-199) reads them coalesced.
 * ft_tree_slot_plan: *grid_out = G and *kb_out = KB (1: one row per TMEM lane, many rows;
 *   8: 16 rows per CTA, few long rows), or G = 0 when the tcgen05 sweep does not apply to this
 *   tree (shape J, R, order, rows, FT_FACTOR_TC=0); with batch_ptr == NULL only G / KB are
 *   returned; else batch_ptr (device int32 [G+1]) is filled and *len_out (HOST) gets the entry
 *   count (batches x 128).  SYNCHRONOUS when batch_ptr != NULL.
 * ft_tree_slot_fill: writes slot_lc / slot_x [len] and slot_pc [len x (N-2)]; must follow
 *   the ft_tree_slot_plan call with batch_ptr of the same tree.  SYNCHRONOUS. */
FT_API int ft_tree_slot_plan(const ft_tree_t *tree, int32_t J, int32_t R, int32_t *grid_out,
                             int32_t *kb_out, int32_t *batch_ptr, int64_t *len_out, void *stream);
FT_API int ft_tree_slot_fill(const ft_tree_t *tree, int32_t grid, const int32_t *batch_ptr,
                             int32_t *slot_lc, int32_t *slot_pc, float *slot_x, void *stream);
/* K2  C = A * Bt^T  (I x R), i.e. refresh_dot_mode (_ckern.pyx:21-33, cache.py:60-70), with the
 * divergence guard of train.py:101-110 fused: if guard != NULL, atomically max-es the IEEE bits
 * of |A| into guard[0] (NaN sorts above +inf, so one word detects both cases). */
FT_API int ft_refresh(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt, float *C,
               uint32_t *guard, void *stream);

/* K2 fused with the C_u all-gather of the row-block-sharded multi-GPU epoch (dist.py): computes
 * the I rows of C = A Bt^T of THIS rank's block and stores them into every destination -- the
 * local C_u and each peer's C_u, all already offset to the block's first row; peer pointers
 * are CUDA-IPC mappings, so on a multi-GPU node the stores travel over NVLink inside the
 * refresh kernel instead of a separate NCCL all-gather.  ndst <= FT_MAX_PEERS.  The caller
 * fences (stream sync + barrier) before any rank reads the gathered C_u. */
FT_API int ft_refresh_scatter(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt,
                              float *const *dsts, int32_t ndst, uint32_t *guard, void *stream);
/* Stream-ordered barrier for the fused refresh + all-gather: publishes `seq` into slot `rank` of
 * every rank's flag array (peer_flags[q] = rank q's array, CUDA-IPC-mapped; world <= FT_MAX_PEERS
 * uint32 slots each) after a system-scope fence, then waits on the device until every slot of
 * local_flags holds >= seq.  Replaces a host synchronize + barrier between the refresh of C_u and
 * the next sweep (no reference counterpart: the reference has no distributed path).
 * Traps after 20 s if a peer never arrives. */
FT_API int ft_peer_barrier(uint32_t *local_flags, uint32_t *const *peer_flags, int32_t world,
                           int32_t rank, uint32_t seq, void *stream);

/* K3b  Exact factor sweep of mode u = tree->root_mode: replaces factor_sweep over the tree
 * rooted at (u+1) mod N (_ckern.pyx:132-199, train.py:152-197).  One warp owns one row of A_u
 * (one root slice of the tree rooted at u) and applies its updates in the reference's serial
 * order; C_m (m != u) and Bt_u are read-only, so the result equals the serial sweep up to fp32
 * rounding.  Requires the cache (model->dots) to be coherent for every m != u. */
FT_API int ft_factor_sweep_rows(const ft_tree_t *tree, const ft_model_t *model, float lr, float reg,
                         void *stream);

/* K3a  Hogwild factor sweep over fibers [fib_lo, fib_hi) of a tree rooted at t = (u+1) mod N,
 * i.e. the reference's own traversal (_ckern.pyx:163-191) with one warp per 32-fiber batch and
 * lock-free row updates (train.py:124-149 with workers > 1): each step is computed from a
 * possibly stale row and added with an L2 atomic, so concurrent steps are never lost.
 * max_warps > 0 caps the number of concurrently sweeping warps (the staleness bound: the
 * reference's hogwild runs <= #cores writers; 0 = one persistent grid). */
FT_API int ft_factor_sweep_fibers(const ft_tree_t *tree, const ft_model_t *model, int64_t fib_lo,
                           int64_t fib_hi, float lr, float reg, int32_t max_warps,
                           void *stream);

/* K4  Core-gradient sweep of mode u = tree->root_mode: replaces core_sweep
 * (_ckern.pyx:202-269, train.py:200-236) in its row form acc = -G^T A_u with
 * G[i,:] = sum_{leaves of row i} e * cross.  Writes one R x J_u partial per block to
 * `partials` (capacity `partials_cap` floats) and the block count to *nblocks_out (HOST).
 * Deterministic (static row->warp map, fixed-order reductions, no atomics).
 * Requires model->dots[u] coherent with (A_u, Bt_u). */
FT_API int ft_core_sweep_rows(const ft_tree_t *tree, const ft_model_t *model, float *partials,
                       int64_t partials_cap, int32_t *nblocks_out, void *stream);

/* Upper bound of `partials` floats ft_core_sweep_rows needs for rank R x J. */
FT_API int64_t ft_core_partials_size(int32_t R, int32_t J);

/* K5  apply_core_update (_ckern.pyx:272-282): acc = -(sum of `nparts` partials, fixed order);
 * Bt -= lr * (acc / omega + reg * Bt).  If acc_out != NULL the reduced acc (R x J, the
 * reference's `acc` buffer) is stored there.  Guard as in ft_refresh, over the new Bt.
 * `partials` may be the output of ft_core_sweep_rows, or (nparts = 1) an allreduced acc
 * negated -- see `acc_is_negated`: 1 means partials hold +G^T A (kernel output), 0 means
 * they hold the reference's acc itself. */
FT_API int ft_core_apply(int32_t R, int32_t J, float *Bt, const float *partials, int32_t nparts,
                  int32_t acc_is_negated, double omega, float lr, float reg, float *acc_out,
                  uint32_t *guard, void *stream);

/* Sum partials only (multi-GPU: reduce locally, then allreduce R*J floats, then apply). */
FT_API int ft_core_reduce(int32_t R, int32_t J, const float *partials, int32_t nparts, float *out,
                   void *stream);

/* K6  predict_batch (model.py:219-230) from the coherent cache: out[m] = sum_r prod_n C_n[i_n,r]. */
FT_API int ft_predict(const ft_model_t *model, int64_t m, const int32_t *idx, float *out, void *stream);

/* K6  evaluate (train.py:91-98): out2[0] = sum (x - xhat)^2, out2[1] = sum |x - xhat| (fp64,
 * DEVICE double[2], deterministic two-level reduction). */
FT_API int ft_sse(const ft_model_t *model, int64_t m, const int32_t *idx, const float *vals,
           double *out2, void *stream);

/* K6b evaluate over the entries a tree holds (the training set): out2 = (sum (x - xhat)^2,
 * sum |x - xhat|) in fp64, walking the tree's row segments with the C rows of its levels --
 * two gathers per entry instead of N (the root mode's C row stays in shared memory per
 * segment).  Same value as ft_sse over those entries up to the summation order.  Needs
 * order 3, R % 4 == 0, the leaf-major index and row segments (FT_ERR_UNSUPPORTED otherwise),
 * and model->dots coherent.  out2 is DEVICE double[2]. */
FT_API int ft_sse_tree(const ft_tree_t *tree, const ft_model_t *model, double *out2, void *stream);
/* K7  Synthetic COO generator (same distribution as coo.generate_synthetic, coo.py:164-213:
 * distinct coordinates uniform without replacement, values U[lo, hi]; NOT the same stream).
 * Writes nnz unique coordinates (row-major int32 [nnz x N]) in a random entry order, and
 * values (so the first k entries are a uniform random test split).  Index spaces wider than
 * 64 bits draw i.i.d. cells without a dedup pass (allowed only when nnz^2 / (2 capacity) <
 * 1e-6; the builder rejects any duplicate).  SYNCHRONOUS. */
FT_API int ft_generate_coo(int32_t N, const int64_t *dims, int64_t nnz, uint64_t seed, float lo,
                    float hi, int32_t *idx, float *vals, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FT_B200_H */
