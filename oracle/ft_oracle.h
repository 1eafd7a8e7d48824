/* TEST INFRASTRUCTURE ONLY -- fp64 CPU restatement of the reference hot path.
 *
 * This header belongs to the parity checker.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load libft_oracle.so.  The product
 * (paper_2210_06014_b200/) never links or calls it.
 *
 * Every function restates one reference function; the file:line it follows is given
 * beside the declaration (paths relative to /root/reference/pkg/src/fastertucker/).
 * Arithmetic is sequential fp64 in the reference's expression order, compiled with
 * -ffp-contract=off, so results are bit-identical to the reference's _ckern/_pykern
 * (pinned by tests/test_oracle.py against tests/golden/).
 */
#ifndef FT_ORACLE_H
#define FT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Counter channel order: counter.py:30-31 */
enum { FTO_CH_DOT = 0, FTO_CH_CHAIN = 1, FTO_CH_COMBINE = 2, FTO_CH_SHARED = 3, FTO_CH_UPDATE = 4 };

/* B-CSF tree build, restating csf.py:101-196 (build_tree).
 * idx: nnz x N row-major int64 (0-based, unique rows); vals: nnz.
 * thr <= 0 means fiber_threshold=None (one subtensor per root value, csf.py:113-114).
 * Output buffers are caller-allocated with capacity:
 *   out_leaf_coord[nnz], out_vals[nnz], out_fiber_ptr[nnz+1], out_fiber_coord[nnz*(N-1)],
 *   out_sub_fiber_ptr[nnz+1], out_sub_leaf_ptr[nnz+1],
 *   out_inds[d] -> buffer of nnz for each depth d, out_ptrs[d] -> buffer of nnz+1 (d < N-1).
 * counts_out[0]=F, [1]=S, [2+d]=nodes at depth d.
 * Returns 0, or -1 on bad arguments / allocation failure. */
int fto_build_tree(int N, int64_t nnz, const int64_t *idx, const double *vals, int root_mode,
                   int64_t thr, int64_t *out_leaf_coord, double *out_vals, int64_t *out_fiber_ptr,
                   int64_t *out_fiber_coord, int64_t *out_sub_fiber_ptr, int64_t *out_sub_leaf_ptr,
                   int64_t **out_inds, int64_t **out_ptrs, int64_t *counts_out);

/* refresh_dot_mode: _ckern.pyx:21-33 / _pykern.py:16-26.  out[i,r] = sum_j A[i,j]*Bt[r,j]. */
void fto_refresh(int64_t I, int64_t J, int64_t R, const double *A, const double *Bt, double *out,
                 int64_t *counts);

/* factor_sweep: _ckern.pyx:132-199 / _pykern.py:69-137.  factors/cores_t/dots are N-pointer
 * tables; dots == NULL selects the uncached plan.  ranks[n] = J_n. */
void fto_factor_sweep(int N, int64_t R, const int64_t *ranks, const int64_t *leaf_coord,
                      const double *leaf_val, const int64_t *fiber_ptr, const int64_t *fiber_coord,
                      const int64_t *prefix_modes, int leaf_mode, double **factors,
                      double *const *cores_t, double *const *dots, double lr, double reg,
                      int64_t *counts, int64_t fib_lo, int64_t fib_hi);

/* core_sweep: _ckern.pyx:202-269 / _pykern.py:140-207.  acc is R x J_u, accumulated. */
void fto_core_sweep(int N, int64_t R, const int64_t *ranks, const int64_t *leaf_coord,
                    const double *leaf_val, const int64_t *fiber_ptr, const int64_t *fiber_coord,
                    const int64_t *prefix_modes, int leaf_mode, double *const *factors,
                    double *const *cores_t, double *const *dots, double *acc, int64_t *counts,
                    int64_t fib_lo, int64_t fib_hi);

/* apply_core_update: _ckern.pyx:272-282 / _pykern.py:210-217. */
void fto_apply_core(int64_t R, int64_t J, double *core_t, const double *acc, double omega,
                    double lr, double reg, int64_t *counts);

/* predict_batch: model.py:219-230 (dots = per-mode I_n x R products, already computed);
 * out[m] = sum_r prod_n dots[n][idx[m,n], r]. */
void fto_predict(int N, int64_t R, int64_t m, const int64_t *idx, double *const *dots, double *out);

#ifdef __cplusplus
}
#endif
#endif
