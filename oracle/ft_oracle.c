/* TEST INFRASTRUCTURE ONLY -- fp64 CPU restatement of the reference hot path.
 * See ft_oracle.h for the contract.  Reference paths are relative to
 * /root/reference/pkg/src/fastertucker/.  Not part of the product.
 */
#define _GNU_SOURCE
#include "ft_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------ */
/* B-CSF build (csf.py:101-196)                                                               */
/* ------------------------------------------------------------------------------------------ */

typedef struct {
    const int64_t *idx;
    int N;
    int perm[64];
} sort_ctx;

/* Lexicographic order of the cyclically permuted coordinates; level 0 is the primary key
 * (csf.py:120-122: np.lexsort(keys.T[::-1]) sorts by keys[:,0] first). Coordinates are
 * unique (coo.py:56-59), so the order is total and any correct sort reproduces it. */
static int cmp_entries(const void *pa, const void *pb, void *vctx) {
    const sort_ctx *c = (const sort_ctx *)vctx;
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    for (int d = 0; d < c->N; ++d) {
        int64_t ka = c->idx[a * c->N + c->perm[d]];
        int64_t kb = c->idx[b * c->N + c->perm[d]];
        if (ka != kb) return ka < kb ? -1 : 1;
    }
    return (a > b) - (a < b);
}

int fto_build_tree(int N, int64_t nnz, const int64_t *idx, const double *vals, int root_mode,
                   int64_t thr, int64_t *out_leaf_coord, double *out_vals, int64_t *out_fiber_ptr,
                   int64_t *out_fiber_coord, int64_t *out_sub_fiber_ptr, int64_t *out_sub_leaf_ptr,
                   int64_t **out_inds, int64_t **out_ptrs, int64_t *counts_out) {
    if (N < 2 || N > 64 || nnz <= 0 || root_mode < 0 || root_mode >= N) return -1;
    if (thr <= 0) thr = nnz + 1; /* fiber_threshold=None: csf.py:113-114 */

    sort_ctx ctx;
    ctx.idx = idx;
    ctx.N = N;
    for (int d = 0; d < N; ++d) ctx.perm[d] = (root_mode + d) % N; /* csf.py:120 */

    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * nnz);
    int64_t *k = (int64_t *)malloc(sizeof(int64_t) * nnz * N); /* sorted level-order keys */
    unsigned char *sub_start = (unsigned char *)calloc(nnz, 1);
    int64_t *fiber_of_entry = (int64_t *)malloc(sizeof(int64_t) * nnz);
    if (!order || !k || !sub_start || !fiber_of_entry) {
        free(order); free(k); free(sub_start); free(fiber_of_entry);
        return -1;
    }
    for (int64_t e = 0; e < nnz; ++e) order[e] = e;
    qsort_r(order, (size_t)nnz, sizeof(int64_t), cmp_entries, &ctx);
    for (int64_t e = 0; e < nnz; ++e) {
        const int64_t *row = idx + order[e] * N;
        for (int d = 0; d < N; ++d) k[e * N + d] = row[ctx.perm[d]];
        out_vals[e] = vals[order[e]];
        out_leaf_coord[e] = row[ctx.perm[N - 1]];
    }

    /* Fibers: runs of equal first N-1 level keys (csf.py:126-133). */
    int64_t F = 0;
    for (int64_t e = 0; e < nnz; ++e) {
        int start = (e == 0);
        if (!start)
            for (int d = 0; d < N - 1; ++d)
                if (k[e * N + d] != k[(e - 1) * N + d]) { start = 1; break; }
        if (start) {
            out_fiber_ptr[F] = e;
            for (int d = 0; d < N - 1; ++d) out_fiber_coord[F * (N - 1) + d] = k[e * N + d];
            ++F;
        }
        fiber_of_entry[e] = F - 1;
    }
    out_fiber_ptr[F] = nnz;

    /* Greedy split of each root run into chunks of <= thr whole fibers (csf.py:135-148). */
    int64_t S = 0;
    int64_t run_start = 0;
    for (int64_t f = 1; f <= F; ++f) {
        int run_end = (f == F) || (out_fiber_coord[f * (N - 1)] != out_fiber_coord[(f - 1) * (N - 1)]);
        if (!run_end) continue;
        for (int64_t s = run_start; s < f; s += thr) out_sub_fiber_ptr[S++] = s;
        run_start = f;
    }
    out_sub_fiber_ptr[S] = F;
    /* Entry-level subtensor starts (csf.py:147-153): first leaf of each chunk's first fiber. */
    for (int64_t s = 0; s < S; ++s) {
        int64_t e = out_fiber_ptr[out_sub_fiber_ptr[s]];
        sub_start[e] = 1;
        out_sub_leaf_ptr[s] = e;
    }
    out_sub_leaf_ptr[S] = nnz;

    /* Per-depth node starts (csf.py:157-166) then inds/ptrs (csf.py:168-178).  A node starts
     * at depth d where the level-(0..d) prefix changes or a subtensor starts; every entry is
     * a leaf node.  ptrs[d][node] = index of the node's first child at depth d+1. */
    int64_t *count_d = counts_out + 2;
    for (int d = 0; d < N; ++d) count_d[d] = 0;
    for (int64_t e = 0; e < nnz; ++e) {
        int changed_depth = N; /* smallest depth whose prefix changed; N = none */
        if (e == 0 || sub_start[e]) {
            changed_depth = 0;
        } else {
            for (int d = 0; d < N - 1; ++d)
                if (k[e * N + d] != k[(e - 1) * N + d]) { changed_depth = d; break; }
        }
        for (int d = 0; d < N; ++d) {
            int starts = (d == N - 1) || (d >= changed_depth);
            if (!starts) continue;
            out_inds[d][count_d[d]] = k[e * N + d];
            if (d < N - 1) out_ptrs[d][count_d[d]] = count_d[d + 1]; /* child about to start */
            count_d[d]++;
        }
    }
    for (int d = 0; d < N - 1; ++d) out_ptrs[d][count_d[d]] = count_d[d + 1];

    counts_out[0] = F;
    counts_out[1] = S;
    free(order);
    free(k);
    free(sub_start);
    free(fiber_of_entry);
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Kernels (_ckern.pyx / _pykern.py)                                                          */
/* ------------------------------------------------------------------------------------------ */

void fto_refresh(int64_t I, int64_t J, int64_t R, const double *A, const double *Bt, double *out,
                 int64_t *counts) {
    for (int64_t i = 0; i < I; ++i)
        for (int64_t r = 0; r < R; ++r) {
            double s = 0.0;
            for (int64_t j = 0; j < J; ++j) s = s + A[i * J + j] * Bt[r * J + j];
            out[i * R + r] = s;
        }
    if (counts) counts[FTO_CH_DOT] += I * J * R;
}

/* Rank products of one fiber: cached (_ckern.pyx:92-103) or rebuilt from fresh dots
 * (_ckern.pyx:106-117), chained left to right over the prefix modes. */
static void rank_products(int n_prefix, int64_t R, const int64_t *ranks, const int64_t *fc,
                          const int64_t *pm, double *const *factors, double *const *cores_t,
                          double *const *dots, double *cross) {
    for (int64_t r = 0; r < R; ++r) {
        double v = 0.0;
        for (int d = 0; d < n_prefix; ++d) {
            int64_t m = pm[d];
            double t;
            if (dots) {
                t = dots[m][fc[d] * R + r];
            } else {
                int64_t Jm = ranks[m];
                const double *a = factors[m] + fc[d] * Jm;
                const double *b = cores_t[m] + r * Jm;
                t = 0.0;
                for (int64_t j = 0; j < Jm; ++j) t = t + a[j] * b[j];
            }
            v = (d == 0) ? t : v * t;
        }
        cross[r] = v;
    }
}

/* Shared vector (_ckern.pyx:120-129): vec[j] = sum_r cross[r] * Bt_u[r,j], r outer. */
static void shared_vector(int64_t R, int64_t Ju, const double *cross, const double *Bu, double *vec) {
    for (int64_t j = 0; j < Ju; ++j) vec[j] = 0.0;
    for (int64_t r = 0; r < R; ++r) {
        double c = cross[r];
        for (int64_t j = 0; j < Ju; ++j) vec[j] = vec[j] + c * Bu[r * Ju + j];
    }
}

static void sweep(int is_core, int N, int64_t R, const int64_t *ranks, const int64_t *leaf_coord,
                  const double *leaf_val, const int64_t *fiber_ptr, const int64_t *fiber_coord,
                  const int64_t *prefix_modes, int leaf_mode, double *const *factors,
                  double *const *cores_t, double *const *dots, double lr, double reg, double *acc,
                  int64_t *counts, int64_t fib_lo, int64_t fib_hi) {
    const int n_prefix = N - 1;
    const int64_t Ju = ranks[leaf_mode];
    double *A_u = factors[leaf_mode];
    const double *B_u = cores_t[leaf_mode];
    double *cross = (double *)malloc(sizeof(double) * (size_t)R);
    double *vec = (double *)malloc(sizeof(double) * (size_t)Ju);
    int64_t dots_per_leaf = 0;
    for (int d = 0; d < n_prefix; ++d) dots_per_leaf += ranks[prefix_modes[d]];
    dots_per_leaf *= R;
    int64_t c_dot = 0, c_chain = 0, c_comb = 0, c_shared = 0, c_upd = 0;

    for (int64_t f = fib_lo; f < fib_hi; ++f) {
        const int64_t *fc = fiber_coord + f * n_prefix;
        if (dots) { /* cached plan: once per fiber (_ckern.pyx:164-169) */
            rank_products(n_prefix, R, ranks, fc, prefix_modes, factors, cores_t, dots, cross);
            shared_vector(R, Ju, cross, B_u, vec);
            c_chain += (N - 2) * R;
            c_comb += Ju * R;
            c_shared += Ju * R + N - 2;
        }
        for (int64_t leaf = fiber_ptr[f]; leaf < fiber_ptr[f + 1]; ++leaf) {
            if (!dots) { /* uncached plan: per leaf from fresh dots (_ckern.pyx:171-177) */
                rank_products(n_prefix, R, ranks, fc, prefix_modes, factors, cores_t, NULL, cross);
                shared_vector(R, Ju, cross, B_u, vec);
                c_dot += dots_per_leaf;
                c_chain += (N - 2) * R;
                c_comb += Ju * R;
                c_shared += Ju * R + N - 2;
            }
            double *arow = A_u + leaf_coord[leaf] * Ju;
            double x = leaf_val[leaf];
            double s = 0.0;
            for (int64_t j = 0; j < Ju; ++j) s = s + arow[j] * vec[j];
            double e = x - s;
            if (!is_core) { /* row SGD step (_ckern.pyx:184-188) */
                for (int64_t j = 0; j < Ju; ++j) {
                    double g = reg * arow[j] - e * vec[j];
                    arow[j] = arow[j] - lr * g;
                }
                c_upd += 4 * Ju;
            } else { /* core gradient accumulation (_ckern.pyx:254-260) */
                for (int64_t r = 0; r < R; ++r) {
                    double c = e * cross[r];
                    for (int64_t j = 0; j < Ju; ++j) acc[r * Ju + j] = acc[r * Ju + j] - c * arow[j];
                }
                c_upd += Ju + R * (1 + Ju);
            }
        }
    }
    if (counts) {
        counts[FTO_CH_DOT] += c_dot;
        counts[FTO_CH_CHAIN] += c_chain;
        counts[FTO_CH_COMBINE] += c_comb;
        counts[FTO_CH_SHARED] += c_shared;
        counts[FTO_CH_UPDATE] += c_upd;
    }
    free(cross);
    free(vec);
}

void fto_factor_sweep(int N, int64_t R, const int64_t *ranks, const int64_t *leaf_coord,
                      const double *leaf_val, const int64_t *fiber_ptr, const int64_t *fiber_coord,
                      const int64_t *prefix_modes, int leaf_mode, double **factors,
                      double *const *cores_t, double *const *dots, double lr, double reg,
                      int64_t *counts, int64_t fib_lo, int64_t fib_hi) {
    sweep(0, N, R, ranks, leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
          factors, cores_t, dots, lr, reg, NULL, counts, fib_lo, fib_hi);
}

void fto_core_sweep(int N, int64_t R, const int64_t *ranks, const int64_t *leaf_coord,
                    const double *leaf_val, const int64_t *fiber_ptr, const int64_t *fiber_coord,
                    const int64_t *prefix_modes, int leaf_mode, double *const *factors,
                    double *const *cores_t, double *const *dots, double *acc, int64_t *counts,
                    int64_t fib_lo, int64_t fib_hi) {
    sweep(1, N, R, ranks, leaf_coord, leaf_val, fiber_ptr, fiber_coord, prefix_modes, leaf_mode,
          factors, cores_t, dots, 0.0, 0.0, acc, counts, fib_lo, fib_hi);
}

void fto_apply_core(int64_t R, int64_t J, double *core_t, const double *acc, double omega,
                    double lr, double reg, int64_t *counts) {
    for (int64_t r = 0; r < R; ++r)
        for (int64_t j = 0; j < J; ++j) {
            double g = acc[r * J + j] / omega + reg * core_t[r * J + j];
            core_t[r * J + j] = core_t[r * J + j] - lr * g;
        }
    if (counts) counts[FTO_CH_UPDATE] += 2 * R * J;
}

void fto_predict(int N, int64_t R, int64_t m, const int64_t *idx, double *const *dots, double *out) {
    for (int64_t e = 0; e < m; ++e) {
        double sum = 0.0;
        for (int64_t r = 0; r < R; ++r) {
            double p = dots[0][idx[e * N + 0] * R + r];
            for (int n = 1; n < N; ++n) p = p * dots[n][idx[e * N + n] * R + r];
            sum = sum + p;
        }
        out[e] = sum;
    }
}
