/*
 * oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * A plain, slow, single-threaded fp64 implementation of the DDG two-level
 * symmetric multiplicative Schwarz preconditioner and of PCG, following
 * PAPER.md (arXiv:1504.00907) step by step.  No blocking, fusion, colouring
 * parallelism or reordering beyond what the paper's algorithm states.
 * Where the paper is silent the DESIGN.md reading is named (R1..R18).
 *
 *   setup (or_setup)
 *     1. parts Omega_I from the partition
 *     2. overlap Omega~_i: graph distance <= Delta in A
 *     3. colours + sweep order (reading R3/R6)
 *     4. local matrices A_i = R~_i A R~_i^T, Cholesky
 *     5. coarse basis: F restricted to Omega_I,
 *        orthonormalised per part (double-double MGS, R6c),
 *        rank-deficient columns discarded (R7)
 *     6. A_0 = R_0 A R_0^T  (A_c = P^T A P), block storage
 *     7. Cholesky of A_0 in envelope storage
 *        (or, for large A_0, the nested-dissection multifrontal
 *        Cholesky of oracle/coarse_nd.py through or_set_coarse_solver)
 *   apply (or_apply_precond)
 *   three levels (or_setup3): the two-level method again on
 *     A_0 with F_0 = R_0 F and a partition of the parts
 *   pcg (or_pcg)
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (see DESIGN.md "Oracle pins"); none is "parity unpinned".
 *
 * Floor mode (or_opts.perturb, SURVEY.md §8(c) "an unavoidable floor"): the
 * same method with harmless rounding changes -- dot products summed in
 * reverse, every local matrix factored with its unknowns in reversed order,
 * the envelope coarse factor built on the reversed coarse order.  The
 * distance between the plain and the perturbed solution is the intrinsic
 * fp64 floor of a configuration.
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];
const char* or_last_error(void) { return g_err; }
static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

struct or_ctx {
    int64_t n;
    int64_t* rp;
    int32_t* ci;
    double* va;
    int k, nparts, overlap;
    double rank_tol;
    int32_t* part;
    /* parts Omega_I: sorted node lists */
    int64_t* bptr;
    int32_t* bidx;
    int32_t* bpos; /* position of node v inside its part's list */
    /* overlapping subdomains Omega~_i: sorted node lists */
    int64_t* optr;
    int32_t* oidx;
    /* colours and sweep order */
    int32_t* colour;
    int ncolours;
    int32_t* order;
    /* local Cholesky factors, packed lower, row-major: L[a][b] at a(a+1)/2 + b */
    int64_t* loff;
    double* L;
    /* coarse basis */
    int32_t* cptr;  /* coarse offset of part I (nparts+1) */
    int64_t* qoff;  /* offset of Q_I (|Omega_I| x r_I column-major) in Q */
    double* Q;
    int dropped;
    double min_ratio;
    int64_t nc;
    int32_t* cpart;  /* part of every coarse unknown (nc) */
    /* A_0 in block form: for part I, blocks (I,J) with
       J <= I adjacent to I in the graph of A (or J = I), J ascending in
       aadj[aptr[I]..aptr[I+1]); block e is r_I x r_J row-major at ablk+aoff[e];
       in diagonal blocks only i >= j is filled */
    int64_t* aptr;
    int32_t* aadj;
    int64_t* aoff;
    double* ablk;
    /* coarse factor, envelope lower storage: row i holds columns efirst[i]..i
       (in floor mode, of the matrix with the coarse order reversed) */
    int64_t* efirst;
    int64_t* eptr;
    double* el;
    /* external exact coarse solve (oracle/coarse_nd.py), replaces el */
    int coarse_external;
    or_coarse_fn ext_fn;
    void* ext_user;
    int perturb;
    /* three-level method: the two-level method applied to
       A_0 with F_0 = R_0 F; when set, it replaces the exact coarse solve */
    struct or_ctx* child;
    const int32_t* colour_in;   /* caller's colouring during setup (borrowed), or NULL */
};

#define ALLOC(p, cnt)                                                        \
    do {                                                                     \
        (p) = calloc((size_t)(cnt) > 0 ? (size_t)(cnt) : 1, sizeof(*(p)));   \
        if (!(p)) return fail(OR_E_OOM, "out of memory (%lld items)", (long long)(cnt)); \
    } while (0)

/* ---------------------------------------------------------------------------
 * double-double arithmetic (reading R6c: orthonormalisation accumulated in
 * double-double so the span of F restricted to a part is resolved to fp64
 * rounding even for ill-conditioned blocks).  Dekker / Knuth error-free
 * transformations.  Compiled with -ffp-contract=off.
 * ------------------------------------------------------------------------- */
typedef struct { double hi, lo; } dd;
static dd two_sum(double a, double b) {
    dd r; double s = a + b, bb = s - a;
    r.hi = s; r.lo = (a - (s - bb)) + (b - bb); return r;
}
static dd quick_two_sum(double a, double b) {
    dd r; double s = a + b; r.hi = s; r.lo = b - (s - a); return r;
}
static dd dd_add(dd x, dd y) {
    dd s = two_sum(x.hi, y.hi), t = two_sum(x.lo, y.lo);
    s.lo += t.hi; s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo; return quick_two_sum(s.hi, s.lo);
}
static dd dd_neg(dd x) { x.hi = -x.hi; x.lo = -x.lo; return x; }
static dd dd_mul(dd x, dd y) {
    double p = x.hi * y.hi;
    double e = fma(x.hi, y.hi, -p);
    e += x.hi * y.lo + x.lo * y.hi;
    return quick_two_sum(p, e);
}
static dd dd_div(dd x, dd y) {
    double q1 = x.hi / y.hi;
    dd r = dd_add(x, dd_neg(dd_mul((dd){q1, 0.0}, y)));
    double q2 = r.hi / y.hi;
    r = dd_add(r, dd_neg(dd_mul((dd){q2, 0.0}, y)));
    double q3 = r.hi / y.hi;
    dd q = quick_two_sum(q1, q2);
    return dd_add(q, (dd){q3, 0.0});
}
static dd dd_sqrt(dd a) {
    if (a.hi <= 0.0) return (dd){0.0, 0.0};
    double x = sqrt(a.hi);
    dd x2 = dd_mul((dd){x, 0.0}, (dd){x, 0.0});
    dd r = dd_add(a, dd_neg(x2));
    return dd_add((dd){x, 0.0}, (dd){r.hi / (2.0 * x), 0.0});
}

/* ---------------------------------------------------------------------------
 * y = A x  (plain CSR row dot products)
 * ------------------------------------------------------------------------- */
int or_spmv(or_ctx* c, const double* x, double* y) {
    for (int64_t i = 0; i < c->n; i++) {
        double s = 0.0;
        for (int64_t e = c->rp[i]; e < c->rp[i + 1]; e++) s += c->va[e] * x[c->ci[e]];
        y[i] = s;
    }
    return OR_OK;
}

/* a^T b, summed in index order (floor mode: in reverse order) */
static double dot(const or_ctx* c, int64_t n, const double* a, const double* b) {
    double s = 0.0;
    if (c->perturb)
        for (int64_t i = n - 1; i >= 0; i--) s += a[i] * b[i];
    else
        for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* ---------------------------------------------------------------------------
 * Step 2: overlap.  "expanding the partition to include nodes within graph
 * distance Delta in the graph defined by A".  Breadth-first
 * level sets over the off-diagonal pattern of A; result sorted.
 * ------------------------------------------------------------------------- */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

static int build_overlap(or_ctx* c) {
    int64_t n = c->n;
    int32_t* mark;   /* mark[v] = 1 + id of last subdomain that took v */
    int32_t* list;
    ALLOC(mark, n);
    ALLOC(list, n);
    /* first pass: sizes, second pass: fill */
    ALLOC(c->optr, c->nparts + 1);
    int64_t total = 0;
    int32_t** lists = calloc((size_t)c->nparts, sizeof(int32_t*));
    int64_t* sizes = calloc((size_t)c->nparts, sizeof(int64_t));
    if (!lists || !sizes) return fail(OR_E_OOM, "oom overlap");
    for (int32_t I = 0; I < c->nparts; I++) {
        int64_t cnt = 0;
        for (int64_t a = c->bptr[I]; a < c->bptr[I + 1]; a++) {
            list[cnt++] = c->bidx[a];
            mark[c->bidx[a]] = I + 1;
        }
        int64_t lev_begin = 0, lev_end = cnt;
        for (int d = 0; d < c->overlap; d++) {
            for (int64_t a = lev_begin; a < lev_end; a++) {
                int32_t v = list[a];
                for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) {
                    int32_t u = c->ci[e];
                    if (u == v || mark[u] == I + 1) continue;
                    mark[u] = I + 1;
                    list[cnt++] = u;
                }
            }
            lev_begin = lev_end;
            lev_end = cnt;
        }
        qsort(list, (size_t)cnt, sizeof(int32_t), cmp_i32);
        lists[I] = malloc((size_t)cnt * sizeof(int32_t));
        if (!lists[I]) return fail(OR_E_OOM, "oom overlap list");
        memcpy(lists[I], list, (size_t)cnt * sizeof(int32_t));
        sizes[I] = cnt;
        total += cnt;
    }
    ALLOC(c->oidx, total);
    c->optr[0] = 0;
    for (int32_t I = 0; I < c->nparts; I++) {
        c->optr[I + 1] = c->optr[I] + sizes[I];
        memcpy(c->oidx + c->optr[I], lists[I], (size_t)sizes[I] * sizeof(int32_t));
        free(lists[I]);
    }
    free(lists); free(sizes); free(mark); free(list);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 3: colours and sweep order (reading R3).  The paper iterates "over all
 * subdomains" one at a time.  The order used is: subdomains
 * sorted by (colour, id), colours from greedy first-fit over increasing id,
 * where i and j conflict iff Omega~_i intersects Omega~_j or its neighbourhood
 * N(Omega~_j).  The oracle still processes this order strictly sequentially.
 * ------------------------------------------------------------------------- */
static int build_colours(or_ctx* c) {
    int64_t n = c->n;
    int np = c->nparts;
    /* cover lists: subdomains containing node v */
    int64_t* cptr_;
    int32_t* cidx;
    ALLOC(cptr_, n + 1);
    for (int64_t a = 0; a < c->optr[np]; a++) cptr_[c->oidx[a] + 1]++;
    for (int64_t v = 0; v < n; v++) cptr_[v + 1] += cptr_[v];
    ALLOC(cidx, c->optr[np]);
    int64_t* fill;
    ALLOC(fill, n);
    for (int32_t i = 0; i < np; i++)
        for (int64_t a = c->optr[i]; a < c->optr[i + 1]; a++) {
            int32_t v = c->oidx[a];
            cidx[cptr_[v] + fill[v]++] = i;
        }
    ALLOC(c->colour, np);
    for (int32_t i = 0; i < np; i++) c->colour[i] = -1;
    int32_t* vmark;
    ALLOC(vmark, n);
    int maxc = 0;
    int cap = 64;
    char* used = calloc((size_t)cap, 1);
    for (int32_t i = 0; i < np; i++) {
        memset(used, 0, (size_t)cap);
        if (c->colour_in) {
            /* caller's colouring: check it with the same conflict rule
               (Omega~_i meets Omega~_j or its neighbours, reading R3) */
            if (c->colour_in[i] < 0 || c->colour_in[i] >= np) {
                free(used); free(vmark); free(cptr_); free(cidx); free(fill);
                return fail(OR_E_COLOURING, "colour %d of subdomain %d outside [0,%d)", c->colour_in[i], i, np);
            }
            for (int64_t a = c->optr[i]; a < c->optr[i + 1]; a++) {
                int32_t v = c->oidx[a];
                for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++)
                    for (int64_t t = cptr_[c->ci[e]]; t < cptr_[c->ci[e] + 1]; t++) {
                        int32_t j = cidx[t];
                        if (j != i && c->colour_in[j] == c->colour_in[i]) {
                            free(used); free(vmark); free(cptr_); free(cidx); free(fill);
                            return fail(OR_E_COLOURING, "subdomains %d and %d are coupled but share colour %d",
                                        i, j, c->colour_in[i]);
                        }
                    }
            }
            c->colour[i] = c->colour_in[i];
            if (c->colour[i] + 1 > maxc) maxc = c->colour[i] + 1;
            continue;
        }
        /* nodes of Omega~_i and their neighbours */
        for (int64_t a = c->optr[i]; a < c->optr[i + 1]; a++) {
            int32_t v = c->oidx[a];
            for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) {
                int32_t u = c->ci[e];
                if (vmark[u] == i + 1) continue;
                vmark[u] = i + 1;
                for (int64_t t = cptr_[u]; t < cptr_[u + 1]; t++) {
                    int32_t j = cidx[t];
                    if (j != i && c->colour[j] >= 0) {
                        if (c->colour[j] >= cap) {
                            int ncap = 2 * c->colour[j] + 2;
                            used = realloc(used, (size_t)ncap);
                            memset(used + cap, 0, (size_t)(ncap - cap));
                            cap = ncap;
                        }
                        used[c->colour[j]] = 1;
                    }
                }
            }
        }
        int col = 0;
        while (col < cap && used[col]) col++;
        c->colour[i] = col;
        if (col + 1 > maxc) maxc = col + 1;
        if (maxc >= cap) {
            used = realloc(used, (size_t)(2 * cap));
            memset(used + cap, 0, (size_t)cap);
            cap *= 2;
        }
    }
    c->ncolours = maxc;
    ALLOC(c->order, np);
    int64_t pos = 0;
    for (int col = 0; col < maxc; col++)
        for (int32_t i = 0; i < np; i++)
            if (c->colour[i] == col) c->order[pos++] = i;
    free(used); free(vmark); free(cptr_); free(cidx); free(fill);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 4: local matrices A_i = R~_i A R~_i^T, exact solves via
 * dense Cholesky A_i = L_i L_i^T (Cholesky-Banachiewicz, row by row).
 * ------------------------------------------------------------------------- */
static int chol_packed(double* L, int64_t m, int32_t blk) {
    for (int64_t i = 0; i < m; i++) {
        double* Li = L + i * (i + 1) / 2;
        for (int64_t j = 0; j <= i; j++) {
            double* Lj = L + j * (j + 1) / 2;
            double s = Li[j];
            for (int64_t t = 0; t < j; t++) s -= Li[t] * Lj[t];
            if (i == j) {
                if (!(s > 0.0))
                    return fail(OR_E_NOT_SPD,
                                "local factor: subdomain %d not positive definite at pivot %lld (%.3e)",
                                blk, (long long)i, s);
                Li[i] = sqrt(s);
            } else {
                Li[j] = s / Lj[j];
            }
        }
    }
    return OR_OK;
}

static void chol_solve_packed(const double* L, int64_t m, double* x) {
    for (int64_t i = 0; i < m; i++) { /* L y = b */
        const double* Li = L + i * (i + 1) / 2;
        double s = x[i];
        for (int64_t t = 0; t < i; t++) s -= Li[t] * x[t];
        x[i] = s / Li[i];
    }
    for (int64_t i = m - 1; i >= 0; i--) { /* L^T x = y */
        const double* Li = L + i * (i + 1) / 2;
        x[i] /= Li[i];
        for (int64_t t = 0; t < i; t++) x[t] -= Li[t] * x[i];
    }
}

static int build_local(or_ctx* c) {
    int np = c->nparts;
    ALLOC(c->loff, np + 1);
    for (int32_t i = 0; i < np; i++) {
        int64_t m = c->optr[i + 1] - c->optr[i];
        c->loff[i + 1] = c->loff[i] + m * (m + 1) / 2;
    }
    ALLOC(c->L, c->loff[np]);
    int32_t* pos;
    ALLOC(pos, c->n);
    for (int64_t v = 0; v < c->n; v++) pos[v] = -1;
    for (int32_t i = 0; i < np; i++) {
        int64_t m = c->optr[i + 1] - c->optr[i];
        const int32_t* idx = c->oidx + c->optr[i];
        for (int64_t a = 0; a < m; a++) pos[idx[a]] = (int32_t)a;
        double* L = c->L + c->loff[i];
        for (int64_t a = 0; a < m; a++) {
            int32_t v = idx[a];
            for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) {
                int32_t b = pos[c->ci[e]];
                if (c->perturb) {                 /* floor mode: unknowns reversed */
                    if (b >= 0 && b >= a) L[(m - 1 - a) * (m - a) / 2 + (m - 1 - b)] = c->va[e];
                } else if (b >= 0 && b <= a) {
                    L[a * (a + 1) / 2 + b] = c->va[e];
                }
            }
        }
        int st = chol_packed(L, m, i);
        for (int64_t a = 0; a < m; a++) pos[idx[a]] = -1;
        if (st) { free(pos); return st; }
    }
    free(pos);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 5: coarse basis.  phi_I = R_I^T R_I F: F restricted
 * to part I; orthogonalised per part; columns for which
 * phi_I is not of full rank discarded.  Modified
 * Gram-Schmidt in double-double over the columns in their given (graded-lex)
 * order; column j kept iff ||v_j|| >= rank_tol * ||F_I e_j||  (R7: the part
 * of column j not in the span of the earlier columns, relative to the column
 * itself, so the test does not depend on how the coordinates are scaled).
 * ------------------------------------------------------------------------- */
static int build_basis(or_ctx* c, const double* F) {
    int np = c->nparts, k = c->k;
    ALLOC(c->cptr, np + 1);
    ALLOC(c->qoff, np + 1);
    int64_t qtotal = 0;
    for (int32_t I = 0; I < np; I++) qtotal += (c->bptr[I + 1] - c->bptr[I]) * (int64_t)k;
    ALLOC(c->Q, qtotal);
    int64_t mmax = 0;
    for (int32_t I = 0; I < np; I++)
        if (c->bptr[I + 1] - c->bptr[I] > mmax) mmax = c->bptr[I + 1] - c->bptr[I];
    dd* V;  /* kept q vectors of this part, dd, column-major mI x k */
    dd* v;
    double* fnrm;  /* ||F_I e_j|| */
    ALLOC(V, mmax * k);
    ALLOC(v, mmax);
    ALLOC(fnrm, k);
    c->dropped = 0;
    c->min_ratio = INFINITY;
    int64_t qpos = 0;
    for (int32_t I = 0; I < np; I++) {
        int64_t mI = c->bptr[I + 1] - c->bptr[I];
        const int32_t* rows = c->bidx + c->bptr[I];
        double fmax = 0.0;
        for (int j = 0; j < k; j++) {
            dd s = {0.0, 0.0};
            for (int64_t a = 0; a < mI; a++) {
                double x = F[(int64_t)j * c->n + rows[a]];
                s = dd_add(s, dd_mul((dd){x, 0.0}, (dd){x, 0.0}));
            }
            fnrm[j] = dd_sqrt(s).hi;
            if (fnrm[j] > fmax) fmax = fnrm[j];
        }
        if (!(fmax > 0.0))
            return fail(OR_E_ZERO_BLOCK, "coarse basis: F restricted to part %d is zero", I);
        int r = 0;
        for (int j = 0; j < k; j++) {
            const double ref = fnrm[j];
            for (int64_t a = 0; a < mI; a++) v[a] = (dd){F[(int64_t)j * c->n + rows[a]], 0.0};
            for (int t = 0; t < r; t++) { /* MGS: v -= (q_t^T v) q_t */
                dd* q = V + (int64_t)t * mI;
                dd s = {0.0, 0.0};
                for (int64_t a = 0; a < mI; a++) s = dd_add(s, dd_mul(q[a], v[a]));
                for (int64_t a = 0; a < mI; a++) v[a] = dd_add(v[a], dd_neg(dd_mul(s, q[a])));
            }
            dd s = {0.0, 0.0};
            for (int64_t a = 0; a < mI; a++) s = dd_add(s, dd_mul(v[a], v[a]));
            dd nrm = dd_sqrt(s);
            double ratio = ref > 0.0 ? nrm.hi / ref : 0.0;
            if (ratio >= c->rank_tol && nrm.hi > 0.0) {
                dd* q = V + (int64_t)r * mI;
                for (int64_t a = 0; a < mI; a++) q[a] = dd_div(v[a], nrm);
                if (ratio < c->min_ratio) c->min_ratio = ratio;
                r++;
            } else {
                c->dropped++;
            }
        }
        c->qoff[I] = qpos;
        for (int t = 0; t < r; t++)
            for (int64_t a = 0; a < mI; a++) c->Q[qpos + (int64_t)t * mI + a] = V[(int64_t)t * mI + a].hi;
        qpos += (int64_t)r * mI;
        c->cptr[I + 1] = c->cptr[I] + r;
    }
    c->qoff[np] = qpos;
    c->nc = c->cptr[np];
    ALLOC(c->cpart, c->nc);
    for (int32_t I = 0; I < np; I++)
        for (int32_t i = c->cptr[I]; i < c->cptr[I + 1]; i++) c->cpart[i] = I;
    free(V); free(v); free(fnrm);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 6: A_0 = R_0 A R_0^T.  Column (J,j) of A_0 is
 * P^T (A p_{J,j}); (A p)[u] = sum_c A[u,c] p[c] evaluated for every row u that
 * can be non-zero (rows in Omega_J and its neighbours).  A_0 is stored by
 * blocks: "the same sparsity pattern as the subdomain adjacency matrix, but
 * with each non-zero replaced with a small dense block".
 * A_0 is symmetric: only entries with row >= column are computed (R9).
 * ------------------------------------------------------------------------- */
static int64_t blk_find(const or_ctx* c, int32_t I, int32_t J) {
    int64_t lo = c->aptr[I], hi = c->aptr[I + 1];
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (c->aadj[mid] < J) lo = mid + 1; else hi = mid;
    }
    return (lo < c->aptr[I + 1] && c->aadj[lo] == J) ? lo : -1;
}

/* A_0[ci, cj] for ci >= cj */
static double a0_entry(const or_ctx* c, int64_t ci, int64_t cj) {
    int32_t I = c->cpart[ci], J = c->cpart[cj];
    int64_t e = blk_find(c, I, J);
    if (e < 0) return 0.0;
    int64_t rJ = c->cptr[J + 1] - c->cptr[J];
    return c->ablk[c->aoff[e] + (ci - c->cptr[I]) * rJ + (cj - c->cptr[J])];
}

static int build_coarse_blocks(or_ctx* c) {
    int np = c->nparts;
    int64_t n = c->n;
    /* block pattern: parts J <= I coupled to I by an entry of A */
    int32_t* mark;
    int32_t* nb;
    ALLOC(mark, np);
    ALLOC(nb, np);
    ALLOC(c->aptr, np + 1);
    for (int pass = 0; pass < 2; pass++) {
        for (int32_t I = 0; I < np; I++) mark[I] = -1;
        for (int32_t I = 0; I < np; I++) {
            int cnt = 0;
            for (int64_t a = c->bptr[I]; a < c->bptr[I + 1]; a++) {
                int32_t v = c->bidx[a];
                for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) {
                    int32_t J = c->part[c->ci[e]];
                    if (J <= I && mark[J] != I) { mark[J] = I; nb[cnt++] = J; }
                }
            }
            if (mark[I] != I) { mark[I] = I; nb[cnt++] = I; }
            if (pass == 0) {
                c->aptr[I + 1] = c->aptr[I] + cnt;
            } else {
                qsort(nb, (size_t)cnt, sizeof(int32_t), cmp_i32);
                memcpy(c->aadj + c->aptr[I], nb, (size_t)cnt * sizeof(int32_t));
            }
        }
        if (pass == 0) ALLOC(c->aadj, c->aptr[np]);
    }
    free(mark); free(nb);
    ALLOC(c->aoff, c->aptr[np] + 1);
    for (int32_t I = 0; I < np; I++)
        for (int64_t e = c->aptr[I]; e < c->aptr[I + 1]; e++) {
            int32_t J = c->aadj[e];
            c->aoff[e + 1] = c->aoff[e] + (int64_t)(c->cptr[I + 1] - c->cptr[I]) * (c->cptr[J + 1] - c->cptr[J]);
        }
    ALLOC(c->ablk, c->aoff[c->aptr[np]]);
    double* w;
    double* p;
    int32_t* touched;
    char* tmark;
    ALLOC(w, n);
    ALLOC(p, n);
    ALLOC(touched, n);
    ALLOC(tmark, n);
    for (int32_t J = 0; J < np; J++) {
        int64_t mJ = c->bptr[J + 1] - c->bptr[J];
        int64_t rJ = c->cptr[J + 1] - c->cptr[J];
        const int32_t* rowsJ = c->bidx + c->bptr[J];
        /* rows where A p can be non-zero */
        int64_t nt = 0;
        for (int64_t a = 0; a < mJ; a++) {
            int32_t v = rowsJ[a];
            for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) {
                int32_t u = c->ci[e];
                if (!tmark[u]) { tmark[u] = 1; touched[nt++] = u; }
            }
        }
        for (int32_t j = 0; j < rJ; j++) {
            int64_t cj = c->cptr[J] + j;
            const double* qJ = c->Q + c->qoff[J] + (int64_t)j * mJ;
            for (int64_t a = 0; a < mJ; a++) p[rowsJ[a]] = qJ[a];
            for (int64_t t = 0; t < nt; t++) {
                int32_t u = touched[t];
                double s = 0.0;
                for (int64_t e = c->rp[u]; e < c->rp[u + 1]; e++) s += c->va[e] * p[c->ci[e]];
                w[u] = s;
            }
            /* A_0[(I,i),(J,j)] = Q_I[:,i]^T w[Omega_I] for parts I touched */
            for (int64_t t = 0; t < nt; t++) {
                int32_t u = touched[t];
                int32_t I = c->part[u];
                if (I < J) continue;
                int64_t mI = c->bptr[I + 1] - c->bptr[I];
                int64_t e = blk_find(c, I, J);
                if (e < 0) return fail(OR_E_ARG, "internal: block (%d,%d) missing", I, J);
                double* blk = c->ablk + c->aoff[e];
                for (int32_t i = 0; i < c->cptr[I + 1] - c->cptr[I]; i++) {
                    int64_t ci_ = c->cptr[I] + i;
                    if (ci_ < cj) continue;
                    double qv = c->Q[c->qoff[I] + (int64_t)i * mI + c->bpos[u]];
                    blk[(int64_t)i * rJ + j] += qv * w[u];
                }
            }
            for (int64_t a = 0; a < mJ; a++) p[rowsJ[a]] = 0.0;
        }
        for (int64_t t = 0; t < nt; t++) tmark[touched[t]] = 0;
    }
    free(w); free(p); free(touched); free(tmark);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Step 7: Cholesky of A_0 within its envelope (exact: no fill outside it;
 * PAPER.md:267 "A_0 u_0 = R_0 f").  Envelope of row i: from the first coarse
 * unknown of the lowest-numbered part adjacent to its part.  Floor mode: the
 * same on the matrix with the coarse order reversed, x'[nc-1-i] = x[i].
 * ------------------------------------------------------------------------- */
static int build_envelope(or_ctx* c) {
    int np = c->nparts;
    int64_t nc = c->nc;
    int32_t* minadj;   /* lowest part J <= I adjacent to I */
    int32_t* maxadj;   /* highest part J >= I adjacent to I */
    ALLOC(minadj, np);
    ALLOC(maxadj, np);
    for (int32_t I = 0; I < np; I++) { minadj[I] = c->aadj[c->aptr[I]]; maxadj[I] = I; }
    for (int32_t I = 0; I < np; I++)
        for (int64_t e = c->aptr[I]; e < c->aptr[I + 1]; e++)
            if (I > maxadj[c->aadj[e]]) maxadj[c->aadj[e]] = I;
    ALLOC(c->efirst, nc);
    ALLOC(c->eptr, nc + 1);
    for (int64_t i = 0; i < nc; i++) {
        int32_t I = c->cpart[i];
        if (c->perturb) /* row nc-1-i of the reversed matrix: columns nc-1-j for j >= i */
            c->efirst[nc - 1 - i] = nc - 1 - (c->cptr[maxadj[I] + 1] - 1);
        else
            c->efirst[i] = c->cptr[minadj[I]];
    }
    free(minadj); free(maxadj);
    for (int64_t i = 0; i < nc; i++) c->eptr[i + 1] = c->eptr[i] + (i - c->efirst[i] + 1);
    ALLOC(c->el, c->eptr[nc]);
    for (int32_t I = 0; I < np; I++) {
        int64_t rI = c->cptr[I + 1] - c->cptr[I];
        for (int64_t e = c->aptr[I]; e < c->aptr[I + 1]; e++) {
            int32_t J = c->aadj[e];
            int64_t rJ = c->cptr[J + 1] - c->cptr[J];
            for (int64_t i = 0; i < rI; i++)
                for (int64_t j = 0; j < rJ; j++) {
                    int64_t ci_ = c->cptr[I] + i, cj = c->cptr[J] + j;
                    if (ci_ < cj) continue;
                    double v = c->ablk[c->aoff[e] + i * rJ + j];
                    int64_t r = ci_, col = cj;
                    if (c->perturb) { r = nc - 1 - cj; col = nc - 1 - ci_; }
                    c->el[c->eptr[r] + (col - c->efirst[r])] = v;
                }
        }
    }
    for (int64_t i = 0; i < nc; i++) {
        double* Li = c->el + c->eptr[i] - c->efirst[i]; /* Li[j] valid for j >= efirst[i] */
        for (int64_t j = c->efirst[i]; j <= i; j++) {
            double* Lj = c->el + c->eptr[j] - c->efirst[j];
            int64_t t0 = c->efirst[i] > c->efirst[j] ? c->efirst[i] : c->efirst[j];
            double s = Li[j];
            for (int64_t t = t0; t < j; t++) s -= Li[t] * Lj[t];
            if (i == j) {
                if (!(s > 0.0))
                    return fail(OR_E_NOT_SPD, "coarse factor: A_0 not positive definite at pivot %lld (%.3e)",
                                (long long)i, s);
                Li[i] = sqrt(s);
            } else {
                Li[j] = s / Lj[j];
            }
        }
    }
    return OR_OK;
}

static void coarse_solve(or_ctx* c, double* x) {
    int64_t nc = c->nc;
    if (c->perturb)
        for (int64_t i = 0; i < nc / 2; i++) { double t = x[i]; x[i] = x[nc - 1 - i]; x[nc - 1 - i] = t; }
    for (int64_t i = 0; i < nc; i++) {
        const double* Li = c->el + c->eptr[i] - c->efirst[i];
        double s = x[i];
        for (int64_t t = c->efirst[i]; t < i; t++) s -= Li[t] * x[t];
        x[i] = s / Li[i];
    }
    for (int64_t i = nc - 1; i >= 0; i--) {
        const double* Li = c->el + c->eptr[i] - c->efirst[i];
        x[i] /= Li[i];
        for (int64_t t = c->efirst[i]; t < i; t++) x[t] -= Li[t] * x[i];
    }
    if (c->perturb)
        for (int64_t i = 0; i < nc / 2; i++) { double t = x[i]; x[i] = x[nc - 1 - i]; x[nc - 1 - i] = t; }
}

/* ---------------------------------------------------------------------------
 * setup
 * ------------------------------------------------------------------------- */
static int setup_impl(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                      const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                      double rank_tol, const or_opts* o, or_ctx** out);

int or_setup(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
             const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
             double rank_tol, or_ctx** out) {
    return setup_impl(n, row_ptr, col, val, F, k, part, nparts, overlap, rank_tol, NULL, out);
}

int or_setup_coloured(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                      const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                      double rank_tol, const int32_t* colour, or_ctx** out) {
    or_opts o = {0};
    o.colour = colour;
    return setup_impl(n, row_ptr, col, val, F, k, part, nparts, overlap, rank_tol, &o, out);
}

int or_setup_ex(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                double rank_tol, const or_opts* o, or_ctx** out) {
    return setup_impl(n, row_ptr, col, val, F, k, part, nparts, overlap, rank_tol, o, out);
}

static int setup_impl(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                      const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                      double rank_tol, const or_opts* o, or_ctx** out) {
    *out = NULL;
    g_err[0] = 0;
    if (n < 1 || !row_ptr || !col || !val || !F || !part || k < 1 || nparts < 1 || overlap < 0)
        return fail(OR_E_ARG, "bad argument (n=%lld k=%d nparts=%d overlap=%d)", (long long)n, k,
                    nparts, overlap);
    if (row_ptr[0] != 0) return fail(OR_E_DIM, "row_ptr[0] != 0");
    for (int64_t i = 0; i < n; i++) {
        if (row_ptr[i + 1] < row_ptr[i]) return fail(OR_E_DIM, "row_ptr decreasing at %lld", (long long)i);
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; e++) {
            if (col[e] < 0 || col[e] >= n) return fail(OR_E_DIM, "column out of range in row %lld", (long long)i);
            if (e > row_ptr[i] && col[e] <= col[e - 1])
                return fail(OR_E_DIM, "columns not strictly increasing in row %lld", (long long)i);
        }
    }
    or_ctx* c = calloc(1, sizeof(or_ctx));
    if (!c) return fail(OR_E_OOM, "oom");
    int st;
    c->n = n; c->k = k; c->nparts = nparts; c->overlap = overlap; c->rank_tol = rank_tol;
    c->colour_in = o ? o->colour : NULL;
    c->perturb = o ? o->perturb : 0;
    c->coarse_external = o ? o->coarse_external : 0;
    int64_t nnz = row_ptr[n];
    c->rp = malloc((size_t)(n + 1) * sizeof(int64_t));
    c->ci = malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    c->va = malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
    c->part = malloc((size_t)n * sizeof(int32_t));
    if (!c->rp || !c->ci || !c->va || !c->part) { or_destroy(c); return fail(OR_E_OOM, "oom"); }
    memcpy(c->rp, row_ptr, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(c->ci, col, (size_t)nnz * sizeof(int32_t));
    memcpy(c->va, val, (size_t)nnz * sizeof(double));
    memcpy(c->part, part, (size_t)n * sizeof(int32_t));
    /* Step 1: parts Omega_I (sorted node lists) */
    c->bptr = calloc((size_t)nparts + 1, sizeof(int64_t));
    c->bidx = malloc((size_t)n * sizeof(int32_t));
    c->bpos = malloc((size_t)n * sizeof(int32_t));
    if (!c->bptr || !c->bidx || !c->bpos) { or_destroy(c); return fail(OR_E_OOM, "oom"); }
    for (int64_t v = 0; v < n; v++) {
        if (part[v] < 0 || part[v] >= nparts) {
            or_destroy(c);
            return fail(OR_E_PART, "part id %d of node %lld out of range [0,%d)", part[v], (long long)v, nparts);
        }
        c->bptr[part[v] + 1]++;
    }
    for (int32_t I = 0; I < nparts; I++) {
        if (c->bptr[I + 1] == 0) { or_destroy(c); return fail(OR_E_PART, "part %d is empty", I); }
        c->bptr[I + 1] += c->bptr[I];
    }
    {
        int64_t* fillp = calloc((size_t)nparts, sizeof(int64_t));
        for (int64_t v = 0; v < n; v++) {
            int32_t I = part[v];
            c->bpos[v] = (int32_t)fillp[I];
            c->bidx[c->bptr[I] + fillp[I]++] = (int32_t)v;
        }
        free(fillp);
    }
    if ((st = build_overlap(c)) || (st = build_colours(c)) || (st = build_local(c)) ||
        (st = build_basis(c, F)) || (st = build_coarse_blocks(c)) ||
        (!c->coarse_external && (st = build_envelope(c)))) {
        or_destroy(c);
        return st;
    }
    c->colour_in = NULL;
    *out = c;
    return OR_OK;
}

void or_destroy(or_ctx* c) {
    if (!c) return;
    free(c->rp); free(c->ci); free(c->va); free(c->part);
    free(c->bptr); free(c->bidx); free(c->bpos);
    free(c->optr); free(c->oidx); free(c->colour); free(c->order);
    free(c->loff); free(c->L);
    free(c->cptr); free(c->qoff); free(c->Q); free(c->cpart);
    free(c->aptr); free(c->aadj); free(c->aoff); free(c->ablk);
    free(c->efirst); free(c->eptr); free(c->el);
    or_destroy(c->child);
    free(c);
}

/* ---------------------------------------------------------------------------
 * Three-level method: "taking the two-level algorithm and
 * applying it again to the coarse matrix A_0 ... a coarsened version of the
 * generating vectors, which are simply F_0 = R_0 F".
 *   - A_0 as a sparse matrix: row (I,i) holds every (J,j) with J = I or J
 *     adjacent to I in the graph of A (reading R19: the structural pattern of
 *     R_0 A R_0^T, explicit zeros kept, so that the overlap and colouring of
 *     the second level follow the graph of A_0 and not cancellation).
 *   - F_0[(I,i), l] = Q_I[:, i]^T F[Omega_I, l]   (R_0 = blockdiag(Q_I^T)).
 *   - second-level partition: coarse unknown (I,i) belongs to part
 *     part2[I] (reading R20: whole fine parts are grouped, which keeps
 *     h/H_0 = H_0/H_1 when part2 groups (H/h)^d neighbouring parts).
 *   - the same Delta and rank tolerance at both levels.
 * ------------------------------------------------------------------------- */
int or_setup3(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
              double rank_tol, const int32_t* part2, int32_t nparts2, or_ctx** out) {
    *out = NULL;
    if (!part2 || nparts2 < 1) return fail(OR_E_ARG, "three levels need a second-level partition");
    for (int32_t I = 0; I < nparts; I++)
        if (part2[I] < 0 || part2[I] >= nparts2)
            return fail(OR_E_PART, "second-level part %d of part %d out of range [0,%d)", part2[I], I, nparts2);
    or_ctx* c;
    int st = or_setup(n, row_ptr, col, val, F, k, part, nparts, overlap, rank_tol, &c);
    if (st) return st;
    int64_t nc = c->nc;
    /* part adjacency in the graph of A */
    char* adj = calloc((size_t)nparts * (size_t)nparts, 1);
    int64_t* rp0 = calloc((size_t)nc + 1, sizeof(int64_t));
    double* F0 = calloc((size_t)(nc > 0 ? nc : 1) * (size_t)k, sizeof(double));
    int32_t* p0 = calloc((size_t)(nc > 0 ? nc : 1), sizeof(int32_t));
    if (!adj || !rp0 || !F0 || !p0) {
        free(adj); free(rp0); free(F0); free(p0); or_destroy(c);
        return fail(OR_E_OOM, "oom");
    }
    for (int64_t v = 0; v < n; v++)
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
            int32_t I = part[v], J = part[col[e]];
            adj[(size_t)I * nparts + J] = adj[(size_t)J * nparts + I] = 1;
        }
    for (int32_t I = 0; I < nparts; I++) adj[(size_t)I * nparts + I] = 1;
    for (int32_t I = 0; I < nparts; I++) {
        int64_t w = 0;
        for (int32_t J = 0; J < nparts; J++)
            if (adj[(size_t)I * nparts + J]) w += c->cptr[J + 1] - c->cptr[J];
        for (int32_t i = c->cptr[I]; i < c->cptr[I + 1]; i++) rp0[i + 1] = w;
    }
    for (int64_t i = 0; i < nc; i++) rp0[i + 1] += rp0[i];
    int32_t* ci0 = malloc((size_t)(rp0[nc] > 0 ? rp0[nc] : 1) * sizeof(int32_t));
    double* va0 = malloc((size_t)(rp0[nc] > 0 ? rp0[nc] : 1) * sizeof(double));
    if (!ci0 || !va0) {
        free(adj); free(rp0); free(F0); free(p0); free(ci0); free(va0); or_destroy(c);
        return fail(OR_E_OOM, "oom");
    }
    for (int32_t I = 0; I < nparts; I++)
        for (int32_t i = c->cptr[I]; i < c->cptr[I + 1]; i++) {
            int64_t e = rp0[i];
            for (int32_t J = 0; J < nparts; J++) {
                if (!adj[(size_t)I * nparts + J]) continue;
                for (int32_t j = c->cptr[J]; j < c->cptr[J + 1]; j++) {
                    /* A_0 is kept lower in the envelope: (max, min) */
                    int64_t hi = i > j ? i : j, lo = i > j ? j : i;
                    ci0[e] = j;
                    va0[e++] = a0_entry(c, hi, lo);
                }
            }
            p0[i] = part2[I];
        }
    /* F_0 = R_0 F (column-major nc x k) */
    for (int32_t I = 0; I < nparts; I++) {
        int64_t mI = c->bptr[I + 1] - c->bptr[I];
        const int32_t* rows = c->bidx + c->bptr[I];
        for (int32_t i = 0; i < c->cptr[I + 1] - c->cptr[I]; i++) {
            const double* q = c->Q + c->qoff[I] + (int64_t)i * mI;
            for (int l = 0; l < k; l++) {
                double s = 0.0;
                for (int64_t a = 0; a < mI; a++) s += q[a] * F[(int64_t)l * n + rows[a]];
                F0[(int64_t)l * nc + c->cptr[I] + i] = s;
            }
        }
    }
    free(adj);
    if (nc < 1) {
        free(rp0); free(F0); free(p0); free(ci0); free(va0); or_destroy(c);
        return fail(OR_E_ARG, "empty coarse space");
    }
    /* every second-level part must own coarse unknowns */
    st = or_setup(nc, rp0, ci0, va0, F0, k, p0, nparts2, overlap, rank_tol, &c->child);
    free(rp0); free(F0); free(p0); free(ci0); free(va0);
    if (st) { or_destroy(c); return st; }
    *out = c;
    return OR_OK;
}

or_ctx* or_child(or_ctx* c) { return c->child; }

/* ---------------------------------------------------------------------------
 * Subdomain update:  u <- u + R~_i^T A_i^{-1} R~_i (f - A u),
 * the residual restricted to Omega~_i recomputed from the current iterate.
 * ------------------------------------------------------------------------- */
static void subdomain_update(or_ctx* c, int32_t i, const double* r, double* z, double* s) {
    int64_t m = c->optr[i + 1] - c->optr[i];
    const int32_t* idx = c->oidx + c->optr[i];
    for (int64_t a = 0; a < m; a++) {
        int32_t v = idx[a];
        double az = 0.0;
        for (int64_t e = c->rp[v]; e < c->rp[v + 1]; e++) az += c->va[e] * z[c->ci[e]];
        s[a] = r[v] - az;
    }
    if (c->perturb) { /* floor mode: the factor holds the reversed ordering */
        for (int64_t a = 0; a < m / 2; a++) { double t = s[a]; s[a] = s[m - 1 - a]; s[m - 1 - a] = t; }
        chol_solve_packed(c->L + c->loff[i], m, s);
        for (int64_t a = 0; a < m / 2; a++) { double t = s[a]; s[a] = s[m - 1 - a]; s[m - 1 - a] = t; }
    } else {
        chol_solve_packed(c->L + c->loff[i], m, s);
    }
    for (int64_t a = 0; a < m; a++) z[idx[a]] += s[a];
}

static int64_t max_m(or_ctx* c) {
    int64_t mm = 0;
    for (int32_t i = 0; i < c->nparts; i++)
        if (c->optr[i + 1] - c->optr[i] > mm) mm = c->optr[i + 1] - c->optr[i];
    return mm;
}

/* one forward pass of one-level multiplicative Schwarz from z = 0 (test hook) */
int or_forward_sweep(or_ctx* c, const double* r, double* z) {
    double* s = malloc((size_t)max_m(c) * sizeof(double));
    if (!s) return fail(OR_E_OOM, "oom");
    memset(z, 0, (size_t)c->n * sizeof(double));
    for (int32_t t = 0; t < c->nparts; t++) subdomain_update(c, c->order[t], r, z, s);
    free(s);
    return OR_OK;
}

/* coarse correction R_0^T A_0^{-1} R_0 r added into z */
static void coarse_add(or_ctx* c, const double* res, double* z) {
    double* b = malloc((size_t)(c->nc > 0 ? c->nc : 1) * sizeof(double));
    for (int32_t I = 0; I < c->nparts; I++) {
        int64_t mI = c->bptr[I + 1] - c->bptr[I];
        const int32_t* rows = c->bidx + c->bptr[I];
        for (int32_t i = 0; i < c->cptr[I + 1] - c->cptr[I]; i++) {
            const double* q = c->Q + c->qoff[I] + (int64_t)i * mI;
            double s = 0.0;
            for (int64_t a = 0; a < mI; a++) s += q[a] * res[rows[a]];
            b[c->cptr[I] + i] = s;
        }
    }
    if (c->child) {
        /* three levels: one V-cycle of the two-level method on A_0 stands in
           for A_0^{-1} */
        double* y = malloc((size_t)(c->nc > 0 ? c->nc : 1) * sizeof(double));
        or_apply_precond(c->child, b, y);
        memcpy(b, y, (size_t)c->nc * sizeof(double));
        free(y);
    } else if (c->coarse_external) {
        c->ext_fn(c->ext_user, c->nc, b);
    } else {
        coarse_solve(c, b);
    }
    for (int32_t I = 0; I < c->nparts; I++) {
        int64_t mI = c->bptr[I + 1] - c->bptr[I];
        const int32_t* rows = c->bidx + c->bptr[I];
        for (int32_t i = 0; i < c->cptr[I + 1] - c->cptr[I]; i++) {
            const double* q = c->Q + c->qoff[I] + (int64_t)i * mI;
            double y = b[c->cptr[I] + i];
            for (int64_t a = 0; a < mI; a++) z[rows[a]] += q[a] * y;
        }
    }
    free(b);
}

int or_coarse_correct(or_ctx* c, const double* r, double* z) {
    if (c->coarse_external && !c->ext_fn) return fail(OR_E_ARG, "external coarse solver not set");
    memset(z, 0, (size_t)c->n * sizeof(double));
    coarse_add(c, r, z);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Two-level symmetric multiplicative preconditioner z = M r:
 * zero initial guess; one pass over the subdomains (pre-smoother); the coarse
 * problem solution on the current residual; another pass in reverse order.
 * ------------------------------------------------------------------------- */
int or_apply_precond(or_ctx* c, const double* r, double* z) {
    int64_t n = c->n;
    if (c->coarse_external && !c->ext_fn) return fail(OR_E_ARG, "external coarse solver not set");
    double* s = malloc((size_t)max_m(c) * sizeof(double));
    double* res = malloc((size_t)n * sizeof(double));
    if (!s || !res) { free(s); free(res); return fail(OR_E_OOM, "oom"); }
    memset(z, 0, (size_t)n * sizeof(double));
    for (int32_t t = 0; t < c->nparts; t++) subdomain_update(c, c->order[t], r, z, s);
    or_spmv(c, z, res);
    for (int64_t v = 0; v < n; v++) res[v] = r[v] - res[v];
    coarse_add(c, res, z);
    for (int32_t t = c->nparts - 1; t >= 0; t--) subdomain_update(c, c->order[t], r, z, s);
    free(s); free(res);
    return OR_OK;
}

/* ---------------------------------------------------------------------------
 * Preconditioned CG (Hestenes-Stiefel) from u_0 = 0.
 * hist[j] = ||r_j||_2 (recurrence residual, reading R2); iterations = number of
 * A p products (R16).  stop_mode: 0 ||r_k|| <= rtol ||r_0||; 1 <= rtol ||r_1||
 * (SPEC.md:398); 2 sqrt(r_k^T z_k) <= rtol sqrt(r_0^T z_0)  (reading R1).
 * ------------------------------------------------------------------------- */
/* PCG as in or_pcg, also recording the CG coefficients alpha_k, beta_k
 * ("condition number estimates derived from the Lanczos
 * coefficients computed during CG"); alphas/betas may be NULL. */
int or_pcg_ab(or_ctx* c, const double* f, double rtol, int max_iter, int stop_mode, double* u,
              int* iters, double* hist, int* converged, double* alphas, double* betas);
int or_pcg(or_ctx* c, const double* f, double rtol, int max_iter, int stop_mode, double* u,
           int* iters, double* hist, int* converged) {
    return or_pcg_ab(c, f, rtol, max_iter, stop_mode, u, iters, hist, converged, NULL, NULL);
}

int or_pcg_ab(or_ctx* c, const double* f, double rtol, int max_iter, int stop_mode, double* u,
              int* iters, double* hist, int* converged, double* alphas, double* betas) {
    int64_t n = c->n;
    double *r = malloc(n * sizeof(double)), *z = malloc(n * sizeof(double)),
           *p = malloc(n * sizeof(double)), *q = malloc(n * sizeof(double));
    if (!r || !z || !p || !q) return fail(OR_E_OOM, "oom");
    int st = OR_OK;
    *converged = 0;
    *iters = 0;
    memset(u, 0, (size_t)n * sizeof(double));
    memcpy(r, f, (size_t)n * sizeof(double));
    double res0 = sqrt(dot(c, n, r, r));
    hist[0] = res0;
    if (res0 == 0.0) { *converged = 1; goto done; }
    or_apply_precond(c, r, z);
    memcpy(p, z, (size_t)n * sizeof(double));
    double rho = dot(c, n, r, z);
    if (!(rho > 0.0)) { st = fail(OR_E_BREAKDOWN, "r^T z <= 0 at iteration 0"); goto done; }
    double pres0 = sqrt(rho), ref = res0;
    for (int it = 0; it < max_iter; it++) {
        or_spmv(c, p, q);
        double sigma = dot(c, n, p, q);
        if (!(sigma > 0.0)) { st = fail(OR_E_BREAKDOWN, "p^T A p <= 0 at iteration %d", it); goto done; }
        double alpha = rho / sigma;
        if (alphas) alphas[it] = alpha;
        for (int64_t v = 0; v < n; v++) { u[v] += alpha * p[v]; r[v] -= alpha * q[v]; }
        double res = sqrt(dot(c, n, r, r));
        hist[it + 1] = res;
        *iters = it + 1;
        if (stop_mode == 1 && it == 0) ref = res;
        if (stop_mode != 2 && res <= rtol * ref && !(stop_mode == 1 && it == 0)) { *converged = 1; break; }
        if (res == 0.0) { *converged = 1; break; }
        or_apply_precond(c, r, z);
        double rho1 = dot(c, n, r, z);
        if (stop_mode == 2 && sqrt(fabs(rho1)) <= rtol * pres0) { *converged = 1; break; }
        if (!(rho1 > 0.0)) { st = fail(OR_E_BREAKDOWN, "r^T z <= 0 at iteration %d", it + 1); goto done; }
        double beta = rho1 / rho;
        if (betas) betas[it] = beta;
        rho = rho1;
        for (int64_t v = 0; v < n; v++) p[v] = z[v] + beta * p[v];
    }
done:
    free(r); free(z); free(p); free(q);
    return st;
}

/* ---------------------------------------------------------------------------
 * accessors for tests
 * ------------------------------------------------------------------------- */
void or_info(or_ctx* c, int64_t* info) {
    int64_t mmin = INT64_MAX, mmax = 0;
    for (int32_t i = 0; i < c->nparts; i++) {
        int64_t m = c->optr[i + 1] - c->optr[i];
        if (m < mmin) mmin = m;
        if (m > mmax) mmax = m;
    }
    info[0] = c->n; info[1] = c->nc; info[2] = c->nparts; info[3] = c->ncolours;
    info[4] = mmin; info[5] = mmax; info[6] = c->k; info[7] = c->dropped;
    info[8] = c->child ? 3 : 2; info[9] = c->child ? c->child->nc : 0;
}
double or_min_rank_ratio(or_ctx* c) { return c->min_ratio; }
int or_get_colours(or_ctx* c, int32_t* colour) {
    memcpy(colour, c->colour, (size_t)c->nparts * sizeof(int32_t));
    return OR_OK;
}
int64_t or_get_overlap(or_ctx* c, int32_t i, int32_t* idx) {
    if (i < 0 || i >= c->nparts) return -1;
    int64_t m = c->optr[i + 1] - c->optr[i];
    if (idx) memcpy(idx, c->oidx + c->optr[i], (size_t)m * sizeof(int32_t));
    return m;
}
int or_get_P_dense(or_ctx* c, double* P) {
    memset(P, 0, (size_t)(c->n * c->nc) * sizeof(double));
    for (int32_t I = 0; I < c->nparts; I++) {
        int64_t mI = c->bptr[I + 1] - c->bptr[I];
        for (int32_t i = 0; i < c->cptr[I + 1] - c->cptr[I]; i++)
            for (int64_t a = 0; a < mI; a++)
                P[(int64_t)(c->cptr[I] + i) * c->n + c->bidx[c->bptr[I] + a]] =
                    c->Q[c->qoff[I] + (int64_t)i * mI + a];
    }
    return OR_OK;
}
int or_get_Ac_dense(or_ctx* c, double* Ac) {
    int64_t nc = c->nc;
    memset(Ac, 0, (size_t)(nc * nc) * sizeof(double));
    for (int64_t i = 0; i < nc; i++)
        for (int64_t j = 0; j <= i; j++) {
            double v = a0_entry(c, i, j);
            Ac[i * nc + j] = v;
            Ac[j * nc + i] = v;
        }
    return OR_OK;
}

/* A_0 as a full symmetric CSR (rows and columns in coarse order, columns
   ascending); with rp == NULL only the entry count is returned */
int64_t or_get_Ac_csr(or_ctx* c, int64_t* rp, int32_t* col, double* val) {
    int np = c->nparts;
    /* full block adjacency: lower part from aadj, upper part by symmetry */
    int64_t* fptr = calloc((size_t)np + 1, sizeof(int64_t));
    if (!fptr) return -1;
    for (int32_t I = 0; I < np; I++)
        for (int64_t e = c->aptr[I]; e < c->aptr[I + 1]; e++) {
            fptr[I + 1]++;
            if (c->aadj[e] != I) fptr[c->aadj[e] + 1]++;
        }
    for (int32_t I = 0; I < np; I++) fptr[I + 1] += fptr[I];
    int32_t* fadj = malloc((size_t)(fptr[np] > 0 ? fptr[np] : 1) * sizeof(int32_t));
    int64_t* fill = calloc((size_t)np, sizeof(int64_t));
    if (!fadj || !fill) { free(fptr); free(fadj); free(fill); return -1; }
    for (int32_t I = 0; I < np; I++)   /* I ascending: each list comes out sorted */
        for (int64_t e = c->aptr[I]; e < c->aptr[I + 1]; e++) {
            int32_t J = c->aadj[e];
            fadj[fptr[I] + fill[I]++] = J;
            if (J != I) fadj[fptr[J] + fill[J]++] = I;
        }
    for (int32_t I = 0; I < np; I++)
        qsort(fadj + fptr[I], (size_t)(fptr[I + 1] - fptr[I]), sizeof(int32_t), cmp_i32);
    int64_t nnz = 0;
    if (rp) rp[0] = 0;
    for (int32_t I = 0; I < np; I++)
        for (int32_t i = c->cptr[I]; i < c->cptr[I + 1]; i++) {
            for (int64_t e = fptr[I]; e < fptr[I + 1]; e++) {
                int32_t J = fadj[e];
                for (int32_t j = c->cptr[J]; j < c->cptr[J + 1]; j++) {
                    if (rp) {
                        col[nnz] = j;
                        val[nnz] = i >= j ? a0_entry(c, i, j) : a0_entry(c, j, i);
                    }
                    nnz++;
                }
            }
            if (rp) rp[i + 1] = nnz;
        }
    free(fptr); free(fadj); free(fill);
    return nnz;
}

void or_set_coarse_solver(or_ctx* c, or_coarse_fn fn, void* user) {
    c->ext_fn = fn;
    c->ext_user = user;
}
int or_get_coarse_offsets(or_ctx* c, int32_t* cptr) {
    memcpy(cptr, c->cptr, (size_t)(c->nparts + 1) * sizeof(int32_t));
    return OR_OK;
}
