/*
 * oracle.h — CPU ORACLE for the DDG-preconditioned CG path.
 *
 * TEST INFRASTRUCTURE ONLY.  This code is the slow, plain, single-threaded
 * fp64 definition of what the CUDA path computes, written from PAPER.md
 * (arXiv:1504.00907).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code,
 * header or helper with the product (paper_1504_00907_b200/, include/ddg.h).
 *
 * Parity pins: see tests/test_oracle_*.py and DESIGN.md §"Oracle pins".
 */
#ifndef DDG_ORACLE_H
#define DDG_ORACLE_H
#include <stdint.h>

typedef struct or_ctx or_ctx;

/* x <- A_0^{-1} x in place (an external exact coarse solve) */
typedef void (*or_coarse_fn)(void* user, int64_t nc, double* x);

typedef struct {
    const int32_t* colour; /* caller's colouring (as or_setup_coloured) or NULL */
    int perturb;           /* floor mode: reversed dot order, reversed local and
                              coarse elimination order */
    int coarse_external;   /* 1: no envelope factor of A_0; the caller supplies
                              A_0^{-1} with or_set_coarse_solver (oracle/coarse_nd.py) */
} or_opts;

/* return codes (own numbering, mirrors the meaning of the product's statuses) */
#define OR_OK 0
#define OR_E_ARG 1
#define OR_E_DIM 2
#define OR_E_PART 3
#define OR_E_ZERO_BLOCK 4
#define OR_E_NOT_SPD 5
#define OR_E_COLOURING 6
#define OR_E_BREAKDOWN 7
#define OR_E_OOM 10

int or_setup(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
             const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
             double rank_tol, or_ctx** out);
/* the same with the caller's colouring colour[nparts] (sweep order: by colour,
   then id); a colouring with two coupled subdomains of one colour fails with
   OR_E_COLOURING.  colour[i] = i is the paper's plain sequential sweep. */
int or_setup_coloured(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                      const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                      double rank_tol, const int32_t* colour, or_ctx** out);
int or_setup_ex(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
                double rank_tol, const or_opts* o, or_ctx** out);
void or_set_coarse_solver(or_ctx* c, or_coarse_fn fn, void* user);
/* A_0 as a full symmetric CSR in coarse order; rp == NULL: returns the entry count */
int64_t or_get_Ac_csr(or_ctx* c, int64_t* rp, int32_t* col, double* val);
/* three levels: the two-level method applied again to A_0,
   with F_0 = R_0 F and second-level part part2[I] for every fine part I */
int or_setup3(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* F, int k, const int32_t* part, int32_t nparts, int overlap,
              double rank_tol, const int32_t* part2, int32_t nparts2, or_ctx** out);
/* the second-level context (borrowed; NULL for two levels) */
or_ctx* or_child(or_ctx* c);
int or_apply_precond(or_ctx* c, const double* r, double* z);
int or_forward_sweep(or_ctx* c, const double* r, double* z);
int or_coarse_correct(or_ctx* c, const double* r, double* z);
int or_spmv(or_ctx* c, const double* x, double* y);
int or_pcg(or_ctx* c, const double* f, double rtol, int max_iter, int stop_mode,
           double* u, int* iters, double* hist, int* converged);
/* the same, recording alpha_k (k < iters) and beta_k (k < iters - 1 or iters) */
int or_pcg_ab(or_ctx* c, const double* f, double rtol, int max_iter, int stop_mode,
              double* u, int* iters, double* hist, int* converged, double* alphas, double* betas);
/* info[0..9] = n, n_c, nparts, ncolours, m_min, m_max, k, dropped, levels, n_c of level 2 */
void or_info(or_ctx* c, int64_t* info);
double or_min_rank_ratio(or_ctx* c);
int or_get_colours(or_ctx* c, int32_t* colour);
int64_t or_get_overlap(or_ctx* c, int32_t i, int32_t* idx);  /* returns |Omega~_i|, fills idx if non-NULL */
int or_get_P_dense(or_ctx* c, double* P);        /* n x n_c column-major (tiny problems) */
int or_get_Ac_dense(or_ctx* c, double* Ac);      /* n_c x n_c, full symmetric (tiny problems) */
int or_get_coarse_offsets(or_ctx* c, int32_t* cptr); /* nparts+1 */
void or_destroy(or_ctx* c);
const char* or_last_error(void);

#endif
