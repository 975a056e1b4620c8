/*
 * ddg.h — C ABI of libddg, the B200-native DDG-preconditioned CG solver.
 *
 * Method: Edwards & Bridson, "The Discretely-Discontinuous Galerkin Coarse
 * Grid for Domain Decomposition", arXiv:1504.00907.  Conjugate
 * gradient (§7) on a sparse SPD system A u = f
 * (Table 1), preconditioned by the two-level symmetric
 * multiplicative overlapping Schwarz method (§6) whose
 * coarse level is the DDG space: each generating vector (column of F,
 * PAPER.md:239-241) restricted to each non-overlapping part Omega_I and
 * orthonormalised per part is one basis function; the
 * coarse matrix is the Galerkin projection A_c = P^T A P (PAPER.md:266,
 * written A_0 = R_0 A R_0^T there; P = R_0^T).  Optionally the coarse solve
 * is one application of the same two-level method built on A_c (the paper's
 * three-level V-cycle; ddg_opts.part2).
 *
 * Everything below runs on one CUDA device per context.  All numerics are
 * IEEE fp64.  There is no CPU fallback: with no usable device every entry
 * point returns DDG_E_CUDA.
 *
 * Ownership: every input pointer is BORROWED for the duration of the call and
 * copied; the context owns all device memory it allocates; outputs go into
 * caller-allocated buffers.  A context is not thread-safe; one context per
 * GPU / rank; a context can be reused for any number of solves.
 *
 * Errors: every int-returning call returns a ddg_status.  On error a
 * stage-labelled, thread-local message is available from ddg_last_error().
 */
#ifndef DDG_H
#define DDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DDG_OK = 0,
    DDG_E_ARG = 1,         /* null pointer, bad size (message carries sizes)          */
    DDG_E_DIM = 2,         /* dimension mismatch / non-canonical CSR                  */
    DDG_E_PART = 3,        /* empty part or part id out of range                      */
    DDG_E_ZERO_BLOCK = 4,  /* F restricted to a part is entirely zero   */
    DDG_E_NOT_SPD = 5,     /* non-positive pivot in a local or the coarse factor
                              (SPEC.md:73); message names stage, block and pivot      */
    DDG_E_COLOURING = 6,   /* ddg_opts.colour has two coupled subdomains in one colour */
    DDG_E_BREAKDOWN = 7,   /* p^T A p <= 0 or r^T z <= 0 inside PCG     */
    DDG_E_CUDA = 8,        /* CUDA runtime error or no device                         */
    DDG_E_NCCL = 9,        /* communicator error                                      */
    DDG_E_OOM = 10         /* device allocation failed                                */
} ddg_status;

typedef struct ddg_ctx ddg_ctx;

/* Stopping rule readings of "a 10^-9 reduction in residual after the first
 * application of the preconditioner"; reading R1. */
enum { DDG_STOP_RES0 = 0,      /* ||r_k||_2 <= rtol ||r_0||_2 (default)              */
       DDG_STOP_RES1 = 1,      /* ||r_k||_2 <= rtol ||r_1||_2           */
       DDG_STOP_PREC = 2 };    /* sqrt(r_k^T z_k) <= rtol sqrt(r_0^T z_0)             */

/* Optional structured-grid description of A (SURVEY.md §8(b) "ddg_stencil"),
 * used matrix-free by the hot-path row kernels (the SpMV q = A p, the residual
 * restrictions s = R~_i (r - A z) and b_c = P^T (r - A z)) instead of reading
 * the CSR.  The CSR passed to ddg_setup stays the definition of A: ddg_setup
 * checks that the stencil reproduces every entry of every row exactly and
 * fails with DDG_E_ARG otherwise.  Rows are the grid points, row index
 * v = x + dims[0] * (y + dims[1] * z); neighbours off the grid are absent
 * (zero Dirichlet values / zero ghosts: BASELINE configs C1, C2, C3, C5).
 * All pointers are host pointers, borrowed for the duration of ddg_setup. */
enum { DDG_STENCIL_NONE = 0,
       DDG_STENCIL_CONST = 1,   /* constant coefficients: npts points (dx, dy, dz) with values coef */
       DDG_STENCIL_FACE7 = 2,   /* 7-point with per-row coefficients: coef = 4 x n, blocks
                                   diag | cx | cy | cz with cx[v] = A[v, v+1],
                                   cy[v] = A[v, v+dims[0]], cz[v] = A[v, v+dims[0]*dims[1]]
                                   (A symmetric: A[v, v-1] = cx[v-1], ...)                     */
       DDG_STENCIL_NODE27 = 3 };/* node-blocked 27-point operator with constant rows per boundary
                                   class (Q1 elements on a uniform grid, BASELINE C4): dims =
                                   nodes per axis, npts = unknowns per node (1..4), row
                                   dof * node + d, node = x + dims[0] (y + dims[1] z); every row
                                   couples to all in-grid nodes at distance <= 1 per axis.  The
                                   values are read from the CSR: all nodes of one class (first /
                                   interior / last per axis, 27 classes) must have identical rows;
                                   offsets and coef are unused                                   */
enum { DDG_STENCIL_MAX_PTS = 16 };
typedef struct {
    int32_t kind;              /* DDG_STENCIL_*                                                 */
    int32_t dims[3];           /* grid points per axis (1 for unused axes)                      */
    int32_t npts;              /* CONST: number of points, <= DDG_STENCIL_MAX_PTS               */
    const int32_t* offsets;    /* CONST: npts x 3 offsets (dx, dy, dz)                          */
    const double* coef;        /* CONST: npts values; FACE7: 4 n values                         */
} ddg_stencil;

typedef struct {
    int overlap;          /* Delta: graph distance in the pattern of A. default 1 */
    double rank_tol;      /* keep column j of a part iff ||v_j|| >= rank_tol * ||F_I e_j||, v_j the
                             part of column j orthogonal to the kept earlier columns
                             (reading R7). default 1e-8            */
    int stop_mode;        /* DDG_STOP_*, default DDG_STOP_RES0                                   */
    int max_iter;         /* default 1000                                         */
    int device;           /* CUDA device ordinal; default 0                                       */
    void* stream;         /* cudaStream_t to run on, or NULL: the context creates its own stream   */
    int use_graphs;       /* 1 (default): capture the preconditioner in a CUDA graph               */
    int verbose;          /* 0 (default): quiet; 1: setup timings on stderr                        */
    int coarse_variant;   /* 0 auto (dense if n_c <= 8192), 1 dense packed inverse of A_c,
                             2 sparse: nested dissection + supernodal block elimination         */
    int block_ndim;       /* 0, or the dimension of block_coords                                    */
    int fuse_gather;      /* R~_i(r - A z) computed inside the SYMV kernel for single-item subdomains:
                             0 never, 1 (default) when the items are large (>= 32 tiles) or the
                             colour is small, 2 always                                               */
    void* comm;           /* ddg_comm* for multi-GPU, or NULL (single GPU)                          */
    int small_kernel;     /* 1 (default): colours of many (>= 16 per SM) single-item subdomains with
                             |Omega~_i| <= 256 use the warp-per-subdomain SYMV                    */
    const int32_t* block_coords; /* optional nparts x block_ndim integer coordinates of the parts
                             (host, borrowed): geometric nested dissection of the coarse graph;
                             NULL: BFS level-set bisection                                       */
    const ddg_stencil* stencil;  /* optional matrix-free description of A (above), or NULL       */
    /* Three levels: when part2 is non-NULL the coarse solve
       A_c^{-1} is replaced by one application of the two-level method built
       on A_c (same Delta and rank_tol), with coarsened generating vectors
       F_0 = R_0 F (the coarse coefficients of F) and second-level parts:
       coarse unknown (I, i) belongs to part2[I].  part2: nparts int32 in
       [0, nparts2), every second-level part non-empty, nparts2 >= 2
       (DDG_E_PART "too small for three levels" otherwise); host, borrowed
       for the duration of ddg_setup.  block_coords2: optional nparts2 x
       block_ndim coordinates of the second-level parts.  coarse_variant then
       selects the second level's coarse solve (0 auto, 1 dense, 2 sparse).
       With opts.comm the second level is distributed over the same ranks
       (its parts by block_coords2 boxes) and only its coarse factor is
       replicated; y_c is assembled on every rank by one allreduce. */
    const int32_t* part2;
    int32_t nparts2;
    const int32_t* block_coords2;
    /* Optional colouring of the subdomains (nparts int32 in [0, nparts), host,
       borrowed for ddg_setup): the sweep visits colours in increasing order,
       subdomains of one colour concurrently (ids increasing within a colour
       for the record).  Two subdomains of one colour must not be coupled
       (Omega~_i meets Omega~_j or its neighbours): DDG_E_COLOURING otherwise.
       colour[i] = i is the paper's plain sequential sweep.
       NULL: greedy first-fit in id order (reading R3). */
    const int32_t* colour;
    /* How the exact local solves A_i^{-1} s ("we solve these
       subdomain problems exactly") are realised:
       DDG_LOCAL_AUTO (0, default) = DDG_LOCAL_INVERSE: the explicit inverse
       A_i^{-1}, formed once by blocked Gauss-Jordan and applied per visit as one
       symmetric matrix-vector product (one read of its packed lower triangle);
       DDG_LOCAL_CHOLESKY (1): the Cholesky factor A_i = L_i L_i^T, applied per
       visit as a forward and a back substitution over 32 x 32 tiles (the
       32 x 32 diagonal blocks stored inverted), one CTA per subdomain of a
       colour.  Both are exact; results agree to rounding (DESIGN.md §7 has
       the measured comparison).  Other values: DDG_E_ARG. */
    int local_variant;
} ddg_opts;

enum { DDG_LOCAL_AUTO = 0, DDG_LOCAL_CHOLESKY = 1, DDG_LOCAL_INVERSE = 2 };

typedef struct {
    int converged;        /* 1 if the stopping rule was met                                     */
    int iters;            /* number of A p products (reading R16)              */
    double res0;          /* ||r_0||_2 = ||f||_2                                                 */
    double res_final;     /* last recurrence residual ||r_k||_2                                  */
    double t_setup;       /* seconds spent in ddg_setup (host clock around device work)          */
    double t_solve;       /* seconds of the last solve (CUDA events on the context stream)       */
    double frac_iters;    /* fractional iteration count                       */
    double cond_est;      /* Lanczos estimate of cond(M A) from the CG coefficients:
                             lambda_max / lambda_min of the CG-Lanczos tridiagonal; 1 if < 2 steps */
    double iter_bound;    /* classical CG bound ln(2/rtol) / ln((sqrt k + 1)/(sqrt k - 1)), k = cond_est */
    double true_res;      /* ||f - A u||_2 of the returned u, computed once after the loop (inside t_solve;
                             the stopping rule uses the recurrence residual, reading R2)           */
    double bytes_per_iter_model;  /* algorithmic HBM bytes of one PCG iteration on this rank
                             (SURVEY.md §8(d)): 2 reads of every local operator, one coarse
                             solve, (64 + 2a) per subdomain row, (144 + 2a + 16k) per row, a =
                             matrix bytes per row (0 stencil, 32 face7, 12 nnz/n + 4 CSR)   */
} ddg_report;

typedef struct {
    int64_t n;            /* fine unknowns                                                      */
    int64_t n_c;          /* coarse unknowns after rank pruning                                 */
    int32_t nparts;       /* number of parts Omega_I = number of overlapping subdomains         */
    int32_t ncolours;     /* colours of the multiplicative sweep                                */
    int32_t m_min, m_max; /* min / max |Omega~_i|                                               */
    int32_t k;            /* generating vectors per part before pruning                          */
    int32_t dropped;      /* total columns dropped by the rank test                              */
    double min_rank_ratio;          /* min over parts and kept j of ||v_j|| / ||F_I e_j|| (R7)       */
    int64_t local_factor_bytes;     /* bytes of the stored local operators (device)            */
    int64_t coarse_factor_bytes;    /* bytes of the stored coarse operator (device); with several
                                       ranks and the sparse coarse solve, this rank's share     */
    int32_t coarse_variant;         /* 1 dense packed inverse, 2 sparse supernodal, 3 three
                                       levels (the second level's own variant in coarse_variant2) */
    int32_t levels;                 /* 2 or 3                                                   */
    int64_t coarse_solve_bytes;     /* operator bytes one coarse solve must read: the packed
                                       inverse once (dense), or 2|G| + |H| over the fronts
                                       (sparse: G read forward and backward, H backward);
                                       three levels: the second level's local operators twice
                                       (two sweeps) plus its own coarse solve bytes; with several
                                       ranks (sparse), the bytes this rank reads per solve     */
    int64_t n_c2;                   /* three levels: coarse unknowns of the second level       */
    int32_t nparts2, ncolours2;     /* three levels: second-level parts and colours            */
    int32_t coarse_variant2;        /* three levels: the second level's coarse variant (1, 2)  */
    int32_t pad2;
} ddg_info;

/* Fills *o with the defaults listed above. */
void ddg_default_opts(ddg_opts* o);

/*
 * ddg_setup — build the preconditioner for A.
 *   n                 fine unknowns (>= 1)
 *   row_ptr[n+1]      int64 CSR row offsets, row_ptr[0] = 0            (host)
 *   col[nnz]          int32 column indices, strictly increasing per row (host)
 *   val[nnz]          fp64 values; A must be symmetric positive definite (host)
 *   F[n*k]            fp64 generating vectors, column-major n x k       (host)
 *   k                 number of generating vectors (1..128)
 *   part[n]           int32 part id of every unknown, 0..nparts-1; every part non-empty
 *   nparts            number of parts
 *   opts              NULL for defaults
 *   out               receives the new context
 * Errors: DDG_E_ARG, DDG_E_DIM, DDG_E_PART, DDG_E_ZERO_BLOCK, DDG_E_NOT_SPD,
 *         DDG_E_CUDA, DDG_E_OOM.  On error *out is NULL.
 */
int ddg_setup(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
              const double* F, int k, const int32_t* part, int32_t nparts,
              const ddg_opts* opts, ddg_ctx** out);

/*
 * ddg_pcg_solve — solve A u = f from u_0 = 0 by PCG with the
 * DDG two-level preconditioner.  HOST buffers: f is copied to the device,
 * u and the residual history are copied back (the end-to-end path).
 *   f[n]              right-hand side (host)
 *   rtol              relative tolerance (> 0)
 *   max_iter          <= 0 means opts.max_iter
 *   u[n]              solution (host, out)
 *   iters             number of A p products (out, may be NULL)
 *   res_hist[cap]     ||r_j||_2 for j = 0..iters (out, may be NULL); entries past
 *                     cap are dropped
 *   rep               report (out, may be NULL)
 * Hitting max_iter is not an error: rep->converged = 0.
 * Errors: DDG_E_ARG, DDG_E_BREAKDOWN, DDG_E_CUDA.
 */
int ddg_pcg_solve(ddg_ctx* ctx, const double* f, double rtol, int max_iter, double* u,
                  int* iters, double* res_hist, int res_hist_cap, ddg_report* rep);

/* Same as ddg_pcg_solve with f and u DEVICE pointers on the context's device
 * (e.g. torch tensors); res_hist stays a host buffer.  No host<->device copy of
 * vectors happens inside. */
int ddg_pcg_solve_device(ddg_ctx* ctx, const double* d_f, double rtol, int max_iter,
                         double* d_u, int* iters, double* res_hist, int res_hist_cap,
                         ddg_report* rep);

/* z = M r, the full two-level symmetric preconditioner;
 * host buffers of length n.  Test hook: symmetry, positivity, linearity. */
int ddg_apply_precond(ddg_ctx* ctx, const double* r, double* z);

/* z = P A_c^{-1} P^T r, the coarse correction alone; host buffers. */
int ddg_coarse_correct(ddg_ctx* ctx, const double* r, double* z);

/* y = A x on the device (test hook for the SpMV kernel); host buffers. */
int ddg_spmv(ddg_ctx* ctx, const double* x, double* y);

/* Size and diagnostics of a built context. */
int ddg_get_info(ddg_ctx* ctx, ddg_info* info);

/* CG coefficients of the last solve: alphas[k] for k < iters and betas[k] for
 * k < iters - 1 (host, out, up to cap entries each; either may be NULL).
 * Returns iters (the number of alphas), or a negative status. */
int ddg_get_lanczos(ddg_ctx* ctx, double* alphas, double* betas, int cap);

/* colour[nparts]: colour of every subdomain in the multiplicative sweep (host, out). */
int ddg_get_colours(ddg_ctx* ctx, int32_t* colour);

/* m[nparts]: |Omega~_i| of every subdomain (host, out). */
int ddg_get_subdomain_sizes(ddg_ctx* ctx, int32_t* m);

/* Number of kernel launches the context issued since the last reset (its own
 * kernels only); `reset` != 0 zeroes the counter after reading. */
int64_t ddg_launch_count(ddg_ctx* ctx, int reset);

/* Per-kernel timing of the hot path (CUDA events on the context stream).
 * While profiling is on, solves run without CUDA graphs and every kernel of
 * the listed classes is bracketed by an event pair; ddg_get_kernel_stats
 * synchronises, sums the pairs recorded since the last call, and resets. */
typedef struct {
    int64_t symv_launches;     /* local colour SYMV launches (a4/a8 dominant kernel)          */
    double symv_ms;            /* their summed device time                                    */
    double symv_alg_bytes;     /* algorithmic bytes they must move: per subdomain visit the
                                  packed inverse 8 m(m+1)/2 + s read 8m + z read-modify-write 16m */
    double gather_ms;          /* residual restriction kernels                                */
    double reduce_ms;          /* partial-sum reduction kernels                               */
    double coarse_ms;          /* coarse restrict + coarse SYMV + prolong                     */
    double vec_ms;             /* SpMV+dot, update, r^T z, direction, fill                    */
    int64_t launches;          /* all kernels timed                                           */
} ddg_kstats;

int ddg_set_profiling(ddg_ctx* ctx, int on);
int ddg_get_kernel_stats(ddg_ctx* ctx, ddg_kstats* st);

/* ---------------------------------------------------------------------------
 * Multi-GPU.  One process / context per GPU.  Every rank
 * passes the same GLOBAL A, F and partition to ddg_setup with opts.comm set;
 * parts are assigned to ranks (boxes of the block grid when block_coords are
 * given), each rank applies only its own subdomains and exchanges, over NCCL:
 * p and r halos once per iteration, the z values written by every colour
 * step, the zero-padded coarse right-hand side (allreduce) and the three CG
 * scalars (allreduce); the coarse factor is replicated.  f and u stay full
 * length on every rank (u is assembled on every rank at the end).
 * ------------------------------------------------------------------------- */
typedef struct ddg_comm ddg_comm;

/* 128-byte NCCL unique id, created on rank 0 and broadcast by the caller. */
int ddg_get_unique_id(void* id128);
int ddg_comm_init(int rank, int nranks, const void* id128, int device, ddg_comm** out);
void ddg_comm_destroy(ddg_comm* comm);

/* Loopback group: nranks VIRTUAL ranks of one process on one device, so the
 * multi-rank path (owned rows and subdomains, halo exchanges, split
 * reductions, the distributed second level) runs and is tested where there
 * are fewer GPUs than ranks.  Each virtual rank is driven by its own host
 * thread (ddg_setup / ddg_pcg_solve with opts.comm = its loopback comm); all
 * of them enqueue on the group's one stream.  A collective is a host
 * rendezvous of every rank; the last to arrive enqueues the data movement
 * (device-to-device copies for halos, a fixed-rank-order sum kernel for
 * allreduces) after all ranks' preceding work -- no kernel waits on another.
 * Graph capture is off for loopback contexts.  nranks <= 16.  The group must
 * outlive its comms and their contexts. */
typedef struct ddg_loop_group ddg_loop_group;
int ddg_loop_group_create(int nranks, int device, ddg_loop_group** out);
void ddg_loop_group_destroy(ddg_loop_group* group);
int ddg_comm_init_loopback(ddg_loop_group* group, int rank, ddg_comm** out);

/* Host-only decomposition plan (no device needed): the same plan ddg_setup
 * builds for a communicator of nranks, exposed for tests and tools. */
typedef struct ddg_plan ddg_plan;
enum { DDG_PLAN_OWNED_ROWS = 0, DDG_PLAN_OWNED_SUBS = 1, DDG_PLAN_P_SEND = 2, DDG_PLAN_P_RECV = 3,
       DDG_PLAN_R_SEND = 4, DDG_PLAN_R_RECV = 5, DDG_PLAN_Z_SEND = 6, DDG_PLAN_Z_RECV = 7,
       DDG_PLAN_PROLONG_PARTS = 8, DDG_PLAN_COLOURS = 9, DDG_PLAN_PART_RANK = 10,
       DDG_PLAN_OVERLAP = 11 };
int ddg_plan_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const int32_t* part,
                    int32_t nparts, int overlap, const int32_t* block_coords, int block_ndim, int rank,
                    int nranks, ddg_plan** out);
/* Number of entries of list `what` (for colour / peer / subdomain where it
 * applies); copies min(count, cap) int32 entries into out when out != NULL. */
int64_t ddg_plan_query(ddg_plan* plan, int what, int colour, int peer, int32_t* out, int64_t cap);
void ddg_plan_destroy(ddg_plan* plan);

/* Release every resource of the context (NULL is a no-op). */
void ddg_destroy(ddg_ctx* ctx);

const char* ddg_status_string(int status);
const char* ddg_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DDG_H */
