// ddg_internal.h — internal types shared by the host setup (setup.cpp) and the
// sm_100a kernels (pcg.cu, symv.cu, coarse.cu, setup_kernels.cu) of libddg.
// Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace ddg {

constexpr int TILE = 32;                 // rows/cols per tile = warp width
constexpr int TILE_ELEMS = TILE * TILE;  // 1024 doubles = 8 KB per tile
constexpr int DIAG_ELEMS = TILE * (TILE + 1) / 2;  // 528: packed diagonal tile (4224 B)

// Compact tail (single-triangle operators with m % 32 != 0): the last tile row
// keeps only its `tail` valid rows -- off-diagonal tiles tail x 32 (element
// (i, j) at j * tail + i), the diagonal tile its packed tail x tail lower
// triangle (column j at tail_col_off(tail, j)), padded to an even number of
// doubles (16-byte bulk copies) -- so no padding row is stored or streamed.
__host__ __device__ inline int tail_diag_doubles(int tail) { return ((tail * (tail + 1) / 2) + 1) & ~1; }
__host__ __device__ inline int tail_col_off(int tail, int j) { return j * tail - j * (j - 1) / 2; }

// doubles of an item's tiles: diagonal tiles of a triangle item are packed;
// tail != 0: its last tile row is compact (above)
__host__ __device__ inline int64_t item_doubles(int tri, int h, int ntiles, int tail = 0) {
    if (tri && tail) {
        const int64_t r = h - 1;    // full rows 0 .. h-2 hold r (r + 1) / 2 tiles, r of them diagonal
        return (r * (r + 1) / 2 - r) * TILE_ELEMS + r * DIAG_ELEMS + r * tail * TILE + tail_diag_doubles(tail);
    }
    return tri ? (int64_t)(ntiles - h) * TILE_ELEMS + (int64_t)h * DIAG_ELEMS : (int64_t)ntiles * TILE_ELEMS;
}
constexpr int SYMV_WARPS = 8;            // consumer warps per SYMV CTA
constexpr int MAX_BT = 16;               // max tiles per item side (smem partial sizing)

// One dense symmetric operator applied by the tiled SYMV kernel: a local
// inverse A_i^{-1} or the dense coarse inverse A_c^{-1}.
// Its lower-triangle tiles are stored item after item, each tile column-major
// (element (i,j) of tile at j*32+i), padded rows/cols zero.
struct OpDesc {
    int32_t m;        // true size
    int32_t mp;       // padded to a multiple of TILE
    int32_t nT;       // tiles per side
    int32_t BT;       // tiles per item-block side
    int32_t nblk;     // item-block rows = ceil(nT / BT)
    int32_t item_base;
    int32_t nitems;   // nblk * (nblk + 1) / 2
    int32_t out_mode; // 0: z[idx[r]] += y[r]; 1: y_out[r] = y[r] (identity, coarse); 2: front (external reduce)
    int64_t tile_off; // first double of its tiles
    int64_t idx_off;  // offset of its index list Omega~_i in d_oidx (out_mode 0)
    int64_t s_off;    // offset of its right-hand side (mp entries) in d_s
    int64_t part_off; // offset of its partial segments (multi-item only)
};

// A work item: the tiles of item-block (bi, bj), bj <= bi, of one operator.
struct ItemDesc {
    int32_t op;       // index into OpDesc array
    int32_t I0, I1;   // tile rows [I0, I1)
    int32_t J0, J1;   // tile cols [J0, J1)
    int32_t tri;      // 1: diagonal block (lower triangle incl. diagonal tiles)
    int32_t ntiles;
    int32_t tail;     // 0, or the valid rows (1..31) of a compact last tile row (whole-operator triangles)
    int64_t tile_off; // first double of this item's tiles
    int64_t part_off; // its partial slot (2 * BT * TILE doubles), -1 if single-item op
};

// Reduction task for multi-item operators: row block b of operator op.
struct RedDesc {
    int32_t op;
    int32_t b;
};

// One front of the sparse coarse factorisation (coarse_sparse.cpp): the
// separator unknowns S of a nested-dissection node, its boundary B (ancestor
// unknowns coupled to its subtree), stored as a tiled dense [S|B] matrix.
struct FrontDesc {
    int32_t nT, nK;          // tiles per side of the [S|B] front, pivot (S) tiles
    int32_t nS, nSp, nB;     // |S|, |S| padded to TILE, |B|
    int32_t parent;          // parent front or -1
    int32_t child_off, nchild;   // children: fchild[child_off .. child_off + nchild)
    int32_t op;              // OpDesc index of its solve operator
    int32_t pad;
    int64_t fvec_off;        // front vector (nT*TILE doubles)
    int64_t w_off;           // w_t: contributions passed to the parent (nB doubles)
    int64_t S_off, B_off;    // coarse index lists
    int64_t map_off;         // B_t -> position in the parent's front (nB ints), -1 at a root
};

// Reduction task of the coarse solve: rows [row0, row0+nrows) of a front op.
struct FRedTask {
    int32_t front, kind;     // kind 0: w_t += (forward), 1: x[S_t] = (backward)
    int32_t row0, nrows;
    int32_t cbeg, cend;      // contributions [cbeg, cend) in the contrib offset list
};

// Per-front schedule of the dataflow coarse solve (k_coarse_dataflow).
struct FrontDF {
    int32_t nG, nGH;          // forward (G) and backward (G + H) work items of the front
    int32_t ft0, ft1;         // its forward reduction tasks [ft0, ft1)
    int32_t bt0, bt1;         // its backward reduction tasks [bt0, bt1)
};
// work-queue entry of the dataflow coarse solve
constexpr int32_t DF_BWD = 1 << 30;       // backward entry (else forward)
constexpr int32_t DF_ASSEMBLE = 1 << 29;  // assemble a leaf front (low bits: front)
constexpr int32_t DF_RED = 1 << 28;       // a reduction task (low bits: task index)
constexpr int32_t DF_IDX = DF_RED - 1;
// device state, zeroed before every solve: [0] queue head, then per front
// fwd_ready, fwd_items_done, fwd_tasks_done, children_done, bwd_ready,
// bwd_items_done, bwd_tasks_done
constexpr int DF_STATE_PER_FRONT = 7;

// Device-side PCG scalars (one struct in device memory).
struct Scalars {
    double rho, sigma, alpha, beta, gamma;
    double res0, ref, pres0, res;
    double rtol;
    int32_t iter, done, status, max_iter;
    int32_t stop_mode, converged, pad0, pad1;
    double loc[5];   // multi-GPU: rank-local sums (init, rz_first, spmv_dot, update, rz)
    double glob[5];  // ... and their allreduced totals
    double* ab;      // CG coefficients: alpha_k at ab[2k], beta_k at ab[2k+1] (Lanczos estimate)
    double tres;     // ||f - A u||_2 after the solve
};

// Reduction scratch: per-block partial sums + a ticket counter.
constexpr int RED_BLOCKS = 148 * 8;
constexpr int VEC_THREADS = 256;

// Matrix-free description of A for the hot-path row kernels (include/ddg.h
// ddg_stencil), validated against the CSR at setup.  CONST points are sorted
// by linear offset, i.e. in the CSR's column order, and FACE7 rows are
// evaluated in that order too, so stencil and CSR rows round identically.
constexpr int STENCIL_MAX_PTS = 16;
struct DevStencil {
    int32_t kind;        // 0 none (CSR), 1 constant, 2 face7, 3 node27 (class table in coef)
    int32_t npts;
    int32_t nx, ny, nz, pad;
    int32_t dx[STENCIL_MAX_PTS], dy[STENCIL_MAX_PTS], dz[STENCIL_MAX_PTS];
    int32_t off[STENCIL_MAX_PTS];   // linear offsets dx + nx (dy + ny dz)
    int32_t rx, ry, rz;             // reach per axis: rows farther than that from the faces need no checks
    int32_t dof;                    // node27: unknowns per node
    double c[STENCIL_MAX_PTS];
    const double* coef;  // face7: diag | cx | cy | cz, 4 n doubles; node27: table[class][offset][d][e] (device)
};

struct DevCSR {
    int64_t n;
    int64_t nnz;
    const int32_t* rp;   // int32 row offsets (nnz < 2^31 checked)
    const int32_t* col;
    const double* val;
    int32_t sw;          // lanes per row in the row kernels (1, 4, 8 or 32; by mean row length)
    int32_t bs;          // 3 or 4: node-blocked columns (bcol/brp below), else 0 (col[] per entry)
    DevStencil st;       // st.kind != 0: rows evaluated matrix-free (sw = 1)
    // Node-blocked column indices: every row of block-row V = v / bs holds the
    // same full, aligned bs-column blocks, so entry j of row v sits in column
    // bcol[brp[V] + j / bs] * bs + j % bs.  val[] keeps the CSR order, so the
    // row sums are bitwise those of the CSR; only the index traffic shrinks
    // (4 B per block per block-row instead of 4 B per entry).
    const int32_t* bcol;
    const int32_t* brp;
};

struct ColourPlan {
    int32_t sub_begin, sub_end;     // sweep positions [begin, end)
    int32_t item_begin, item_end;   // items of this colour
    int32_t red_begin, red_end;     // reduction tasks of multi-item ops
    int32_t max_rows;               // max m over the colour's subdomains
    int32_t max_rows_t;             // max rows touched by one SYMV item (smem sizing)
    int32_t all_single;             // every operator of the colour is one item (gather may be fused)
    int32_t max_ntiles;             // largest item of the colour (tiles)
    int32_t ring_off;               // its k_symv_ring CTA partition in ctx::h_ring (-1: none)
    // multi-GPU boundary-first split: ops [sub_begin, sub_mid) write
    // z values another rank reads, [sub_mid, sub_end) do not; their items, reduction
    // tasks and ring partitions ([*_begin, *_mid) / [*_mid, *_end)); sub_mid = sub_end: no split
    int32_t sub_mid, item_mid, red_mid;
    int32_t ring_b, ring_i;
};

// streams on which chain kernels launch without programmatic dependent launch
// (the loopback group's stream, shared by several host threads; symv.cu)
void register_no_pdl_stream(cudaStream_t st);
void release_no_pdl_stream(cudaStream_t st);
// ---- kernel launchers (pcg.cu, symv.cu, coarse.cu, setup_kernels.cu) --------
void launch_symv(cudaStream_t st, const OpDesc* ops, const ItemDesc* items, int item_begin,
                 int nitems, const double* tiles, const double* s, const int32_t* oidx, double* z,
                 double* y_out, double* partials, const int32_t* done, int max_rows_t, unsigned* tickets,
                 int gather_mode = 0, DevCSR A = DevCSR{}, const double* r = nullptr, bool small_ok = false);
// persistent bulk-copy-ring SYMV (k_symv_ring); cta_part[0..ncta]: item ranges
// (relative to item_begin) of the CTAs.  Requires every item's rows <= 512.
constexpr int RING_MAX_ROWS = 512;
void symv_ring_init();   // once per device, before any capture
extern int g_compact;    // 1: whole-triangle operators store a compact last tile row (DDG_COMPACT)
int symv_ring_trace(unsigned long long* out);   // debug counters (DDG_RING_TRACE)
// max_rows_r / max_rows_c: the launch's largest row block and (rectangles)
// column block, in rows (ring_dims)
void launch_symv_ring(cudaStream_t st, const OpDesc* ops, const ItemDesc* items, int item_begin,
                      const int32_t* cta_part, int ncta, int max_rows_r, int max_rows_c, const double* tiles,
                      const double* s, const int32_t* oidx, double* z, double* y_out, double* partials,
                      const int32_t* done, bool triangles = false);
void launch_symv_reduce(cudaStream_t st, const OpDesc* ops, const ItemDesc* items,
                        const RedDesc* red, int red_begin, int nred, const int32_t* oidx,
                        const double* partials, double* z, double* y_out, const int32_t* done);
// s[x] = r[g] - (A z)[g] with g = gidx[x] (gidx < 0: padding, left untouched)
// for x in [x0, x1): the residual restriction of a whole colour, flat over
// the colour's contiguous s segments
void launch_gather_flat(cudaStream_t st, int64_t x0, int64_t x1, const int32_t* gidx, DevCSR A, const double* r,
                        const double* z, double* s, bool z_is_zero, const int32_t* done);
void launch_coarse_restrict(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* bidx,
                            const int32_t* cptr, const int64_t* qoff, const double* Q, DevCSR A,
                            const double* r, const double* z, double* bc, int maxmI,
                            const int32_t* done, const int32_t* parts = nullptr);
void launch_restrict_dot(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* cptr, const int64_t* qoff,
                         const double* Q, const double* res, double* bc, int maxmI, const int32_t* done);
void launch_prolong_flat(cudaStream_t st, int64_t n, const int32_t* xpart, const int64_t* bptr, const int32_t* bidx,
                         const int32_t* cptr, const int64_t* qoff, const double* Q, const double* yc, double* z,
                         const int32_t* done);
void launch_prolong(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* bidx,
                    const int32_t* cptr, const int64_t* qoff, const double* Q, const double* yc,
                    double* z, int maxmI, const int32_t* done, const int32_t* parts = nullptr);
void launch_fill(cudaStream_t st, double* x, int64_t n, double v, const int32_t* done);
void launch_spmv(cudaStream_t st, DevCSR A, const double* x, double* y);

// PCG pieces (all read/write the device Scalars; all exit early once done != 0).
// rows/nrows: the rank's owned rows (rows == nullptr: 0..nrows-1); dist != 0:
// reductions leave the rank-local sum in sc->loc[slot] (then allreduce +
// launch_pcg_finalize).
void launch_pcg_init(cudaStream_t st, int64_t n, const double* f, double* r, double* u, const int32_t* rows,
                     int64_t nrows, Scalars* sc, double* hist, double* red, unsigned* ticket, int dist);
void launch_pcg_rz_first(cudaStream_t st, const double* r, const double* z, double* p, const int32_t* rows,
                         int64_t nrows, Scalars* sc, double* red, unsigned* ticket, int dist);
void launch_true_res(cudaStream_t st, DevCSR A, const double* f, const double* u, int64_t n, Scalars* sc,
                     double* red, unsigned* ticket);
void launch_pcg_spmv_dot(cudaStream_t st, DevCSR A, const double* p, double* q, const int32_t* rows,
                         int64_t nrows, Scalars* sc, double* red, unsigned* ticket, int dist);
void launch_pcg_update(cudaStream_t st, const double* p, const double* q, double* u, double* r,
                       const int32_t* rows, int64_t nrows, Scalars* sc, double* hist, double* red,
                       unsigned* ticket, int dist);
void launch_pcg_rz(cudaStream_t st, const double* r, const double* z, const int32_t* rows, int64_t nrows,
                   Scalars* sc, double* red, unsigned* ticket, int dist);
void launch_pcg_direction(cudaStream_t st, const double* z, double* p, const int32_t* rows, int64_t nrows,
                          Scalars* sc);
void launch_pcg_finalize(cudaStream_t st, int slot, Scalars* sc, double* hist);
// k_pcg_small (pcg.cu): the whole solve of a small problem in one cluster kernel
struct SmallArgs {
    DevCSR A;
    int64_t n;
    const double* f;
    double *u, *r, *z, *p, *q;
    Scalars* sc;
    double* hist;
    double* part;                 // [2][SMALL_MAX_G] block sums
    const OpDesc* ops;
    const ItemDesc* items;
    const double* tiles;
    const int32_t* oidx;
    const int32_t* cops;          // [ncolours + 1] operator ranges of the colours (sweep order)
    int ncolours;
    int nparts;
    const int64_t* bptr;
    const int32_t* bidx;
    const int32_t* cptr;
    const int64_t* qoff;
    const double* Q;
    int coarse_item;
    double* bc;
    // shared-memory plan (small_plan, setup.cpp): resident arena (doubles and
    // ints, the largest over the cluster's CTAs), scratch row length, padded
    // coarse size, coarse tile rows, bytes; cluster size
    int ad, ai, pw, ncp, nTc, G;
    size_t smem;
    int dbg;                    // DDG_SMALL_TRACE=2: timestamps inside the colour steps too
};
bool small_cluster_ok(int G, size_t smem);   // a cluster of G CTAs with smem bytes each fits
int small_trace(int on, unsigned long long* out, int cap);   // debug (DDG_SMALL_TRACE)
bool launch_pcg_small(cudaStream_t st, const SmallArgs& args);
void launch_pcg_cond(cudaStream_t st, const Scalars* sc, unsigned long long handle);
void launch_halo_pack(cudaStream_t st, const double* v, const int32_t* idx, double* buf, int64_t n);
void launch_halo_unpack(cudaStream_t st, const double* buf, const int32_t* idx, double* v, int64_t n);
void launch_copy_rows(cudaStream_t st, const double* in, double* out, const int32_t* rows, int64_t nrows);

// setup kernels
void launch_extract_local(cudaStream_t st, int nops, const int32_t* op_ids, const OpDesc* ops,
                          const int32_t* oidx, DevCSR A, double* scratch,
                          const int64_t* scratch_off);
// Gauss-Jordan exchange on the first nK pivot tiles of nmat tiled dense
// matrices (nK = nT: full inverse; nK < nT: partial, Schur complement left in
// the trailing block).  ids[i] is reported in err[0] on a non-positive pivot.
void launch_gj_batched(cudaStream_t st, int nmat, const int32_t* nT, const int32_t* nK,
                       double* const* mats, const int32_t* ids, int32_t* err);
// blocked exchange (128-column pivot blocks, fp64 GEMM updates) over a batch,
// used for matrices of at least GJB_MIN_T tiles per side;
// mats/nT/nK/ids are device arrays of nmat entries, maxT/maxK their maxima
constexpr int GJB_MIN_T = 16;
// sym: 1 the experimental symmetric exchange (R22), 0 the full exchange, -1 the DDG_GJ_SYM switch
void launch_gj_blocked(cudaStream_t st, int nmat, int maxT, int maxK, double* const* mats, const int32_t* nT,
                       const int32_t* nK, const int32_t* ids, int32_t* err, int sym = -1);
// coarse space on the device (basis.cu): per-part dd-MGS basis (one warp per
// part), compaction to Q, and the Galerkin blocks A_c[I, J] (one CTA per block)
void launch_basis_mgs(cudaStream_t st, int nparts, int k, int64_t n, const double* F, const int64_t* bptr,
                      const int32_t* bidx, const int64_t* voff, double2* V, double* Qw, int32_t* rank,
                      double* ratio, double rank_tol, int32_t* err);
void launch_basis_compact(cudaStream_t st, int nparts, const int64_t* bptr, const int64_t* voff,
                          const int64_t* qoff, const double* Qw, double* Q);
void launch_galerkin_blocks(cudaStream_t st, int nblocks, int maxk, const int32_t* bI, const int32_t* bJ,
                            const int64_t* boff, const int64_t* bptr, const int32_t* bidx, const int32_t* cptr,
                            const int64_t* qoff, const double* Q, const int32_t* part, const int32_t* bpos,
                            const int32_t* rp, const int32_t* col, const double* val, double* out);
// Cholesky factor storage (chol.cu): tile row I holds I full 32 x 32 tiles L_IJ
// (J < I) and then the packed lower triangle of L_II^{-1} (DIAG_ELEMS doubles)
__host__ __device__ inline int64_t chol_row_off(int I) {
    return (int64_t)TILE_ELEMS * I * (I - 1) / 2 + (int64_t)DIAG_ELEMS * I;
}
__host__ __device__ inline int64_t chol_doubles(int nT) { return chol_row_off(nT); }
// local_variant = DDG_LOCAL_CHOLESKY (chol.cu): tile Cholesky of nmat tiled
// dense matrices (one CTA each), packing of the lower tiles at each op's
// tile_off, and one colour's forward + back substitutions (one CTA per op)
void launch_chol_local(cudaStream_t st, int nmat, const int32_t* nT, double* const* mats, const int32_t* ids,
                       int32_t* err);
void launch_chol_pack(cudaStream_t st, int nops, int max_tiles, const int32_t* op_ids, const OpDesc* ops,
                      const double* scratch, const int64_t* scratch_off, double* out);
void launch_chol_solve(cudaStream_t st, const OpDesc* ops, int op_begin, int nops, int max_mp, const double* fac,
                       const double* s, const int32_t* oidx, double* z, const int32_t* done);
// sparse coarse factorisation / solve
void launch_front_scatter(cudaStream_t st, int64_t ntrip, const int32_t* frow, const int32_t* fcol,
                          const double* fval, const int32_t* ffront, const FrontDesc* fronts,
                          double* const* fptr);
void launch_front_extend_add(cudaStream_t st, int ntask, const int32_t* child, const FrontDesc* fronts,
                             double* const* fptr, const int32_t* map, int64_t max_elems);
void launch_front_pack(cudaStream_t st, int i0, int i1, int item_base, const int32_t* item_front,
                       const FrontDesc* fronts, double* const* fptr, const ItemDesc* items, double* ctiles);
void launch_front_fwd_assemble(cudaStream_t st, int f0, int nf, const FrontDesc* fronts, const int32_t* fchild,
                               const int32_t* fS, const int32_t* map, const double* bc, double* fvec,
                               double* w, const int32_t* done);
void launch_front_bwd_gather(cudaStream_t st, int f0, int nf, const FrontDesc* fronts,
                             const int32_t* fB, const double* x, double* fvec, const int32_t* done);
void launch_copy_segments(cudaStream_t st, int nseg, const int64_t* seg, const double* src, double* dst);
void launch_gather_masked(cudaStream_t st, int64_t n, const int32_t* idx, const uint8_t* mask, const double* src,
                          double* dst);
void launch_front_reduce(cudaStream_t st, const FRedTask* tasks, int t0, int nt, const int64_t* contrib,
                         const FrontDesc* fronts, const int32_t* fS, const double* partials, double* w,
                         double* x, const int32_t* done);
// whole sparse coarse solve y = A_c^{-1} b_c in one launch (see coarse.cu)
void launch_coarse_dataflow(cudaStream_t st, int nwork, const int32_t* work, const FrontDesc* fronts,
                            const int32_t* fchild,
                            const FrontDF* fdf, const int32_t* item_front, int item_base, const OpDesc* ops,
                            const ItemDesc* items, const double* ctiles, const FRedTask* fwd, const FRedTask* bwd,
                            const int64_t* contrib, const int32_t* fS, const int32_t* fB, const int32_t* map,
                            const double* bc, double* fvec, double* w, double* x, double* partials,
                            int32_t* state, int max_rows_t, const int32_t* done, uint64_t* trace = nullptr);
void launch_scatter_coarse(cudaStream_t st, int64_t nent, const int32_t* row, const int32_t* col,
                           const double* val, int nT, int n_c, double* M);
void launch_pack(cudaStream_t st, int nops, const int32_t* op_ids, const OpDesc* ops,
                 const ItemDesc* items, const double* scratch, const int64_t* scratch_off,
                 double* tiles);

int num_sms();

}  // namespace ddg
