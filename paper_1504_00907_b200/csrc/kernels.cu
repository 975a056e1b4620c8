// kernels.cu — sm_100a kernels of libddg.
//
// Hot path, one PCG iteration:
//   a1 pcg_spmv_dot      q = A p, sigma = p^T q, alpha = rho / sigma
//   a2 pcg_update        u += alpha p, r -= alpha q, gamma = r^T r, history, stop test
//   a4 gather + symv     per colour: s_i = R~_i (r - A z); z[Omega~_i] += A_i^{-1} s_i
//   a5 coarse_restrict   b_c = P^T (r - A z)
//   a6 symv (coarse op)  y_c = A_c^{-1} b_c (dense packed inverse, small n_c)
//   a7 prolong           z += P y_c
//   a8 gather + symv     reverse colour order
//   a9 pcg_rz, direction rho' = r^T z, beta, p = z + beta p
// Setup: extract_local, Gauss-Jordan block inversion (batched / big), pack.
//
// Every reduction is deterministic (fixed partition, fixed order, last-block
// finalisation with a ticket; no floating-point atomics), so runs are bitwise
// repeatable.  Every PCG kernel exits immediately once the device flag
// `done` is set, so the host can enqueue several iterations without syncing.
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ddg_internal.h"

namespace ddg {

#define FULL 0xffffffffu

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// (A x)[v] from the stencil, in the CSR's column order (see DevStencil)
__device__ __forceinline__ double stencil_dot(const DevStencil& st, int64_t v, const double* __restrict__ x) {
    const int nx = st.nx, ny = st.ny;
    const int ix = (int)(v % nx);
    const int64_t r = v / nx;
    const int iy = (int)(r % ny), iz = (int)(r / ny);
    double s = 0.0;
    if (st.kind == 1) {
        const double* xv = x + v;
        if (ix >= st.rx && ix < nx - st.rx && iy >= st.ry && iy < ny - st.ry && iz >= st.rz && iz < st.nz - st.rz) {
#pragma unroll
            for (int k = 0; k < STENCIL_MAX_PTS; ++k) {    // interior: every point on the grid
                if (k >= st.npts) break;
                s = fma(st.c[k], xv[st.off[k]], s);
            }
            return s;
        }
#pragma unroll
        for (int k = 0; k < STENCIL_MAX_PTS; ++k) {
            if (k >= st.npts) break;
            const int a = ix + st.dx[k], b = iy + st.dy[k], c = iz + st.dz[k];
            if (a >= 0 && a < nx && b >= 0 && b < ny && c >= 0 && c < st.nz) s = fma(st.c[k], xv[st.off[k]], s);
        }
        return s;
    }
    const int64_t n = (int64_t)nx * ny * st.nz, sy = nx, sz = (int64_t)nx * ny;
    const double* D = st.coef;
    const double* CX = D + n;
    const double* CY = CX + n;
    const double* CZ = CY + n;
    if (iz > 0) s = fma(CZ[v - sz], x[v - sz], s);
    if (iy > 0) s = fma(CY[v - sy], x[v - sy], s);
    if (ix > 0) s = fma(CX[v - 1], x[v - 1], s);
    s = fma(D[v], x[v], s);
    if (ix + 1 < nx) s = fma(CX[v], x[v + 1], s);
    if (iy + 1 < ny) s = fma(CY[v], x[v + sy], s);
    if (iz + 1 < st.nz) s = fma(CZ[v], x[v + sz], s);
    return s;
}

// (A x)[v] by one thread: stencil or CSR row
__device__ __forceinline__ double row_dot1(const DevCSR& A, int64_t v, const double* __restrict__ x) {
    if (A.st.kind) return stencil_dot(A.st, v, x);
    double s = 0.0;
    for (int e = A.rp[v]; e < A.rp[v + 1]; e++) s += A.val[e] * x[A.col[e]];
    return s;
}

// CSR row only: the fused gathers of the per-item SYMV kernels (the stencil
// code would double their register allocation; the CSR rounds identically)
__device__ __forceinline__ double row_dot_csr(const DevCSR& A, int64_t v, const double* __restrict__ x) {
    double s = 0.0;
    for (int e = A.rp[v]; e < A.rp[v + 1]; e++) s += A.val[e] * x[A.col[e]];
    return s;
}

// (A x)[v] by SW lanes (an aligned group of the warp; sl = lane in group).
// Every lane of the warp must call it (the group reduction shuffles); rows
// with valid == false contribute 0.
template <int SW>
__device__ __forceinline__ double row_dot(const DevCSR& A, int64_t v, bool valid, const double* __restrict__ x,
                                          int sl) {
    double s = 0.0;
    if (SW == 1) return valid ? row_dot1(A, v, x) : 0.0;
    if (valid) {
        const int e1 = A.rp[v + 1];
        for (int e = A.rp[v] + sl; e < e1; e += SW) s += A.val[e] * x[A.col[e]];
    }
#pragma unroll
    for (int o = SW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    return s;
}

// block-wide sum; result valid in every thread. blockDim.x multiple of 32, <= 1024
__device__ double block_sum(double v) {
    __shared__ double ws[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) ws[w] = v;
    __syncthreads();
    double t = (threadIdx.x < nw) ? ws[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) ws[0] = t;
    __syncthreads();
    return ws[0];
}

// Grid reduction: every block contributes v; the last block to arrive sums
// the block partials in index order and calls fin(total) in thread 0.
template <typename Fin>
__device__ void grid_reduce(double v, double* red, unsigned* ticket, Fin fin) {
    __shared__ bool last;
    double b = block_sum(v);
    if (threadIdx.x == 0) {
        red[blockIdx.x] = b;
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        __threadfence();
        double s = 0.0;
        for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) s += __ldcg(red + i);
        s = block_sum(s);
        if (threadIdx.x == 0) {
            fin(s);
            *ticket = 0u;
        }
    }
}

// =============================================================================
// PCG vector kernels
// Rows: the rank's owned rows (rows == nullptr: rows 0..nrows-1).  Reductions
// end either in the last block (single rank) or, with `dist`, by storing the
// rank-local sum in sc->loc[slot] for an NCCL allreduce followed by
// k_pcg_finalize (multi-GPU).
// =============================================================================

#define ROW(i) (rows ? (int64_t)rows[i] : (i))

__device__ void fin_init(Scalars* sc, double* hist, double s) {
    const double r0 = sqrt(s);
    sc->res0 = r0;
    sc->ref = r0;
    sc->res = r0;
    hist[0] = r0;
    sc->iter = 0;
    sc->status = 0;
    sc->converged = (r0 == 0.0);
    sc->done = (r0 == 0.0);
}
__device__ void fin_rz_first(Scalars* sc, double s) {
    if (!(s > 0.0)) {
        sc->status = 7;  // DDG_E_BREAKDOWN
        sc->done = 1;
    } else {
        sc->rho = s;
        sc->pres0 = sqrt(s);
    }
}
__device__ void fin_spmv_dot(Scalars* sc, double s) {
    sc->sigma = s;
    if (!(s > 0.0)) {
        sc->status = 7;
        sc->done = 1;
    } else {
        sc->alpha = sc->rho / s;
        if (sc->ab) sc->ab[2 * sc->iter] = sc->alpha;
    }
}
__device__ void fin_update(Scalars* sc, double* hist, double s) {
    const double res = sqrt(s);
    const int it = sc->iter + 1;
    sc->iter = it;
    sc->res = res;
    hist[it] = res;
    if (sc->stop_mode == 1 && it == 1) sc->ref = res;
    bool conv = false;
    if (sc->stop_mode == 0) conv = res <= sc->rtol * sc->ref;
    if (sc->stop_mode == 1) conv = (it > 1) && res <= sc->rtol * sc->ref;
    if (res == 0.0) conv = true;
    if (conv) {
        sc->converged = 1;
        sc->done = 1;
    } else if (it >= sc->max_iter) {
        sc->done = 1;
    }
}
__device__ void fin_rz(Scalars* sc, double s) {
    if (sc->stop_mode == 2 && sqrt(fabs(s)) <= sc->rtol * sc->pres0) {
        sc->converged = 1;
        sc->done = 1;
    } else if (!(s > 0.0)) {
        sc->status = 7;
        sc->done = 1;
    } else {
        sc->beta = s / sc->rho;
        sc->rho = s;
        if (sc->ab) sc->ab[2 * (sc->iter - 1) + 1] = sc->beta;
    }
}

__global__ void k_pcg_init(int64_t n, const double* __restrict__ f, double* __restrict__ r,
                           double* __restrict__ u, const int32_t* __restrict__ rows, int64_t nrows, Scalars* sc,
                           double* hist, double* red, unsigned* ticket, int dist) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        r[i] = f[i];
        u[i] = 0.0;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = f[ROW(i)];
        acc += v * v;
    }
    grid_reduce(acc, red, ticket, [&](double s) {
        if (dist) { sc->loc[0] = s; sc->done = 0; return; }
        fin_init(sc, hist, s);
    });
}

// rho = r^T z ; p = z  (first direction)
__global__ void k_pcg_rz_first(const double* __restrict__ r, const double* __restrict__ z,
                               double* __restrict__ p, const int32_t* __restrict__ rows, int64_t nrows,
                               Scalars* sc, double* red, unsigned* ticket, int dist) {
    if (sc->done) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ROW(i);
        const double zi = z[v];
        p[v] = zi;
        acc += r[v] * zi;
    }
    grid_reduce(acc, red, ticket, [&](double s) {
        if (dist) { sc->loc[1] = s; return; }
        fin_rz_first(sc, s);
    });
}

// q = A p ; sigma = p^T q ; alpha = rho / sigma
template <int SW>
__global__ void k_pcg_spmv_dot(DevCSR A, const double* __restrict__ p, double* __restrict__ q,
                               const int32_t* __restrict__ rows, int64_t nrows, Scalars* sc, double* red,
                               unsigned* ticket, int dist) {
    if (sc->done) return;
    double acc = 0.0;
    const int64_t ng = (int64_t)gridDim.x * blockDim.x / SW;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / SW;
    const int sl = threadIdx.x % SW;
    for (int64_t base = 0; base < nrows; base += ng) {
        const int64_t i = base + g;
        const bool ok = i < nrows;
        const int64_t v = ok ? ROW(i) : 0;
        const double s = row_dot<SW>(A, v, ok, p, sl);
        if (ok && sl == 0) {
            q[v] = s;
            acc += p[v] * s;
        }
    }
    grid_reduce(acc, red, ticket, [&](double s) {
        if (dist) { sc->loc[2] = s; return; }
        fin_spmv_dot(sc, s);
    });
}

// u += alpha p ; r -= alpha q ; ||r|| ; history ; stopping rule (reading R1)
__global__ void k_pcg_update(const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ u,
                             double* __restrict__ r, const int32_t* __restrict__ rows, int64_t nrows, Scalars* sc,
                             double* hist, double* red, unsigned* ticket, int dist) {
    if (sc->done) return;
    const double alpha = sc->alpha;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ROW(i);
        u[v] += alpha * p[v];
        const double ri = r[v] - alpha * q[v];
        r[v] = ri;
        acc += ri * ri;
    }
    grid_reduce(acc, red, ticket, [&](double s) {
        if (dist) { sc->loc[3] = s; return; }
        fin_update(sc, hist, s);
    });
}

// rho' = r^T z ; beta = rho' / rho
__global__ void k_pcg_rz(const double* __restrict__ r, const double* __restrict__ z,
                         const int32_t* __restrict__ rows, int64_t nrows, Scalars* sc, double* red,
                         unsigned* ticket, int dist) {
    if (sc->done) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ROW(i);
        acc += r[v] * z[v];
    }
    grid_reduce(acc, red, ticket, [&](double s) {
        if (dist) { sc->loc[4] = s; return; }
        fin_rz(sc, s);
    });
}

// p = z + beta p
__global__ void k_pcg_direction(const double* __restrict__ z, double* __restrict__ p,
                                const int32_t* __restrict__ rows, int64_t nrows, const Scalars* sc) {
    if (sc->done) return;
    const double beta = sc->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = ROW(i);
        p[v] = z[v] + beta * p[v];
    }
}

// multi-GPU: apply the stopping / step logic to the allreduced sum
__global__ void k_pcg_finalize(int slot, Scalars* sc, double* hist) {
    const double s = sc->glob[slot];
    if (slot == 0) { fin_init(sc, hist, s); return; }
    if (sc->done) return;
    if (slot == 1) fin_rz_first(sc, s);
    else if (slot == 2) fin_spmv_dot(sc, s);
    else if (slot == 3) fin_update(sc, hist, s);
    else fin_rz(sc, s);
}

// halo exchange pack / unpack
__global__ void k_halo_pack(const double* __restrict__ v, const int32_t* __restrict__ idx, double* __restrict__ buf,
                            int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = v[idx[i]];
}
__global__ void k_halo_unpack(const double* __restrict__ buf, const int32_t* __restrict__ idx, double* __restrict__ v,
                              int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[idx[i]] = buf[i];
}
// out[rows] = in[rows] (assembly of rank-owned rows before an allreduce)
__global__ void k_copy_rows(const double* __restrict__ in, double* __restrict__ out,
                            const int32_t* __restrict__ rows, int64_t nrows) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
        out[rows[i]] = in[rows[i]];
}

__global__ void k_fill(double* x, int64_t n, double v, const int32_t* done) {
    if (done && *done) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void k_spmv(DevCSR A, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        y[i] = row_dot1(A, i, x);
    }
}

// =============================================================================
// Multiplicative Schwarz colour step
// =============================================================================

// flat residual restriction of one colour: x over its s segments
template <int SW>
__global__ void __launch_bounds__(256)
k_gather_flat(int64_t x0, int64_t x1, const int32_t* __restrict__ gidx, DevCSR A, const double* __restrict__ r,
              const double* __restrict__ z, double* __restrict__ s, int z_is_zero, const int32_t* done) {
    if (*done) return;
    const int64_t ng = (int64_t)gridDim.x * blockDim.x / SW;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / SW;
    const int sl = threadIdx.x % SW;
    for (int64_t base = x0; base < x1; base += ng) {
        const int64_t x = base + g;
        const int v = x < x1 ? gidx[x] : -1;
        const bool ok = v >= 0;
        const double az = z_is_zero ? 0.0 : row_dot<SW>(A, v, ok, z, sl);
        if (ok && sl == 0) s[x] = r[v] - az;
    }
}

__device__ __forceinline__ void item_tile(const ItemDesc& it, int l, int& I, int& J) {
    if (!it.tri) {
        const int wJ = it.J1 - it.J0;
        I = it.I0 + l / wJ;
        J = it.J0 + l % wJ;
    } else {
        int rr = (int)((sqrtf(8.0f * (float)l + 1.0f) - 1.0f) * 0.5f);
        while ((rr + 1) * (rr + 2) / 2 <= l) rr++;
        while (rr * (rr + 1) / 2 > l) rr--;
        I = it.I0 + rr;
        J = it.J0 + (l - rr * (rr + 1) / 2);
    }
}

// Diagonal tiles are stored as their lower triangle, column-major packed,
// with the diagonal halved: D = L' + L'^T, so a diagonal tile is applied
// exactly like an off-diagonal one (direct + transposed) from half the bytes.
__device__ __forceinline__ int diag_col_off(int j) { return j * TILE - j * (j - 1) / 2; }

// offset (doubles) of local tile l = (I, J) inside its item
__device__ __forceinline__ int64_t item_tile_off(const ItemDesc& it, int l, int I) {
    if (!it.tri) return (int64_t)l * TILE_ELEMS;
    const int rr = I - it.I0;                  // diagonal tiles of rows 0..rr-1 precede l
    return (int64_t)(l - rr) * TILE_ELEMS + (int64_t)rr * DIAG_ELEMS;
}

// lane i loads row i of tile (I, J) (packed form when I == J)
__device__ __forceinline__ void load_tile_row(double* a, const double* T, bool diag, int lane) {
    if (!diag) {
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] = __ldcs(T + j * TILE + lane);
    } else {
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] = lane >= j ? __ldcs(T + diag_col_off(j) + lane - j) : 0.0;
    }
}

// butterfly reduce-scatter of 32 per-lane values: afterwards v[0] of lane l
// holds sum over lanes of the original v[l].
template <int OFF>
__device__ __forceinline__ void rs_stage(double* v, int lane) {
    const bool upper = (lane & OFF) != 0;
#pragma unroll
    for (int j = 0; j < OFF; ++j) {
        double send = upper ? v[j] : v[j + OFF];
        double keep = upper ? v[j + OFF] : v[j];
        v[j] = keep + __shfl_xor_sync(FULL, send, OFF);
    }
}

// Tiled symmetric matrix-vector product y = S s over one item-block of a
// packed symmetric operator.  Warp w handles tiles w, w+W, ...; lane i owns
// row i of each tile: direct part y_I += S_IJ s_J by per-lane dot products,
// transposed part y_J += S_IJ^T s_I by a butterfly reduce-scatter.  Per-warp
// partials in shared memory are summed in warp order (deterministic).
__global__ void __launch_bounds__(SYMV_WARPS * 32)
k_symv(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin,
       const double* __restrict__ tiles, const double* __restrict__ s,
       const int32_t* __restrict__ oidx, double* __restrict__ z, double* __restrict__ y_out,
       double* __restrict__ partials, const int32_t* done, unsigned* __restrict__ tickets,
       int gather_mode, DevCSR A, const double* __restrict__ rvec) {
    if (*done) return;
    extern __shared__ double sm[];
    const ItemDesc it = items[item_begin + blockIdx.x];
    const OpDesc op = ops[it.op];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rows_r = (it.I1 - it.I0) * TILE;
    const int rows_c = it.tri ? 0 : (it.J1 - it.J0) * TILE;
    const int rows_t = rows_r + rows_c;
    double* s_sm = sm;                          // [rows_t]: s over row block, then col block
    double* part = sm + rows_t;                 // [SYMV_WARPS][rows_t]
    const double* tbase = tiles + it.tile_off;
    // issue this warp's first tile loads now: their latency overlaps the prologue
    double a[TILE];
    if (w < it.ntiles) {
        int I0_, J0_;
        item_tile(it, w, I0_, J0_);
        load_tile_row(a, tbase + item_tile_off(it, w, I0_), I0_ == J0_, lane);
    }
    if (gather_mode) {
        // fused residual restriction (single-item operators): s = R~_i (r - A z)
        const int32_t* idx = oidx + op.idx_off;
        for (int x = threadIdx.x; x < rows_t; x += blockDim.x) {
            double v = 0.0;
            if (x < op.m) {
                const int node = idx[x];
                double az = 0.0;
                if (gather_mode == 1)
                    az = row_dot_csr(A, node, z);
                v = rvec[node] - az;
            }
            s_sm[x] = v;
        }
    } else {
        const double* sop = s + op.s_off;
        for (int x = threadIdx.x; x < rows_t; x += blockDim.x) {
            int g = x < rows_r ? it.I0 * TILE + x : it.J0 * TILE + (x - rows_r);
            s_sm[x] = sop[g];
        }
    }
    for (int x = threadIdx.x; x < SYMV_WARPS * rows_t; x += blockDim.x) part[x] = 0.0;
    __syncthreads();
    double* pw = part + w * rows_t;
    for (int l = w; l < it.ntiles; l += SYMV_WARPS) {
        int I, J;
        item_tile(it, l, I, J);
        if (l != w) load_tile_row(a, tbase + item_tile_off(it, l, I), I == J, lane);
        const int ri = (I - it.I0) * TILE;                           // row offset in s_sm / pw
        const int cj = it.tri ? (J - it.I0) * TILE : rows_r + (J - it.J0) * TILE;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < TILE; ++j) acc += a[j] * s_sm[cj + j];
        const double si = s_sm[ri + lane];
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] *= si;
        rs_stage<16>(a, lane);
        rs_stage<8>(a, lane);
        rs_stage<4>(a, lane);
        rs_stage<2>(a, lane);
        rs_stage<1>(a, lane);
        if (I != J) {
            pw[ri + lane] += acc;
            pw[cj + lane] += a[0];
        } else {
            pw[ri + lane] += acc + a[0];
        }
    }
    __syncthreads();
    const bool single = it.part_off < 0;
    for (int x = threadIdx.x; x < rows_t; x += blockDim.x) {
        double y = 0.0;
#pragma unroll
        for (int ww = 0; ww < SYMV_WARPS; ++ww) y += part[ww * rows_t + x];
        if (single) {
            const int g = it.I0 * TILE + x;     // single-item op: one triangle from 0
            if (g < op.m) {
                if (op.out_mode == 0) z[oidx[op.idx_off + g]] += y;
                else y_out[g] = y;
            }
        } else {
            partials[it.part_off + x] = y;
        }
    }
    if (single || op.out_mode == 2) return;   // fronts: reduced by k_front_reduce
    // multi-item operator: the last CTA to finish it sums every row's partial
    // segments in fixed item order (deterministic) and applies the result
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(&tickets[it.op], 1u) == (unsigned)op.nitems - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int rb = op.BT * TILE;
    for (int g = threadIdx.x; g < op.m; g += blockDim.x) {
        const int b = g / rb, x = g % rb;
        double y = 0.0;
        for (int j = 0; j <= b; ++j) {
            const ItemDesc& ij = items[op.item_base + b * (b + 1) / 2 + j];
            y += __ldcg(partials + ij.part_off + x);
        }
        for (int i = b + 1; i < op.nblk; ++i) {
            const ItemDesc& ii = items[op.item_base + i * (i + 1) / 2 + b];
            y += __ldcg(partials + ii.part_off + (ii.I1 - ii.I0) * TILE + x);
        }
        if (op.out_mode == 0) z[oidx[op.idx_off + g]] += y;
        else y_out[g] = y;
    }
    if (threadIdx.x == 0) tickets[it.op] = 0u;
}

// ---- warp-per-subdomain SYMV for small single-item operators (nT <= 8) ----
// Each warp owns one subdomain end to end: fused residual restriction, all
// tiles (two in flight: register double buffer), its own shared y, scatter.
// No CTA barrier anywhere, so warps of a CTA stream independently.
constexpr int SMALL_MAXROWS = 256;

__device__ __forceinline__ void tile_apply(const double* __restrict__ a_in, double* a, const double* s,
                                           double* y, int ri, int cj, bool diag, int lane) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < TILE; ++j) acc += a_in[j] * s[cj + j];
    const double si = s[ri + lane];
#pragma unroll
    for (int j = 0; j < TILE; ++j) a[j] = a_in[j] * si;
    rs_stage<16>(a, lane);
    rs_stage<8>(a, lane);
    rs_stage<4>(a, lane);
    rs_stage<2>(a, lane);
    rs_stage<1>(a, lane);
    if (!diag) {
        y[ri + lane] += acc;
        __syncwarp();
        y[cj + lane] += a[0];
    } else {
        y[ri + lane] += acc + a[0];
    }
    __syncwarp();
}

__global__ void __launch_bounds__(256)
k_symv_small(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin, int nitems,
             const double* __restrict__ tiles, const double* __restrict__ s, const int32_t* __restrict__ oidx,
             double* __restrict__ z, double* __restrict__ y_out, const int32_t* done, int gather_mode, DevCSR A,
             const double* __restrict__ rvec) {
    if (*done) return;
    __shared__ double ssm[8][SMALL_MAXROWS];
    __shared__ double ysm[8][SMALL_MAXROWS];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ii = blockIdx.x * 8 + w;
    if (ii >= nitems) return;
    const ItemDesc it = items[item_begin + ii];
    const OpDesc op = ops[it.op];
    const double* tb = tiles + it.tile_off;
    double a[TILE], b[TILE];
    int I = 0, J = 0;
    item_tile(it, 0, I, J);
    load_tile_row(a, tb + item_tile_off(it, 0, I), I == J, lane);       // first tile in flight
    double* sw = ssm[w];
    double* yw = ysm[w];
    const int32_t* idx = oidx + op.idx_off;
    for (int x = lane; x < op.mp; x += 32) {
        double v = 0.0;
        if (x < op.m) {
            if (gather_mode) {
                const int node = idx[x];
                double az = 0.0;
                if (gather_mode == 1)
                    az = row_dot_csr(A, node, z);
                v = rvec[node] - az;
            } else {
                v = s[op.s_off + x];
            }
        }
        sw[x] = v;
        yw[x] = 0.0;
    }
    __syncwarp();
    for (int l = 0; l < it.ntiles; l += 2) {
        int I1 = 0, J1 = 0;
        const bool has1 = l + 1 < it.ntiles;
        if (has1) {
            item_tile(it, l + 1, I1, J1);
            load_tile_row(b, tb + item_tile_off(it, l + 1, I1), I1 == J1, lane);
        }
        tile_apply(a, a, sw, yw, I * TILE, J * TILE, I == J, lane);
        if (l + 2 < it.ntiles) {
            item_tile(it, l + 2, I, J);
            load_tile_row(a, tb + item_tile_off(it, l + 2, I), I == J, lane);
        }
        if (has1) tile_apply(b, b, sw, yw, I1 * TILE, J1 * TILE, I1 == J1, lane);
    }
    for (int x = lane; x < op.m; x += 32) {
        if (op.out_mode == 0) z[idx[x]] += yw[x];
        else y_out[x] = yw[x];
    }
}

// ---- mbarrier / bulk-copy helpers (TMA, sm_90+) -----------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// ---- persistent streaming SYMV: bulk-copy ring, warp-specialised ----------
// One CTA per SM walks a byte-balanced contiguous range of the launch's items
// (host partition `cta_part`).  Roles:
//  * warp 8 lane 0 (producer): streams each item's s segment(s) and its tiles
//    (RING_TILES tiles per chunk, <= 32 KB) into shared memory with
//    cp.async.bulk + mbarrier complete_tx, up to RING_NST chunks ahead and
//    across item boundaries, so HBM never waits on the consumers;
//  * warps 0-7 (consumers): each owns a fixed set of the item's tiles and
//    progresses independently of the other consumer warps.  Tile (I, J):
//    direct part y_I += S_IJ s_J by per-lane dot products into the warp's
//    partial rows; transposed part y_J += S_IJ^T s_I accumulated per lane in
//    registers (t[j] += S_IJ[lane][j] s_I[lane]) over the warp's consecutive
//    tiles of the same column J, then one butterfly reduce-scatter per column
//    run.  Owner of a tile: l % 8 in rectangular items (= its column for the
//    8-wide blocks), (J + item counter) % 8 in triangles (one column per warp,
//    rotated across items so the long columns are spread over the warps);
//  * warp 9 (epilogue): sums the 8 warps' partial rows in warp order
//    (deterministic) and applies them -- z[idx] += y with idx and z prefetched
//    before the item finishes (same-colour subdomains are disjoint), y_out = y,
//    or the partial segment of a multi-item operator (reduced later).
// Partial rows are double-buffered by item parity, so consumer warps never
// wait for each other.  Measured ceiling of this access pattern:
// tools/bwprobe.cu ("tma ring" rows).
constexpr int RING_EPI_WARPS = 2;
constexpr int RING_THREADS = (SYMV_WARPS + 1 + RING_EPI_WARPS) * 32;
constexpr int RING_MAX_NST = 24;
constexpr int RING_MAX_NB = 8;
// shared memory of a launch: nst slots of RT tiles; nb item buffers, each the
// item's s (maxr rows), the 8 consumer warps' partial rows and a descriptor;
// barriers
__host__ __device__ constexpr size_t ring_smem(int RT, int nst, int nb, int R, int Cr) {
    return (size_t)nst * RT * TILE_ELEMS * 8 + (size_t)nb * (R + Cr) * 8 + (size_t)nb * (SYMV_WARPS * R + Cr) * 8 +
           (size_t)nb * 8 * 4 + (2 * (size_t)nst + 4 * (size_t)nb) * 8;
}

// first double of tile l of item it (l == ntiles: one past the last tile)
__device__ __forceinline__ int64_t item_tile_off_l(const ItemDesc& it, int l) {
    if (l >= it.ntiles) return item_doubles(it.tri, it.I1 - it.I0, it.ntiles);
    int I, J;
    item_tile(it, l, I, J);
    return item_tile_off(it, l, I);
}

// descriptors of the next items, fetched ahead so no role stalls on them
struct DescPipe {
    ItemDesc it1, it2;
    OpDesc op1;
    __device__ __forceinline__ void init(const ItemDesc* items, const OpDesc* ops, int i0, int i1) {
        it1 = items[i0];
        op1 = ops[it1.op];
        if (i0 + 1 < i1) it2 = items[i0 + 1];
    }
    __device__ __forceinline__ void next(const ItemDesc* items, const OpDesc* ops, int ii, int i1, ItemDesc& it,
                                         OpDesc& op) {
        it = it1;
        op = op1;
        if (ii + 1 < i1) {
            it1 = it2;
            op1 = ops[it1.op];
        }
        if (ii + 2 < i1) it2 = items[ii + 2];
    }
};

__device__ __forceinline__ void flush_column(double* t, double* pw, int cj, int lane) {
    rs_stage<16>(t, lane);
    rs_stage<8>(t, lane);
    rs_stage<4>(t, lane);
    rs_stage<2>(t, lane);
    rs_stage<1>(t, lane);
    pw[cj + lane] += t[0];
}

template <int RT>
__global__ void __launch_bounds__(RING_THREADS, 1)
k_symv_ring(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin,
            const int32_t* __restrict__ cta_part, const double* __restrict__ tiles, const double* __restrict__ s,
            const int32_t* __restrict__ oidx, double* __restrict__ z, double* __restrict__ y_out,
            double* __restrict__ partials, const int32_t* done, int nst, int nb, int R, int Cr,
            unsigned long long* rtrace) {
    constexpr int SLOT = RT * TILE_ELEMS;
    // item buffers: s over R + Cr rows; partial rows: the row block replicated
    // per consumer warp ([8][R], every warp adds direct parts to any row) and
    // the column block of rectangles once ([Cr], each column has one owner)
    const int maxr = R + Cr, PB = SYMV_WARPS * R + Cr;
    // DDG_RING_TRACE: cycles per role and wait (debug; rtrace == nullptr otherwise)
    unsigned long long tw[4] = {0, 0, 0, 0}, tstart = rtrace ? clock64() : 0, ntile = 0, nflush = 0;
#define RT_WAIT(k, call)                                        \
    do {                                                        \
        if (rtrace) {                                           \
            const unsigned long long t0_ = clock64();           \
            call;                                               \
            tw[k] += clock64() - t0_;                           \
        } else {                                                \
            call;                                               \
        }                                                       \
    } while (0)
#define RT_FLUSH(base)                                                                  \
    do {                                                                                \
        if (rtrace && lane == 0) {                                                      \
            atomicAdd(&rtrace[(base)], tw[0]);                                          \
            atomicAdd(&rtrace[(base) + 1], tw[1]);                                      \
            atomicAdd(&rtrace[(base) + 2], tw[2]);                                      \
            atomicAdd(&rtrace[(base) + 3], clock64() - tstart);                         \
            atomicAdd(&rtrace[(base) + 4], ntile);                                      \
            atomicAdd(&rtrace[(base) + 5], nflush);                                     \
            atomicAdd(&rtrace[(base) + 6], tw[3]);                                      \
        }                                                                               \
    } while (0)
    if (*done) return;
    extern __shared__ __align__(128) double rsm[];
    double* ring = rsm;                                          // [nst][SLOT]
    double* s_sm = ring + (size_t)nst * SLOT;                    // [nb][maxr]
    double* part = s_sm + (size_t)nb * maxr;                     // [nb][PB]
    int32_t* dsc = reinterpret_cast<int32_t*>(part + (size_t)nb * PB);   // [nb][8]
    uint64_t* full = reinterpret_cast<uint64_t*>(dsc + nb * 8);
    uint64_t* empty = full + nst;
    uint64_t* sfull = empty + nst;    // [nb] s + descriptor of the item landed
    uint64_t* sempty = sfull + nb;    // [nb] consumers done with the item's s
    uint64_t* pdone = sempty + nb;    // [nb] consumers' partial rows final
    uint64_t* pfree = pdone + nb;     // [nb] epilogue done with the partial rows
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = item_begin + cta_part[blockIdx.x], i1 = item_begin + cta_part[blockIdx.x + 1];
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], SYMV_WARPS);                  // every consumer warp, every chunk
        }
        for (int b = 0; b < nb; ++b) {
            mbar_init(&sfull[b], 1);
            mbar_init(&sempty[b], SYMV_WARPS);
            mbar_init(&pdone[b], SYMV_WARPS * 32);
            mbar_init(&pfree[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (i0 >= i1) return;
    if (warp == SYMV_WARPS) {                                    // ---- producer warp ----
        // Lane 0 owns the barriers; the tile copies of a triangle chunk are
        // issued by lanes 0..nt-1 in one instruction (a bulk-copy issue costs
        // the issuing thread a few hundred cycles: one per lane overlaps them).
        DescPipe dp;
        dp.init(items, ops, i0, i1);
        unsigned slot = 0, sph = 0;                                // ring slot and its fill count
        int bi = 0;
        unsigned bph = 0;                                          // item buffer and its use count
        for (int ii = i0; ii < i1; ++ii) {
            ItemDesc it;
            OpDesc op;
            RT_WAIT(2, dp.next(items, ops, ii, i1, it, op); it.tri += 0);
            const int rows_r = (it.I1 - it.I0) * TILE, rows_c = it.tri ? 0 : (it.J1 - it.J0) * TILE;
            if (bph > 0) RT_WAIT(0, mbar_wait(&sempty[bi], (bph - 1) & 1));
            if (lane == 0) {
                int32_t* d = dsc + bi * 8;
                d[0] = it.I0; d[1] = it.I1; d[2] = it.J0; d[3] = it.J1; d[4] = it.tri; d[5] = it.ntiles;
                mbar_expect_tx(&sfull[bi], (unsigned)(rows_r + rows_c) * 8u);
            }
            __syncwarp();
            const double* sop = s + op.s_off;
            double* sb = s_sm + (size_t)bi * maxr;
            if (lane == 0) bulk_g2s(sb, sop + it.I0 * TILE, rows_r * 8u, &sfull[bi]);
            if (lane == 1 && rows_c) bulk_g2s(sb + rows_r, sop + it.J0 * TILE, rows_c * 8u, &sfull[bi]);
            if (++bi == nb) { bi = 0; ++bph; }
            // tile q of a chunk always lands at q * 8 KB of its slot; rectangular
            // items are contiguous full tiles (one copy per chunk), triangles
            // copy tile by tile (packed diagonal tiles are 4224 B)
            const double* src = tiles + it.tile_off;
            for (int l0 = 0; l0 < it.ntiles; l0 += RT) {
                const int nt = min(RT, it.ntiles - l0);
                if (sph > 0) RT_WAIT(1, mbar_wait(&empty[slot], (sph - 1) & 1));
                const unsigned long long tc0 = rtrace ? clock64() : 0;
                double* dst = ring + (size_t)slot * SLOT;
                if (!it.tri) {
                    if (lane == 0) {
                        mbar_expect_tx(&full[slot], (unsigned)nt * TILE_ELEMS * 8u);
                        bulk_g2s(dst, src + (int64_t)l0 * TILE_ELEMS, (unsigned)nt * TILE_ELEMS * 8u, &full[slot]);
                    }
                } else {
                    unsigned tb = 0;
                    int64_t toff = 0;
                    if (lane < nt) {
                        int I_, J_;
                        item_tile(it, l0 + lane, I_, J_);
                        tb = (I_ == J_ ? DIAG_ELEMS : TILE_ELEMS) * 8u;
                        toff = item_tile_off(it, l0 + lane, I_);
                    }
                    unsigned bytes = tb;
#pragma unroll
                    for (int o = 1; o < RT; o <<= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
                    if (lane == 0) mbar_expect_tx(&full[slot], bytes);
                    __syncwarp();
                    if (lane < nt) bulk_g2s(dst + lane * TILE_ELEMS, src + toff, tb, &full[slot]);
                }
                if (rtrace) tw[3] += clock64() - tc0;
                if (++slot == (unsigned)nst) { slot = 0; ++sph; }
            }
        }
        RT_FLUSH(0);
        return;
    }
    if (warp > SYMV_WARPS) {                                     // ---- epilogue warps ----
        const int e = warp - SYMV_WARPS - 1;                      // handles items ki = e, e+E, ...
        for (int ii = i0 + e, ki = e; ii < i1; ii += RING_EPI_WARPS, ki += RING_EPI_WARPS) {
            const ItemDesc it = items[ii];
            const OpDesc op = ops[it.op];
            const int b = ki % nb;
            const unsigned ph = (unsigned)(ki / nb);
            const int rows_t = (it.I1 - it.I0 + (it.tri ? 0 : it.J1 - it.J0)) * TILE;
            const int g0 = it.I0 * TILE;
            const int nr = min(rows_t, op.m - g0);                // single-item ops only
            const bool scat = it.part_off < 0 && op.out_mode == 0;
            int ix[RING_MAX_ROWS / 32];
            double zv[RING_MAX_ROWS / 32];
            if (scat) {
                const int32_t* idx = oidx + op.idx_off + g0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) ix[r] = (lane + 32 * r < nr) ? idx[lane + 32 * r] : 0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) zv[r] = (lane + 32 * r < nr) ? z[ix[r]] : 0.0;
            }
            RT_WAIT(0, mbar_wait(&pdone[b], ph & 1));
            const double* pp = part + (size_t)b * PB;
            const int rows_r = (it.I1 - it.I0) * TILE;
#pragma unroll
            for (int r = 0; r < RING_MAX_ROWS / 32; ++r) {
                const int x = lane + 32 * r;
                if (x < rows_t) {
                    double y = 0.0;
                    if (x < rows_r) {
#pragma unroll
                        for (int ww = 0; ww < SYMV_WARPS; ++ww) y += pp[ww * R + x];
                    } else {
                        y = pp[SYMV_WARPS * R + x - rows_r];       // column block (one owner)
                    }
                    if (it.part_off >= 0) partials[it.part_off + x] = y;
                    else if (x < nr) {
                        if (scat) z[ix[r]] = zv[r] + y;
                        else y_out[g0 + x] = y;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfree[b]);
        }
        RT_FLUSH(8);
        return;
    }
    // ---- consumers (warps 0..7): each walks only its own tiles ----
    unsigned slot = 0, sph = 0;
    int bi = 0;
    unsigned bph = 0;
    for (int ki = 0; ki < i1 - i0; ++ki) {
        RT_WAIT(0, mbar_wait(&sfull[bi], bph & 1));
        const int32_t* d = dsc + bi * 8;
        const int I0 = d[0], I1 = d[1], J0 = d[2], J1 = d[3], tri = d[4], ntiles = d[5];
        const double* ss = s_sm + (size_t)bi * maxr;
        const int rows_r = (I1 - I0) * TILE;
        const int rows_t = rows_r + (tri ? 0 : (J1 - J0) * TILE);
        double* pw = part + (size_t)bi * PB + (size_t)warp * R;    // this warp's row-block rows
        double* pcb = part + (size_t)bi * PB + SYMV_WARPS * R;     // column block (rectangles)
        if (bph > 0) RT_WAIT(1, mbar_wait(&pfree[bi], (bph - 1) & 1));
        for (int x = lane; x < rows_r; x += 32) pw[x] = 0.0;
        __syncwarp();
        double t[TILE];
#pragma unroll
        for (int j = 0; j < TILE; ++j) t[j] = 0.0;
        int curJ = -1;
        auto tile = [&](const double* T, int I, int J) {
            const int ri = (I - I0) * TILE;
            const int cj = tri ? (J - I0) * TILE : rows_r + (J - J0) * TILE;
            ++ntile;
            if (J != curJ) {
                if (curJ >= 0) {                                   // (triangles only: one column per
                    ++nflush;                                      //  warp in a rectangle)
                    flush_column(t, pw, (curJ - I0) * TILE, lane);
#pragma unroll
                    for (int j = 0; j < TILE; ++j) t[j] = 0.0;
                }
                curJ = J;
            }
            double a[TILE];
            if (I != J) {
#pragma unroll
                for (int j = 0; j < TILE; ++j) a[j] = T[j * TILE + lane];
            } else {
#pragma unroll
                for (int j = 0; j < TILE; ++j) a[j] = lane >= j ? T[diag_col_off(j) + lane - j] : 0.0;
            }
            const double2* sJ = reinterpret_cast<const double2*>(ss + cj);
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int j = 0; j < TILE; j += 4) {
                const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                d0 = fma(a[j], u.x, d0);
                d1 = fma(a[j + 1], u.y, d1);
                d2 = fma(a[j + 2], v.x, d2);
                d3 = fma(a[j + 3], v.y, d3);
            }
            pw[ri + lane] += (d0 + d1) + (d2 + d3);
            const double si = ss[ri + lane];
#pragma unroll
            for (int j = 0; j < TILE; ++j) t[j] = fma(a[j], si, t[j]);
        };
        // own-tile iterator, in increasing l.  Rectangles: column warp of every
        // row (l = r * wd + warp; warps >= wd idle); each column has one owner.
        // Triangles: columns c0 = (warp - ki) mod 8, c0+8, ... of rows r >= c.
        int l = -1, I = 0, J = 0, r = 0, c = 0;
        const int h = I1 - I0, wd = J1 - J0, c0 = (warp - ki) & (SYMV_WARPS - 1);
        if (!tri) {
            if (warp < wd) { l = warp; I = I0; J = J0 + warp; }
        } else if (c0 < h) {
            r = c0; c = c0; l = r * (r + 1) / 2 + c; I = I0 + r; J = J0 + c;
        }
        auto advance = [&]() {
            if (!tri) {
                l += wd;
                ++I;
                if (I >= I1) l = -1;
            } else {
                c += SYMV_WARPS;
                if (c > r) { ++r; c = c0; }
                if (r >= h) { l = -1; return; }
                l = r * (r + 1) / 2 + c; I = I0 + r; J = J0 + c;
            }
        };
        // every warp visits every chunk in order (keeps the mbarrier phases
        // of each slot in step), consuming only its own tiles
        for (int l0 = 0; l0 < ntiles; l0 += RT) {
            RT_WAIT(2, mbar_wait(&full[slot], sph & 1));
            const double* C = ring + (size_t)slot * SLOT;
            while (l >= 0 && l < l0 + RT) {
                tile(C + (l - l0) * TILE_ELEMS, I, J);
                advance();
            }
            __syncwarp();                                          // every lane has consumed its rows
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == (unsigned)nst) { slot = 0; ++sph; }
        }
        if (curJ >= 0) {
            if (tri) {
                flush_column(t, pw, (curJ - I0) * TILE, lane);
            } else {                                               // sole owner of this column
                rs_stage<16>(t, lane);
                rs_stage<8>(t, lane);
                rs_stage<4>(t, lane);
                rs_stage<2>(t, lane);
                rs_stage<1>(t, lane);
                pcb[(curJ - J0) * TILE + lane] = t[0];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[bi]);
        mbar_arrive(&pdone[bi]);                                   // every lane (release its rows)
        if (++bi == nb) { bi = 0; ++bph; }
    }
    RT_FLUSH(16);
#undef RT_WAIT
#undef RT_FLUSH
}

// ---- k_symv_ring2: row warps + column warps ----------------------------------
// Same producer, ring, item buffers and epilogue as k_symv_ring; the 16
// consumer warps split each tile's two products by role:
//  * row warps (0-7): own tile rows r (owner (r + item counter) mod 8); lane i
//    accumulates the direct part y_I[i] += sum_j S_IJ[i][j] s_J[j] in one
//    register across the row's tiles, then writes pr[row] once;
//  * column warps (8-15): own tile columns c; lane j accumulates the
//    transposed part y_J[j] += sum_i S_IJ[i][j] s_I[i] walking the tile along a
//    rotated diagonal (i = (t + j) mod 32: two wavefronts per load, no bank
//    conflicts) with s_I rotated by shuffles; one register per owned column,
//    written to pc[column] at the end of the item.
// Every row and column has a single owner, so the item's result is
// y = pr + pc (triangles) or pr | pc (rectangles: row block | column block)
// -- two partial arrays instead of eight, no butterfly, ~40 registers per
// consumer thread.
constexpr int R2_ROWW = 8, R2_COLW = 8, R2_CONS = R2_ROWW + R2_COLW;
constexpr int RING2_THREADS = (R2_CONS + 1 + RING_EPI_WARPS) * 32;
__host__ __device__ constexpr size_t ring2_smem(int RT, int nst, int nb, int maxr) {
    return (size_t)nst * RT * TILE_ELEMS * 8 + (size_t)nb * 3 * maxr * 8 + (size_t)nb * 8 * 4 +
           (2 * (size_t)nst + 4 * (size_t)nb) * 8;
}

template <int RT>
__global__ void __launch_bounds__(RING2_THREADS, 1)
k_symv_ring2(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin,
             const int32_t* __restrict__ cta_part, const double* __restrict__ tiles, const double* __restrict__ s,
             const int32_t* __restrict__ oidx, double* __restrict__ z, double* __restrict__ y_out,
             double* __restrict__ partials, const int32_t* done, int nst, int nb, int maxr) {
    constexpr int SLOT = RT * TILE_ELEMS;
    if (*done) return;
    extern __shared__ __align__(128) double rsm[];
    double* ring = rsm;                                          // [nst][SLOT]
    double* s_sm = ring + (size_t)nst * SLOT;                    // [nb][maxr]
    double* pr_sm = s_sm + (size_t)nb * maxr;                    // [nb][maxr]  row (direct) parts
    double* pc_sm = pr_sm + (size_t)nb * maxr;                   // [nb][maxr]  column (transposed) parts
    int32_t* dsc = reinterpret_cast<int32_t*>(pc_sm + (size_t)nb * maxr);   // [nb][8]
    uint64_t* full = reinterpret_cast<uint64_t*>(dsc + nb * 8);
    uint64_t* empty = full + nst;
    uint64_t* sfull = empty + nst;
    uint64_t* sempty = sfull + nb;
    uint64_t* pdone = sempty + nb;
    uint64_t* pfree = pdone + nb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = item_begin + cta_part[blockIdx.x], i1 = item_begin + cta_part[blockIdx.x + 1];
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], R2_CONS);
        }
        for (int b = 0; b < nb; ++b) {
            mbar_init(&sfull[b], 1);
            mbar_init(&sempty[b], R2_CONS);
            mbar_init(&pdone[b], R2_CONS * 32);
            mbar_init(&pfree[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (i0 >= i1) return;
    if (warp == R2_CONS) {                                       // ---- producer warp ----
        DescPipe dp;
        dp.init(items, ops, i0, i1);
        unsigned slot = 0, sph = 0;
        int bi = 0;
        unsigned bph = 0;
        for (int ii = i0; ii < i1; ++ii) {
            ItemDesc it;
            OpDesc op;
            dp.next(items, ops, ii, i1, it, op);
            const int rows_r = (it.I1 - it.I0) * TILE, rows_c = it.tri ? 0 : (it.J1 - it.J0) * TILE;
            if (bph > 0) mbar_wait(&sempty[bi], (bph - 1) & 1);
            if (lane == 0) {
                int32_t* d = dsc + bi * 8;
                d[0] = it.I0; d[1] = it.I1; d[2] = it.J0; d[3] = it.J1; d[4] = it.tri; d[5] = it.ntiles;
                mbar_expect_tx(&sfull[bi], (unsigned)(rows_r + rows_c) * 8u);
            }
            __syncwarp();
            const double* sop = s + op.s_off;
            double* sb = s_sm + (size_t)bi * maxr;
            if (lane == 0) bulk_g2s(sb, sop + it.I0 * TILE, rows_r * 8u, &sfull[bi]);
            if (lane == 1 && rows_c) bulk_g2s(sb + rows_r, sop + it.J0 * TILE, rows_c * 8u, &sfull[bi]);
            if (++bi == nb) { bi = 0; ++bph; }
            const double* src = tiles + it.tile_off;
            for (int l0 = 0; l0 < it.ntiles; l0 += RT) {
                const int nt = min(RT, it.ntiles - l0);
                if (sph > 0) mbar_wait(&empty[slot], (sph - 1) & 1);
                double* dst = ring + (size_t)slot * SLOT;
                if (!it.tri) {
                    if (lane == 0) {
                        mbar_expect_tx(&full[slot], (unsigned)nt * TILE_ELEMS * 8u);
                        bulk_g2s(dst, src + (int64_t)l0 * TILE_ELEMS, (unsigned)nt * TILE_ELEMS * 8u, &full[slot]);
                    }
                } else {
                    unsigned tb = 0;
                    int64_t toff = 0;
                    if (lane < nt) {
                        int I_, J_;
                        item_tile(it, l0 + lane, I_, J_);
                        tb = (I_ == J_ ? DIAG_ELEMS : TILE_ELEMS) * 8u;
                        toff = item_tile_off(it, l0 + lane, I_);
                    }
                    unsigned bytes = tb;
#pragma unroll
                    for (int o = 1; o < RT; o <<= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
                    if (lane == 0) mbar_expect_tx(&full[slot], bytes);
                    __syncwarp();
                    if (lane < nt) bulk_g2s(dst + lane * TILE_ELEMS, src + toff, tb, &full[slot]);
                }
                if (++slot == (unsigned)nst) { slot = 0; ++sph; }
            }
        }
        return;
    }
    if (warp > R2_CONS) {                                        // ---- epilogue warps ----
        const int e = warp - R2_CONS - 1;
        for (int ii = i0 + e, ki = e; ii < i1; ii += RING_EPI_WARPS, ki += RING_EPI_WARPS) {
            const ItemDesc it = items[ii];
            const OpDesc op = ops[it.op];
            const int b = ki % nb;
            const unsigned ph = (unsigned)(ki / nb);
            const int rows_r = (it.I1 - it.I0) * TILE;
            const int rows_t = rows_r + (it.tri ? 0 : (it.J1 - it.J0) * TILE);
            const int g0 = it.I0 * TILE;
            const int nr = min(rows_t, op.m - g0);
            const bool scat = it.part_off < 0 && op.out_mode == 0;
            int ix[RING_MAX_ROWS / 32];
            double zv[RING_MAX_ROWS / 32];
            if (scat) {
                const int32_t* idx = oidx + op.idx_off + g0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) ix[r] = (lane + 32 * r < nr) ? idx[lane + 32 * r] : 0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) zv[r] = (lane + 32 * r < nr) ? z[ix[r]] : 0.0;
            }
            mbar_wait(&pdone[b], ph & 1);
            const double* pr = pr_sm + (size_t)b * maxr;
            const double* pc = pc_sm + (size_t)b * maxr;
#pragma unroll
            for (int r = 0; r < RING_MAX_ROWS / 32; ++r) {
                const int x = lane + 32 * r;
                if (x < rows_t) {
                    const double y = it.tri ? pr[x] + pc[x] : (x < rows_r ? pr[x] : pc[x]);
                    if (it.part_off >= 0) partials[it.part_off + x] = y;
                    else if (x < nr) {
                        if (scat) z[ix[r]] = zv[r] + y;
                        else y_out[g0 + x] = y;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfree[b]);
        }
        return;
    }
    // ---- consumers: row warps 0..7, column warps 8..15 ----
    const bool colw = warp >= R2_ROWW;
    const int wr = colw ? warp - R2_ROWW : warp;
    unsigned slot = 0, sph = 0;
    int bi = 0;
    unsigned bph = 0;
    for (int ki = 0; ki < i1 - i0; ++ki) {
        mbar_wait(&sfull[bi], bph & 1);
        const int32_t* d = dsc + bi * 8;
        const int I0 = d[0], I1 = d[1], J1 = d[3], tri = d[4], ntiles = d[5];
        const int J0 = d[2];
        const double* ss = s_sm + (size_t)bi * maxr;
        const int h = I1 - I0, wd = tri ? h : J1 - J0;
        const int rows_r = h * TILE;
        double* pr = pr_sm + (size_t)bi * maxr;
        double* pc = pc_sm + (size_t)bi * maxr;
        if (bph > 0) mbar_wait(&pfree[bi], (bph - 1) & 1);
        // own tiles in increasing stream index l:
        //   row warp:    rows a, a + 8 (a = (wr - ki) mod 8), each row's tiles in order
        //   column warp: columns a, a + 8; per row r both owned columns in order
        const int a = (wr - ki) & 7;
        int l = -1, r = 0, c = 0, ccur = 0;
        double acc = 0.0, acc0 = 0.0, acc1 = 0.0;
        auto rowstart = [&](int rr) { return tri ? rr * (rr + 1) / 2 : rr * wd; };
        auto rowlen = [&](int rr) { return tri ? rr + 1 : wd; };
        if (!colw) {
            if (a < h) { r = a; c = 0; l = rowstart(r); }
        } else {
            if (a < wd) {
                r = tri ? a : 0;
                ccur = 0;                                          // 0: column a, 1: column a + 8
                c = a;
                l = rowstart(r) + c;
            }
        }
        auto advance = [&]() {
            if (!colw) {
                if (++c < rowlen(r)) { ++l; return; }
                r += 8;
                if (r >= h) { l = -1; return; }
                c = 0;
                l = rowstart(r);
            } else {
                const int c1 = a + 8;
                if (ccur == 0 && c1 < wd && (!tri || c1 <= r)) {
                    ccur = 1;
                    c = c1;
                } else {
                    ++r;
                    if (r >= h) { l = -1; return; }
                    ccur = 0;
                    c = a;
                }
                l = rowstart(r) + c;
            }
        };
        for (int l0 = 0; l0 < ntiles; l0 += RT) {
            mbar_wait(&full[slot], sph & 1);
            const double* C = ring + (size_t)slot * SLOT;
            while (l >= 0 && l < l0 + RT) {
                const double* T = C + (l - l0) * TILE_ELEMS;
                const bool diag = tri && r == c;
                if (!colw) {
                    // direct part: lane = row, s_J broadcast
                    const double2* sJ = reinterpret_cast<const double2*>(ss + (tri ? c * TILE : rows_r + c * TILE));
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
                    if (!diag) {
#pragma unroll
                        for (int j = 0; j < TILE; j += 4) {
                            const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                            d0 = fma(T[j * TILE + lane], u.x, d0);
                            d1 = fma(T[(j + 1) * TILE + lane], u.y, d1);
                            d2 = fma(T[(j + 2) * TILE + lane], v.x, d2);
                            d3 = fma(T[(j + 3) * TILE + lane], v.y, d3);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < TILE; j += 4) {
                            const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                            if (lane >= j) d0 = fma(T[diag_col_off(j) + lane - j], u.x, d0);
                            if (lane >= j + 1) d1 = fma(T[diag_col_off(j + 1) + lane - j - 1], u.y, d1);
                            if (lane >= j + 2) d2 = fma(T[diag_col_off(j + 2) + lane - j - 2], v.x, d2);
                            if (lane >= j + 3) d3 = fma(T[diag_col_off(j + 3) + lane - j - 3], v.y, d3);
                        }
                    }
                    acc += (d0 + d1) + (d2 + d3);
                    if (c == rowlen(r) - 1) {                      // row complete
                        pr[r * TILE + lane] = acc;
                        acc = 0.0;
                    }
                } else {
                    // transposed part: lane = column, rotated walk of the tile
                    const double sI = ss[r * TILE + lane];
                    double d0 = 0.0, d1 = 0.0;
                    if (!diag) {
#pragma unroll
                        for (int t = 0; t < TILE; t += 2) {
                            const int ia = (t + lane) & 31, ib = (t + 1 + lane) & 31;
                            d0 = fma(T[lane * TILE + ia], __shfl_sync(FULL, sI, ia), d0);
                            d1 = fma(T[lane * TILE + ib], __shfl_sync(FULL, sI, ib), d1);
                        }
                    } else {
                        const double* Tc = T + diag_col_off(lane) - lane;   // element (i, lane) at Tc[i], i >= lane
#pragma unroll
                        for (int t = 0; t < TILE; t += 2) {
                            const int ia = (t + lane) & 31, ib = (t + 1 + lane) & 31;
                            const double va = __shfl_sync(FULL, sI, ia), vb = __shfl_sync(FULL, sI, ib);
                            if (ia >= lane) d0 = fma(Tc[ia], va, d0);
                            if (ib >= lane) d1 = fma(Tc[ib], vb, d1);
                        }
                    }
                    if (ccur == 0) acc0 += d0 + d1;
                    else acc1 += d0 + d1;
                }
                advance();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
            if (++slot == (unsigned)nst) { slot = 0; ++sph; }
        }
        if (colw && a < wd) {
            pc[(tri ? a * TILE : rows_r + a * TILE) + lane] = acc0;
            if (a + 8 < wd) pc[(tri ? (a + 8) * TILE : rows_r + (a + 8) * TILE) + lane] = acc1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[bi]);
        mbar_arrive(&pdone[bi]);                                   // every lane (release its rows)
        if (++bi == nb) { bi = 0; ++bph; }
    }
}

// Sum the partial segments of multi-item operators for one row block, in
// fixed item order, and apply the result.
__global__ void k_symv_reduce(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items,
                              const RedDesc* __restrict__ red, int red_begin,
                              const int32_t* __restrict__ oidx, const double* __restrict__ partials,
                              double* __restrict__ z, double* __restrict__ y_out,
                              const int32_t* done) {
    if (*done) return;
    const RedDesc rd = red[red_begin + blockIdx.x];
    const OpDesc op = ops[rd.op];
    const int b = rd.b;
    const int rows_b = (min(op.nT, (b + 1) * op.BT) - b * op.BT) * TILE;
    for (int x = threadIdx.x; x < rows_b; x += blockDim.x) {
        const int g = b * op.BT * TILE + x;
        double y = 0.0;
        for (int j = 0; j <= b; ++j) {                       // items (b, j): row segments
            const ItemDesc& it = items[op.item_base + b * (b + 1) / 2 + j];
            y += partials[it.part_off + x];
        }
        for (int i = b + 1; i < op.nblk; ++i) {              // items (i, b): col segments
            const ItemDesc& it = items[op.item_base + i * (i + 1) / 2 + b];
            y += partials[it.part_off + (it.I1 - it.I0) * TILE + x];
        }
        if (g < op.m) {
            if (op.out_mode == 0) z[oidx[op.idx_off + g]] += y;
            else y_out[g] = y;
        }
    }
}

// =============================================================================
// Coarse correction
// =============================================================================

// b_c[I,:] = Q_I^T (r - A z)[Omega_I]
__global__ void k_coarse_restrict(const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                                  const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff,
                                  const double* __restrict__ Q, DevCSR A, const double* __restrict__ r,
                                  const double* __restrict__ z, double* __restrict__ bc,
                                  const int32_t* done, const int32_t* __restrict__ parts) {
    if (*done) return;
    extern __shared__ double res[];
    const int I = parts ? parts[blockIdx.x] : blockIdx.x;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    const int sw = A.sw >= 8 ? 8 : 1;                              // lanes per row
    const int gpb = blockDim.x / sw, g = threadIdx.x / sw, sl = threadIdx.x % sw;
    for (int base = 0; base < mI; base += gpb) {
        const int a = base + g;
        const bool ok = a < mI;
        const int v = ok ? bidx[b0 + a] : 0;
        const double az = sw == 8 ? row_dot<8>(A, v, ok, z, sl) : row_dot<1>(A, v, ok, z, sl);
        if (ok && sl == 0) res[a] = r[v] - az;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int ncI = cptr[I + 1] - cptr[I];
    const double* QI = Q + qoff[I];
    for (int i = w; i < ncI; i += nw) {
        double acc = 0.0;
        for (int a = lane; a < mI; a += 32) acc += QI[(int64_t)i * mI + a] * res[a];
        acc = warp_sum(acc);
        if (lane == 0) bc[cptr[I] + i] = acc;
    }
}

// Warp per part (|Omega_I| <= 32 R, short rows): the residual rows live in
// registers, each coarse column is one warp reduction.
template <int R>
__global__ void __launch_bounds__(256)
k_restrict_warp(int nparts, const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff, const double* __restrict__ Q,
                DevCSR A, const double* __restrict__ r, const double* __restrict__ z, double* __restrict__ bc,
                const int32_t* done, const int32_t* __restrict__ parts) {
    if (*done) return;
    const int wg = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (wg >= nparts) return;                                     // whole warp
    const int I = parts ? parts[wg] : wg;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    double res[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int a = lane + 32 * k;
        res[k] = 0.0;
        if (a < mI) {
            const int v = bidx[b0 + a];
            double az = 0.0;
            az = row_dot1(A, v, z);
            res[k] = r[v] - az;
        }
    }
    const int c0 = cptr[I], ncI = cptr[I + 1] - c0;
    const double* QI = Q + qoff[I];
    for (int i = 0; i < ncI; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int a = lane + 32 * k;
            if (a < mI) acc += QI[(int64_t)i * mI + a] * res[k];
        }
        acc = warp_sum(acc);
        if (lane == 0) bc[c0 + i] = acc;
    }
}

// z[Omega_I] += Q_I y_c[I,:], warp per part
template <int R>
__global__ void __launch_bounds__(256)
k_prolong_warp(int nparts, const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
               const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff, const double* __restrict__ Q,
               const double* __restrict__ yc, double* __restrict__ z, const int32_t* done,
               const int32_t* __restrict__ parts) {
    if (*done) return;
    const int wg = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (wg >= nparts) return;
    const int I = parts ? parts[wg] : wg;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    const int c0 = cptr[I], ncI = cptr[I + 1] - c0;
    const double y0 = lane < ncI ? yc[c0 + lane] : 0.0, y1 = lane + 32 < ncI ? yc[c0 + 32 + lane] : 0.0;
    const double* QI = Q + qoff[I];
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    for (int i = 0; i < ncI; ++i) {
        const double yi = __shfl_sync(FULL, i < 32 ? y0 : y1, i & 31);
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int a = lane + 32 * k;
            if (a < mI) acc[k] += QI[(int64_t)i * mI + a] * yi;
        }
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int a = lane + 32 * k;
        if (a < mI) z[bidx[b0 + a]] += acc[k];
    }
}

// z[Omega_I] += Q_I y_c[I,:]
__global__ void k_prolong(const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                          const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff,
                          const double* __restrict__ Q, const double* __restrict__ yc,
                          double* __restrict__ z, const int32_t* done, const int32_t* __restrict__ parts) {
    if (*done) return;
    __shared__ double ys[64];
    const int I = parts ? parts[blockIdx.x] : blockIdx.x;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    const int ncI = cptr[I + 1] - cptr[I];
    if (threadIdx.x < ncI) ys[threadIdx.x] = yc[cptr[I] + threadIdx.x];
    __syncthreads();
    const double* QI = Q + qoff[I];
    for (int a = threadIdx.x; a < mI; a += blockDim.x) {
        double acc = 0.0;
        for (int i = 0; i < ncI; i++) acc += QI[(int64_t)i * mI + a] * ys[i];
        z[bidx[b0 + a]] += acc;
    }
}

// =============================================================================
// Sparse coarse solve as one dataflow kernel
// =============================================================================
// The multifrontal solve of coarse_sparse.cpp without level barriers.  CTAs
// pull entries from a queue ordered leaves -> root (forward G items, after
// the leaf assemblies) then root -> leaves (backward G + H items); an entry
// only ever waits for fronts whose entries come earlier in the queue, so the
// schedule is deadlock-free without co-residency.  Per-front tickets: the
// CTA finishing a front's last item reduces its partial segments in fixed
// order, then (forward) assembles the parent once both children are done --
// children in fixed order, so the result is deterministic -- or (backward)
// writes x[S_t] and gathers x[B_c] into each child's front vector.  Flags are
// published with __threadfence + st.release and observed with ld.acquire by
// one thread followed by __syncthreads; data written by other CTAs is read
// with __ldcg.
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct DFCtx {
    const FrontDesc* fronts;
    const FrontDF* fdf;
    const FRedTask* fwd;
    const FRedTask* bwd;
    const int64_t* contrib;
    const int32_t *fS, *fB, *map;
    const double* bc;
    double *fvec, *w, *x, *partials;
    int32_t* state;
};

__device__ __forceinline__ int32_t* df_flag(const DFCtx& d, int t, int k) {
    return d.state + 1 + (int64_t)t * DF_STATE_PER_FRONT + k;
}

// front vector and w of front t from b_c and its children's w (children in order)
__device__ void df_assemble(const DFCtx& d, int t) {
    const FrontDesc f = d.fronts[t];
    double* fv = d.fvec + f.fvec_off;
    double* wt = d.w + f.w_off;
    const int ntot = f.nT * TILE;
    for (int a = threadIdx.x; a < ntot; a += blockDim.x) fv[a] = a < f.nS ? d.bc[d.fS[f.S_off + a]] : 0.0;
    for (int a = threadIdx.x; a < f.nB; a += blockDim.x) wt[a] = 0.0;
    __syncthreads();
    for (int k = 0; k < 2; ++k) {
        const int ci = k == 0 ? f.child0 : f.child1;
        if (ci < 0) continue;
        const FrontDesc c = d.fronts[ci];
        for (int j = threadIdx.x; j < c.nB; j += blockDim.x) {
            const int pos = d.map[c.map_off + j];
            const double v = __ldcg(d.w + c.w_off + j);
            if (pos < f.nSp) fv[pos] += v;
            else wt[pos - f.nSp] += v;
        }
        __syncthreads();
    }
}

// reduction tasks [t0, t1): forward w_t[B] += sum, backward x[S_t] = sum
__device__ void df_reduce(const DFCtx& d, const FRedTask* tasks, int t0, int t1) {
    for (int q = t0; q < t1; ++q) {
        const FRedTask t = tasks[q];
        const FrontDesc f = d.fronts[t.front];
        for (int r = threadIdx.x; r < t.nrows; r += blockDim.x) {
            // 8 independent loads in flight per step; fixed combine order
            double s = 0.0;
            int c = t.cbeg;
            for (; c + 8 <= t.cend; c += 8) {
                double v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = __ldcg(d.partials + d.contrib[c + k] + r);
                s += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
            }
            for (; c < t.cend; ++c) s += __ldcg(d.partials + d.contrib[c] + r);
            const int row = t.row0 + r;
            if (t.kind == 0) {
                const int b = row - f.nSp;
                if (b >= 0 && b < f.nB) d.w[f.w_off + b] += s;
            } else if (row < f.nS) {
                d.x[d.fS[f.S_off + row]] = s;
            }
        }
    }
}

// flag slots (df_flag k)
enum { DFF_READY = 0, DFF_ITEMS = 1, DFF_TASKS = 2, DFF_CHILDREN = 3, DFB_READY = 4, DFB_ITEMS = 5, DFB_TASKS = 6 };

// forward step of front t complete: count it at the parent; the last child
// assembles the parent, and fronts without G items complete on assembly
__device__ void df_forward_complete(const DFCtx& d, int t, int* sh) {
    for (;;) {
        const FrontDesc f = d.fronts[t];
        __threadfence();
        __syncthreads();
        if (f.parent < 0) {                                       // a root: backward may start
            if (threadIdx.x == 0) st_release(df_flag(d, t, DFB_READY), 1);
            return;
        }
        if (threadIdx.x == 0) {
            const FrontDesc p = d.fronts[f.parent];
            const int nch = (p.child0 >= 0) + (p.child1 >= 0);
            sh[0] = atomicAdd(df_flag(d, f.parent, DFF_CHILDREN), 1) == nch - 1;
        }
        __syncthreads();
        if (!sh[0]) return;
        __threadfence();
        t = f.parent;
        df_assemble(d, t);
        if (d.fdf[t].nG > 0) {                                    // its G items may run
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) st_release(df_flag(d, t, DFF_READY), 1);
            return;
        }
    }
}

// a leaf front was assembled
__device__ void df_leaf_ready(const DFCtx& d, int t, int* sh) {
    if (d.fdf[t].nG > 0) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) st_release(df_flag(d, t, DFF_READY), 1);
        return;
    }
    df_forward_complete(d, t, sh);
}

// tiled SYMV of one front item into its partial segment (k_symv's arithmetic)
__device__ void df_item(const OpDesc* __restrict__ ops, const ItemDesc& it, const double* __restrict__ ctiles,
                        const double* __restrict__ fvec, double* __restrict__ partials, double* sm) {
    const OpDesc op = ops[it.op];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rows_r = (it.I1 - it.I0) * TILE;
    const int rows_c = it.tri ? 0 : (it.J1 - it.J0) * TILE;
    const int rows_t = rows_r + rows_c;
    double* s_sm = sm;
    double* part = sm + rows_t;
    const double* tbase = ctiles + it.tile_off;
    const double* sop = fvec + op.s_off;
    for (int x = threadIdx.x; x < rows_t; x += blockDim.x) {
        const int g = x < rows_r ? it.I0 * TILE + x : it.J0 * TILE + (x - rows_r);
        s_sm[x] = __ldcg(sop + g);
    }
    for (int x = threadIdx.x; x < SYMV_WARPS * rows_t; x += blockDim.x) part[x] = 0.0;
    __syncthreads();
    double* pw = part + w * rows_t;
    for (int l = w; l < it.ntiles; l += SYMV_WARPS) {
        int I, J;
        item_tile(it, l, I, J);
        double a[TILE];
        load_tile_row(a, tbase + item_tile_off(it, l, I), I == J, lane);
        const int ri = (I - it.I0) * TILE;
        const int cj = it.tri ? (J - it.I0) * TILE : rows_r + (J - it.J0) * TILE;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < TILE; ++j) acc += a[j] * s_sm[cj + j];
        const double si = s_sm[ri + lane];
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] *= si;
        rs_stage<16>(a, lane);
        rs_stage<8>(a, lane);
        rs_stage<4>(a, lane);
        rs_stage<2>(a, lane);
        rs_stage<1>(a, lane);
        if (I != J) {
            pw[ri + lane] += acc;
            pw[cj + lane] += a[0];
        } else {
            pw[ri + lane] += acc + a[0];
        }
    }
    __syncthreads();
    for (int x = threadIdx.x; x < rows_t; x += blockDim.x) {
        double y = 0.0;
#pragma unroll
        for (int ww = 0; ww < SYMV_WARPS; ++ww) y += part[ww * rows_t + x];
        partials[it.part_off + x] = y;
    }
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(SYMV_WARPS * 32)
k_coarse_dataflow(int nwork, const int32_t* __restrict__ work, DFCtx d, const int32_t* __restrict__ item_front,
                  int item_base, const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items,
                  const double* __restrict__ ctiles, const int32_t* done, uint64_t* trace) {
    if (*done) return;
    extern __shared__ double sm[];
    __shared__ int sh[2];
    for (int prevq = -1;; ) {
        if (trace && prevq >= 0 && threadIdx.x == 0) trace[4 * prevq + 3] = gtimer();
        if (threadIdx.x == 0) sh[0] = atomicAdd(d.state, 1);
        __syncthreads();
        const int q = sh[0];
        __syncthreads();
        if (q >= nwork) return;
        prevq = q;
        if (trace && threadIdx.x == 0) trace[4 * q] = gtimer();
        const int32_t e = work[q];
        if (e & DF_ASSEMBLE) {
            const int t = e & DF_IDX;
            df_assemble(d, t);
            df_leaf_ready(d, t, sh);
            continue;
        }
        const bool bwd = (e & DF_BWD) != 0;
        const int idx = e & DF_IDX;
        if (e & DF_RED) {                                          // reduction task of a front
            const FRedTask tk = (bwd ? d.bwd : d.fwd)[idx];
            const int t = tk.front;
            const FrontDF fd = d.fdf[t];
            if (threadIdx.x == 0) {
                const int32_t* fl = df_flag(d, t, bwd ? DFB_ITEMS : DFF_ITEMS);
                const int need = bwd ? fd.nGH : fd.nG;
                while (ld_acquire(fl) < need) __nanosleep(100);
                if (trace) trace[4 * q + 1] = gtimer();
            }
            __syncthreads();
            df_reduce(d, bwd ? d.bwd : d.fwd, idx, idx + 1);     // w_t += -G b_S  /  x[S_t] = H b_S - G^T x_B
            if (trace && threadIdx.x == 0) trace[4 * q + 2] = gtimer();
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int ntask = bwd ? fd.bt1 - fd.bt0 : fd.ft1 - fd.ft0;
                sh[1] = atomicAdd(df_flag(d, t, bwd ? DFB_TASKS : DFF_TASKS), 1) == ntask - 1;
            }
            __syncthreads();
            if (!sh[1]) continue;
            __threadfence();
            if (!bwd) {
                df_forward_complete(d, t, sh);
            } else {
                const FrontDesc f = d.fronts[t];
                for (int k = 0; k < 2; ++k) {                      // children: gather x[B_c]
                    const int ci = k == 0 ? f.child0 : f.child1;
                    if (ci < 0) continue;
                    const FrontDesc c = d.fronts[ci];
                    double* fv = d.fvec + c.fvec_off + c.nSp;
                    const int nBp = c.nT * TILE - c.nSp;
                    for (int a = threadIdx.x; a < nBp; a += blockDim.x)
                        fv[a] = a < c.nB ? __ldcg(d.x + d.fB[c.B_off + a]) : 0.0;
                    __threadfence();
                    __syncthreads();
                    if (threadIdx.x == 0) st_release(df_flag(d, ci, DFB_READY), 1);
                }
            }
            continue;
        }
        const int t = item_front[idx - item_base];                 // a work item of front t
        if (threadIdx.x == 0) {
            const int32_t* fl = df_flag(d, t, bwd ? DFB_READY : DFF_READY);
            while (!ld_acquire(fl)) __nanosleep(100);
            if (trace) trace[4 * q + 1] = gtimer();
        }
        __syncthreads();
        const ItemDesc it = items[idx];
        df_item(ops, it, ctiles, d.fvec, d.partials, sm);
        if (trace && threadIdx.x == 0) trace[4 * q + 2] = gtimer();
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(df_flag(d, t, bwd ? DFB_ITEMS : DFF_ITEMS), 1);
    }
}

void launch_coarse_dataflow(cudaStream_t st, int nwork, const int32_t* work, const FrontDesc* fronts,
                            const FrontDF* fdf, const int32_t* item_front, int item_base, const OpDesc* ops,
                            const ItemDesc* items, const double* ctiles, const FRedTask* fwd, const FRedTask* bwd,
                            const int64_t* contrib, const int32_t* fS, const int32_t* fB, const int32_t* map,
                            const double* bc, double* fvec, double* w, double* x, double* partials,
                            int32_t* state, int max_rows_t, const int32_t* done, uint64_t* trace) {
    if (nwork <= 0) return;
    DFCtx d{fronts, fdf, fwd, bwd, contrib, fS, fB, map, bc, fvec, w, x, partials, state};
    const size_t smem = (size_t)max_rows_t * (SYMV_WARPS + 1) * sizeof(double);
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(k_coarse_dataflow, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        init = true;
    }
    const int grid = std::min(nwork, num_sms() * 2);
    k_coarse_dataflow<<<grid, SYMV_WARPS * 32, smem, st>>>(nwork, work, d, item_front, item_base, ops, items,
                                                           ctiles, done, trace);
}

// =============================================================================
// Setup: local matrices and their explicit inverses
// =============================================================================

// element (R, C) of a tiled dense mp x mp matrix (tile (I,J) at (J*nT+I)*1024)
__device__ __forceinline__ int64_t tix(int nT, int R, int C) {
    return ((int64_t)(C / TILE) * nT + R / TILE) * TILE_ELEMS + (C % TILE) * TILE + (R % TILE);
}

__global__ void k_extract_local(const int32_t* __restrict__ op_ids, const OpDesc* __restrict__ ops,
                                const int32_t* __restrict__ oidx, DevCSR A, double* scratch,
                                const int64_t* __restrict__ scratch_off) {
    const OpDesc op = ops[op_ids[blockIdx.x]];
    double* M = scratch + scratch_off[blockIdx.x];
    const int64_t tot = (int64_t)op.mp * op.mp;
    for (int64_t x = threadIdx.x; x < tot; x += blockDim.x) M[x] = 0.0;
    __syncthreads();
    const int32_t* idx = oidx + op.idx_off;
    for (int a = threadIdx.x; a < op.mp; a += blockDim.x) {
        if (a >= op.m) {
            M[tix(op.nT, a, a)] = 1.0;   // identity on the padding keeps the matrix SPD
            continue;
        }
        const int v = idx[a];
        for (int e = A.rp[v]; e < A.rp[v + 1]; e++) {
            const int c = A.col[e];
            int lo = 0, hi = op.m;       // binary search in the sorted Omega~_i
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (idx[mid] < c) lo = mid + 1; else hi = mid;
            }
            if (lo < op.m && idx[lo] == c) M[tix(op.nT, a, lo)] = A.val[e];
        }
    }
}

// ---- Gauss-Jordan exchange inversion, tile level ------------------------------
// For pivot tile k (PAPER.md's exact local solves realised as A_i^{-1}):
//   P = A_kk^{-1};  A_kj <- -P A_kj;  A_ij <- A_ij + A_ik A_kj;  A_ik <- A_ik P.
// After all k the matrix holds its inverse.  SPD input => all pivots > 0.

// invert the 32x32 tile in shared memory by scalar exchange (256 threads)
__device__ void tile_exchange_inverse(double* P, int32_t* err, int op_id, int kbase) {
    for (int p = 0; p < TILE; ++p) {
        const double d = P[p * TILE + p];
        double rowp[4], colp[4], old[4];
        const double inv = 1.0 / d;
        for (int q = 0; q < 4; ++q) {
            int e = threadIdx.x + q * 256;
            int i = e % TILE, j = e / TILE;   // element (i, j) at j*32+i
            old[q] = P[e];
            colp[q] = P[p * TILE + i];        // (i, p)
            rowp[q] = P[j * TILE + p];        // (p, j)
        }
        if (threadIdx.x == 0 && !(d > 0.0) && err) {
            if (atomicCAS(err, -1, op_id) == -1) err[1] = kbase + p;
        }
        __syncthreads();
        for (int q = 0; q < 4; ++q) {
            int e = threadIdx.x + q * 256;
            int i = e % TILE, j = e / TILE;
            double nv;
            if (i == p && j == p) nv = inv;
            else if (i == p) nv = -rowp[q] * inv;
            else if (j == p) nv = colp[q] * inv;
            else nv = old[q] - colp[q] * rowp[q] * inv;
            P[e] = nv;
        }
        __syncthreads();
    }
}

// warp: C (32x32 tile, global) = alpha * Ps(smem) * B (global tile), lane = row
__device__ __forceinline__ void warp_left_mul(const double* Ps, const double* B, double* C,
                                              double* Bs, double alpha) {
    const int lane = threadIdx.x & 31;
#pragma unroll 4
    for (int j = 0; j < TILE; ++j) Bs[j * TILE + lane] = B[j * TILE + lane];
    __syncwarp();
    double prow[TILE];
#pragma unroll
    for (int t = 0; t < TILE; ++t) prow[t] = Ps[t * TILE + lane];
    for (int j = 0; j < TILE; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < TILE; ++t) acc += prow[t] * Bs[j * TILE + t];
        C[j * TILE + lane] = alpha * acc;
    }
    __syncwarp();
}

// warp: C += Arow-tile(global) * Bs(smem), lane = row
__device__ __forceinline__ void warp_gemm_acc(const double* Ag, const double* Bs, double* C) {
    const int lane = threadIdx.x & 31;
    double arow[TILE];
#pragma unroll
    for (int t = 0; t < TILE; ++t) arow[t] = Ag[t * TILE + lane];
    for (int j = 0; j < TILE; ++j) {
        double acc = C[j * TILE + lane];
#pragma unroll
        for (int t = 0; t < TILE; ++t) acc += arow[t] * Bs[j * TILE + t];
        C[j * TILE + lane] = acc;
    }
}

// warp: C = C * Ps  (C global tile, right-multiplied in place), lane = row
__device__ __forceinline__ void warp_right_mul(double* C, const double* Ps) {
    const int lane = threadIdx.x & 31;
    double crow[TILE];
#pragma unroll
    for (int t = 0; t < TILE; ++t) crow[t] = C[t * TILE + lane];
    for (int j = 0; j < TILE; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < TILE; ++t) acc += crow[t] * Ps[j * TILE + t];
        C[j * TILE + lane] = acc;
    }
}

// one CTA (8 warps) runs the exchange over the first nK pivot tiles of one
// tiled dense matrix in place (nK = nT: full inverse)
__global__ void __launch_bounds__(256)
k_gj_batched(const int32_t* __restrict__ nTs, const int32_t* __restrict__ nKs, double* const* mats,
             const int32_t* __restrict__ ids, int32_t* err) {
    extern __shared__ double gjsm[];
    double* Ps = gjsm;
    double (*Bs)[TILE_ELEMS] = reinterpret_cast<double (*)[TILE_ELEMS]>(gjsm + TILE_ELEMS);
    const int nT = nTs[blockIdx.x], nK = nKs[blockIdx.x];
    const int opid = ids[blockIdx.x];
    double* M = mats[blockIdx.x];
    const int w = threadIdx.x >> 5;
    auto tile = [&](int I, int J) { return M + ((int64_t)J * nT + I) * TILE_ELEMS; };
    for (int k = 0; k < nK; ++k) {
        for (int e = threadIdx.x; e < TILE_ELEMS; e += 256) Ps[e] = tile(k, k)[e];
        __syncthreads();
        tile_exchange_inverse(Ps, err, opid, k * TILE);
        for (int e = threadIdx.x; e < TILE_ELEMS; e += 256) tile(k, k)[e] = Ps[e];
        // row panel: A_kj <- -P A_kj
        for (int j = w; j < nT; j += 8)
            if (j != k) warp_left_mul(Ps, tile(k, j), tile(k, j), Bs[w], -1.0);
        __syncthreads();
        // trailing update: A_ij += A_ik A_kj  (i, j != k)
        for (int j = w; j < nT; j += 8) {
            if (j == k) continue;
            const double* B = tile(k, j);
            const int lane = threadIdx.x & 31;
            for (int c = 0; c < TILE; ++c) Bs[w][c * TILE + lane] = B[c * TILE + lane];
            __syncwarp();
            for (int i = 0; i < nT; ++i)
                if (i != k) warp_gemm_acc(tile(i, k), Bs[w], tile(i, j));
            __syncwarp();
        }
        __syncthreads();
        // column panel: A_ik <- A_ik P
        for (int i = w; i < nT; i += 8)
            if (i != k) warp_right_mul(tile(i, k), Ps);
        __syncthreads();
    }
}

// ---- blocked Gauss-Jordan exchange (setup) ----------------
// The same exchange with pivot blocks of GJB_BT tiles (128 columns): per
// block, P = A_kk^{-1} (tile exchange restricted to the block, one CTA), then
// A_kj <- -P A_kj, A_ij <- A_ij + A_ik A_kj, A_ik <- A_ik P as register-blocked
// fp64 GEMMs (k_gjb_gemm): the matrix streams through HBM once per 128
// columns instead of once per 32, and each pass does 128 FMAs per element.
// A batch of matrices (tiled layout, possibly different sizes) runs together;
// matrix b has nT[b] tiles per side and eliminates its first nK[b] tiles.
constexpr int GJB_BT = 4;                  // pivot block / output block side (tiles)
constexpr int GJB_N = GJB_BT * TILE;       // 128
constexpr int GJB_BPAD = GJB_N + 2;        // padded row of the transposed B stage

struct GJBatch {
    double* const* mats;
    const int32_t* nT;
    const int32_t* nK;
    const int32_t* ids;
    int32_t* err;
};

// P = inverse of the pivot block [k0, k0 + nb) (tile exchange inside the block)
__global__ void __launch_bounds__(256) k_gjb_pivot(GJBatch bt, int k0) {
    extern __shared__ double gjsm[];
    double* Ps = gjsm;
    double (*Bs)[TILE_ELEMS] = reinterpret_cast<double (*)[TILE_ELEMS]>(gjsm + TILE_ELEMS);
    const int b = blockIdx.x;
    const int nT = bt.nT[b], nK = bt.nK[b];
    if (k0 >= nK) return;
    const int k1 = min(k0 + GJB_BT, nK);
    double* M = bt.mats[b];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto tile = [&](int I, int J) { return M + ((int64_t)J * nT + I) * TILE_ELEMS; };
    for (int k = k0; k < k1; ++k) {
        for (int e = threadIdx.x; e < TILE_ELEMS; e += 256) Ps[e] = tile(k, k)[e];
        __syncthreads();
        tile_exchange_inverse(Ps, bt.err, bt.ids[b], k * TILE);
        for (int e = threadIdx.x; e < TILE_ELEMS; e += 256) tile(k, k)[e] = Ps[e];
        for (int j = k0 + w; j < k1; j += 8)
            if (j != k) warp_left_mul(Ps, tile(k, j), tile(k, j), Bs[w], -1.0);
        __syncthreads();
        for (int j = k0 + w; j < k1; j += 8) {
            if (j == k) continue;
            const double* B = tile(k, j);
            for (int c = 0; c < TILE; ++c) Bs[w][c * TILE + lane] = B[c * TILE + lane];
            __syncwarp();
            for (int i = k0; i < k1; ++i)
                if (i != k) warp_gemm_acc(tile(i, k), Bs[w], tile(i, j));
            __syncwarp();
        }
        __syncthreads();
        for (int i = k0 + w; i < k1; i += 8)
            if (i != k) warp_right_mul(tile(i, k), Ps);
        __syncthreads();
    }
}

// mode 0 (row panel):  C(kb, J) = -P C(kb, J)          for tile columns J outside kb
// mode 1 (trailing):   C(I, J) += C(I, kb) C(kb, J)     for I, J outside kb
// mode 2 (col panel):  C(I, kb) = C(I, kb) P            for tile rows I outside kb
// CTA: a 4 x 4-tile (128 x 128) output block; thread: 8 x 8 elements.
// grid.x: output blocks of one matrix (by 4-tile rows and columns), grid.y: batch
__global__ void __launch_bounds__(256) k_gjb_gemm(GJBatch bt, int k0, int mode) {
    extern __shared__ double gsm[];
    double* As = gsm;                               // [TILE][GJB_N]   A(row, kk), kk-major
    double* Bs = gsm + TILE * GJB_N;                // [TILE][GJB_BPAD] B(kk, col), kk-major
    const int b = blockIdx.y;
    const int nT = bt.nT[b], nK = bt.nK[b];
    if (k0 >= nK) return;
    const int k1 = min(k0 + GJB_BT, nK);
    const int nb = (nT + GJB_BT - 1) / GJB_BT;      // output blocks per side
    int bi, bj;
    if (mode == 1) {
        if ((int)blockIdx.x >= nb * nb) return;
        bi = blockIdx.x % nb;
        bj = blockIdx.x / nb;
    } else {
        if ((int)blockIdx.x >= nb) return;
        bi = mode == 0 ? k0 / GJB_BT : blockIdx.x;
        bj = mode == 0 ? blockIdx.x : k0 / GJB_BT;
    }
    const int i0 = bi * GJB_BT, j0 = bj * GJB_BT;
    auto in_kb = [&](int t) { return t >= k0 && t < k1; };
    // does this block own any output tile?
    {
        bool any = false;
        for (int I = i0; I < min(i0 + GJB_BT, nT); ++I)
            for (int J = j0; J < min(j0 + GJB_BT, nT); ++J) {
                const bool ok = mode == 0 ? (in_kb(I) && !in_kb(J))
                              : mode == 1 ? (!in_kb(I) && !in_kb(J)) : (!in_kb(I) && in_kb(J));
                any |= ok;
            }
        if (!any) return;
    }
    double* M = bt.mats[b];
    auto tile = [&](int I, int J) { return M + ((int64_t)J * nT + I) * TILE_ELEMS; };
    const int tr = (threadIdx.x >> 4) * 8;          // output rows tr..tr+7 (one tile row)
    const int tc = (threadIdx.x & 15) * 2;          // output cols 32 m + tc, +1 (m = 0..3): consecutive
                                                    // lanes read consecutive 16 B of a B row
    double acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = 0.0;
    // inner dimension: the pivot block's tiles q (A's column tile, B's row tile)
    for (int q = k0; q < k1; ++q) {
        // A = (rows i0.., tile column q) [mode 0: P = (kb, q)]; B = (tile row q, cols j0..) [mode 2: P]
        for (int e = threadIdx.x; e < GJB_BT * TILE_ELEMS; e += 256) {
            const int ti = e / TILE_ELEMS, o = e % TILE_ELEMS;   // o = kk * 32 + r
            const int I = (mode == 0 ? k0 : i0) + ti;
            const int kk = o / TILE, r = o % TILE;
            As[kk * GJB_N + ti * TILE + r] = (I < nT && (mode != 0 || I < k1)) ? tile(I, q)[o] : 0.0;
        }
        for (int e = threadIdx.x; e < GJB_BT * TILE_ELEMS; e += 256) {
            const int tj = e / TILE_ELEMS, o = e % TILE_ELEMS;   // o = c * 32 + kk
            const int J = (mode == 2 ? k0 : j0) + tj;
            const int c = o / TILE, kk = o % TILE;
            Bs[kk * GJB_BPAD + tj * TILE + c] = (J < nT && (mode != 2 || J < k1)) ? tile(q, J)[o] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < TILE; ++kk) {
            double a[8], bv[8];
            const double2* ap = reinterpret_cast<const double2*>(As + kk * GJB_N + tr);
            const double* brow = Bs + kk * GJB_BPAD + tc;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double2 x = ap[u], y = *reinterpret_cast<const double2*>(brow + u * TILE);
                a[2 * u] = x.x; a[2 * u + 1] = x.y;
                bv[2 * u] = y.x; bv[2 * u + 1] = y.y;
            }
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[r][c] = fma(a[r], bv[c], acc[r][c]);
        }
        __syncthreads();
    }
    // epilogue: rows tr..tr+7 lie in tile row I; columns 2u, 2u+1 of acc are
    // columns tc, tc+1 of tile column j0 + u
    const int I = i0 + tr / TILE;
    if (I >= nT) return;
    const int rr = tr % TILE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int J = j0 + u;
        if (J >= nT) break;
        const bool ok = mode == 0 ? (in_kb(I) && !in_kb(J)) : mode == 1 ? (!in_kb(I) && !in_kb(J))
                                                                         : (!in_kb(I) && in_kb(J));
        if (!ok) continue;
        double* T = tile(I, J);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double* p = T + (tc + c) * TILE + rr + r;
                const double v = acc[r][2 * u + c];
                *p = mode == 1 ? *p + v : (mode == 0 ? -v : v);
            }
    }
}

// Dense tiled A_c from its lower-triangle entries (mirrored => exactly symmetric,
// reading R9); identity on the padding.
__global__ void k_scatter_coarse(int64_t nent, const int32_t* __restrict__ row,
                                 const int32_t* __restrict__ col, const double* __restrict__ val,
                                 int nT, int n_c, double* M) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nent;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int R = row[e], C = col[e];
        M[tix(nT, R, C)] = val[e];
        M[tix(nT, C, R)] = val[e];
    }
    for (int64_t a = n_c + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < (int64_t)nT * TILE;
         a += (int64_t)gridDim.x * blockDim.x)
        M[tix(nT, (int)a, (int)a)] = 1.0;
}

// Pack the lower-triangle tiles of the inverse into item order; diagonal
// tiles symmetrised, padding rows/cols zeroed.
__global__ void k_pack(const int32_t* __restrict__ op_ids, const OpDesc* __restrict__ ops,
                       const ItemDesc* __restrict__ items, const double* __restrict__ scratch,
                       const int64_t* __restrict__ scratch_off, double* __restrict__ tiles) {
    const int opid = op_ids[blockIdx.y];
    const OpDesc op = ops[opid];
    const double* M = scratch + scratch_off[blockIdx.y];
    for (int itx = blockIdx.x; itx < op.nitems; itx += gridDim.x) {
        const ItemDesc it = items[op.item_base + itx];
        for (int l = 0; l < it.ntiles; ++l) {
            int I, J;
            item_tile(it, l, I, J);
            const double* src = M + ((int64_t)J * op.nT + I) * TILE_ELEMS;
            double* dst = tiles + it.tile_off + item_tile_off(it, l, I);
            for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
                const int i = e % TILE, j = e / TILE;
                double v = src[e];
                if (I * TILE + i >= op.m || J * TILE + j >= op.m) v = 0.0;
                if (I != J) {
                    dst[e] = v;
                } else if (i >= j) {           // packed lower, diagonal halved, symmetrised
                    double vt = (I * TILE + i >= op.m || J * TILE + j >= op.m) ? 0.0 : src[i * TILE + j];
                    dst[diag_col_off(j) + i - j] = i == j ? 0.5 * v : 0.5 * (v + vt);
                }
            }
        }
    }
}

// =============================================================================
// Sparse coarse factorisation and solve (coarse_sparse.cpp)
// =============================================================================

__global__ void k_front_scatter(int64_t ntrip, const int32_t* __restrict__ frow,
                                const int32_t* __restrict__ fcol, const double* __restrict__ fval,
                                const int32_t* __restrict__ ffront, const FrontDesc* __restrict__ fronts,
                                double* const* fptr) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ntrip;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int f = ffront[e];
        double* M = fptr[f];
        const int nT = fronts[f].nT;
        M[tix(nT, frow[e], fcol[e])] = fval[e];
        M[tix(nT, fcol[e], frow[e])] = fval[e];
    }
}

// parent front += child's Schur complement (its B x B block), through the map
__global__ void k_front_extend_add(const int32_t* __restrict__ child, const FrontDesc* __restrict__ fronts,
                                   double* const* fptr, const int32_t* __restrict__ map) {
    const FrontDesc c = fronts[child[blockIdx.y]];
    const FrontDesc p = fronts[c.parent];
    const double* Fc = fptr[child[blockIdx.y]];
    double* Fp = fptr[c.parent];
    const int32_t* mp = map + c.map_off;
    const int64_t tot = (int64_t)c.nB * c.nB;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e % c.nB), b = (int)(e / c.nB);
        Fp[tix(p.nT, mp[a], mp[b])] += Fc[tix(c.nT, c.nSp + a, c.nSp + b)];
    }
}

// tiles of the front's solve operator K_t = [[A_SS^-1, .], [-A_BS A_SS^-1, 0]]
__global__ void k_front_pack(int i0, int i1, int item_base, const int32_t* __restrict__ item_front,
                             const FrontDesc* __restrict__ fronts, double* const* fptr,
                             const ItemDesc* __restrict__ items, double* __restrict__ ctiles) {
    for (int itx = i0 + blockIdx.x; itx < i1; itx += gridDim.x) {
        const ItemDesc it = items[itx];
        const int fi = item_front[itx - item_base];
        const FrontDesc fr = fronts[fi];
        const double* M = fptr[fi];
        for (int l = 0; l < it.ntiles; ++l) {
            int I, J;
            item_tile(it, l, I, J);
            const double* src = M + ((int64_t)J * fr.nT + I) * TILE_ELEMS;
            double* dst = ctiles + it.tile_off + item_tile_off(it, l, I);
            for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
                const int i = e % TILE, j = e / TILE;
                const int R = I * TILE + i, C = J * TILE + j;
                double v = src[e];
                if (I < fr.nK) {                    // H = A_SS^{-1}
                    if (R >= fr.nS || C >= fr.nS) v = 0.0;
                    if (I != J) {
                        dst[e] = v;
                    } else if (i >= j) {            // packed lower, diagonal halved, symmetrised
                        const double vt = (R >= fr.nS || C >= fr.nS) ? 0.0 : src[i * TILE + j];
                        dst[diag_col_off(j) + i - j] = i == j ? 0.5 * v : 0.5 * (v + vt);
                    }
                } else {                             // -G = -A_BS A_SS^{-1}
                    v = -v;
                    if (R - fr.nSp >= fr.nB || C >= fr.nS) v = 0.0;
                    dst[e] = v;
                }
            }
        }
    }
}

// forward: front vector [b_S ; 0] and w_t = incoming contributions to B
__global__ void k_front_fwd_assemble(int f0, const FrontDesc* __restrict__ fronts,
                                     const int32_t* __restrict__ fS, const int32_t* __restrict__ map,
                                     const double* __restrict__ bc, double* __restrict__ fvec,
                                     double* __restrict__ w, const int32_t* done) {
    if (*done) return;
    const FrontDesc f = fronts[f0 + blockIdx.x];
    double* fv = fvec + f.fvec_off;
    double* wt = w + f.w_off;
    const int ntot = f.nT * TILE;
    for (int a = threadIdx.x; a < ntot; a += blockDim.x) fv[a] = a < f.nS ? bc[fS[f.S_off + a]] : 0.0;
    for (int a = threadIdx.x; a < f.nB; a += blockDim.x) wt[a] = 0.0;
    __syncthreads();
    for (int s = 0; s < 2; ++s) {
        const int ci = s == 0 ? f.child0 : f.child1;
        if (ci < 0) continue;
        const FrontDesc c = fronts[ci];
        for (int j = threadIdx.x; j < c.nB; j += blockDim.x) {
            const int pos = map[c.map_off + j];
            const double v = w[c.w_off + j];
            if (pos < f.nSp) fv[pos] += v;
            else wt[pos - f.nSp] += v;
        }
        __syncthreads();
    }
}

// backward: B part of the front vector = x[B_t] (solved by ancestors)
__global__ void k_front_bwd_gather(int f0, const FrontDesc* __restrict__ fronts,
                                   const int32_t* __restrict__ fB, const double* __restrict__ x,
                                   double* __restrict__ fvec, const int32_t* done) {
    if (*done) return;
    const FrontDesc f = fronts[f0 + blockIdx.x];
    double* fv = fvec + f.fvec_off + f.nSp;
    const int nBp = f.nT * TILE - f.nSp;
    for (int a = threadIdx.x; a < nBp; a += blockDim.x) fv[a] = a < f.nB ? x[fB[f.B_off + a]] : 0.0;
}

__global__ void k_front_reduce(const FRedTask* __restrict__ tasks, int t0,
                               const int64_t* __restrict__ contrib, const FrontDesc* __restrict__ fronts,
                               const int32_t* __restrict__ fS, const double* __restrict__ partials,
                               double* __restrict__ w, double* __restrict__ x, const int32_t* done) {
    if (*done) return;
    const FRedTask t = tasks[t0 + blockIdx.x];
    const FrontDesc f = fronts[t.front];
    for (int r = threadIdx.x; r < t.nrows; r += blockDim.x) {
        double s = 0.0;
        for (int c = t.cbeg; c < t.cend; ++c) s += partials[contrib[c] + r];
        const int row = t.row0 + r;
        if (t.kind == 0) {
            const int b = row - f.nSp;
            if (b >= 0 && b < f.nB) w[f.w_off + b] += s;
        } else if (row < f.nS) {
            x[fS[f.S_off + row]] = s;
        }
    }
}

// =============================================================================
// launchers
// =============================================================================

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static inline int vec_grid(int64_t n) {
    int64_t g = (n + VEC_THREADS - 1) / VEC_THREADS;
    return (int)(g < RED_BLOCKS ? (g > 0 ? g : 1) : RED_BLOCKS);
}

void launch_gather_flat(cudaStream_t st, int64_t x0, int64_t x1, const int32_t* gidx, DevCSR A, const double* r,
                        const double* z, double* s, bool z_is_zero, const int32_t* done) {
    if (x1 <= x0) return;
    const int sw = z_is_zero ? 1 : std::max(1, A.sw);
    const int64_t want = ((x1 - x0) * sw + 255) / 256;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * 8));
    const int zz = z_is_zero ? 1 : 0;
    switch (sw) {
        case 4: k_gather_flat<4><<<g, 256, 0, st>>>(x0, x1, gidx, A, r, z, s, zz, done); break;
        case 8: k_gather_flat<8><<<g, 256, 0, st>>>(x0, x1, gidx, A, r, z, s, zz, done); break;
        case 32: k_gather_flat<32><<<g, 256, 0, st>>>(x0, x1, gidx, A, r, z, s, zz, done); break;
        default: k_gather_flat<1><<<g, 256, 0, st>>>(x0, x1, gidx, A, r, z, s, zz, done);
    }
}

static size_t symv_smem(int max_rows_t) {
    return (size_t)max_rows_t * (SYMV_WARPS + 1) * sizeof(double);
}

void launch_symv(cudaStream_t st, const OpDesc* ops, const ItemDesc* items, int item_begin,
                 int nitems, const double* tiles, const double* s, const int32_t* oidx, double* z,
                 double* y_out, double* partials, const int32_t* done, int max_rows_t, unsigned* tickets,
                 int gather_mode, DevCSR A, const double* r, bool small_ok) {
    if (nitems <= 0) return;
    if (max_rows_t <= 0) max_rows_t = 2 * MAX_BT * TILE;
    if (small_ok && max_rows_t <= SMALL_MAXROWS) {
        k_symv_small<<<(nitems + 7) / 8, 256, 0, st>>>(ops, items, item_begin, nitems, tiles, s, oidx, z, y_out,
                                                      done, gather_mode, A, r);
        return;
    }
    const size_t smem = symv_smem(max_rows_t);
    cudaFuncSetAttribute(k_symv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_symv<<<nitems, SYMV_WARPS * 32, smem, st>>>(ops, items, item_begin, tiles, s, oidx, z, y_out,
                                                  partials, done, tickets, gather_mode, A, r);
}

static bool g_ring_init[64] = {};
static int g_ring_rt = 4, g_ring_nb = 0, g_ring_nst = 0, g_ring_v2 = 0;
static unsigned long long* g_ring_trace = nullptr;   // DDG_RING_TRACE (debug)
// per device, once, outside any stream capture (called from ddg_setup)
void symv_ring_init() {
    g_ring_rt = 4;
    if (const char* e = getenv("DDG_RING_TILES")) g_ring_rt = atoi(e);
    if (g_ring_rt != 1 && g_ring_rt != 2 && g_ring_rt != 8) g_ring_rt = 4;
    g_ring_nb = 0;
    if (const char* e = getenv("DDG_RING_NB")) g_ring_nb = std::max(2, std::min(RING_MAX_NB, atoi(e)));
    g_ring_nst = 0;
    if (const char* e = getenv("DDG_RING_NST")) g_ring_nst = std::max(2, std::min(RING_MAX_NST, atoi(e)));
    g_ring_v2 = getenv("DDG_RING_V2") ? atoi(getenv("DDG_RING_V2")) : -1;   // -1: auto

    if (getenv("DDG_RING_TRACE") && !g_ring_trace) {
        if (cudaMalloc(&g_ring_trace, 32 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(g_ring_trace, 0, 32 * sizeof(unsigned long long));
        else
            g_ring_trace = nullptr;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_ring_init[dev & 63]) return;
    const size_t mx = 227 * 1024;
    cudaFuncSetAttribute(k_symv_ring<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaFuncSetAttribute(k_symv_ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaFuncSetAttribute(k_symv_ring<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaFuncSetAttribute(k_symv_ring2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaFuncSetAttribute(k_symv_ring2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    cudaFuncSetAttribute(k_symv_ring2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    g_ring_init[dev & 63] = true;
}

// debug: read and zero the DDG_RING_TRACE counters (24 values; see k_symv_ring)
int symv_ring_trace(unsigned long long* out) {
    if (!g_ring_trace) return -1;
    cudaDeviceSynchronize();
    cudaMemcpy(out, g_ring_trace, 24 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemset(g_ring_trace, 0, 32 * sizeof(unsigned long long));
    return 0;
}

void launch_symv_ring(cudaStream_t st, const OpDesc* ops, const ItemDesc* items, int item_begin,
                      const int32_t* cta_part, int ncta, int max_rows_r, int max_rows_c, const double* tiles,
                      const double* s, const int32_t* oidx, double* z, double* y_out, double* partials,
                      const int32_t* done, bool triangles) {
    const int RT = g_ring_rt;
    const int R = std::max(TILE, max_rows_r), Cr = std::max(0, max_rows_c);
    const int maxr = std::min(RING_MAX_ROWS, R + Cr);
    const size_t budget = 227 * 1024;
    // row/column-warp consumers for launches of whole-subdomain triangles
    // (measured: C3 +4%, C5 +1%; the 8-warp column consumers win on the
    // 8-wide rectangles of split operators); DDG_RING_V2=0/1 forces either
    if (g_ring_v2 == 1 || (g_ring_v2 < 0 && triangles) || RT == 8) {
        int nb2 = g_ring_nb > 0 ? g_ring_nb : (maxr <= 256 ? 4 : 2);
        int nst2 = 2;
        const int cap = g_ring_nst > 0 ? g_ring_nst : RING_MAX_NST;
        while (nst2 < cap && ring2_smem(RT, nst2 + 1, nb2, maxr) <= budget) ++nst2;
        const size_t smem2 = ring2_smem(RT, nst2, nb2, maxr);
        if (RT == 2)
            k_symv_ring2<2><<<ncta, RING2_THREADS, smem2, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z,
                                                                 y_out, partials, done, nst2, nb2, maxr);
        else if (RT == 8)
            k_symv_ring2<8><<<ncta, RING2_THREADS, smem2, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z,
                                                                 y_out, partials, done, nst2, nb2, maxr);
        else
            k_symv_ring2<4><<<ncta, RING2_THREADS, smem2, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z,
                                                                 y_out, partials, done, nst2, nb2, maxr);
        return;
    }
    // item buffers: deep for small items (s copies and epilogues overlap
    // several items), two for large ones; the rest of shared memory is ring
    int nb = g_ring_nb > 0 ? g_ring_nb : (maxr <= 256 ? 3 : 2);
    while (nb > 2 && ring_smem(RT, 4, nb, R, Cr) > budget) --nb;
    int nst = 2;
    const int nst_cap = g_ring_nst > 0 ? g_ring_nst : RING_MAX_NST;
    while (nst < nst_cap && ring_smem(RT, nst + 1, nb, R, Cr) <= budget) ++nst;
    const size_t smem = ring_smem(RT, nst, nb, R, Cr);
    if (RT == 1)
        k_symv_ring<1><<<ncta, RING_THREADS, smem, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z, y_out,
                                                         partials, done, nst, nb, R, Cr, g_ring_trace);
    else if (RT == 2)
        k_symv_ring<2><<<ncta, RING_THREADS, smem, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z, y_out,
                                                         partials, done, nst, nb, R, Cr, g_ring_trace);
    else
        k_symv_ring<4><<<ncta, RING_THREADS, smem, st>>>(ops, items, item_begin, cta_part, tiles, s, oidx, z, y_out,
                                                         partials, done, nst, nb, R, Cr, g_ring_trace);
}

void launch_symv_reduce(cudaStream_t st, const OpDesc* ops, const ItemDesc* items,
                        const RedDesc* red, int red_begin, int nred, const int32_t* oidx,
                        const double* partials, double* z, double* y_out, const int32_t* done) {
    if (nred <= 0) return;
    k_symv_reduce<<<nred, 256, 0, st>>>(ops, items, red, red_begin, oidx, partials, z, y_out, done);
}

void launch_coarse_restrict(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* bidx,
                            const int32_t* cptr, const int64_t* qoff, const double* Q, DevCSR A,
                            const double* r, const double* z, double* bc, int maxmI,
                            const int32_t* done, const int32_t* parts) {
    if (nparts <= 0) return;
    if (A.sw <= 1 && maxmI <= 512) {
        const int g = (nparts + 7) / 8;
        if (maxmI <= 64)
            k_restrict_warp<2><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
        else if (maxmI <= 128)
            k_restrict_warp<4><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
        else if (maxmI <= 256)
            k_restrict_warp<8><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
        else
            k_restrict_warp<16><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
        return;
    }
    const size_t smem = (size_t)maxmI * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_coarse_restrict, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_coarse_restrict<<<nparts, 256, smem, st>>>(bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
}

void launch_prolong(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* bidx,
                    const int32_t* cptr, const int64_t* qoff, const double* Q, const double* yc,
                    double* z, int maxmI, const int32_t* done, const int32_t* parts) {
    if (nparts <= 0) return;
    if (maxmI <= 512) {
        const int g = (nparts + 7) / 8;
        if (maxmI <= 64)
            k_prolong_warp<2><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, yc, z, done, parts);
        else if (maxmI <= 128)
            k_prolong_warp<4><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, yc, z, done, parts);
        else if (maxmI <= 256)
            k_prolong_warp<8><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, yc, z, done, parts);
        else
            k_prolong_warp<16><<<g, 256, 0, st>>>(nparts, bptr, bidx, cptr, qoff, Q, yc, z, done, parts);
        return;
    }
    k_prolong<<<nparts, 256, 0, st>>>(bptr, bidx, cptr, qoff, Q, yc, z, done, parts);
}

void launch_fill(cudaStream_t st, double* x, int64_t n, double v, const int32_t* done) {
    k_fill<<<vec_grid(n), VEC_THREADS, 0, st>>>(x, n, v, done);
}

void launch_spmv(cudaStream_t st, DevCSR A, const double* x, double* y) {
    k_spmv<<<vec_grid(A.n), VEC_THREADS, 0, st>>>(A, x, y);
}

void launch_pcg_init(cudaStream_t st, int64_t n, const double* f, double* r, double* u, const int32_t* rows,
                     int64_t nrows, Scalars* sc, double* hist, double* red, unsigned* ticket, int dist) {
    k_pcg_init<<<vec_grid(n), VEC_THREADS, 0, st>>>(n, f, r, u, rows, nrows, sc, hist, red, ticket, dist);
}
void launch_pcg_rz_first(cudaStream_t st, const double* r, const double* z, double* p, const int32_t* rows,
                         int64_t nrows, Scalars* sc, double* red, unsigned* ticket, int dist) {
    k_pcg_rz_first<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(r, z, p, rows, nrows, sc, red, ticket, dist);
}
void launch_pcg_spmv_dot(cudaStream_t st, DevCSR A, const double* p, double* q, const int32_t* rows,
                         int64_t nrows, Scalars* sc, double* red, unsigned* ticket, int dist) {
    const int g = vec_grid(nrows * std::max(1, A.sw));
    switch (A.sw) {
        case 4: k_pcg_spmv_dot<4><<<g, VEC_THREADS, 0, st>>>(A, p, q, rows, nrows, sc, red, ticket, dist); break;
        case 8: k_pcg_spmv_dot<8><<<g, VEC_THREADS, 0, st>>>(A, p, q, rows, nrows, sc, red, ticket, dist); break;
        case 32: k_pcg_spmv_dot<32><<<g, VEC_THREADS, 0, st>>>(A, p, q, rows, nrows, sc, red, ticket, dist); break;
        default: k_pcg_spmv_dot<1><<<g, VEC_THREADS, 0, st>>>(A, p, q, rows, nrows, sc, red, ticket, dist);
    }
}
void launch_pcg_update(cudaStream_t st, const double* p, const double* q, double* u, double* r,
                       const int32_t* rows, int64_t nrows, Scalars* sc, double* hist, double* red,
                       unsigned* ticket, int dist) {
    k_pcg_update<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(p, q, u, r, rows, nrows, sc, hist, red, ticket, dist);
}
void launch_pcg_rz(cudaStream_t st, const double* r, const double* z, const int32_t* rows, int64_t nrows,
                   Scalars* sc, double* red, unsigned* ticket, int dist) {
    k_pcg_rz<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(r, z, rows, nrows, sc, red, ticket, dist);
}
void launch_pcg_direction(cudaStream_t st, const double* z, double* p, const int32_t* rows, int64_t nrows,
                          Scalars* sc) {
    k_pcg_direction<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(z, p, rows, nrows, sc);
}
void launch_pcg_finalize(cudaStream_t st, int slot, Scalars* sc, double* hist) {
    k_pcg_finalize<<<1, 1, 0, st>>>(slot, sc, hist);
}
void launch_halo_pack(cudaStream_t st, const double* v, const int32_t* idx, double* buf, int64_t n) {
    if (n > 0) k_halo_pack<<<vec_grid(n), VEC_THREADS, 0, st>>>(v, idx, buf, n);
}
void launch_halo_unpack(cudaStream_t st, const double* buf, const int32_t* idx, double* v, int64_t n) {
    if (n > 0) k_halo_unpack<<<vec_grid(n), VEC_THREADS, 0, st>>>(buf, idx, v, n);
}
void launch_copy_rows(cudaStream_t st, const double* in, double* out, const int32_t* rows, int64_t nrows) {
    if (nrows > 0) k_copy_rows<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(in, out, rows, nrows);
}

void launch_extract_local(cudaStream_t st, int nops, const int32_t* op_ids, const OpDesc* ops,
                          const int32_t* oidx, DevCSR A, double* scratch,
                          const int64_t* scratch_off) {
    if (nops <= 0) return;
    k_extract_local<<<nops, 256, 0, st>>>(op_ids, ops, oidx, A, scratch, scratch_off);
}

void launch_gj_batched(cudaStream_t st, int nmat, const int32_t* nT, const int32_t* nK,
                       double* const* mats, const int32_t* ids, int32_t* err) {
    if (nmat <= 0) return;
    const int smem = 9 * TILE_ELEMS * sizeof(double);
    cudaFuncSetAttribute(k_gj_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_gj_batched<<<nmat, 256, smem, st>>>(nT, nK, mats, ids, err);
}

void launch_gj_blocked(cudaStream_t st, int nmat, int maxT, int maxK, double* const* mats, const int32_t* nT,
                       const int32_t* nK, const int32_t* ids, int32_t* err) {
    if (nmat <= 0) return;
    static bool init = false;
    const int smem_p = 9 * TILE_ELEMS * sizeof(double);
    const int smem_g = (TILE * GJB_N + TILE * GJB_BPAD) * sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_gjb_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p);
        cudaFuncSetAttribute(k_gjb_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_g);
        init = true;
    }
    GJBatch bt{mats, nT, nK, ids, err};
    const int nb = (maxT + GJB_BT - 1) / GJB_BT;
    for (int k0 = 0; k0 < maxK; k0 += GJB_BT) {
        k_gjb_pivot<<<nmat, 256, smem_p, st>>>(bt, k0);
        k_gjb_gemm<<<dim3(nb, nmat), 256, smem_g, st>>>(bt, k0, 0);
        k_gjb_gemm<<<dim3(nb * nb, nmat), 256, smem_g, st>>>(bt, k0, 1);
        k_gjb_gemm<<<dim3(nb, nmat), 256, smem_g, st>>>(bt, k0, 2);
    }
}

void launch_scatter_coarse(cudaStream_t st, int64_t nent, const int32_t* row, const int32_t* col,
                           const double* val, int nT, int n_c, double* M) {
    k_scatter_coarse<<<RED_BLOCKS, 256, 0, st>>>(nent, row, col, val, nT, n_c, M);
}

void launch_pack(cudaStream_t st, int nops, const int32_t* op_ids, const OpDesc* ops,
                 const ItemDesc* items, const double* scratch, const int64_t* scratch_off,
                 double* tiles) {
    if (nops <= 0) return;
    k_pack<<<dim3(8, nops), 256, 0, st>>>(op_ids, ops, items, scratch, scratch_off, tiles);
}

}  // namespace ddg

namespace ddg {
void launch_front_scatter(cudaStream_t st, int64_t ntrip, const int32_t* frow, const int32_t* fcol,
                          const double* fval, const int32_t* ffront, const FrontDesc* fronts,
                          double* const* fptr) {
    if (ntrip <= 0) return;
    k_front_scatter<<<RED_BLOCKS, 256, 0, st>>>(ntrip, frow, fcol, fval, ffront, fronts, fptr);
}
void launch_front_extend_add(cudaStream_t st, int ntask, const int32_t* child, const FrontDesc* fronts,
                             double* const* fptr, const int32_t* map, int64_t max_elems) {
    if (ntask <= 0) return;
    int gx = (int)std::min<int64_t>(std::max<int64_t>(1, (max_elems + 255) / 256), 4096);
    k_front_extend_add<<<dim3(gx, ntask), 256, 0, st>>>(child, fronts, fptr, map);
}
void launch_front_pack(cudaStream_t st, int i0, int i1, int item_base, const int32_t* item_front,
                       const FrontDesc* fronts, double* const* fptr, const ItemDesc* items, double* ctiles) {
    if (i1 <= i0) return;
    k_front_pack<<<std::min(i1 - i0, 4096), 256, 0, st>>>(i0, i1, item_base, item_front, fronts, fptr, items,
                                                          ctiles);
}
void launch_front_fwd_assemble(cudaStream_t st, int f0, int nf, const FrontDesc* fronts,
                               const int32_t* fS, const int32_t* map, const double* bc, double* fvec,
                               double* w, const int32_t* done) {
    if (nf <= 0) return;
    k_front_fwd_assemble<<<nf, 256, 0, st>>>(f0, fronts, fS, map, bc, fvec, w, done);
}
void launch_front_bwd_gather(cudaStream_t st, int f0, int nf, const FrontDesc* fronts,
                             const int32_t* fB, const double* x, double* fvec, const int32_t* done) {
    if (nf <= 0) return;
    k_front_bwd_gather<<<nf, 256, 0, st>>>(f0, fronts, fB, x, fvec, done);
}
void launch_front_reduce(cudaStream_t st, const FRedTask* tasks, int t0, int nt, const int64_t* contrib,
                         const FrontDesc* fronts, const int32_t* fS, const double* partials, double* w,
                         double* x, const int32_t* done) {
    if (nt <= 0) return;
    k_front_reduce<<<nt, 256, 0, st>>>(tasks, t0, contrib, fronts, fS, partials, w, x, done);
}
}  // namespace ddg
