// pcg.cu — PCG vector kernels, halo pack/unpack
// (part of libddg's sm_100a kernels; shared device helpers in kernel_common.cuh)
#include "kernel_common.cuh"

namespace ddg {
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
    pdl_wait();
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

// ||f - A u||_2 once after the solve (SURVEY.md §8(c) PCG step 3: the true
// residual, reported beside the recurrence residual the stopping rule uses)
template <int SW>
__global__ void k_true_res(DevCSR A, const double* __restrict__ f, const double* __restrict__ u, int64_t n,
                           Scalars* sc, double* red, unsigned* ticket) {
    double acc = 0.0;
    const int64_t ng = (int64_t)gridDim.x * blockDim.x / SW;
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / SW;
    const int sl = threadIdx.x % SW;
    for (int64_t base = 0; base < n; base += ng) {
        const int64_t v = base + g;
        const bool ok = v < n;
        const double s = row_dot<SW>(A, ok ? v : 0, ok, u, sl);
        if (ok && sl == 0) {
            const double d = f[v] - s;
            acc += d * d;
        }
    }
    grid_reduce(acc, red, ticket, [&](double t) { sc->tres = sqrt(t); });
}

// u += alpha p ; r -= alpha q ; ||r|| ; history ; stopping rule (reading R1)
__global__ void k_pcg_update(const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ u,
                             double* __restrict__ r, const int32_t* __restrict__ rows, int64_t nrows, Scalars* sc,
                             double* hist, double* red, unsigned* ticket, int dist) {
    pdl_wait();
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
    pdl_wait();
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
    pdl_wait();
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
    {
        const int64_t v = rows ? (int64_t)rows[i] : i;   // rows == nullptr: every row (one rank)
        out[v] = in[v];
    }
}

__global__ void k_fill(double* x, int64_t n, double v, const int32_t* done) {
    pdl_wait();
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


// ---- launchers ----

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

void launch_fill(cudaStream_t st, double* x, int64_t n, double v, const int32_t* done) {
    launch_pdl(k_fill, vec_grid(n), VEC_THREADS, 0, st, x, n, v, done);
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
        case 4: launch_pdl(k_pcg_spmv_dot<4>, g, VEC_THREADS, 0, st, A, p, q, rows, nrows, sc, red, ticket, dist); break;
        case 8: launch_pdl(k_pcg_spmv_dot<8>, g, VEC_THREADS, 0, st, A, p, q, rows, nrows, sc, red, ticket, dist); break;
        case 32: launch_pdl(k_pcg_spmv_dot<32>, g, VEC_THREADS, 0, st, A, p, q, rows, nrows, sc, red, ticket, dist); break;
        default: launch_pdl(k_pcg_spmv_dot<1>, g, VEC_THREADS, 0, st, A, p, q, rows, nrows, sc, red, ticket, dist);
    }
}

void launch_true_res(cudaStream_t st, DevCSR A, const double* f, const double* u, int64_t n, Scalars* sc,
                     double* red, unsigned* ticket) {
    const int g = vec_grid(n * std::max(1, A.sw));
    switch (A.sw) {
        case 4: k_true_res<4><<<g, VEC_THREADS, 0, st>>>(A, f, u, n, sc, red, ticket); break;
        case 8: k_true_res<8><<<g, VEC_THREADS, 0, st>>>(A, f, u, n, sc, red, ticket); break;
        case 32: k_true_res<32><<<g, VEC_THREADS, 0, st>>>(A, f, u, n, sc, red, ticket); break;
        default: k_true_res<1><<<g, VEC_THREADS, 0, st>>>(A, f, u, n, sc, red, ticket);
    }
}

void launch_pcg_update(cudaStream_t st, const double* p, const double* q, double* u, double* r,
                       const int32_t* rows, int64_t nrows, Scalars* sc, double* hist, double* red,
                       unsigned* ticket, int dist) {
    launch_pdl(k_pcg_update, vec_grid(nrows), VEC_THREADS, 0, st, p, q, u, r, rows, nrows, sc, hist, red, ticket, dist);
}

void launch_pcg_rz(cudaStream_t st, const double* r, const double* z, const int32_t* rows, int64_t nrows,
                   Scalars* sc, double* red, unsigned* ticket, int dist) {
    launch_pdl(k_pcg_rz, vec_grid(nrows), VEC_THREADS, 0, st, r, z, rows, nrows, sc, red, ticket, dist);
}

void launch_pcg_direction(cudaStream_t st, const double* z, double* p, const int32_t* rows, int64_t nrows,
                          Scalars* sc) {
    launch_pdl(k_pcg_direction, vec_grid(nrows), VEC_THREADS, 0, st, z, p, rows, nrows, sc);
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

// device-side iteration control: the condition of a graph IF / WHILE node
// becomes "not done" (setup.cpp build_solve_graph)
__global__ void k_pcg_cond(const Scalars* sc, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, sc->done ? 0u : 1u);
}
void launch_pcg_cond(cudaStream_t st, const Scalars* sc, unsigned long long h) {
    k_pcg_cond<<<1, 1, 0, st>>>(sc, (cudaGraphConditionalHandle)h);
}

// loopback allreduce (comm.cpp): fixed rank order
struct LoopPtrs {
    const double* p[16];
};
__global__ void k_loop_sum(LoopPtrs P, int n, double* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += P.p[r][i];
        out[i] = s;
    }
}
void launch_loop_sum(cudaStream_t st, const double* const* ptrs, int n, double* out, int64_t count) {
    LoopPtrs P{};
    for (int r = 0; r < n && r < 16; ++r) P.p[r] = ptrs[r];
    const int grid = (int)std::min<int64_t>((count + 255) / 256, 4096);
    if (count > 0) k_loop_sum<<<grid, 256, 0, st>>>(P, n, out, count);
}

void launch_copy_rows(cudaStream_t st, const double* in, double* out, const int32_t* rows, int64_t nrows) {
    if (nrows > 0) k_copy_rows<<<vec_grid(nrows), VEC_THREADS, 0, st>>>(in, out, rows, nrows);
}

}  // namespace ddg
