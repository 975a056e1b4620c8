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
    if (hist) hist[0] = r0;
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
    if (hist) hist[it] = res;
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



// =============================================================================
// The whole PCG solve in one kernel for small problems (C1-sized; VERDICT r1
// item 9): one thread-block cluster of G CTAs runs every phase of
// PAPER.md:605-608 with the two-level preconditioner PAPER.md:552-564 between
// cluster barriers (barrier.cluster, release / acquire at cluster scope):
// 2C + 7 barriers per iteration instead of ~4C + 8 kernel launches.
//  * CTA g owns the operators t = g, g + G, ... of every colour and keeps
//    their tiles (compact last rows) and index lists in shared memory for the
//    whole solve; a colour step is a gather from L2, a SYMV by its 8 warps from
//    shared memory, and the z update (z at the subdomain rows is captured by
//    the gather: same-colour subdomains are disjoint);
//  * warp w of CTA g owns the parts I = g + G w (+ 8 G ...) of the
//    restriction and prolongation, with their Q_I and row lists resident;
//  * CTA G - 1 - s (s < nT_c) keeps tile row s and tile column s of the dense
//    coarse inverse and computes y_c's segment s; the restriction broadcasts b_c and
//    the coarse step broadcasts y_c through distributed shared memory;
//  * sums: per-CTA block sums to a two-slot scratch, one barrier, then every
//    CTA adds the G partials in CTA order, so every CTA takes the same
//    (deterministic) step and runs the stopping rule itself; CTA 0 writes the
//    history, the CG coefficients and the final scalars.
// Vectors other CTAs write are read through L2 (ld.global.cg): L1 is not
// coherent.  Eligibility and the shared-memory plan: small_plan (setup.cpp).
// =============================================================================
constexpr int SMALL_MAX_G = 16;
constexpr int SMALL_MAX_OWN = 32;
constexpr int SMALL_MAX_COL = 64;

__device__ unsigned long long* g_small_trace = nullptr;   // DDG_SMALL_TRACE: %globaltimer per barrier (CTA 0)
__device__ int g_small_ntrace = 0;
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (g_small_trace && threadIdx.x == 0 && blockIdx.x == 0 && g_small_ntrace < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_small_trace[g_small_ntrace++] = t;
    }
}
__device__ __forceinline__ void small_stamp() {   // DDG_SMALL_TRACE: globaltimer and clock64 (CTA 0, thread 0)
    if (g_small_trace && threadIdx.x == 0 && blockIdx.x == 0 && g_small_ntrace < 4094) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_small_trace[g_small_ntrace++] = t;
        g_small_trace[g_small_ntrace++] = clock64() | (1ull << 63);
    }
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// store v at the same shared-memory location of CTA `rank` of the cluster
__device__ __forceinline__ void st_cluster(double* local, unsigned rank, double v) {
    unsigned la = smem_u32(local), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
// lane i: row i of a tile in shared memory (packed diagonal, compact tail rows th)
__device__ __forceinline__ void smem_tile_row(double* a, const double* T, bool diag, int lane, int th) {
    if (th == TILE) {
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] = diag ? (lane >= j ? T[diag_col_off(j) + lane - j] : 0.0) : T[j * TILE + lane];
        return;
    }
#pragma unroll
    for (int j = 0; j < TILE; ++j)
        a[j] = lane < th ? (diag ? (lane >= j ? T[tail_col_off(th, j) + lane - j] : 0.0) : T[j * th + lane]) : 0.0;
}
// one tile: direct part (lane = row) and transposed part (butterfly: lane = column)
__device__ __forceinline__ void small_tile(double* a, const double* sJ, double si, double& dir, double& tr, int lane) {
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
    for (int j = 0; j < TILE; j += 4) {
        d0 = fma(a[j], sJ[j], d0);
        d1 = fma(a[j + 1], sJ[j + 1], d1);
        d2 = fma(a[j + 2], sJ[j + 2], d2);
        d3 = fma(a[j + 3], sJ[j + 3], d3);
    }
    const double acc = (d0 + d1) + (d2 + d3);
#pragma unroll
    for (int j = 0; j < TILE; ++j) a[j] *= si;
    rs_stage<16>(a, lane);
    rs_stage<8>(a, lane);
    rs_stage<4>(a, lane);
    rs_stage<2>(a, lane);
    rs_stage<1>(a, lane);
    dir = acc;
    tr = a[0];
}

struct SmallOwn {
    ItemDesc it;     // the operator's single item (descriptors cached for the whole solve)
    int32_t m, mp;
    int32_t toff;    // doubles into the arena
    int32_t ioff;    // ints into the index arena
};

__global__ void __launch_bounds__(256) k_pcg_small(SmallArgs a) {
    extern __shared__ __align__(16) double dsm[];
    __shared__ SmallOwn own[SMALL_MAX_OWN];
    __shared__ int own_col[SMALL_MAX_COL + 1];
    __shared__ int coarse_toff, part_doff[8], part_ioff[8];
    __shared__ double psum[2 * SMALL_MAX_G];
    __shared__ Scalars ss;
    const unsigned g = cluster_rank(), G = gridDim.x;
    const int cseg = (int)G - 1 - (int)g;           // the coarse segment this CTA applies (if < nT_c)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int PW = a.pw;
    double* arena = dsm;                         // resident tiles, coarse tiles, Q blocks
    double* s_sm = arena + a.ad;                 // [PW]
    double* zc = s_sm + PW;                      // [PW]
    double* pw = zc + PW;                        // [8][PW]
    double* bcv = pw + 8 * PW;                   // [ncp] b_c (every CTA)
    double* ycv = bcv + a.ncp;                   // [ncp] y_c (every CTA)
    int32_t* iarena = reinterpret_cast<int32_t*>(ycv + a.ncp);   // index lists, part rows
    const bool writer = g == 0;
    // ---- the resident plan (the same walk as small_plan on the host) ----
    if (tid == 0) {
        int n = 0, od = 0, oi = 0;
        for (int cc = 0; cc < a.ncolours; ++cc) {
            own_col[cc] = n;
            for (int t = a.cops[cc] + (int)g; t < a.cops[cc + 1]; t += G) {
                const OpDesc op = a.ops[t];
                const ItemDesc it = a.items[op.item_base];
                own[n++] = SmallOwn{it, op.m, op.mp, od, oi};
                od += (int)((item_doubles(1, it.I1 - it.I0, it.ntiles, it.tail) + 1) & ~1);
                oi += (op.m + 3) & ~3;
            }
        }
        own_col[a.ncolours] = n;
        coarse_toff = od;
        if (cseg < a.nTc) od += (a.nTc - 1) * TILE_ELEMS + DIAG_ELEMS;
        for (int ww = 0; ww < 8; ++ww) {
            part_doff[ww] = od;
            part_ioff[ww] = oi;
            for (int I = (int)g + (int)G * ww; I < a.nparts; I += (int)G * 8) {
                const int mI = (int)(a.bptr[I + 1] - a.bptr[I]);
                od += ((mI * (a.cptr[I + 1] - a.cptr[I])) + 1) & ~1;
                oi += (mI + 3) & ~3;
            }
        }
        ss = *a.sc;
        if (!writer) ss.ab = nullptr;
    }
    __syncthreads();
    // ---- load the resident data once ----
    // b_c and y_c: the restriction writes only the n_c real entries, while the
    // coarse tile products read whole tiles, so the padding must hold zeros (not
    // stale shared memory: 0 * NaN is NaN); zeroed before the first cluster
    // barrier, i.e. before any CTA stores into another's copy
    for (int x = tid; x < 2 * a.ncp; x += blockDim.x) bcv[x] = 0.0;
    for (int e = 0; e < own_col[a.ncolours]; ++e) {
        const ItemDesc& it = own[e].it;
        const OpDesc op = a.ops[it.op];
        const int64_t nd = item_doubles(1, it.I1 - it.I0, it.ntiles, it.tail);
        for (int64_t x = tid; x < nd; x += blockDim.x) arena[own[e].toff + x] = __ldg(a.tiles + it.tile_off + x);
        for (int x = tid; x < op.m; x += blockDim.x) iarena[own[e].ioff + x] = __ldg(a.oidx + op.idx_off + x);
    }
    if (cseg < a.nTc) {            // coarse tiles (s, 0..s) then (s+1..nTc-1, s): full tiles, diagonal packed
        const ItemDesc it = a.items[a.coarse_item];
        int o = coarse_toff;
        for (int q = 0; q < a.nTc; ++q) {
            const int I = q <= cseg ? cseg : q, J = q <= cseg ? q : cseg;
            const int l = I * (I + 1) / 2 + J;
            const double* src = a.tiles + it.tile_off + item_tile_off(it, l, I);
            const int nd = I == J ? DIAG_ELEMS : TILE_ELEMS;
            for (int x = tid; x < nd; x += blockDim.x) arena[o + x] = __ldg(src + x);
            o += nd;
        }
    }
    for (int ww = 0; ww < 8; ++ww) {
        int od = part_doff[ww], oi = part_ioff[ww];
        for (int I = (int)g + (int)G * ww; I < a.nparts; I += (int)G * 8) {
            const int64_t b0 = a.bptr[I];
            const int mI = (int)(a.bptr[I + 1] - b0), nc = a.cptr[I + 1] - a.cptr[I];
            for (int x = tid; x < mI * nc; x += blockDim.x) arena[od + x] = __ldg(a.Q + a.qoff[I] + x);
            for (int x = tid; x < mI; x += blockDim.x) iarena[oi + x] = __ldg(a.bidx + b0 + x);
            od += ((mI * nc) + 1) & ~1;
            oi += (mI + 3) & ~3;
        }
    }
    __syncthreads();
    const int64_t gt = (int64_t)g * blockDim.x + tid, gs = (int64_t)G * blockDim.x;
    int red = 0;
    auto csum = [&](double v) -> double {           // cluster sum: block sums all-gathered through DSMEM
        const double b = block_sum(v);
        double* slot = psum + (red & 1) * SMALL_MAX_G;  // two slots: the next sum never overwrites one being read
        ++red;
        if (tid < (int)G) st_cluster(slot + g, tid, b);
        cluster_barrier();
        double t = 0.0;
        for (unsigned i = 0; i < G; ++i) t += slot[i];
        return t;
    };
    auto finish = [&](auto&& fn) {
        if (tid == 0) fn();
        __syncthreads();
    };
    // one colour: s = R~_i (r - A z), z[Omega~_i] += A_i^{-1} s for the CTA's operators
    auto colour = [&](int cc, bool zzero) {
        for (int e = own_col[cc]; e < own_col[cc + 1]; ++e) {
            const ItemDesc& it = own[e].it;
            const int m = own[e].m, mp = own[e].mp;
            const int32_t* idx = iarena + own[e].ioff;
            const double* T0 = arena + own[e].toff;
            for (int x = tid; x < mp; x += blockDim.x) {
                double v = 0.0, zv = 0.0;
                if (x < m) {
                    const int node = idx[x];
                    if (!zzero) zv = __ldcg(a.z + node);
                    v = __ldcg(a.r + node) - (zzero ? 0.0 : row_dot1<true>(a.A, node, a.z));
                }
                s_sm[x] = v;
                zc[x] = zv;
            }
            for (int x = tid; x < 8 * PW; x += blockDim.x) pw[x] = 0.0;
            __syncthreads();
            if (a.dbg) small_stamp();
            for (int l = w; l < it.ntiles; l += 8) {
                int I, J;
                item_tile(it, l, I, J);
                double t[TILE], dir, tr;
                smem_tile_row(t, T0 + item_tile_off(it, l, I), I == J, lane, item_tile_rows(it, I));
                small_tile(t, s_sm + J * TILE, s_sm[I * TILE + lane], dir, tr, lane);
                double* pwr = pw + w * PW;
                if (I != J) {
                    pwr[I * TILE + lane] += dir;
                    pwr[J * TILE + lane] += tr;
                } else {
                    pwr[I * TILE + lane] += dir + tr;
                }
            }
            __syncthreads();
            if (a.dbg) small_stamp();
            for (int x = tid; x < m; x += blockDim.x) {
                double y = 0.0;
#pragma unroll
                for (int ww = 0; ww < 8; ++ww) y += pw[ww * PW + x];
                a.z[idx[x]] = zc[x] + y;
            }
            __syncthreads();
            if (a.dbg) small_stamp();
        }
        cluster_barrier();
    };
    auto precond = [&]() {                          // PAPER.md:552-564; z = 0 on entry
        for (int cc = 0; cc < a.ncolours; ++cc) colour(cc, cc == 0);
        // b_c = P^T (r - A z) (warp per part), broadcast to every CTA
        {
            int od = part_doff[w], oi = part_ioff[w];
            double* res = pw + w * PW;
            for (int I = (int)g + (int)G * w; I < a.nparts; I += (int)G * 8) {
                const int mI = (int)(a.bptr[I + 1] - a.bptr[I]), c0 = a.cptr[I], nc = a.cptr[I + 1] - c0;
                const double* QI = arena + od;
                const int32_t* rows = iarena + oi;
                for (int x = lane; x < mI; x += 32) {
                    const int v = rows[x];
                    res[x] = __ldcg(a.r + v) - row_dot1<true>(a.A, v, a.z);
                }
                __syncwarp();
                for (int i = 0; i < nc; ++i) {
                    double acc = 0.0;
                    for (int x = lane; x < mI; x += 32) acc += QI[i * mI + x] * res[x];
                    acc = warp_sum(acc);
                    if (lane < (int)G) st_cluster(bcv + c0 + i, lane, acc);
                }
                __syncwarp();
                od += ((mI * nc) + 1) & ~1;
                oi += (mI + 3) & ~3;
            }
        }
        cluster_barrier();
        // y_c segment g = row g and column g of A_c^{-1} times b_c, broadcast
        if (cseg < a.nTc) {
            pw[w * PW + lane] = 0.0;
            __syncwarp();
            for (int q = w; q < a.nTc; q += 8) {
                const int I = q <= cseg ? cseg : q, J = q <= cseg ? q : cseg;
                const int toff = q <= cseg ? q * TILE_ELEMS : (q - 1) * TILE_ELEMS + DIAG_ELEMS;
                double t[TILE], dir, tr;
                smem_tile_row(t, arena + coarse_toff + toff, I == J, lane, TILE);
                small_tile(t, bcv + J * TILE, bcv[I * TILE + lane], dir, tr, lane);
                pw[w * PW + lane] += I == J ? dir + tr : (I == cseg ? dir : tr);
            }
            __syncthreads();
            if (w == 0) {
                double y = 0.0;
#pragma unroll
                for (int ww = 0; ww < 8; ++ww) y += pw[ww * PW + lane];
                for (unsigned c = 0; c < G; ++c) st_cluster(ycv + cseg * TILE + lane, c, y);
            }
        }
        cluster_barrier();
        // z += P y_c (warp per part)
        {
            int od = part_doff[w], oi = part_ioff[w];
            for (int I = (int)g + (int)G * w; I < a.nparts; I += (int)G * 8) {
                const int mI = (int)(a.bptr[I + 1] - a.bptr[I]), c0 = a.cptr[I], nc = a.cptr[I + 1] - c0;
                const double* QI = arena + od;
                const int32_t* rows = iarena + oi;
                for (int x = lane; x < mI; x += 32) {
                    const int v = rows[x];
                    double acc = 0.0;
                    for (int i = 0; i < nc; ++i) acc += QI[i * mI + x] * ycv[c0 + i];
                    a.z[v] = __ldcg(a.z + v) + acc;
                }
                od += ((mI * nc) + 1) & ~1;
                oi += (mI + 3) & ~3;
            }
        }
        cluster_barrier();
        for (int cc = a.ncolours - 1; cc >= 0; --cc) colour(cc, false);
    };
    double* hist = writer ? a.hist : nullptr;
    // r = f, u = 0, ||f||
    {
        double acc = 0.0;
        for (int64_t i = gt; i < a.n; i += gs) {
            const double v = a.f[i];
            a.r[i] = v;
            a.u[i] = 0.0;
            a.z[i] = 0.0;                           // M r starts from z = 0
            acc += v * v;
        }
        const double t = csum(acc);
        finish([&] { fin_init(&ss, hist, t); });
    }
    if (!ss.done) {
        precond();
        double acc = 0.0;                           // rho = r^T z, p = z
        for (int64_t i = gt; i < a.n; i += gs) {
            const double zi = __ldcg(a.z + i);
            a.p[i] = zi;
            acc += __ldcg(a.r + i) * zi;
        }
        const double t = csum(acc);
        finish([&] { fin_rz_first(&ss, t); });
    }
    while (!ss.done) {
        double acc = 0.0;                           // q = A p, sigma = p^T q
        for (int64_t i = gt; i < a.n; i += gs) {
            const double v = row_dot1<true>(a.A, i, a.p);
            a.q[i] = v;
            a.z[i] = 0.0;                           // for this iteration's M r
            acc += __ldcg(a.p + i) * v;
        }
        double t = csum(acc);
        finish([&] { fin_spmv_dot(&ss, t); });
        if (ss.done) break;
        const double alpha = ss.alpha;              // u += alpha p, r -= alpha q, ||r||, stopping rule
        acc = 0.0;
        for (int64_t i = gt; i < a.n; i += gs) {
            a.u[i] += alpha * __ldcg(a.p + i);
            const double ri = __ldcg(a.r + i) - alpha * __ldcg(a.q + i);
            a.r[i] = ri;
            acc += ri * ri;
        }
        t = csum(acc);
        finish([&] { fin_update(&ss, hist, t); });
        if (ss.done) break;
        precond();
        acc = 0.0;                                  // rho' = r^T z, beta
        for (int64_t i = gt; i < a.n; i += gs) acc += __ldcg(a.r + i) * __ldcg(a.z + i);
        t = csum(acc);
        finish([&] { fin_rz(&ss, t); });
        if (ss.done) break;
        const double beta = ss.beta;                // p = z + beta p
        for (int64_t i = gt; i < a.n; i += gs) a.p[i] = __ldcg(a.z + i) + beta * __ldcg(a.p + i);
        cluster_barrier();
    }
    if (writer && tid == 0) {
        ss.ab = a.sc->ab;
        *a.sc = ss;
    }
}

// debug (DDG_SMALL_TRACE): enable the barrier timestamps / read them back
int small_trace(int on, unsigned long long* out, int cap) {
    static unsigned long long* buf = nullptr;
    if (on) {
        if (!buf) cudaMalloc(&buf, 4096 * sizeof(unsigned long long));
        int z = 0;
        cudaMemcpyToSymbol(g_small_trace, &buf, sizeof buf);
        cudaMemcpyToSymbol(g_small_ntrace, &z, sizeof z);
        return 0;
    }
    int n = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&n, g_small_ntrace, sizeof n);
    n = std::min(n, cap);
    if (buf && n > 0) cudaMemcpy(out, buf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long* none = nullptr;
    cudaMemcpyToSymbol(g_small_trace, &none, sizeof none);
    return n;
}

// can one cluster of G CTAs with `smem` bytes of dynamic shared memory each be
// launched: a trial launch of an empty kernel with the same shape (the
// occupancy query reports 0 for non-portable cluster sizes here)
__global__ void __launch_bounds__(256) k_cluster_probe(int* out) {
    extern __shared__ double probe_sm[];
    if (threadIdx.x == 0) probe_sm[0] = 1.0;
    cluster_barrier();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = (int)(probe_sm[0] + gridDim.x) - 1;
}
bool small_cluster_ok(int G, size_t smem) {
    static bool init = false;
    static int* d_out = nullptr;
    if (!init) {
        int dev = 0, optin = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        for (auto k : {(const void*)k_pcg_small, (const void*)k_cluster_probe}) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, k);      // the dynamic maximum excludes the static shared memory
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
            cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        cudaMalloc(&d_out, sizeof(int));
        cudaGetLastError();
        init = true;
    }
    if (!d_out) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem + 4096;             // + the small kernel's static shared memory
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int h = 0;
    cudaMemset(d_out, 0, sizeof(int));
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster_probe, d_out);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&h, d_out, sizeof(int), cudaMemcpyDeviceToHost);
    if (getenv("DDG_VERBOSE"))
        fprintf(stderr, "[ddg] cluster probe: %d CTAs x %zu B: %s (%d)\n", G, smem, cudaGetErrorString(e), h);
    cudaGetLastError();
    return e == cudaSuccess && h == G;
}

bool launch_pcg_small(cudaStream_t st, const SmallArgs& args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(args.G);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cfg.dynamicSmemBytes = args.smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = args.G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_pcg_small, args);
    if (e != cudaSuccess) {
        if (getenv("DDG_VERBOSE")) fprintf(stderr, "[ddg] k_pcg_small: %s\n", cudaGetErrorString(e));
        cudaGetLastError();
        return false;
    }
    return true;
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
