// coarse.cu — coarse correction (a5-a7): restriction, prolongation, the sparse coarse solve (dataflow and level kernels)
// (part of libddg's sm_100a kernels; shared device helpers in kernel_common.cuh)
#include "kernel_common.cuh"

namespace ddg {
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

// Two-stage restriction (single GPU): k_gather_flat first writes the
// residual res[x] = (r - A z)[bidx[x]] for every position x in part order
// (one coalesced pass at streaming speed), then b_c[I,:] = Q_I^T res[Omega_I]
// reads Q_I and res contiguously, warp per part.
template <int R>
__global__ void __launch_bounds__(256)
k_restrict_dot(int nparts, const int64_t* __restrict__ bptr, const int32_t* __restrict__ cptr,
               const int64_t* __restrict__ qoff, const double* __restrict__ Q, const double* __restrict__ res,
               double* __restrict__ bc, const int32_t* done) {
    pdl_wait();
    if (*done) return;
    const int I = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (I >= nparts) return;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    const int c0 = cptr[I], ncI = cptr[I + 1] - c0;
    const double* QI = Q + qoff[I];
    double rv[R];
#pragma unroll
    for (int k = 0; k < R; ++k) rv[k] = lane + 32 * k < mI ? res[b0 + lane + 32 * k] : 0.0;
    for (int i = 0; i < ncI; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int a = lane + 32 * k;
            if (a < mI) acc += QI[(int64_t)i * mI + a] * rv[k];
        }
        acc = warp_sum(acc);
        if (lane == 0) bc[c0 + i] = acc;
    }
}

// large parts: block per part, one block reduction per coarse column
__global__ void __launch_bounds__(256)
k_restrict_dot_block(const int64_t* __restrict__ bptr, const int32_t* __restrict__ cptr,
                     const int64_t* __restrict__ qoff, const double* __restrict__ Q,
                     const double* __restrict__ res, double* __restrict__ bc, const int32_t* done) {
    pdl_wait();
    if (*done) return;
    const int I = blockIdx.x;
    const int64_t b0 = bptr[I];
    const int mI = (int)(bptr[I + 1] - b0);
    const int c0 = cptr[I], ncI = cptr[I + 1] - c0;
    const double* QI = Q + qoff[I];
    for (int i = 0; i < ncI; ++i) {
        double acc = 0.0;
        for (int a = threadIdx.x; a < mI; a += blockDim.x) acc += QI[(int64_t)i * mI + a] * res[b0 + a];
        acc = block_sum(acc);
        if (threadIdx.x == 0) bc[c0 + i] = acc;
    }
}

// Flat prolongation (single GPU): thread per position x of the part order,
// z[bidx[x]] += sum_i Q_I[a, i] y_c[I, i] with I = xpart[x], a = x - bptr[I].
__global__ void __launch_bounds__(256)
k_prolong_flat(int64_t n, const int32_t* __restrict__ xpart, const int64_t* __restrict__ bptr,
               const int32_t* __restrict__ bidx, const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff,
               const double* __restrict__ Q, const double* __restrict__ yc, double* __restrict__ z,
               const int32_t* done) {
    pdl_wait();
    if (*done) return;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int I = xpart[x];
        const int64_t b0 = bptr[I];
        const int64_t mI = bptr[I + 1] - b0;
        const int c0 = cptr[I], ncI = cptr[I + 1] - c0;
        const double* q = Q + qoff[I] + (x - b0);
        double acc = 0.0;
        for (int i = 0; i < ncI; ++i) acc += q[i * mI] * yc[c0 + i];
        z[bidx[x]] += acc;
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
    double yq[4];                                                  // k <= 128 coarse columns
#pragma unroll
    for (int h = 0; h < 4; ++h) yq[h] = lane + 32 * h < ncI ? yc[c0 + 32 * h + lane] : 0.0;
    const double* QI = Q + qoff[I];
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    for (int i = 0; i < ncI; ++i) {
        const double ysel = i < 32 ? yq[0] : i < 64 ? yq[1] : i < 96 ? yq[2] : yq[3];
        const double yi = __shfl_sync(FULL, ysel, i & 31);
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
    __shared__ double ys[128];
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
    const int32_t* fchild;
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
// The index loads of one CTA over a front of up to ~25k rows are a chain of
// dependent global round trips per element (index, then value): each thread
// keeps DF_U independent elements in flight (measured: a 24k-row assembly took
// ~150 us one element at a time, on the coarse solve's critical path).
constexpr int DF_U = 8;
__device__ void df_gather_idx(double* __restrict__ out, int n, int ntot, const int32_t* __restrict__ idx,
                              const double* __restrict__ src, bool cg) {
    for (int a0 = threadIdx.x; a0 < ntot; a0 += blockDim.x * DF_U) {
        int ix[DF_U];
#pragma unroll
        for (int u = 0; u < DF_U; ++u) {
            const int a = a0 + u * blockDim.x;
            ix[u] = a < n ? idx[a] : -1;
        }
        double v[DF_U];
#pragma unroll
        for (int u = 0; u < DF_U; ++u) v[u] = ix[u] >= 0 ? (cg ? __ldcg(src + ix[u]) : src[ix[u]]) : 0.0;
#pragma unroll
        for (int u = 0; u < DF_U; ++u) {
            const int a = a0 + u * blockDim.x;
            if (a < ntot) out[a] = v[u];
        }
    }
}
__device__ void df_assemble(const DFCtx& d, int t) {
    const FrontDesc f = d.fronts[t];
    double* fv = d.fvec + f.fvec_off;
    double* wt = d.w + f.w_off;
    const int ntot = f.nT * TILE;
    df_gather_idx(fv, f.nS, ntot, d.fS + f.S_off, d.bc, false);
    for (int a = threadIdx.x; a < f.nB; a += blockDim.x) wt[a] = 0.0;
    __syncthreads();
    for (int k = 0; k < f.nchild; ++k) {                      // children in fixed order
        const int ci = d.fchild[f.child_off + k];
        const FrontDesc c = d.fronts[ci];
        for (int j0 = threadIdx.x; j0 < c.nB; j0 += blockDim.x * DF_U) {
            int pos[DF_U];
            double v[DF_U];
#pragma unroll
            for (int u = 0; u < DF_U; ++u) {
                const int j = j0 + u * blockDim.x;
                pos[u] = j < c.nB ? d.map[c.map_off + j] : -1;
                v[u] = j < c.nB ? __ldcg(d.w + c.w_off + j) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < DF_U; ++u) {   // positions are distinct within a child
                if (pos[u] < 0) continue;
                if (pos[u] < f.nSp) fv[pos[u]] += v[u];
                else wt[pos[u] - f.nSp] += v[u];
            }
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
            sh[0] = atomicAdd(df_flag(d, f.parent, DFF_CHILDREN), 1) == p.nchild - 1;
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
                  const double* __restrict__ ctiles, const int32_t* done, uint64_t* trace, int pf) {
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
        if (pf > 0 && threadIdx.x == 0 && q + pf < nwork) {     // L2 prefetch of a later work item's tiles
            const int32_t ep = work[q + pf];
            if (!(ep & (DF_ASSEMBLE | DF_RED))) {
                const ItemDesc ip = items[ep & DF_IDX];
                bulk_prefetch_l2(ctiles + ip.tile_off, (unsigned)(item_doubles(ip.tri, ip.I1 - ip.I0, ip.ntiles) * 8));
            }
        }
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
                for (int k = 0; k < f.nchild; ++k) {               // children: gather x[B_c]
                    const int ci = d.fchild[f.child_off + k];
                    const FrontDesc c = d.fronts[ci];
                    double* fv = d.fvec + c.fvec_off + c.nSp;
                    df_gather_idx(fv, c.nB, c.nT * TILE - c.nSp, d.fB + c.B_off, d.x, true);
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
                            const int32_t* fchild,
                            const FrontDF* fdf, const int32_t* item_front, int item_base, const OpDesc* ops,
                            const ItemDesc* items, const double* ctiles, const FRedTask* fwd, const FRedTask* bwd,
                            const int64_t* contrib, const int32_t* fS, const int32_t* fB, const int32_t* map,
                            const double* bc, double* fvec, double* w, double* x, double* partials,
                            int32_t* state, int max_rows_t, const int32_t* done, uint64_t* trace) {
    if (nwork <= 0) return;
    DFCtx d{fronts, fchild, fdf, fwd, bwd, contrib, fS, fB, map, bc, fvec, w, x, partials, state};
    const size_t smem = (size_t)max_rows_t * (SYMV_WARPS + 1) * sizeof(double);
    static bool init_dev[64] = {};   // function attributes are per device
    int dev_ = 0;
    cudaGetDevice(&dev_);
    bool& init = init_dev[dev_ & 63];
    if (!init) {
        cudaFuncSetAttribute(k_coarse_dataflow, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        init = true;
    }
    const int grid = std::min(nwork, num_sms() * 2);
    static int pfq = getenv("DDG_DF_PF") ? atoi(getenv("DDG_DF_PF")) : 0;   // work entries ahead (0: off)
    k_coarse_dataflow<<<grid, SYMV_WARPS * 32, smem, st>>>(nwork, work, d, item_front, item_base, ops, items,
                                                           ctiles, done, trace, pfq);
}

// forward: front vector [b_S ; 0] and w_t = incoming contributions to B
__global__ void k_front_fwd_assemble(int f0, const FrontDesc* __restrict__ fronts, const int32_t* __restrict__ fchild,
                                     const int32_t* __restrict__ fS, const int32_t* __restrict__ map,
                                     const double* __restrict__ bc, double* __restrict__ fvec,
                                     double* __restrict__ w, const int32_t* done) {
    if (*done) return;
    const FrontDesc f = fronts[f0 + blockIdx.x];
    double* fv = fvec + f.fvec_off;
    double* wt = w + f.w_off;
    const int ntot = f.nT * TILE;
    df_gather_idx(fv, f.nS, ntot, fS + f.S_off, bc, false);
    for (int a = threadIdx.x; a < f.nB; a += blockDim.x) wt[a] = 0.0;
    __syncthreads();
    for (int s = 0; s < f.nchild; ++s) {
        const int ci = fchild[f.child_off + s];
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
    df_gather_idx(fv, f.nB, f.nT * TILE - f.nSp, fB + f.B_off, x, false);
}

__global__ void k_front_reduce(const FRedTask* __restrict__ tasks, int t0,
                               const int64_t* __restrict__ contrib, const FrontDesc* __restrict__ fronts,
                               const int32_t* __restrict__ fS, const double* __restrict__ partials,
                               double* __restrict__ w, double* __restrict__ x, const int32_t* done) {
    if (*done) return;
    const FRedTask t = tasks[t0 + blockIdx.x];
    const FrontDesc f = fronts[t.front];
    for (int r = threadIdx.x; r < t.nrows; r += blockDim.x) {
        // df_reduce's combine order (k_coarse_dataflow), so the level-by-level and the
        // distributed top-front steps give the dataflow solve's values bitwise
        double s = 0.0;
        int c = t.cbeg;
        for (; c + 8 <= t.cend; c += 8) {
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = partials[contrib[c + k] + r];
            s += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        }
        for (; c < t.cend; ++c) s += partials[contrib[c] + r];
        const int row = t.row0 + r;
        if (t.kind == 0) {
            const int b = row - f.nSp;
            if (b >= 0 && b < f.nB) w[f.w_off + b] += s;
        } else if (row < f.nS) {
            x[fS[f.S_off + row]] = s;
        }
    }
}


// ---- launchers ----

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
    if (smem > 48 * 1024) DDG_MAX_DYN_SMEM(k_coarse_restrict);
    k_coarse_restrict<<<nparts, 256, smem, st>>>(bptr, bidx, cptr, qoff, Q, A, r, z, bc, done, parts);
}

void launch_restrict_dot(cudaStream_t st, int nparts, const int64_t* bptr, const int32_t* cptr, const int64_t* qoff,
                         const double* Q, const double* res, double* bc, int maxmI, const int32_t* done) {
    if (nparts <= 0) return;
    const int g = (nparts + 7) / 8;
    if (maxmI <= 64) launch_pdl(k_restrict_dot<2>, g, 256, 0, st, nparts, bptr, cptr, qoff, Q, res, bc, done);
    else if (maxmI <= 128) launch_pdl(k_restrict_dot<4>, g, 256, 0, st, nparts, bptr, cptr, qoff, Q, res, bc, done);
    else if (maxmI <= 256) launch_pdl(k_restrict_dot<8>, g, 256, 0, st, nparts, bptr, cptr, qoff, Q, res, bc, done);
    else if (maxmI <= 512) launch_pdl(k_restrict_dot<16>, g, 256, 0, st, nparts, bptr, cptr, qoff, Q, res, bc, done);
    else launch_pdl(k_restrict_dot_block, nparts, 256, 0, st, bptr, cptr, qoff, Q, res, bc, done);
}

void launch_prolong_flat(cudaStream_t st, int64_t n, const int32_t* xpart, const int64_t* bptr, const int32_t* bidx,
                         const int32_t* cptr, const int64_t* qoff, const double* Q, const double* yc, double* z,
                         const int32_t* done) {
    if (n <= 0) return;
    launch_pdl(k_prolong_flat, vec_grid(n), 256, 0, st, n, xpart, bptr, bidx, cptr, qoff, Q, yc, z, done);
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

void launch_front_fwd_assemble(cudaStream_t st, int f0, int nf, const FrontDesc* fronts, const int32_t* fchild,
                               const int32_t* fS, const int32_t* map, const double* bc, double* fvec,
                               double* w, const int32_t* done) {
    if (nf <= 0) return;
    k_front_fwd_assemble<<<nf, 256, 0, st>>>(f0, fronts, fchild, fS, map, bc, fvec, w, done);
}

void launch_front_bwd_gather(cudaStream_t st, int f0, int nf, const FrontDesc* fronts,
                             const int32_t* fB, const double* x, double* fvec, const int32_t* done) {
    if (nf <= 0) return;
    k_front_bwd_gather<<<nf, 256, 0, st>>>(f0, fronts, fB, x, fvec, done);
}

// distributed coarse solve (coarse_sparse.cpp) --------------
// dst[k] = mask[k] ? src[idx ? idx[k] : k] : 0  (a rank's share of an allreduce)
__global__ void k_gather_masked(int64_t n, const int32_t* __restrict__ idx, const uint8_t* __restrict__ mask,
                                const double* __restrict__ src, double* __restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        dst[k] = mask[k] ? src[idx ? idx[k] : k] : 0.0;
}
// copy segments [src_off, src_off + len) -> [dst_off, ...), one CTA per segment
__global__ void k_copy_segments(const int64_t* __restrict__ seg, const double* __restrict__ src,
                                double* __restrict__ dst) {
    const int64_t so = seg[3 * blockIdx.x], doff = seg[3 * blockIdx.x + 1], len = seg[3 * blockIdx.x + 2];
    for (int64_t x = threadIdx.x; x < len; x += blockDim.x) dst[doff + x] = src[so + x];
}
void launch_copy_segments(cudaStream_t st, int nseg, const int64_t* seg, const double* src, double* dst) {
    for (int s0 = 0; s0 < nseg; s0 += 65535)
        k_copy_segments<<<std::min(65535, nseg - s0), 256, 0, st>>>(seg + 3 * (int64_t)s0, src, dst);
}
void launch_gather_masked(cudaStream_t st, int64_t n, const int32_t* idx, const uint8_t* mask, const double* src,
                          double* dst) {
    if (n > 0) k_gather_masked<<<vec_grid(n), VEC_THREADS, 0, st>>>(n, idx, mask, src, dst);
}

void launch_front_reduce(cudaStream_t st, const FRedTask* tasks, int t0, int nt, const int64_t* contrib,
                         const FrontDesc* fronts, const int32_t* fS, const double* partials, double* w,
                         double* x, const int32_t* done) {
    if (nt <= 0) return;
    k_front_reduce<<<nt, 256, 0, st>>>(tasks, t0, contrib, fronts, fS, partials, w, x, done);
}

}  // namespace ddg
