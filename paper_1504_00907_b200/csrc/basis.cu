// basis.cu — the DDG coarse space on the device:
//   * per-part orthonormal basis Q_I of span F[Omega_I, :] (PAPER.md:253-264,
//     269-280): modified Gram-Schmidt in double-double (reading R6c), one warp
//     per part, columns in the given order, column j kept iff
//     ||v_j|| >= rank_tol ||F_I e_j|| (reading R7);
//   * the Galerkin product A_c = P^T A P block by block:
//     A_c[I, J] = Q_I^T (A[Omega_I, Omega_J] Q_J) for adjacent parts I >= J
//     (the block pattern of PAPER.md:282-287), one CTA per block.
// Every sum runs in a fixed order (lanes strided, butterfly combine; rows of
// Omega_I ascending), so setup is bitwise repeatable.
#include "kernel_common.cuh"

namespace ddg {

// ---- double-double arithmetic (error-free transformations) -----------------
struct dd_t {
    double hi, lo;
};
__device__ __forceinline__ dd_t dd_quick(double a, double b) {   // |a| >= |b|
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ dd_t dd_exact_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd_t dd_add(dd_t x, dd_t y) {
    dd_t s = dd_exact_sum(x.hi, y.hi);
    const dd_t t = dd_exact_sum(x.lo, y.lo);
    s = dd_quick(s.hi, s.lo + t.hi);
    return dd_quick(s.hi, s.lo + t.lo);
}
__device__ __forceinline__ dd_t dd_mul(dd_t x, dd_t y) {
    const double p = x.hi * y.hi;
    return dd_quick(p, fma(x.hi, y.hi, -p) + (x.hi * y.lo + x.lo * y.hi));
}
__device__ __forceinline__ dd_t dd_neg(dd_t x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd_t dd_divide(dd_t x, dd_t y) {   // three correction steps
    const double q1 = x.hi / y.hi;
    dd_t r = dd_add(x, dd_neg(dd_mul({q1, 0.0}, y)));
    const double q2 = r.hi / y.hi;
    r = dd_add(r, dd_neg(dd_mul({q2, 0.0}, y)));
    const double q3 = r.hi / y.hi;
    return dd_add(dd_quick(q1, q2), {q3, 0.0});
}
__device__ __forceinline__ dd_t dd_root(dd_t a) {   // one Newton step from the double root
    if (a.hi <= 0.0) return {0.0, 0.0};
    const double x = sqrt(a.hi);
    const dd_t r = dd_add(a, dd_neg(dd_mul({x, 0.0}, {x, 0.0})));
    return dd_add({x, 0.0}, {r.hi / (2.0 * x), 0.0});
}
__device__ __forceinline__ dd_t dd_warp_sum(dd_t v) {   // identical on every lane
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const dd_t w = {__shfl_xor_sync(FULL, v.hi, o), __shfl_xor_sync(FULL, v.lo, o)};
        v = dd_add(v, w);
    }
    return v;
}

// ---- per-part basis: one warp per part ---------------------------------------
// V (scratch, double2 {hi, lo}): part I's columns at voff[I] + slot * m_I;
// kept columns are compacted to slots 0 .. rank-1.  Outputs: rank[I],
// ratio[I] (min over kept columns of ||v_j|| / ||F_I e_j||), Qw[voff[I] + ...]
// = hi parts of the kept columns; err[0] = a part whose F block is zero.
__global__ void __launch_bounds__(256) k_basis_mgs(int nparts, int k, int64_t n, const double* __restrict__ F,
                                                   const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                                                   const int64_t* __restrict__ voff, double2* __restrict__ V,
                                                   double* __restrict__ Qw, int32_t* __restrict__ rank,
                                                   double* __restrict__ ratio, double rank_tol, int32_t* err) {
    const int lane = threadIdx.x & 31;
    const int I = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (I >= nparts) return;
    const int64_t m = bptr[I + 1] - bptr[I];
    const int32_t* rows = bidx + bptr[I];
    double2* Vp = V + voff[I];
    int r = 0;
    double minrt = INFINITY;
    bool any = false;
    for (int j = 0; j < k; ++j) {
        const double* Fj = F + (int64_t)j * n;
        double2* v = Vp + (int64_t)r * m;          // the candidate goes to the next free slot
        dd_t fs = {0.0, 0.0};
        for (int64_t a = lane; a < m; a += 32) {
            const double x = Fj[rows[a]];
            v[a] = make_double2(x, 0.0);
            fs = dd_add(fs, dd_mul({x, 0.0}, {x, 0.0}));
        }
        const double fn = dd_root(dd_warp_sum(fs)).hi;
        any |= fn > 0.0;
        __syncwarp();
        for (int t = 0; t < r; ++t) {              // v -= (q_t . v) q_t, in dd
            const double2* q = Vp + (int64_t)t * m;
            dd_t s = {0.0, 0.0};
            for (int64_t a = lane; a < m; a += 32) {
                const double2 qa = q[a], va = v[a];
                s = dd_add(s, dd_mul({qa.x, qa.y}, {va.x, va.y}));
            }
            s = dd_neg(dd_warp_sum(s));
            for (int64_t a = lane; a < m; a += 32) {
                const double2 qa = q[a], va = v[a];
                const dd_t nv = dd_add({va.x, va.y}, dd_mul(s, {qa.x, qa.y}));
                v[a] = make_double2(nv.hi, nv.lo);
            }
            __syncwarp();
        }
        dd_t ss = {0.0, 0.0};
        for (int64_t a = lane; a < m; a += 32) {
            const double2 va = v[a];
            ss = dd_add(ss, dd_mul({va.x, va.y}, {va.x, va.y}));
        }
        const dd_t nrm = dd_root(dd_warp_sum(ss));
        const double rt = fn > 0.0 ? nrm.hi / fn : 0.0;
        if (rt >= rank_tol && nrm.hi > 0.0) {       // keep: normalise in place
            for (int64_t a = lane; a < m; a += 32) {
                const double2 va = v[a];
                const dd_t q = dd_divide({va.x, va.y}, nrm);
                v[a] = make_double2(q.hi, q.lo);
                Qw[voff[I] + (int64_t)r * m + a] = q.hi;
            }
            minrt = fmin(minrt, rt);
            ++r;
        }
        __syncwarp();
    }
    if (lane == 0) {
        rank[I] = r;
        ratio[I] = minrt;
        if (!any) atomicCAS(err, -1, I);
    }
}

// compact the kept columns: Q_I (m_I x rank_I, column-major) at qoff[I]
__global__ void k_basis_compact(int nparts, const int64_t* __restrict__ bptr, const int64_t* __restrict__ voff,
                                const int64_t* __restrict__ qoff, const double* __restrict__ Qw,
                                double* __restrict__ Q) {
    for (int I = blockIdx.x; I < nparts; I += gridDim.x) {
        const int64_t len = qoff[I + 1] - qoff[I];
        for (int64_t x = threadIdx.x; x < len; x += blockDim.x) Q[qoff[I] + x] = Qw[voff[I] + x];
    }
}

// ---- Galerkin blocks: one CTA per adjacent pair (I >= J) ----------------------
// out[boff[b] + i * rJ + j] = sum_{u in Omega_I, ascending} Q_I(u, i) w_J(u, j),
// w_J(u, j) = sum over row u's entries x with part(col x) = J of
//             val_x Q_J(pos(col x), j)           (CSR order)
// Rows in batches of GAL_RB: the batch's Q_I rows and w_J values are staged in
// shared memory, then each thread adds its outputs in row order.
constexpr int GAL_THREADS = 128, GAL_RB = 32, GAL_OUT = 8;   // outputs per thread per pass
__global__ void __launch_bounds__(GAL_THREADS)
k_galerkin_blocks(const int32_t* __restrict__ bI, const int32_t* __restrict__ bJ, const int64_t* __restrict__ boff,
                  const int64_t* __restrict__ bptr, const int32_t* __restrict__ bidx,
                  const int32_t* __restrict__ cptr, const int64_t* __restrict__ qoff, const double* __restrict__ Q,
                  const int32_t* __restrict__ part, const int32_t* __restrict__ bpos, const int32_t* __restrict__ rp,
                  const int32_t* __restrict__ col, const double* __restrict__ val, double* __restrict__ out) {
    extern __shared__ double gs[];
    const int b = blockIdx.x;
    const int I = bI[b], J = bJ[b];
    const int rI = cptr[I + 1] - cptr[I], rJ = cptr[J + 1] - cptr[J];
    const int64_t mI = bptr[I + 1] - bptr[I], mJ = bptr[J + 1] - bptr[J];
    const double* QI = Q + qoff[I];
    const double* QJ = Q + qoff[J];
    double* qs = gs;                    // [GAL_RB][rI]
    double* ws = gs + GAL_RB * rI;      // [GAL_RB][rJ]
    const int nout = rI * rJ;
    for (int o0 = 0; o0 < nout; o0 += GAL_THREADS * GAL_OUT) {
        double acc[GAL_OUT];
#pragma unroll
        for (int t = 0; t < GAL_OUT; ++t) acc[t] = 0.0;
        for (int64_t a0 = 0; a0 < mI; a0 += GAL_RB) {
            const int nr = (int)(mI - a0 < GAL_RB ? mI - a0 : GAL_RB);
            __syncthreads();
            for (int e = threadIdx.x; e < nr * rI; e += GAL_THREADS) {
                const int rr = e / rI, i = e % rI;
                qs[rr * rI + i] = QI[(int64_t)i * mI + a0 + rr];
            }
            for (int e = threadIdx.x; e < nr * rJ; e += GAL_THREADS) {
                const int rr = e / rJ, j = e % rJ;
                const int u = bidx[bptr[I] + a0 + rr];
                double w = 0.0;
                for (int x = rp[u]; x < rp[u + 1]; ++x) {
                    const int cc = col[x];
                    if (part[cc] == J) w += val[x] * QJ[(int64_t)j * mJ + bpos[cc]];
                }
                ws[rr * rJ + j] = w;
            }
            __syncthreads();
#pragma unroll
            for (int t = 0; t < GAL_OUT; ++t) {
                const int o = o0 + t * GAL_THREADS + threadIdx.x;
                if (o < nout) {
                    const int i = o / rJ, j = o % rJ;
                    double s = acc[t];
                    for (int rr = 0; rr < nr; ++rr) s += qs[rr * rI + i] * ws[rr * rJ + j];
                    acc[t] = s;
                }
            }
        }
#pragma unroll
        for (int t = 0; t < GAL_OUT; ++t) {
            const int o = o0 + t * GAL_THREADS + threadIdx.x;
            if (o < nout) out[boff[b] + o] = acc[t];
        }
    }
}

void launch_basis_mgs(cudaStream_t st, int nparts, int k, int64_t n, const double* F, const int64_t* bptr,
                      const int32_t* bidx, const int64_t* voff, double2* V, double* Qw, int32_t* rank,
                      double* ratio, double rank_tol, int32_t* err) {
    if (nparts > 0)
        k_basis_mgs<<<(nparts + 7) / 8, 256, 0, st>>>(nparts, k, n, F, bptr, bidx, voff, V, Qw, rank, ratio,
                                                      rank_tol, err);
}
void launch_basis_compact(cudaStream_t st, int nparts, const int64_t* bptr, const int64_t* voff,
                          const int64_t* qoff, const double* Qw, double* Q) {
    if (nparts > 0) k_basis_compact<<<std::min(nparts, 65535), 128, 0, st>>>(nparts, bptr, voff, qoff, Qw, Q);
}
void launch_galerkin_blocks(cudaStream_t st, int nblocks, int maxk, const int32_t* bI, const int32_t* bJ,
                            const int64_t* boff, const int64_t* bptr, const int32_t* bidx, const int32_t* cptr,
                            const int64_t* qoff, const double* Q, const int32_t* part, const int32_t* bpos,
                            const int32_t* rp, const int32_t* col, const double* val, double* out) {
    if (nblocks <= 0) return;
    const size_t smem = (size_t)GAL_RB * 2 * maxk * sizeof(double);
    if (smem > 48 * 1024) DDG_MAX_DYN_SMEM(k_galerkin_blocks);
    for (int b0 = 0; b0 < nblocks; b0 += 1 << 30)
        k_galerkin_blocks<<<std::min(nblocks - b0, 1 << 30), GAL_THREADS, smem, st>>>(
            bI + b0, bJ + b0, boff + b0, bptr, bidx, cptr, qoff, Q, part, bpos, rp, col, val, out);
}

}  // namespace ddg
