// setup_kernels.cu — setup kernels: local matrix extraction, Gauss-Jordan inversion (tile and blocked), packing, front assembly
// (part of libddg's sm_100a kernels; shared device helpers in kernel_common.cuh)
#include "kernel_common.cuh"

namespace ddg {
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
    double* strip;          // symmetric variant: the new row panel of matrix b at strip + b * strip_stride
    int64_t strip_stride;   // (tile (t, J) of the panel at ((J * GJB_BT + t) * TILE_ELEMS)); nullptr: full
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
// Symmetric variant (bt.strip set, reading R22 in DESIGN.md): the exchange keeps
// M(X,Y) = s M(Y,X)^T (s = -1 when exactly one of X, Y is pivoted).  The
// block-upper tiles whose row and column are both pivoted or both unpivoted
// are not updated; the unpivoted-unpivoted ones are read transposed from
// their mirror (s = +1) where the row panel needs them.  The mixed tiles
// (pivoted rows, unpivoted columns) are kept exactly as in the full exchange.
// The new row panel goes to a strip first (mode 1 still needs the old one),
// and mode 2 copies it back.  About a third of the trailing flops saved.
// MMA: the 128 x 128 block product on the fp64 tensor path (mma.sync m8n8k4,
// each warp a 32 x 64 tile of 4 x 8 fragments): the fragments are read from
// shared memory once per 4-deep k step instead of per FMA, which is what
// bounds the FMA variant (16 B of operands per 8 FMAs).
constexpr int GJB_LDM = GJB_N + 8;         // MMA stage row: conflict-free 8 x 4 fragment loads
template <bool MMA>
__global__ void __launch_bounds__(256) k_gjb_gemm(GJBatch bt, int k0, int mode) {
    constexpr int LDA = MMA ? GJB_LDM : GJB_N, LDB = MMA ? GJB_LDM : GJB_BPAD;
    extern __shared__ double gsm[];
    double* As = gsm;                               // [TILE][LDA] A(row, kk), kk-major
    double* Bs = gsm + TILE * LDA;                  // [TILE][LDB] B(kk, col), kk-major
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
    const bool sym = bt.strip != nullptr;
    const int bk = k0 / GJB_BT;
    double* strip = sym ? bt.strip + (int64_t)b * bt.strip_stride : nullptr;
    auto stile = [&](int t, int J) { return strip + ((int64_t)J * GJB_BT + t) * TILE_ELEMS; };
    // block-upper tiles with both row and column pivoted, or both unpivoted, follow by
    // symmetry; the mixed ones (pivoted rows, unpivoted columns) are kept as in the full
    // exchange, so pivoted rows never take a transposed operand
    if (sym && mode == 1 && bi < bj && !(bi < bk && bj >= bk)) return;
    if (sym && mode == 2) {
        // the new row panel (kb, J), J in block bi, back from the strip
        for (int J = i0; J < min(i0 + GJB_BT, nT); ++J) {
            if (in_kb(J)) continue;
            for (int t = 0; t < k1 - k0; ++t) {
                const double* src = stile(t, J);
                double* dst = bt.mats[b] + ((int64_t)J * nT + k0 + t) * TILE_ELEMS;
                for (int e = threadIdx.x; e < TILE_ELEMS; e += 256) dst[e] = src[e];
            }
        }
    }
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
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wr = (wid & 3) * 32, wc = (wid >> 2) * 64;   // MMA: this warp's 32 x 64 output tile
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
            double v = 0.0;
            if (I < nT && (mode != 0 || I < k1)) {
                v = tile(I, q)[o];
            }
            As[kk * LDA + ti * TILE + r] = v;
        }
        for (int e = threadIdx.x; e < GJB_BT * TILE_ELEMS; e += 256) {
            const int tj = e / TILE_ELEMS, o = e % TILE_ELEMS;   // o = c * 32 + kk
            const int J = (mode == 2 ? k0 : j0) + tj;
            const int c = o / TILE, kk = o % TILE;
            double v = 0.0;
            if (J < nT && (mode != 2 || J < k1)) {
                if (sym && mode == 1) v = stile(q - k0, J)[o];                           // the new row panel
                else if (sym && mode == 0 && J / GJB_BT > bk) v = tile(J, q)[kk * TILE + c];   // both unpivoted
                else v = tile(q, J)[o];
            }
            Bs[kk * LDB + tj * TILE + c] = v;
        }
        __syncthreads();
        if constexpr (MMA) {
            // value v = 16 mi + 2 ni + h of acc (acc[v / 8][v % 8]) is
            // C(wr + 8 mi + lane / 4, wc + 8 ni + 2 (lane % 4) + h)
#pragma unroll 2
            for (int kq = 0; kq < TILE; kq += 4) {
                double af[4], bf[8];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) af[mi] = As[(kq + (lane & 3)) * LDA + wr + 8 * mi + (lane >> 2)];
#pragma unroll
                for (int ni = 0; ni < 8; ++ni) bf[ni] = Bs[(kq + (lane & 3)) * LDB + wc + 8 * ni + (lane >> 2)];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 8; ++ni)
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                     : "+d"(acc[2 * mi + ni / 4][(2 * ni) % 8]), "+d"(acc[2 * mi + ni / 4][(2 * ni) % 8 + 1])
                                     : "d"(af[mi]), "d"(bf[ni]));
            }
            __syncthreads();
            continue;
        }
#pragma unroll 4
        for (int kk = 0; kk < TILE; ++kk) {
            double a[8], bv[8];
            const double2* ap = reinterpret_cast<const double2*>(As + kk * LDA + tr);
            const double* brow = Bs + kk * LDB + tc;
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
    if constexpr (MMA) {
        // rows wr + 8 mi + lane / 4 lie in tile row i0 + wr / 32; columns
        // wc + 8 ni + 2 (lane % 4) + h in tile column j0 + (wc + 8 ni) / 32
        const int I = i0 + wr / TILE;
        if (I >= nT) return;
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) {
            const int J = j0 + (wc + 8 * ni) / TILE;
            if (J >= nT) continue;
            const bool ok = mode == 0 ? (in_kb(I) && !in_kb(J)) : mode == 1 ? (!in_kb(I) && !in_kb(J))
                                                                             : (!in_kb(I) && in_kb(J));
            if (!ok) continue;
            double* T = sym && mode == 0 ? stile(I - k0, J) : tile(I, J);
            const int cc = (wc + 8 * ni) % TILE + 2 * (lane & 3);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double* p = T + (cc + h) * TILE + 8 * mi + (lane >> 2);
                    const double v = acc[2 * mi + ni / 4][(2 * ni) % 8 + h];
                    *p = mode == 1 ? *p + v : (mode == 0 ? -v : v);
                }
        }
        return;
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
        double* T = sym && mode == 0 ? stile(I - k0, J) : tile(I, J);
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

// Pipelined full-exchange block product (the default for the blocked exchange):
// the same three modes as k_gjb_gemm<true> with the operand tiles streamed by
// 16-byte cp.async into GJP_STAGES shared-memory stages (stage q + 2 in flight
// while q computes), B stored column-major per output column so both fragment
// loads are conflict-free; the trailing mode's C tiles are bulk-prefetched into
// L2 at the start, so the epilogue's C + A B read-modify-write hits L2.  (Adding
// the products onto C inside the accumulators instead was measured: the same
// speed, but 1e-14 instead of 3e-15 against numpy's inverse in tools/gjunit.py.)
constexpr int GJP_LDA = GJB_N + 8;                          // As[kk][row]
constexpr int GJP_LDK = TILE + 4;                           // Bs[col][kk]
// BNT: output block width in tiles (4: 128 x 128 per CTA, 8 warps, 3 stages,
// one CTA per SM; 2: 128 x 64 per CTA, 4 warps, 2 stages of 53 KB, two CTAs per
// SM, so one CTA's prologue and epilogue overlap the other's products)
template <int BNT> struct GJP {
    static constexpr int W = 2 * BNT;                                    // warps (32 x 64 outputs each)
    static constexpr int STAGE = TILE * GJP_LDA + BNT * TILE * GJP_LDK;  // doubles per stage
    static constexpr int STAGES = BNT == 4 ? 3 : 2;
};
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
template <int BNT>
__global__ void __launch_bounds__(GJP<BNT>::W * 32) k_gjb_gemm_pipe(GJBatch bt, int k0, int mode) {
    constexpr int W = GJP<BNT>::W, NTH = W * 32, STAGE = GJP<BNT>::STAGE, STAGES = GJP<BNT>::STAGES;
    extern __shared__ __align__(16) double psm[];
    const int b = blockIdx.y;
    const int nT = bt.nT[b], nK = bt.nK[b];
    if (k0 >= nK) return;
    const int k1 = min(k0 + GJB_BT, nK);
    const int nbr = (nT + GJB_BT - 1) / GJB_BT, nbc = (nT + BNT - 1) / BNT;   // row / column blocks
    int i0, j0;
    if (mode == 1) {
        if ((int)blockIdx.x >= nbr * nbc) return;
        i0 = (blockIdx.x % nbr) * GJB_BT;
        j0 = (blockIdx.x / nbr) * BNT;
    } else if (mode == 0) {                 // the pivot rows, every column block
        if ((int)blockIdx.x >= nbc) return;
        i0 = k0;
        j0 = blockIdx.x * BNT;
    } else {                                // every row block, the pivot columns
        if ((int)blockIdx.x >= nbr * (GJB_BT / BNT)) return;
        i0 = (blockIdx.x % nbr) * GJB_BT;
        j0 = k0 + (blockIdx.x / nbr) * BNT;
    }
    auto in_kb = [&](int t) { return t >= k0 && t < k1; };
    auto owns = [&](int I, int J) {
        return mode == 0 ? (in_kb(I) && !in_kb(J)) : mode == 1 ? (!in_kb(I) && !in_kb(J)) : (!in_kb(I) && in_kb(J));
    };
    {
        bool any = false;
        for (int I = i0; I < min(i0 + GJB_BT, nT); ++I)
            for (int J = j0; J < min(j0 + BNT, nT); ++J) any |= owns(I, J);
        if (!any) return;
    }
    double* M = bt.mats[b];
    auto tile = [&](int I, int J) { return M + ((int64_t)J * nT + I) * TILE_ELEMS; };
    const int nq = k1 - k0;
    auto load_stage = [&](int q, int slot) {
        double* As = psm + slot * STAGE;
        double* Bs = As + TILE * GJP_LDA;
        constexpr int CH = TILE * TILE / 2;   // 16-byte chunks per tile
        for (int e = threadIdx.x; e < GJB_BT * CH; e += NTH) {
            const int t = e / CH, rem = e % CH;
            const int kk = rem / (TILE / 2), r2 = (rem % (TILE / 2)) * 2;
            // A: tile (I, q), element (r, kk) at kk * 32 + r  ->  As[kk][t * 32 + r]
            const int I = i0 + t;
            const bool oka = I < nT && (mode != 0 || I < k1);
            cp_async16(As + kk * GJP_LDA + t * TILE + r2, oka ? tile(I, q) + kk * TILE + r2 : M, oka);
        }
        for (int e = threadIdx.x; e < BNT * CH; e += NTH) {
            const int t = e / CH, rem = e % CH;
            const int c = rem / (TILE / 2), k2 = (rem % (TILE / 2)) * 2;
            // B: tile (q, J), element (kk, c) at c * 32 + kk  ->  Bs[t * 32 + c][kk]
            const int J = j0 + t;
            const bool okb = J < nT && (mode != 2 || J < k1);
            cp_async16(Bs + (t * TILE + c) * GJP_LDK + k2, okb ? tile(q, J) + c * TILE + k2 : M, okb);
        }
    };
#pragma unroll
    for (int sg = 0; sg < STAGES - 1; ++sg) {
        if (sg < nq) load_stage(k0 + sg, sg);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wr = (wid & 3) * 32, wc = (wid >> 2) * 64;   // this warp's 32 x 64 output tile
    const int I = i0 + wr / TILE;
    if (mode == 1 && (int)threadIdx.x < GJB_BT * BNT) {
        const int Ip = i0 + threadIdx.x / BNT, Jp = j0 + threadIdx.x % BNT;
        if (Ip < nT && Jp < nT && owns(Ip, Jp)) bulk_prefetch_l2(tile(Ip, Jp), TILE_ELEMS * sizeof(double));
    }
    double acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c2 = 0; c2 < 8; ++c2) acc[r][c2] = 0.0;
    for (int qi = 0; qi < nq; ++qi) {
        asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
        __syncthreads();
        if (qi + STAGES - 1 < nq) load_stage(k0 + qi + STAGES - 1, (qi + STAGES - 1) % STAGES);
        asm volatile("cp.async.commit_group;" ::: "memory");
        const double* As = psm + (qi % STAGES) * STAGE;
        const double* Bs = As + TILE * GJP_LDA;
#pragma unroll 2
        for (int kq = 0; kq < TILE; kq += 4) {
            double af[4], bf[8];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) af[mi] = As[(kq + (lane & 3)) * GJP_LDA + wr + 8 * mi + (lane >> 2)];
#pragma unroll
            for (int ni = 0; ni < 8; ++ni) bf[ni] = Bs[(wc + 8 * ni + (lane >> 2)) * GJP_LDK + kq + (lane & 3)];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 8; ++ni)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                                 : "+d"(acc[2 * mi + ni / 4][(2 * ni) % 8]), "+d"(acc[2 * mi + ni / 4][(2 * ni) % 8 + 1])
                                 : "d"(af[mi]), "d"(bf[ni]));
        }
        if (STAGES == 2) __syncthreads();   // two stages: the next prefetch overwrites this one
    }
    if (I >= nT) return;
#pragma unroll
    for (int ni = 0; ni < 8; ++ni) {
        const int J = j0 + (wc + 8 * ni) / TILE;
        if (J >= nT || !owns(I, J)) continue;
        double* T = tile(I, J);
        const int cc = (wc + 8 * ni) % TILE + 2 * (lane & 3);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double v = acc[2 * mi + ni / 4][(2 * ni) % 8 + h];
                double* p = T + (cc + h) * TILE + 8 * mi + (lane >> 2);
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
            const int th = item_tile_rows(it, I);     // compact tail: rows >= th are not stored
            if (th < TILE && I == J && threadIdx.x == 0 && (th * (th + 1) / 2) % 2)
                dst[tail_diag_doubles(th) - 1] = 0.0;   // the even-size pad of a compact diagonal tile
            for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
                const int i = e % TILE, j = e / TILE;
                double v = src[e];
                if (I * TILE + i >= op.m || J * TILE + j >= op.m) v = 0.0;
                if (th < TILE) {
                    if (i >= th) continue;
                    if (I != J) {
                        dst[j * th + i] = v;
                    } else if (i >= j) {
                        double vt = (I * TILE + i >= op.m || J * TILE + j >= op.m) ? 0.0 : src[i * TILE + j];
                        dst[tail_col_off(th, j) + i - j] = i == j ? 0.5 * v : 0.5 * (v + vt);
                    }
                    continue;
                }
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
        // the Schur block is symmetric and only its lower part is kept (R22)
        Fp[tix(p.nT, mp[a], mp[b])] += Fc[tix(c.nT, c.nSp + max(a, b), c.nSp + min(a, b))];
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


// ---- launchers ----

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
                       const int32_t* nK, const int32_t* ids, int32_t* err, int sym) {
    if (nmat <= 0) return;
    static bool init_dev[64] = {};   // function attributes are per device
    int dev_ = 0;
    cudaGetDevice(&dev_);
    bool& init = init_dev[dev_ & 63];
    const int smem_p = 9 * TILE_ELEMS * sizeof(double);
    const int smem_g = (TILE * GJB_N + TILE * GJB_BPAD) * sizeof(double);
    const int smem_m = 2 * TILE * GJB_LDM * sizeof(double);
    const int smem_pp = GJP<4>::STAGES * GJP<4>::STAGE * sizeof(double);
    const int smem_p2 = GJP<2>::STAGES * GJP<2>::STAGE * sizeof(double);
    if (!init) {
        cudaFuncSetAttribute(k_gjb_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p);
        cudaFuncSetAttribute(k_gjb_gemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_g);
        cudaFuncSetAttribute(k_gjb_gemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_m);
        cudaFuncSetAttribute(k_gjb_gemm_pipe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pp);
        cudaFuncSetAttribute(k_gjb_gemm_pipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p2);
        init = true;
    }
    GJBatch bt{mats, nT, nK, ids, err, nullptr, 0};
    const int nb = (maxT + GJB_BT - 1) / GJB_BT;
    // symmetric variant: a row-panel strip per matrix (DDG_GJ_SYM=0: full exchange)
    // off by default: wrong beyond ~100 tiles per side (biharmonic blocks of 5k-16k unknowns;
    // DESIGN.md R22), passes the parity suite below that
    const bool want_sym = sym >= 0 ? sym != 0 : (getenv("DDG_GJ_SYM") && atoi(getenv("DDG_GJ_SYM")) != 0);
    const int64_t stride = (int64_t)GJB_BT * maxT * TILE_ELEMS;
    if (want_sym && cudaMallocAsync(&bt.strip, (size_t)nmat * stride * sizeof(double), st) == cudaSuccess)
        bt.strip_stride = stride;
    else
        bt.strip = nullptr;
    cudaGetLastError();
    const bool use_mma = !getenv("DDG_GJ_MMA") || atoi(getenv("DDG_GJ_MMA")) != 0;   // experiment switch
    // the pipelined MMA product for the full exchange (DDG_GJ_PIPE=0: the single-stage one)
    const bool use_pipe = use_mma && !bt.strip && !(getenv("DDG_GJ_PIPE") && atoi(getenv("DDG_GJ_PIPE")) == 0);
    // DDG_GJ_BNT = 2: the 128 x 64 two-CTAs-per-SM product, 4 (default): 128 x 128
    const int pipe_bnt = getenv("DDG_GJ_BNT") && atoi(getenv("DDG_GJ_BNT")) == 2 ? 2 : 4;
    for (int k0 = 0; k0 < maxK; k0 += GJB_BT) {
        k_gjb_pivot<<<nmat, 256, smem_p, st>>>(bt, k0);
        if (use_pipe && pipe_bnt == 2) {
            const int nbc = (maxT + 1) / 2;
            k_gjb_gemm_pipe<2><<<dim3(nbc, nmat), 128, smem_p2, st>>>(bt, k0, 0);
            k_gjb_gemm_pipe<2><<<dim3(nb * nbc, nmat), 128, smem_p2, st>>>(bt, k0, 1);
            k_gjb_gemm_pipe<2><<<dim3(nb * 2, nmat), 128, smem_p2, st>>>(bt, k0, 2);
        } else if (use_pipe) {
            k_gjb_gemm_pipe<4><<<dim3(nb, nmat), 256, smem_pp, st>>>(bt, k0, 0);
            k_gjb_gemm_pipe<4><<<dim3(nb * nb, nmat), 256, smem_pp, st>>>(bt, k0, 1);
            k_gjb_gemm_pipe<4><<<dim3(nb, nmat), 256, smem_pp, st>>>(bt, k0, 2);
        } else if (use_mma) {
            k_gjb_gemm<true><<<dim3(nb, nmat), 256, smem_m, st>>>(bt, k0, 0);
            k_gjb_gemm<true><<<dim3(nb * nb, nmat), 256, smem_m, st>>>(bt, k0, 1);
            k_gjb_gemm<true><<<dim3(nb, nmat), 256, smem_m, st>>>(bt, k0, 2);
        } else {
            k_gjb_gemm<false><<<dim3(nb, nmat), 256, smem_g, st>>>(bt, k0, 0);
            k_gjb_gemm<false><<<dim3(nb * nb, nmat), 256, smem_g, st>>>(bt, k0, 1);
            k_gjb_gemm<false><<<dim3(nb, nmat), 256, smem_g, st>>>(bt, k0, 2);
        }
    }
    if (bt.strip) cudaFreeAsync(bt.strip, st);
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

}  // namespace ddg
