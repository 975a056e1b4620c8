// chol.cu — local_variant = DDG_LOCAL_CHOLESKY: the exact local solves as the
// north star words them, "a batched triangular solve against per-subdomain
// Cholesky factors".  PAPER.md:550-551 ("we solve these subdomain problems
// exactly"): A_i = L_i L_i^T once at setup, then every visit of subdomain i
// in a colour step solves L_i L_i^T delta = s_i by a forward and a back
// substitution over 32 x 32 tiles.
//
// Factor storage (one factor after another in ddg_ctx::d_tiles at the local
// op's tile_off): tile rows I = 0 .. nT-1 at chol_row_off(I) (ddg_internal.h),
// each row the I full tiles L_IJ (J < I, tile (I, J) at + J * 1024, column-major
// like the SYMV tiles: element (i, j) at j * 32 + i) and then D_I = L_II^{-1}
// as a packed lower triangle (element (i, j), i >= j, at diag_col_off(j) + i - j;
// 4224 B instead of 8 KB, so a 5-tile-row factor (C3) fits twice per SM when
// staged).  Both substitutions are dot products within a warp:
//     forward  y_I = L_II^{-1} (s_I - sum_{J<I} L_IJ y_J)
//     back     x_J = L_JJ^{-T} (y_J - sum_{I>J} L_IJ^T x_I)
// (the inverted 32 x 32 diagonal blocks remove the scalar recurrence inside a
// tile; the tile-row recurrence is the triangular solve itself).
#include "kernel_common.cuh"

namespace ddg {

// element (R, C) of the tiled dense mp x mp setup scratch (tile (I,J) at (J*nT+I)*1024)
__device__ __forceinline__ double* stile(double* M, int nT, int I, int J) {
    return M + ((int64_t)J * nT + I) * TILE_ELEMS;
}
constexpr int CP = TILE + 1;   // padded shared-memory tile column (conflict-free row and column walks)

// ---- setup: right-looking tile Cholesky, one CTA (256 threads) per matrix ----
// On exit the lower tiles of the scratch hold L_IJ (I > J) and T_I (I = J).
__global__ void __launch_bounds__(256) k_chol_local(const int32_t* __restrict__ nTs, double* const* __restrict__ mats,
                                                    const int32_t* __restrict__ ids, int32_t* err) {
    __shared__ double Ls[TILE * CP];   // the pivot tile: L_kk, then the panel operand
    __shared__ double Ds[TILE * CP];   // D = L_kk^{-1}
    __shared__ double Bs[TILE * CP];   // second operand of the trailing update
    __shared__ int bad;
    const int nT = nTs[blockIdx.x];
    double* M = mats[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) bad = 0;
    for (int k = 0; k < nT; ++k) {
        // 1. L_kk = chol(A_kk) (lower triangle read), warp 0, scalar right-looking
        const double* Akk = stile(M, nT, k, k);
        for (int e = tid; e < TILE_ELEMS; e += 256) Ls[(e / TILE) * CP + e % TILE] = Akk[e];
        __syncthreads();
        if (warp == 0) {
            for (int p = 0; p < TILE; ++p) {
                const double d = Ls[p * CP + p];
                if (!(d > 0.0)) {
                    if (lane == 0) {
                        bad = 1;
                        if (atomicCAS(&err[0], -1, ids[blockIdx.x]) == -1) err[1] = k * TILE + p;
                    }
                    break;
                }
                const double piv = sqrt(d);
                const double li = lane > p ? Ls[p * CP + lane] / piv : 0.0;
                __syncwarp();
                if (lane == p) Ls[p * CP + p] = piv;
                if (lane > p) Ls[p * CP + lane] = li;
                // trailing 32x32 update: row `lane` of columns p+1 .. lane
                for (int j = p + 1; j < TILE; ++j) {
                    const double lj = __shfl_sync(FULL, li, j);
                    if (lane >= j) Ls[j * CP + lane] -= li * lj;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (bad) return;
        // 2. D = L_kk^{-1}: thread c < 32 solves L d_c = e_c (column c, rows c..31)
        if (tid < TILE) {
            const int cc = tid;
            for (int i = 0; i < TILE; ++i) {
                double v;
                if (i < cc) {
                    v = 0.0;
                } else {
                    double acc = (i == cc) ? 1.0 : 0.0;
                    for (int t = cc; t < i; ++t) acc -= Ls[t * CP + i] * Ds[cc * CP + t];
                    v = acc / Ls[i * CP + i];
                }
                Ds[cc * CP + i] = v;
            }
        }
        __syncthreads();
        // T_k: lower = D, strict upper = D^T
        {
            double* Tk = stile(M, nT, k, k);
            for (int e = tid; e < TILE_ELEMS; e += 256) {
                const int i = e % TILE, j = e / TILE;
                Tk[e] = i >= j ? Ds[j * CP + i] : Ds[i * CP + j];
            }
        }
        // 3. panel: L_Ik = A_Ik L_kk^{-T} = A_Ik D^T,  L(i,j) = sum_{t<=j} A(i,t) D(j,t)
        for (int I = k + 1; I < nT; ++I) {
            double* AIk = stile(M, nT, I, k);
            __syncthreads();
            for (int e = tid; e < TILE_ELEMS; e += 256) Bs[(e / TILE) * CP + e % TILE] = AIk[e];
            __syncthreads();
            for (int e = tid; e < TILE_ELEMS; e += 256) {
                const int i = e % TILE, j = e / TILE;
                double acc = 0.0;
                for (int t = 0; t <= j; ++t) acc += Bs[t * CP + i] * Ds[t * CP + j];
                AIk[e] = acc;
            }
        }
        __syncthreads();
        // 4. trailing update: A_IJ -= L_Ik L_Jk^T for k < J <= I (lower tiles only)
        for (int J = k + 1; J < nT; ++J) {
            const double* LJk = stile(M, nT, J, k);
            __syncthreads();
            for (int e = tid; e < TILE_ELEMS; e += 256) Bs[(e / TILE) * CP + e % TILE] = LJk[e];
            for (int I = J; I < nT; ++I) {
                const double* LIk = stile(M, nT, I, k);
                double* AIJ = stile(M, nT, I, J);
                __syncthreads();
                for (int e = tid; e < TILE_ELEMS; e += 256) Ls[(e / TILE) * CP + e % TILE] = LIk[e];
                __syncthreads();
                // thread: rows i0, i0+16 x columns j0, j0+16 (2 x 2 register block)
                const int i0 = tid % 16, j0 = tid / 16;
                double a00 = 0, a01 = 0, a10 = 0, a11 = 0;
#pragma unroll 8
                for (int t = 0; t < TILE; ++t) {
                    const double x0 = Ls[t * CP + i0], x1 = Ls[t * CP + i0 + 16];
                    const double y0 = Bs[t * CP + j0], y1 = Bs[t * CP + j0 + 16];
                    a00 += x0 * y0;
                    a01 += x0 * y1;
                    a10 += x1 * y0;
                    a11 += x1 * y1;
                }
                AIJ[j0 * TILE + i0] -= a00;
                AIJ[(j0 + 16) * TILE + i0] -= a01;
                AIJ[j0 * TILE + i0 + 16] -= a10;
                AIJ[(j0 + 16) * TILE + i0 + 16] -= a11;
            }
        }
        __syncthreads();
    }
}

// copy the lower tiles of the factored scratch into the factor storage
// (padding rows / columns >= m zeroed: s is zero there, so y and x stay zero)
__global__ void k_chol_pack(const int32_t* __restrict__ op_ids, const OpDesc* __restrict__ ops,
                            const double* __restrict__ scratch, const int64_t* __restrict__ scratch_off,
                            double* __restrict__ out) {
    const OpDesc op = ops[op_ids[blockIdx.y]];
    const double* M = scratch + scratch_off[blockIdx.y];
    const int ntl = op.nT * (op.nT + 1) / 2;
    for (int t = blockIdx.x; t < ntl; t += gridDim.x) {
        int I = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
        while (I * (I + 1) / 2 > t) --I;
        while ((I + 1) * (I + 2) / 2 <= t) ++I;
        const int J = t - I * (I + 1) / 2;
        const double* src = M + ((int64_t)J * op.nT + I) * TILE_ELEMS;
        double* dst = out + op.tile_off + chol_row_off(I) + (int64_t)J * TILE_ELEMS;
        if (J < I) {
            for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
                const int i = e % TILE, j = e / TILE;
                const bool ok = I * TILE + i < op.m && J * TILE + j < op.m;
                dst[e] = ok ? src[e] : 0.0;
            }
        } else {                       // D_I packed lower (the lower part of T_I)
            for (int e = threadIdx.x; e < TILE_ELEMS; e += blockDim.x) {
                const int i = e % TILE, j = e / TILE;
                if (i < j) continue;
                const bool ok = I * TILE + i < op.m;
                dst[diag_col_off(j) + i - j] = ok ? src[e] : 0.0;
            }
        }
    }
}

// ---- hot path: one colour's local solves, one CTA (8 warps) per subdomain ----
// s_i = R~_i (r - A z) is in s[op.s_off ..] (k_gather_flat); z[Omega~_i] += x.
// STAGED (factors of at most CHOL_STAGE_T tile rows, C1 and C3): the whole
// factor is bulk-copied into shared memory, one copy and one mbarrier per tile
// row, issued at kernel start; the forward pass consumes the rows as they land
// and the back pass re-reads them on chip, so the factor crosses HBM once.
// Otherwise the tiles are read from global memory by both passes (the back
// pass mostly from L2).
constexpr int CHOL_WARPS = 8;
constexpr int CHOL_STAGE_T = 6;    // 15 full tiles + 6 packed diagonals = 148 KB (C3, 5 rows: 103 KB, two CTAs per SM)
template <bool STAGED>
__device__ __forceinline__ double ldt(const double* p) {
    if constexpr (STAGED) return *p;
    else return __ldg(p);
}
template <bool STAGED>
__global__ void __launch_bounds__(CHOL_WARPS * 32)
k_chol_solve(const OpDesc* __restrict__ ops, int op_begin, const double* __restrict__ fac,
             const double* __restrict__ s, const int32_t* __restrict__ oidx, double* __restrict__ z,
             const int32_t* done) {
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar[CHOL_STAGE_T];
    pdl_wait();
    if (*done) return;
    const OpDesc op = ops[op_begin + blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* tiles = sm;                                  // STAGED: the whole factor
    double* y = sm + (STAGED ? chol_doubles(op.nT) : 0); // mp: s, then y, then x (in place)
    double* part = y + op.mp;                            // CHOL_WARPS x 32 partial rows
    double* dsm = part + CHOL_WARPS * TILE;              // !STAGED: a packed diagonal block, for the
                                                         // back pass's column walk (coalesced load)
    const double* L = STAGED ? tiles : fac + op.tile_off;
    if constexpr (STAGED) {
        if (threadIdx.x == 0) {
            for (int I = 0; I < op.nT; ++I) mbar_init(&bar[I], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int I = 0; I < op.nT; ++I) {
                const unsigned bytes = (unsigned)(chol_row_off(I + 1) - chol_row_off(I)) * 8;
                mbar_expect_tx(&bar[I], bytes);
                bulk_g2s(tiles + chol_row_off(I), fac + op.tile_off + chol_row_off(I), bytes, &bar[I]);
            }
        }
    }
    for (int r = threadIdx.x; r < op.mp; r += blockDim.x) y[r] = s[op.s_off + r];
    __syncthreads();
    // forward: L y = s
    for (int I = 0; I < op.nT; ++I) {
        if constexpr (STAGED) mbar_wait(&bar[I], 0);
        const double* row = L + chol_row_off(I);
        double acc = 0.0;
        for (int J = warp; J < I; J += CHOL_WARPS) {
            const double* T = row + (int64_t)J * TILE_ELEMS;
            const double* yj = y + J * TILE;
#pragma unroll
            for (int j = 0; j < TILE; ++j) acc += ldt<STAGED>(T + j * TILE + lane) * yj[j];
        }
        part[warp * TILE + lane] = acc;
        __syncthreads();
        if (warp == 0) {
            double t = y[I * TILE + lane];
            for (int w = 0; w < CHOL_WARPS; ++w) t -= part[w * TILE + lane];
            const double* D = row + (int64_t)I * TILE_ELEMS;     // packed lower D_I
            double yi = 0.0;
#pragma unroll
            for (int j = 0; j < TILE; ++j) {
                const double tj = __shfl_sync(FULL, t, j);
                if (j <= lane) yi += ldt<STAGED>(D + diag_col_off(j) + lane - j) * tj;
            }
            y[I * TILE + lane] = yi;
        }
        __syncthreads();
    }
    // back: L^T x = y
    for (int J = op.nT - 1; J >= 0; --J) {
        double v[TILE];
#pragma unroll
        for (int j = 0; j < TILE; ++j) v[j] = 0.0;
        for (int I = J + 1 + warp; I < op.nT; I += CHOL_WARPS) {
            const double* T = L + chol_row_off(I) + (int64_t)J * TILE_ELEMS;
            const double xi = y[I * TILE + lane];
#pragma unroll
            for (int j = 0; j < TILE; ++j) v[j] += ldt<STAGED>(T + j * TILE + lane) * xi;
        }
        rs_stage<16>(v, lane);
        rs_stage<8>(v, lane);
        rs_stage<4>(v, lane);
        rs_stage<2>(v, lane);
        rs_stage<1>(v, lane);
        part[warp * TILE + lane] = v[0];
        __syncthreads();
        if (warp == 0) {
            double t = y[J * TILE + lane];
            for (int w = 0; w < CHOL_WARPS; ++w) t -= part[w * TILE + lane];
            const double* D = L + chol_row_off(J) + (int64_t)J * TILE_ELEMS;   // packed lower D_J
            if constexpr (!STAGED) {      // lane j reads column j of D_J: stage it in shared memory
                for (int k = lane; k < DIAG_ELEMS; k += TILE) dsm[k] = __ldg(D + k);
                __syncwarp();
                D = dsm;
            }
            double xj = 0.0;
#pragma unroll
            for (int j = 0; j < TILE; ++j) {
                const double tj = __shfl_sync(FULL, t, j);
                if (j >= lane) xj += D[diag_col_off(lane) + j - lane] * tj;   // D_J(j, lane), shared memory
            }
            y[J * TILE + lane] = xj;
        }
        __syncthreads();
    }
    const int32_t* idx = oidx + op.idx_off;
    for (int r = threadIdx.x; r < op.m; r += blockDim.x) z[idx[r]] += y[r];
}

void launch_chol_local(cudaStream_t st, int nmat, const int32_t* nT, double* const* mats, const int32_t* ids,
                       int32_t* err) {
    if (nmat > 0) k_chol_local<<<nmat, 256, 0, st>>>(nT, mats, ids, err);
}
void launch_chol_pack(cudaStream_t st, int nops, int max_tiles, const int32_t* op_ids, const OpDesc* ops,
                      const double* scratch, const int64_t* scratch_off, double* out) {
    if (nops > 0) k_chol_pack<<<dim3(std::min(max_tiles, 64), nops), 256, 0, st>>>(op_ids, ops, scratch, scratch_off, out);
}
void launch_chol_solve(cudaStream_t st, const OpDesc* ops, int op_begin, int nops, int max_mp, const double* fac,
                       const double* s, const int32_t* oidx, double* z, const int32_t* done) {
    if (nops <= 0) return;
    const int maxT = max_mp / TILE;
    const bool staged = maxT <= CHOL_STAGE_T && !getenv("DDG_CHOL_GLOBAL");
    const size_t smem = (size_t)(max_mp + CHOL_WARPS * TILE) * sizeof(double) +
                        (staged ? (size_t)chol_doubles(maxT) : (size_t)DIAG_ELEMS) * sizeof(double);
    if (smem > 48 * 1024) {
        if (staged) DDG_MAX_DYN_SMEM(k_chol_solve<true>);
        else DDG_MAX_DYN_SMEM(k_chol_solve<false>);
    }
    if (staged) launch_pdl(k_chol_solve<true>, nops, CHOL_WARPS * 32, smem, st, ops, op_begin, fac, s, oidx, z, done);
    else launch_pdl(k_chol_solve<false>, nops, CHOL_WARPS * 32, smem, st, ops, op_begin, fac, s, oidx, z, done);
}

}  // namespace ddg
