// kernel_common.cuh — device helpers shared by libddg's sm_100a kernels
// (pcg.cu, symv.cu, coarse.cu, setup_kernels.cu).  Overview of the kernels:
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
// Setup: extract_local, Gauss-Jordan block inversion (tile / blocked), pack.
//
// Every reduction is deterministic (fixed partition, fixed order, last-block
// finalisation with a ticket; no floating-point atomics), so runs are bitwise
// repeatable.  Every PCG kernel exits immediately once the device flag
// `done` is set, so the host can enqueue several iterations without syncing.
#pragma once
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

// x loads of the row kernels: plain, or L2-only (CG: vectors other CTAs of a
// cluster wrote since this SM last read them; L1 is not coherent)
template <bool CG>
__device__ __forceinline__ double ldx(const double* p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
}

// (A x)[v] from the stencil, in the CSR's column order (see DevStencil)
template <bool CG = false>
__device__ __forceinline__ double stencil_dot(const DevStencil& st, int64_t v, const double* __restrict__ x) {
    const int nx = st.nx, ny = st.ny;
    // 32-bit index arithmetic (n < 2^31: int32 CSR offsets, checked at setup)
    const unsigned vv = (unsigned)v, r = vv / (unsigned)nx;
    const int ix = (int)(vv - r * (unsigned)nx);
    const unsigned r2 = r / (unsigned)ny;
    const int iy = (int)(r - r2 * (unsigned)ny), iz = (int)r2;
    double s = 0.0;
    if (st.kind == 1) {
        const double* xv = x + v;
        if constexpr (!CG) {
            // streaming kernels: enough warps in flight hide each load
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
        // k_pcg_small: every load is issued before the first product (a break
        // between them would make each multiply-add wait out an L2 latency in
        // turn); the products stay in column order, so the rounding is the CSR's
        double xk[STENCIL_MAX_PTS];
        if (ix >= st.rx && ix < nx - st.rx && iy >= st.ry && iy < ny - st.ry && iz >= st.rz && iz < st.nz - st.rz) {
#pragma unroll
            for (int k = 0; k < STENCIL_MAX_PTS; ++k)     // interior: every point on the grid
                xk[k] = k < st.npts ? ldx<CG>(xv + st.off[k]) : 0.0;
#pragma unroll
            for (int k = 0; k < STENCIL_MAX_PTS; ++k)
                if (k < st.npts) s = fma(st.c[k], xk[k], s);
            return s;
        }
        bool in[STENCIL_MAX_PTS];
#pragma unroll
        for (int k = 0; k < STENCIL_MAX_PTS; ++k) {
            const int a = ix + st.dx[k], b = iy + st.dy[k], c = iz + st.dz[k];
            in[k] = k < st.npts && a >= 0 && a < nx && b >= 0 && b < ny && c >= 0 && c < st.nz;
            xk[k] = in[k] ? ldx<CG>(xv + st.off[k]) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < STENCIL_MAX_PTS; ++k)
            if (in[k]) s = fma(st.c[k], xk[k], s);
        return s;
    }
    if (st.kind == 3) {
        // node27: row v = dof * node + d; the node's class (first / interior / last per
        // axis) selects its table rows; neighbours in ascending node order, then e --
        // the CSR's column order, so the multiply-adds round as the CSR row does
        const int dof = st.dof;
        const unsigned node = vv / (unsigned)dof, d = vv - node * (unsigned)dof;
        const unsigned q = node / (unsigned)nx;
        const int jx = (int)(node - q * (unsigned)nx);
        const unsigned q2 = q / (unsigned)ny;
        const int jy = (int)(q - q2 * (unsigned)ny), jz = (int)q2;
        const int cls = (jx == 0 ? 0 : jx == nx - 1 ? 2 : 1) + 3 * (jy == 0 ? 0 : jy == ny - 1 ? 2 : 1) +
                        9 * (jz == 0 ? 0 : jz == st.nz - 1 ? 2 : 1);
        const double* T = st.coef + ((size_t)cls * 27 * dof + d) * dof;   // [offset][d][e], offset-major
        for (int dz = -1; dz <= 1; ++dz) {
            if (jz + dz < 0 || jz + dz >= st.nz) continue;
            for (int dy = -1; dy <= 1; ++dy) {
                if (jy + dy < 0 || jy + dy >= ny) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    if (jx + dx < 0 || jx + dx >= nx) continue;
                    const int o = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
                    const int64_t nb = (int64_t)node + dx + (int64_t)nx * (dy + (int64_t)ny * dz);
                    const double* Te = T + (size_t)o * dof * dof;
                    for (int e = 0; e < dof; ++e) s = fma(__ldg(Te + e), ldx<CG>(x + nb * dof + e), s);
                }
            }
        }
        return s;
    }
    const int64_t n = (int64_t)nx * ny * st.nz, sy = nx, sz = (int64_t)nx * ny;
    const double* D = st.coef;
    const double* CX = D + n;
    const double* CY = CX + n;
    const double* CZ = CY + n;
    if (iz > 0) s = fma(CZ[v - sz], ldx<CG>(&x[v - sz]), s);
    if (iy > 0) s = fma(CY[v - sy], ldx<CG>(&x[v - sy]), s);
    if (ix > 0) s = fma(CX[v - 1], ldx<CG>(&x[v - 1]), s);
    s = fma(D[v], ldx<CG>(x + v), s);
    if (ix + 1 < nx) s = fma(CX[v], ldx<CG>(&x[v + 1]), s);
    if (iy + 1 < ny) s = fma(CY[v], ldx<CG>(&x[v + sy]), s);
    if (iz + 1 < st.nz) s = fma(CZ[v], ldx<CG>(&x[v + sz]), s);
    return s;
}

// lane sl of SW: its entries e = rp[v] + sl, + SW, ... in order (node-blocked columns)
template <int BS, int SW, bool CG = false>
__device__ __forceinline__ double row_dot_nb(const DevCSR& A, int64_t v, const double* __restrict__ x, int sl) {
    const int e0 = A.rp[v], e1 = A.rp[v + 1];
    const int32_t* bc = A.bcol + A.brp[v / BS];
    double s = 0.0;
    for (int e = e0 + sl; e < e1; e += SW) {
        const int j = e - e0;
        s += A.val[e] * ldx<CG>(x + bc[j / BS] * BS + j % BS);
    }
    return s;
}

// (A x)[v] by one thread: stencil or CSR row
template <bool CG = false>
__device__ __forceinline__ double row_dot1(const DevCSR& A, int64_t v, const double* __restrict__ x) {
    if (A.st.kind) return stencil_dot<CG>(A.st, v, x);
    if (A.bs == 3) return row_dot_nb<3, 1, CG>(A, v, x, 0);
    if (A.bs == 4) return row_dot_nb<4, 1, CG>(A, v, x, 0);
    double s = 0.0;
    for (int e = A.rp[v]; e < A.rp[v + 1]; e++) s += A.val[e] * ldx<CG>(x + A.col[e]);
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
        if (A.bs == 3) {
            s = row_dot_nb<3, SW>(A, v, x, sl);
        } else if (A.bs == 4) {
            s = row_dot_nb<4, SW>(A, v, x, sl);
        } else {
            const int e1 = A.rp[v + 1];
            for (int e = A.rp[v] + sl; e < e1; e += SW) s += A.val[e] * x[A.col[e]];
        }
    }
#pragma unroll
    for (int o = SW / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    return s;
}

// block-wide sum; result valid in every thread. blockDim.x multiple of 32, <= 1024
static __device__ double block_sum(double v) {
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

// offset (doubles) of local tile l = (I, J) inside its item (compact last
// row when it.tail != 0, ddg_internal.h)
__device__ __forceinline__ int64_t item_tile_off(const ItemDesc& it, int l, int I) {
    if (!it.tri) return (int64_t)l * TILE_ELEMS;
    const int rr = I - it.I0;                  // diagonal tiles of rows 0..rr-1 precede l
    if (it.tail && I == it.I1 - 1)
        return (int64_t)(rr * (rr + 1) / 2 - rr) * TILE_ELEMS + (int64_t)rr * DIAG_ELEMS +
               (int64_t)(l - rr * (rr + 1) / 2) * it.tail * TILE;
    return (int64_t)(l - rr) * TILE_ELEMS + (int64_t)rr * DIAG_ELEMS;
}
// doubles stored for tile (I, J) of an item (packed diagonal, compact tail)
__device__ __forceinline__ int item_tile_doubles(const ItemDesc& it, int I, int J) {
    const bool t = it.tail && I == it.I1 - 1;
    return I == J && it.tri ? (t ? tail_diag_doubles(it.tail) : DIAG_ELEMS) : (t ? it.tail * TILE : TILE_ELEMS);
}
// valid rows stored for tile row I of an item: 32, or the compact tail
__device__ __forceinline__ int item_tile_rows(const ItemDesc& it, int I) {
    return (it.tail && I == it.I1 - 1) ? it.tail : TILE;
}

// lane i loads row i of tile (I, J) (packed form when I == J); th < 32: a
// compact tail tile (rows >= th are zero)
__device__ __forceinline__ void load_tile_row(double* a, const double* T, bool diag, int lane, int th = TILE) {
    if (th == TILE) {
        if (!diag) {
#pragma unroll
            for (int j = 0; j < TILE; ++j) a[j] = __ldcs(T + j * TILE + lane);
        } else {
#pragma unroll
            for (int j = 0; j < TILE; ++j) a[j] = lane >= j ? __ldcs(T + diag_col_off(j) + lane - j) : 0.0;
        }
        return;
    }
    if (!diag) {
#pragma unroll
        for (int j = 0; j < TILE; ++j) a[j] = lane < th ? __ldcs(T + j * th + lane) : 0.0;
    } else {
#pragma unroll
        for (int j = 0; j < TILE; ++j)
            a[j] = (lane >= j && lane < th) ? __ldcs(T + tail_col_off(th, j) + lane - j) : 0.0;
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
// bulk prefetch of [src, src + bytes) into L2 (no shared memory, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Programmatic dependent launch along the colour-step chain (gather -> ring
// -> reduce -> gather ...): the next kernel is launched while the previous
// one drains, and waits in pdl_wait() for it to complete before reading.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
extern int g_pdl;   // 1: chain launches carry the programmatic-serialization attribute (DDG_PDL)
// streams shared by several host threads (the loopback group's stream): launched
// without the attribute (comm.cpp registers them)
bool no_pdl_stream(cudaStream_t st);
template <typename... KArgs, typename... Args>
static inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl && !no_pdl_stream(st);
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, args...);
}

// Raise a kernel's dynamic shared-memory limit to the device maximum once per
// device.  Setting it to each launch's own size races when several host
// threads launch the same kernel with different sizes (the loopback ranks):
// one thread's smaller value lands between another's set and launch, and that
// launch fails with an invalid argument.  A single maximal value cannot race.
#define DDG_MAX_DYN_SMEM(kern)                                                                        \
    do {                                                                                              \
        static bool done_[64] = {};                                                                   \
        int d_ = 0;                                                                                   \
        cudaGetDevice(&d_);                                                                           \
        if (!done_[d_ & 63]) {                                                                        \
            cudaFuncAttributes fa_{};                                                                 \
            cudaFuncGetAttributes(&fa_, (const void*)(kern));                                         \
            int optin_ = 0;                                                                           \
            cudaDeviceGetAttribute(&optin_, cudaDevAttrMaxSharedMemoryPerBlockOptin, d_);             \
            cudaFuncSetAttribute((const void*)(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                 optin_ - (int)fa_.sharedSizeBytes);                                  \
            done_[d_ & 63] = true;                                                                    \
        }                                                                                             \
    } while (0)

static inline int vec_grid(int64_t n) {
    int64_t g = (n + VEC_THREADS - 1) / VEC_THREADS;
    return (int)(g < RED_BLOCKS ? (g > 0 ? g : 1) : RED_BLOCKS);
}

}  // namespace ddg
