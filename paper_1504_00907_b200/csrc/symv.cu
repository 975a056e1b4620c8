// symv.cu — colour-sweep kernels (a4, a8): flat residual gather, per-item SYMV, the persistent bulk-copy-ring SYMVs, partial reduction
// (part of libddg's sm_100a kernels; shared device helpers in kernel_common.cuh)
#include <cstring>

#include <atomic>
#include <mutex>

#include "kernel_common.cuh"

namespace ddg {
int g_pdl = 1;
static std::mutex g_nopdl_mu;
static std::vector<cudaStream_t> g_nopdl;   // live loopback streams (registered / released by comm.cpp)
static std::atomic<int> g_nopdl_n{0};
bool no_pdl_stream(cudaStream_t st) {
    if (g_nopdl_n.load(std::memory_order_acquire) == 0) return false;   // no loopback group alive
    std::lock_guard<std::mutex> lk(g_nopdl_mu);
    for (cudaStream_t x : g_nopdl)
        if (x == st) return true;
    return false;
}
void register_no_pdl_stream(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_nopdl_mu);
    g_nopdl.push_back(st);
    g_nopdl_n.store((int)g_nopdl.size(), std::memory_order_release);
}
void release_no_pdl_stream(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_nopdl_mu);
    for (size_t i = 0; i < g_nopdl.size(); ++i)
        if (g_nopdl[i] == st) {
            g_nopdl[i] = g_nopdl.back();
            g_nopdl.pop_back();
            g_nopdl_n.store((int)g_nopdl.size(), std::memory_order_release);
            return;
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
    pdl_wait();
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
        load_tile_row(a, tbase + item_tile_off(it, w, I0_), I0_ == J0_, lane, item_tile_rows(it, I0_));
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
        if (l != w) load_tile_row(a, tbase + item_tile_off(it, l, I), I == J, lane, item_tile_rows(it, I));
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
    load_tile_row(a, tb + item_tile_off(it, 0, I), I == J, lane, item_tile_rows(it, I));   // first tile in flight
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
            load_tile_row(b, tb + item_tile_off(it, l + 1, I1), I1 == J1, lane, item_tile_rows(it, I1));
        }
        tile_apply(a, a, sw, yw, I * TILE, J * TILE, I == J, lane);
        if (l + 2 < it.ntiles) {
            item_tile(it, l + 2, I, J);
            load_tile_row(a, tb + item_tile_off(it, l + 2, I), I == J, lane, item_tile_rows(it, I));
        }
        if (has1) tile_apply(b, b, sw, yw, I1 * TILE, J1 * TILE, I1 == J1, lane);
    }
    for (int x = lane; x < op.m; x += 32) {
        if (op.out_mode == 0) z[idx[x]] += yw[x];
        else y_out[x] = yw[x];
    }
}

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
    pdl_wait();
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

// ---- tile products of whole-operator triangles (k_symv_whole, k_symv_ring2) --
// th = 32: a full tile (diagonal tiles packed, kernel_common.cuh); th < 32: a
// compact last-row tile (ddg_internal.h).
// direct part of tile (r, c): lane = row i, sum_j T(i, j) s_c[j]
__device__ __forceinline__ double tile_direct(const double* __restrict__ T, const double* __restrict__ ss, int r,
                                              int c, int th, int lane) {
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    if (th == TILE) {
        if (r != c) {
            const double2* sJ = reinterpret_cast<const double2*>(ss + c * TILE);
#pragma unroll
            for (int j = 0; j < TILE; j += 4) {
                const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                d0 = fma(T[j * TILE + lane], u.x, d0);
                d1 = fma(T[(j + 1) * TILE + lane], u.y, d1);
                d2 = fma(T[(j + 2) * TILE + lane], v.x, d2);
                d3 = fma(T[(j + 3) * TILE + lane], v.y, d3);
            }
        } else {
            const double2* sJ = reinterpret_cast<const double2*>(ss + r * TILE);
#pragma unroll
            for (int j = 0; j < TILE; j += 4) {
                const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                if (lane >= j) d0 = fma(T[diag_col_off(j) + lane - j], u.x, d0);
                if (lane >= j + 1) d1 = fma(T[diag_col_off(j + 1) + lane - j - 1], u.y, d1);
                if (lane >= j + 2) d2 = fma(T[diag_col_off(j + 2) + lane - j - 2], v.x, d2);
                if (lane >= j + 3) d3 = fma(T[diag_col_off(j + 3) + lane - j - 3], v.y, d3);
            }
        }
    } else if (lane < th) {                                // compact tail row
        if (r != c) {
            const double* sJ = ss + c * TILE;
#pragma unroll 8
            for (int j = 0; j < TILE; j += 2) {
                d0 = fma(T[j * th + lane], sJ[j], d0);
                d1 = fma(T[(j + 1) * th + lane], sJ[j + 1], d1);
            }
        } else {
            const double* sJ = ss + r * TILE;
            for (int j = 0; j <= lane; ++j) d0 = fma(T[tail_col_off(th, j) + lane - j], sJ[j], d0);
        }
    }
    return (d0 + d1) + (d2 + d3);
}

// transposed part of tile (r, c): lane = column j, sum_i T(i, j) s_r[i]
__device__ __forceinline__ double tile_trans(const double* __restrict__ T, const double* __restrict__ ss, int r,
                                             int c, int th, int lane) {
    const double* sI = ss + r * TILE;
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    if (th == TILE) {
        if (r != c) {
            // 16-byte pairs along the rotated diagonal: lanes 8p..8p+7 of a
            // quarter-warp phase hit 8 distinct 16-byte bank groups
            const double2* Tc = reinterpret_cast<const double2*>(T + lane * TILE);
            const double2* s2 = reinterpret_cast<const double2*>(sI);
#pragma unroll
            for (int t = 0; t < TILE / 2; t += 2) {
                const int ua = (t + lane) & 15, ub = (t + 1 + lane) & 15;
                const double2 a = Tc[ua], sa = s2[ua], b = Tc[ub], sb = s2[ub];
                d0 = fma(a.x, sa.x, d0);
                d1 = fma(a.y, sa.y, d1);
                d2 = fma(b.x, sb.x, d2);
                d3 = fma(b.y, sb.y, d3);
            }
        } else {
            const double* Tc = T + diag_col_off(lane) - lane;   // (i, lane) at Tc[i], i >= lane
#pragma unroll
            for (int t = 0; t < TILE; t += 2) {
                const int ia = (t + lane) & 31, ib = (t + 1 + lane) & 31;
                if (ia >= lane) d0 = fma(Tc[ia], sI[ia], d0);
                if (ib >= lane) d1 = fma(Tc[ib], sI[ib], d1);
            }
        }
    } else if (r != c) {                                   // compact tail tile: rows i < th
        const double* Tc = T + lane * th;
        for (int i = 0; i < th; ++i) d0 = fma(Tc[i], sI[i], d0);
    } else if (lane < th) {
        const double* Tc = T + tail_col_off(th, lane) - lane;
        for (int i = lane; i < th; ++i) d0 = fma(Tc[i], sI[i], d0);
    }
    return (d0 + d1) + (d2 + d3);
}

// ---- k_symv_ring2: row warps + column warps ----------------------------------
// Same producer, ring, item buffers and epilogue as k_symv_ring; the 16
// consumer warps split each tile's two products by role:
//  * row warps (0-7): own tile rows r; lane i accumulates the direct part
//    y_I[i] += sum_j S_IJ[i][j] s_J[j] in one register across the row's
//    tiles, then writes its partial row once.  split = 2 (default): warps 2p
//    and 2p + 1 share rows r = (p + item counter) mod 4 (+4, +8, +12), one
//    taking columns j < 16 of every tile, the other j >= 16 (partials pr, pr2),
//    so a row streamed as consecutive chunks is consumed by two warps at once;
//    split = 1: one warp per row (owner (r + item counter) mod 8);
//  * column warps (8-15): own tile columns c; lane j accumulates the
//    transposed part y_J[j] += sum_i S_IJ[i][j] s_I[i] walking the tile along a
//    rotated diagonal (i = (t + j) mod 32: two wavefronts per load, no bank
//    conflicts) with s_I rotated by shuffles; one register per owned column,
//    written to pc[column] at the end of the item.
// Every row half and column has a single owner, so the item's result is
// y = (pr + pr2) + pc (triangles) or pr + pr2 | pc (rectangles: row block |
// column block) -- three partial arrays instead of eight, no butterfly.
constexpr int R2_ROWW = 8, R2_COLW = 8, R2_CONS = R2_ROWW + R2_COLW;
constexpr int RING2_THREADS = (R2_CONS + 1 + RING_EPI_WARPS) * 32;
__host__ __device__ constexpr size_t ring2_smem(int RT, int nst, int nb, int maxr) {
    return (size_t)nst * RT * TILE_ELEMS * 8 + (size_t)nb * 4 * maxr * 8 + (size_t)nb * 8 * 4 +
           (2 * (size_t)nst + 4 * (size_t)nb) * 8 + (size_t)RING_EPI_WARPS * maxr * 8;
}

template <int RT>
__global__ void __launch_bounds__(RING2_THREADS, 1)
k_symv_ring2(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin,
             const int32_t* __restrict__ cta_part, const double* __restrict__ tiles, const double* __restrict__ s,
             const int32_t* __restrict__ oidx, double* __restrict__ z, double* __restrict__ y_out,
             double* __restrict__ partials, const int32_t* done, int nst, int nb, int maxr, int pf, int split_) {
    pdl_wait();
    constexpr int SLOT = RT * TILE_ELEMS;
    const bool copy_only = split_ & 0x100;                       // DDG_RING2_COPYONLY: bandwidth probe (debug)
    const bool merge = split_ & 0x200;                           // DDG_RING2_MERGE=1: one copy per contiguous run (measured no gain)
    // DDG_RING2_BARE_EPI (probes): 1 the epilogue only hands buffers back; 2 it skips the tail strip only
    const bool bare_epi = split_ & 0x400, no_strip = split_ & 0xC00;
    const int split = split_ & 0xff;
    if (*done) return;
    extern __shared__ __align__(128) double rsm[];
    double* ring = rsm;                                          // [nst][SLOT]
    double* s_sm = ring + (size_t)nst * SLOT;                    // [nb][maxr]
    double* pr_sm = s_sm + (size_t)nb * maxr;                    // [nb][maxr]  row (direct) parts
    double* pc_sm = pr_sm + (size_t)nb * maxr;                   // [nb][maxr]  column (transposed) parts
    double* pr2_sm = pc_sm + (size_t)nb * maxr;                  // [nb][maxr]  second row half (split = 2)
    int32_t* dsc = reinterpret_cast<int32_t*>(pr2_sm + (size_t)nb * maxr);  // [nb][8]
    uint64_t* full = reinterpret_cast<uint64_t*>(dsc + nb * 8);
    uint64_t* empty = full + nst;
    uint64_t* sfull = empty + nst;
    uint64_t* sempty = sfull + nb;
    uint64_t* pdone = sempty + nb;
    uint64_t* pfree = pdone + nb;
    double* yt_sm = reinterpret_cast<double*>(pfree + nb);      // [RING_EPI_WARPS][maxr] strip transposed parts
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
            if (pf > 0 && lane == 0 && ii + pf < i1) {           // L2 prefetch pf items ahead
                const ItemDesc ip = items[ii + pf];
                bulk_prefetch_l2(tiles + ip.tile_off,
                                 (unsigned)(item_doubles(ip.tri, ip.I1 - ip.I0, ip.ntiles, ip.tail) * 8));
            }
            const int rows_r = (it.I1 - it.I0) * TILE, rows_c = it.tri ? 0 : (it.J1 - it.J0) * TILE;
            if (it.tail) {                      // compact last row: the epilogue warp applies it (strip);
                it.ntiles -= it.I1 - it.I0;     // the ring streams the full rows 0 .. nT-2
                it.I1 -= 1;
                it.J1 -= 1;
                it.tail = 0;
            }
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
                        tb = (unsigned)item_tile_doubles(it, I_, J_) * 8u;
                        toff = item_tile_off(it, l0 + lane, I_);
                    }
                    unsigned bytes = tb;
#pragma unroll
                    for (int o = 1; o < RT; o <<= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
                    if (lane == 0) mbar_expect_tx(&full[slot], bytes);
                    __syncwarp();
                    if (merge) {
                        // one copy per run of stream-contiguous tiles: full tiles
                        // of a row are adjacent in the packed operator and in the
                        // slot; a (shorter, packed) diagonal tile ends a run
                        const unsigned ptb = __shfl_up_sync(FULL, tb, 1);
                        const bool start = lane < nt && (lane == 0 || ptb != (unsigned)TILE_ELEMS * 8u);
                        unsigned rb = 0;
                        bool open = true;
#pragma unroll
                        for (int k = 0; k < RT; ++k) {              // run bytes from this lane on
                            const unsigned tk = __shfl_sync(FULL, tb, k);
                            if (k >= lane && k < nt && open) {
                                rb += tk;
                                open = tk == (unsigned)TILE_ELEMS * 8u;
                            }
                        }
                        if (start) bulk_g2s(dst + lane * TILE_ELEMS, src + toff, rb, &full[slot]);
                    } else if (lane < nt) {
                        bulk_g2s(dst + lane * TILE_ELEMS, src + toff, tb, &full[slot]);
                    }
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
            const bool scat = it.part_off < 0 && op.out_mode == 0 && !bare_epi;
            int ix[RING_MAX_ROWS / 32];
            double zv[RING_MAX_ROWS / 32];
            if (scat) {
                const int32_t* idx = oidx + op.idx_off + g0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) ix[r] = (lane + 32 * r < nr) ? idx[lane + 32 * r] : 0;
#pragma unroll
                for (int r = 0; r < RING_MAX_ROWS / 32; ++r) zv[r] = (lane + 32 * r < nr) ? z[ix[r]] : 0.0;
            }
            // compact last row (whole-operator triangles): the strip S (th x W,
            // column-major, W = (nT - 1) 32) and its packed th x th diagonal
            // tile, read from global memory while the consumers stream the
            // rest: lane j of column block c adds S(:, 32c + j)^T s_tail to
            // row 32c + j (a register per block), and the direct parts
            // S(i, :) s are per-lane partials reduced over the warp
            double* yT = yt_sm + (size_t)e * maxr;             // row 32 cb + lane: this lane's own entries
            double ys = 0.0;
            const int th = no_strip ? 0 : it.tail, W = (it.I1 - it.I0 - 1) * TILE;
            if (th) {
                const double* S = tiles + it.tile_off + item_tile_off(it, (it.I1 - it.I0 - 1) * (it.I1 - it.I0) / 2,
                                                                      it.I1 - 1);
                const double* sv = s + op.s_off + g0;              // s from global (L2): no hold on the s buffer
                for (int x = lane; x < W; x += TILE) yT[x] = 0.0;
                for (int i = 0; i < th; ++i) {                    // strip row i (L1 serves the re-reads)
                    const double si = __ldg(sv + W + i);
                    double d = 0.0;
#pragma unroll
                    for (int cb = 0; cb < RING_MAX_ROWS / 32; ++cb)
                        if (cb * TILE < W) {
                            const double v = __ldg(S + (int64_t)(cb * TILE + lane) * th + i);
                            yT[cb * TILE + lane] = fma(v, si, yT[cb * TILE + lane]);
                            d = fma(v, __ldg(sv + cb * TILE + lane), d);
                        }
                    d = warp_sum(d);
                    if (lane == i) ys = d;
                }
                // diagonal tile: lane i < th, direct L'(i, :) and transposed L'(:, i)^T parts
                const double* D = S + (int64_t)W * th;
                if (lane < th) {
                    double dg = 0.0;
                    for (int j = 0; j <= lane; ++j) dg = fma(D[tail_col_off(th, j) + lane - j], __ldg(sv + W + j), dg);
                    for (int i = lane; i < th; ++i)
                        dg = fma(D[tail_col_off(th, lane) + i - lane], __ldg(sv + W + i), dg);
                    ys += dg;
                }
            }
            mbar_wait(&pdone[b], ph & 1);
            if (bare_epi) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfree[b]);
                continue;
            }
            const double* pr = pr_sm + (size_t)b * maxr;
            const double* pc = pc_sm + (size_t)b * maxr;
            const double* pr2 = pr2_sm + (size_t)b * maxr;
#pragma unroll
            for (int r = 0; r < RING_MAX_ROWS / 32; ++r) {
                const int x = lane + 32 * r;
                if (x < rows_t) {
                    const double pxr = split == 2 ? pr[x] + pr2[x] : pr[x];
                    const double y = th ? (x < W ? pxr + pc[x] + yT[x] : ys)
                                        : (it.tri ? pxr + pc[x] : (x < rows_r ? pxr : pc[x]));
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
        //   row warp:    rows a, a + rstep, ... (split 1: a = (wr - ki) mod 8, rstep 8;
        //                split 2: a = (wr / 2 - ki) mod 4, rstep 4, column half wr & 1)
        //   column warp: columns a, a + 8; per row r both owned columns in order
        const int rstep = (!colw && split == 2) ? 4 : 8, hh = (!colw && split == 2) ? (wr & 1) : 0;
        const int a = (!colw && split == 2) ? ((wr >> 1) - ki) & 3 : (wr - ki) & 7;
        if (hh) pr = pr2_sm + (size_t)bi * maxr;
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
                r += rstep;
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
            while (!copy_only && l >= 0 && l < l0 + RT) {
                const double* T = C + (l - l0) * TILE_ELEMS;
                const bool diag = tri && r == c;
                if (!colw) {
                    // direct part: lane = row, s_J broadcast; columns [j0, j0 + jn)
                    const double2* sJ = reinterpret_cast<const double2*>(ss + (tri ? c * TILE : rows_r + c * TILE));
                    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
                    if (!diag) {
                        if (split == 2) {
                            const double* Th = T + hh * 16 * TILE;
                            const double2* sh = sJ + hh * 8;
#pragma unroll
                            for (int j = 0; j < 16; j += 4) {
                                const double2 u = sh[j / 2], v = sh[j / 2 + 1];
                                d0 = fma(Th[j * TILE + lane], u.x, d0);
                                d1 = fma(Th[(j + 1) * TILE + lane], u.y, d1);
                                d2 = fma(Th[(j + 2) * TILE + lane], v.x, d2);
                                d3 = fma(Th[(j + 3) * TILE + lane], v.y, d3);
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < TILE; j += 4) {
                                const double2 u = sJ[j / 2], v = sJ[j / 2 + 1];
                                d0 = fma(T[j * TILE + lane], u.x, d0);
                                d1 = fma(T[(j + 1) * TILE + lane], u.y, d1);
                                d2 = fma(T[(j + 2) * TILE + lane], v.x, d2);
                                d3 = fma(T[(j + 3) * TILE + lane], v.y, d3);
                            }
                        }
                    } else {
                        const int j0 = split == 2 ? hh * 16 : 0, jn = split == 2 ? 16 : TILE;
#pragma unroll 4
                        for (int jj = 0; jj < jn; jj += 4) {
                            const int j = j0 + jj;
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

// ---- k_symv_whole: whole small triangles, one bulk copy per item -------------
// For colours whose operators are single small triangles (C3: m <= 160, at most
// 5 x 5 tiles = 103 KB) the whole item fits in shared memory twice.  Item k of
// a CTA's byte-balanced range lands in buffer k & 1 by one bulk copy of its
// contiguous tiles (compact last row) plus its s segment and its index list
// (one mbarrier); the producer writes the item's sizes next to them.  The 16
// consumer warps split the item's (nT + 1) nT contributions -- for output
// segment g: the direct parts of tiles (g, 0..g), the transposed part of
// diagonal tile (g, g), the transposed parts of tiles (g+1..nT-1, g) -- two per
// warp, each a 32-vector written to shared memory.  One named barrier per item;
// then thread x sums segment x / 32's contributions in that fixed order
// (deterministic) and applies z[idx[x]] += y.  Its z value is loaded as soon
// as the item lands, so the load overlaps the item's products (same-colour
// subdomains are disjoint), and no consumer ever waits on a descriptor or
// index load from global memory.
constexpr int WH_MAX_NT = 5;
constexpr int WH_MAX_ROWS = WH_MAX_NT * TILE;
constexpr int WH_CONS = 16;
__host__ __device__ constexpr int64_t wh_item_doubles(int nT) {
    return (int64_t)(nT * (nT + 1) / 2 - nT) * TILE_ELEMS + (int64_t)nT * DIAG_ELEMS;
}
// tiles [2][BUFD] | s [2][nT 32] | contributions [2][(nT+1) nT][32] | row indices [2][160] |
// item sizes [2][4] | mbarriers full[2], empty[2]
__host__ __device__ constexpr size_t wh_smem(int nT) {
    return 2 * (size_t)((wh_item_doubles(nT) + 15) / 16 * 16) * 8 + 2 * (size_t)nT * TILE * 8 +
           2 * (size_t)(nT + 1) * nT * TILE * 8 + 2 * (size_t)WH_MAX_ROWS * 4 + 2 * 4 * 4 + 4 * 8;
}
// first double of tile (r, c) of a whole-operator triangle (tail: compact last row)
__device__ __forceinline__ int wh_toff(int r, int c, int nT, int tail) {
    const int base = (r * (r + 1) / 2 - r) * TILE_ELEMS + r * DIAG_ELEMS;   // rows 0..r-1
    return base + c * ((tail && r == nT - 1) ? tail * TILE : TILE_ELEMS);
}

// Work plan of the 16 consumer warps for a triangle of nT <= 5 tile rows: up
// to 3 contributions q = g (nT + 1) + k each, balanced by longest-processing-
// time first over measured-cost weights (host wh_plan_init).
constexpr int WH_PLAN_U = 3;
constexpr int WH_PLANS = 2;   // 0: q = warp, warp + 16; 1: LPT
__constant__ int8_t c_wh_plan[WH_PLANS][WH_MAX_NT + 1][WH_CONS][WH_PLAN_U];

// contribution (g, k) of a triangle with nT tile rows (see above)
__device__ __forceinline__ double wh_contrib(const double* __restrict__ T0, const double* __restrict__ ss, int nT,
                                             int tail, int g, int k, int lane) {
    const int thg = (tail && g == nT - 1) ? tail : TILE;
    if (k <= g) return tile_direct(T0 + wh_toff(g, k, nT, tail), ss, g, k, thg, lane);
    if (k == g + 1) return tile_trans(T0 + wh_toff(g, g, nT, tail), ss, g, g, thg, lane);
    const int r = k - 1;
    return tile_trans(T0 + wh_toff(r, g, nT, tail), ss, r, g, (tail && r == nT - 1) ? tail : TILE, lane);
}

__global__ void __launch_bounds__((WH_CONS + 1) * 32, 1)   // 5 warps on one SM sub-partition: 96 registers
k_symv_whole(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items, int item_begin,
             const int32_t* __restrict__ cta_part, const double* __restrict__ tiles, const double* __restrict__ s,
             const int32_t* __restrict__ oidx, double* __restrict__ z, const int32_t* done, int nTmax, int split,
             int plan) {
    pdl_wait();
    if (*done) return;
    extern __shared__ __align__(128) double wsm[];
    const int64_t BUFD = (wh_item_doubles(nTmax) + 15) / 16 * 16;
    double* tbuf = wsm;                                        // [2][BUFD]
    double* sbuf = tbuf + 2 * BUFD;                            // [2][nTmax * 32]
    double* cbuf = sbuf + 2 * nTmax * TILE;                    // [2][(nTmax + 1) nTmax][32]
    int32_t* ibuf = reinterpret_cast<int32_t*>(cbuf + 2 * (nTmax + 1) * nTmax * TILE);   // [2][WH_MAX_ROWS]
    int32_t* dbuf = ibuf + 2 * WH_MAX_ROWS;                    // [2][4]: nT, m, tail
    uint64_t* full = reinterpret_cast<uint64_t*>(dbuf + 8);    // [2] tiles, s, idx landed
    uint64_t* empty = full + 2;                                // [2] consumed
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = item_begin + cta_part[blockIdx.x], i1 = item_begin + cta_part[blockIdx.x + 1];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (i0 >= i1) return;
    if (warp == WH_CONS) {                                     // ---- producer: bulk copies ----
        if (lane != 0) return;
        DescPipe dp;
        dp.init(items, ops, i0, i1);
        for (int k = 0; k < i1 - i0; ++k) {
            const int b = k & 1;
            ItemDesc it;
            OpDesc op;
            dp.next(items, ops, i0 + k, i1, it, op);
            if (k >= 2) mbar_wait(&empty[b], ((k - 2) >> 1) & 1);
            const int h = it.I1 - it.I0;
            int32_t* d = dbuf + b * 4;
            d[0] = h;
            d[1] = op.m;
            d[2] = it.tail;
            const unsigned tb = (unsigned)(item_doubles(1, h, it.ntiles, it.tail) * 8),
                           sb = (unsigned)(h * TILE * 8), ib = (unsigned)((op.m + 3) / 4 * 16);
            mbar_expect_tx(&full[b], tb + sb + ib);            // arrive (release: the sizes)
            bulk_g2s(sbuf + b * nTmax * TILE, s + op.s_off, sb, &full[b]);
            bulk_g2s(ibuf + b * WH_MAX_ROWS, oidx + op.idx_off, ib, &full[b]);
            const double* src = tiles + it.tile_off;
            double* dst = tbuf + b * BUFD;
            if ((split & 0xff) <= 1 || it.tail) {
                bulk_g2s(dst, src, tb, &full[b]);
            } else {                                           // one copy per tile row (experiment)
                for (int r = 0; r < h; ++r) {
                    const int64_t o0 = (int64_t)(r * (r + 1) / 2 - r) * TILE_ELEMS + (int64_t)r * DIAG_ELEMS;
                    const unsigned rb = (unsigned)((r * TILE_ELEMS + DIAG_ELEMS) * 8);
                    bulk_g2s(dst + o0, src + o0, rb, &full[b]);
                }
            }
        }
        return;
    }
    // ---- consumers: contributions q = warp, warp + 16 of each item ----
    const int tid = threadIdx.x;
    for (int k = 0; k < i1 - i0; ++k) {
        const int b = k & 1;
        mbar_wait(&full[b], (k >> 1) & 1);
        const int32_t* d = dbuf + b * 4;
        const int nT = d[0], nr = d[1], tail = d[2];
        int ixk = 0;
        double zvk = 0.0;
        if (tid < nr) {                                        // z now, used after the products
            ixk = ibuf[b * WH_MAX_ROWS + tid];
            zvk = z[ixk];
        }
        const double* T0 = tbuf + b * BUFD;
        const double* ss = sbuf + b * nTmax * TILE;
        double* cb = cbuf + b * (nTmax + 1) * nTmax * TILE;
        const int inv = (256 + nT) / (nT + 1);                 // q / (nT + 1) = (q * inv) >> 8, q < 32
        if (!(split & 0x100))                                  // DDG_RING_WHOLE bit 8: copy-only probe (debug)
#pragma unroll
            for (int u = 0; u < WH_PLAN_U; ++u) {
                const int q = c_wh_plan[plan][nT][warp][u];
                if (q < 0) break;
                const int g = (q * inv) >> 8, kk = q - g * (nT + 1);
                cb[q * TILE + lane] = wh_contrib(T0, ss, nT, tail, g, kk, lane);
            }
        asm volatile("bar.sync 1, %0;" ::"n"(WH_CONS * 32) : "memory");
        if (tid == 0) mbar_arrive(&empty[b]);                  // tiles, s and idx of buffer b consumed
        if (tid < nr) {
            const int g = tid >> 5;
            const double* c = cb + g * (nT + 1) * TILE + (tid & 31);
            double y = 0.0;
            for (int kk = 0; kk <= nT; ++kk) y += c[kk * TILE];
            z[ixk] = zvk + y;
        }
    }
}

// Sum the partial segments of multi-item operators for one row block, in
// fixed item order, and apply the result.  The block's segment offsets are
// staged in shared memory first, and each row's index and z value are
// fetched before its partial sums, so no load waits on a descriptor.
__global__ void k_symv_reduce(const OpDesc* __restrict__ ops, const ItemDesc* __restrict__ items,
                              const RedDesc* __restrict__ red, int red_begin,
                              const int32_t* __restrict__ oidx, const double* __restrict__ partials,
                              double* __restrict__ z, double* __restrict__ y_out,
                              const int32_t* done) {
    pdl_wait();
    if (*done) return;
    __shared__ int64_t off[64];
    const RedDesc rd = red[red_begin + blockIdx.x];
    const OpDesc op = ops[rd.op];
    const int b = rd.b, nblk = op.nblk;
    auto seg = [&](int j) -> int64_t {
        if (j <= b) return items[op.item_base + b * (b + 1) / 2 + j].part_off;   // items (b, j): row segments
        const ItemDesc it = items[op.item_base + j * (j + 1) / 2 + b];           // items (j, b): column segments
        return it.part_off + (int64_t)(it.I1 - it.I0) * TILE;
    };
    for (int j = threadIdx.x; j < min(nblk, 64); j += blockDim.x) off[j] = seg(j);
    __syncthreads();
    const int rows_b = (min(op.nT, (b + 1) * op.BT) - b * op.BT) * TILE;
    for (int x = threadIdx.x; x < rows_b; x += blockDim.x) {
        const int g = b * op.BT * TILE + x;
        const bool ok = g < op.m;
        const bool scat = ok && op.out_mode == 0;
        const int ix = scat ? oidx[op.idx_off + g] : 0;
        const double zv = scat ? z[ix] : 0.0;
        double y = 0.0;
#pragma unroll 8
        for (int j = 0; j < min(nblk, 64); ++j) y += partials[off[j] + x];
        for (int j = 64; j < nblk; ++j) y += partials[seg(j) + x];     // very large dense operators
        if (scat) z[ix] = zv + y;
        else if (ok) y_out[g] = y;
    }
}


// ---- launchers ----

void launch_gather_flat(cudaStream_t st, int64_t x0, int64_t x1, const int32_t* gidx, DevCSR A, const double* r,
                        const double* z, double* s, bool z_is_zero, const int32_t* done) {
    if (x1 <= x0) return;
    const int sw = z_is_zero ? 1 : std::max(1, A.sw);
    const int64_t want = ((x1 - x0) * sw + 255) / 256;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)num_sms() * 8));
    const int zz = z_is_zero ? 1 : 0;
    switch (sw) {
        case 4: launch_pdl(k_gather_flat<4>, g, 256, 0, st, x0, x1, gidx, A, r, z, s, zz, done); break;
        case 8: launch_pdl(k_gather_flat<8>, g, 256, 0, st, x0, x1, gidx, A, r, z, s, zz, done); break;
        case 32: launch_pdl(k_gather_flat<32>, g, 256, 0, st, x0, x1, gidx, A, r, z, s, zz, done); break;
        default: launch_pdl(k_gather_flat<1>, g, 256, 0, st, x0, x1, gidx, A, r, z, s, zz, done);
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
    DDG_MAX_DYN_SMEM(k_symv);
    k_symv<<<nitems, SYMV_WARPS * 32, smem, st>>>(ops, items, item_begin, tiles, s, oidx, z, y_out,
                                                  partials, done, tickets, gather_mode, A, r);
}

static bool g_ring_init[64] = {};
static int g_ring_rt = 4, g_ring_nb = 0, g_ring_nst = 0, g_ring_v2 = 0, g_ring_whole = 1, g_ring_pf = 0,
           g_ring2_split = 2;
int g_compact = 1;   // compact tails for whole-triangle colours (DDG_COMPACT)
static unsigned long long* g_ring_trace = nullptr;   // DDG_RING_TRACE (debug)
static void wh_plan_init();
static int g_whole_plan = 0;   // DDG_WHOLE_PLAN (WH_PLANS; 0 measured best: C3 0.949 vs LPT 0.914)
// per device, once, outside any stream capture (called from ddg_setup)
void symv_ring_init() {
    // every switch computed in locals and stored once: ddg_setup may run in several
    // host threads at a time (loopback ranks), so no global may pass through a
    // transient value another thread could read
    int rt = 4;
    if (const char* e = getenv("DDG_RING_TILES")) rt = atoi(e);
    if (rt != 1 && rt != 2 && rt != 8) rt = 4;
    int nb = 0;
    if (const char* e = getenv("DDG_RING_NB")) nb = std::max(2, std::min(RING_MAX_NB, atoi(e)));
    int nst = 0;
    if (const char* e = getenv("DDG_RING_NST")) nst = std::max(2, std::min(RING_MAX_NST, atoi(e)));
    const int v2 = getenv("DDG_RING_V2") ? atoi(getenv("DDG_RING_V2")) : -1;   // -1: auto
    // DDG_COMPACT (default 1): whole-triangle operators store their last tile
    // row compact (no padding rows streamed); read by every kernel but the
    // 8-warp ring, which is only chosen for triangles when forced (DDG_RING_V2=0)
    int compact = (v2 == 0) ? 0 : 1;
    if (const char* e = getenv("DDG_COMPACT")) compact = atoi(e) != 0;
    g_ring_rt = rt;
    g_ring_nb = nb;
    g_ring_nst = nst;
    g_ring_v2 = v2;
    g_pdl = getenv("DDG_PDL") ? (atoi(getenv("DDG_PDL")) != 0) : 1;
    // DDG_RING_WHOLE: 0 off, 1 (default) one copy per item, n > 1 one copy per tile row
    g_ring_whole = getenv("DDG_RING_WHOLE") ? atoi(getenv("DDG_RING_WHOLE")) : 1;
    g_ring2_split = ((getenv("DDG_RING2_SPLIT") && atoi(getenv("DDG_RING2_SPLIT")) == 1) ? 1 : 2) |
                    ((getenv("DDG_RING2_COPYONLY") && atoi(getenv("DDG_RING2_COPYONLY")) != 0) ? 0x100 : 0) |
                    ((getenv("DDG_RING2_MERGE") && atoi(getenv("DDG_RING2_MERGE")) != 0) ? 0x200 : 0) |
                    (!getenv("DDG_RING2_BARE_EPI") ? 0 : atoi(getenv("DDG_RING2_BARE_EPI")) == 1 ? 0x400
                     : atoi(getenv("DDG_RING2_BARE_EPI")) == 2 ? 0x800 : 0);
    g_ring_pf = getenv("DDG_RING_PF") ? atoi(getenv("DDG_RING_PF")) : 0;      // ... by k_symv_ring2
    g_compact = compact;

    if (getenv("DDG_RING_TRACE") && !g_ring_trace) {
        if (cudaMalloc(&g_ring_trace, 32 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(g_ring_trace, 0, 32 * sizeof(unsigned long long));
        else
            g_ring_trace = nullptr;
    }
    g_whole_plan = getenv("DDG_WHOLE_PLAN") ? std::max(0, std::min(WH_PLANS - 1, atoi(getenv("DDG_WHOLE_PLAN")))) : 0;
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
    cudaFuncSetAttribute(k_symv_whole, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    wh_plan_init();
    g_ring_init[dev & 63] = true;
}

// k_symv_whole work plan (c_wh_plan): longest processing time first.  Unit
// costs (relative instructions per warp, from the ncu source page): direct
// full tile 1, direct diagonal 1.2, transposed full tile 1.6, transposed pass
// over the packed diagonal tile 3.
static void wh_plan_init() {
    int8_t plans[WH_PLANS][WH_MAX_NT + 1][WH_CONS][WH_PLAN_U];
    memset(plans, -1, sizeof plans);
    for (int mode = 0; mode < WH_PLANS; ++mode)
    for (int nT = 1; nT <= WH_MAX_NT; ++nT) {
        auto& plan = plans[mode];
        if (mode == 0) {
            for (int q = 0; q < (nT + 1) * nT; ++q) plan[nT][q % WH_CONS][q / WH_CONS] = (int8_t)q;
            continue;
        }
        std::vector<std::pair<double, int>> units;
        for (int g = 0; g < nT; ++g)
            for (int k = 0; k <= nT; ++k) {
                const int q = g * (nT + 1) + k;
                units.push_back({k < g ? 1.0 : k == g ? 1.2 : k == g + 1 ? 3.0 : 1.6, q});
            }
        std::stable_sort(units.begin(), units.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
        double load[WH_CONS] = {};
        int cnt[WH_CONS] = {};
        for (const auto& u : units) {
            int w = 0;
            for (int v = 1; v < WH_CONS; ++v)
                if (cnt[v] < WH_PLAN_U && (cnt[w] >= WH_PLAN_U || load[v] < load[w])) w = v;
            plan[nT][w][cnt[w]++] = (int8_t)u.second;
            load[w] += u.first;
        }
    }
    cudaMemcpyToSymbol(c_wh_plan, plans, sizeof plans);
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
    // whole small triangles (C3): one bulk copy per item, k_symv_whole
    const int nTw = (std::max(TILE, max_rows_r) + TILE - 1) / TILE;
    if (triangles && g_ring_whole && nTw <= WH_MAX_NT && max_rows_c == 0 && wh_smem(nTw) <= budget) {
        launch_pdl(k_symv_whole, ncta, (WH_CONS + 1) * 32, wh_smem(nTw), st, ops, items, item_begin, cta_part, tiles,
                   s, oidx, z, done, nTw, g_ring_whole, g_whole_plan);
        return;
    }
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
            launch_pdl(k_symv_ring2<2>, ncta, RING2_THREADS, smem2, st, ops, items, item_begin, cta_part, tiles, s,
                       oidx, z, y_out, partials, done, nst2, nb2, maxr, g_ring_pf, g_ring2_split);
        else if (RT == 8)
            launch_pdl(k_symv_ring2<8>, ncta, RING2_THREADS, smem2, st, ops, items, item_begin, cta_part, tiles, s,
                       oidx, z, y_out, partials, done, nst2, nb2, maxr, g_ring_pf, g_ring2_split);
        else
            launch_pdl(k_symv_ring2<4>, ncta, RING2_THREADS, smem2, st, ops, items, item_begin, cta_part, tiles, s,
                       oidx, z, y_out, partials, done, nst2, nb2, maxr, g_ring_pf, g_ring2_split);
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
        launch_pdl(k_symv_ring<1>, ncta, RING_THREADS, smem, st, ops, items, item_begin, cta_part, tiles, s, oidx,
                   z, y_out, partials, done, nst, nb, R, Cr, g_ring_trace);
    else if (RT == 2)
        launch_pdl(k_symv_ring<2>, ncta, RING_THREADS, smem, st, ops, items, item_begin, cta_part, tiles, s, oidx,
                   z, y_out, partials, done, nst, nb, R, Cr, g_ring_trace);
    else
        launch_pdl(k_symv_ring<4>, ncta, RING_THREADS, smem, st, ops, items, item_begin, cta_part, tiles, s, oidx,
                   z, y_out, partials, done, nst, nb, R, Cr, g_ring_trace);
}

void launch_symv_reduce(cudaStream_t st, const OpDesc* ops, const ItemDesc* items,
                        const RedDesc* red, int red_begin, int nred, const int32_t* oidx,
                        const double* partials, double* z, double* y_out, const int32_t* done) {
    if (nred <= 0) return;
    launch_pdl(k_symv_reduce, nred, 256, 0, st, ops, items, red, red_begin, oidx, partials, z, y_out, done);
}

}  // namespace ddg
