// bwprobe.cu — read-bandwidth ceilings on this B200 for the access patterns
// the SYMV kernels can use (standalone; not part of libddg).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bwprobe tools/bwprobe.cu && ./bwprobe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_fill(double* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 1e-3 * (i & 1023);
}

// K1: grid-stride double2 streaming loads
__global__ void k_read_v2(const double2* __restrict__ p, size_t n2, double* out) {
    double s = 0;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
#pragma unroll 4
    for (; i < n2; i += st) { double2 v = __ldcs(p + i); s += v.x + v.y; }
    if (s == 12345.678) out[0] = s;
}

// K2: warp per 8 KB tile, lane = row, 32 coalesced 256 B loads (k_symv's pattern)
__global__ void k_read_tiles(const double* __restrict__ p, size_t ntiles, double* out) {
    const int lane = threadIdx.x & 31;
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    double s = 0;
    for (; w < ntiles; w += nw) {
        const double* T = p + w * 1024;
        double a[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = __ldcs(T + j * 32 + lane);
#pragma unroll
        for (int j = 0; j < 32; ++j) s += a[j];
    }
    if (s == 12345.678) out[0] = s;
}

// K3: warp streams a contiguous chunk of tiles (per-warp contiguous ranges, 2 tiles in flight)
__global__ void k_read_tiles2(const double* __restrict__ p, size_t ntiles, double* out) {
    const int lane = threadIdx.x & 31;
    size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    double s = 0;
    for (; w < ntiles; w += 2 * nw) {
        const double* T = p + w * 1024;
        const double* U = p + (w + nw < ntiles ? w + nw : w) * 1024;
        double a[32], b[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = __ldcs(T + j * 32 + lane);
#pragma unroll
        for (int j = 0; j < 32; ++j) b[j] = __ldcs(U + j * 32 + lane);
#pragma unroll
        for (int j = 0; j < 32; ++j) s += a[j] * b[j];
    }
    if (s == 12345.678) out[0] = s;
}

// K4: TMA bulk ring: 1 producer lane, 8 consumer warps, S stages of CH bytes
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
__global__ void __launch_bounds__(288) k_read_tma(const double* __restrict__ p, size_t nch, int CH, int S, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    double* ring = (double*)(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {
        if (lane) return;
        unsigned k = 0;
        for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
            unsigned slot = k % S, n = k / S;
            if (n) mb_wait(&empty[slot], (n - 1) & 1);
            mb_expect(&full[slot], CH);
            bulk((char*)ring + (size_t)slot * CH, (const char*)p + c * CH, CH, &full[slot]);
        }
        return;
    }
    double s = 0;
    unsigned k = 0;
    const int per = CH / 8;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
        unsigned slot = k % S;
        mb_wait(&full[slot], (k / S) & 1);
        const double* T = ring + (size_t)slot * per;
        for (int x = warp * 32 + lane; x < per; x += 256) s += T[x];
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[slot]);
    }
    if (s == 12345.678) out[0] = s;
}

// K5: 32 KB slots filled by NC copies each (the ring's per-tile copies),
// optional packed "diagonal" copies of 4224 B every `diag_every` copies
__global__ void __launch_bounds__(288) k_read_tma_nc(const double* __restrict__ p, size_t nslots, int NC, int S,
                                                     int diag_every, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    double* ring = (double*)(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned CH = 32768, cb = CH / NC;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {
        if (lane) return;
        unsigned k = 0, cnt = 0;
        const char* src = (const char*)p + (size_t)blockIdx.x * CH;
        for (size_t c = blockIdx.x; c < nslots; c += gridDim.x, ++k) {
            unsigned slot = k % S, n = k / S;
            if (n) mb_wait(&empty[slot], (n - 1) & 1);
            unsigned bytes[8], tot = 0;
            for (int q = 0; q < NC; ++q, ++cnt) {
                bytes[q] = (diag_every && cnt % diag_every == 0) ? 4224 : cb;
                tot += bytes[q];
            }
            mb_expect(&full[slot], tot);
            const char* s0 = (const char*)p + c * CH;
            for (int q = 0; q < NC; ++q)
                bulk((char*)ring + (size_t)slot * CH + q * cb, s0 + q * cb, bytes[q], &full[slot]);
        }
        (void)src;
        return;
    }
    double s = 0;
    unsigned k = 0;
    for (size_t c = blockIdx.x; c < nslots; c += gridDim.x, ++k) {
        unsigned slot = k % S;
        mb_wait(&full[slot], (k / S) & 1);
        const double* T = ring + (size_t)slot * 4096;
        s += T[warp * 512 + lane];
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[slot]);
    }
    if (s == 12345.678) out[0] = s;
}

// K6: like K5 with 4 copies per 32 KB slot, the first copy of each slot of
// `first` bytes (the rest 8 KB): the cost of a short / unaligned-size copy
__global__ void __launch_bounds__(288) k_read_tma_first(const double* __restrict__ p, size_t nslots, int S,
                                                        unsigned first, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    double* ring = (double*)(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned CH = 32768;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {
        if (lane) return;
        unsigned k = 0;
        for (size_t c = blockIdx.x; c < nslots; c += gridDim.x, ++k) {
            unsigned slot = k % S, n = k / S;
            if (n) mb_wait(&empty[slot], (n - 1) & 1);
            mb_expect(&full[slot], first + 3 * 8192);
            const char* s0 = (const char*)p + c * CH;
            char* d0 = (char*)ring + (size_t)slot * CH;
            bulk(d0, s0, first, &full[slot]);
            for (int q = 1; q < 4; ++q) bulk(d0 + q * 8192, s0 + q * 8192, 8192, &full[slot]);
        }
        return;
    }
    double sum = 0;
    unsigned k = 0;
    for (size_t c = blockIdx.x; c < nslots; c += gridDim.x, ++k) {
        unsigned slot = k % S;
        mb_wait(&full[slot], (k / S) & 1);
        const double* T = ring + (size_t)slot * 4096;
        sum += T[warp * 512 + lane];
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[slot]);
    }
    if (sum == 12345.678) out[0] = sum;
}

// K7: 4 x 8 KB copies per 32 KB slot; source misaligned by `mis` bytes;
// `contig`: CTA b streams its own contiguous range (the ring's partition)
// instead of slots strided across the grid
__global__ void __launch_bounds__(288) k_read_tma_pat(const double* __restrict__ p, size_t nslots, int S,
                                                      unsigned mis, int contig, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    double* ring = (double*)(smem + 1024);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned CH = 32768;
    const size_t per = nslots / gridDim.x;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {
        if (lane) return;
        for (size_t k = 0; k < per; ++k) {
            const size_t c = contig ? blockIdx.x * per + k : blockIdx.x + k * gridDim.x;
            unsigned slot = k % S, n = k / S;
            if (n) mb_wait(&empty[slot], (n - 1) & 1);
            mb_expect(&full[slot], 4 * 8192);
            const char* s0 = (const char*)p + c * CH + mis;
            char* d0 = (char*)ring + (size_t)slot * CH;
            for (int q = 0; q < 4; ++q) bulk(d0 + q * 8192, s0 + q * 8192, 8192, &full[slot]);
        }
        return;
    }
    double sum = 0;
    for (size_t k = 0; k < per; ++k) {
        unsigned slot = k % S;
        mb_wait(&full[slot], (k / S) & 1);
        const double* T = ring + (size_t)slot * 4096;
        sum += T[warp * 512 + lane];
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[slot]);
    }
    if (sum == 12345.678) out[0] = sum;
}

int main() {
    const size_t bytes = 8ull << 30, n = bytes / 8;
    double *p, *out;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMalloc(&out, 64));
    k_fill<<<148 * 8, 256>>>(p, n);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto fn) {
        fn();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        cudaError_t e = cudaGetLastError();
        printf("%-44s %8.1f GB/s  (%.3f ms)%s\n", name, bytes / (best * 1e-3) / 1e9, best, e ? cudaGetErrorString(e) : "");
    };
    for (int bpsm : {4, 8, 16})
        for (int th : {256, 512}) {
            char nm[96];
            snprintf(nm, sizeof nm, "read_v2 grid=148x%d thr=%d", bpsm, th);
            timeit(nm, [&] { k_read_v2<<<148 * bpsm, th>>>((const double2*)p, n / 2, out); });
        }
    for (int bpsm : {2, 4, 8}) {
        char nm[96];
        snprintf(nm, sizeof nm, "read_tiles (1 tile/warp) 148x%d x256", bpsm);
        timeit(nm, [&] { k_read_tiles<<<148 * bpsm, 256>>>(p, n / 1024, out); });
        snprintf(nm, sizeof nm, "read_tiles2 (2 tiles/warp) 148x%d x256", bpsm);
        timeit(nm, [&] { k_read_tiles2<<<148 * bpsm, 256>>>(p, n / 1024, out); });
    }
    for (int CH : {8192, 16384, 32768})
        for (int S : {4, 8, 12}) {
            size_t sm = 1024 + (size_t)CH * S;
            if (sm > 227 * 1024) continue;
            cudaFuncSetAttribute(k_read_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            for (int cps : {1, 2}) {
                if (sm * cps > 228 * 1024) continue;
                char nm[96];
                snprintf(nm, sizeof nm, "tma ring CH=%dK S=%d ctas/sm=%d", CH / 1024, S, cps);
                timeit(nm, [&] { k_read_tma<<<148 * cps, 288, sm>>>(p, bytes / CH, CH, S, out); });
            }
        }
    for (int contig : {0, 1})
        for (unsigned mis : {0u, 128u, 4224u % 8192u}) {
            const int S = 5;
            const size_t sm = 1024 + (size_t)32768 * S;
            cudaFuncSetAttribute(k_read_tma_pat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            const size_t nslots = bytes / 32768 - 1;
            const double moved = (double)(nslots / 148) * 148 * 32768;
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(e0);
                k_read_tma_pat<<<148, 288, sm>>>(p, nslots, S, mis, contig, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("4x8KB copies/slot, contiguous-per-CTA %d, source offset %4u B: %8.1f GB/s\n", contig, mis,
                   moved / (best * 1e-3) / 1e9);
        }
    return 0;
}
