// ctx.h — the ddg_ctx object shared by setup.cpp and coarse_sparse.cpp (internal).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include <string>
#include <functional>
#include <vector>

#include "../../include/ddg.h"
#include "comm.h"
#include "ddg_internal.h"
#include "dist.h"

using namespace ddg;

int set_err(int code, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return set_err(_e == cudaErrorMemoryAllocation ? DDG_E_OOM : DDG_E_CUDA,     \
                           "%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
    } while (0)


// host work split over the hardware threads: fn(begin, end, thread) on chunks of [0, n)
void parallel_for(int64_t n, const std::function<void(int64_t, int64_t, int)>& fn);

struct SparseCoarse;   // coarse_sparse.cpp
void sparse_coarse_free(SparseCoarse* sc);

template <typename T>
static int dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess)
        return set_err(DDG_E_OOM, "cudaMalloc of %zu bytes failed: %s", count * sizeof(T),
                       cudaGetErrorString(e));
    static const int fill = getenv("DDG_DEBUG_FILL") ? atoi(getenv("DDG_DEBUG_FILL")) : -1;
    if (fill >= 0) {   // debug: 0 zeroes, 255 poisons (NaN)
        cudaMemset(*p, fill, count * sizeof(T));
        cudaDeviceSynchronize();
    }
    return DDG_OK;
}

struct ddg_ctx {
    ddg_opts opts{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t n = 0, nnz = 0;
    int k = 0, nparts = 0;
    // host structures
    std::vector<int64_t> bptr;
    std::vector<int32_t> bidx, bpos, part;
    std::vector<int64_t> optr;
    std::vector<int32_t> oidx;
    std::vector<int32_t> colour, order;
    int ncolours = 0;
    std::vector<ColourPlan> plans;
    std::vector<int32_t> cptr;
    std::vector<int64_t> qoff;
    std::vector<double> Q;
    int64_t nc = 0;
    int dropped = 0;
    double min_ratio = INFINITY;
    std::vector<OpDesc> ops;
    std::vector<ItemDesc> items;
    std::vector<RedDesc> red;
    int coarse_op = -1;
    int coarse_item_begin = 0, coarse_item_end = 0, coarse_red_begin = 0, coarse_red_end = 0;
    int coarse_rows_t = 0;
    int maxmI = 0;
    int64_t tiles_doubles = 0, s_doubles = 0, part_doubles = 0;
    // device
    DevCSR A{};
    int32_t *d_rp = nullptr, *d_col = nullptr;
    double* d_val = nullptr;
    int32_t* d_oidx = nullptr;
    OpDesc* d_ops = nullptr;
    ItemDesc* d_items = nullptr;
    RedDesc* d_red = nullptr;
    double *d_tiles = nullptr, *d_s = nullptr, *d_partials = nullptr;
    int64_t* d_bptr = nullptr;
    int32_t *d_bidx = nullptr, *d_cptr = nullptr;
    int64_t* d_qoff = nullptr;
    double *d_Q = nullptr, *d_yc = nullptr;
    double *d_r = nullptr, *d_z = nullptr, *d_p = nullptr, *d_q = nullptr, *d_f = nullptr,
           *d_u = nullptr, *d_x = nullptr;
    Scalars* d_sc = nullptr;
    double* d_hist = nullptr;
    double* d_ab = nullptr;             // CG coefficients of the current solve (Scalars::ab)
    std::vector<double> last_alpha, last_beta;
    int hist_cap = 0;
    double* d_redbuf = nullptr;
    unsigned* d_ticket = nullptr;
    int32_t* d_zero = nullptr;  // a device int that stays 0 (`done` for test hooks)
    unsigned* d_tickets = nullptr;  // per-operator completion tickets of k_symv
    Scalars* h_sc = nullptr;    // pinned mirror
    cudaGraph_t g_iter = nullptr;
    cudaGraphExec_t ge_iter = nullptr;
    const double* g_iter_u = nullptr;  // u pointer baked into the captured graph
    int64_t launches = 0;
    int64_t launches_per_iter = 0;
    // device-side loop (one graph per solve: WHILE(not done){ a1-a3; IF(not done){ a4-a9 } })
    cudaGraph_t g_solve = nullptr;
    cudaGraphExec_t ge_solve = nullptr;
    const double* g_solve_u = nullptr;
    int64_t launches_a = 0, launches_b = 0;
    int device_loop = 1;       // DDG_DEVICE_LOOP=0: host-stepped chunks
    int loop_graph_used = 0;
    int64_t local_bytes = 0, coarse_bytes = 0;
    double t_setup = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // multi-GPU (NCCL): the z halo of a colour's boundary subdomains runs on a side
    // stream while the interior subdomains compute (colour_step)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // profiling (ddg_set_profiling)
    bool profiling = false;
    std::vector<cudaEvent_t> evpool;
    struct ProfRec { int cat; int e0, e1; double bytes; };
    std::vector<ProfRec> recs;
    std::vector<double> colour_alg_bytes;
    // coarse solver variant: 1 dense packed inverse, 2 sparse supernodal (coarse_sparse.cpp)
    int coarse_variant = 1;   // 1 dense, 2 sparse, 3 three levels (child two-level context on A_c)
    bool flat_coarse = true;           // two-stage restriction + flat prolongation (single GPU)
    double* d_res = nullptr;           // r - A z in part order (flat restriction)
    int32_t* d_xpart = nullptr;        // part of every position of the part order
    // small problems: the whole solve in one cluster kernel (k_pcg_small, pcg.cu)
    bool small_ok = false;
    SmallArgs small{};                 // its shared-memory plan (small_plan)
    int32_t* d_cops = nullptr;         // [ncolours + 1] operator ranges of the colours
    int32_t *d_brp = nullptr, *d_bcol = nullptr;   // node-blocked columns of A (DevCSR::bs)
    struct ddg_ctx* child = nullptr;   // three levels: the two-level method on A_c
    double* d_bc = nullptr;            // three levels: coarse right-hand side R_0 (r - A z)
    SparseCoarse* sparse = nullptr;
    // multi-GPU (dist.cpp / comm.cpp)
    ddg_comm* comm = nullptr;
    bool dist = false;
    int rank = 0, nranks = 1;
    int comm_err = 0;
    ddg::DistPlan plan;
    int32_t* d_rows = nullptr;          // owned rows (nullptr: all rows)
    int64_t nrows = 0;
    ddg::Halo h_p, h_r;
    std::vector<ddg::Halo> h_z;         // one per colour
    int32_t* d_restrict_parts = nullptr;
    int n_restrict = 0;
    int32_t* d_prolong_parts = nullptr;
    int n_prolong = 0;
    std::vector<int32_t> op_sub;        // subdomain id of every local operator
    std::vector<int32_t> block_coords;  // optional nparts x block_ndim
    int block_ndim = 0;
    // SYMV kernel choice (DDG_SYMV: "ring" default, "classic") and the
    // byte-balanced CTA partitions of every k_symv_ring launch
    int symv_mode = 0;                  // 0 ring, 1 classic per-item k_symv
    bool chol = false;                  // local_variant DDG_LOCAL_CHOLESKY: factors instead of inverses (chol.cu)
    std::vector<int32_t> h_ring;
    std::vector<std::pair<int, std::pair<int, int>>> ring_rc;   // partition offset -> (max rows_r, max rows_c)
    int32_t* d_ring = nullptr;
    int32_t* d_gidx = nullptr;          // s position -> fine row (-1: padding)
    double* d_stencil_coef = nullptr;   // ddg_stencil FACE7 coefficients (device)
    int coarse_ring_off = -1;
    double ring_min_bytes = 16e6;       // launches moving less use the per-item k_symv
};

// append the CTA partition of items [b, e) for k_symv_ring; returns its offset
// in c->h_ring, or -1 when the range is empty or an item exceeds the ring's rows
int ring_partition(ddg_ctx* c, int b, int e);
// largest row block and column block (rows) of the items of partition `off`
void ring_dims(const ddg_ctx* c, int off, int* max_rows_r, int* max_rows_c);
// launch the colour/coarse SYMV over items [b, e) with the context's kernel choice
bool ring_ok(const ddg_ctx* c, int off);

enum { PC_SYMV = 0, PC_GATHER, PC_REDUCE, PC_COARSE, PC_VEC, PC_N };

static int prof_event(ddg_ctx* c) {
    int need = 0;
    for (auto& r : c->recs) need = std::max(need, std::max(r.e0, r.e1) + 1);
    if ((int)c->evpool.size() <= need) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        c->evpool.push_back(e);
    }
    return need;
}
// bracket the launches issued by fn with an event pair when profiling
template <typename Fn>
static void prof(ddg_ctx* c, int cat, double bytes, Fn fn) {
    if (!c->profiling) { fn(); return; }
    ddg_ctx::ProfRec r{cat, 0, 0, bytes};
    r.e0 = prof_event(c);
    c->recs.push_back(r);
    cudaEventRecord(c->evpool[r.e0], c->stream);
    fn();
    int e1 = prof_event(c);
    c->recs.back().e1 = e1;
    cudaEventRecord(c->evpool[e1], c->stream);
}


// Every host<->device transfer of the library is ordered on the context
// stream (a legacy-stream cudaMemcpy/cudaMemset is NOT ordered with the
// context's non-blocking stream, and a pageable H2D cudaMemcpy may return
// before its DMA lands).
static inline int h2d(cudaStream_t s, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return DDG_OK;
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DDG_OK;
}
static inline int d2h(cudaStream_t s, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return DDG_OK;
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return DDG_OK;
}
