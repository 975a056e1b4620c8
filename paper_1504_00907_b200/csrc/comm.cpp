// comm.cpp — NCCL communicator of libddg.  NCCL is loaded
// with dlopen (the copy torch ships, or the system one), so libddg itself
// loads and runs single-GPU without it.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "ctx.h"

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

int load_nccl() {
    if (g_nccl.h) return DDG_OK;
    const char* cands[] = {"libnccl.so.2", DDG_NCCL_DIR "/libnccl.so.2", "libnccl.so"};
    for (const char* c : cands) {
        g_nccl.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.h) break;
    }
    if (!g_nccl.h) return set_err(DDG_E_NCCL, "cannot dlopen libnccl.so.2: %s", dlerror());
#define SYM(f, name)                                                        \
    g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(g_nccl.h, name)); \
    if (!g_nccl.f) return set_err(DDG_E_NCCL, "NCCL symbol %s missing", name);
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(allReduce, "ncclAllReduce");
    SYM(send, "ncclSend");
    SYM(recv, "ncclRecv");
    SYM(groupStart, "ncclGroupStart");
    SYM(groupEnd, "ncclGroupEnd");
    SYM(errStr, "ncclGetErrorString");
#undef SYM
    return DDG_OK;
}

#define NCCL_TRY(expr)                                                                     \
    do {                                                                                   \
        ncclResult_t _r = (expr);                                                          \
        if (_r != ncclSuccess) return set_err(DDG_E_NCCL, "%s: %s", #expr, g_nccl.errStr(_r)); \
    } while (0)

}  // namespace

namespace ddg {

constexpr int LOOP_MAX_RANKS = 16;

}  // namespace ddg

struct ddg_loop_group {
    int n = 0, device = 0;
    cudaStream_t stream = nullptr;
    std::mutex mu;
    std::condition_variable cv;
    uint64_t gen = 0;
    int arrived = 0, kind = 0, err = 0;
    int broken = 0;        // a failed collective poisons the group: later calls fail at once
    std::vector<const double*> send;
    std::vector<double*> recv;
    std::vector<size_t> count;
    std::vector<const Halo*> halo;
    double* d_tmp = nullptr;
    size_t tmp_cap = 0;
};

namespace ddg {

cudaStream_t loop_stream(ddg_comm* c) { return c && c->loop ? c->loop->stream : nullptr; }

// the data movement of the current collective (called by the last arrival)
static int loop_execute(ddg_loop_group& g) {
    if (g.kind == 1) {                                  // allreduce (sum)
        const size_t cnt = g.count[0];
        for (int r = 1; r < g.n; ++r)
            if (g.count[r] != cnt) return set_err(DDG_E_NCCL, "loopback allreduce: ranks disagree on the count");
        if (cnt == 0) return DDG_OK;
        if (cnt > g.tmp_cap) {
            if (g.d_tmp) cudaFree(g.d_tmp);
            g.d_tmp = nullptr;
            if (cudaMalloc(&g.d_tmp, cnt * sizeof(double)) != cudaSuccess)
                return set_err(DDG_E_OOM, "loopback allreduce buffer (%zu doubles)", cnt);
            g.tmp_cap = cnt;
        }
        launch_loop_sum(g.stream, g.send.data(), g.n, g.d_tmp, (int64_t)cnt);
        for (int r = 0; r < g.n; ++r)
            if (cudaMemcpyAsync(g.recv[r], g.d_tmp, cnt * sizeof(double), cudaMemcpyDeviceToDevice, g.stream) !=
                cudaSuccess)
                return set_err(DDG_E_CUDA, "loopback allreduce copy");
        return cudaGetLastError() == cudaSuccess ? DDG_OK : set_err(DDG_E_CUDA, "loopback allreduce kernel");
    }
    // halo exchange: rank r's send segment for p lands in p's receive segment for r
    for (int r = 0; r < g.n; ++r)
        for (int p = 0; p < g.n; ++p) {
            const Halo& hs = *g.halo[r];
            const Halo& hr = *g.halo[p];
            const int64_t ns = hs.send_off[p + 1] - hs.send_off[p];
            const int64_t nr = hr.recv_off[r + 1] - hr.recv_off[r];
            if (ns != nr)
                return set_err(DDG_E_NCCL, "loopback exchange: rank %d sends %lld values to %d, which expects %lld", r,
                               (long long)ns, p, (long long)nr);
            if (ns > 0 && cudaMemcpyAsync(hr.d_rbuf + hr.recv_off[r], hs.d_sbuf + hs.send_off[p], ns * sizeof(double),
                                          cudaMemcpyDeviceToDevice, g.stream) != cudaSuccess)
                return set_err(DDG_E_CUDA, "loopback exchange copy");
        }
    return DDG_OK;
}

// rendezvous: deposit this rank's arguments; the last arrival moves the data
static int loop_collective(ddg_comm* c, int kind, const double* send, double* recv, size_t count, const Halo* h) {
    ddg_loop_group& g = *c->loop;
    std::unique_lock<std::mutex> lk(g.mu);
    if (g.broken) return set_err(DDG_E_NCCL, "loopback group failed earlier");
    const uint64_t my = g.gen;
    if (g.arrived == 0) {
        g.kind = kind;
        g.err = 0;
    } else if (g.kind != kind) {
        g.err = set_err(DDG_E_NCCL, "loopback: ranks called different collectives");
    }
    g.send[c->rank] = send;
    g.recv[c->rank] = recv;
    g.count[c->rank] = count;
    g.halo[c->rank] = h;
    if (++g.arrived == g.n) {
        if (!g.err) g.err = loop_execute(g);
        if (g.err) g.broken = 1;
        g.arrived = 0;
        ++g.gen;
        g.cv.notify_all();
    } else {
        g.cv.wait(lk, [&] { return g.gen != my; });
    }
    if (g.err) return set_err(DDG_E_NCCL, "loopback collective failed");   // thread-local message
    return DDG_OK;
}

}  // namespace ddg

extern "C" int ddg_loop_group_create(int nranks, int device, ddg_loop_group** out) {
    if (!out || nranks < 1 || nranks > ddg::LOOP_MAX_RANKS) return set_err(DDG_E_ARG, "loop group: 1..%d ranks", ddg::LOOP_MAX_RANKS);
    CUDA_TRY(cudaSetDevice(device));
    auto* g = new ddg_loop_group();
    g->n = nranks;
    g->device = device;
    g->send.assign(nranks, nullptr);
    g->recv.assign(nranks, nullptr);
    g->count.assign(nranks, 0);
    g->halo.assign(nranks, nullptr);
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete g;
        return set_err(DDG_E_CUDA, "loop group stream");
    }
    ddg::register_no_pdl_stream(g->stream);
    *out = g;
    return DDG_OK;
}

extern "C" void ddg_loop_group_destroy(ddg_loop_group* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->d_tmp) cudaFree(g->d_tmp);
    if (g->stream) {
        ddg::release_no_pdl_stream(g->stream);
        cudaStreamDestroy(g->stream);
    }
    delete g;
}

extern "C" int ddg_comm_init_loopback(ddg_loop_group* g, int rank, ddg_comm** out) {
    if (!g || !out || rank < 0 || rank >= g->n) return set_err(DDG_E_ARG, "ddg_comm_init_loopback: bad argument");
    ddg_comm* c = new ddg_comm();
    c->rank = rank;
    c->nranks = g->n;
    c->device = g->device;
    c->loop = g;
    *out = c;
    return DDG_OK;
}

extern "C" int ddg_get_unique_id(void* id128) {
    if (!id128) return set_err(DDG_E_ARG, "null id");
    int st = load_nccl();
    if (st) return st;
    ncclUniqueId id;
    NCCL_TRY(g_nccl.getUniqueId(&id));
    memcpy(id128, &id, sizeof id);
    return DDG_OK;
}

extern "C" int ddg_comm_init(int rank, int nranks, const void* id128, int device, ddg_comm** out) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return set_err(DDG_E_ARG, "ddg_comm_init: bad argument");
    *out = nullptr;
    int st = load_nccl();
    if (st) return st;
    CUDA_TRY(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ddg_comm* c = new ddg_comm();
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    ncclResult_t r = g_nccl.commInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return set_err(DDG_E_NCCL, "ncclCommInitRank: %s", g_nccl.errStr(r));
    }
    *out = c;
    return DDG_OK;
}

extern "C" void ddg_comm_destroy(ddg_comm* c) {
    if (!c) return;
    if (c->comm && g_nccl.commDestroy) g_nccl.commDestroy(c->comm);
    delete c;
}

namespace ddg {

int comm_allreduce_sum(ddg_comm* c, const double* send, double* recv, size_t count, cudaStream_t st) {
    if (c->loop) return loop_collective(c, 1, send, recv, count, nullptr);
    NCCL_TRY(g_nccl.allReduce(send, recv, count, ncclFloat64, ncclSum, c->comm, st));
    return DDG_OK;
}

int comm_exchange(ddg_comm* c, const Halo& h, cudaStream_t st) {
    if (c->loop) return loop_collective(c, 2, nullptr, nullptr, 0, &h);   // every rank arrives
    if (h.send_total == 0 && h.recv_total == 0) return DDG_OK;
    NCCL_TRY(g_nccl.groupStart());
    ncclResult_t err = ncclSuccess;
    for (int p = 0; p < c->nranks && err == ncclSuccess; ++p) {
        const int64_t ns = h.send_off[p + 1] - h.send_off[p];
        const int64_t nr = h.recv_off[p + 1] - h.recv_off[p];
        if (ns > 0) err = g_nccl.send(h.d_sbuf + h.send_off[p], ns, ncclFloat64, p, c->comm, st);
        if (nr > 0 && err == ncclSuccess) err = g_nccl.recv(h.d_rbuf + h.recv_off[p], nr, ncclFloat64, p, c->comm, st);
    }
    const ncclResult_t e2 = g_nccl.groupEnd();        // close the group even after a failed call
    if (err != ncclSuccess) return set_err(DDG_E_NCCL, "ncclSend/ncclRecv: %s", g_nccl.errStr(err));
    if (e2 != ncclSuccess) return set_err(DDG_E_NCCL, "ncclGroupEnd: %s", g_nccl.errStr(e2));
    return DDG_OK;
}

}  // namespace ddg
