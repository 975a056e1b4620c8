// comm.cpp — NCCL communicator of libddg.  NCCL is loaded
// with dlopen (the copy torch ships, or the system one), so libddg itself
// loads and runs single-GPU without it.
#include <dlfcn.h>
#include <stdio.h>
#include <string.h>

#include <string>

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
    NCCL_TRY(g_nccl.allReduce(send, recv, count, ncclFloat64, ncclSum, c->comm, st));
    return DDG_OK;
}

int comm_exchange(ddg_comm* c, const Halo& h, cudaStream_t st) {
    if (h.send_total == 0 && h.recv_total == 0) return DDG_OK;
    NCCL_TRY(g_nccl.groupStart());
    for (int p = 0; p < c->nranks; ++p) {
        const int64_t ns = h.send_off[p + 1] - h.send_off[p];
        const int64_t nr = h.recv_off[p + 1] - h.recv_off[p];
        if (ns > 0) NCCL_TRY(g_nccl.send(h.d_sbuf + h.send_off[p], ns, ncclFloat64, p, c->comm, st));
        if (nr > 0) NCCL_TRY(g_nccl.recv(h.d_rbuf + h.recv_off[p], nr, ncclFloat64, p, c->comm, st));
    }
    NCCL_TRY(g_nccl.groupEnd());
    return DDG_OK;
}

}  // namespace ddg
