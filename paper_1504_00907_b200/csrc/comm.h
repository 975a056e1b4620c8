// comm.h — NCCL communicator and halo exchange plans (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "nccl.h"

struct ddg_loop_group;

struct ddg_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, device = 0;
    ddg_loop_group* loop = nullptr;   // loopback: virtual ranks of one process on one device
};

namespace ddg {

// Loopback group (include/ddg.h ddg_loop_group_create): nranks virtual ranks,
// one host thread each, every context on the group's single stream.  A
// collective is a host rendezvous of all ranks; the last rank to arrive
// enqueues the data movement (device copies, a fixed-order sum kernel) on the
// shared stream, after every rank's preceding work and before any rank's
// following work.  No kernel ever waits on another.
cudaStream_t loop_stream(ddg_comm* c);
// out[i] = sum_{r < n} ptrs[r][i] in rank order (pcg.cu)
void launch_loop_sum(cudaStream_t st, const double* const* ptrs, int n, double* out, int64_t count);

// One exchange: this rank packs vec[send_idx] per peer, sends, receives and
// unpacks into vec[recv_idx].  Index lists concatenated over peers.
struct Halo {
    std::vector<int64_t> send_off, recv_off;   // nranks + 1
    int64_t send_total = 0, recv_total = 0;
    int32_t* d_sidx = nullptr;
    int32_t* d_ridx = nullptr;
    double* d_sbuf = nullptr;
    double* d_rbuf = nullptr;
};

int comm_allreduce_sum(ddg_comm* c, const double* send, double* recv, size_t count, cudaStream_t st);
int comm_exchange(ddg_comm* c, const Halo& h, cudaStream_t st);

}  // namespace ddg
