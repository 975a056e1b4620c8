// comm.h — NCCL communicator and halo exchange plans (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "nccl.h"

struct ddg_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, device = 0;
};

namespace ddg {

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
