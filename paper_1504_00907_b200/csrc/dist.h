// dist.h — multi-GPU decomposition plan (dist.cpp), internal.
#pragma once
#include <stdint.h>

#include <vector>

namespace ddg {

struct DistPlan {
    int rank = 0, nranks = 1, ncolours = 0;
    std::vector<int32_t> part_rank;                    // owner rank of every part / subdomain
    std::vector<int64_t> rows_per_rank;
    std::vector<int32_t> owned_rows;                   // natural numbering, increasing
    std::vector<int32_t> owned_subs;                   // subdomain (part) ids owned here
    std::vector<std::vector<int32_t>> p_send, p_recv;  // [peer] row lists (send: owned rows)
    std::vector<std::vector<int32_t>> r_send, r_recv;
    std::vector<std::vector<int32_t>> z_send, z_recv;  // [colour * nranks + peer]
    std::vector<int32_t> prolong_parts;                // parts whose rows this rank reads or owns
};

int build_dist_plan(DistPlan& P, int64_t n, const int64_t* rp, const int32_t* col, const int32_t* part,
                    int32_t nparts, const int64_t* bptr, const int32_t* bidx, const int64_t* optr,
                    const int32_t* oidx, const int32_t* colour, int ncolours, const int32_t* block_coords,
                    int block_ndim, int rank, int nranks);

}  // namespace ddg
