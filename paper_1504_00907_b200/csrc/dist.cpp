// dist.cpp — host-side decomposition plan for running the DDG-PCG path on
// several GPUs.  Pure integer work, no device: it is used
// by ddg_setup when a communicator is given, and exported through the
// ddg_plan_* entry points so that tests can check it on the CPU.
//
// Model (correct by construction):
//  * parts are assigned to ranks (geometric boxes of the block grid when
//    block coordinates are known, contiguous balanced id ranges otherwise);
//    a rank owns the rows of its parts and the overlapping subdomains built
//    on them;
//  * every rank keeps full-length vectors but only computes on what it owns;
//  * after every step that writes a vector another rank reads, the written
//    values are sent to exactly the ranks that read them:
//      p   after the direction update   -> readers for A p  (cols of owned rows)
//      r   after the residual update    -> readers for R~_i r (rows of owned subdomains)
//      z   after every colour step      -> readers of z (neighbourhoods of owned
//                                          subdomains and of owned rows, owned rows)
//    Within a colour every row is written by at most one subdomain, so the
//    exchange overwrites (no summation), and a rank's view of every vector it
//    reads equals the single-GPU one;
//  * the coarse right-hand side is summed over ranks (allreduce of a
//    zero-padded n_c vector), the coarse solve is replicated, and every rank
//    prolongates all parts that touch rows it reads.
#include <algorithm>
#include <numeric>
#include <vector>

#include "dist.h"

namespace ddg {

static void assign_ranks_geom(const std::vector<int32_t>& idx, const int32_t* coords, int ndim, int r0,
                              int nr, std::vector<int32_t>& out) {
    if (nr == 1 || idx.size() <= 1) {
        for (int32_t b : idx) out[b] = r0;
        return;
    }
    int axis = 0;
    int32_t best = -1;
    for (int d = 0; d < ndim; ++d) {
        int32_t lo = INT32_MAX, hi = INT32_MIN;
        for (int32_t b : idx) {
            lo = std::min(lo, coords[(int64_t)b * ndim + d]);
            hi = std::max(hi, coords[(int64_t)b * ndim + d]);
        }
        if (hi - lo > best) { best = hi - lo; axis = d; }
    }
    std::vector<int32_t> s(idx);
    std::stable_sort(s.begin(), s.end(), [&](int32_t a, int32_t b) {
        const int32_t ca = coords[(int64_t)a * ndim + axis], cb = coords[(int64_t)b * ndim + axis];
        return ca != cb ? ca < cb : a < b;
    });
    const int nl = nr / 2;
    size_t cut = s.size() * nl / nr;
    // keep whole slabs together when possible (cut on a coordinate change)
    while (cut > 0 && cut < s.size() &&
           coords[(int64_t)s[cut] * ndim + axis] == coords[(int64_t)s[cut - 1] * ndim + axis]) {
        size_t up = cut, dn = cut;
        while (up < s.size() && coords[(int64_t)s[up] * ndim + axis] == coords[(int64_t)s[cut - 1] * ndim + axis]) ++up;
        while (dn > 0 && coords[(int64_t)s[dn - 1] * ndim + axis] == coords[(int64_t)s[cut] * ndim + axis]) --dn;
        const size_t ideal = s.size() * nl / nr;
        cut = (up - ideal <= ideal - dn) ? up : dn;
        if (cut == 0 || cut == s.size()) cut = ideal;
        break;
    }
    std::vector<int32_t> L(s.begin(), s.begin() + cut), R(s.begin() + cut, s.end());
    assign_ranks_geom(L, coords, ndim, r0, nl, out);
    assign_ranks_geom(R, coords, ndim, r0 + nl, nr - nl, out);
}

int build_dist_plan(DistPlan& P, int64_t n, const int64_t* rp, const int32_t* col, const int32_t* part,
                    int32_t nparts, const int64_t* bptr, const int32_t* bidx, const int64_t* optr,
                    const int32_t* oidx, const int32_t* colour, int ncolours, const int32_t* block_coords,
                    int block_ndim, int rank, int nranks) {
    P.rank = rank;
    P.nranks = nranks;
    P.ncolours = ncolours;
    P.part_rank.assign(nparts, 0);
    if (nranks > 1) {
        if (block_coords && block_ndim > 0) {
            std::vector<int32_t> all(nparts);
            std::iota(all.begin(), all.end(), 0);
            assign_ranks_geom(all, block_coords, block_ndim, 0, nranks, P.part_rank);
        } else {
            // contiguous id ranges balanced by row count
            int64_t acc = 0;
            for (int32_t I = 0; I < nparts; ++I) {
                const int64_t mI = bptr[I + 1] - bptr[I];
                P.part_rank[I] = (int32_t)std::min<int64_t>(nranks - 1, (acc + mI / 2) * nranks / n);
                acc += mI;
            }
        }
    }
    auto row_rank = [&](int64_t v) { return P.part_rank[part[v]]; };
    // owned rows (natural order), owned subdomains (ids), counts per rank
    P.owned_rows.clear();
    P.rows_per_rank.assign(nranks, 0);
    for (int64_t v = 0; v < n; ++v) {
        const int r = row_rank(v);
        P.rows_per_rank[r]++;
        if (r == rank) P.owned_rows.push_back((int32_t)v);
    }
    P.owned_subs.clear();
    for (int32_t i = 0; i < nparts; ++i)
        if (P.part_rank[i] == rank) P.owned_subs.push_back(i);
    // read sets (stamp arrays per rank would be n*nranks; build per reader h)
    std::vector<int32_t> stamp_p(n, -1), stamp_r(n, -1), stamp_z(n, -1);
    P.p_send.assign(nranks, {});
    P.p_recv.assign(nranks, {});
    P.r_send.assign(nranks, {});
    P.r_recv.assign(nranks, {});
    P.z_send.assign((size_t)ncolours * nranks, {});
    P.z_recv.assign((size_t)ncolours * nranks, {});
    P.prolong_parts.clear();
    std::vector<char> part_needed(nparts, 0);
    for (int h = 0; h < nranks; ++h) {
        // mark the rows h reads
        for (int64_t v = 0; v < n; ++v) {
            if (row_rank(v) != h) continue;
            stamp_z[v] = h;                                  // rho' = r^T z on owned rows
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                stamp_p[col[e]] = h;                         // q = A p on owned rows
                stamp_z[col[e]] = h;                         // coarse restriction reads z at cols
            }
        }
        for (int32_t i = 0; i < nparts; ++i) {
            if (P.part_rank[i] != h) continue;
            for (int64_t a = optr[i]; a < optr[i + 1]; ++a) {
                const int32_t v = oidx[a];
                stamp_r[v] = h;                              // gather reads r on Omega~_i
                for (int64_t e = rp[v]; e < rp[v + 1]; ++e) stamp_z[col[e]] = h;  // and z on N[Omega~_i]
            }
        }
        if (h == rank) {
            for (int64_t v = 0; v < n; ++v)
                if (stamp_z[v] == h) part_needed[part[v]] = 1;
        }
        // sends g -> h for vectors owned/written by g
        for (int g = 0; g < nranks; ++g) {
            if (g == h) continue;
            const bool mine_send = (g == rank), mine_recv = (h == rank);
            if (!mine_send && !mine_recv) continue;
            std::vector<int32_t> lp, lr;
            for (int64_t v = 0; v < n; ++v) {
                if (row_rank(v) != g) continue;
                if (stamp_p[v] == h) lp.push_back((int32_t)v);
                if (stamp_r[v] == h) lr.push_back((int32_t)v);
            }
            if (mine_send) { P.p_send[h] = lp; P.r_send[h] = lr; }
            if (mine_recv) { P.p_recv[g] = lp; P.r_recv[g] = lr; }
            // z written by g in colour c: Omega~_i of g's subdomains of colour c
            for (int c = 0; c < ncolours; ++c) {
                std::vector<int32_t> lz;
                for (int32_t i = 0; i < nparts; ++i) {
                    if (P.part_rank[i] != g || colour[i] != c) continue;
                    for (int64_t a = optr[i]; a < optr[i + 1]; ++a)
                        if (stamp_z[oidx[a]] == h) lz.push_back(oidx[a]);
                }
                std::sort(lz.begin(), lz.end());
                if (mine_send) P.z_send[(size_t)c * nranks + h] = lz;
                if (mine_recv) P.z_recv[(size_t)c * nranks + g] = lz;
            }
        }
    }
    for (int32_t I = 0; I < nparts; ++I)
        if (part_needed[I] || P.part_rank[I] == rank) P.prolong_parts.push_back(I);
    return 0;
}

}  // namespace ddg
