// coarse_sparse.cpp — sparse direct solve of the DDG coarse system
// A_c y = b_c, exploiting its block sparsity: "the same
// sparsity pattern as the subdomain adjacency matrix, but with each non-zero
// replaced with a small dense block".
//
// Symbolic (host): nested dissection of the part-adjacency graph (geometric
// bisection when block coordinates are given, BFS level-set bisection
// otherwise; every cut is verified to separate), supernodes = separators and
// leaf boxes, boundary sets B_t = ancestor unknowns coupled to the subtree.
// Numeric (device, level by level from the leaves): each front [S_t | B_t] is
// assembled from A_c entries and the children's Schur complements
// (extend-add), then the S_t pivots are eliminated by block Gauss-Jordan
// exchange, which leaves H_t = A_SS^{-1}, G_t = A_BS A_SS^{-1} and the Schur
// complement A_BB - A_BS A_SS^{-1} A_SB for the parent.
// Solve (device): forward w_t = inc_B - G_t b_S (leaves to root), backward
// x_S = H_t b_S - G_t^T x_B (root to leaves), each level one tiled SYMV launch
// over the operator K_t = [[H_t, .], [-G_t, 0]] plus gather/reduce launches.
// Bytes per solve: 2|G| + |H| (H packed lower) -- below the 2|L_c| of
// Cholesky forward/back substitution.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <numeric>

#include "ctx.h"
#include "comm.h"

namespace {

// Tunables of one symbolic phase, per call (not globals: contexts are set up
// concurrently by the loopback ranks' threads, and a global reset to its default
// in one thread was seen by another's tree builder -- different trees per rank)
constexpr int64_t MERGE_MAX = 12288; // merged top separators stay below this many unknowns

struct NDNode {
    std::vector<int32_t> sep;  // blocks eliminated at this node
    std::vector<int> child;    // children in elimination order (2 from a bisection, more when merged)
    int parent = -1;
    int height = 0;
};

}  // namespace

struct SparseCoarse {
    int nfront = 0, nlevels = 0;
    std::vector<FrontDesc> fr;
    std::vector<int32_t> fS, fB, fmap, fchild;
    std::vector<int> lb;                       // fronts of level h: [lb[h], lb[h+1])
    std::vector<int> g_begin, g_end, h_begin, h_end;
    std::vector<int> fwd_b, bwd_b;             // task ranges per level (size nlevels+1)
    std::vector<int> ring_fwd, ring_bwd;       // k_symv_ring partitions per level (-1: none)
    // dataflow solve (k_coarse_dataflow): work queue, per-front schedule, state
    std::vector<int32_t> dfwork;
    std::vector<FrontDF> fdf;
    int32_t *d_dfwork = nullptr, *d_dfstate = nullptr;
    FrontDF* d_fdf = nullptr;
    bool dataflow = true;
    uint64_t* d_trace = nullptr;                // DDG_DF_TRACE: per-entry timestamps (debug)
    std::vector<FRedTask> fwd, bwd;
    std::vector<int64_t> contrib;
    std::vector<int32_t> item_front;           // item (relative to item_base) -> front
    int item_base = 0, item_end = 0;
    int max_rows_t = 0;
    int64_t fvec_doubles = 0, w_doubles = 0, ctile_doubles = 0;
    // triplets per level (front-local row, col, value, front)
    std::vector<std::vector<int32_t>> tr_r, tr_c, tr_f;
    std::vector<std::vector<double>> tr_v;
    // device
    FrontDesc* d_fr = nullptr;
    int32_t *d_fS = nullptr, *d_fB = nullptr, *d_fmap = nullptr, *d_item_front = nullptr, *d_fchild = nullptr;
    FRedTask *d_fwd = nullptr, *d_bwd = nullptr;
    int64_t* d_contrib = nullptr;
    double *d_fvec = nullptr, *d_w = nullptr, *d_ctiles = nullptr, *d_bc = nullptr;
    int64_t factor_bytes = 0;
    // distributed solve (sparse_coarse_dist_setup): the top fronts replicated,
    // every subtree below them solved by one rank
    bool dist = false;
    int nw1 = 0, nw3 = 0;
    int64_t nwx = 0, rank_solve_bytes = 0;
    int32_t *d_work1 = nullptr, *d_work3 = nullptr, *d_wx_idx = nullptr;
    uint8_t *d_wx_mask = nullptr, *d_y_mask = nullptr;
    FrontDesc* d_fr1 = nullptr;
    double *d_wx_buf = nullptr, *d_y_buf = nullptr;
    int ntop = 0, nsub = 0;
    // the top fronts' work split over the ranks (phase 2):
    // per front its G and H item ranges and reduction tasks; a rank computes its
    // share of every range, the partial segments are allreduced, the reductions
    // run everywhere
    struct Top { int f, depth, g0, g1, h0, h1, ft0, ft1, bt0, bt1; };
    std::vector<Top> tops;          // deepest first
    std::vector<int> own_roots;     // this rank's subtree roots
};

int64_t sparse_coarse_solve_bytes(ddg_ctx* c);

void sparse_coarse_free(SparseCoarse* s) {
    if (!s) return;
    void* p[] = {s->d_fr, s->d_fchild, s->d_fS, s->d_fB, s->d_fmap, s->d_item_front, s->d_fwd, s->d_bwd,
                 s->d_contrib, s->d_fvec, s->d_w, s->d_ctiles, s->d_bc, s->d_dfwork, s->d_dfstate, s->d_fdf,
                 s->d_trace, s->d_work1, s->d_work3,
                 s->d_wx_idx, s->d_wx_mask, s->d_y_mask, s->d_fr1, s->d_wx_buf, s->d_y_buf};
    for (void* x : p)
        if (x) cudaFree(x);
    delete s;
}

// --------------------------------------------------------------------------
// nested dissection of the part-adjacency graph
// --------------------------------------------------------------------------
namespace {

struct NDBuilder {
    const std::vector<std::vector<int32_t>>& adj;
    const std::vector<int32_t>& rank;
    const int32_t* coords;
    int ndim;
    std::vector<NDNode> nodes;
    std::vector<int32_t> mark;   // 0 none, 1 L, 2 R, 3 S, 4 in V (scratch)
    std::vector<int32_t> lev;

    int64_t leaf_unknowns = 256;   // nested dissection stops below this many unknowns (DDG_ND_LEAF)

    NDBuilder(const std::vector<std::vector<int32_t>>& a, const std::vector<int32_t>& r,
              const int32_t* co, int nd, int64_t leaf)
        : adj(a), rank(r), coords(co), ndim(nd), mark(a.size(), 0), lev(a.size(), -1), leaf_unknowns(leaf) {}

    int64_t unknowns(const std::vector<int32_t>& V) const {
        int64_t s = 0;
        for (int32_t v : V) s += rank[v];
        return s;
    }

    bool split_geom(const std::vector<int32_t>& V, std::vector<int32_t>& L, std::vector<int32_t>& R,
                    std::vector<int32_t>& S) {
        if (!coords) return false;
        int axis = -1;
        int32_t best = 0;
        for (int d = 0; d < ndim; ++d) {
            int32_t lo = INT32_MAX, hi = INT32_MIN;
            for (int32_t v : V) {
                lo = std::min(lo, coords[(int64_t)v * ndim + d]);
                hi = std::max(hi, coords[(int64_t)v * ndim + d]);
            }
            if (hi - lo > best) { best = hi - lo; axis = d; }
        }
        if (axis < 0) return false;
        std::vector<int32_t> vals;
        vals.reserve(V.size());
        for (int32_t v : V) vals.push_back(coords[(int64_t)v * ndim + axis]);
        std::nth_element(vals.begin(), vals.begin() + vals.size() / 2, vals.end());
        const int32_t m = vals[vals.size() / 2];
        L.clear(); R.clear(); S.clear();
        for (int32_t v : V) {
            const int32_t x = coords[(int64_t)v * ndim + axis];
            if (x < m) L.push_back(v); else if (x > m) R.push_back(v); else S.push_back(v);
        }
        if (L.empty() || R.empty()) return false;
        fix_separation(L, R, S);
        return true;
    }

    // move every R endpoint of an L-R edge into S
    void fix_separation(std::vector<int32_t>& L, std::vector<int32_t>& R, std::vector<int32_t>& S) {
        for (int32_t v : L) mark[v] = 1;
        for (int32_t v : R) mark[v] = 2;
        for (int32_t v : S) mark[v] = 3;
        for (int32_t v : L)
            for (int32_t u : adj[v])
                if (mark[u] == 2) mark[u] = 3;
        std::vector<int32_t> R2;
        for (int32_t v : R) {
            if (mark[v] == 3) S.push_back(v); else R2.push_back(v);
        }
        R.swap(R2);
        for (int32_t v : L) mark[v] = 0;
        for (int32_t v : R) mark[v] = 0;
        for (int32_t v : S) mark[v] = 0;
    }

    // BFS level-structure bisection from a pseudo-peripheral node (induced subgraph)
    void split_bfs(const std::vector<int32_t>& V, std::vector<int32_t>& L, std::vector<int32_t>& R,
                   std::vector<int32_t>& S) {
        for (int32_t v : V) mark[v] = 4;
        auto bfs = [&](int32_t s, std::vector<int32_t>& order) {
            order.clear();
            for (int32_t v : V) lev[v] = -1;
            lev[s] = 0;
            order.push_back(s);
            for (size_t h = 0; h < order.size(); ++h) {
                int32_t v = order[h];
                for (int32_t u : adj[v])
                    if (mark[u] == 4 && lev[u] < 0) { lev[u] = lev[v] + 1; order.push_back(u); }
            }
        };
        std::vector<int32_t> order;
        bfs(V[0], order);
        bfs(order.back(), order);
        const int maxlev = lev[order.back()];
        std::vector<int64_t> cnt(maxlev + 2, 0);
        for (int32_t v : order) cnt[lev[v]]++;
        int64_t cum = 0;
        int cut = 0;
        for (int l = 0; l <= maxlev; ++l) {
            cum += cnt[l];
            if (cum * 2 > (int64_t)V.size()) { cut = l; break; }
        }
        if (cut == 0 && maxlev >= 1) cut = 1;
        L.clear(); R.clear(); S.clear();
        for (int32_t v : V) {
            if (lev[v] < 0) R.push_back(v);          // other components
            else if (lev[v] < cut) L.push_back(v);
            else if (lev[v] == cut) S.push_back(v);
            else R.push_back(v);
        }
        for (int32_t v : V) { mark[v] = 0; lev[v] = -1; }
    }

    int build(std::vector<int32_t> V) {
        const int id = (int)nodes.size();
        nodes.emplace_back();
        if (V.size() <= 1 || unknowns(V) <= leaf_unknowns) {
            std::sort(V.begin(), V.end());
            nodes[id].sep = std::move(V);
            return id;
        }
        std::vector<int32_t> L, R, S;
        if (!split_geom(V, L, R, S)) split_bfs(V, L, R, S);
        if (S.empty() && (L.empty() || R.empty())) {
            std::sort(V.begin(), V.end());
            nodes[id].sep = std::move(V);
            return id;
        }
        if (S.empty()) {          // disconnected halves: eliminate one block here
            S.push_back(R.back());
            R.pop_back();
        }
        std::sort(S.begin(), S.end());
        nodes[id].sep = S;
        for (auto* part : {&L, &R}) {
            if (part->empty()) continue;
            int ch = build(std::move(*part));
            nodes[id].child.push_back(ch);
            nodes[ch].parent = id;
        }
        return id;
    }

    // The top `levels` bisections merged into one root front: its separator is
    // the union of theirs and the remaining regions are its children.  One
    // dense front replaces `levels` sequential steps of the solve's critical
    // path at the top of the tree, where the fronts are few and small.
    int build_top(std::vector<int32_t> V, int levels) {
        if (levels <= 0) return build(std::move(V));
        const int id = (int)nodes.size();
        nodes.emplace_back();
        std::vector<std::vector<int32_t>> frontier, finals;
        std::vector<int32_t> seps;
        frontier.push_back(std::move(V));
        for (int l = 0; l < levels && !frontier.empty(); ++l) {
            if (l > 0 && unknowns(seps) >= MERGE_MAX) break;
            std::vector<std::vector<int32_t>> next;
            for (auto& R0 : frontier) {
                if (R0.size() <= 1 || unknowns(R0) <= leaf_unknowns) { finals.push_back(std::move(R0)); continue; }
                std::vector<int32_t> L, R, S;
                if (!split_geom(R0, L, R, S)) split_bfs(R0, L, R, S);
                if (S.empty() && (L.empty() || R.empty())) { finals.push_back(std::move(R0)); continue; }
                if (S.empty()) {
                    S.push_back(R.back());
                    R.pop_back();
                }
                seps.insert(seps.end(), S.begin(), S.end());
                if (!L.empty()) next.push_back(std::move(L));
                if (!R.empty()) next.push_back(std::move(R));
            }
            frontier.swap(next);
        }
        for (auto& R0 : frontier) finals.push_back(std::move(R0));
        std::sort(seps.begin(), seps.end());
        nodes[id].sep = seps;
        for (auto& R0 : finals) {
            const int ch = build(std::move(R0));
            nodes[id].child.push_back(ch);
            nodes[ch].parent = id;
        }
        return id;
    }
};

}  // namespace

// --------------------------------------------------------------------------
// symbolic phase: fronts, items, reduction tasks, triplets
// --------------------------------------------------------------------------
int sparse_coarse_symbolic(ddg_ctx* c, const int64_t* rp, const int32_t* col,
                           const std::vector<int32_t>& er, const std::vector<int32_t>& ec,
                           const std::vector<double>& ev) {
    const int np = c->nparts;
    SparseCoarse* sc = new SparseCoarse();
    c->sparse = sc;
    int FRONT_BT = 8;   // tiles per item side of the front operators (DDG_FRONT_BT)
    if (const char* e = getenv("DDG_FRONT_BT")) FRONT_BT = std::max(1, std::min(8, atoi(e)));
    // small coarse systems (C2, C5): bigger leaves, fewer levels on the solve's
    // critical path; large ones (C3): smaller leaves, fewer bytes (measured)
    int64_t leaf = c->nc <= 262144 ? 1024 : 256;
    if (const char* e = getenv("DDG_ND_LEAF")) leaf = std::max(16, atoi(e));
    int MERGE_LEVELS = 0;   // top bisection levels merged into the root front (DDG_ND_MERGE)
    if (const char* e = getenv("DDG_ND_MERGE")) MERGE_LEVELS = std::max(0, atoi(e));
    // part adjacency
    std::vector<std::vector<int32_t>> adj(np);
    parallel_for(np, [&](int64_t b, int64_t e2, int) {
        for (int64_t I = b; I < e2; ++I) {
            auto& a = adj[I];
            for (int64_t x = c->bptr[I]; x < c->bptr[I + 1]; ++x) {
                const int32_t v = c->bidx[x];
                for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                    const int32_t J = c->part[col[e]];
                    if (J != (int32_t)I) a.push_back(J);
                }
            }
            std::sort(a.begin(), a.end());
            a.erase(std::unique(a.begin(), a.end()), a.end());
        }
    });
    std::vector<int32_t> rank(np);
    for (int I = 0; I < np; ++I) rank[I] = c->cptr[I + 1] - c->cptr[I];
    NDBuilder nd(adj, rank, c->block_coords.empty() ? nullptr : c->block_coords.data(), c->block_ndim, leaf);
    // one tree per connected component of the part graph
    {
        std::vector<int32_t> comp(np, -1);
        std::vector<int32_t> stack;
        for (int s = 0; s < np; ++s) {
            if (comp[s] >= 0) continue;
            std::vector<int32_t> V{s};
            comp[s] = s;
            stack.assign(1, s);
            while (!stack.empty()) {
                int32_t v = stack.back();
                stack.pop_back();
                for (int32_t u : adj[v])
                    if (comp[u] < 0) { comp[u] = s; V.push_back(u); stack.push_back(u); }
            }
            nd.build_top(std::move(V), MERGE_LEVELS);
        }
    }
    auto& nodes = nd.nodes;
    const int nn = (int)nodes.size();
    // postorder, heights, Euler intervals
    std::vector<int> post;
    std::vector<int> tin(nn), tout(nn);
    {
        int timer = 0;
        std::function<void(int)> dfs = [&](int t) {
            tin[t] = timer++;
            for (int ch : nodes[t].child) dfs(ch);
            int h = 0;
            for (int ch : nodes[t].child) h = std::max(h, nodes[ch].height + 1);
            nodes[t].height = h;
            post.push_back(t);
            tout[t] = timer++;
        };
        for (int t = 0; t < nn; ++t)
            if (nodes[t].parent < 0) dfs(t);
    }
    std::vector<int> postidx(nn);
    for (int i = 0; i < nn; ++i) postidx[post[i]] = i;
    auto is_anc = [&](int a, int b) { return tin[a] <= tin[b] && tout[b] <= tout[a]; };  // a ancestor-or-self of b
    std::vector<int32_t> snode(np, -1);
    for (int t = 0; t < nn; ++t)
        for (int32_t b : nodes[t].sep) snode[b] = t;
    // boundary block sets, bottom-up
    std::vector<std::vector<int32_t>> Bblk(nn);
    for (int t : post) {
        std::vector<int32_t> cand;
        for (int32_t b : nodes[t].sep) cand.insert(cand.end(), adj[b].begin(), adj[b].end());
        for (int ch : nodes[t].child) {
            const auto& cb = Bblk[ch];
            cand.insert(cand.end(), cb.begin(), cb.end());
        }
        std::vector<int32_t> keep;
        for (int32_t u : cand) {
            const int su = snode[u];
            if (su != t && is_anc(su, t)) keep.push_back(u);
        }
        std::sort(keep.begin(), keep.end(), [&](int32_t a, int32_t b) {
            return postidx[snode[a]] != postidx[snode[b]] ? postidx[snode[a]] < postidx[snode[b]] : a < b;
        });
        keep.erase(std::unique(keep.begin(), keep.end()), keep.end());
        Bblk[t] = std::move(keep);
    }
    // fronts ordered by (height, postorder)
    std::vector<int> order(nn);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        return nodes[a].height != nodes[b].height ? nodes[a].height < nodes[b].height : postidx[a] < postidx[b];
    });
    std::vector<int> fid(nn);
    for (int i = 0; i < nn; ++i) fid[order[i]] = i;
    sc->nfront = nn;
    sc->nlevels = nn ? nodes[order.back()].height + 1 : 0;
    sc->lb.assign(sc->nlevels + 1, 0);
    for (int i = 0; i < nn; ++i) sc->lb[nodes[order[i]].height + 1]++;
    for (int h = 0; h < sc->nlevels; ++h) sc->lb[h + 1] += sc->lb[h];
    sc->fr.assign(nn, FrontDesc{});
    for (int i = 0; i < nn; ++i) {
        const int t = order[i];
        FrontDesc& f = sc->fr[i];
        f.parent = nodes[t].parent >= 0 ? fid[nodes[t].parent] : -1;
        f.child_off = (int32_t)sc->fchild.size();
        f.nchild = (int32_t)nodes[t].child.size();
        for (int ch : nodes[t].child) sc->fchild.push_back(fid[ch]);
        f.S_off = (int64_t)sc->fS.size();
        for (int32_t b : nodes[t].sep)
            for (int32_t q = c->cptr[b]; q < c->cptr[b + 1]; ++q) sc->fS.push_back(q);
        f.nS = (int32_t)(sc->fS.size() - f.S_off);
        f.B_off = (int64_t)sc->fB.size();
        for (int32_t b : Bblk[t])
            for (int32_t q = c->cptr[b]; q < c->cptr[b + 1]; ++q) sc->fB.push_back(q);
        f.nB = (int32_t)(sc->fB.size() - f.B_off);
        f.nSp = ((f.nS + TILE - 1) / TILE) * TILE;
        const int nBp = ((f.nB + TILE - 1) / TILE) * TILE;
        f.nK = f.nSp / TILE;
        f.nT = (f.nSp + nBp) / TILE;
        f.fvec_off = sc->fvec_doubles;
        sc->fvec_doubles += (int64_t)f.nT * TILE;
        f.w_off = sc->w_doubles;
        sc->w_doubles += f.nB;
        f.map_off = -1;
    }
    // child -> parent position maps
    std::vector<int32_t> pos(c->nc, -1);
    for (int i = 0; i < nn; ++i) {
        FrontDesc& p = sc->fr[i];
        for (int a = 0; a < p.nS; ++a) pos[sc->fS[p.S_off + a]] = a;
        for (int j = 0; j < p.nB; ++j) pos[sc->fB[p.B_off + j]] = p.nSp + j;
        for (int k = 0; k < p.nchild; ++k) {
            const int ci = sc->fchild[p.child_off + k];
            FrontDesc& ch = sc->fr[ci];
            ch.map_off = (int64_t)sc->fmap.size();
            for (int j = 0; j < ch.nB; ++j) {
                const int32_t q = sc->fB[ch.B_off + j];
                if (pos[q] < 0) {
                    delete sc;
                    c->sparse = nullptr;
                    return set_err(DDG_E_COLOURING, "sparse coarse: boundary unknown %d of front %d not in parent", q, ci);
                }
                sc->fmap.push_back(pos[q]);
            }
        }
        for (int a = 0; a < p.nS; ++a) pos[sc->fS[p.S_off + a]] = -1;
        for (int j = 0; j < p.nB; ++j) pos[sc->fB[p.B_off + j]] = -1;
    }
    // A_c entries -> the front eliminated first (the deeper supernode)
    std::vector<int32_t> cblock(c->nc);
    for (int I = 0; I < np; ++I)
        for (int32_t q = c->cptr[I]; q < c->cptr[I + 1]; ++q) cblock[q] = I;
    std::vector<std::vector<int64_t>> byfront(nn);
    for (size_t e = 0; e < ev.size(); ++e) {
        const int tr = snode[cblock[er[e]]], tc = snode[cblock[ec[e]]];
        const int t = is_anc(tc, tr) ? tr : tc;   // descendant-or-self
        byfront[fid[t]].push_back((int64_t)e);
    }
    sc->tr_r.assign(sc->nlevels, {});
    sc->tr_c.assign(sc->nlevels, {});
    sc->tr_f.assign(sc->nlevels, {});
    sc->tr_v.assign(sc->nlevels, {});
    for (int i = 0; i < nn; ++i) {
        const FrontDesc& f = sc->fr[i];
        const int h = nodes[order[i]].height;
        for (int a = 0; a < f.nS; ++a) pos[sc->fS[f.S_off + a]] = a;
        for (int j = 0; j < f.nB; ++j) pos[sc->fB[f.B_off + j]] = f.nSp + j;
        for (int64_t e : byfront[i]) {
            const int pr = pos[er[e]], pc = pos[ec[e]];
            if (pr < 0 || pc < 0) {
                delete sc;
                c->sparse = nullptr;
                return set_err(DDG_E_COLOURING, "sparse coarse: A_c entry (%d,%d) outside front %d", er[e], ec[e], i);
            }
            sc->tr_r[h].push_back(pr);
            sc->tr_c[h].push_back(pc);
            sc->tr_f[h].push_back(i);
            sc->tr_v[h].push_back(ev[e]);
        }
        for (int a = f.nS; a < f.nSp; ++a) {      // identity on the S padding
            sc->tr_r[h].push_back(a);
            sc->tr_c[h].push_back(a);
            sc->tr_f[h].push_back(i);
            sc->tr_v[h].push_back(1.0);
        }
        for (int a = 0; a < f.nS; ++a) pos[sc->fS[f.S_off + a]] = -1;
        for (int j = 0; j < f.nB; ++j) pos[sc->fB[f.B_off + j]] = -1;
    }
    // solve operators: ops + items (per level: all G items, then all H items)
    // Item block size per level: the largest of 8, 4, 2 tiles that still gives
    // the level ~2 work items per SM (upper levels have few, large fronts; in
    // the dataflow solve each item is one CTA on the critical path).
    std::vector<int> lvl_bt(sc->nlevels, FRONT_BT);
    if (!getenv("DDG_FRONT_BT")) {
        std::vector<double> lvl_tiles(sc->nlevels, 0.0);
        for (int i = 0; i < nn; ++i) {
            const FrontDesc& f = sc->fr[i];
            lvl_tiles[nodes[order[i]].height] += (double)f.nK * f.nT;   // S columns of the [S|B] front
        }
        for (int h = 0; h < sc->nlevels; ++h) {
            int bt = 8;
            while (bt > 2 && lvl_tiles[h] / ((double)bt * bt) < 2.0 * num_sms()) bt /= 2;
            lvl_bt[h] = bt;
        }
    }
    std::vector<std::vector<int>> rowblk(nn);   // row-block starts (tiles) per front
    for (int i = 0; i < nn; ++i) {
        FrontDesc& f = sc->fr[i];
        auto& rb = rowblk[i];
        const int bt = lvl_bt[nodes[order[i]].height];
        for (int t0 = 0; t0 < f.nK; t0 += bt) rb.push_back(t0);
        for (int t0 = f.nK; t0 < f.nT; t0 += bt) rb.push_back(t0);
        rb.push_back(f.nT);
        OpDesc op{};
        op.m = f.nS;
        op.mp = f.nT * TILE;
        op.nT = f.nT;
        op.BT = bt;
        op.nblk = (int)rb.size() - 1;
        op.out_mode = 2;
        op.idx_off = -1;
        op.s_off = f.fvec_off;
        op.part_off = 0;
        f.op = (int)c->ops.size();
        c->ops.push_back(op);
    }
    sc->item_base = (int)c->items.size();
    struct PendingItem { int front, bi, bj; };
    std::vector<std::vector<int>> item_of(nn);   // item index per (bi, bj) pair, row-major over all blocks
    auto nblkS = [&](int i) {
        int k = 0;
        for (size_t b = 0; b + 1 < rowblk[i].size(); ++b)
            if (rowblk[i][b] < sc->fr[i].nK) ++k;
        return k;
    };
    auto add_item = [&](int i, int bi, int bj) {
        const FrontDesc& f = sc->fr[i];
        const auto& rb = rowblk[i];
        ItemDesc it{};
        it.op = f.op;
        it.I0 = rb[bi];
        it.I1 = rb[bi + 1];
        it.J0 = rb[bj];
        it.J1 = rb[bj + 1];
        it.tri = (bi == bj);
        const int h = it.I1 - it.I0, wd = it.J1 - it.J0;
        it.ntiles = it.tri ? h * (h + 1) / 2 : h * wd;
        it.tile_off = sc->ctile_doubles;
        sc->ctile_doubles += item_doubles(it.tri, h, it.ntiles);
        it.part_off = c->part_doubles;
        c->part_doubles += (int64_t)(h + (it.tri ? 0 : wd)) * TILE;
        sc->max_rows_t = std::max(sc->max_rows_t, (h + (it.tri ? 0 : wd)) * TILE);
        item_of[i][bi * (rowblk[i].size() - 1) + bj] = (int)c->items.size();
        c->items.push_back(it);
        sc->item_front.push_back(i);
    };
    for (int i = 0; i < nn; ++i) item_of[i].assign((rowblk[i].size() - 1) * (rowblk[i].size() - 1), -1);
    sc->g_begin.assign(sc->nlevels, 0);
    sc->g_end.assign(sc->nlevels, 0);
    sc->h_begin.assign(sc->nlevels, 0);
    sc->h_end.assign(sc->nlevels, 0);
    for (int h = 0; h < sc->nlevels; ++h) {
        sc->g_begin[h] = (int)c->items.size();
        for (int i = sc->lb[h]; i < sc->lb[h + 1]; ++i) {
            const int nb = (int)rowblk[i].size() - 1, ns = nblkS(i);
            for (int bi = ns; bi < nb; ++bi)
                for (int bj = 0; bj < ns; ++bj) add_item(i, bi, bj);
        }
        sc->g_end[h] = sc->h_begin[h] = (int)c->items.size();
        for (int i = sc->lb[h]; i < sc->lb[h + 1]; ++i) {
            const int ns = nblkS(i);
            for (int bi = 0; bi < ns; ++bi)
                for (int bj = 0; bj <= bi; ++bj) add_item(i, bi, bj);
        }
        sc->h_end[h] = (int)c->items.size();
    }
    sc->item_end = (int)c->items.size();
    // reduction tasks
    sc->fdf.assign(nn, FrontDF{});
    sc->fwd_b.assign(sc->nlevels + 1, 0);
    sc->bwd_b.assign(sc->nlevels + 1, 0);
    for (int h = 0; h < sc->nlevels; ++h) {
        sc->fwd_b[h] = (int)sc->fwd.size();
        sc->bwd_b[h] = (int)sc->bwd.size();
        for (int i = sc->lb[h]; i < sc->lb[h + 1]; ++i) {
            const auto& rb = rowblk[i];
            const int nb = (int)rb.size() - 1, ns = nblkS(i);
            auto idx = [&](int bi, int bj) { return item_of[i][bi * nb + bj]; };
            sc->fdf[i].ft0 = (int)sc->fwd.size();
            sc->fdf[i].bt0 = (int)sc->bwd.size();
            for (int bi = ns; bi < nb; ++bi) {       // forward: rows in B
                FRedTask t{i, 0, rb[bi] * TILE, (rb[bi + 1] - rb[bi]) * TILE, (int)sc->contrib.size(), 0};
                for (int bj = 0; bj < ns; ++bj) sc->contrib.push_back(c->items[idx(bi, bj)].part_off);
                t.cend = (int)sc->contrib.size();
                sc->fwd.push_back(t);
            }
            for (int b = 0; b < ns; ++b) {            // backward: rows in S
                FRedTask t{i, 1, rb[b] * TILE, (rb[b + 1] - rb[b]) * TILE, (int)sc->contrib.size(), 0};
                for (int bj = 0; bj <= b; ++bj) sc->contrib.push_back(c->items[idx(b, bj)].part_off);
                for (int bi = b + 1; bi < nb; ++bi) {
                    const ItemDesc& it = c->items[idx(bi, b)];
                    sc->contrib.push_back(it.part_off + (int64_t)(it.I1 - it.I0) * TILE);
                }
                t.cend = (int)sc->contrib.size();
                sc->bwd.push_back(t);
            }
            sc->fdf[i].ft1 = (int)sc->fwd.size();
            sc->fdf[i].bt1 = (int)sc->bwd.size();
        }
    }
    sc->fwd_b[sc->nlevels] = (int)sc->fwd.size();
    sc->bwd_b[sc->nlevels] = (int)sc->bwd.size();
    sc->factor_bytes = sc->ctile_doubles * 8;
    // dataflow work queue: leaf assemblies, forward G items leaves -> root,
    // backward G + H items root -> leaves
    for (int h = 0; h < sc->nlevels; ++h)
        for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) {
            FrontDF& d = sc->fdf[sc->item_front[q - sc->item_base]];
            if (q < sc->g_end[h]) ++d.nG;
            ++d.nGH;
        }
    sc->dfwork.clear();
    for (int i = 0; i < nn; ++i)
        if (sc->fr[i].nchild == 0) sc->dfwork.push_back(DF_ASSEMBLE | i);
    for (int h = 0; h < sc->nlevels; ++h) {
        for (int q = sc->g_begin[h]; q < sc->g_end[h]; ++q) sc->dfwork.push_back(q);
        for (int k = sc->fwd_b[h]; k < sc->fwd_b[h + 1]; ++k) sc->dfwork.push_back(DF_RED | k);
    }
    for (int h = sc->nlevels - 1; h >= 0; --h) {
        for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) sc->dfwork.push_back(DF_BWD | q);
        for (int k = sc->bwd_b[h]; k < sc->bwd_b[h + 1]; ++k) sc->dfwork.push_back(DF_BWD | DF_RED | k);
    }
    if ((int64_t)c->items.size() >= DF_RED || (int64_t)sc->fwd.size() >= DF_RED || (int64_t)sc->bwd.size() >= DF_RED)
        sc->dataflow = false;   // entry indices must fit below the flag bits
    if (const char* e = getenv("DDG_COARSE_DATAFLOW")) sc->dataflow = atoi(e) != 0;
    if (getenv("DDG_DF_TRACE")) {
        if (cudaMalloc(&sc->d_trace, sc->dfwork.size() * 4 * sizeof(uint64_t)) != cudaSuccess) sc->d_trace = nullptr;
        else cudaMemset(sc->d_trace, 0, sc->dfwork.size() * 4 * sizeof(uint64_t));
    }
    sc->ring_fwd.assign(sc->nlevels, -1);
    sc->ring_bwd.assign(sc->nlevels, -1);
    for (int h = 0; h < sc->nlevels; ++h) {
        sc->ring_fwd[h] = ring_partition(c, sc->g_begin[h], sc->g_end[h]);
        sc->ring_bwd[h] = ring_partition(c, sc->g_begin[h], sc->h_end[h]);
    }
    return DDG_OK;
}

template <typename T>
static int up_s(cudaStream_t s, T** d, const std::vector<T>& h) {
    int st = dalloc(d, h.size());
    if (st) return st;
    return h2d(s, *d, h.data(), h.size() * sizeof(T));
}
#define up(d, h) up_s(c->stream, d, h)

// --------------------------------------------------------------------------
// distributed solve plan
// --------------------------------------------------------------------------
// The nested-dissection tree is cut at depth D = ceil(log2 P): the fronts
// above the cut (the top separators) are solved redundantly by every rank,
// every subtree below it by one rank (greedy by solve bytes).  One solve:
//   phase 1  forward elimination over this rank's subtrees (dataflow kernel;
//            the subtree roots stop there, as if they were roots)
//   exchange the subtree roots' contributions w_t to their top ancestors:
//            one allreduce of their concatenation (zeros from non-owners)
//   phase 2  forward + backward over the top fronts, front by front, each
//            front's G and H item ranges split over the ranks: a rank zeroes
//            the range's partial segments, computes its share (k_symv), the
//            segments are allreduced, the front's reductions run everywhere
//   phase 3  backward substitution over this rank's subtrees
//   y_c      one allreduce: each unknown contributed by exactly one rank (a
//            subtree's owner, rank 0 for the top), so every rank holds the
//            same y_c bitwise.
// Every partial segment and every y_c entry is computed by exactly one rank
// and the allreduces only add zeros, so the result equals the replicated
// solve bitwise.  The factor stays replicated in memory (the top fronts need
// every subtree's Schur complement at setup); each rank READS its subtrees and
// 1/P of the top fronts per solve, which is what bounds the coarse step.
struct DistSplit {
    std::vector<char> top, sroot;
    std::vector<int> owner, roots;
    std::vector<double> fbytes;
};
static void dist_split(ddg_ctx* c, int P, DistSplit& ds) {
    SparseCoarse* sc = c->sparse;
    const int nn = sc->nfront;
    std::vector<char>& top = ds.top;
    std::vector<char>& sroot = ds.sroot;
    std::vector<int>& owner = ds.owner;
    std::vector<int>& roots = ds.roots;
    std::vector<double>& fbytes = ds.fbytes;
    top.assign(nn, 0);
    sroot.assign(nn, 0);
    roots.clear();
    int D = 0;
    while ((1 << D) < P) ++D;
    std::vector<int> depth(nn, 0);
    for (int i = nn - 1; i >= 0; --i) depth[i] = sc->fr[i].parent < 0 ? 0 : depth[sc->fr[i].parent] + 1;
    for (int i = 0; i < nn; ++i) top[i] = depth[i] < D;
    // solve bytes per front (G twice, H once)
    fbytes.assign(nn, 0.0);
    for (int h = 0; h < sc->nlevels; ++h)
        for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) {
            const ItemDesc& d = c->items[q];
            fbytes[sc->item_front[q - sc->item_base]] +=
                item_doubles(d.tri, d.I1 - d.I0, d.ntiles) * 8.0 * (q < sc->g_end[h] ? 2 : 1);
        }
    std::vector<double> sub(nn, 0.0);   // subtree bytes (children have lower indices)
    for (int i = 0; i < nn; ++i) {
        sub[i] += fbytes[i];
        if (sc->fr[i].parent >= 0) sub[sc->fr[i].parent] += sub[i];
    }
    for (int i = 0; i < nn; ++i)
        if (!top[i] && (sc->fr[i].parent < 0 || top[sc->fr[i].parent])) {
            sroot[i] = 1;
            roots.push_back(i);
        }
    owner.assign(nn, -1);
    std::vector<int> sorted = roots;
    std::stable_sort(sorted.begin(), sorted.end(), [&](int a, int b) { return sub[a] > sub[b]; });
    std::vector<double> load(P, 0.0);
    for (int r : sorted) {
        const int k = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        owner[r] = k;
        load[k] += sub[r];
    }
    for (int i = nn - 1; i >= 0; --i)
        if (!top[i] && !sroot[i]) owner[i] = owner[sc->fr[i].parent];
}

static int sparse_coarse_dist_setup(ddg_ctx* c) {
    SparseCoarse* sc = c->sparse;
    const int nn = sc->nfront, P = c->nranks, me = c->rank;
    DistSplit ds;
    dist_split(c, P, ds);
    const std::vector<char>& top = ds.top;
    const std::vector<int>& owner = ds.owner;
    const std::vector<int>& roots = ds.roots;
    const std::vector<double>& fbytes = ds.fbytes;
    if (roots.empty()) return DDG_OK;   // the whole tree is above the cut: replicated solve
    int D = 0;
    while ((1 << D) < P) ++D;
    auto mine = [&](int f) { return !top[f] && owner[f] == me; };
    auto entry_front = [&](int32_t e) {
        const int idx = e & DF_IDX;
        if (e & DF_ASSEMBLE) return idx;
        if (e & DF_RED) return (e & DF_BWD) ? sc->bwd[idx].front : sc->fwd[idx].front;
        return (int)sc->item_front[idx - sc->item_base];
    };
    std::vector<int32_t> w1, w3;
    for (int32_t e : sc->dfwork) {
        const int f = entry_front(e);
        if (mine(f)) (e & DF_BWD ? w3 : w1).push_back(e);
    }
    // phase-1 fronts: subtree roots end the forward elimination like roots
    std::vector<FrontDesc> fr1 = sc->fr;
    for (int r : roots) fr1[r].parent = -1;
    // w exchange: the subtree roots' w, concatenated (zero slot for non-owners)
    std::vector<int32_t> wx;
    std::vector<uint8_t> wm;
    for (int r : roots)
        for (int j = 0; j < sc->fr[r].nB; ++j) {
            wx.push_back((int32_t)(sc->fr[r].w_off + j));
            wm.push_back(owner[r] == me);
        }
    // y_c: who contributes each coarse unknown
    std::vector<uint8_t> ym(c->nc, 0);
    for (int i = 0; i < nn; ++i) {
        const bool contrib = top[i] ? me == 0 : owner[i] == me;
        if (!contrib) continue;
        for (int a = 0; a < sc->fr[i].nS; ++a) ym[sc->fS[sc->fr[i].S_off + a]] = 1;
    }
    int st;
    if ((st = up(&sc->d_work1, w1)) || (st = up(&sc->d_work3, w3)) ||
        (st = up(&sc->d_fr1, fr1)) || (st = up(&sc->d_wx_idx, wx)) || (st = up(&sc->d_wx_mask, wm)) ||
        (st = dalloc(&sc->d_wx_buf, std::max<size_t>(1, wx.size()))) || (st = up(&sc->d_y_mask, ym)) ||
        (st = dalloc(&sc->d_y_buf, std::max<int64_t>(1, c->nc))))
        return st;
    sc->nw1 = (int)w1.size();
    sc->nw3 = (int)w3.size();
    sc->nwx = (int64_t)wx.size();
    sc->ntop = 0;
    for (int i = 0; i < nn; ++i) sc->ntop += top[i];
    sc->nsub = (int)roots.size();
    // top fronts: item ranges per front (a front's G items, and its H items, are
    // contiguous in c->items, and so are their partial segments)
    sc->tops.clear();
    sc->own_roots.clear();
    for (int r : roots)
        if (owner[r] == me) sc->own_roots.push_back(r);
    {
        std::vector<int> dep(nn, 0);
        for (int i = nn - 1; i >= 0; --i) dep[i] = sc->fr[i].parent < 0 ? 0 : dep[sc->fr[i].parent] + 1;
        std::vector<int> g0(nn, INT32_MAX), g1(nn, -1), h0(nn, INT32_MAX), h1(nn, -1);
        for (int h = 0; h < sc->nlevels; ++h)
            for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) {
                const int f = sc->item_front[q - sc->item_base];
                if (q < sc->g_end[h]) { g0[f] = std::min(g0[f], q); g1[f] = std::max(g1[f], q + 1); }
                else { h0[f] = std::min(h0[f], q); h1[f] = std::max(h1[f], q + 1); }
            }
        for (int i = 0; i < nn; ++i) {
            if (!top[i]) continue;
            SparseCoarse::Top t{i, dep[i], g1[i] < 0 ? 0 : g0[i], g1[i] < 0 ? 0 : g1[i], h1[i] < 0 ? 0 : h0[i],
                                h1[i] < 0 ? 0 : h1[i], sc->fdf[i].ft0, sc->fdf[i].ft1, sc->fdf[i].bt0, sc->fdf[i].bt1};
            sc->tops.push_back(t);
        }
        std::stable_sort(sc->tops.begin(), sc->tops.end(),
                         [](const SparseCoarse::Top& a, const SparseCoarse::Top& b) { return a.depth > b.depth; });
    }
    double rb = 0, tb = 0;
    for (int i = 0; i < nn; ++i) {
        if (top[i]) tb += fbytes[i];
        else if (owner[i] == me) rb += fbytes[i];
    }
    rb += tb / P;    // the top fronts' item ranges are split evenly by item count
    sc->rank_solve_bytes = (int64_t)rb;
    // keep only the front operators this rank reads (its subtrees, its chunk of every
    // top range): the factor was built replicated (the top fronts need every
    // subtree's Schur complement), the solve needs a 1/P share of it
    if (!(getenv("DDG_COARSE_KEEP_ALL") && atoi(getenv("DDG_COARSE_KEEP_ALL")) != 0)) {
        std::vector<char> keep(c->items.size(), 0);
        for (int h = 0; h < sc->nlevels; ++h)
            for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q)
                if (mine(sc->item_front[q - sc->item_base])) keep[q] = 1;
        auto chunk = [&](int q0, int q1) {
            const int64_t len = q1 - q0;
            for (int q = q0 + (int)(len * me / P); q < q0 + (int)(len * (me + 1) / P); ++q) keep[q] = 1;
        };
        for (const auto& t : sc->tops) {
            chunk(t.g0, t.g1);
            chunk(t.h0, t.h1);
        }
        std::vector<int64_t> seg;
        int64_t nd = 0;
        for (int q = sc->item_base; q < sc->item_end; ++q) {
            if (!keep[q]) continue;
            ItemDesc& it = c->items[q];
            const int64_t len = item_doubles(it.tri, it.I1 - it.I0, it.ntiles);
            seg.push_back(it.tile_off);
            seg.push_back(nd);
            seg.push_back(len);
            it.tile_off = nd;
            nd += len;
        }
        double* d_new = nullptr;
        int64_t* d_seg = nullptr;
        if ((st = dalloc(&d_new, std::max<int64_t>(1, nd))) || (st = up(&d_seg, seg))) return st;
        launch_copy_segments(c->stream, (int)(seg.size() / 3), d_seg, sc->d_ctiles, d_new);
        for (int q = sc->item_base; q < sc->item_end; ++q)
            if (!keep[q]) c->items[q].tile_off = -1;   // never read on this rank
        CUDA_TRY(cudaMemcpyAsync(c->d_items + sc->item_base, c->items.data() + sc->item_base,
                                 (size_t)(sc->item_end - sc->item_base) * sizeof(ItemDesc), cudaMemcpyHostToDevice,
                                 c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        CUDA_TRY(cudaGetLastError());
        cudaFree(d_seg);
        cudaFree(sc->d_ctiles);
        sc->d_ctiles = d_new;
        sc->factor_bytes = nd * 8;
    }
    sc->dist = true;
    if (c->opts.verbose)
        fprintf(stderr, "[ddg_setup] distributed coarse solve: depth %d cut, %d top fronts, %d subtrees; rank %d "
                "reads %.2f of %.2f GB per solve\n", D, sc->ntop, sc->nsub, me, rb / 1e9,
                (double)sparse_coarse_solve_bytes(c) / 1e9);
    return DDG_OK;
}

// --------------------------------------------------------------------------
// numeric phase (device)
// --------------------------------------------------------------------------
int sparse_coarse_numeric(ddg_ctx* c) {
    SparseCoarse* sc = c->sparse;
    int st;
    if ((st = up(&sc->d_fr, sc->fr)) || (st = up(&sc->d_fchild, sc->fchild)) || (st = up(&sc->d_fS, sc->fS)) ||
        (st = up(&sc->d_fB, sc->fB)) ||
        (st = up(&sc->d_fmap, sc->fmap)) || (st = up(&sc->d_item_front, sc->item_front)) ||
        (st = up(&sc->d_fwd, sc->fwd)) || (st = up(&sc->d_bwd, sc->bwd)) ||
        (st = up(&sc->d_contrib, sc->contrib)) || (st = up(&sc->d_dfwork, sc->dfwork)) ||
        (st = up(&sc->d_fdf, sc->fdf)) ||
        (st = dalloc(&sc->d_dfstate, 1 + (size_t)DF_STATE_PER_FRONT * sc->nfront)) ||
        (st = dalloc(&sc->d_fvec, sc->fvec_doubles)) ||
        (st = dalloc(&sc->d_w, sc->w_doubles)) || (st = dalloc(&sc->d_ctiles, sc->ctile_doubles)) ||
        (st = dalloc(&sc->d_bc, c->nc)))
        return st;
    const int nn = sc->nfront;
    double** d_fptr = nullptr;
    int32_t *d_err = nullptr, *d_ids = nullptr, *d_nT = nullptr, *d_nK = nullptr, *d_tasks = nullptr;
    if ((st = dalloc(&d_fptr, nn)) || (st = dalloc(&d_err, 2)) || (st = dalloc(&d_ids, nn)) ||
        (st = dalloc(&d_nT, nn)) || (st = dalloc(&d_nK, nn)) || (st = dalloc(&d_tasks, nn)))
        return st;
    int32_t herr[2] = {-1, -1};
    { int _s = h2d(c->stream, d_err, herr, sizeof herr); if (_s) return _s; }
    std::vector<double*> fptr(nn, nullptr);
    std::vector<double*> level_buf(sc->nlevels, nullptr);
    std::vector<int> max_parent_h(sc->nlevels, -1);
    auto height_of = [&](int f) {
        int h = 0;
        while (!(sc->lb[h] <= f && f < sc->lb[h + 1])) ++h;
        return h;
    };
    for (int h = 0; h < sc->nlevels; ++h)
        for (int i = sc->lb[h]; i < sc->lb[h + 1]; ++i)
            if (sc->fr[i].parent >= 0) max_parent_h[h] = std::max(max_parent_h[h], height_of(sc->fr[i].parent));
    for (int h = 0; h < sc->nlevels; ++h) {
        const int f0 = sc->lb[h], f1 = sc->lb[h + 1], nf = f1 - f0;
        int64_t tot = 0;
        for (int i = f0; i < f1; ++i) tot += (int64_t)sc->fr[i].nT * sc->fr[i].nT * TILE_ELEMS;
        if ((st = dalloc(&level_buf[h], tot))) return st;
        CUDA_TRY(cudaMemsetAsync(level_buf[h], 0, tot * sizeof(double), c->stream));
        int64_t off = 0;
        for (int i = f0; i < f1; ++i) {
            fptr[i] = level_buf[h] + off;
            off += (int64_t)sc->fr[i].nT * sc->fr[i].nT * TILE_ELEMS;
        }
        CUDA_TRY(cudaMemcpyAsync(d_fptr + f0, fptr.data() + f0, nf * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
        // assemble A_c entries
        {
            int32_t *dr = nullptr, *dc = nullptr, *df = nullptr;
            double* dv = nullptr;
            if ((st = up(&dr, sc->tr_r[h])) || (st = up(&dc, sc->tr_c[h])) || (st = up(&df, sc->tr_f[h])) ||
                (st = up(&dv, sc->tr_v[h])))
                return st;
            launch_front_scatter(c->stream, (int64_t)sc->tr_v[h].size(), dr, dc, dv, df, sc->d_fr, d_fptr);
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            cudaFree(dr); cudaFree(dc); cudaFree(df); cudaFree(dv);
        }
        // extend-add the children's Schur complements (slot by slot: no write conflicts)
        int maxch = 0;
        for (int i = f0; i < f1; ++i) maxch = std::max(maxch, (int)sc->fr[i].nchild);
        for (int slot = 0; slot < maxch; ++slot) {
            std::vector<int32_t> tasks;
            int64_t maxe = 0;
            for (int i = f0; i < f1; ++i) {
                const int ch = slot < sc->fr[i].nchild ? sc->fchild[sc->fr[i].child_off + slot] : -1;
                if (ch >= 0 && sc->fr[ch].nB > 0) {
                    tasks.push_back(ch);
                    maxe = std::max<int64_t>(maxe, (int64_t)sc->fr[ch].nB * sc->fr[ch].nB);
                }
            }
            if (tasks.empty()) continue;
            CUDA_TRY(cudaMemcpyAsync(d_tasks, tasks.data(), tasks.size() * 4, cudaMemcpyHostToDevice, c->stream));
            launch_front_extend_add(c->stream, (int)tasks.size(), d_tasks, sc->d_fr, d_fptr, sc->d_fmap, maxe);
            CUDA_TRY(cudaStreamSynchronize(c->stream));
        }
        static const bool dbg = getenv("DDG_DEBUG_CHECK") != nullptr;
        auto dump = [&](const char* tag) -> int {
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            for (int i = f0; i < f1; ++i) {
                const FrontDesc& f = sc->fr[i];
                const int64_t ne = (int64_t)f.nT * f.nT * TILE_ELEMS;
                std::vector<double> hv(ne);
                { int _s = d2h(c->stream, hv.data(), fptr[i], ne * 8); if (_s) return _s; }
                const int N = f.nT * TILE;
                auto at = [&](int R, int Cc) {
                    return hv[((int64_t)(Cc / TILE) * f.nT + R / TILE) * TILE_ELEMS + (Cc % TILE) * TILE + R % TILE];
                };
                double cs = 0, asym = 0, dmin = 1e300;
                for (int R = 0; R < N; ++R)
                    for (int Cc = 0; Cc < N; ++Cc) {
                        cs += fabs(at(R, Cc)) * (1 + (R * 7 + Cc * 13) % 5);
                        if (!(R < f.nSp && Cc < f.nSp) && !(R >= f.nSp && Cc >= f.nSp)) continue;
                        asym = std::max(asym, fabs(at(R, Cc) - at(Cc, R)));
                    }
                for (int R = 0; R < f.nS; ++R) dmin = std::min(dmin, at(R, R));
                fprintf(stderr, "[dbg] %s lvl %d front %d nS %d nB %d nT %d nch %d cs %.17g asym %.3g dmin %.3g\n",
                        tag, h, i, f.nS, f.nB, f.nT, f.nchild, cs, asym, dmin);
            }
            return DDG_OK;
        };
        if (dbg && (st = dump("assembled"))) return st;
        // eliminate the S pivots: small fronts one CTA each (tile exchange), the
        // rest with the blocked exchange (fp64 GEMM updates), each as one batch
        std::vector<int32_t> ids, nTs, nKs;
        std::vector<double*> mats;
        int nsmall = 0, maxT = 0, maxK = 0;
        for (int pass = 0; pass < 2; ++pass)
            for (int i = f0; i < f1; ++i) {
                const FrontDesc& f = sc->fr[i];
                if ((f.nT < GJB_MIN_T) != (pass == 0)) continue;
                ids.push_back(i);
                nTs.push_back(f.nT);
                nKs.push_back(f.nK);
                mats.push_back(fptr[i]);
                if (pass == 0) ++nsmall;
                else { maxT = std::max(maxT, f.nT); maxK = std::max(maxK, f.nK); }
            }
        if (!ids.empty()) {
            double** d_m = nullptr;
            if ((st = dalloc(&d_m, ids.size()))) return st;
            CUDA_TRY(cudaMemcpyAsync(d_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(cudaMemcpyAsync(d_nT, nTs.data(), ids.size() * 4, cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(cudaMemcpyAsync(d_nK, nKs.data(), ids.size() * 4, cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(cudaMemcpyAsync(d_m, mats.data(), ids.size() * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
            if (nsmall) launch_gj_batched(c->stream, nsmall, d_nT, d_nK, d_m, d_ids, d_err);
            const int nbig = (int)ids.size() - nsmall;
            if (nbig)
                launch_gj_blocked(c->stream, nbig, maxT, maxK, d_m + nsmall, d_nT + nsmall, d_nK + nsmall,
                                  d_ids + nsmall, d_err);
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            cudaFree(d_m);
        }
        // pack the level's solve operators
        launch_front_pack(c->stream, sc->g_begin[h], sc->h_end[h], sc->item_base, sc->d_item_front, sc->d_fr,
                          d_fptr, c->d_items, sc->d_ctiles);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (dbg && (st = dump("factored"))) return st;
        // release levels whose fronts have all been absorbed by their parents
        for (int l = 0; l < h; ++l)
            if (level_buf[l] && max_parent_h[l] <= h) {
                cudaFree(level_buf[l]);
                level_buf[l] = nullptr;
            }
        if (c->opts.verbose) {
            double gb = 0, hb = 0;
            for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) {
                const ItemDesc& d = c->items[q];
                (q < sc->g_end[h] ? gb : hb) += item_doubles(d.tri, d.I1 - d.I0, d.ntiles) * 8.0;
            }
            fprintf(stderr, "[ddg_setup] coarse level %2d: %5d fronts, max front %d, G items %d (%.1f MB), "
                    "H items %d (%.1f MB)\n", h, nf,
                    [&] { int m = 0; for (int i = f0; i < f1; ++i) m = std::max(m, sc->fr[i].nT * TILE); return m; }(),
                    sc->g_end[h] - sc->g_begin[h], gb / 1e6, sc->h_end[h] - sc->h_begin[h], hb / 1e6);
        }
    }
    for (auto* b : level_buf)
        if (b) cudaFree(b);
    { int _s = d2h(c->stream, herr, d_err, sizeof herr); if (_s) return _s; }
    cudaFree(d_fptr); cudaFree(d_err); cudaFree(d_ids); cudaFree(d_nT); cudaFree(d_nK); cudaFree(d_tasks);
    if (herr[0] >= 0)
        return set_err(DDG_E_NOT_SPD, "coarse factor: front %d not positive definite at pivot %d", herr[0], herr[1]);
    if (c->dist && c->nranks > 1 && sc->dataflow && !(getenv("DDG_COARSE_REPLICATED") &&
                                                      atoi(getenv("DDG_COARSE_REPLICATED")) != 0))
        return sparse_coarse_dist_setup(c);
    return DDG_OK;
}

// --------------------------------------------------------------------------
// solve: y_c = A_c^{-1} b_c
// --------------------------------------------------------------------------
double* sparse_coarse_rhs(ddg_ctx* c) { return c->sparse->d_bc; }
int64_t sparse_coarse_bytes(ddg_ctx* c) { return c->sparse ? c->sparse->factor_bytes : 0; }
// forward reads every G item, backward every G and H item
int64_t sparse_coarse_solve_bytes(ddg_ctx* c) {
    if (!c->sparse) return 0;
    const SparseCoarse* sc = c->sparse;
    if (sc->dist) return sc->rank_solve_bytes;
    int64_t b = 0;
    for (int h = 0; h < sc->nlevels; ++h)
        for (int q = sc->g_begin[h]; q < sc->h_end[h]; ++q) {
            const ItemDesc& d = c->items[q];
            b += item_doubles(d.tri, d.I1 - d.I0, d.ntiles) * 8 * (q < sc->g_end[h] ? 2 : 1);
        }
    return b;
}
int sparse_coarse_levels(ddg_ctx* c) { return c->sparse ? c->sparse->nlevels : 0; }
int sparse_coarse_nfront(ddg_ctx* c) { return c->sparse ? c->sparse->nfront : 0; }

int sparse_coarse_enqueue_solve(ddg_ctx* c, double* d_x, const int32_t* done) {
    SparseCoarse* sc = c->sparse;
    int launches = 0;
    if (sc->dist) {
        auto df = [&](int nw, const int32_t* work, const FrontDesc* fr) {
            launch_coarse_dataflow(c->stream, nw, work, fr, sc->d_fchild, sc->d_fdf, sc->d_item_front, sc->item_base,
                                   c->d_ops, c->d_items, sc->d_ctiles, sc->d_fwd, sc->d_bwd, sc->d_contrib, sc->d_fS,
                                   sc->d_fB, sc->d_fmap, sc->d_bc, sc->d_fvec, sc->d_w, d_x, c->d_partials,
                                   sc->d_dfstate, sc->max_rows_t, done, nullptr);
        };
        int err = 0;
        cudaMemsetAsync(sc->d_dfstate, 0, (1 + (size_t)DF_STATE_PER_FRONT * sc->nfront) * sizeof(int32_t), c->stream);
        df(sc->nw1, sc->d_work1, sc->d_fr1);                                       // phase 1: own subtrees, forward
        launch_gather_masked(c->stream, sc->nwx, sc->d_wx_idx, sc->d_wx_mask, sc->d_w, sc->d_wx_buf);
        err |= ddg::comm_allreduce_sum(c->comm, sc->d_wx_buf, sc->d_wx_buf, (size_t)sc->nwx, c->stream);
        launch_halo_unpack(c->stream, sc->d_wx_buf, sc->d_wx_idx, sc->d_w, sc->nwx);
        {
            // phase 2, the top fronts' items split over the ranks: per item range
            // zero its partial segments, compute this rank's share, allreduce
            const int P = c->nranks, me = c->rank;
            auto sym_range = [&](int q0, int q1) {
                if (q1 <= q0) return;
                const ItemDesc& a = c->items[q0];
                const ItemDesc& b = c->items[q1 - 1];
                const int64_t lo = a.part_off;
                const int64_t hi = b.part_off + (int64_t)(b.I1 - b.I0 + (b.tri ? 0 : b.J1 - b.J0)) * TILE;
                cudaMemsetAsync(c->d_partials + lo, 0, (size_t)(hi - lo) * sizeof(double), c->stream);
                const int64_t len = q1 - q0;
                const int m0 = q0 + (int)(len * me / P), m1 = q0 + (int)(len * (me + 1) / P);
                if (m1 > m0)
                    launch_symv(c->stream, c->d_ops, c->d_items, m0, m1 - m0, sc->d_ctiles, sc->d_fvec, nullptr,
                                nullptr, nullptr, c->d_partials, done, sc->max_rows_t, c->d_tickets);
                err |= ddg::comm_allreduce_sum(c->comm, c->d_partials + lo, c->d_partials + lo, (size_t)(hi - lo),
                                               c->stream);
                launches += 2;
            };
            for (const auto& t : sc->tops) {                                       // forward, deepest first
                launch_front_fwd_assemble(c->stream, t.f, 1, sc->d_fr, sc->d_fchild, sc->d_fS, sc->d_fmap, sc->d_bc,
                                          sc->d_fvec, sc->d_w, done);
                sym_range(t.g0, t.g1);
                launch_front_reduce(c->stream, sc->d_fwd, t.ft0, t.ft1 - t.ft0, sc->d_contrib, sc->d_fr, sc->d_fS,
                                    c->d_partials, sc->d_w, d_x, done);
                launches += 2;
            }
            for (auto it = sc->tops.rbegin(); it != sc->tops.rend(); ++it) {        // backward, root first
                launch_front_bwd_gather(c->stream, it->f, 1, sc->d_fr, sc->d_fB, d_x, sc->d_fvec, done);
                sym_range(it->g0, it->g1);
                sym_range(it->h0, it->h1);
                launch_front_reduce(c->stream, sc->d_bwd, it->bt0, it->bt1 - it->bt0, sc->d_contrib, sc->d_fr,
                                    sc->d_fS, c->d_partials, sc->d_w, d_x, done);
                launches += 2;
            }
            for (int r : sc->own_roots)                                            // x[B] of the subtree roots
                launch_front_bwd_gather(c->stream, r, 1, sc->d_fr, sc->d_fB, d_x, sc->d_fvec, done);
            launches += (int)sc->own_roots.size();
        }
        cudaMemsetAsync(sc->d_dfstate, 0, sizeof(int32_t), c->stream);
        df(sc->nw3, sc->d_work3, sc->d_fr);                                        // phase 3: own subtrees, back
        launch_gather_masked(c->stream, c->nc, nullptr, sc->d_y_mask, d_x, sc->d_y_buf);
        err |= ddg::comm_allreduce_sum(c->comm, sc->d_y_buf, d_x, (size_t)c->nc, c->stream);
        if (err && !c->comm_err) c->comm_err = err;
        return launches + 8;
    }
    if (sc->dataflow) {
        cudaMemsetAsync(sc->d_dfstate, 0, (1 + (size_t)DF_STATE_PER_FRONT * sc->nfront) * sizeof(int32_t),
                        c->stream);
        launch_coarse_dataflow(c->stream, (int)sc->dfwork.size(), sc->d_dfwork, sc->d_fr, sc->d_fchild, sc->d_fdf,
                               sc->d_item_front, sc->item_base, c->d_ops, c->d_items, sc->d_ctiles, sc->d_fwd,
                               sc->d_bwd, sc->d_contrib, sc->d_fS, sc->d_fB, sc->d_fmap, sc->d_bc, sc->d_fvec,
                               sc->d_w, d_x, c->d_partials, sc->d_dfstate, sc->max_rows_t, done, sc->d_trace);
        return 1;
    }
    for (int h = 0; h < sc->nlevels; ++h) {
        const int f0 = sc->lb[h], nf = sc->lb[h + 1] - f0;
        launch_front_fwd_assemble(c->stream, f0, nf, sc->d_fr, sc->d_fchild, sc->d_fS, sc->d_fmap, sc->d_bc, sc->d_fvec,
                                  sc->d_w, done);
        if (ring_ok(c, sc->ring_fwd[h]))
        {
            int mr, mc;
            ring_dims(c, sc->ring_fwd[h], &mr, &mc);
            launch_symv_ring(c->stream, c->d_ops, c->d_items, sc->g_begin[h], c->d_ring + sc->ring_fwd[h], num_sms(), mr, mc,
                             sc->d_ctiles, sc->d_fvec, nullptr, nullptr, nullptr, c->d_partials, done);
        } else
            launch_symv(c->stream, c->d_ops, c->d_items, sc->g_begin[h], sc->g_end[h] - sc->g_begin[h],
                        sc->d_ctiles, sc->d_fvec, nullptr, nullptr, nullptr, c->d_partials, done, sc->max_rows_t,
                        c->d_tickets);
        launch_front_reduce(c->stream, sc->d_fwd, sc->fwd_b[h], sc->fwd_b[h + 1] - sc->fwd_b[h], sc->d_contrib,
                            sc->d_fr, sc->d_fS, c->d_partials, sc->d_w, d_x, done);
        launches += 1 + (sc->g_end[h] > sc->g_begin[h]) + (sc->fwd_b[h + 1] > sc->fwd_b[h]);
    }
    for (int h = sc->nlevels - 1; h >= 0; --h) {
        const int f0 = sc->lb[h], nf = sc->lb[h + 1] - f0;
        launch_front_bwd_gather(c->stream, f0, nf, sc->d_fr, sc->d_fB, d_x, sc->d_fvec, done);
        if (ring_ok(c, sc->ring_bwd[h]))
        {
            int mr, mc;
            ring_dims(c, sc->ring_bwd[h], &mr, &mc);
            launch_symv_ring(c->stream, c->d_ops, c->d_items, sc->g_begin[h], c->d_ring + sc->ring_bwd[h], num_sms(), mr, mc,
                             sc->d_ctiles, sc->d_fvec, nullptr, nullptr, nullptr, c->d_partials, done);
        } else
            launch_symv(c->stream, c->d_ops, c->d_items, sc->g_begin[h], sc->h_end[h] - sc->g_begin[h],
                        sc->d_ctiles, sc->d_fvec, nullptr, nullptr, nullptr, c->d_partials, done, sc->max_rows_t,
                        c->d_tickets);
        launch_front_reduce(c->stream, sc->d_bwd, sc->bwd_b[h], sc->bwd_b[h + 1] - sc->bwd_b[h], sc->d_contrib,
                            sc->d_fr, sc->d_fS, c->d_partials, sc->d_w, d_x, done);
        launches += 3;
    }
    return launches;
}

// debug (not part of include/ddg.h): the distributed coarse solve's split for
// P ranks on this context's tree (the plan sparse_coarse_dist_setup makes):
// coarse solve bytes of each rank's own subtrees into bytes[0 .. P), the
// top fronts' total into *top (read by every rank when replicated, 1/P of it
// per rank when split, the default); returns the number of
// subtrees (0: the whole tree lies above the cut), -1 without a sparse coarse
extern "C" int ddg_debug_coarse_split(ddg_ctx* c, int P, double* bytes, double* top) {
    if (!c || !c->sparse || P < 1) return -1;
    DistSplit ds;
    dist_split(c, P, ds);
    double tb = 0;
    for (int p = 0; p < P; ++p) bytes[p] = 0;
    for (size_t i = 0; i < ds.top.size(); ++i) {
        if (ds.top[i]) tb += ds.fbytes[i];
        else bytes[ds.owner[i]] += ds.fbytes[i];
    }
    *top = tb;
    return (int)ds.roots.size();
}

// debug (not part of include/ddg.h): the dataflow trace of the last coarse
// solve -- per work entry {start | cta << 52, dependency met, item done,
// entry finished} in ns -- and the work entries; returns the entry count
extern "C" int ddg_debug_df_trace(ddg_ctx* c, uint64_t* trace, int32_t* work, int cap) {
    if (!c || !c->sparse || !c->sparse->d_trace) return -1;
    SparseCoarse* sc = c->sparse;
    const int n = (int)sc->dfwork.size();
    if (cap < n) return -n;
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(trace, sc->d_trace, (size_t)n * 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    memcpy(work, sc->dfwork.data(), (size_t)n * sizeof(int32_t));
    return n;
}
