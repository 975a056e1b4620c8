// setup.cpp — host side of libddg: the C ABI (include/ddg.h), the setup
// pipeline, and the PCG driver that enqueues the sm_100a kernels.
//
// Setup, SURVEY.md §3 call stack (1):
//   parts Omega_I -> overlap Omega~_i (BFS, Delta) -> colours + sweep order
//   -> per-part double-double MGS basis (R6c, R7) -> Galerkin A_c = P^T A P
//   (host, threaded) -> device: local inverses A_i^{-1} (extract + batched
//   Gauss-Jordan + pack) and the coarse inverse A_c^{-1}.
// Solve: PCG whose every vector operation and every
// preconditioner step runs in the .cu kernels; the host only enqueues (one CUDA
// graph per iteration) and polls the device `done` flag every few iterations.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ddg.h"
#include "ddg_internal.h"

using namespace ddg;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

int set_err(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

extern "C" const char* ddg_last_error(void) { return g_last_error.c_str(); }

extern "C" const char* ddg_status_string(int s) {
    switch (s) {
        case DDG_OK: return "ok";
        case DDG_E_ARG: return "invalid argument";
        case DDG_E_DIM: return "dimension mismatch / non-canonical CSR";
        case DDG_E_PART: return "invalid partition";
        case DDG_E_ZERO_BLOCK: return "generating vectors vanish on a part";
        case DDG_E_NOT_SPD: return "matrix not positive definite";
        case DDG_E_COLOURING: return "colouring conflict";
        case DDG_E_BREAKDOWN: return "CG breakdown";
        case DDG_E_CUDA: return "CUDA error";
        case DDG_E_NCCL: return "NCCL error";
        case DDG_E_OOM: return "out of device memory";
        default: return "unknown status";
    }
}

extern "C" void ddg_default_opts(ddg_opts* o) {
    memset(o, 0, sizeof *o);
    o->overlap = 1;
    o->rank_tol = 1e-8;
    o->stop_mode = DDG_STOP_RES0;
    o->max_iter = 1000;
    o->device = 0;
    o->stream = nullptr;
    o->use_graphs = 1;
    o->verbose = 0;
    o->fuse_gather = 1;
    o->small_kernel = 1;
}

// ---------------------------------------------------------------------------
// small host helpers
// ---------------------------------------------------------------------------
void parallel_for(int64_t n, const std::function<void(int64_t, int64_t, int)>& fn) {
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 32);
    if (n < 64 || nt == 1) { fn(0, n, 0); return; }
    nt = (int)std::min<int64_t>(nt, n);
    std::vector<std::thread> th;
    std::atomic<int64_t> next{0};
    const int64_t chunk = std::max<int64_t>(1, n / (nt * 16));
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (;;) {
                int64_t b = next.fetch_add(chunk);
                if (b >= n) break;
                fn(b, std::min(n, b + chunk), t);
            }
        });
    for (auto& x : th) x.join();
}

static int hw_threads() {
    return (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
}

// ---------------------------------------------------------------------------
// the context
// ---------------------------------------------------------------------------
#include "ctx.h"
#include "comm.h"
#include "dist.h"

// coarse_sparse.cpp
int sparse_coarse_symbolic(ddg_ctx* c, const int64_t* rp, const int32_t* col, const std::vector<int32_t>& er,
                           const std::vector<int32_t>& ec, const std::vector<double>& ev);
int sparse_coarse_numeric(ddg_ctx* c);
int sparse_coarse_enqueue_solve(ddg_ctx* c, double* d_x, const int32_t* done);
double* sparse_coarse_rhs(ddg_ctx* c);
int64_t sparse_coarse_bytes(ddg_ctx* c);
int64_t sparse_coarse_solve_bytes(ddg_ctx* c);

static void free_ctx(ddg_ctx* c) {
    if (!c) return;
    if (c->child) free_ctx(c->child);   // borrows this context's stream
    if (c->device >= 0) cudaSetDevice(c->device);
    if (c->ge_iter) cudaGraphExecDestroy(c->ge_iter);
    if (c->g_iter) cudaGraphDestroy(c->g_iter);
    if (c->ge_solve) cudaGraphExecDestroy(c->ge_solve);
    if (c->g_solve) cudaGraphDestroy(c->g_solve);
    void* ptrs[] = {c->d_rp, c->d_col, c->d_val, c->d_oidx, c->d_ops, c->d_items, c->d_red,
                    c->d_tiles, c->d_s, c->d_partials, c->d_bptr, c->d_bidx, c->d_cptr,
                    c->d_qoff, c->d_Q, c->d_yc, c->d_r, c->d_z, c->d_p, c->d_q, c->d_f,
                    c->d_u, c->d_x, c->d_sc, c->d_hist, c->d_redbuf, c->d_ticket, c->d_zero, c->d_tickets,
                    c->d_ring, c->d_gidx, c->d_stencil_coef, c->d_ab, c->d_bc, c->d_res, c->d_xpart, c->d_brp, c->d_bcol,
                    c->d_cops};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->h_sc) cudaFreeHost(c->h_sc);
    for (auto e : c->evpool) cudaEventDestroy(e);
    if (c->sparse) sparse_coarse_free(c->sparse);
    {
        std::vector<ddg::Halo*> hs{&c->h_p, &c->h_r};
        for (auto& h : c->h_z) hs.push_back(&h);
        for (auto* h : hs) {
            if (h->d_sidx) cudaFree(h->d_sidx);
            if (h->d_ridx) cudaFree(h->d_ridx);
            if (h->d_sbuf) cudaFree(h->d_sbuf);
            if (h->d_rbuf) cudaFree(h->d_rbuf);
        }
        if (c->d_rows) cudaFree(c->d_rows);
        if (c->d_restrict_parts) cudaFree(c->d_restrict_parts);
        if (c->d_prolong_parts) cudaFree(c->d_prolong_parts);
    }
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    delete c;
}

extern "C" void ddg_destroy(ddg_ctx* c) { free_ctx(c); }

// ---------------------------------------------------------------------------
// setup steps (host)
// ---------------------------------------------------------------------------

// Omega~_i: nodes within graph distance Delta of Omega_i, sorted
static void build_overlap(ddg_ctx* c, const int64_t* rp, const int32_t* col) {
    const int np = c->nparts;
    std::vector<std::vector<int32_t>> lists(np);
    const int nt = hw_threads();
    std::vector<std::vector<int32_t>> marks(nt);
    parallel_for(np, [&](int64_t b, int64_t e, int t) {
        auto& mark = marks[t];
        if (mark.empty()) mark.assign(c->n, -1);
        for (int64_t I = b; I < e; ++I) {
            auto& L = lists[I];
            for (int64_t a = c->bptr[I]; a < c->bptr[I + 1]; ++a) {
                L.push_back(c->bidx[a]);
                mark[c->bidx[a]] = (int32_t)I;
            }
            size_t lb = 0, le = L.size();
            for (int d = 0; d < c->opts.overlap; ++d) {
                for (size_t a = lb; a < le; ++a) {
                    const int32_t v = L[a];
                    for (int64_t x = rp[v]; x < rp[v + 1]; ++x) {
                        const int32_t u = col[x];
                        if (u != v && mark[u] != (int32_t)I) {
                            mark[u] = (int32_t)I;
                            L.push_back(u);
                        }
                    }
                }
                lb = le;
                le = L.size();
            }
            std::sort(L.begin(), L.end());
        }
    });
    c->optr.assign(np + 1, 0);
    for (int I = 0; I < np; ++I) c->optr[I + 1] = c->optr[I] + (int64_t)lists[I].size();
    c->oidx.resize(c->optr[np]);
    for (int I = 0; I < np; ++I)
        std::copy(lists[I].begin(), lists[I].end(), c->oidx.begin() + c->optr[I]);
}

// Greedy first-fit colours over increasing id; i, j conflict iff Omega~_i meets
// Omega~_j or its neighbourhood (the pull-form residual of j reads there).
// Sweep order: (colour, id).  Reading R3.
static int build_colours(ddg_ctx* c, const int64_t* rp, const int32_t* col) {
    const int64_t n = c->n;
    const int np = c->nparts;
    std::vector<int64_t> cp(n + 1, 0);
    for (int32_t v : c->oidx) cp[v + 1]++;
    for (int64_t v = 0; v < n; ++v) cp[v + 1] += cp[v];
    std::vector<int32_t> cov(cp[n]);
    {
        std::vector<int64_t> fill(cp.begin(), cp.end() - 1);
        for (int i = 0; i < np; ++i)
            for (int64_t a = c->optr[i]; a < c->optr[i + 1]; ++a) cov[fill[c->oidx[a]]++] = i;
    }
    // the conflict graph, in parallel: j conflicts with i iff some row of
    // Omega~_i or one of its neighbours lies in Omega~_j (sorted, j != i)
    std::vector<std::vector<int32_t>> conf(np);
    {
        const int nt = hw_threads();
        std::vector<std::vector<int32_t>> marks(nt);
        parallel_for(np, [&](int64_t b, int64_t e, int t) {
            auto& mark = marks[t];
            if (mark.empty()) mark.assign(np, -1);
            for (int64_t i = b; i < e; ++i) {
                auto& L = conf[i];
                for (int64_t a = c->optr[i]; a < c->optr[i + 1]; ++a) {
                    const int32_t v = c->oidx[a];
                    for (int64_t x = rp[v]; x < rp[v + 1]; ++x) {
                        const int32_t u = col[x];
                        for (int64_t q = cp[u]; q < cp[u + 1]; ++q) {
                            const int j = cov[q];
                            if (j != (int)i && mark[j] != (int32_t)i) {
                                mark[j] = (int32_t)i;
                                L.push_back(j);
                            }
                        }
                    }
                }
                std::sort(L.begin(), L.end());
            }
        });
    }
    c->colour.assign(np, -1);
    std::vector<char> used;
    int maxc = 0;
    if (const int32_t* uc = c->opts.colour) {
        // the caller's colouring (ddg_opts.colour), checked with the same
        // conflict rule: Omega~_i meets Omega~_j or its neighbours (reading R3)
        for (int i = 0; i < np; ++i)
            if (uc[i] < 0 || uc[i] >= np)
                return set_err(DDG_E_COLOURING, "colour %d of subdomain %d outside [0,%d)", uc[i], i, np);
        for (int i = 0; i < np; ++i) {
            for (int32_t j : conf[i])
                if (uc[j] == uc[i])
                    return set_err(DDG_E_COLOURING, "subdomains %d and %d are coupled but share colour %d",
                                   std::min(i, j), std::max(i, j), uc[i]);
            c->colour[i] = uc[i];
            maxc = std::max(maxc, uc[i] + 1);
        }
    }
    // greedy first-fit over increasing id (reading R3): the smallest colour no
    // already-coloured conflicting subdomain has
    for (int i = 0; i < np && !c->opts.colour; ++i) {
        used.assign(maxc + 1, 0);
        for (int32_t j : conf[i])
            if (c->colour[j] >= 0) used[c->colour[j]] = 1;
        int cc = 0;
        while (cc <= maxc && used[cc]) ++cc;
        c->colour[i] = cc;
        maxc = std::max(maxc, cc + 1);
    }
    c->ncolours = maxc;
    c->order.resize(np);
    for (int i = 0; i < np; ++i) c->order[i] = i;
    std::stable_sort(c->order.begin(), c->order.end(),
                     [&](int a, int b) { return c->colour[a] < c->colour[b]; });   // (colour, id)
    return DDG_OK;
}

// Operator descriptors, work items and reduction tasks for the tiled SYMV.
static void add_op(ddg_ctx* c, int32_t m, int out_mode, int64_t idx_off, bool allow_single, bool compact = false) {
    OpDesc op{};
    op.m = m;
    op.mp = ((m + TILE - 1) / TILE) * TILE;
    op.nT = op.mp / TILE;
    const int single_max = getenv("DDG_SINGLE_MAX_NT") ? atoi(getenv("DDG_SINGLE_MAX_NT")) : MAX_BT;
    if (allow_single && op.nT <= single_max) op.BT = op.nT;
    else op.BT = (op.nT > 512) ? MAX_BT : 8;
    if (op.BT > op.nT) op.BT = op.nT;
    op.nblk = (op.nT + op.BT - 1) / op.BT;
    op.item_base = (int32_t)c->items.size();
    op.nitems = op.nblk * (op.nblk + 1) / 2;
    op.out_mode = out_mode;
    op.tile_off = c->tiles_doubles;
    op.idx_off = idx_off;
    op.s_off = c->s_doubles;
    op.part_off = -1;
    const int opi = (int)c->ops.size();
    for (int bi = 0; bi < op.nblk; ++bi)
        for (int bj = 0; bj <= bi; ++bj) {
            ItemDesc it{};
            it.op = opi;
            it.I0 = bi * op.BT;
            it.I1 = std::min(op.nT, (bi + 1) * op.BT);
            it.J0 = bj * op.BT;
            it.J1 = std::min(op.nT, (bj + 1) * op.BT);
            it.tri = (bi == bj);
            const int h = it.I1 - it.I0, wd = it.J1 - it.J0;
            it.ntiles = it.tri ? h * (h + 1) / 2 : h * wd;
            // compact last tile row (ddg_internal.h) for whole-operator triangles
            it.tail = (compact && op.nblk == 1 && m % TILE) ? m % TILE : 0;
            it.tile_off = c->tiles_doubles;
            c->tiles_doubles += item_doubles(it.tri, h, it.ntiles, it.tail);
            if (op.nitems > 1) {
                it.part_off = c->part_doubles;
                c->part_doubles += (int64_t)(h + (it.tri ? 0 : wd)) * TILE;
            } else {
                it.part_off = -1;
            }
            c->items.push_back(it);
        }
    if (op.nitems > 1)
        for (int b = 0; b < op.nblk; ++b) c->red.push_back(RedDesc{opi, b});
    c->s_doubles += op.mp;
    c->ops.push_back(op);
}

// ddg_stencil (include/ddg.h): check that it reproduces every CSR row exactly
// and build the device description (CONST points sorted into column order).
// DDG_STENCIL_NODE27: the class table from the CSR, every row checked against it
static int build_node27(const ddg_stencil* S, int64_t n, const int64_t* rp, const int32_t* col, const double* val,
                        DevStencil& D, std::vector<double>& table) {
    const int64_t nx = S->dims[0], ny = S->dims[1], nz = S->dims[2], dof = S->npts;
    if (dof < 1 || dof > 4 || nx < 1 || ny < 1 || nz < 1 || nx * ny * nz * dof != n)
        return set_err(DDG_E_ARG, "node27 stencil: dims %lld x %lld x %lld x %lld unknowns per node != n = %lld",
                       (long long)nx, (long long)ny, (long long)nz, (long long)dof, (long long)n);
    D.kind = 3;
    D.nx = (int32_t)nx;
    D.ny = (int32_t)ny;
    D.nz = (int32_t)nz;
    D.dof = (int32_t)dof;
    const size_t per_class = 27 * (size_t)dof * dof;
    table.assign(27 * per_class, 0.0);
    std::vector<int64_t> rep(27, -1);               // the node whose rows define each class
    auto cls_of = [&](int64_t ix, int64_t iy, int64_t iz) {
        return (int)((ix == 0 ? 0 : ix == nx - 1 ? 2 : 1) + 3 * (iy == 0 ? 0 : iy == ny - 1 ? 2 : 1) +
                     9 * (iz == 0 ? 0 : iz == nz - 1 ? 2 : 1));
    };
    // expected columns of row (node, d) and the table slot of each, in CSR order
    auto walk = [&](int64_t node, const std::function<bool(int64_t colv, size_t slot)>& f) {
        const int64_t ix = node % nx, iy = (node / nx) % ny, iz = node / (nx * ny);
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (ix + dx < 0 || ix + dx >= nx || iy + dy < 0 || iy + dy >= ny || iz + dz < 0 || iz + dz >= nz)
                        continue;
                    const int o = (dx + 1) + 3 * ((dy + 1) + 3 * (dz + 1));
                    const int64_t nb = node + dx + nx * (dy + ny * (int64_t)dz);
                    for (int e = 0; e < dof; ++e)
                        if (!f(nb * dof + e, (size_t)o * dof * dof + e)) return false;
                }
        return true;
    };
    const int64_t nnode = nx * ny * nz;
    for (int64_t node = 0; node < nnode; ++node) {   // first node of each class fills its table rows
        const int cl = cls_of(node % nx, (node / nx) % ny, node / (nx * ny));
        if (rep[cl] >= 0) continue;
        rep[cl] = node;
        for (int d = 0; d < dof; ++d) {
            const int64_t v = node * dof + d;
            int64_t k = rp[v];
            const bool ok = walk(node, [&](int64_t colv, size_t slot) {
                if (k >= rp[v + 1] || col[k] != colv) return false;
                table[cl * per_class + slot + (size_t)d * dof] = val[k++];
                return true;
            });
            if (!ok || k != rp[v + 1])
                return set_err(DDG_E_ARG, "node27 stencil: row %lld is not a full 27-point node row", (long long)v);
        }
    }
    std::atomic<int64_t> bad{-1};
    parallel_for(nnode, [&](int64_t b, int64_t e, int) {
        for (int64_t node = b; node < e && bad.load() < 0; ++node) {
            const int cl = cls_of(node % nx, (node / nx) % ny, node / (nx * ny));
            for (int d = 0; d < dof; ++d) {
                const int64_t v = node * dof + d;
                int64_t k = rp[v];
                const bool ok = walk(node, [&](int64_t colv, size_t slot) {
                    const bool same = k < rp[v + 1] && col[k] == colv &&
                                      val[k] == table[cl * per_class + slot + (size_t)d * dof];
                    ++k;
                    return same;
                });
                if (!ok || k != rp[v + 1]) {
                    int64_t exp = -1;
                    bad.compare_exchange_strong(exp, v);
                }
            }
        }
    });
    if (bad.load() >= 0)
        return set_err(DDG_E_ARG, "node27 stencil does not reproduce row %lld of the CSR matrix", (long long)bad.load());
    return DDG_OK;
}

static int build_stencil(ddg_ctx* c, const ddg_stencil* S, int64_t n, const int64_t* rp, const int32_t* col,
                         const double* val, DevStencil& D, std::vector<double>& coef) {
    D = DevStencil{};
    if (!S || S->kind == DDG_STENCIL_NONE) return DDG_OK;
    const int64_t nx = S->dims[0], ny = S->dims[1], nz = S->dims[2];
    if (S->kind == DDG_STENCIL_NODE27) return build_node27(S, n, rp, col, val, D, coef);
    if (nx < 1 || ny < 1 || nz < 1 || nx * ny * nz != n)
        return set_err(DDG_E_ARG, "stencil dims %lld x %lld x %lld do not match n = %lld", (long long)nx,
                       (long long)ny, (long long)nz, (long long)n);
    D.nx = (int32_t)nx;
    D.ny = (int32_t)ny;
    D.nz = (int32_t)nz;
    std::vector<int> ord;
    if (S->kind == DDG_STENCIL_CONST) {
        if (S->npts < 1 || S->npts > STENCIL_MAX_PTS || !S->offsets || !S->coef)
            return set_err(DDG_E_ARG, "stencil: npts = %d (1..%d) and offsets/coef required", S->npts,
                           STENCIL_MAX_PTS);
        D.kind = 1;
        D.npts = S->npts;
        ord.resize(S->npts);
        std::iota(ord.begin(), ord.end(), 0);
        auto lin = [&](int k) {
            return S->offsets[3 * k] + nx * (S->offsets[3 * k + 1] + ny * (int64_t)S->offsets[3 * k + 2]);
        };
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lin(a) < lin(b); });
        for (int q = 0; q < S->npts; ++q) {
            const int k = ord[q];
            D.dx[q] = S->offsets[3 * k];
            D.dy[q] = S->offsets[3 * k + 1];
            D.dz[q] = S->offsets[3 * k + 2];
            D.c[q] = S->coef[k];
            const int64_t lo = lin(k);
            if (lo < INT32_MIN || lo > INT32_MAX) return set_err(DDG_E_ARG, "stencil offset out of range");
            D.off[q] = (int32_t)lo;
            D.rx = std::max(D.rx, std::abs(D.dx[q]));
            D.ry = std::max(D.ry, std::abs(D.dy[q]));
            D.rz = std::max(D.rz, std::abs(D.dz[q]));
        }
    } else if (S->kind == DDG_STENCIL_FACE7) {
        if (!S->coef) return set_err(DDG_E_ARG, "stencil: coef (4 n values) required");
        D.kind = 2;
        coef.assign(S->coef, S->coef + 4 * n);
    } else {
        return set_err(DDG_E_ARG, "stencil: unknown kind %d", S->kind);
    }
    // exact reproduction of the CSR, row by row
    std::atomic<int64_t> bad{-1};
    parallel_for(n, [&](int64_t b, int64_t e, int) {
        std::vector<std::pair<int64_t, double>> ent;
        for (int64_t v = b; v < e && bad.load() < 0; ++v) {
            const int64_t ix = v % nx, iy = (v / nx) % ny, iz = v / (nx * ny);
            ent.clear();
            if (D.kind == 1) {
                for (int q = 0; q < D.npts; ++q) {
                    const int64_t a = ix + D.dx[q], bb = iy + D.dy[q], cc = iz + D.dz[q];
                    if (a >= 0 && a < nx && bb >= 0 && bb < ny && cc >= 0 && cc < nz)
                        ent.push_back({v + D.dx[q] + nx * (D.dy[q] + ny * (int64_t)D.dz[q]), D.c[q]});
                }
            } else {
                const double* Dg = coef.data();
                const double *CX = Dg + n, *CY = CX + n, *CZ = CY + n;
                const int64_t sy = nx, sz = nx * ny;
                if (iz > 0) ent.push_back({v - sz, CZ[v - sz]});
                if (iy > 0) ent.push_back({v - sy, CY[v - sy]});
                if (ix > 0) ent.push_back({v - 1, CX[v - 1]});
                ent.push_back({v, Dg[v]});
                if (ix + 1 < nx) ent.push_back({v + 1, CX[v]});
                if (iy + 1 < ny) ent.push_back({v + sy, CY[v]});
                if (iz + 1 < nz) ent.push_back({v + sz, CZ[v]});
            }
            bool ok = (int64_t)ent.size() == rp[v + 1] - rp[v];
            for (size_t k = 0; ok && k < ent.size(); ++k)
                ok = col[rp[v] + k] == ent[k].first && val[rp[v] + k] == ent[k].second;
            if (!ok) {
                int64_t exp = -1;
                bad.compare_exchange_strong(exp, v);
            }
        }
    });
    if (bad.load() >= 0)
        return set_err(DDG_E_ARG, "stencil does not reproduce row %lld of the CSR matrix", (long long)bad.load());
    (void)c;
    return DDG_OK;
}

// Contiguous partition of n weighted items over G parts: out[0] = 0,
// out[G] = n, non-decreasing; part g starts at the item whose weight prefix
// pre[] (n + 1 entries, pre[0] = 0) is nearest to g/G of the total.
static void balanced_partition(const double* pre, int n, int G, int32_t* out) {
    out[0] = 0;
    int cur = 0;
    for (int g = 1; g < G; ++g) {
        const double target = pre[n] * g / G;
        while (cur < n && pre[cur + 1] <= target) ++cur;
        int pick = cur;
        if (cur < n && target - pre[cur] > pre[cur + 1] - target) pick = cur + 1;
        out[g] = std::max(pick, out[g - 1]);
    }
    out[G] = n;
}

// debug / test export (not part of include/ddg.h): balanced_partition of
// weights w[0..n) into G parts, out[0..G]
extern "C" int ddg_debug_partition(const double* w, int n, int G, int32_t* out) {
    if (!w || !out || n < 0 || G < 1) return DDG_E_ARG;
    std::vector<double> pre(n + 1, 0.0);
    for (int i = 0; i < n; ++i) pre[i + 1] = pre[i] + w[i];
    balanced_partition(pre.data(), n, G, out);
    return DDG_OK;
}

// Byte-balanced contiguous partition of items [b, e) over the persistent
// k_symv_ring CTAs (one per SM): CTA g gets the items whose byte prefix starts
// nearest to g/G of the total (each item weighted by its bytes plus 8 KB for
// its fixed per-item work).
int ring_partition(ddg_ctx* c, int b, int e) {
    if (e <= b) return -1;
    const int G = num_sms();
    std::vector<double> pre(e - b + 1, 0.0);
    int mr = 0, mc = 0;
    for (int i = b; i < e; ++i) {
        const ItemDesc& d = c->items[i];
        const int rows = (d.I1 - d.I0 + (d.tri ? 0 : d.J1 - d.J0)) * TILE;
        if (rows > RING_MAX_ROWS) return -1;
        mr = std::max(mr, (d.I1 - d.I0) * TILE);
        if (!d.tri) mc = std::max(mc, (d.J1 - d.J0) * TILE);
        pre[i - b + 1] = pre[i - b] + item_doubles(d.tri, d.I1 - d.I0, d.ntiles, d.tail) * 8.0 + 8192.0;
    }
    const int off = (int)c->h_ring.size();
    c->h_ring.resize(off + G + 1);
    balanced_partition(pre.data(), e - b, G, c->h_ring.data() + off);
    // small launches (C1, the upper coarse levels) stay on the per-item
    // kernel: the persistent ring's fixed cost (148 CTAs, ~200 KB shared
    // memory and barrier set-up each) outweighs its streaming advantage
    if (pre.back() < c->ring_min_bytes) {
        c->h_ring.resize(off);
        return -1;
    }
    c->ring_rc.push_back({off, {mr, mc}});
    return off;
}
void ring_dims(const ddg_ctx* c, int off, int* max_rows_r, int* max_rows_c) {
    *max_rows_r = RING_MAX_ROWS;
    *max_rows_c = 0;
    for (const auto& e : c->ring_rc)
        if (e.first == off) {
            *max_rows_r = e.second.first;
            *max_rows_c = e.second.second;
        }
}
bool ring_ok(const ddg_ctx* c, int off) { return c->symv_mode == 0 && off >= 0; }

static int build_plans(ddg_ctx* c) {
    c->ops.clear();
    c->items.clear();
    c->red.clear();
    c->plans.assign(c->ncolours, ColourPlan{});
    // subdomain operators in sweep order; the index lists are stored in that order
    std::vector<int32_t> sorted_idx;
    sorted_idx.reserve(c->oidx.size());
    int pos = 0;
    c->op_sub.clear();
    for (int cc = 0; cc < c->ncolours; ++cc) {
        ColourPlan& pl = c->plans[cc];
        pl.sub_begin = (int)c->ops.size();
        pl.item_begin = (int)c->items.size();
        pl.red_begin = (int)c->red.size();
        pl.max_rows = 0;
        // compact last tile rows (ddg_internal.h, DDG_COMPACT) only in colours
        // whose operators are all whole triangles: the rectangle items of split
        // operators are read as full tiles
        bool compact = g_compact != 0;
        {
            const int single_max = getenv("DDG_SINGLE_MAX_NT") ? atoi(getenv("DDG_SINGLE_MAX_NT")) : MAX_BT;
            int64_t max_nt = 0;
            for (int q = pos; q < c->nparts && c->colour[c->order[q]] == cc; ++q) {
                const int i = c->order[q];
                const int64_t m = c->optr[i + 1] - c->optr[i];
                if ((m + TILE - 1) / TILE > single_max) compact = false;
                max_nt = std::max<int64_t>(max_nt, (m + TILE - 1) / TILE);
            }
            // colours of small triangles (nT <= 5) run k_symv_whole on full tiles
            if (max_nt <= 5) compact = false;
        }
        // this rank's subdomains of the colour; with several ranks, those whose
        // writes another rank reads (the colour's z halo) first
        std::vector<int> subs;
        while (pos < c->nparts && c->colour[c->order[pos]] == cc) {
            const int i = c->order[pos++];
            if (c->dist && c->plan.part_rank[i] != c->rank) continue;   // another rank's
            subs.push_back(i);
        }
        int nbound = (int)subs.size();
        static const bool no_split = getenv("DDG_NO_BOUNDARY_FIRST") && atoi(getenv("DDG_NO_BOUNDARY_FIRST")) != 0;
        if (c->dist && c->nranks > 1 && !no_split) {
            std::vector<char> sent(c->n, 0);
            for (int h = 0; h < c->nranks; ++h)
                for (int32_t v : c->plan.z_send[(size_t)cc * c->nranks + h]) sent[v] = 1;
            auto is_b = [&](int i) {
                for (int64_t a = c->optr[i]; a < c->optr[i + 1]; ++a)
                    if (sent[c->oidx[a]]) return true;
                return false;
            };
            auto mid = std::stable_partition(subs.begin(), subs.end(), is_b);
            nbound = (int)(mid - subs.begin());
        }
        for (size_t qq = 0; qq < subs.size(); ++qq) {
            if ((int)qq == nbound) {
                pl.sub_mid = (int)c->ops.size();
                pl.item_mid = (int)c->items.size();
                pl.red_mid = (int)c->red.size();
            }
            const int i = subs[qq];
            const int64_t m = c->optr[i + 1] - c->optr[i];
            c->op_sub.push_back(i);
            const int64_t off = (int64_t)sorted_idx.size();
            sorted_idx.insert(sorted_idx.end(), c->oidx.begin() + c->optr[i],
                              c->oidx.begin() + c->optr[i + 1]);
            // every list starts 16-byte aligned (k_symv_whole bulk-copies it)
            while (sorted_idx.size() % 4) sorted_idx.push_back(0);
            if (c->chol) {
                // Cholesky factor (chol.cu): nT (nT + 1) / 2 full tiles at tile_off,
                // no SYMV items read, no partial segments
                const int64_t t0 = c->tiles_doubles, p0 = c->part_doubles;
                add_op(c, (int32_t)m, 0, off, true, false);
                OpDesc& op = c->ops.back();
                op.tile_off = t0;
                c->tiles_doubles = t0 + chol_doubles(op.nT);
                c->part_doubles = p0;
            } else {
                add_op(c, (int32_t)m, 0, off, true, compact);
            }
            pl.max_rows = std::max<int>(pl.max_rows, (int)m);
        }
        pl.sub_end = (int)c->ops.size();
        pl.item_end = (int)c->items.size();
        if (nbound >= (int)subs.size() || nbound == 0) {   // nothing to overlap
            pl.sub_mid = pl.sub_end;
            pl.item_mid = pl.item_end;
            pl.red_mid = -1;
        }
        pl.max_rows_t = 0;
        pl.all_single = 1;
        pl.max_ntiles = 0;
        for (int q = pl.sub_begin; q < pl.sub_end; ++q)
            if (c->ops[q].nitems != 1) pl.all_single = 0;
        for (int it = pl.item_begin; it < pl.item_end; ++it) {
            const ItemDesc& d = c->items[it];
            pl.max_rows_t = std::max(pl.max_rows_t, (d.I1 - d.I0 + (d.tri ? 0 : d.J1 - d.J0)) * TILE);
            pl.max_ntiles = std::max(pl.max_ntiles, d.ntiles);
        }
        pl.red_end = (int)c->red.size();
        if (pl.red_mid < 0) pl.red_mid = pl.red_end;
        pl.ring_off = ring_partition(c, pl.item_begin, pl.item_end);
        pl.ring_b = pl.ring_i = -1;
        if (pl.sub_mid < pl.sub_end) {
            pl.ring_b = ring_partition(c, pl.item_begin, pl.item_mid);
            pl.ring_i = ring_partition(c, pl.item_mid, pl.item_end);
        }
    }
    c->oidx.swap(sorted_idx);  // now in sweep order; optr no longer valid for oidx
    c->colour_alg_bytes.assign(c->ncolours, 0.0);
    for (int cc = 0; cc < c->ncolours; ++cc)
        for (int q = c->plans[cc].sub_begin; q < c->plans[cc].sub_end; ++q) {
            const double m = c->ops[q].m;   // local operators of this rank
            c->colour_alg_bytes[cc] += 8.0 * m * (m + 1) / 2 + 24.0 * m;
        }
    if (c->coarse_variant != 1) return DDG_OK;
    // dense coarse inverse
    c->coarse_op = (int)c->ops.size();
    c->coarse_item_begin = (int)c->items.size();
    c->coarse_red_begin = (int)c->red.size();
    add_op(c, (int32_t)c->nc, 1, -1, true);
    c->coarse_item_end = (int)c->items.size();
    for (int it = c->coarse_item_begin; it < c->coarse_item_end; ++it) {
        const ItemDesc& d = c->items[it];
        c->coarse_rows_t = std::max(c->coarse_rows_t, (d.I1 - d.I0 + (d.tri ? 0 : d.J1 - d.J0)) * TILE);
    }
    c->coarse_red_end = (int)c->red.size();
    c->coarse_ring_off = ring_partition(c, c->coarse_item_begin, c->coarse_item_end);
    return DDG_OK;
}

// ---------------------------------------------------------------------------
// device setup: local inverses and the coarse inverse
// ---------------------------------------------------------------------------
static int invert_locals(ddg_ctx* c) {
    const int np = (int)c->op_sub.size();
    if (np == 0) return DDG_OK;
    size_t freeb = 0, totb = 0;
    CUDA_TRY(cudaMemGetInfo(&freeb, &totb));
    int64_t budget = std::min<int64_t>((int64_t)freeb / 4, (int64_t)8 << 30);
    budget = std::max<int64_t>(budget, (int64_t)64 << 20);
    double* scratch = nullptr;
    int64_t max_single = 0;
    for (int q = 0; q < np; ++q) max_single = std::max<int64_t>(max_single, (int64_t)c->ops[q].mp * c->ops[q].mp);
    const int64_t cap = std::max<int64_t>(budget / 8, max_single);
    int st = dalloc(&scratch, cap);
    if (st) return st;
    int32_t *d_ids = nullptr, *d_err = nullptr, *d_nT = nullptr, *d_ids2 = nullptr, *d_nT2 = nullptr;
    int64_t* d_soff = nullptr;
    double **d_ptr = nullptr, **d_ptr2 = nullptr;
    if ((st = dalloc(&d_ids, np)) || (st = dalloc(&d_soff, np)) || (st = dalloc(&d_err, 2)) ||
        (st = dalloc(&d_nT, np)) || (st = dalloc(&d_ptr, np)) || (st = dalloc(&d_ids2, np)) ||
        (st = dalloc(&d_nT2, np)) || (st = dalloc(&d_ptr2, np))) {
        cudaFree(scratch);
        return st;
    }
    int32_t herr[2] = {-1, -1};
    { int _s = h2d(c->stream, d_err, herr, sizeof herr); if (_s) return _s; }
    std::vector<int32_t> ids, nTs;
    std::vector<int64_t> soff;
    std::vector<double*> ptrs;
    int q = 0;
    while (q < np) {
        ids.clear();
        soff.clear();
        nTs.clear();
        ptrs.clear();
        int64_t used = 0;
        while (q < np && (ids.empty() || used + (int64_t)c->ops[q].mp * c->ops[q].mp <= cap)) {
            ids.push_back(q);
            soff.push_back(used);
            nTs.push_back(c->ops[q].nT);
            ptrs.push_back(scratch + used);
            used += (int64_t)c->ops[q].mp * c->ops[q].mp;
            ++q;
        }
        const size_t nb = ids.size();
        CUDA_TRY(cudaMemcpyAsync(d_ids, ids.data(), nb * 4, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(d_soff, soff.data(), nb * 8, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(d_nT, nTs.data(), nb * 4, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(d_ptr, ptrs.data(), nb * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
        launch_extract_local(c->stream, (int)nb, d_ids, c->d_ops, c->d_oidx, c->A, scratch, d_soff);
        // small operators: one CTA each (tile exchange); operators of >= GJB_MIN_T
        // tiles: blocked exchange with fp64 GEMM updates (entries [nsmall, nb))
        {
            std::vector<int> order(nb);
            std::iota(order.begin(), order.end(), 0);
            std::stable_partition(order.begin(), order.end(), [&](int i) { return nTs[i] < GJB_MIN_T; });
            std::vector<int32_t> oids(nb), onT(nb);
            std::vector<double*> optr(nb);
            int nsmall = 0, maxT = 0;
            for (size_t i = 0; i < nb; ++i) {
                oids[i] = ids[order[i]];
                onT[i] = nTs[order[i]];
                optr[i] = ptrs[order[i]];
                if (onT[i] < GJB_MIN_T) ++nsmall;
                else maxT = std::max(maxT, onT[i]);
            }
            CUDA_TRY(cudaMemcpyAsync(d_ids2, oids.data(), nb * 4, cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(cudaMemcpyAsync(d_nT2, onT.data(), nb * 4, cudaMemcpyHostToDevice, c->stream));
            CUDA_TRY(cudaMemcpyAsync(d_ptr2, optr.data(), nb * sizeof(double*), cudaMemcpyHostToDevice, c->stream));
            if (c->chol) {
                launch_chol_local(c->stream, (int)nb, d_nT2, d_ptr2, d_ids2, d_err);
                nsmall = (int)nb;
            } else if (nsmall) {
                launch_gj_batched(c->stream, nsmall, d_nT2, d_nT2, d_ptr2, d_ids2, d_err);
            }
            if ((int)nb > nsmall)
                launch_gj_blocked(c->stream, (int)nb - nsmall, maxT, maxT, d_ptr2 + nsmall, d_nT2 + nsmall,
                                  d_nT2 + nsmall, d_ids2 + nsmall, d_err);
        }
        if (c->chol) {
            int maxT = 0;
            for (int32_t t : nTs) maxT = std::max(maxT, (int)t);
            launch_chol_pack(c->stream, (int)nb, maxT * (maxT + 1) / 2, d_ids, c->d_ops, scratch, d_soff, c->d_tiles);   // tiles of the largest
        } else {
            launch_pack(c->stream, (int)nb, d_ids, c->d_ops, c->d_items, scratch, d_soff, c->d_tiles);
        }
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    { int _s = d2h(c->stream, herr, d_err, sizeof herr); if (_s) return _s; }
    cudaFree(scratch);
    cudaFree(d_ids);
    cudaFree(d_soff);
    cudaFree(d_err);
    cudaFree(d_nT);
    cudaFree(d_ptr);
    cudaFree(d_ids2);
    cudaFree(d_nT2);
    cudaFree(d_ptr2);
    if (herr[0] >= 0)
        return set_err(DDG_E_NOT_SPD,
                       c->chol ? "local Cholesky: subdomain %d not positive definite at pivot %d"
                               : "local inverse: subdomain %d not positive definite at pivot %d",
                       c->op_sub[herr[0]], herr[1]);
    return DDG_OK;
}

static int invert_coarse(ddg_ctx* c, const std::vector<int32_t>& er, const std::vector<int32_t>& ec,
                         const std::vector<double>& ev) {
    const OpDesc& op = c->ops[c->coarse_op];
    const int64_t tot = (int64_t)op.mp * op.mp;
    double* M = nullptr;
    int32_t *d_r = nullptr, *d_c = nullptr, *d_err = nullptr, *d_ids = nullptr, *d_nT = nullptr;
    double* d_v = nullptr;
    int64_t* d_soff = nullptr;
    double** d_ptr = nullptr;
    int st;
    if ((st = dalloc(&M, tot)) || (st = dalloc(&d_r, er.size())) || (st = dalloc(&d_c, ec.size())) ||
        (st = dalloc(&d_v, ev.size())) || (st = dalloc(&d_err, 2)) || (st = dalloc(&d_ids, 1)) ||
        (st = dalloc(&d_soff, 1)) || (st = dalloc(&d_nT, 1)) || (st = dalloc(&d_ptr, 1)))
        return st;
    int32_t herr[2] = {-1, -1};
    int32_t id = c->coarse_op, nT = op.nT;
    int64_t zero = 0;
    CUDA_TRY(cudaMemsetAsync(M, 0, tot * sizeof(double), c->stream));
    { int _s = h2d(c->stream, d_r, er.data(), er.size() * 4); if (_s) return _s; }
    { int _s = h2d(c->stream, d_c, ec.data(), ec.size() * 4); if (_s) return _s; }
    { int _s = h2d(c->stream, d_v, ev.data(), ev.size() * 8); if (_s) return _s; }
    { int _s = h2d(c->stream, d_err, herr, sizeof herr); if (_s) return _s; }
    { int _s = h2d(c->stream, d_ids, &id, 4); if (_s) return _s; }
    { int _s = h2d(c->stream, d_soff, &zero, 8); if (_s) return _s; }
    { int _s = h2d(c->stream, d_nT, &nT, 4); if (_s) return _s; }
    { int _s = h2d(c->stream, d_ptr, &M, sizeof(double*)); if (_s) return _s; }
    launch_scatter_coarse(c->stream, (int64_t)ev.size(), d_r, d_c, d_v, op.nT, op.m, M);
    if (op.nT < GJB_MIN_T) launch_gj_batched(c->stream, 1, d_nT, d_nT, d_ptr, d_ids, d_err);
    else launch_gj_blocked(c->stream, 1, op.nT, op.nT, d_ptr, d_nT, d_nT, d_ids, d_err);
    launch_pack(c->stream, 1, d_ids, c->d_ops, c->d_items, M, d_soff, c->d_tiles);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    { int _s = d2h(c->stream, herr, d_err, sizeof herr); if (_s) return _s; }
    cudaFree(M); cudaFree(d_r); cudaFree(d_c); cudaFree(d_v); cudaFree(d_err); cudaFree(d_ids);
    cudaFree(d_soff); cudaFree(d_nT); cudaFree(d_ptr);
    if (herr[0] >= 0)
        return set_err(DDG_E_NOT_SPD, "coarse inverse: A_c not positive definite at pivot %d", herr[1]);
    return DDG_OK;
}

// Three levels: "taking the two-level algorithm and
// applying it again to the coarse matrix A_0", with "F_0 = R_0 F".  The
// second level is an ordinary two-level context on A_c (host CSR built from
// the Galerkin triplets, structural pattern = part adjacency, reading R19),
// F_0 = blockdiag(Q_I^T) F, coarse unknown (I,i) in part part2[I] (R20), the
// same Delta and rank tolerance, on this context's device and stream.
static int build_child(ddg_ctx* c, const double* F, const std::vector<int32_t>& er,
                       const std::vector<int32_t>& ec, const std::vector<double>& ev) {
    const int64_t nc = c->nc;
    const int k = c->k;
    const int32_t* part2 = c->opts.part2;
    const int np2 = c->opts.nparts2;
    // CSR of A_c, both triangles, columns increasing
    std::vector<int64_t> rp(nc + 1, 0);
    for (size_t e = 0; e < er.size(); ++e) {
        rp[er[e] + 1]++;
        if (er[e] != ec[e]) rp[ec[e] + 1]++;
    }
    for (int64_t i = 0; i < nc; ++i) rp[i + 1] += rp[i];
    if (rp[nc] >= (int64_t)INT32_MAX) return set_err(DDG_E_ARG, "A_c has too many entries for three levels");
    std::vector<int32_t> col(rp[nc]);
    std::vector<double> val(rp[nc]);
    {
        std::vector<int64_t> fill(rp.begin(), rp.end() - 1);
        for (size_t e = 0; e < er.size(); ++e) {
            col[fill[er[e]]] = ec[e];
            val[fill[er[e]]++] = ev[e];
            if (er[e] != ec[e]) {
                col[fill[ec[e]]] = er[e];
                val[fill[ec[e]]++] = ev[e];
            }
        }
        parallel_for(nc, [&](int64_t b, int64_t e, int) {
            std::vector<std::pair<int32_t, double>> row;
            for (int64_t i = b; i < e; ++i) {
                row.clear();
                for (int64_t x = rp[i]; x < rp[i + 1]; ++x) row.push_back({col[x], val[x]});
                std::sort(row.begin(), row.end(),
                          [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b2) {
                              return a.first < b2.first;
                          });
                for (int64_t x = rp[i]; x < rp[i + 1]; ++x) {
                    col[x] = row[x - rp[i]].first;
                    val[x] = row[x - rp[i]].second;
                }
            }
        });
    }
    // F_0 = R_0 F (column-major nc x k) and the second-level partition
    std::vector<double> F0((size_t)nc * k);
    std::vector<int32_t> p0(nc);
    parallel_for(c->nparts, [&](int64_t b, int64_t e, int) {
        for (int64_t I = b; I < e; ++I) {
            const int64_t mI = c->bptr[I + 1] - c->bptr[I];
            const int32_t* rows = c->bidx.data() + c->bptr[I];
            for (int i = 0; i < c->cptr[I + 1] - c->cptr[I]; ++i) {
                const double* q = c->Q.data() + c->qoff[I] + (int64_t)i * mI;
                for (int l = 0; l < k; ++l) {
                    double sum = 0;
                    for (int64_t a = 0; a < mI; ++a) sum += q[a] * F[(int64_t)l * c->n + rows[a]];
                    F0[(size_t)l * nc + c->cptr[I] + i] = sum;
                }
                p0[c->cptr[I] + i] = part2[I];
            }
        }
    });
    ddg_opts o = c->opts;
    o.stream = c->stream;
    o.comm = c->opts.comm;     // multi-GPU: the second level is distributed over the same ranks
    o.stencil = nullptr;
    o.part2 = nullptr;
    o.nparts2 = 0;
    o.block_coords = c->opts.block_coords2;
    o.block_ndim = c->opts.block_coords2 ? c->opts.block_ndim : 0;
    o.block_coords2 = nullptr;
    o.coarse_variant = c->opts.coarse_variant;   // selects the last level's coarse solve
    int st = ddg_setup(nc, rp.data(), col.data(), val.data(), F0.data(), k, p0.data(), np2, &o, &c->child);
    if (st) return st;   // the child's message stands
    return DDG_OK;
}

// Node-blocked column structure (DevCSR::bs): n % bs == 0 and the bs rows of
// every block-row share one column list made of whole aligned bs-blocks.
static bool node_blocks(int64_t n, const int64_t* rp, const int32_t* col, int bs, std::vector<int32_t>& brp,
                        std::vector<int32_t>& bcol) {
    if (n % bs) return false;
    const int64_t nbr = n / bs;
    brp.assign(nbr + 1, 0);
    bcol.clear();
    for (int64_t V = 0; V < nbr; ++V) {
        const int64_t v0 = V * bs;
        const int64_t len = rp[v0 + 1] - rp[v0];
        if (len % bs) return false;
        for (int64_t j = 0; j < len; j += bs) {
            const int32_t c0 = col[rp[v0] + j];
            if (c0 % bs) return false;
            bcol.push_back(c0 / bs);
        }
        for (int r = 0; r < bs; ++r) {
            const int64_t v = v0 + r;
            if (rp[v + 1] - rp[v] != len) return false;
            for (int64_t j = 0; j < len; ++j)
                if (col[rp[v] + j] != bcol[brp[V] + j / bs] * bs + (int32_t)(j % bs)) return false;
        }
        brp[V + 1] = (int32_t)bcol.size();
    }
    return true;
}

template <typename T>
static int upload_s(cudaStream_t s, T** d, const std::vector<T>& h) {
    int st = dalloc(d, h.size());
    if (st) return st;
    return h2d(s, *d, h.data(), h.size() * sizeof(T));
}
#define upload(d, h) upload_s(c->stream, d, h)

// Per-part orthonormal basis of F[Omega_I,:] on the device (basis.cu,
// PAPER.md:253-264; readings R6c, R7): cptr, qoff, d_Q, and the host copy of
// Q when the three-level child needs it (build_child).
static int device_basis(ddg_ctx* c, const double* F, int32_t* d_part) {
    (void)d_part;
    const int np = c->nparts, k = c->k;
    const int64_t n = c->n;
    std::vector<int64_t> voff(np + 1, 0);
    for (int I = 0; I < np; ++I) voff[I + 1] = voff[I] + (c->bptr[I + 1] - c->bptr[I]) * k;
    double *dF = nullptr, *dQw = nullptr, *dratio = nullptr;
    double2* dV = nullptr;
    int64_t* dvoff = nullptr;
    int32_t *drank = nullptr, *derr = nullptr;
    auto done = [&](int st) {
        cudaFree(dF); cudaFree(dQw); cudaFree(dratio); cudaFree(dV); cudaFree(dvoff); cudaFree(drank);
        cudaFree(derr);
        return st;
    };
    int st;
    if ((st = dalloc(&dF, (size_t)n * k)) || (st = h2d(c->stream, dF, F, (size_t)n * k * 8)) ||
        (st = upload(&dvoff, voff)) || (st = dalloc(&dV, (size_t)voff[np])) || (st = dalloc(&dQw, (size_t)voff[np])) ||
        (st = dalloc(&drank, np)) || (st = dalloc(&dratio, np)) || (st = dalloc(&derr, 1)))
        return done(st);
    const int32_t neg = -1;
    if ((st = h2d(c->stream, derr, &neg, 4))) return done(st);
    launch_basis_mgs(c->stream, np, k, n, dF, c->d_bptr, c->d_bidx, dvoff, dV, dQw, drank, dratio,
                     c->opts.rank_tol, derr);
    std::vector<int32_t> rank(np);
    std::vector<double> ratio(np);
    int32_t bad = -1;
    if ((st = d2h(c->stream, rank.data(), drank, np * 4)) || (st = d2h(c->stream, ratio.data(), dratio, np * 8)) ||
        (st = d2h(c->stream, &bad, derr, 4)))
        return done(st);
    if (bad >= 0) return done(set_err(DDG_E_ZERO_BLOCK, "coarse basis: F restricted to part %d is zero", bad));
    c->cptr.assign(np + 1, 0);
    c->qoff.assign(np + 1, 0);
    c->dropped = 0;
    for (int I = 0; I < np; ++I) {
        c->cptr[I + 1] = c->cptr[I] + rank[I];
        c->qoff[I + 1] = c->qoff[I] + (int64_t)rank[I] * (c->bptr[I + 1] - c->bptr[I]);
        c->dropped += k - rank[I];
        c->min_ratio = std::min(c->min_ratio, ratio[I]);
    }
    c->nc = c->cptr[np];
    if ((st = upload(&c->d_cptr, c->cptr)) || (st = upload(&c->d_qoff, c->qoff)) ||
        (st = dalloc(&c->d_Q, std::max<int64_t>(1, c->qoff[np]))))
        return done(st);
    launch_basis_compact(c->stream, np, c->d_bptr, dvoff, c->d_qoff, dQw, c->d_Q);
    CUDA_TRY(cudaGetLastError());
    if (c->opts.part2) {
        c->Q.resize(c->qoff[np]);
        if ((st = d2h(c->stream, c->Q.data(), c->d_Q, c->qoff[np] * 8))) return done(st);
    }
    return done(DDG_OK);
}

// Galerkin product A_c = P^T A P on the device (basis.cu), one
// block A_c[I, J] = Q_I^T A[Omega_I, Omega_J] Q_J per adjacent pair I >= J;
// triplets (row >= col only, reading R9) in (J, j, I, i) order for the coarse
// factorisation.
static int device_galerkin(ddg_ctx* c, const int64_t* rp, const int32_t* col, const int32_t* d_part,
                           const int32_t* d_bpos, std::vector<int32_t>& er, std::vector<int32_t>& ec,
                           std::vector<double>& ev) {
    const int np = c->nparts;
    // adjacent parts I >= J of every J (structural pattern of A)
    std::vector<std::vector<int32_t>> adj(np);
    const int nt = (int)std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
    std::vector<std::vector<int32_t>> marks(nt);
    parallel_for(np, [&](int64_t b, int64_t e, int t) {
        auto& mark = marks[t];
        if (mark.empty()) mark.assign(np, -1);
        for (int64_t J = b; J < e; ++J) {
            auto& L = adj[J];
            for (int64_t a = c->bptr[J]; a < c->bptr[J + 1]; ++a) {
                const int32_t v = c->bidx[a];
                for (int64_t x = rp[v]; x < rp[v + 1]; ++x) {
                    const int32_t I = c->part[col[x]];
                    if (I >= J && mark[I] != (int32_t)J) {
                        mark[I] = (int32_t)J;
                        L.push_back(I);
                    }
                }
            }
            std::sort(L.begin(), L.end());
        }
    });
    std::vector<int32_t> bI, bJ;
    std::vector<int64_t> boff(1, 0);
    int maxk = 1;
    for (int J = 0; J < np; ++J)
        for (int32_t I : adj[J]) {
            bI.push_back(I);
            bJ.push_back(J);
            boff.push_back(boff.back() + (int64_t)(c->cptr[I + 1] - c->cptr[I]) * (c->cptr[J + 1] - c->cptr[J]));
        }
    for (int I = 0; I < np; ++I) maxk = std::max(maxk, c->cptr[I + 1] - c->cptr[I]);
    const int nb = (int)bI.size();
    int32_t *dbI = nullptr, *dbJ = nullptr;
    int64_t* dboff = nullptr;
    double* dout = nullptr;
    auto done = [&](int st) {
        cudaFree(dbI); cudaFree(dbJ); cudaFree(dboff); cudaFree(dout);
        return st;
    };
    int st;
    if ((st = upload(&dbI, bI)) || (st = upload(&dbJ, bJ)) || (st = upload(&dboff, boff)) ||
        (st = dalloc(&dout, std::max<int64_t>(1, boff.back()))))
        return done(st);
    launch_galerkin_blocks(c->stream, nb, maxk, dbI, dbJ, dboff, c->d_bptr, c->d_bidx, c->d_cptr, c->d_qoff, c->d_Q,
                           d_part, d_bpos, c->d_rp, c->d_col, c->d_val, dout);
    CUDA_TRY(cudaGetLastError());
    std::vector<double> hb(boff.back());
    if ((st = d2h(c->stream, hb.data(), dout, hb.size() * 8))) return done(st);
    er.clear(); ec.clear(); ev.clear();
    er.reserve(hb.size()); ec.reserve(hb.size()); ev.reserve(hb.size());
    int64_t b0 = 0;
    for (int J = 0; J < np; ++J) {
        const int rJ = c->cptr[J + 1] - c->cptr[J];
        const int64_t nbJ = (int64_t)adj[J].size();
        for (int j = 0; j < rJ; ++j) {
            const int32_t cj = c->cptr[J] + j;
            for (int64_t q = 0; q < nbJ; ++q) {
                const int I = bI[b0 + q];
                const int rI = c->cptr[I + 1] - c->cptr[I];
                const double* blk = hb.data() + boff[b0 + q];
                for (int i = (I == J ? j : 0); i < rI; ++i) {
                    er.push_back(c->cptr[I] + i);
                    ec.push_back(cj);
                    ev.push_back(blk[(int64_t)i * rJ + j]);
                }
            }
        }
        b0 += nbJ;
    }
    return done(DDG_OK);
}

// Shared-memory plan of k_pcg_small (pcg.cu), the same walk the kernel makes:
// CTA g of G keeps its operators t = g, g + G, ... of every colour (tiles and
// index lists), tile row and column s = G - 1 - g of the coarse inverse
// (s < nT_c), and the Q_I blocks and row lists of its warps' parts
// I = g + G w (+ 8 G ...).
static int small_plan(ddg_ctx* c) {
    c->small_ok = false;
    if (c->dist || c->coarse_variant != 1 || c->n > 65536 || c->coarse_op < 0 ||
        c->coarse_item_end - c->coarse_item_begin != 1 || c->ncolours > 64)
        return DDG_OK;
    const int nTc = c->ops[c->coarse_op].nT;
    int maxmp = 32;
    for (size_t q = 0; q < c->op_sub.size(); ++q) {
        if (c->ops[q].nitems != 1 || c->ops[q].mp > 512) return DDG_OK;
        maxmp = std::max(maxmp, c->ops[q].mp);
    }
    for (int cc = 0; cc + 1 < c->ncolours; ++cc)
        if (c->plans[cc].sub_end != c->plans[cc + 1].sub_begin) return DDG_OK;
    const int PW = std::max(maxmp, c->maxmI);
    for (int G : {16, 8}) {
        if (nTc > G) continue;
        int64_t ad = 0, ai = 0;
        bool fits = true;
        for (int g = 0; g < G; ++g) {
            int64_t od = 0, oi = 0, nown = 0;
            for (int cc = 0; cc < c->ncolours; ++cc)
                for (int t = c->plans[cc].sub_begin + g; t < c->plans[cc].sub_end; t += G) {
                    const OpDesc& op = c->ops[t];
                    const ItemDesc& it = c->items[op.item_base];
                    od += (item_doubles(1, it.I1 - it.I0, it.ntiles, it.tail) + 1) & ~1;
                    oi += (op.m + 3) & ~3;
                    ++nown;
                }
            if (nown > 32) fits = false;
            if (G - 1 - g < nTc) od += (int64_t)(nTc - 1) * TILE_ELEMS + DIAG_ELEMS;
            for (int w = 0; w < 8; ++w)
                for (int I = g + G * w; I < c->nparts; I += G * 8) {
                    const int64_t mI = c->bptr[I + 1] - c->bptr[I];
                    od += (mI * (c->cptr[I + 1] - c->cptr[I]) + 1) & ~1;
                    oi += (mI + 3) & ~3;
                }
            ad = std::max(ad, od);
            ai = std::max(ai, oi);
        }
        const int ncp = nTc * TILE;
        const size_t smem = 8 * (size_t)(ad + 10 * (int64_t)PW + 2 * ncp) + 4 * (size_t)ai;
        fits = fits && smem <= 220 * 1024 && small_cluster_ok(G, smem);
        if (c->opts.verbose)
            fprintf(stderr, "[ddg_setup] k_pcg_small plan: G %d, %zu bytes of shared memory per CTA%s\n", G, smem,
                    fits ? "" : " (does not fit)");
        if (!fits) continue;
        std::vector<int32_t> cops(c->ncolours + 1);
        for (int cc = 0; cc < c->ncolours; ++cc) cops[cc] = c->plans[cc].sub_begin;
        cops[c->ncolours] = c->ncolours ? c->plans[c->ncolours - 1].sub_end : 0;
        int st = upload(&c->d_cops, cops);
        if (st) return st;
        c->small = SmallArgs{};
        c->small.ad = (int)ad;
        c->small.ai = (int)ai;
        c->small.pw = PW;
        c->small.ncp = ncp;
        c->small.nTc = nTc;
        c->small.G = G;
        c->small.smem = smem;
        c->small_ok = true;
        return DDG_OK;
    }
    return DDG_OK;
}

// ---------------------------------------------------------------------------
// ddg_setup
// ---------------------------------------------------------------------------
extern "C" int ddg_setup(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                         const double* F, int k, const int32_t* part, int32_t nparts,
                         const ddg_opts* opts, ddg_ctx** out) {
    if (!out) return set_err(DDG_E_ARG, "out is NULL");
    *out = nullptr;
    g_last_error.clear();
    if (n < 1 || !row_ptr || !col || !val || !F || !part || k < 1 || k > 128 || nparts < 1)
        return set_err(DDG_E_ARG, "bad argument (n=%lld k=%d nparts=%d)", (long long)n, k, nparts);
    if (n >= (int64_t)INT32_MAX) return set_err(DDG_E_ARG, "n=%lld too large for int32 indices", (long long)n);
    auto t0 = std::chrono::steady_clock::now();
    ddg_ctx* c = new ddg_ctx();
    if (opts) c->opts = *opts;
    else ddg_default_opts(&c->opts);
    if (c->opts.overlap < 0) { free_ctx(c); return set_err(DDG_E_ARG, "overlap < 0"); }
    if (c->opts.max_iter <= 0) c->opts.max_iter = 1000;
    if (c->opts.local_variant < DDG_LOCAL_AUTO || c->opts.local_variant > DDG_LOCAL_INVERSE) {
        int lv = c->opts.local_variant;
        free_ctx(c);
        return set_err(DDG_E_ARG, "local_variant %d not one of DDG_LOCAL_*", lv);
    }
    c->chol = c->opts.local_variant == DDG_LOCAL_CHOLESKY;
    c->n = n;
    c->k = k;
    c->nparts = nparts;
    c->nnz = row_ptr[n];
    if (row_ptr[0] != 0 || c->nnz < n) { free_ctx(c); return set_err(DDG_E_DIM, "row_ptr[0] != 0 or nnz < n"); }
    if (c->nnz >= (int64_t)INT32_MAX) { free_ctx(c); return set_err(DDG_E_ARG, "nnz too large"); }
    for (int64_t i = 0; i < n; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) { free_ctx(c); return set_err(DDG_E_DIM, "row_ptr decreasing at row %lld", (long long)i); }
        for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            if (col[e] < 0 || col[e] >= n) { free_ctx(c); return set_err(DDG_E_DIM, "column %d out of range in row %lld", col[e], (long long)i); }
            if (e > row_ptr[i] && col[e] <= col[e - 1]) { free_ctx(c); return set_err(DDG_E_DIM, "columns not strictly increasing in row %lld", (long long)i); }
        }
    }
    // parts Omega_I
    c->part.assign(part, part + n);
    c->bptr.assign(nparts + 1, 0);
    for (int64_t v = 0; v < n; ++v) {
        if (part[v] < 0 || part[v] >= nparts) {
            int pv = part[v];
            free_ctx(c);
            return set_err(DDG_E_PART, "part id %d of unknown %lld outside [0,%d)", pv, (long long)v, nparts);
        }
        c->bptr[part[v] + 1]++;
    }
    for (int I = 0; I < nparts; ++I) {
        if (c->bptr[I + 1] == 0) { free_ctx(c); return set_err(DDG_E_PART, "part %d is empty", I); }
        c->bptr[I + 1] += c->bptr[I];
    }
    c->bidx.resize(n);
    c->bpos.resize(n);
    {
        std::vector<int64_t> fill(c->bptr.begin(), c->bptr.end() - 1);
        for (int64_t v = 0; v < n; ++v) {
            const int I = part[v];
            c->bpos[v] = (int32_t)(fill[I] - c->bptr[I]);
            c->bidx[fill[I]++] = (int32_t)v;
        }
    }
    int st;
    // device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        free_ctx(c);
        return set_err(DDG_E_CUDA, "no CUDA device available (libddg has no CPU fallback)");
    }
    c->device = c->opts.device;
    if (cudaSetDevice(c->device) != cudaSuccess) {
        free_ctx(c);
        return set_err(DDG_E_CUDA, "cudaSetDevice(%d) failed", c->opts.device);
    }
    if (c->opts.comm && ((ddg_comm*)c->opts.comm)->loop) {
        // loopback virtual ranks share the group's stream; no graph capture
        // (another rank's thread enqueues on the same stream between collectives)
        c->stream = ddg::loop_stream((ddg_comm*)c->opts.comm);
        c->opts.use_graphs = 0;
    } else if (c->opts.stream) {
        c->stream = (cudaStream_t)c->opts.stream;
    } else {
        if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
            free_ctx(c);
            return set_err(DDG_E_CUDA, "stream creation failed");
        }
        c->own_stream = true;
    }
    auto tick = [&](const char* what) {
        if (c->opts.verbose) {
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            fprintf(stderr, "[ddg_setup] %-28s %8.3f s\n", what, s);
        }
    };
    build_overlap(c, row_ptr, col);
    tick("overlap");
    if ((st = build_colours(c, row_ptr, col))) { free_ctx(c); return st; }
    c->opts.colour = nullptr;   // borrowed for the duration of ddg_setup only
    tick("colours");
    if (c->opts.block_coords && c->opts.block_ndim > 0)
        c->block_coords.assign(c->opts.block_coords, c->opts.block_coords + (int64_t)nparts * c->opts.block_ndim);
    c->block_ndim = c->opts.block_ndim;
    if (c->opts.comm) {
        c->comm = (ddg_comm*)c->opts.comm;
        c->dist = true;
        c->rank = c->comm->rank;
        c->nranks = c->comm->nranks;
        ddg::build_dist_plan(c->plan, n, row_ptr, col, part, nparts, c->bptr.data(), c->bidx.data(),
                             c->optr.data(), c->oidx.data(), c->colour.data(), c->ncolours,
                             c->block_coords.empty() ? nullptr : c->block_coords.data(), c->block_ndim, c->rank,
                             c->nranks);
        tick("decomposition plan");
    }
    // A, the parts and the row positions on the device: the coarse space is
    // built there (basis.cu), and the hot path keeps A, bptr and bidx
    {
        std::vector<int32_t> rp32(n + 1);
        for (int64_t i = 0; i <= n; ++i) rp32[i] = (int32_t)row_ptr[i];
        if ((st = upload(&c->d_rp, rp32)) || (st = dalloc(&c->d_col, c->nnz)) || (st = dalloc(&c->d_val, c->nnz)) ||
            (st = h2d(c->stream, c->d_col, col, c->nnz * 4)) || (st = h2d(c->stream, c->d_val, val, c->nnz * 8)) ||
            (st = upload(&c->d_bptr, c->bptr)) || (st = upload(&c->d_bidx, c->bidx))) {
            free_ctx(c);
            return st;
        }
    }
    int32_t *d_part = nullptr, *d_bpos = nullptr;
    if ((st = upload(&d_part, c->part)) || (st = upload(&d_bpos, c->bpos))) {
        cudaFree(d_part);
        free_ctx(c);
        return st;
    }
    tick("upload A");
    std::vector<int32_t> er, ec;
    std::vector<double> ev;
    if ((st = device_basis(c, F, d_part))) { cudaFree(d_part); cudaFree(d_bpos); free_ctx(c); return st; }
    tick("basis (dd-MGS, GPU)");
    st = device_galerkin(c, row_ptr, col, d_part, d_bpos, er, ec, ev);
    cudaFree(d_part);
    cudaFree(d_bpos);
    if (st) { free_ctx(c); return st; }
    tick("galerkin (GPU)");
    // environment overrides for experiments (documented in DESIGN.md)
    if (const char* e = getenv("DDG_FUSE_GATHER")) c->opts.fuse_gather = atoi(e);
    if (const char* e = getenv("DDG_SMALL_KERNEL")) c->opts.small_kernel = atoi(e);
    if (const char* e = getenv("DDG_SYMV")) c->symv_mode = e[0] == 'c' ? 1 : 0;
    if (const char* e = getenv("DDG_RING_MIN_MB")) c->ring_min_bytes = atof(e) * 1e6;
    if (const char* e = getenv("DDG_FLAT_COARSE")) c->flat_coarse = atoi(e) != 0;
    c->coarse_variant = c->opts.coarse_variant;
    if (c->coarse_variant == 0) c->coarse_variant = c->nc <= 8192 ? 1 : 2;
    if (c->opts.part2) {   // three levels
        if (c->opts.nparts2 < 2) {
            int np2 = c->opts.nparts2;
            free_ctx(c);
            return set_err(DDG_E_PART, "too small for three levels: %d second-level part(s)", np2);
        }
        std::vector<char> seen(c->opts.nparts2, 0);
        for (int I = 0; I < nparts; ++I) {
            const int J = c->opts.part2[I];
            if (J < 0 || J >= c->opts.nparts2) {
                free_ctx(c);
                return set_err(DDG_E_PART, "second-level part %d of part %d outside [0,%d)", J, I,
                               c->opts.nparts2);
            }
            if (c->cptr[I + 1] > c->cptr[I]) seen[J] = 1;
        }
        for (int J = 0; J < c->opts.nparts2; ++J)
            if (!seen[J]) { free_ctx(c); return set_err(DDG_E_PART, "second-level part %d is empty", J); }
        c->coarse_variant = 3;
    }
    if (c->coarse_variant == 1 && c->nc > 131072) {
        int64_t nc = c->nc;
        free_ctx(c);
        return set_err(DDG_E_ARG, "n_c = %lld: the dense coarse inverse is limited to 131072 unknowns",
                       (long long)nc);
    }
    symv_ring_init();          // reads the SYMV switches (g_band) build_plans depends on
    build_plans(c);
    c->device_loop = getenv("DDG_DEVICE_LOOP") ? atoi(getenv("DDG_DEVICE_LOOP")) : 1;
    if (c->coarse_variant == 2) {
        if ((st = sparse_coarse_symbolic(c, row_ptr, col, er, ec, ev))) { free_ctx(c); return st; }
        tick("coarse symbolic (nested dissection)");
    }
    // uploads
    {
        const double mean = (double)c->nnz / (double)std::max<int64_t>(1, n);
        int sw = mean <= 16 ? 1 : mean <= 48 ? 4 : mean <= 128 ? 8 : 32;
        DevStencil ds;
        std::vector<double> scoef;
        if (getenv("DDG_NO_STENCIL")) c->opts.stencil = nullptr;
        if ((st = build_stencil(c, c->opts.stencil, n, row_ptr, col, val, ds, scoef))) { free_ctx(c); return st; }
        if (!scoef.empty()) {
            if ((st = upload(&c->d_stencil_coef, scoef))) { free_ctx(c); return st; }
            ds.coef = c->d_stencil_coef;
        }
        if (const char* e = getenv("DDG_ROW_SW")) sw = atoi(e);   // experiment: lanes per CSR row
        if (sw != 1 && sw != 4 && sw != 8 && sw != 32) sw = 8;
        if (ds.kind) sw = 1;
        c->A = DevCSR{n, c->nnz, c->d_rp, c->d_col, c->d_val, sw, 0, ds, nullptr, nullptr};
        if (!ds.kind && !getenv("DDG_NO_NODE_BLOCKS")) {
            // node-blocked columns (C4's 3 DoFs per node, a three-level child's k per part)
            for (int bs : {4, 3}) {
                std::vector<int32_t> brp, bcol;
                if (!node_blocks(n, row_ptr, col, bs, brp, bcol)) continue;
                if ((st = upload(&c->d_brp, brp)) || (st = upload(&c->d_bcol, bcol))) { free_ctx(c); return st; }
                c->A.bs = bs;
                c->A.brp = c->d_brp;
                c->A.bcol = c->d_bcol;
                break;
            }
        }
        c->opts.stencil = nullptr;   // borrowed for the duration of ddg_setup only
    }
    {   // s position -> fine row (padding -1), for the flat colour gather
        std::vector<int32_t> g(std::max<int64_t>(1, c->s_doubles), -1);
        for (size_t q = 0; q < c->op_sub.size(); ++q) {
            const OpDesc& op = c->ops[q];
            for (int a = 0; a < op.m; ++a) g[op.s_off + a] = c->oidx[op.idx_off + a];
        }
        if ((st = upload(&c->d_gidx, g))) { free_ctx(c); return st; }
    }
    if ((st = upload(&c->d_oidx, c->oidx)) || (st = upload(&c->d_ops, c->ops)) ||
        (st = upload(&c->d_items, c->items)) || (st = upload(&c->d_red, c->red)) ||
        (st = dalloc(&c->d_tiles, c->tiles_doubles)) || (st = dalloc(&c->d_s, c->s_doubles)) ||
        (st = dalloc(&c->d_partials, c->part_doubles)) ||
        (st = dalloc(&c->d_yc, c->nc)) || (st = dalloc(&c->d_r, n)) || (st = dalloc(&c->d_z, n)) ||
        (st = dalloc(&c->d_p, n)) || (st = dalloc(&c->d_q, n)) || (st = dalloc(&c->d_f, n)) ||
        (st = dalloc(&c->d_u, n)) || (st = dalloc(&c->d_x, n)) || (st = dalloc(&c->d_sc, 1)) ||
        (st = dalloc(&c->d_redbuf, RED_BLOCKS)) || (st = dalloc(&c->d_ticket, 1)) ||
        (st = dalloc(&c->d_zero, 1)) || (st = dalloc(&c->d_tickets, c->ops.size())) ||
        (st = upload(&c->d_ring, c->h_ring)) ||
        (c->coarse_variant == 3 && (st = dalloc(&c->d_bc, std::max<int64_t>(1, c->nc))))) {
        free_ctx(c);
        return st;
    }
    if (c->dist) c->flat_coarse = false;
    if (c->flat_coarse) {
        std::vector<int32_t> xp(n);
        for (int I = 0; I < nparts; ++I)
            for (int64_t x = c->bptr[I]; x < c->bptr[I + 1]; ++x) xp[x] = I;
        if ((st = dalloc(&c->d_res, n)) || (st = upload(&c->d_xpart, xp))) {
            free_ctx(c);
            return st;
        }
    }
    if (cudaMemsetAsync(c->d_s, 0, c->s_doubles * 8, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->d_ticket, 0, sizeof(unsigned), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->d_zero, 0, sizeof(int32_t), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->d_tickets, 0, c->ops.size() * sizeof(unsigned), c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->d_sc, 0, sizeof(Scalars), c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess ||
        cudaMallocHost(&c->h_sc, sizeof(Scalars)) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
        free_ctx(c);
        return set_err(DDG_E_CUDA, "device initialisation failed");
    }
    c->maxmI = 0;
    for (int I = 0; I < nparts; ++I) c->maxmI = std::max<int>(c->maxmI, (int)(c->bptr[I + 1] - c->bptr[I]));
    c->nrows = n;
    c->n_restrict = nparts;
    c->n_prolong = nparts;
    c->h_z.assign(c->ncolours, ddg::Halo{});
    if (c->dist && c->nranks > 1 && !c->comm->loop && !getenv("DDG_NO_HALO_OVERLAP")) {
        if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
            free_ctx(c);
            return set_err(DDG_E_CUDA, "side stream creation failed");
        }
    }
    if (c->dist && c->nranks > 1) {
        const ddg::DistPlan& P = c->plan;
        if ((st = upload(&c->d_rows, P.owned_rows)) || (st = upload(&c->d_restrict_parts, P.owned_subs)) ||
            (st = upload(&c->d_prolong_parts, P.prolong_parts))) {
            free_ctx(c);
            return st;
        }
        c->nrows = (int64_t)P.owned_rows.size();
        c->n_restrict = (int)P.owned_subs.size();
        c->n_prolong = (int)P.prolong_parts.size();
        auto mk = [&](ddg::Halo& h, const std::vector<std::vector<int32_t>>& snd,
                      const std::vector<std::vector<int32_t>>& rcv, size_t base) -> int {
            h.send_off.assign(c->nranks + 1, 0);
            h.recv_off.assign(c->nranks + 1, 0);
            std::vector<int32_t> si, ri;
            for (int p = 0; p < c->nranks; ++p) {
                const auto& a = snd[base + p];
                const auto& b = rcv[base + p];
                si.insert(si.end(), a.begin(), a.end());
                ri.insert(ri.end(), b.begin(), b.end());
                h.send_off[p + 1] = (int64_t)si.size();
                h.recv_off[p + 1] = (int64_t)ri.size();
            }
            h.send_total = (int64_t)si.size();
            h.recv_total = (int64_t)ri.size();
            int e;
            if ((e = upload(&h.d_sidx, si)) || (e = upload(&h.d_ridx, ri)) || (e = dalloc(&h.d_sbuf, si.size())) ||
                (e = dalloc(&h.d_rbuf, ri.size())))
                return e;
            return DDG_OK;
        };
        if ((st = mk(c->h_p, P.p_send, P.p_recv, 0)) || (st = mk(c->h_r, P.r_send, P.r_recv, 0))) {
            free_ctx(c);
            return st;
        }
        for (int cc = 0; cc < c->ncolours; ++cc)
            if ((st = mk(c->h_z[cc], P.z_send, P.z_recv, (size_t)cc * c->nranks))) {
                free_ctx(c);
                return st;
            }
        tick("halo plans");
    }
    // the whole solve in one cluster kernel (k_pcg_small): one GPU, dense single-item
    // coarse inverse with at most G tile rows, single-item local operators, n small,
    // and everything a CTA keeps resident within its shared memory (small_plan)
    // (DDG_SMALL_FUSED=0: off)
    if (!c->chol && !(getenv("DDG_SMALL_FUSED") && atoi(getenv("DDG_SMALL_FUSED")) == 0)) {
        if ((st = small_plan(c))) { free_ctx(c); return st; }
    }
    tick("upload");
    if ((st = invert_locals(c))) { free_ctx(c); return st; }
    tick("local inverses (GPU)");
    if (c->coarse_variant == 1) {
        if ((st = invert_coarse(c, er, ec, ev))) { free_ctx(c); return st; }
        tick("coarse inverse (GPU)");
    } else if (c->coarse_variant == 2) {
        if ((st = sparse_coarse_numeric(c))) { free_ctx(c); return st; }
        tick("coarse inverse (GPU)");
    } else {
        if ((st = build_child(c, F, er, ec, ev))) {
            std::string msg = g_last_error;
            free_ctx(c);
            return set_err(st, "second level: %s", msg.c_str());
        }
        tick("second level (two-level setup on A_c)");
    }
    c->local_bytes = 0;
    for (int q = 0; q < (int)c->op_sub.size(); ++q) {
        const OpDesc& op = c->ops[q];
        if (c->chol) {
            c->local_bytes += chol_doubles(op.nT) * 8;
            continue;
        }
        for (int t = 0; t < op.nitems; ++t) {
            const ItemDesc& d = c->items[op.item_base + t];
            c->local_bytes += item_doubles(d.tri, d.I1 - d.I0, d.ntiles, d.tail) * 8;
        }
    }
    c->coarse_bytes = c->coarse_variant == 1   ? (c->tiles_doubles * 8) - c->local_bytes
                      : c->coarse_variant == 2 ? sparse_coarse_bytes(c)
                                               : c->child->local_bytes + c->child->coarse_bytes;
    c->opts.part2 = nullptr;   // borrowed for the duration of ddg_setup only
    c->opts.block_coords2 = nullptr;
    c->t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c;
    return DDG_OK;
}

// ---------------------------------------------------------------------------
// preconditioner and PCG enqueue
// ---------------------------------------------------------------------------
// multi-GPU helpers (no-ops on a single GPU) --------------------------------
static void comm_check(ddg_ctx* c, int st) {
    if (st && !c->comm_err) c->comm_err = st;
}
// after a reduction kernel: allreduce the rank-local sum, then apply its logic
static void dist_finish(ddg_ctx* c, int slot) {
    if (!c->dist) return;
    comm_check(c, comm_allreduce_sum(c->comm, &c->d_sc->loc[slot], &c->d_sc->glob[slot], 1, c->stream));
    launch_pcg_finalize(c->stream, slot, c->d_sc, c->d_hist);
    c->launches += 1;
}
// send the values this rank wrote to the ranks that read them
static void halo_on(ddg_ctx* c, ddg::Halo& h, double* v, cudaStream_t st) {
    if (!c->dist || c->nranks == 1) return;
    launch_halo_pack(st, v, h.d_sidx, h.d_sbuf, h.send_total);
    comm_check(c, comm_exchange(c->comm, h, st));
    launch_halo_unpack(st, h.d_rbuf, h.d_ridx, v, h.recv_total);
    c->launches += (h.send_total > 0) + (h.recv_total > 0);
}
static void halo(ddg_ctx* c, ddg::Halo& h, double* v) { halo_on(c, h, v, c->stream); }
// boundary-first colour step: the z halo of the boundary
// subdomains goes out on the side stream while the interior ones compute
// (loopback ranks share one stream: in order there)
static void halo_fork(ddg_ctx* c, ddg::Halo& h, double* v) {
    if (!c->side) { halo(c, h, v); return; }
    cudaEventRecord(c->ev_fork, c->stream);
    cudaStreamWaitEvent(c->side, c->ev_fork, 0);
    halo_on(c, h, v, c->side);
    cudaEventRecord(c->ev_join, c->side);
}
static void halo_join(ddg_ctx* c) {
    if (c->side) cudaStreamWaitEvent(c->stream, c->ev_join, 0);
}

static void colour_step(ddg_ctx* c, int cc, const double* r, double* z, bool z_zero, const int32_t* done) {
    const ColourPlan& pl = c->plans[cc];
    if (c->chol) {   // DDG_LOCAL_CHOLESKY: gather s, then forward + back substitution per subdomain
        if (pl.sub_end > pl.sub_begin) {
            const OpDesc& lo = c->ops[pl.sub_begin];
            const OpDesc& hi = c->ops[pl.sub_end - 1];
            prof(c, PC_GATHER, 0, [&] {
                launch_gather_flat(c->stream, lo.s_off, hi.s_off + hi.mp, c->d_gidx, c->A, r, z, c->d_s, z_zero,
                                   done);
            });
            const int mp = (pl.max_rows + TILE - 1) / TILE * TILE;
            prof(c, PC_SYMV, c->colour_alg_bytes[cc], [&] {
                launch_chol_solve(c->stream, c->d_ops, pl.sub_begin, pl.sub_mid - pl.sub_begin, mp, c->d_tiles,
                                  c->d_s, c->d_oidx, z, done);
                if (pl.sub_mid < pl.sub_end) {
                    halo_fork(c, c->h_z[cc], z);
                    launch_chol_solve(c->stream, c->d_ops, pl.sub_mid, pl.sub_end - pl.sub_mid, mp, c->d_tiles,
                                      c->d_s, c->d_oidx, z, done);
                    halo_join(c);
                }
            });
            c->launches += 2 + (pl.sub_mid < pl.sub_end);
            if (pl.sub_mid < pl.sub_end) return;
        }
        halo(c, c->h_z[cc], z);
        return;
    }
    if (pl.sub_mid < pl.sub_end) {   // several ranks: boundary subdomains, halo out, interior ones
        const OpDesc& lo = c->ops[pl.sub_begin];
        const OpDesc& hi = c->ops[pl.sub_end - 1];
        prof(c, PC_GATHER, 0, [&] {
            launch_gather_flat(c->stream, lo.s_off, hi.s_off + hi.mp, c->d_gidx, c->A, r, z, c->d_s, z_zero, done);
        });
        c->launches += 1;
        auto run = [&](int ib, int ie, int rb, int re, int roff) {
            if (ie <= ib) return;
            if (ring_ok(c, roff)) {
                int mr, mc;
                ring_dims(c, roff, &mr, &mc);
                launch_symv_ring(c->stream, c->d_ops, c->d_items, ib, c->d_ring + roff, num_sms(), mr, mc,
                                 c->d_tiles, c->d_s, c->d_oidx, z, nullptr, c->d_partials, done, pl.all_single != 0);
                if (re > rb)
                    launch_symv_reduce(c->stream, c->d_ops, c->d_items, c->d_red, rb, re - rb, c->d_oidx,
                                       c->d_partials, z, nullptr, done);
                c->launches += 1 + (re > rb);
            } else {
                launch_symv(c->stream, c->d_ops, c->d_items, ib, ie - ib, c->d_tiles, c->d_s, c->d_oidx, z, nullptr,
                            c->d_partials, done, pl.max_rows_t, c->d_tickets);
                c->launches += 1;
            }
        };
        prof(c, PC_SYMV, c->colour_alg_bytes[cc], [&] {
            run(pl.item_begin, pl.item_mid, pl.red_begin, pl.red_mid, pl.ring_b);
            halo_fork(c, c->h_z[cc], z);
            run(pl.item_mid, pl.item_end, pl.red_mid, pl.red_end, pl.ring_i);
            halo_join(c);
        });
        return;
    }
    int gmode = 0;
    const bool ring = ring_ok(c, pl.ring_off);
    const bool fuse = !ring && pl.all_single && (c->opts.fuse_gather == 2 ||
                                        (c->opts.fuse_gather == 1 &&
                                         (pl.max_ntiles >= 32 || pl.sub_end - pl.sub_begin <= 2 * num_sms())));
    if (pl.sub_end > pl.sub_begin) {
        if (fuse) {
            gmode = z_zero ? 2 : 1;
        } else {
            prof(c, PC_GATHER, 0, [&] {
                const OpDesc& lo = c->ops[pl.sub_begin];
                const OpDesc& hi = c->ops[pl.sub_end - 1];
                launch_gather_flat(c->stream, lo.s_off, hi.s_off + hi.mp, c->d_gidx, c->A, r, z, c->d_s, z_zero,
                                   done);
            });
            c->launches += 1;
        }
        if (ring) {
            prof(c, PC_SYMV, c->colour_alg_bytes[cc], [&] {
                int mr, mc;
                ring_dims(c, pl.ring_off, &mr, &mc);
                launch_symv_ring(c->stream, c->d_ops, c->d_items, pl.item_begin, c->d_ring + pl.ring_off,
                                 num_sms(), mr, mc, c->d_tiles, c->d_s, c->d_oidx, z, nullptr, c->d_partials, done,
                                 pl.all_single != 0);
            });
            c->launches += 1;
            if (pl.red_end > pl.red_begin) {
                prof(c, PC_REDUCE, 0, [&] {
                    launch_symv_reduce(c->stream, c->d_ops, c->d_items, c->d_red, pl.red_begin,
                                       pl.red_end - pl.red_begin, c->d_oidx, c->d_partials, z, nullptr, done);
                });
                c->launches += 1;
            }
            halo(c, c->h_z[cc], z);
            return;
        }
        prof(c, PC_SYMV, c->colour_alg_bytes[cc], [&] {
            launch_symv(c->stream, c->d_ops, c->d_items, pl.item_begin, pl.item_end - pl.item_begin,
                        c->d_tiles, c->d_s, c->d_oidx, z, nullptr, c->d_partials, done, pl.max_rows_t,
                        c->d_tickets, gmode, c->A, r,
                        pl.all_single && c->opts.small_kernel != 0 && !fuse &&
                            pl.sub_end - pl.sub_begin >= 16 * num_sms());
        });
        c->launches += 1;
    }
    halo(c, c->h_z[cc], z);
}

static void enqueue_precond(ddg_ctx* c, const double* r, double* z, const int32_t* done);

static void coarse_add(ddg_ctx* c, const double* r, double* z, const int32_t* done) {
    double* bc = c->coarse_variant == 2 ? sparse_coarse_rhs(c)
                 : c->coarse_variant == 3 ? c->d_bc
                                          : c->d_s + c->ops[c->coarse_op].s_off;
    const bool multi = c->dist && c->nranks > 1;
    prof(c, PC_COARSE, 0, [&] {
        if (multi) cudaMemsetAsync(bc, 0, c->nc * sizeof(double), c->stream);
        if (c->flat_coarse) {   // residual in part order at streaming speed, then Q_I^T res per part
            launch_gather_flat(c->stream, 0, c->n, c->d_bidx, c->A, r, z, c->d_res, false, done);
            launch_restrict_dot(c->stream, c->nparts, c->d_bptr, c->d_cptr, c->d_qoff, c->d_Q, c->d_res, bc,
                                c->maxmI, done);
            c->launches += 1;
        } else {
            launch_coarse_restrict(c->stream, c->n_restrict, c->d_bptr, c->d_bidx, c->d_cptr, c->d_qoff, c->d_Q,
                                   c->A, r, z, bc, c->maxmI, done, c->d_restrict_parts);
        }
        if (multi) comm_check(c, comm_allreduce_sum(c->comm, bc, bc, c->nc, c->stream));
        if (c->coarse_variant == 3) {
            // three levels: y_c = M_2 b_c, one V-cycle of the two-level method on A_c
            const int64_t l0 = c->child->launches;
            ddg_ctx* ch = c->child;
            enqueue_precond(ch, bc, c->d_yc, done);
            if (c->dist) {
                // each rank holds y_c on the second level's rows it owns (and halos):
                // assemble it everywhere for this rank's prolongation
                launch_fill(c->stream, ch->d_q, ch->n, 0.0, done);
                launch_copy_rows(c->stream, c->d_yc, ch->d_q, ch->d_rows, ch->nrows);
                comm_check(c, comm_allreduce_sum(c->comm, ch->d_q, c->d_yc, ch->n, c->stream));
                c->comm_err |= ch->comm_err;
                ch->launches += 2;
            }
            c->launches += ch->launches - l0;
        } else if (c->coarse_variant == 2) {
            c->launches += sparse_coarse_enqueue_solve(c, c->d_yc, done);
        } else if (ring_ok(c, c->coarse_ring_off)) {
            int mr, mc;
            ring_dims(c, c->coarse_ring_off, &mr, &mc);
            launch_symv_ring(c->stream, c->d_ops, c->d_items, c->coarse_item_begin, c->d_ring + c->coarse_ring_off,
                             num_sms(), mr, mc, c->d_tiles, c->d_s, c->d_oidx, nullptr, c->d_yc, c->d_partials, done);
            c->launches += 1;
            if (c->coarse_red_end > c->coarse_red_begin) {
                launch_symv_reduce(c->stream, c->d_ops, c->d_items, c->d_red, c->coarse_red_begin,
                                   c->coarse_red_end - c->coarse_red_begin, c->d_oidx, c->d_partials, nullptr,
                                   c->d_yc, done);
                c->launches += 1;
            }
        } else {
            launch_symv(c->stream, c->d_ops, c->d_items, c->coarse_item_begin,
                        c->coarse_item_end - c->coarse_item_begin, c->d_tiles, c->d_s, c->d_oidx, nullptr,
                        c->d_yc, c->d_partials, done, c->coarse_rows_t, c->d_tickets);
            c->launches += 1;
        }
        if (c->flat_coarse)
            launch_prolong_flat(c->stream, c->n, c->d_xpart, c->d_bptr, c->d_bidx, c->d_cptr, c->d_qoff, c->d_Q,
                                c->d_yc, z, done);
        else
            launch_prolong(c->stream, c->n_prolong, c->d_bptr, c->d_bidx, c->d_cptr, c->d_qoff, c->d_Q, c->d_yc, z,
                           c->maxmI, done, c->d_prolong_parts);
    });
    c->launches += 2;
}

// z = M r: zero guess, forward sweep, coarse, reverse sweep
static void enqueue_precond(ddg_ctx* c, const double* r, double* z, const int32_t* done) {
    prof(c, PC_VEC, 0, [&] { launch_fill(c->stream, z, c->n, 0.0, done); });
    c->launches += 1;
    for (int cc = 0; cc < c->ncolours; ++cc) colour_step(c, cc, r, z, cc == 0, done);
    coarse_add(c, r, z, done);
    for (int cc = c->ncolours - 1; cc >= 0; --cc) colour_step(c, cc, r, z, false, done);
}

// a1 + a2: q = A p, sigma, alpha; u, r update, ||r||, stop test; r halo
static void enqueue_step_a(ddg_ctx* c, double* u) {
    Scalars* sc = c->d_sc;
    const int dist = c->dist ? 1 : 0;
    prof(c, PC_VEC, 0, [&] {
        launch_pcg_spmv_dot(c->stream, c->A, c->d_p, c->d_q, c->d_rows, c->nrows, sc, c->d_redbuf, c->d_ticket,
                            dist);
        dist_finish(c, 2);
        launch_pcg_update(c->stream, c->d_p, c->d_q, u, c->d_r, c->d_rows, c->nrows, sc, c->d_hist, c->d_redbuf,
                          c->d_ticket, dist);
        dist_finish(c, 3);
        halo(c, c->h_r, c->d_r);
    });
    c->launches += 2;
}
// a9: rho' = r^T z, beta; p = z + beta p; p halo
static void enqueue_step_b(ddg_ctx* c) {
    Scalars* sc = c->d_sc;
    const int dist = c->dist ? 1 : 0;
    prof(c, PC_VEC, 0, [&] {
        launch_pcg_rz(c->stream, c->d_r, c->d_z, c->d_rows, c->nrows, sc, c->d_redbuf, c->d_ticket, dist);
        dist_finish(c, 4);
        launch_pcg_direction(c->stream, c->d_z, c->d_p, c->d_rows, c->nrows, sc);
        halo(c, c->h_p, c->d_p);
    });
    c->launches += 2;
}

static void enqueue_iteration(ddg_ctx* c, double* u) {
    enqueue_step_a(c, u);
    enqueue_precond(c, c->d_r, c->d_z, &c->d_sc->done);
    enqueue_step_b(c);
}

// Lanczos condition estimate from the CG coefficients:
// tridiagonal T with T_kk = 1/a_k + b_{k-1}/a_{k-1}, T_{k,k+1} = sqrt(b_k)/a_k;
// its extreme eigenvalues by Sturm-count bisection; kappa = max/min and the
// classical CG bound ln(2/tol) / ln((sqrt(kappa)+1)/(sqrt(kappa)-1)).
static void lanczos_condition(const std::vector<double>& a, const std::vector<double>& b, double tol,
                              double* kappa, double* bound) {
    *kappa = 1.0;
    *bound = 1.0;
    const int k = (int)a.size();
    if (k < 2) return;
    std::vector<double> d(k), e(k, 0.0);
    for (int j = 0; j < k; ++j) {
        d[j] = 1.0 / a[j] + (j > 0 ? b[j - 1] / a[j - 1] : 0.0);
        if (j + 1 < k) e[j] = sqrt(b[j]) / a[j];
    }
    double lo = INFINITY, hi = -INFINITY;                     // Gershgorin interval
    for (int j = 0; j < k; ++j) {
        const double r = (j > 0 ? fabs(e[j - 1]) : 0.0) + fabs(e[j]);
        lo = std::min(lo, d[j] - r);
        hi = std::max(hi, d[j] + r);
    }
    auto below = [&](double x) {                              // eigenvalues < x (Sturm sequence)
        int cnt = 0;
        double q = 1.0;
        for (int j = 0; j < k; ++j) {
            q = d[j] - x - (j > 0 ? e[j - 1] * e[j - 1] / q : 0.0);
            if (q == 0.0) q = -1e-300;
            if (q < 0.0) ++cnt;
        }
        return cnt;
    };
    auto kth = [&](int want) {                                // smallest x with below(x) >= want
        double l = lo, h = hi;
        for (int it = 0; it < 200; ++it) {
            const double m = 0.5 * (l + h);
            if (below(m) >= want) h = m; else l = m;
        }
        return 0.5 * (l + h);
    };
    const double lmin = kth(1), lmax = kth(k);
    if (!(lmin > 0.0)) return;
    *kappa = lmax / lmin;
    const double sk = sqrt(*kappa);
    if (*kappa > 1.0) *bound = log(2.0 / tol) / log((sk + 1.0) / (sk - 1.0));
}

// The whole iteration loop as one graph with device-side control (CUDA
// conditional nodes): no iteration is launched after convergence and the host
// waits once per solve.
//   top:  k_pcg_cond(while) -> WHILE { body }
//   body: a1 spmv+dot, a2 update + a3 test, k_pcg_cond(if) -> IF { a4..a8
//         preconditioner, a9 r^T z + direction } -> k_pcg_cond(while)
// Returns false (and leaves no graph) where the driver cannot build it; the
// caller then steps the loop from the host.
static bool build_solve_graph(ddg_ctx* c, double* d_u) {
    if (c->ge_solve) cudaGraphExecDestroy(c->ge_solve);
    if (c->g_solve) cudaGraphDestroy(c->g_solve);
    c->ge_solve = nullptr;
    c->g_solve = nullptr;
    cudaGraph_t g = nullptr;
    auto fail = [&]() {
        cudaStreamCaptureStatus cs;
        if (cudaStreamIsCapturing(c->stream, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(c->stream, &junk);
            if (junk && junk != g) cudaGraphDestroy(junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return false;
    };
    if (cudaGraphCreate(&g, 0) != cudaSuccess) return fail();
    cudaGraphConditionalHandle hw;
    if (cudaGraphConditionalHandleCreate(&hw, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
    // top: the WHILE condition from the state after the prologue
    if (cudaStreamBeginCaptureToGraph(c->stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return fail();
    launch_pcg_cond(c->stream, c->d_sc, (unsigned long long)hw);
    cudaGraph_t tmp = nullptr;
    if (cudaStreamEndCapture(c->stream, &tmp) != cudaSuccess) return fail();
    cudaGraphNode_t pre;
    size_t nn = 1;
    if (cudaGraphGetNodes(g, &pre, &nn) != cudaSuccess || nn != 1) return fail();
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wn;
    if (cudaGraphAddNode(&wn, g, &pre, 1, &wp) != cudaSuccess) return fail();
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    cudaGraphConditionalHandle hi;
    if (cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
    // body: a1-a3, then the IF condition
    const int64_t l0 = c->launches;
    if (cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return fail();
    enqueue_step_a(c, d_u);
    launch_pcg_cond(c->stream, c->d_sc, (unsigned long long)hi);
    c->launches_a = c->launches - l0 + 1;
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    if (cudaStreamGetCaptureInfo(c->stream, &cs, nullptr, nullptr, &deps, &nd) != cudaSuccess) return fail();
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t in;
    if (cudaGraphAddNode(&in, body, deps, nd, &ip) != cudaSuccess) return fail();
    if (cudaStreamUpdateCaptureDependencies(c->stream, &in, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
        return fail();
    launch_pcg_cond(c->stream, c->d_sc, (unsigned long long)hw);
    if (cudaStreamEndCapture(c->stream, &tmp) != cudaSuccess) return fail();
    // IF body: a4-a8 (preconditioner) and a9
    cudaGraph_t ib = ip.conditional.phGraph_out[0];
    const int64_t l1 = c->launches;
    if (cudaStreamBeginCaptureToGraph(c->stream, ib, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return fail();
    enqueue_precond(c, c->d_r, c->d_z, &c->d_sc->done);
    enqueue_step_b(c);
    if (cudaStreamEndCapture(c->stream, &tmp) != cudaSuccess) return fail();
    c->launches_b = c->launches - l1 + 1;          // + the WHILE condition kernel
    c->launches = l0;
    if (cudaGraphInstantiate(&c->ge_solve, g, 0) != cudaSuccess) return fail();
    c->g_solve = g;
    c->g_solve_u = d_u;
    return true;
}

// SURVEY.md §8(d) byte model of one PCG iteration on this rank
static double bytes_per_iter_model(ddg_ctx* c) {
    const double a = (c->A.st.kind == 1 || c->A.st.kind == 3) ? 0.0
                     : c->A.st.kind == 2 ? 32.0 : 12.0 * (double)c->nnz / (double)c->n + 4.0;
    double local = 0.0, msum = 0.0;
    for (size_t q = 0; q < c->op_sub.size(); ++q) {      // the subdomain operators come first
        const double m = c->ops[q].m;
        local += 2.0 * 8.0 * m * (m + 1) / 2;
        msum += m;
    }
    ddg_info inf;
    ddg_get_info(c, &inf);
    return local + (double)inf.coarse_solve_bytes + (64.0 + 2 * a) * msum + (144.0 + 2 * a + 16.0 * c->k) * (double)c->nrows;
}

static int run_pcg(ddg_ctx* c, const double* d_f, double* d_u, double rtol, int max_iter,
                   int* iters, double* res_hist, int cap, ddg_report* rep) {
    if (!(rtol > 0)) return set_err(DDG_E_ARG, "rtol must be > 0");
    if (max_iter <= 0) max_iter = c->opts.max_iter;
    if (max_iter + 1 > c->hist_cap) {
        if (c->d_hist) cudaFree(c->d_hist);
        if (c->d_ab) cudaFree(c->d_ab);
        c->d_hist = nullptr;
        c->d_ab = nullptr;
        int st = dalloc(&c->d_hist, max_iter + 1);
        if (!st) st = dalloc(&c->d_ab, 2 * (size_t)(max_iter + 1));
        if (st) return st;
        c->hist_cap = max_iter + 1;
        if (c->ge_iter) { cudaGraphExecDestroy(c->ge_iter); c->ge_iter = nullptr; }   // d_hist is baked in
        if (c->g_iter) { cudaGraphDestroy(c->g_iter); c->g_iter = nullptr; }
        if (c->ge_solve) { cudaGraphExecDestroy(c->ge_solve); c->ge_solve = nullptr; }
        if (c->g_solve) { cudaGraphDestroy(c->g_solve); c->g_solve = nullptr; }
    }
    c->comm_err = 0;
    c->loop_graph_used = 0;
    const int dist = c->dist ? 1 : 0;
    Scalars init{};
    init.rtol = rtol;
    init.max_iter = max_iter;
    init.stop_mode = c->opts.stop_mode;
    init.ab = c->d_ab;
    *c->h_sc = init;
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_sc, c->h_sc, sizeof(Scalars), cudaMemcpyHostToDevice, c->stream));
    int done_iters = 0;
    bool use_graph = c->opts.use_graphs != 0 && !c->profiling;
    if (c->small_ok && !c->profiling) {
        SmallArgs a = c->small;
        a.dbg = getenv("DDG_SMALL_TRACE") ? atoi(getenv("DDG_SMALL_TRACE")) >= 2 : 0;
        a.A = c->A;
        a.n = c->n;
        a.f = d_f;
        a.u = d_u;
        a.r = c->d_r;
        a.z = c->d_z;
        a.p = c->d_p;
        a.q = c->d_q;
        a.sc = c->d_sc;
        a.hist = c->d_hist;
        a.part = c->d_redbuf;
        a.ops = c->d_ops;
        a.items = c->d_items;
        a.tiles = c->d_tiles;
        a.oidx = c->d_oidx;
        a.cops = c->d_cops;
        a.ncolours = c->ncolours;
        a.nparts = c->nparts;
        a.bptr = c->d_bptr;
        a.bidx = c->d_bidx;
        a.cptr = c->d_cptr;
        a.qoff = c->d_qoff;
        a.Q = c->d_Q;
        a.coarse_item = c->coarse_item_begin;
        a.bc = c->d_s + c->ops[c->coarse_op].s_off;
        if (!launch_pcg_small(c->stream, a)) {
            if (c->opts.verbose) fprintf(stderr, "[ddg] k_pcg_small launch failed: multi-kernel iteration\n");
        } else {
            c->launches += 1;
            done_iters = max_iter;
            use_graph = false;
            goto solved;
        }
    }
    launch_pcg_init(c->stream, c->n, d_f, c->d_r, d_u, c->d_rows, c->nrows, c->d_sc, c->d_hist, c->d_redbuf,
                    c->d_ticket, dist);
    dist_finish(c, 0);
    enqueue_precond(c, c->d_r, c->d_z, &c->d_sc->done);
    launch_pcg_rz_first(c->stream, c->d_r, c->d_z, c->d_p, c->d_rows, c->nrows, c->d_sc, c->d_redbuf,
                        c->d_ticket, dist);
    dist_finish(c, 1);
    halo(c, c->h_p, c->d_p);
    c->launches += 2;
    CUDA_TRY(cudaGetLastError());
    // iteration graph (captured once per u pointer)
    if (use_graph && (!c->ge_iter || c->g_iter_u != d_u)) {
        if (c->ge_iter) cudaGraphExecDestroy(c->ge_iter);
        if (c->g_iter) cudaGraphDestroy(c->g_iter);
        c->ge_iter = nullptr;
        c->g_iter = nullptr;
        int64_t l0 = c->launches;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        enqueue_iteration(c, d_u);
        cudaError_t e = cudaStreamEndCapture(c->stream, &c->g_iter);
        if (e != cudaSuccess) return set_err(DDG_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
        CUDA_TRY(cudaGraphInstantiate(&c->ge_iter, c->g_iter, 0));
        c->launches_per_iter = c->launches - l0;
        c->launches = l0;
        c->g_iter_u = d_u;
    }
    {
    int chunk = 2;
    // device-side loop: one graph launch per solve (single context; the
    // host-stepped chunks below remain for multi-rank contexts and profiling)
    if (use_graph && !c->dist && c->device_loop && !c->profiling) {
        if (!c->ge_solve || c->g_solve_u != d_u) {
            if (!build_solve_graph(c, d_u)) c->device_loop = 0;
        }
        if (c->ge_solve) {
            CUDA_TRY(cudaGraphLaunch(c->ge_solve, c->stream));
            c->launches += 1;                          // the WHILE condition before the loop
            done_iters = max_iter;
            c->loop_graph_used = 1;
        }
    }
    if (c->profiling) {
        // profiled solve: step on the host so that no kernel is enqueued after
        // convergence (every timed launch does real work)
        for (int t = 0; t < max_iter; ++t) {
            { int _s = d2h(c->stream, c->h_sc, c->d_sc, sizeof(Scalars)); if (_s) return _s; }
            if (c->h_sc->done) break;
            enqueue_step_a(c, d_u);
            { int _s = d2h(c->stream, c->h_sc, c->d_sc, sizeof(Scalars)); if (_s) return _s; }
            if (c->h_sc->done) break;
            enqueue_precond(c, c->d_r, c->d_z, &c->d_sc->done);
            enqueue_step_b(c);
        }
        done_iters = max_iter;
    }
    while (done_iters < max_iter) {
        const int todo = std::min(chunk, max_iter - done_iters);
        for (int t = 0; t < todo; ++t) {
            if (use_graph) {
                CUDA_TRY(cudaGraphLaunch(c->ge_iter, c->stream));
                c->launches += c->launches_per_iter;
            } else {
                enqueue_iteration(c, d_u);
            }
        }
        done_iters += todo;
        CUDA_TRY(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (c->h_sc->done) break;
        chunk = std::min(chunk * 2, 8);
    }
    }
solved:
    if (c->dist && c->nranks > 1) {
        // assemble u on every rank: u is zero outside the owned rows
        comm_check(c, comm_allreduce_sum(c->comm, d_u, d_u, c->n, c->stream));
    }
    // true residual ||f - A u|| once (u is complete on every rank here)
    launch_true_res(c->stream, c->A, d_f, d_u, c->n, c->d_sc, c->d_redbuf, c->d_ticket);
    c->launches += 1;
    CUDA_TRY(cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    CUDA_TRY(cudaGetLastError());   // a launch that failed (bad configuration) must not pass silently
    if (c->comm_err) return set_err(DDG_E_NCCL, "NCCL failure inside the solve");
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    const Scalars s = *c->h_sc;
    const int it = s.iter;
    if (c->loop_graph_used) {     // kernels the device loop ran: every body, the IF bodies taken
        const int nif = (c->opts.stop_mode != 2 && s.status == 0) ? std::max(0, it - 1) : it;
        c->launches += (int64_t)it * c->launches_a + (int64_t)nif * c->launches_b;
        c->loop_graph_used = 0;
    }
    if (iters) *iters = it;
    if (res_hist && cap > 0) {
        int cnt = std::min(cap, it + 1);
        { int _s = d2h(c->stream, res_hist, c->d_hist, cnt * sizeof(double)); if (_s) return _s; }
    }
    if (rep) {
        rep->converged = s.converged;
        rep->iters = it;
        rep->res0 = s.res0;
        rep->res_final = s.res;
        rep->true_res = s.tres;
        rep->t_setup = c->t_setup;
        rep->t_solve = ms * 1e-3;
        rep->frac_iters = (double)it;
        rep->bytes_per_iter_model = bytes_per_iter_model(c);
        rep->cond_est = 1.0;
        rep->iter_bound = 1.0;
        c->last_alpha.clear();
        c->last_beta.clear();
        if (it >= 1) {
            std::vector<double> ab(2 * (size_t)it);
            if (d2h(c->stream, ab.data(), c->d_ab, ab.size() * sizeof(double)) == DDG_OK) {
                for (int k = 0; k < it; ++k) c->last_alpha.push_back(ab[2 * k]);
                for (int k = 0; k + 1 < it; ++k) c->last_beta.push_back(ab[2 * k + 1]);
                lanczos_condition(c->last_alpha, c->last_beta, rtol, &rep->cond_est, &rep->iter_bound);
            }
        }
        if (it >= 1 && s.converged && s.res > 0) {
            std::vector<double> h(it + 1);
            if (d2h(c->stream, h.data(), c->d_hist, (it + 1) * sizeof(double)) == DDG_OK) {
                double tol = s.rtol * s.ref;
                double a = log10(h[it - 1]), b = log10(h[it]), lt = log10(tol);
                // SPEC.md:373-377 interpolates the residual history; under stop_mode 2
                // the rule tests sqrt(r^T z), so the interpolant is kept inside
                // [it - 1, it] (frac <= iters <= frac + 1 in every mode)
                if (a != b) rep->frac_iters = std::min((double)it, std::max((double)(it - 1), (it - 1) + (a - lt) / (a - b)));
            }
        }
    }
    if (s.status) return set_err(s.status, "PCG breakdown (p^T A p <= 0 or r^T z <= 0) at iteration %d", it);
    return DDG_OK;
}

extern "C" int ddg_pcg_solve_device(ddg_ctx* c, const double* d_f, double rtol, int max_iter, double* d_u,
                                    int* iters, double* res_hist, int res_hist_cap, ddg_report* rep) {
    if (!c || !d_f || !d_u) return set_err(DDG_E_ARG, "null argument");
    if (cudaSetDevice(c->device) != cudaSuccess) return set_err(DDG_E_CUDA, "cudaSetDevice failed");
    return run_pcg(c, d_f, d_u, rtol, max_iter, iters, res_hist, res_hist_cap, rep);
}

extern "C" int ddg_pcg_solve(ddg_ctx* c, const double* f, double rtol, int max_iter, double* u,
                             int* iters, double* res_hist, int res_hist_cap, ddg_report* rep) {
    if (!c || !f || !u) return set_err(DDG_E_ARG, "null argument");
    if (cudaSetDevice(c->device) != cudaSuccess) return set_err(DDG_E_CUDA, "cudaSetDevice failed");
    CUDA_TRY(cudaMemcpyAsync(c->d_f, f, c->n * 8, cudaMemcpyHostToDevice, c->stream));
    int st = run_pcg(c, c->d_f, c->d_u, rtol, max_iter, iters, res_hist, res_hist_cap, rep);
    if (st) return st;
    CUDA_TRY(cudaMemcpyAsync(u, c->d_u, c->n * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return DDG_OK;
}

static int host_vec_op(ddg_ctx* c, const double* in, double* out, int which) {
    if (!c || !in || !out) return set_err(DDG_E_ARG, "null argument");
    if (cudaSetDevice(c->device) != cudaSuccess) return set_err(DDG_E_CUDA, "cudaSetDevice failed");
    c->comm_err = 0;
    CUDA_TRY(cudaMemcpyAsync(c->d_x, in, c->n * 8, cudaMemcpyHostToDevice, c->stream));
    if (which == 0) {
        enqueue_precond(c, c->d_x, c->d_z, c->d_zero);
    } else if (which == 1) {
        launch_fill(c->stream, c->d_z, c->n, 0.0, nullptr);
        coarse_add(c, c->d_x, c->d_z, c->d_zero);
    } else {
        launch_spmv(c->stream, c->A, c->d_x, c->d_z);
        c->launches += 1;
    }
    double* res = c->d_z;
    if (c->dist && c->nranks > 1) {   // assemble: each rank contributes its owned rows
        launch_fill(c->stream, c->d_q, c->n, 0.0, nullptr);
        launch_copy_rows(c->stream, c->d_z, c->d_q, c->d_rows, c->nrows);
        comm_check(c, comm_allreduce_sum(c->comm, c->d_q, c->d_q, c->n, c->stream));
        res = c->d_q;
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, res, c->n * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->comm_err) return set_err(DDG_E_NCCL, "NCCL failure");
    return DDG_OK;
}

extern "C" int ddg_apply_precond(ddg_ctx* c, const double* r, double* z) { return host_vec_op(c, r, z, 0); }
extern "C" int ddg_coarse_correct(ddg_ctx* c, const double* r, double* z) { return host_vec_op(c, r, z, 1); }
extern "C" int ddg_spmv(ddg_ctx* c, const double* x, double* y) { return host_vec_op(c, x, y, 2); }

extern "C" int ddg_get_info(ddg_ctx* c, ddg_info* info) {
    if (!c || !info) return set_err(DDG_E_ARG, "null argument");
    memset(info, 0, sizeof *info);
    info->n = c->n;
    info->n_c = c->nc;
    info->nparts = c->nparts;
    info->ncolours = c->ncolours;
    int mmin = INT32_MAX, mmax = 0;
    for (int i = 0; i < c->nparts; ++i) {
        const int m = (int)(c->optr[i + 1] - c->optr[i]);
        mmin = std::min(mmin, m);
        mmax = std::max(mmax, m);
    }
    info->m_min = mmin;
    info->m_max = mmax;
    info->k = c->k;
    info->dropped = c->dropped;
    info->min_rank_ratio = c->min_ratio;
    info->local_factor_bytes = c->local_bytes;
    info->coarse_factor_bytes = c->coarse_bytes;
    info->coarse_variant = c->coarse_variant;
    info->levels = c->child ? 3 : 2;
    if (c->child) {
        ddg_info ci;
        ddg_get_info(c->child, &ci);
        info->n_c2 = ci.n_c;
        info->nparts2 = ci.nparts;
        info->ncolours2 = ci.ncolours;
        info->coarse_variant2 = ci.coarse_variant;
        info->coarse_solve_bytes = 2 * ci.local_factor_bytes + ci.coarse_solve_bytes;
    } else {
        info->coarse_solve_bytes = c->coarse_variant == 1 ? c->coarse_bytes : sparse_coarse_solve_bytes(c);
    }
    return DDG_OK;
}

extern "C" int ddg_get_colours(ddg_ctx* c, int32_t* colour) {
    if (!c || !colour) return set_err(DDG_E_ARG, "null argument");
    std::copy(c->colour.begin(), c->colour.end(), colour);
    return DDG_OK;
}

extern "C" int ddg_get_subdomain_sizes(ddg_ctx* c, int32_t* m) {
    if (!c || !m) return set_err(DDG_E_ARG, "null argument");
    for (int i = 0; i < c->nparts; ++i) m[i] = (int32_t)(c->optr[i + 1] - c->optr[i]);
    return DDG_OK;
}

extern "C" int64_t ddg_launch_count(ddg_ctx* c, int reset) {
    if (!c) return -1;
    int64_t v = c->launches;
    if (reset) c->launches = 0;
    return v;
}

extern "C" int ddg_set_profiling(ddg_ctx* c, int on) {
    if (!c) return set_err(DDG_E_ARG, "null argument");
    c->profiling = on != 0;
    c->recs.clear();
    return DDG_OK;
}

extern "C" int ddg_get_kernel_stats(ddg_ctx* c, ddg_kstats* st) {
    if (!c || !st) return set_err(DDG_E_ARG, "null argument");
    memset(st, 0, sizeof *st);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (auto& r : c->recs) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->evpool[r.e0], c->evpool[r.e1]));
        switch (r.cat) {
            case PC_SYMV: st->symv_launches++; st->symv_ms += ms; st->symv_alg_bytes += r.bytes; break;
            case PC_GATHER: st->gather_ms += ms; break;
            case PC_REDUCE: st->reduce_ms += ms; break;
            case PC_COARSE: st->coarse_ms += ms; break;
            default: st->vec_ms += ms; break;
        }
        st->launches++;
    }
    c->recs.clear();
    return DDG_OK;
}

// ---------------------------------------------------------------------------
// host-only decomposition plan (tests / tools)
// ---------------------------------------------------------------------------
#include "dist.h"

struct ddg_plan {
    ddg::DistPlan P;
    std::vector<int32_t> colour;
    std::vector<int64_t> optr;
    std::vector<int32_t> oidx;
};

extern "C" int ddg_plan_create(int64_t n, const int64_t* row_ptr, const int32_t* col, const int32_t* part,
                               int32_t nparts, int overlap, const int32_t* block_coords, int block_ndim,
                               int rank, int nranks, ddg_plan** out) {
    if (!out || n < 1 || !row_ptr || !col || !part || nparts < 1 || nranks < 1 || rank < 0 || rank >= nranks ||
        overlap < 0)
        return set_err(DDG_E_ARG, "ddg_plan_create: bad argument");
    *out = nullptr;
    ddg_ctx c;
    ddg_default_opts(&c.opts);
    c.opts.overlap = overlap;
    c.n = n;
    c.nparts = nparts;
    c.part.assign(part, part + n);
    c.bptr.assign(nparts + 1, 0);
    for (int64_t v = 0; v < n; ++v) {
        if (part[v] < 0 || part[v] >= nparts) return set_err(DDG_E_PART, "part id out of range");
        c.bptr[part[v] + 1]++;
    }
    for (int I = 0; I < nparts; ++I) c.bptr[I + 1] += c.bptr[I];
    c.bidx.resize(n);
    c.bpos.resize(n);
    {
        std::vector<int64_t> fill(c.bptr.begin(), c.bptr.end() - 1);
        for (int64_t v = 0; v < n; ++v) {
            c.bpos[v] = (int32_t)(fill[part[v]] - c.bptr[part[v]]);
            c.bidx[fill[part[v]]++] = (int32_t)v;
        }
    }
    build_overlap(&c, row_ptr, col);
    build_colours(&c, row_ptr, col);
    ddg_plan* p = new ddg_plan();
    build_dist_plan(p->P, n, row_ptr, col, part, nparts, c.bptr.data(), c.bidx.data(), c.optr.data(),
                    c.oidx.data(), c.colour.data(), c.ncolours, block_coords, block_ndim, rank, nranks);
    p->colour = c.colour;
    p->optr = c.optr;
    p->oidx = c.oidx;
    c.device = -1;
    *out = p;
    return DDG_OK;
}

extern "C" int64_t ddg_plan_query(ddg_plan* p, int what, int colour, int peer, int32_t* out, int64_t cap) {
    if (!p) return -1;
    const ddg::DistPlan& P = p->P;
    const std::vector<int32_t>* v = nullptr;
    std::vector<int32_t> tmp;
    auto zidx = [&](int c, int q) { return (size_t)c * P.nranks + q; };
    const bool peer_ok = peer >= 0 && peer < P.nranks;
    const bool col_ok = colour >= 0 && colour < P.ncolours;
    switch (what) {
        case DDG_PLAN_OWNED_ROWS: v = &P.owned_rows; break;
        case DDG_PLAN_OWNED_SUBS: v = &P.owned_subs; break;
        case DDG_PLAN_P_SEND: if (!peer_ok) return -1; v = &P.p_send[peer]; break;
        case DDG_PLAN_P_RECV: if (!peer_ok) return -1; v = &P.p_recv[peer]; break;
        case DDG_PLAN_R_SEND: if (!peer_ok) return -1; v = &P.r_send[peer]; break;
        case DDG_PLAN_R_RECV: if (!peer_ok) return -1; v = &P.r_recv[peer]; break;
        case DDG_PLAN_Z_SEND: if (!peer_ok || !col_ok) return -1; v = &P.z_send[zidx(colour, peer)]; break;
        case DDG_PLAN_Z_RECV: if (!peer_ok || !col_ok) return -1; v = &P.z_recv[zidx(colour, peer)]; break;
        case DDG_PLAN_PROLONG_PARTS: v = &P.prolong_parts; break;
        case DDG_PLAN_COLOURS: v = &p->colour; break;
        case DDG_PLAN_PART_RANK: v = &P.part_rank; break;
        case DDG_PLAN_OVERLAP:
            if (peer < 0 || peer + 1 >= (int64_t)p->optr.size()) return -1;
            tmp.assign(p->oidx.begin() + p->optr[peer], p->oidx.begin() + p->optr[peer + 1]);
            v = &tmp;
            break;
        default: return -1;
    }
    const int64_t cnt = (int64_t)v->size();
    if (out) std::copy(v->begin(), v->begin() + std::min<int64_t>(cnt, cap), out);
    return cnt;
}

extern "C" void ddg_plan_destroy(ddg_plan* p) { delete p; }

// debug (not part of include/ddg.h): k_symv_ring role/wait cycle counters
// accumulated since the last call (DDG_RING_TRACE=1); 24 values
extern "C" int ddg_debug_ring_trace(unsigned long long* out) { return symv_ring_trace(out); }
// debug: k_pcg_small barrier timestamps (on = 1: arm; on = 0: read up to cap, returns the count)
extern "C" int ddg_debug_small_trace(int on, unsigned long long* out, int cap) { return small_trace(on, out, cap); }

// CG coefficients of the last solve (include/ddg.h)
extern "C" int ddg_get_lanczos(ddg_ctx* c, double* alphas, double* betas, int cap) {
    if (!c) return set_err(DDG_E_ARG, "null argument");
    const int k = (int)c->last_alpha.size();
    for (int j = 0; j < std::min(k, cap); ++j) {
        if (alphas) alphas[j] = c->last_alpha[j];
        if (betas && j + 1 < k) betas[j] = c->last_beta[j];
    }
    return k;
}

// Debug: blocked Gauss-Jordan on nmat host matrices (tiled layout, nTs[b] tiles
// per side, all pivoted, concatenated), in place; sym selects the symmetric
// variant (tools/gjunit.py only).
extern "C" int ddg_debug_gj(int nmat, const int32_t* nTs, double* mats, int sym) {
    std::vector<int64_t> off(nmat + 1, 0);
    int maxT = 0;
    for (int b = 0; b < nmat; ++b) {
        off[b + 1] = off[b] + (int64_t)nTs[b] * nTs[b] * TILE_ELEMS;
        maxT = std::max(maxT, (int)nTs[b]);
    }
    double* d = nullptr;
    double** dp = nullptr;
    int32_t *dn = nullptr, *dids = nullptr, *derr = nullptr;
    if (cudaMalloc(&d, off[nmat] * 8) || cudaMalloc(&dp, nmat * sizeof(double*)) || cudaMalloc(&dn, nmat * 4) ||
        cudaMalloc(&dids, nmat * 4) || cudaMalloc(&derr, 8))
        return set_err(DDG_E_OOM, "debug gj alloc");
    std::vector<double*> ptr(nmat);
    std::vector<int32_t> ids(nmat);
    for (int b = 0; b < nmat; ++b) { ptr[b] = d + off[b]; ids[b] = b; }
    int32_t herr[2] = {-1, -1};
    cudaMemcpy(d, mats, off[nmat] * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, ptr.data(), nmat * sizeof(double*), cudaMemcpyHostToDevice);
    cudaMemcpy(dn, nTs, nmat * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dids, ids.data(), nmat * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(derr, herr, 8, cudaMemcpyHostToDevice);
    launch_gj_blocked(nullptr, nmat, maxT, maxT, dp, dn, dn, dids, derr, sym ? 1 : 0);
    cudaDeviceSynchronize();
    cudaMemcpy(mats, d, off[nmat] * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(herr, derr, 8, cudaMemcpyDeviceToHost);
    cudaFree(d); cudaFree(dp); cudaFree(dn); cudaFree(dids); cudaFree(derr);
    return herr[0] >= 0 ? DDG_E_NOT_SPD : DDG_OK;
}
