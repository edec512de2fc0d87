// slab_group.cuh — one problem slab-partitioned over several contexts
// (BASELINE north_star: "large fine grids are slab-partitioned
// across 2/4/8 GPUs ... with NVLink halo exchange per smoothing sweep and
// coarse levels agglomerated below a size threshold").
//
// Included at the end of ibmg.cu (same translation unit: it drives the
// single-context kernels and helpers defined there).
//
// Partition.  Slab r owns the fine rows [r N/P, (r+1) N/P) and, on every
// distributed level l < la, the rows [r n_l/P, (r+1) n_l/P).  A slab is a full
// ibmg_ctx (whole-level vectors, so a slab's kernels index the level exactly
// as on one GPU; it computes only its own rows) whose Krylov basis holds only
// its fine rows (compact: 3 planes x rows x N).  Levels la.. are agglomerated:
// every slab holds the whole level and runs the rest of the V-cycle
// redundantly (bitwise identical on all slabs), which replaces gather-to-one
// plus broadcast by a single allgather of the restricted residual.
//
// Exchange.  Every pass that writes a distributed level is followed by
//   (1) the seam merge: a box of a slab's top cell row also owns the v face
//       in the next slab's first row (v(i, j+1), SPEC.md:418-426 box DOFs).
//       The next slab takes every entry of that row its neighbour changed
//       in the pass (k_seam_merge against a snapshot taken before it);
//   (2) the halo push: each slab copies its first and last kHalo owned rows
//       (3 planes) into the neighbours' copies, peer to peer (NVLink on
//       distinct GPUs, a device copy when slabs share one GPU).
// Ordering is by CUDA events between the slab streams; no kernel ever waits
// on another slab, so slabs may share a GPU.  The colour passes are those of
// the single-GPU schedule (4 tile colours, then the big-block colours one
// launch each), so the smoother result equals the one-context result.
//
// FGMRES dots: each slab reduces its rows (the fused CGS2 sweeps unchanged),
// then every slab sums the P partials in rank order (k_sum_ranks), so all
// slabs take bitwise identical Krylov decisions.
#pragma once

namespace {

constexpr int kHalo = 24;   // >= 2 E' reaches (<= 7 cells, checked at setup) + restriction stencil
constexpr int kStash = 64;  // doubles per partial-dot stash slot (>= 2 (restart + 2))

struct SlabPlan {
    int P = 1, nlev = 0, la = 0;
    std::vector<int> n;
    // owned rows of slab r on level l (level 0 is always row-partitioned: the
    // Krylov vectors; levels la.. (l > 0) are whole on every slab)
    int y0(int r, int l) const { return (l < la || l == 0) ? r * (n[l] / P) : 0; }
    int y1(int r, int l) const { return (l < la || l == 0) ? (r + 1) * (n[l] / P) : n[l]; }
};

SlabPlan make_plan(int N, int coarsest, int P, int min_rows, long min_cells) {
    SlabPlan S;
    S.P = P;
    for (int n = N;; n /= 2) {
        S.n.push_back(n);
        if (n <= coarsest) break;
    }
    S.nlev = int(S.n.size());
    if (P > 1)
        while (S.la < S.nlev) {
            const int n = S.n[S.la], rows = n / P;
            if (n % P || n <= kCoarseMaxN || rows % (2 * kTile) || rows < std::max(min_rows, kHalo) ||
                long(rows) * n < min_cells)
                break;
            ++S.la;
        }
    return S;
}

}  // namespace

struct ibmg_group {
    ibmg_params prm{};
    std::string err;
    SlabPlan plan;
    std::vector<ibmg_ctx*> c;
    std::vector<int> dev;
    struct Per {
        double *kb = nullptr, *kx = nullptr, *kr = nullptr;  // compact rhs, solution, residual
        double* stash = nullptr;                             // [2][kStash] partial dots
        std::vector<double*> seam_in, seam_old;              // per distributed level: n doubles
        cudaEvent_t ea = nullptr, eb = nullptr;
    };
    std::vector<Per> s;
    unsigned red_seq = 0;
    size_t Mk = 0;
    int rows = 0;  // fine rows per slab
    long long exchanges = 0;
};

namespace {

enum { VW = 0, VB = 1 };

double* lvec(ibmg_group* g, int r, int l, int which) {
    return which == VW ? g->c[r]->lev[l].w : g->c[r]->lev[l].b;
}

template <class Fn>
void each(ibmg_group* g, Fn&& fn) {
    for (int r = 0; r < g->plan.P; ++r) {
        CK(cudaSetDevice(g->dev[r]));
        fn(r, g->c[r]);
    }
}

// rows [row0, row0 + cnt) of the 3 planes of a level vector, src slab -> dst slab
// (same offsets: both hold the whole level), on the source slab's stream
void copy_rows(ibmg_group* g, int dst, int src, int l, int which, int row0, int cnt) {
    if (cnt <= 0) return;
    const size_t n = size_t(g->plan.n[l]), nn = n * n;
    double* d = lvec(g, dst, l, which) + size_t(row0) * n;
    const double* s = lvec(g, src, l, which) + size_t(row0) * n;
    CK(cudaMemcpy2DAsync(d, nn * sizeof(double), s, nn * sizeof(double), cnt * n * sizeof(double), 3,
                         cudaMemcpyDefault, g->c[src]->s));
}

// snapshot of the slab's first v row before a pass on a distributed level
void seam_snapshot(ibmg_group* g, int l) {
    const size_t n = size_t(g->plan.n[l]), nn = n * n;
    each(g, [&](int r, ibmg_ctx* c) {
        const double* row = c->lev[l].w + nn + size_t(g->plan.y0(r, l)) * n;
        CK(cudaMemcpyAsync(g->s[r].seam_old[l], row, n * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
    });
}

// seam merge (after a colour pass) and halo push of a distributed level's vector
void exchange(ibmg_group* g, int l, int which, bool seam) {
    const int P = g->plan.P, n = g->plan.n[l];
    const size_t nn = size_t(n) * n;
    ++g->exchanges;
    if (seam) {
        each(g, [&](int r, ibmg_ctx* c) {
            const int nx = (r + 1) % P;
            const double* row = c->lev[l].w + nn + size_t(g->plan.y1(r, l) % n) * n;
            CK(cudaMemcpyAsync(g->s[nx].seam_in[l], row, n * sizeof(double), cudaMemcpyDefault, c->s));
            CK(cudaEventRecord(g->s[r].ea, c->s));
        });
        each(g, [&](int r, ibmg_ctx* c) {
            const int pv = (r + P - 1) % P;
            CK(cudaStreamWaitEvent(c->s, g->s[pv].ea, 0));
            double* row = c->lev[l].w + nn + size_t(g->plan.y0(r, l)) * n;
            LAUNCH(c, k_seam_merge, nblk(n), 256, 0, row, (const double*)g->s[r].seam_in[l],
                   (const double*)g->s[r].seam_old[l], n);
        });
    }
    each(g, [&](int r, ibmg_ctx*) {
        const int pv = (r + P - 1) % P, nx = (r + 1) % P;
        const int y0 = g->plan.y0(r, l), y1 = g->plan.y1(r, l);
        copy_rows(g, pv, r, l, which, y0, kHalo);
        copy_rows(g, nx, r, l, which, y1 - kHalo, kHalo);
        CK(cudaEventRecord(g->s[r].eb, g->c[r]->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaStreamWaitEvent(c->s, g->s[(r + P - 1) % P].eb, 0));
        CK(cudaStreamWaitEvent(c->s, g->s[(r + 1) % P].eb, 0));
    });
}

// every slab's owned rows of a level vector to every other slab (the
// agglomeration onto all slabs; level 0 when nothing is distributed)
void allgather(ibmg_group* g, int l, int which, int lrows_of) {
    const int P = g->plan.P;
    ++g->exchanges;
    each(g, [&](int r, ibmg_ctx* c) {
        const int y0 = r * (g->plan.n[lrows_of] / P) >> (l - lrows_of);
        const int cnt = (g->plan.n[lrows_of] / P) >> (l - lrows_of);
        for (int d = 0; d < P; ++d)
            if (d != r) copy_rows(g, d, r, l, which, y0, cnt);
        CK(cudaEventRecord(g->s[r].eb, c->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        for (int d = 0; d < P; ++d)
            if (d != r) CK(cudaStreamWaitEvent(c->s, g->s[d].eb, 0));
    });
}

// make level 0's vector valid where the next consumer reads it
void sync0(ibmg_group* g, int which) {
    if (g->plan.la > 0) exchange(g, 0, which, false);
    else allgather(g, 0, which, 0);
}

// dh[off, off + len) of every slab <- sum over slabs (rank order)
void allreduce(ibmg_group* g, int off, int len) {
    const int P = g->plan.P;
    if (len > kStash) throw InvalidArg("allreduce: too many values");
    const int p = int(g->red_seq++ & 1u);
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaMemcpyAsync(g->s[r].stash + p * kStash, c->dh + off, len * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->s));
        CK(cudaEventRecord(g->s[r].ea, c->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        RankPtrs rp{};
        for (int d = 0; d < P; ++d) {
            if (d != r) CK(cudaStreamWaitEvent(c->s, g->s[d].ea, 0));
            rp.p[d] = g->s[d].stash + p * kStash;
        }
        LAUNCH(c, k_sum_ranks, 1, 64, 0, rp, P, len, c->dh + off);
    });
}

// compact (owned fine rows) <-> whole-level level-0 vector
void pack(ibmg_group* g, int r, const double* full, double* compact) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    CK(cudaMemcpy2DAsync(compact, w * sizeof(double), full + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double),
                         w * sizeof(double), 3, cudaMemcpyDeviceToDevice, g->c[r]->s));
}
void unpack(ibmg_group* g, int r, const double* compact, double* full) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    CK(cudaMemcpy2DAsync(full + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double), compact, w * sizeof(double),
                         w * sizeof(double), 3, cudaMemcpyDeviceToDevice, g->c[r]->s));
}

// one multicolour sweep of a distributed level: the single-GPU pass order
// (4 tile colours, then the big-block colours), each pass over the slab's own
// tiles / blocks, each followed by the seam merge and the halo push
void sweep_group(ibmg_group* g, int l) {
    const int n = g->plan.n[l], ntile = n / kTile, half = ntile / 2;
    const int rows = n / g->plan.P;
    for (int tc = 0; tc < 4; ++tc) {
        seam_snapshot(g, l);
        each(g, [&](int r, ibmg_ctx* c) {
            LevelBuf& lb = c->lev[l];
            LAUNCH(c, k_plain_tiles, half * (rows / (2 * kTile)), 32, 0, lb.L, tc, (const double*)lb.b, lb.w,
                   (const uint8_t*)lb.big, g->plan.y0(r, l) / kTile);
        });
        exchange(g, l, VW, true);
    }
    const LevelBuf& l0 = g->c[0]->lev[l];
    const int nbk = n / 4;
    for (int col = 0; col < l0.ncol; ++col) {
        // owned blocks of this colour: ids ascend within a colour, id = bx + by nbk
        std::vector<std::pair<int, int>> rng(g->plan.P);
        bool any = false;
        for (int r = 0; r < g->plan.P; ++r) {
            const LevelBuf& lb = g->c[r]->lev[l];
            const int* a = lb.h_ids.data() + lb.coff[col];
            const int* e = lb.h_ids.data() + lb.coff[col + 1];
            const int lo = int(std::lower_bound(a, e, (g->plan.y0(r, l) / 4) * nbk) - lb.h_ids.data());
            const int hi = int(std::lower_bound(a, e, (g->plan.y1(r, l) / 4) * nbk) - lb.h_ids.data());
            rng[r] = {lo, hi};
            any |= hi > lo;
        }
        if (!any) continue;
        seam_snapshot(g, l);
        each(g, [&](int r, ibmg_ctx* c) {
            const int lo = rng[r].first, hi = rng[r].second;
            if (hi <= lo) return;
            LevelBuf& lb = c->lev[l];
            BigColours BC{};
            BC.ncol = 1;
            BC.off[0] = lo;
            BC.off[1] = hi;
            const BigDeps DP{nullptr, nullptr, nullptr, 0u};
            const int grid = std::min(hi - lo, c->big_grid_max);
            if (c->prof) prof_begin(c, "k_big_phase");
            launch_k(c, k_big_phase, dim3(grid), dim3(kBigThreads), kBigSmem, true, lb.L, slabs(lb), BC, DP,
                     (const double*)lb.b, lb.w);
            if (c->prof) prof_end(c);
            ++c->launches;
        });
        exchange(g, l, VW, true);
    }
}

// coarse b (owned coarse rows) = R (b - A w) of distributed level l; coarse w = 0
void restrict_group(ibmg_group* g, int l) {
    each(g, [&](int r, ibmg_ctx* c) {
        LevelBuf& lb = c->lev[l];
        LevelBuf& nx = c->lev[l + 1];
        const int nc = nx.L.n, yc0 = g->plan.y0(r, l) / 2, yc1 = g->plan.y1(r, l) / 2;
        const PForce pf = pforce(c, lb, lb.w, nx.FL.nf > 0);
        const int ng = int(nblk(size_t(yc1 - yc0) * nc));
        Gather G = gather(c, nx, nx.b, 1.0, pf, ng);
        G.lg = nx.L.lg;
        G.jlo = yc0;
        G.jhi = yc1;
        LAUNCH(c, k_residual_restrict, pf.nblk + ng + G.nblk, 256, 0, lb.L, (const double*)lb.b,
               (const double*)lb.w, nx.b, (double*)nullptr, pf, G, ng, yc0 * nc, yc1 * nc);
        CK(cudaMemsetAsync(nx.w, 0, sizeof(double) * 3 * size_t(nx.L.nn), c->s));
    });
    if (l + 1 < g->plan.la) exchange(g, l + 1, VB, false);
    else allgather(g, l + 1, VB, l);
}

// out (owned rows of level 0) = A w, w valid on the owned rows + halo
void apply_owned(ibmg_group* g, int r, const double* w, double* out) {
    ibmg_ctx* c = g->c[r];
    LevelBuf& lb = c->lev[0];
    const int n = lb.L.n, y0 = g->plan.y0(r, 0), y1 = g->plan.y1(r, 0);
    const PForce pf = pforce(c, lb, w, lb.FL.nf > 0);
    const int ng = int(nblk(size_t(y1 - y0) * n));
    Gather G = gather(c, lb, out, -1.0, pf, ng);
    G.lg = lb.L.lg;
    G.jlo = y0;
    G.jhi = y1;
    LAUNCH(c, k_stokes_apply, pf.nblk + ng + G.nblk, 256, 0, lb.L, w, out, pf, G, ng, y0 * n, y1 * n);
}

// The V-cycle below the distributed levels on one slab: levels la..nlev-1
// with b = lev[la].b (whole) and w = lev[la].w (zero), as vcycle() does.
void vtail(ibmg_ctx* c, int la) {
    if (la >= c->lc) {
        coarse_cycle(c, c->lev[c->lc].b, c->lev[c->lc].w, c->lc > 0 ? c->lev[c->lc - 1].w : nullptr);
        return;
    }
    for (int l = la; l < c->lc; ++l) {
        LevelBuf& lb = c->lev[l];
        LevelBuf& nx = c->lev[l + 1];
        for (int s = 0; s < c->prm.nu1; ++s) sweep_level(c, l, lb.b, lb.w);
        const PForce pf = pforce(c, lb, lb.w, nx.FL.nf > 0);
        const int ng = int(nblk(nx.L.nn));
        const Gather G = gather(c, nx, nx.b, 1.0, pf, ng);
        LAUNCH(c, k_residual_restrict, pf.nblk + ng + G.nblk, 256, 0, lb.L, (const double*)lb.b,
               (const double*)lb.w, nx.b, nx.w, pf, G, ng, 0, nx.L.nn);
    }
    coarse_cycle(c, c->lev[c->lc].b, c->lev[c->lc].w, c->lev[c->lc - 1].w);
    for (int l = c->lc - 1; l >= la; --l) {
        LevelBuf& lb = c->lev[l];
        if (l < c->lc - 1)
            LAUNCH(c, k_prolong_add, nblk(lb.L.nn), 256, 0, lb.L.n, (const double*)c->lev[l + 1].w, lb.w, 0, lb.L.nn);
        for (int s = 0; s < c->prm.nu2; ++s) sweep_level(c, l, lb.b, lb.w);
    }
}

// z (compact) = V(nu1, nu2)(0, b (compact)), no mean projection (as inside FGMRES)
void vcycle_group(ibmg_group* g, const std::vector<const double*>& kb, const std::vector<double*>& kz) {
    const int la = g->plan.la;
    each(g, [&](int r, ibmg_ctx* c) {
        unpack(g, r, kb[r], c->lev[0].b);
        CK(cudaMemsetAsync(c->lev[0].w, 0, sizeof(double) * c->M, c->s));
    });
    sync0(g, VB);
    for (int l = 0; l < la; ++l) {
        for (int s = 0; s < g->prm.nu1; ++s) sweep_group(g, l);
        restrict_group(g, l);
    }
    each(g, [&](int, ibmg_ctx* c) { vtail(c, la); });
    for (int l = la - 1; l >= 0; --l) {
        // the coarse kernel already prolonged into level lc - 1 (all rows)
        if (!(l + 1 == la && la == g->c[0]->lc))
            each(g, [&](int r, ibmg_ctx* c) {
                LevelBuf& lb = c->lev[l];
                const int n = lb.L.n, y0 = g->plan.y0(r, l), y1 = g->plan.y1(r, l);
                LAUNCH(c, k_prolong_add, nblk(size_t(y1 - y0) * n), 256, 0, n, (const double*)c->lev[l + 1].w, lb.w,
                       y0 * n, y1 * n);
            });
        exchange(g, l, VW, false);
        for (int s = 0; s < g->prm.nu2; ++s) sweep_group(g, l);
    }
    each(g, [&](int r, ibmg_ctx* c) { pack(g, r, c->lev[0].w, kz[r]); });
}

// dh[off] of every slab = global a . b (compact vectors of length Mk)
void gdot(ibmg_group* g, const std::vector<const double*>& a, const std::vector<const double*>& b, size_t len, int off) {
    each(g, [&](int r, ibmg_ctx* c) {
        LAUNCH(c, k_multidot_partial, dim3(kRedBlocks, 1), kRedThreads, 0, a[r], len, b[r], len, c->partial);
        LAUNCH(c, k_finish_dots, 1, 32, 0, (const double*)c->partial, kRedBlocks, c->dh + off, 0);
    });
    allreduce(g, off, 1);
}

double read0(ibmg_group* g, int off) {
    ibmg_ctx* c = g->c[0];
    CK(cudaSetDevice(g->dev[0]));
    CK(cudaMemcpyAsync(c->hpin, c->dh + off, sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return c->hpin[0];
}

template <class Fn>
std::vector<double*> per_slab(ibmg_group* g, Fn&& fn) {
    std::vector<double*> v(g->plan.P);
    for (int r = 0; r < g->plan.P; ++r) v[r] = fn(r);
    return v;
}
std::vector<const double*> cst(const std::vector<double*>& v) { return std::vector<const double*>(v.begin(), v.end()); }

// mean-zero pressure of the compact vectors x (project_pressure_mean, fields.cpp:78-85)
void pressure_mean_zero_group(ibmg_group* g, const std::vector<double*>& x) {
    const size_t cnt = size_t(g->rows) * g->prm.N, tot = size_t(g->prm.N) * g->prm.N;
    const int off = 2 * (g->prm.restart + 2);
    auto p = per_slab(g, [&](int r) { return x[r] + 2 * cnt; });
    auto ones = per_slab(g, [&](int r) { return g->c[r]->ones; });
    gdot(g, cst(p), cst(ones), cnt, off);
    each(g, [&](int r, ibmg_ctx* c) { LAUNCH(c, k_sub_mean, nblk(cnt), 256, 0, p[r], cnt, tot, (const double*)c->dh + off); });
}

// r (compact) = b - A x (compact), returns ||r||^2 (global)
double true_residual(ibmg_group* g, const std::vector<double*>& x, const std::vector<double*>& b,
                     const std::vector<double*>& rres) {
    each(g, [&](int r, ibmg_ctx* c) { unpack(g, r, x[r], c->lev[0].w); });
    sync0(g, VW);
    each(g, [&](int r, ibmg_ctx* c) {
        apply_owned(g, r, c->lev[0].w, c->wv);
        pack(g, r, c->wv, rres[r]);
        LAUNCH(c, k_b_minus, nblk(g->Mk), 256, 0, (const double*)b[r], rres[r], g->Mk);
    });
    gdot(g, cst(rres), cst(rres), g->Mk, 0);
    return read0(g, 0);
}

// FGMRES(m) over the slabs: fgmres() with compact vectors, allreduced dots
// and the slab V-cycle (oracle fgmres()).
int fgmres_group(ibmg_group* g, ibmg_stats* st) {
    const int m = g->prm.restart;
    const size_t Mk = g->Mk;
    const int hoff = 0, h2off = m + 2;
    std::vector<double> H(size_t(m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), y(m);
    st->iters = st->restarts = st->converged = 0;
    st->relres = 0.0;
    auto kb = per_slab(g, [&](int r) { return g->s[r].kb; });
    auto kx = per_slab(g, [&](int r) { return g->s[r].kx; });
    auto kr = per_slab(g, [&](int r) { return g->s[r].kr; });
    each(g, [&](int r, ibmg_ctx* c) { CK(cudaMemsetAsync(kx[r], 0, sizeof(double) * Mk, c->s)); });
    gdot(g, cst(kb), cst(kb), Mk, hoff);
    const double bnorm = std::sqrt(read0(g, hoff));
    if (bnorm == 0.0) {
        st->converged = 1;
        return IBMG_OK;
    }
    const double tol = g->prm.rtol * bnorm;
    double beta = bnorm;
    std::vector<double*> rvec = kb;
    int it = 0, restarts = 0;
    ibmg_ctx* c0 = g->c[0];
    while (true) {
        each(g, [&](int r, ibmg_ctx* c) {
            LAUNCH(c, k_scale_by_norm, nblk(Mk), 256, 0, (const double*)rvec[r], c->V, Mk, (const double*)nullptr,
                   beta, (double*)nullptr);
        });
        std::fill(gv.begin(), gv.end(), 0.0);
        gv[0] = beta;
        int kdim = 0;
        for (int j = 0; j < m; ++j) {
            auto Vj = per_slab(g, [&](int r) { return g->c[r]->V + g->c[r]->Mst * j; });
            auto Zj = per_slab(g, [&](int r) { return g->c[r]->Z + g->c[r]->Mst * j; });
            vcycle_group(g, cst(Vj), Zj);
            // w = A z_j from the V-cycle's level-0 w (owned rows + halo valid)
            each(g, [&](int r, ibmg_ctx* c) {
                apply_owned(g, r, c->lev[0].w, c->wv);
                pack(g, r, c->wv, c->stage_a);
            });
            auto w = per_slab(g, [&](int r) { return g->c[r]->stage_a; });
            each(g, [&](int r, ibmg_ctx* c) { cgs_sweep(c, 0, j + 1, nullptr, w[r], hoff); });
            allreduce(g, hoff, j + 1);
            each(g, [&](int r, ibmg_ctx* c) { cgs_sweep(c, 1, j + 1, c->dh + hoff, w[r], h2off); });
            allreduce(g, h2off, j + 1);
            each(g, [&](int r, ibmg_ctx* c) { cgs_sweep(c, 2, j + 1, c->dh + h2off, w[r], h2off + j + 1); });
            allreduce(g, h2off + j + 1, 1);
            CK(cudaSetDevice(g->dev[0]));
            CK(cudaMemcpyAsync(c0->hpin, c0->dh, sizeof(double) * (2 * (m + 2)), cudaMemcpyDeviceToHost, c0->s));
            CK(cudaEventRecord(c0->ev_dots, c0->s));
            if (j + 1 < m)
                each(g, [&](int r, ibmg_ctx* c) {
                    LAUNCH(c, k_scale_by_norm, nblk(Mk), 256, 0, (const double*)w[r], c->V + c->Mst * (j + 1), Mk,
                           (const double*)(c->dh + h2off + j + 1), 0.0, (double*)nullptr);
                });
            CK(cudaEventSynchronize(c0->ev_dots));
            for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = c0->hpin[hoff + i] + c0->hpin[h2off + i];
            const double hnext = std::sqrt(c0->hpin[h2off + j + 1]);
            H[size_t(j + 1) * m + j] = hnext;
            for (int i = 0; i < j; ++i) {
                const double a = H[size_t(i) * m + j], cc = H[size_t(i + 1) * m + j];
                H[size_t(i) * m + j] = cs[i] * a + sn[i] * cc;
                H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * cc;
            }
            const double a = H[size_t(j) * m + j], cc = H[size_t(j + 1) * m + j];
            const double den = std::hypot(a, cc);
            cs[j] = a / den;
            sn[j] = cc / den;
            H[size_t(j) * m + j] = den;
            H[size_t(j + 1) * m + j] = 0.0;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            ++it;
            kdim = j + 1;
            if (!std::isfinite(gv[j + 1])) throw CudaError("FGMRES: non-finite residual estimate");
            if (std::fabs(gv[j + 1]) <= tol || it >= g->prm.max_iters || hnext == 0.0) break;
        }
        for (int i = kdim - 1; i >= 0; --i) {
            double sacc = gv[i];
            for (int k = i + 1; k < kdim; ++k) sacc -= H[size_t(i) * m + k] * y[k];
            y[i] = sacc / H[size_t(i) * m + i];
        }
        each(g, [&](int r, ibmg_ctx* c) {
            CK(cudaStreamSynchronize(c->s));  // hpin of this slab is free
            std::copy(y.begin(), y.begin() + kdim, c->hpin);
            CK(cudaMemcpyAsync(c->dh + h2off, c->hpin, sizeof(double) * kdim, cudaMemcpyHostToDevice, c->s));
            LAUNCH(c, k_multi_axpy_add, nblk(Mk), 256, 0, (const double*)c->Z, c->Mst, kdim,
                   (const double*)(c->dh + h2off), kx[r], Mk);
        });
        beta = std::sqrt(true_residual(g, kx, kb, kr));
        rvec = kr;
        if (beta <= tol) {
            st->converged = 1;
            break;
        }
        if (it >= g->prm.max_iters) break;
        ++restarts;
    }
    pressure_mean_zero_group(g, kx);
    st->iters = it;
    st->restarts = restarts;
    st->relres = beta / bnorm;
    return st->converged ? IBMG_OK : IBMG_NOT_CONVERGED;
}

// host whole-grid vector (3 planes) -> each slab's compact rows, and back
void scatter_host(ibmg_group* g, const double* h, const std::vector<double*>& k) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaMemcpy2DAsync(k[r], w * sizeof(double), h + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double),
                             w * sizeof(double), 3, cudaMemcpyHostToDevice, c->s));
    });
}
void gather_host(ibmg_group* g, const std::vector<double*>& k, double* h, int planes = 3, double* h_p = nullptr) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    each(g, [&](int r, ibmg_ctx* c) {
        const size_t o = size_t(g->plan.y0(r, 0)) * N;
        CK(cudaMemcpy2DAsync(h + o, nn * sizeof(double), k[r], w * sizeof(double), w * sizeof(double), planes,
                             cudaMemcpyDeviceToHost, c->s));
        if (h_p)
            CK(cudaMemcpyAsync(h_p + o, k[r] + 2 * w, w * sizeof(double), cudaMemcpyDeviceToHost, c->s));
    });
    each(g, [&](int, ibmg_ctx* c) { CK(cudaStreamSynchronize(c->s)); });
}

int gfail(ibmg_group* g, const std::exception& e, int code) {
    if (g) g->err = e.what();
    return code;
}

template <class Fn>
int gapi(ibmg_group* g, Fn&& fn) {
    if (!g) return IBMG_INVALID;
    try {
        const int rc = fn();
        for (int r = 0; r < g->plan.P; ++r) {
            CK(cudaSetDevice(g->dev[r]));
            CK(cudaStreamSynchronize(g->c[r]->s));
        }
        return rc;
    } catch (const std::invalid_argument& e) {
        return gfail(g, e, IBMG_INVALID);
    } catch (const std::exception& e) {
        return gfail(g, e, IBMG_CUDA);
    }
}

}  // namespace

extern "C" {

int ibmg_slab_plan(int N, int coarsest_n, int nslabs, int min_rows, long min_cells, int* rows_out) {
    if (N < 8 || (N & (N - 1)) || coarsest_n < 1 || nslabs < 1 || nslabs > kMaxSlabs) return -1;
    const SlabPlan S = make_plan(N, coarsest_n, nslabs, min_rows, min_cells);
    if (rows_out)
        for (int r = 0; r < nslabs; ++r)
            for (int l = 0; l < S.nlev; ++l) {
                rows_out[(size_t(r) * S.nlev + l) * 2] = S.y0(r, l);
                rows_out[(size_t(r) * S.nlev + l) * 2 + 1] = S.y1(r, l);
            }
    return S.la;
}

void ibmg_group_destroy(ibmg_group* g) {
    if (!g) return;
    for (size_t r = 0; r < g->c.size(); ++r) {
        cudaSetDevice(g->dev[r]);
        if (g->c[r]) cudaStreamSynchronize(g->c[r]->s);
        if (r < g->s.size()) {
            auto& P = g->s[r];
            dfree(P.kb);
            dfree(P.kx);
            dfree(P.kr);
            dfree(P.stash);
            for (auto& p : P.seam_in) dfree(p);
            for (auto& p : P.seam_old) dfree(p);
            if (P.ea) cudaEventDestroy(P.ea);
            if (P.eb) cudaEventDestroy(P.eb);
        }
        ibmg_destroy(g->c[r]);
    }
    delete g;
}

int ibmg_group_create(const ibmg_params* p, int nslabs, const int* devices, int min_rows, long min_cells,
                      ibmg_group** out) {
    if (!p || !out || nslabs < 1 || nslabs > kMaxSlabs) return IBMG_INVALID;
    *out = nullptr;
    if (p->N < 8 || (p->N & (p->N - 1)) || p->N % nslabs) return IBMG_INVALID;
    ibmg_group* g = new ibmg_group;
    g->prm = *p;
    g->plan = make_plan(p->N, p->coarsest_n, nslabs, min_rows, min_cells);
    g->rows = p->N / nslabs;
    for (int r = 0; r < nslabs; ++r) g->dev.push_back(devices ? devices[r] : p->device);
    try {
        for (int r = 0; r < nslabs; ++r) {
            ibmg_params q = *p;
            q.device = g->dev[r];
            ibmg_ctx* c = nullptr;
            const int rc = create_ctx(&q, g->rows, &c);
            if (rc != IBMG_OK) {
                ibmg_group_destroy(g);
                return rc;
            }
            g->c.push_back(c);
        }
        for (int r = 0; r < nslabs; ++r)
            for (int d = 0; d < nslabs; ++d)
                if (g->dev[r] != g->dev[d]) {
                    CK(cudaSetDevice(g->dev[r]));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[d], 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                    cudaGetLastError();
                }
        g->Mk = g->c[0]->Mk;
        g->s.resize(nslabs);
        for (int r = 0; r < nslabs; ++r) {
            CK(cudaSetDevice(g->dev[r]));
            auto& P = g->s[r];
            P.kb = dalloc<double>(g->Mk);
            P.kx = dalloc<double>(g->Mk);
            P.kr = dalloc<double>(g->Mk);
            P.stash = dalloc<double>(2 * kStash);
            CK(cudaMemset(P.stash, 0, sizeof(double) * 2 * kStash));
            for (int l = 0; l < g->plan.la; ++l) {
                P.seam_in.push_back(dalloc<double>(g->plan.n[l]));
                P.seam_old.push_back(dalloc<double>(g->plan.n[l]));
            }
            CK(cudaEventCreateWithFlags(&P.ea, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&P.eb, cudaEventDisableTiming));
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ibmg_group_create: %s\n", e.what());
        ibmg_group_destroy(g);
        return IBMG_CUDA;
    }
    *out = g;
    return IBMG_OK;
}

const char* ibmg_group_last_error(const ibmg_group* g) { return g ? g->err.c_str() : "null group"; }
int ibmg_group_distributed_levels(const ibmg_group* g) { return g ? g->plan.la : -1; }
long long ibmg_group_kernel_launches(const ibmg_group* g) {
    if (!g) return -1;
    long long s = 0;
    for (auto* c : g->c) s += c->launches;
    return s;
}
long long ibmg_group_exchanges(const ibmg_group* g) { return g ? g->exchanges : -1; }

int ibmg_group_set_structures(ibmg_group* g, int n_mem, const int* nb, const double* kappa, const double* ds,
                              const double* X) {
    return gapi(g, [&]() -> int {
        if (n_mem > 0 && (!nb || !kappa || !ds || !X)) throw InvalidArg("null structure arrays");
        each(g, [&](int, ibmg_ctx* c) { set_structures(c, n_mem, nb, kappa, ds, X, IBMG_PTR_HOST); });
        return IBMG_OK;
    });
}

int ibmg_group_sweep(ibmg_group* g, int level, const double* b, double* w) {
    return gapi(g, [&]() -> int {
        if (level < 0 || level >= g->plan.la) throw InvalidArg("group sweep: level is not distributed");
        const size_t m = 3 * size_t(g->plan.n[level]) * g->plan.n[level];
        each(g, [&](int, ibmg_ctx* c) {
            CK(cudaMemcpyAsync(c->lev[level].b, b, m * sizeof(double), cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(c->lev[level].w, w, m * sizeof(double), cudaMemcpyHostToDevice, c->s));
        });
        sweep_group(g, level);
        const size_t n = size_t(g->plan.n[level]), nn = n * n;
        each(g, [&](int r, ibmg_ctx* c) {
            const size_t o = size_t(g->plan.y0(r, level)) * n, cnt = size_t(g->plan.y1(r, level)) * n - o;
            CK(cudaMemcpy2DAsync(w + o, nn * sizeof(double), c->lev[level].w + o, nn * sizeof(double),
                                 cnt * sizeof(double), 3, cudaMemcpyDeviceToHost, c->s));
        });
        return IBMG_OK;
    });
}

int ibmg_group_vcycle(ibmg_group* g, const double* b, double* z) {
    return gapi(g, [&]() -> int {
        auto kb = per_slab(g, [&](int r) { return g->s[r].kb; });
        auto kx = per_slab(g, [&](int r) { return g->s[r].kx; });
        scatter_host(g, b, kb);
        vcycle_group(g, cst(kb), kx);
        pressure_mean_zero_group(g, kx);
        gather_host(g, kx, z);
        return IBMG_OK;
    });
}

int ibmg_group_solve(ibmg_group* g, const double* b, double* x, ibmg_stats* st) {
    ibmg_stats local{};
    if (!st) st = &local;
    return gapi(g, [&]() -> int {
        const double t0 = now_ms();
        scatter_host(g, b, per_slab(g, [&](int r) { return g->s[r].kb; }));
        const int rc = fgmres_group(g, st);
        gather_host(g, per_slab(g, [&](int r) { return g->s[r].kx; }), x);
        st->solve_ms = now_ms() - t0;
        st->total_ms = st->solve_ms;
        return rc;
    });
}

int ibmg_group_step(ibmg_group* g, double* u, double* p, double* X, ibmg_stats* st) {
    ibmg_stats local{};
    if (!st) st = &local;
    return gapi(g, [&]() -> int {
        if (!g->c[0]->have_structs) throw InvalidArg("ibmg_group_step: call ibmg_group_set_structures first");
        const double t0 = now_ms();
        const size_t nn = size_t(g->prm.N) * g->prm.N;
        // lagged operators at X^n on every slab (redundant setup), RHS rows
        each(g, [&](int r, ibmg_ctx* c) {
            if (c->npts)
                CK(cudaMemcpyAsync(c->X, X, sizeof(double) * 2 * c->npts, cudaMemcpyHostToDevice, c->s));
            rebuild(c);
            CK(cudaMemcpyAsync(c->stage_a, u, sizeof(double) * 2 * nn, cudaMemcpyHostToDevice, c->s));
            build_rhs(c, c->stage_a, c->bv);
            pack(g, r, c->bv, g->s[r].kb);
        });
        each(g, [&](int, ibmg_ctx* c) { CK(cudaStreamSynchronize(c->s)); });
        const double t1 = now_ms();
        const int rc = fgmres_group(g, st);
        auto kx = per_slab(g, [&](int r) { return g->s[r].kx; });
        gather_host(g, kx, u, 2, p);
        const double t2 = now_ms();
        // X^{n+1} = X^n + dt S^T u^{n+1} on every slab (whole u^{n+1})
        each(g, [&](int, ibmg_ctx* c) {
            CK(cudaMemcpyAsync(c->stage_a, u, sizeof(double) * 2 * nn, cudaMemcpyHostToDevice, c->s));
            if (c->npts)
                LAUNCH(c, k_interp, nblk(c->npts, 128), 128, 0, c->lev[0].W, c->npts, c->prm.N, c->lev[0].L.h,
                       (const double*)c->stage_a, (double*)nullptr, c->X, c->prm.dt);
        });
        ibmg_ctx* c0 = g->c[0];
        CK(cudaSetDevice(g->dev[0]));
        if (c0->npts) CK(cudaMemcpyAsync(X, c0->X, sizeof(double) * 2 * c0->npts, cudaMemcpyDeviceToHost, c0->s));
        st->setup_ms = t1 - t0;
        st->solve_ms = t2 - t1;
        st->total_ms = now_ms() - t0;
        return rc;
    });
}

}  // extern "C"
