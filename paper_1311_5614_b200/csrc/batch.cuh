// batch.cuh — a batch of independent problems (C5: 512 independent N = 256
// implicit steps) stepped in LOCKSTEP through one set of launches.
//
// Each problem keeps its own context (structures, hierarchy, box inverses,
// Krylov basis: ibmg_ctx), rebuilt on the context's own stream; the solve of
// all of them then runs on the batch stream, one launch per phase for the
// whole batch:
// * the dataflow sweep of a level (k_sweep_df_b) runs the tile tasks and the
//   big-block tasks of ALL active problems as one DAG: tile task t belongs to
//   problem act[t mod nA], big-block tasks come in colour-major order with the
//   problems interleaved inside a colour.  Every task still waits only on
//   tasks of its own problem that come earlier in the order, so the result is
//   each problem's colour-ordered schedule (bitwise the per-context sweep),
//   while one problem's dependency waits are filled with the other problems'
//   tasks: per-problem latency chains become throughput;
// * restriction, prolongation, the operator apply and the two CGS2 passes put
//   the problem index in grid.y; the coarse cycle runs one CTA per problem;
// * FGMRES(m) advances all active problems one Arnoldi step per round: one
//   device-to-host copy of every problem's dots per round, the Givens updates
//   on the host per problem; a converged problem leaves the active set.  A
//   problem that reaches the restart length unconverged, or whose true
//   residual misses the tolerance, is finished by the single-context FGMRES.
//
// Requires every level n >= 64 to be a dataflow level (N <= 512): C5 is 256.
#pragma once

namespace ibmg {

constexpr int kBMaxLev = 4;  // multi-tile levels of a batch problem (512 .. 64)

// One problem, one multi-tile level l < lc.
struct BLev {
    DfArgs df;         // sweep; df.b / df.w are unused on level 0 (V_j, Z_j)
    double* ec;        // w of level l + 1 (prolongation source; l + 1 < lc)
    // residual + restriction into level l + 1
    double* bc;        // b of level l + 1
    double* wcz;       // w of level l + 1 (zeroed)
    PForce pf;         // pf.w set at launch
    Gather G;          // G.cnt: the problem's batch counter, target = producer CTAs
    ERes R;            // E'-row variant: R.cnt the same counter
    int mode;          // 0 tiled + factored E', 1 tiled + E' rows
    int ngrid, nnc, total;
};

struct BProb {
    BLev lv[kBMaxLev];
    int lc;
    CoarseArgs co;     // co.w_fine replaced by Z_j when lc == 1
    Lev L0;
    PForce apf;        // apply on level 0 (out = wv)
    Gather aG;
    int ang, atotal;
    double *wv, *rv, *V, *Z;
    size_t Mst, M;
    double* partial;
    double* dh;
    unsigned* ticket;
    unsigned long long* cnt;  // batch-owned, reset before each fused launch
};

struct BTask {
    int b, q;  // problem (slot), big-block list position
};

__device__ __forceinline__ const double* blev_b(const BProb& P, int l, int j) {
    return l == 0 ? P.V + (size_t)j * P.Mst : P.lv[l].df.b;
}
__device__ __forceinline__ double* blev_w(const BProb& P, int l, int j) {
    return l == 0 ? P.Z + (size_t)j * P.Mst : P.lv[l].df.w;
}

// Batched dataflow sweep of level l (cooperative: all CTAs co-resident).
template <bool ES>
__global__ void __launch_bounds__(32 * kDfWarps, ES ? 2 : 1)
    k_sweep_df_b(const BProb* __restrict__ P, int l, int j, unsigned eadd, const int* __restrict__ act, int nA,
                 const BTask* __restrict__ bt, int nbt) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char dsm[];
    SlabSlot* slot = reinterpret_cast<SlabSlot*>(dsm);
    ESlot* eslot = reinterpret_cast<ESlot*>(dsm);
    __shared__ BigScratch S;
    const int t = threadIdx.x, wid = t >> 5, G = gridDim.x;
    const int n = P[act[0]].lv[l].df.L.n, nn = n * n;
    const int nt = n / kTile, ntiles = nt * nt, per = ntiles / 4, half = nt >> 1, nbk = n >> 2;
    double* sw = reinterpret_cast<double*>(dsm + (ES ? sizeof(ESlot) : 2 * sizeof(SlabSlot)) + wid * kDfTileStride);
    double* sb = sw + kDfWDoubles;
    int k = blockIdx.x;  // this CTA's big tasks: k, k + G, ...
    if (k < nbt) {
        const BTask it = bt[k];
        const Slabs& SL = P[it.b].lv[l].df.SL;
        if (ES) eslot_issue(*eslot, SL, it.q, t, 32 * kDfWarps);
        else slab_issue(slot[0], SL, it.q, t, 32 * kDfWarps);
    }
    cp_async_commit();
    // ---- plain tasks of every active problem: task t -> problem act[t mod nA]
    for (int task = blockIdx.x * kDfWarps + wid; task < nA * ntiles; task += G * kDfWarps) {
        const int b = act[task % nA], loc = task / nA;
        const int tc = loc / per, i = loc - tc * per;
        const BProb& PB = P[b];
        const DfArgs& A = PB.lv[l].df;
        const Lev L = A.L;
        df_plain_tile(L, blev_b(PB, l, j), blev_w(PB, l, j), A.big, A.tflags, A.DP.epoch + eadd,
                      2 * (i % half) + (tc & 1), 2 * (i / half) + (tc >> 1), tc, sw, sb, nullptr);
    }
    __syncthreads();
    // ---- big tasks (colour-major, problems interleaved within a colour)
    for (int r = 0; k < nbt; k += G, ++r) {
        const BTask it = bt[k];
        const int kn = k + G;
        const BProb& PB = P[it.b];
        const DfArgs& A = PB.lv[l].df;
        const Lev L = A.L;
        if (!ES) {
            if (kn < nbt) {
                const BTask nx = bt[kn];
                slab_issue(slot[(r + 1) & 1], P[nx.b].lv[l].df.SL, nx.q, t, 32 * kDfWarps);
            }
            cp_async_commit();
        }
        const unsigned epoch = A.DP.epoch + eadd;
        double* w = blev_w(PB, l, j);
        const double* bb = blev_b(PB, l, j);
        const int q = it.q;
        const int Bk = A.SL.rp[(size_t)q * 48 + 47];
        const int bi = 4 * (Bk % nbk), bj = 4 * (Bk / nbk);
        for (int e = A.DP.poff[q] + t; e < A.DP.poff[q + 1]; e += 32 * kDfWarps)
            while (ld_acquire(A.DP.flags + A.DP.pred[e]) != epoch) __nanosleep(8);
        if (t < 9) {  // plain tiles within 8 cells of the block
            const int tx0 = (bi - 8) >> 4, ty0 = (bj - 8) >> 4;
            const int tx = tx0 + t % 3, ty = ty0 + t / 3;
            if (tx * kTile <= bi + 11 && ty * kTile <= bj + 11)
                while (ld_acquire(A.tflags + wr(tx, nt) + wr(ty, nt) * nt) != epoch) __nanosleep(8);
        }
        __syncthreads();
        if (ES) cp_async_wait<0>();
        else cp_async_wait<1>();
        __syncthreads();
        GAccCG Wg{w, n, nn};
        GAccB Bg{bb, n, nn};
        auto wadd = [&](int f, int i, int jj, double old, double d) {
            __stcg(w + (size_t)f * nn + i + (size_t)jj * n, old + d);
        };
        if (ES) {
            big_block_es<0>(L, *eslot, A.SL.Ainv + (size_t)q * 3136, bi, bj, Wg, FlatCG{w}, Bg, wadd, S, t,
                            [] { __syncthreads(); },
                            [&] {
                                if (kn < nbt) {
                                    const BTask nx = bt[kn];
                                    eslot_issue(*eslot, P[nx.b].lv[l].df.SL, nx.q, t, 32 * kDfWarps);
                                }
                                cp_async_commit();
                            },
                            nullptr, nullptr, SlabTail{&A.SL, q});
        } else {
            big_block_slab(L, slot[r & 1], bi, bj, Wg, FlatCG{w}, FlatCG{w}, Bg, wadd, S, t, nullptr,
                           SlabTail{&A.SL, q});
        }
        __syncthreads();
        if (t == 0) st_release(A.DP.flags + q, epoch);
    }
    cp_async_wait<0>();
}

// Split form of a batched sweep (throughput regime: many problems): the
// plain phase of every active problem as one launch of one-warp CTAs (13 per
// SM by shared memory; tile tasks colour-major, problems interleaved), then
// the big blocks as one launch of 128-thread CTAs (4 per SM: one E'-row slot,
// the inverse streamed into registers; k_big_phase's scheme) over the batch's
// colour-major task list.  The blocks no longer overlap the tiles, but twice
// as many tasks are in flight per SM as in the one-launch sweep.
__global__ void __launch_bounds__(32) k_plain_b(const BProb* __restrict__ P, int l, int j, unsigned eadd,
                                                const int* __restrict__ act, int nA) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char pdm[];
    double* sw = reinterpret_cast<double*>(pdm);
    double* sb = sw + kDfWDoubles;
    const int n = P[act[0]].lv[l].df.L.n, nt = n / kTile, ntiles = nt * nt, per = ntiles / 4, half = nt >> 1;
    for (int task = blockIdx.x; task < nA * ntiles; task += gridDim.x) {
        const int b = act[task % nA], loc = task / nA;
        const int tc = loc / per, i = loc - tc * per;
        const BProb& PB = P[b];
        const DfArgs& A = PB.lv[l].df;
        const Lev L = A.L;
        df_plain_tile(L, blev_b(PB, l, j), blev_w(PB, l, j), A.big, A.tflags, A.DP.epoch + eadd,
                      2 * (i % half) + (tc & 1), 2 * (i / half) + (tc >> 1), tc, sw, sb, nullptr);
    }
}

__global__ void __launch_bounds__(kBigThreads) k_big_b(const BProb* __restrict__ P, int l, int j, unsigned eadd,
                                                       const BTask* __restrict__ bt, int nbt) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char dsm[];
    ESlot* slot = reinterpret_cast<ESlot*>(dsm);
    __shared__ BigScratch S;
    const int t = threadIdx.x, G = gridDim.x;
    int k = blockIdx.x;
    if (k < nbt) eslot_issue(*slot, P[bt[k].b].lv[l].df.SL, bt[k].q, t, kBigThreads);
    cp_async_commit();
    for (; k < nbt; k += G) {
        const BTask it = bt[k];
        const int kn = k + G;
        const BProb& PB = P[it.b];
        const DfArgs& A = PB.lv[l].df;
        const Lev L = A.L;
        const int n = L.n, nn = L.nn, nbk = n >> 2, q = it.q;
        const unsigned epoch = A.DP.epoch + eadd;
        double* w = blev_w(PB, l, j);
        const double* bb = blev_b(PB, l, j);
        for (int e = A.DP.poff[q] + t; e < A.DP.poff[q + 1]; e += kBigThreads)
            while (ld_acquire(A.DP.flags + A.DP.pred[e]) != epoch) __nanosleep(8);
        cp_async_wait<0>();
        __syncthreads();
        const int Bk = slot->rp[47];
        GAccCG Wg{w, n, nn};
        GAccB Bg{bb, n, nn};
        big_block_es(L, *slot, A.SL.Ainv + (size_t)q * 3136, 4 * (Bk % nbk), 4 * (Bk / nbk), Wg, FlatCG{w}, Bg,
                     [&](int f, int i, int jj, double old, double d) {
                         __stcg(w + (size_t)f * nn + i + (size_t)jj * n, old + d);
                     },
                     S, t, [] { __syncthreads(); },
                     [&] {
                         if (kn < nbt) eslot_issue(*slot, P[bt[kn].b].lv[l].df.SL, bt[kn].q, t, kBigThreads);
                         cp_async_commit();
                     },
                     nullptr, nullptr, SlabTail{&A.SL, q});
        __syncthreads();
        if (t == 0) st_release(A.DP.flags + q, epoch);
    }
    cp_async_wait<0>();
}

// Batched residual + restriction of level l (grid.y = active problem).
__global__ void __launch_bounds__(256) k_rr_b(const BProb* __restrict__ P, int l, int j, const int* __restrict__ act) {
    __shared__ __align__(16) RrSmem S;
    pdl_enter();
    const BProb& PB = P[act[blockIdx.y]];
    const BLev& R = PB.lv[l];
    const int bid = blockIdx.x;
    if (bid >= R.total) return;
    const double* bb = blev_b(PB, l, j);
    const double* w = blev_w(PB, l, j);
    const Lev F = R.df.L;
    if (R.mode == 1) {
        ERes E = R.R;
        E.cnt = PB.cnt;
        residual_restrict_e_at(F, bb, w, R.bc, R.wcz, E, 0, R.nnc, bid, S);
    } else {
        PForce pf = R.pf;
        pf.w = w;
        Gather G = R.G;
        G.cnt = PB.cnt;
        fused_launch_at(pf, G, R.ngrid, bid,
                        [&](int blk) { residual_restrict_tile(F, bb, w, R.bc, R.wcz, blk, 0, R.nnc, S); });
    }
}

// Batched prolongation + add into level l from level l + 1 (l + 1 < lc).
__global__ void k_prolong_b(const BProb* __restrict__ P, int l, int j, const int* __restrict__ act) {
    pdl_enter();
    const BProb& PB = P[act[blockIdx.y]];
    const int nf = PB.lv[l].df.L.n, nnf = nf * nf;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nnf) return;
    double* wf = blev_w(PB, l, j);
    GAcc acc{PB.lv[l].ec, nf >> 1, (nf >> 1) * (nf >> 1)};
    double du, dv, dp;
    prolong_rows(nf, acc, q % nf, q / nf, du, dv, dp);
    wf[q] += du;
    wf[nnf + q] += dv;
    wf[2 * nnf + q] += dp;
}

// Batched coarse cycle: one CTA per active problem.
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_cycle_b(const BProb* __restrict__ P, int j,
                                                                    const int* __restrict__ act) {
    pdl_enter();
    const BProb& PB = P[act[blockIdx.x]];
    coarse_cycle_body(PB.co, PB.lc == 1 ? PB.Z + (size_t)j * PB.Mst : PB.co.w_fine);
}

// Batched operator apply on level 0: wv = A Z_j (grid.y = active problem).
__global__ void __launch_bounds__(256) k_apply_b(const BProb* __restrict__ P, int j, const int* __restrict__ act) {
    __shared__ __align__(16) ApSmem S;
    pdl_enter();
    const BProb& PB = P[act[blockIdx.y]];
    const int bid = blockIdx.x;
    if (bid >= PB.atotal) return;
    const double* w = PB.Z + (size_t)j * PB.Mst;
    PForce pf = PB.apf;
    pf.w = w;
    Gather G = PB.aG;
    G.cnt = PB.cnt;
    const Lev L0 = PB.L0;
    fused_launch_at(pf, G, PB.ang, bid, [&](int blk) { apply_tile(L0, w, PB.wv, blk, 0, L0.nn, S); });
}

template <int KMAX, bool FLAT = false>
__global__ void __launch_bounds__(kRedThreads, KMAX > 16 ? 2 : 3)
    k_ortho_dots_b(const BProb* __restrict__ P, int k, int ld, const int* __restrict__ act) {
    pdl_enter();
    const BProb& PB = P[act[blockIdx.y]];
    ortho_dots_at<KMAX, false, FLAT>(PB.V, PB.Mst, k, PB.wv, PB.M, PB.partial, PB.dh, ld, PB.ticket, (int)blockIdx.x,
                        (int)gridDim.x);
}

template <int KMAX>
__global__ void __launch_bounds__(kRedThreads, 4 / (KMAX > 16 ? 2 : 1))
    k_ortho_update_b(const BProb* __restrict__ P, int k, int ld, int more, const int* __restrict__ act) {
    pdl_enter();
    const BProb& PB = P[act[blockIdx.y]];
    ortho_update_at<KMAX>(PB.V, PB.Mst, k, PB.wv, more ? PB.V + (size_t)k * PB.Mst : PB.rv,
                          more ? PB.Z + (size_t)k * PB.Mst : nullptr, PB.M, PB.partial, PB.dh, ld, PB.ticket,
                          (int)blockIdx.x, (int)gridDim.x);
}

// The first `cnt` entries of every active problem's dh, contiguous (one copy to the host).
__global__ void k_gather_dh(const BProb* __restrict__ P, const int* __restrict__ act, int nA, int cnt,
                            double* __restrict__ out) {
    pdl_enter();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nA * cnt; i += gridDim.x * blockDim.x) {
        const int a = i / cnt;
        out[i] = P[act[a]].dh[i - a * cnt];
    }
}

}  // namespace ibmg

// ---------------- host side ----------------
struct ibmg_batch {
    ibmg_params prm{};
    std::string err;
    std::vector<ibmg_ctx*> ctx;
    std::vector<cudaEvent_t> ev_ready;
    cudaStream_t s = nullptr;
    cudaEvent_t ev_dots = nullptr, ev_done = nullptr;
    bool pdl = true;
    long long launches = 0;
    int df_grid_es = 1, df_grid = 1;
    ibmg::BProb* dP = nullptr;   // device table
    ibmg::BProb* hP = nullptr;   // pinned host table
    int* d_act = nullptr;
    int* h_act = nullptr;
    unsigned long long* d_cnt = nullptr;
    ibmg::BTask* d_bt = nullptr;  // all levels' big-task lists, level-major
    ibmg::BTask* h_bt = nullptr;  // pinned
    long bt_cap = 0;
    int bt_off[ibmg::kBMaxLev + 1] = {0};
    double* d_dh = nullptr;
    double* h_dh = nullptr;  // pinned
    int prepared = 0;        // slots rebuilt by ibmg_batch_prepare, awaiting ibmg_batch_solve
    int prep_threads = 4;    // host threads of ibmg_batch_prepare (IBMG_BATCH_THREADS)
    bool split = true;       // split sweeps from split_min active problems (IBMG_BATCH_SPLIT=0: one launch)
    int split_min = 8;
    int pdf_grid = 1, big_grid = 1;
    double prep_ms = 0.0;
};

namespace {

template <typename... KArgs, typename... Args>
void launch_b(ibmg_batch* B, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, bool coop, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = B->s;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (B->pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
    ++B->launches;
}

// The per-problem launch table of the current structures (after the rebuilds).
void batch_table(ibmg_batch* B, int count) {
    using namespace ibmg;
    for (int k = 0; k < count; ++k) {
        ibmg_ctx* c = B->ctx[k];
        BProb& P = B->hP[k];
        P = BProb{};
        P.lc = c->lc;
        for (int l = 0; l < c->lc; ++l) {
            LevelBuf& lb = c->lev[l];
            LevelBuf& nx = c->lev[l + 1];
            BLev& BL = P.lv[l];
            BigColours BC;
            BC.ncol = lb.ncol;
            for (int q = 0; q <= kMaxColours; ++q) BC.off[q] = lb.coff[q];
            BL.df = DfArgs{lb.L, slabs(lb), BC, BigDeps{lb.pred, lb.poff, lb.flags, lb.epoch}, lb.tflags, lb.big,
                           lb.b, lb.w, nullptr};
            BL.ec = nx.w;
            BL.bc = nx.b;
            BL.wcz = nx.w;
            const int nc = nx.L.n;
            BL.nnc = nc * nc;
            BL.ngrid = (nc / kRrTx) * ((nc + kRrTy - 1) / kRrTy);
            if (lb.rr_csr) {
                BL.mode = 1;
                BL.R = ERes{lb.FL, lb.E, lb.escr, int(nblk(lb.FL.nf, 8)), nullptr, 0ull};
                BL.R.target = (unsigned long long)BL.R.nblk;
                BL.total = BL.R.nblk + BL.ngrid;
            } else {
                BL.mode = 0;
                BL.pf = pforce(c, lb, nullptr, nx.FL.nf > 0);
                BL.G = Gather{nx.FL, nx.W, c->F, nx.b, nx.L.nn, 1.0, 0, nullptr, 0ull};
                BL.G.sub = nx.maxrow <= 32 ? 8 : 32;
                if (BL.pf.nblk) {
                    BL.G.nblk = int(nblk(nx.FL.nf, gather_faces_per_cta(BL.G.sub)));
                    BL.G.target = (unsigned long long)(BL.pf.nblk + BL.ngrid);
                }
                BL.total = BL.pf.nblk + BL.ngrid + BL.G.nblk;
            }
        }
        P.co = coarse_args(c, c->lev[c->lc].b, c->lev[c->lc].w, c->lc > 1 ? c->lev[c->lc - 1].w : nullptr);
        LevelBuf& l0 = c->lev[0];
        P.L0 = l0.L;
        P.apf = pforce(c, l0, nullptr, l0.FL.nf > 0);
        P.ang = (l0.L.n / kApTx) * (l0.L.n / kApTy);
        P.aG = Gather{l0.FL, l0.W, c->F, c->wv, l0.L.nn, -1.0, 0, nullptr, 0ull};
        P.aG.sub = l0.maxrow <= 32 ? 8 : 32;
        if (P.apf.nblk) {
            P.aG.nblk = int(nblk(l0.FL.nf, gather_faces_per_cta(P.aG.sub)));
            P.aG.target = (unsigned long long)(P.apf.nblk + P.ang);
        }
        P.atotal = P.apf.nblk + P.ang + P.aG.nblk;
        P.wv = c->wv;
        P.rv = c->rv;
        P.V = c->V;
        P.Z = c->Z;
        P.Mst = c->Mst;
        P.M = c->M;
        P.partial = c->partial;
        P.dh = c->dh;
        P.ticket = c->ticket;
        P.cnt = B->d_cnt + k;
    }
    CK(cudaMemcpyAsync(B->dP, B->hP, sizeof(BProb) * size_t(count), cudaMemcpyHostToDevice, B->s));
}

// Active list + every level's big-task list (colour-major, problems
// interleaved within a colour) for the given active problems.
void batch_tasks(ibmg_batch* B, const std::vector<int>& act) {
    using namespace ibmg;
    const int nA = int(act.size());
    for (int a = 0; a < nA; ++a) B->h_act[a] = act[a];
    const int lc = B->ctx[act[0]]->lc;
    long tot = 0;
    for (int l = 0; l < lc; ++l)
        for (int b : act) tot += B->ctx[b]->lev[l].nbig;
    if (tot > B->bt_cap) {
        if (B->h_bt) CK(cudaFreeHost(B->h_bt));
        dfree(B->d_bt);
        B->bt_cap = grow_cap(tot, B->bt_cap);
        CK(cudaMallocHost(&B->h_bt, sizeof(BTask) * size_t(B->bt_cap)));
        B->d_bt = dalloc<BTask>(size_t(B->bt_cap));
    }
    long o = 0;
    for (int l = 0; l < lc; ++l) {
        B->bt_off[l] = int(o);
        int maxc = 0;
        for (int b : act) maxc = std::max(maxc, B->ctx[b]->lev[l].ncol);
        for (int col = 0; col < maxc; ++col) {
            int maxr = 0;
            for (int b : act) {
                const LevelBuf& lb = B->ctx[b]->lev[l];
                if (col < lb.ncol) maxr = std::max(maxr, lb.coff[col + 1] - lb.coff[col]);
            }
            for (int r = 0; r < maxr; ++r)
                for (int b : act) {
                    const LevelBuf& lb = B->ctx[b]->lev[l];
                    if (col < lb.ncol && r < lb.coff[col + 1] - lb.coff[col]) B->h_bt[o++] = BTask{b, lb.coff[col] + r};
                }
        }
    }
    B->bt_off[lc] = int(o);
    CK(cudaMemcpyAsync(B->d_act, B->h_act, sizeof(int) * size_t(nA), cudaMemcpyHostToDevice, B->s));
    if (o) CK(cudaMemcpyAsync(B->d_bt, B->h_bt, sizeof(BTask) * size_t(o), cudaMemcpyHostToDevice, B->s));
}

void batch_sweep(ibmg_batch* B, int l, int j, unsigned eadd, int nA) {
    using namespace ibmg;
    const int nbt = B->bt_off[l + 1] - B->bt_off[l];
    const BTask* bt = B->d_bt + B->bt_off[l];
    if (B->split && nA >= B->split_min) {  // throughput regime: split launches (k_plain_b / k_big_b)
        const int nt = B->ctx[0]->lev[l].L.n / kTile;
        launch_b(B, k_plain_b, dim3(std::min(B->pdf_grid, nA * nt * nt)), dim3(32), kPdfSmem, true,
                 (const BProb*)B->dP, l, j, eadd, (const int*)B->d_act, nA);
        if (nbt)
            launch_b(B, k_big_b, dim3(std::min(B->big_grid, nbt)), dim3(kBigThreads), kBigSmem, true,
                     (const BProb*)B->dP, l, j, eadd, bt, nbt);
        return;
    }
    // E'-row-slot variant (2 CTAs/SM) when the batch's blocks outnumber 1 CTA/SM (kDfEsMinBig)
    if (nbt >= kDfEsMinBig)
        launch_b(B, k_sweep_df_b<true>, dim3(B->df_grid_es), dim3(32 * kDfWarps), kDfSmemES, true,
                 (const BProb*)B->dP, l, j, eadd, (const int*)B->d_act, nA, bt, nbt);
    else
        launch_b(B, k_sweep_df_b<false>, dim3(B->df_grid), dim3(32 * kDfWarps), kDfSmem, true, (const BProb*)B->dP,
                 l, j, eadd, (const int*)B->d_act, nA, bt, nbt);
}

// One V(nu1, nu2) cycle of every active problem on (V_j, Z_j); Z_j is zero.
void batch_vcycle(ibmg_batch* B, int j, int nA, std::vector<unsigned>& eadd) {
    using namespace ibmg;
    ibmg_ctx* c0 = B->ctx[B->h_act[0]];
    const int lc = c0->lc, nu1 = c0->prm.nu1, nu2 = c0->prm.nu2;
    int maxtot[kBMaxLev] = {0};
    for (int l = 0; l < lc; ++l)
        for (int a = 0; a < nA; ++a) maxtot[l] = std::max(maxtot[l], B->hP[B->h_act[a]].lv[l].total);
    for (int l = 0; l < lc; ++l) {
        for (int s = 0; s < nu1; ++s) batch_sweep(B, l, j, ++eadd[l], nA);
        CK(cudaMemsetAsync(B->d_cnt, 0, sizeof(unsigned long long) * B->ctx.size(), B->s));
        launch_b(B, k_rr_b, dim3(maxtot[l], nA), dim3(256), 0, false, (const BProb*)B->dP, l, j,
                 (const int*)B->d_act);
    }
    launch_b(B, k_coarse_cycle_b, dim3(nA), dim3(kCoarseThreads), coarse_smem(c0), false, (const BProb*)B->dP, j,
             (const int*)B->d_act);
    for (int l = lc - 1; l >= 0; --l) {
        if (l < lc - 1)
            launch_b(B, k_prolong_b, dim3(nblk(c0->lev[l].L.nn), nA), dim3(256), 0, false, (const BProb*)B->dP, l, j,
                     (const int*)B->d_act);
        for (int s = 0; s < nu2; ++s) batch_sweep(B, l, j, ++eadd[l], nA);
    }
}

template <int KM, bool FLAT = false>
void batch_ortho_k(ibmg_batch* B, int k, int ld, int more, int nA) {
    using namespace ibmg;
    const size_t M = B->ctx[0]->Mk;
    const int pc = B->ctx[0]->ortho_per_cta;
    launch_b(B, (k_ortho_dots_b<KM, FLAT>), dim3(ortho_dots_grid<KM>(M, pc), nA), dim3(kRedThreads), 0, false,
             (const BProb*)B->dP, k, ld, (const int*)B->d_act);
}
template <int KM>
void batch_update_k(ibmg_batch* B, int k, int ld, int more, int nA) {
    using namespace ibmg;
    const size_t M = B->ctx[0]->Mk;
    const int pc = B->ctx[0]->ortho_per_cta;
    launch_b(B, k_ortho_update_b<KM>, dim3(ortho_update_grid(M, pc), nA), dim3(kRedThreads), 0, false, (const BProb*)B->dP, k, ld,
             more, (const int*)B->d_act);
}
void batch_ortho(ibmg_batch* B, int k, int ld, int more, int nA) {
    if (k <= ibmg::kOrthoFlatK) batch_ortho_k<8, true>(B, k, ld, more, nA);
    else if (k <= 8) batch_ortho_k<8>(B, k, ld, more, nA);
    else if (k <= 16) batch_ortho_k<16>(B, k, ld, more, nA);
    else batch_ortho_k<32>(B, k, ld, more, nA);
    if (k - 1 <= 8) batch_update_k<8>(B, k, ld, more, nA);
    else if (k - 1 <= 16) batch_update_k<16>(B, k, ld, more, nA);
    else if (k - 1 <= 24) batch_update_k<24>(B, k, ld, more, nA);
    else batch_update_k<32>(B, k, ld, more, nA);
}

// Per-problem FGMRES state on the host (the arithmetic of fgmres2).
struct BState {
    std::vector<double> Hx, Ha, cs, sn, g, y;
    double bnorm = -1.0, tol = 0.0, beta = 0.0, nu0 = 1.0;
    int it = 0, kdim = 0;
    bool active = true, finish = false, fallback = false, converged = false;
};

// Runs fn with the context's work on the batch stream (the context's own
// stream is idle while the batch solves).
template <class Fn>
void on_batch_stream(ibmg_batch* B, ibmg_ctx* c, Fn&& fn) {
    cudaStream_t own = c->s;
    c->s = B->s;
    try {
        fn();
    } catch (...) {
        c->s = own;
        throw;
    }
    c->s = own;
}

// Lockstep FGMRES(m) (fgmres2 per problem) over problems 0..count-1:
// x_k = ctx_k->xv solves A_k x = ctx_k->bv.  Returns per-problem stats.
void batch_fgmres(ibmg_batch* B, int count, std::vector<ibmg_stats>& st) {
    using namespace ibmg;
    const int m = B->prm.restart, ld = m + 2, SC = 5 * ld, bslot = 6 * ld + 2, cnt = bslot + 1;
    std::vector<BState> S(count);
    for (int k = 0; k < count; ++k) {
        ibmg_ctx* c = B->ctx[k];
        BState& P = S[k];
        P.Hx.assign(size_t(m + 1) * m, 0.0);
        P.Ha.assign(size_t(m + 1) * m, 0.0);
        P.cs.assign(m, 0.0);
        P.sn.assign(m, 0.0);
        P.g.assign(m + 1, 0.0);
        P.y.assign(m, 0.0);
        on_batch_stream(B, c, [&] {
            CK(cudaMemsetAsync(c->xv, 0, sizeof(double) * c->M, c->s));
            multidot(c, c->bv, 1, c->bv, bslot, 0);
            LAUNCH(c, k_scale_by_norm, nblk(c->M), 256, 0, (const double*)c->bv, c->V, c->M,
                   (const double*)(c->dh + bslot), 0.0, c->Z);
        });
    }
    std::vector<int> act;
    for (int k = 0; k < count; ++k) act.push_back(k);
    batch_tasks(B, act);
    const int lc = B->ctx[0]->lc;
    std::vector<unsigned> eadd(lc, 0u);
    for (int j = 0; j < m && !act.empty(); ++j) {
        const int nA = int(act.size());
        const bool more = j + 1 < m;
        batch_vcycle(B, j, nA, eadd);
        int maxat = 0;
        for (int b : act) maxat = std::max(maxat, B->hP[b].atotal);
        CK(cudaMemsetAsync(B->d_cnt, 0, sizeof(unsigned long long) * B->ctx.size(), B->s));
        launch_b(B, k_apply_b, dim3(maxat, nA), dim3(256), 0, false, (const BProb*)B->dP, j, (const int*)B->d_act);
        batch_ortho(B, j + 1, ld, more ? 1 : 0, nA);
        launch_b(B, k_gather_dh, dim3(std::max(1, (nA * cnt + 255) / 256)), dim3(256), 0, false, (const BProb*)B->dP,
                 (const int*)B->d_act, nA, cnt, B->d_dh);
        CK(cudaMemcpyAsync(B->h_dh, B->d_dh, sizeof(double) * size_t(nA) * cnt, cudaMemcpyDeviceToHost, B->s));
        CK(cudaEventRecord(B->ev_dots, B->s));
        CK(cudaEventSynchronize(B->ev_dots));
        std::vector<int> fin;
        for (int a = 0; a < nA; ++a) {
            const int k = act[a];
            BState& P = S[k];
            ibmg_ctx* c = B->ctx[k];
            const double* hp = B->h_dh + size_t(a) * cnt;
            if (P.bnorm < 0.0) {
                check_deferred_err(c);
                P.bnorm = std::sqrt(hp[bslot]);
                P.tol = c->prm.rtol * P.bnorm;
                P.beta = P.bnorm;
                P.g[0] = P.beta;
                if (P.bnorm == 0.0) {  // x = 0
                    P.converged = true;
                    P.active = false;
                    fin.push_back(-1 - k);
                    continue;
                }
            }
            const double nu = hp[SC + 2], h = hp[SC + 3], bnext = std::sqrt(hp[SC + 4]);
            if (j > 0 && !(nu > 0.0)) {  // breakdown
                for (int i = 0; i < j; ++i) P.Hx[size_t(i) * m + j - 1] += hp[ld + i];
                P.Hx[size_t(j) * m + j - 1] = 0.0;
                fin.push_back(k);
                continue;
            }
            if (j == 0) {
                P.nu0 = nu;
            } else {
                for (int i = 0; i < j; ++i) P.Hx[size_t(i) * m + j - 1] += hp[ld + i];
                P.Hx[size_t(j) * m + j - 1] = nu;
            }
            for (int i = 0; i < j; ++i) P.Hx[size_t(i) * m + j] = hp[i];
            P.Hx[size_t(j) * m + j] = h;
            P.Hx[size_t(j + 1) * m + j] = bnext;
            for (int i = 0; i <= j + 1; ++i) P.Ha[size_t(i) * m + j] = P.Hx[size_t(i) * m + j];
            for (int i = 0; i < j; ++i) {
                const double aa = P.Ha[size_t(i) * m + j], cc = P.Ha[size_t(i + 1) * m + j];
                P.Ha[size_t(i) * m + j] = P.cs[i] * aa + P.sn[i] * cc;
                P.Ha[size_t(i + 1) * m + j] = -P.sn[i] * aa + P.cs[i] * cc;
            }
            const double aa = P.Ha[size_t(j) * m + j], cc = P.Ha[size_t(j + 1) * m + j];
            const double den = std::hypot(aa, cc);
            P.cs[j] = aa / den;
            P.sn[j] = cc / den;
            P.g[j + 1] = -P.sn[j] * P.g[j];
            P.g[j] = P.cs[j] * P.g[j];
            ++P.it;
            P.kdim = j + 1;
            if (!std::isfinite(P.g[j + 1])) throw CudaError("batched FGMRES: non-finite residual estimate");
            if (std::fabs(P.g[j + 1]) <= P.tol || P.it >= c->prm.max_iters || bnext == 0.0 || !more) fin.push_back(k);
        }
        if (fin.empty()) continue;
        // finishing problems: least squares, x = Z y, true residual (their own launches, batch stream)
        std::vector<int> chk;
        for (int f : fin) {
            if (f < 0) continue;
            const int k = f;
            BState& P = S[k];
            ibmg_ctx* c = B->ctx[k];
            P.active = false;
            on_batch_stream(B, c, [&] {
                hessenberg_lsq(P.Hx, m, P.kdim, P.beta * P.nu0, P.y);
                std::copy(P.y.begin(), P.y.begin() + P.kdim, c->hpin);
                CK(cudaMemcpyAsync(c->dh + 4 * ld, c->hpin, sizeof(double) * P.kdim, cudaMemcpyHostToDevice, c->s));
                LAUNCH(c, k_multi_axpy_add, nblk(c->M), 256, 0, c->Z, c->Mst, P.kdim, c->dh + 4 * ld, c->xv, c->M);
                apply_level(c, 0, c->xv, c->rv);
                LAUNCH(c, k_b_minus, nblk(c->M), 256, 0, c->bv, c->rv, c->M);
                multidot(c, c->rv, 1, c->rv, 0, 0);
                CK(cudaMemcpyAsync(c->hpin + ld, c->dh, sizeof(double), cudaMemcpyDeviceToHost, c->s));
            });
            chk.push_back(k);
        }
        if (!chk.empty()) CK(cudaStreamSynchronize(B->s));
        for (int k : chk) {
            BState& P = S[k];
            P.beta = std::sqrt(B->ctx[k]->hpin[ld]);
            if (P.beta <= P.tol) P.converged = true;
            else P.fallback = true;  // restart needed: finished by the single-context FGMRES
        }
        std::vector<int> nact;
        for (int k : act)
            if (S[k].active) nact.push_back(k);
        act.swap(nact);
        if (!act.empty()) batch_tasks(B, act);
    }
    // epochs: every batched sweep advanced each level's epoch by one
    for (int k = 0; k < count; ++k)
        for (int l = 0; l < lc; ++l) B->ctx[k]->lev[l].epoch += eadd[l];
    st.assign(count, ibmg_stats{});
    for (int k = 0; k < count; ++k) {
        ibmg_ctx* c = B->ctx[k];
        BState& P = S[k];
        if (P.fallback || P.active) {  // single-context FGMRES from x = 0, on the batch stream
            on_batch_stream(B, c, [&] { fgmres(c, c->bv, c->xv, &st[k]); });
            st[k].iters += P.it;  // the lockstep iterations spent as well
            continue;
        }
        on_batch_stream(B, c, [&] { pressure_mean_zero(c, c->xv); });
        st[k].iters = P.it;
        st[k].restarts = 0;
        st[k].converged = P.converged ? 1 : 0;
        st[k].relres = P.bnorm > 0.0 ? P.beta / P.bnorm : 0.0;
    }
}

int bfail(ibmg_batch* B, const std::exception& e, int code) {
    if (B) B->err = e.what();
    return code;
}

template <class Fn>
int bapi(ibmg_batch* B, Fn&& fn) {
    if (!B) return IBMG_INVALID;
    try {
        CK(cudaSetDevice(B->prm.device));
        return fn();
    } catch (const std::invalid_argument& e) {
        return bfail(B, e, IBMG_INVALID);
    } catch (const std::exception& e) {
        return bfail(B, e, IBMG_CUDA);
    }
}

}  // namespace

extern "C" {

int ibmg_batch_create(const ibmg_params* p, int nslots, ibmg_batch** out) {
    using namespace ibmg;
    if (!p || !out || nslots < 1 || nslots > 256) return IBMG_INVALID;
    if (p->N < 64 || p->N > kDataflowMaxN) return IBMG_INVALID;  // every multi-tile level a dataflow level
    *out = nullptr;
    ibmg_batch* B = new ibmg_batch;
    B->prm = *p;
    B->pdl = std::getenv("IBMG_NO_PDL") == nullptr;
    if (const char* e = std::getenv("IBMG_BATCH_THREADS")) B->prep_threads = std::max(1, std::atoi(e));
    try {
        CK(cudaSetDevice(p->device));
        for (int k = 0; k < nslots; ++k) {
            ibmg_ctx* c = nullptr;
            const int rc = create_ctx(p, p->N, &c);
            if (rc != IBMG_OK) throw CudaError("ibmg_batch_create: context creation failed");
            B->ctx.push_back(c);
            if (c->cl_ok || c->lc > kBMaxLev || c->df_maxn < p->N)
                throw InvalidArg("ibmg_batch_create: the batch runs the dataflow path only (IBMG_CLUSTER / IBMG_DF_MAXN)");
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            B->ev_ready.push_back(e);
        }
        B->df_grid = B->ctx[0]->df_grid_max;
        B->df_grid_es = B->ctx[0]->df_grid_max_es;
        CK(cudaFuncSetAttribute(k_sweep_df_b<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDfSmem)));
        CK(cudaFuncSetAttribute(k_sweep_df_b<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kDfSmemES)));
        {
            int per_sm = 0, sms = 0;
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_df_b<true>, 32 * kDfWarps, kDfSmemES));
            B->df_grid_es = std::max(1, per_sm * sms);
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_df_b<false>, 32 * kDfWarps, kDfSmem));
            B->df_grid = std::max(1, per_sm * sms);
        }
        CK(cudaFuncSetAttribute(k_coarse_cycle_b, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(coarse_smem(B->ctx[0]))));
        CK(cudaFuncSetAttribute(k_plain_b, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPdfSmem)));
        CK(cudaFuncSetAttribute(k_big_b, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kBigSmem)));
        {
            int per_sm = 0, sms = 0;
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_plain_b, 32, kPdfSmem));
            B->pdf_grid = std::max(1, per_sm * sms);
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_big_b, kBigThreads, kBigSmem));
            B->big_grid = std::max(1, per_sm * sms);
        }
        if (const char* e = std::getenv("IBMG_BATCH_SPLIT")) B->split = std::atoi(e) != 0;
        CK(cudaStreamCreateWithFlags(&B->s, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&B->ev_dots, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&B->ev_done, cudaEventDisableTiming));
        B->dP = dalloc<BProb>(size_t(nslots));
        CK(cudaMallocHost(&B->hP, sizeof(BProb) * size_t(nslots)));
        B->d_act = dalloc<int>(size_t(nslots));
        CK(cudaMallocHost(&B->h_act, sizeof(int) * size_t(nslots)));
        B->d_cnt = dalloc<unsigned long long>(size_t(nslots));
        const int cnt = 6 * (p->restart + 2) + 3;
        B->d_dh = dalloc<double>(size_t(nslots) * cnt);
        CK(cudaMallocHost(&B->h_dh, sizeof(double) * size_t(nslots) * cnt));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ibmg_batch_create: %s\n", e.what());
        ibmg_batch_destroy(B);
        return IBMG_CUDA;
    }
    *out = B;
    return IBMG_OK;
}

void ibmg_batch_destroy(ibmg_batch* B) {
    if (!B) return;
    cudaSetDevice(B->prm.device);
    if (B->s) cudaStreamSynchronize(B->s);
    for (auto* c : B->ctx) ibmg_destroy(c);
    for (auto e : B->ev_ready) cudaEventDestroy(e);
    dfree(B->dP);
    dfree(B->d_act);
    dfree(B->d_cnt);
    dfree(B->d_bt);
    dfree(B->d_dh);
    if (B->hP) cudaFreeHost(B->hP);
    if (B->h_act) cudaFreeHost(B->h_act);
    if (B->h_bt) cudaFreeHost(B->h_bt);
    if (B->h_dh) cudaFreeHost(B->h_dh);
    if (B->ev_dots) cudaEventDestroy(B->ev_dots);
    if (B->ev_done) cudaEventDestroy(B->ev_done);
    if (B->s) cudaStreamDestroy(B->s);
    delete B;
}

const char* ibmg_batch_last_error(const ibmg_batch* B) { return B ? B->err.c_str() : "null batch"; }
long long ibmg_batch_kernel_launches(const ibmg_batch* B) {
    if (!B) return -1;
    long long n = B->launches;
    for (auto* c : B->ctx) n += c->launches;
    return n;
}
void* ibmg_batch_stream(const ibmg_batch* B) { return B ? (void*)B->s : nullptr; }

int ibmg_batch_set_structures(ibmg_batch* B, int slot, int n_mem, const int* nb, const double* kappa,
                              const double* ds, const double* X) {
    return bapi(B, [&]() -> int {
        if (slot < 0 || slot >= int(B->ctx.size())) throw InvalidArg("batch slot out of range");
        if (n_mem > 0 && (!nb || !kappa || !ds || !X)) throw InvalidArg("null structure arrays");
        set_structures(B->ctx[slot], n_mem, nb, kappa, ds, X, IBMG_PTR_HOST, true);
        return IBMG_OK;
    });
}

// Phase 1 of a batch step: X^n and u^n in, every slot's operators rebuilt at
// X^n and its RHS built, on the slots' own streams (another thread may run
// ibmg_batch_solve of ANOTHER batch meanwhile: the host colouring and the
// rebuild kernels overlap that batch's solve).
int ibmg_batch_prepare(ibmg_batch* B, int count, double* const* u, double* const* X, int ptr_kind) {
    using namespace ibmg;
    return bapi(B, [&]() -> int {
        if (count < 1 || count > int(B->ctx.size()) || !u || !X) throw InvalidArg("batch prepare arguments");
        const double t0 = now_ms();
        const size_t nn = size_t(B->prm.N) * B->prm.N;
        for (int k = 0; k < count; ++k)
            if (!B->ctx[k]->have_structs) throw InvalidArg("ibmg_batch_prepare: set the structures of every slot first");
        // the slots' rebuilds (host colouring + setup kernels with their host
        // round trips) on worker threads, slots round-robin: each context
        // has its own streams and pinned buffers
        auto work = [&](int w, int nw) {
            CK(cudaSetDevice(B->prm.device));
            for (int k = w; k < count; k += nw) {
                ibmg_ctx* c = B->ctx[k];
                wait_inputs(c, ptr_kind);
                const cudaMemcpyKind kin =
                    ptr_kind == IBMG_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
                if (c->npts) CK(cudaMemcpyAsync(c->X, X[k], sizeof(double) * 2 * c->npts, kin, c->s));
                CK(cudaMemcpyAsync(c->stage_a, u[k], sizeof(double) * 2 * nn, kin, c->s));
                rebuild(c, true);
                c->built_dirty = false;
                build_rhs(c, c->stage_a, c->bv);
                CK(cudaEventRecord(B->ev_ready[k], c->s));
            }
        };
        const int nw = std::max(1, std::min(B->prep_threads, count));
        std::vector<std::future<void>> jobs;
        for (int w = 1; w < nw; ++w) jobs.push_back(std::async(std::launch::async, work, w, nw));
        std::exception_ptr first;
        try {
            work(0, nw);
        } catch (...) {
            first = std::current_exception();
        }
        for (auto& j : jobs) {
            try {
                j.get();
            } catch (...) {
                if (!first) first = std::current_exception();
            }
        }
        if (first) std::rethrow_exception(first);
        B->prepared = count;
        B->prep_ms = now_ms() - t0;
        return IBMG_OK;
    });
}

// Phase 2: the lockstep solve of the prepared slots, X^{n+1} = X^n + dt S*u,
// results out (u[k] 2N^2, p[k] N^2, X[k]).
int ibmg_batch_solve(ibmg_batch* B, int count, double* const* u, double* const* p, double* const* X,
                     ibmg_stats* stats, int ptr_kind) {
    using namespace ibmg;
    return bapi(B, [&]() -> int {
        if (count < 1 || count != B->prepared || !u || !p || !X)
            throw InvalidArg("batch solve: call ibmg_batch_prepare with the same count first");
        B->prepared = 0;
        const double t1 = now_ms();
        const size_t nn = size_t(B->prm.N) * B->prm.N;
        for (int k = 0; k < count; ++k) CK(cudaStreamWaitEvent(B->s, B->ev_ready[k], 0));
        batch_table(B, count);
        std::vector<ibmg_stats> st;
        batch_fgmres(B, count, st);
        const cudaMemcpyKind kout = ptr_kind == IBMG_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        for (int k = 0; k < count; ++k) {
            ibmg_ctx* c = B->ctx[k];
            on_batch_stream(B, c, [&] {
                if (c->npts)
                    LAUNCH(c, k_interp, nblk(c->npts, 128), 128, 0, c->lev[0].W, c->npts, c->prm.N, c->lev[0].L.h,
                           c->xv, (double*)nullptr, c->X, c->prm.dt);
                CK(cudaMemcpyAsync(u[k], c->xv, sizeof(double) * 2 * nn, kout, c->s));
                CK(cudaMemcpyAsync(p[k], c->xv + 2 * nn, sizeof(double) * nn, kout, c->s));
                if (c->npts) CK(cudaMemcpyAsync(X[k], c->X, sizeof(double) * 2 * c->npts, kout, c->s));
            });
        }
        CK(cudaStreamSynchronize(B->s));
        // the slots' own streams follow the batch stream (their next rebuild
        // must not overwrite what this solve used)
        CK(cudaEventRecord(B->ev_done, B->s));
        for (int k = 0; k < count; ++k) CK(cudaStreamWaitEvent(B->ctx[k]->s, B->ev_done, 0));
        const double t2 = now_ms();
        int rc = IBMG_OK;
        for (int k = 0; k < count; ++k) {
            if (stats) {
                stats[k] = st[k];
                stats[k].setup_ms = B->prep_ms / count;
                stats[k].solve_ms = (t2 - t1) / count;
                stats[k].total_ms = (B->prep_ms + t2 - t1) / count;
            }
            if (!st[k].converged) rc = IBMG_NOT_CONVERGED;
        }
        return rc;
    });
}

// One implicit step of problems 0..count-1 (SPEC.md:548-552 each), in lockstep:
// u[k] (2N^2 in/out), p[k] (N^2 out), X[k] (in/out) host or device arrays.
int ibmg_batch_step(ibmg_batch* B, int count, double* const* u, double* const* p, double* const* X,
                    ibmg_stats* stats, int ptr_kind) {
    const int rc = ibmg_batch_prepare(B, count, u, X, ptr_kind);
    if (rc != IBMG_OK) return rc;
    return ibmg_batch_solve(B, count, u, p, X, stats, ptr_kind);
}

}  // extern "C"
