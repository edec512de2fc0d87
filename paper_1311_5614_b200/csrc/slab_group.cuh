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
//   (2) the halo push: each slab's first and last kHalo owned rows (3 planes)
//       go to the neighbours' copies.
// In-process groups do both inside the pass kernels (peer stores of the
// boundary rows into the neighbours' copies, common.cuh Mirror) and only
// synchronise with the neighbours afterwards; NCCL groups exchange after it.
// The colour passes are those of the single-GPU schedule (4 tile colours,
// then the big-block colours one launch each), so a distributed sweep equals
// the one-context sweep bit for bit (tests/test_slab_group.py).
//
// Two transports, the same schedule:
//   * in-process group (ibmg_group_create): all P slabs in one process, slab
//     r on devices[r]; exchanges are peer copies (NVLink between GPUs, a
//     device copy when slabs share a GPU) ordered by CUDA events between the
//     slab streams — no kernel waits on another slab, so slabs may share a GPU;
//   * NCCL group (ibmg_group_create_nccl): one slab per process (torchrun, one
//     rank per GPU); halos and seams are ncclSend/ncclRecv pairs, dots an
//     ncclAllReduce and the agglomeration an in-place ncclAllGather, all
//     stream-ordered on the slab's stream (no host synchronisation).
//
// FGMRES dots: each slab reduces its rows (the fused CGS2 sweeps unchanged),
// then the P partials are summed (in rank order in-process; by NCCL, whose
// result is identical on every rank), so all slabs take the same Krylov
// decisions.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

namespace {

// NCCL is resolved at run time (dlopen of libnccl.so.2) the first time an NCCL
// group is made: single-GPU use needs no NCCL, and a process that already
// loaded torch's NCCL shares that copy instead of loading a second one.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
};

const NcclApi* nccl_load() {
    static NcclApi api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
#define IBMG_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    IBMG_NCCL_SYM(GetUniqueId);
    IBMG_NCCL_SYM(CommInitRank);
    IBMG_NCCL_SYM(CommDestroy);
    IBMG_NCCL_SYM(GetErrorString);
    IBMG_NCCL_SYM(GroupStart);
    IBMG_NCCL_SYM(GroupEnd);
    IBMG_NCCL_SYM(Send);
    IBMG_NCCL_SYM(Recv);
    IBMG_NCCL_SYM(AllReduce);
    IBMG_NCCL_SYM(AllGather);
#undef IBMG_NCCL_SYM
    const bool ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GetErrorString && api.GroupStart &&
                    api.GroupEnd && api.Send && api.Recv && api.AllReduce && api.AllGather;
    return ok ? &api : nullptr;
}
const NcclApi* nccl_api() {
    static const NcclApi* api = nccl_load();  // thread-safe one-time initialisation
    return api;
}
const NcclApi& nccl() {
    const NcclApi* a = nccl_api();
    if (!a) throw std::runtime_error("libnccl.so.2 not found (NCCL slab groups need it)");
    return *a;
}

constexpr int kHalo = kHaloRows;  // >= 2 E' reaches (<= 7 cells, checked at setup) + restriction stencil
constexpr int kStash = 64;  // doubles per partial-dot stash slot (>= restart + 1)

struct SlabPlan {
    int P = 1, nlev = 0, la = 0;
    std::vector<int> n;
    // owned rows of slab r on level l (level 0 is always row-partitioned: the
    // Krylov vectors; levels la.. (l > 0) are whole on every slab)
    int y0(int r, int l) const { return (l < la || l == 0) ? r * (n[l] / P) : 0; }
    int y1(int r, int l) const { return (l < la || l == 0) ? (r + 1) * (n[l] / P) : n[l]; }
};

// min_rows < 0: test mode, levels are distributed even for P = 1 (every
// exchange then goes to the slab itself).
SlabPlan make_plan(int N, int coarsest, int P, int min_rows, long min_cells) {
    SlabPlan S;
    S.P = P;
    for (int n = N;; n /= 2) {
        S.n.push_back(n);
        if (n <= coarsest) break;
    }
    S.nlev = int(S.n.size());
    if (P > 1 || min_rows < 0)
        while (S.la < S.nlev) {
            const int n = S.n[S.la], rows = n / P;
            if (n % P || n <= kCoarseMaxN || rows % (2 * kTile) || rows < std::max(min_rows, kHalo) ||
                long(rows) * n < min_cells)
                break;
            ++S.la;
        }
    return S;
}

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define NC(x)                                                                                              \
    do {                                                                                                   \
        ncclResult_t e_ = (x);                                                                             \
        if (e_ != ncclSuccess)                                                                             \
            throw NcclError(std::string(#x) + ": " + nccl().GetErrorString(e_) + " @" + std::to_string(__LINE__)); \
    } while (0)

}  // namespace

struct ibmg_group {
    ibmg_params prm{};
    std::string err;
    SlabPlan plan;
    // local slabs: ranks r0 .. r0 + c.size() - 1 (in-process group: all P
    // slabs, r0 = 0; NCCL group: this process's one slab, r0 = its rank)
    int r0 = 0;
    ncclComm_t comm = nullptr;
    std::vector<ibmg_ctx*> c;
    std::vector<int> dev;
    struct Per {
        double *kb = nullptr, *kx = nullptr, *kr = nullptr;  // compact rhs, solution, residual
        double* stash = nullptr;                             // [2][kStash] partial dots (in-process)
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

// slab r's context / scratch (r must be local)
ibmg_ctx* cx(ibmg_group* g, int r) { return g->c[size_t(r - g->r0)]; }
ibmg_group::Per& pr(ibmg_group* g, int r) { return g->s[size_t(r - g->r0)]; }

double* lvec(ibmg_group* g, int r, int l, int which) {
    return which == VW ? cx(g, r)->lev[l].w : cx(g, r)->lev[l].b;
}

// fn(rank, ctx) over the local slabs, each with its device current
template <class Fn>
void each(ibmg_group* g, Fn&& fn) {
    for (size_t i = 0; i < g->c.size(); ++i) {
        CK(cudaSetDevice(g->dev[i]));
        fn(g->r0 + int(i), g->c[i]);
    }
}

// rows [row0, row0 + cnt) of the 3 planes of a level vector, src slab -> dst
// slab (same offsets: both hold the whole level), on the source slab's stream
void copy_rows(ibmg_group* g, int dst, int src, int l, int which, int row0, int cnt) {
    if (cnt <= 0) return;
    const size_t n = size_t(g->plan.n[l]), nn = n * n;
    double* d = lvec(g, dst, l, which) + size_t(row0) * n;
    const double* s = lvec(g, src, l, which) + size_t(row0) * n;
    if (d == s) return;  // a one-slab test group exchanging with itself
    CK(cudaMemcpy2DAsync(d, nn * sizeof(double), s, nn * sizeof(double), cnt * n * sizeof(double), 3,
                         cudaMemcpyDefault, cx(g, src)->s));
}

// snapshot of the slab's first v row before a pass on a distributed level
void seam_snapshot(ibmg_group* g, int l) {
    const size_t n = size_t(g->plan.n[l]), nn = n * n;
    each(g, [&](int r, ibmg_ctx* c) {
        const double* row = c->lev[l].w + nn + size_t(g->plan.y0(r, l)) * n;
        CK(cudaMemcpyAsync(pr(g, r).seam_old[l], row, n * sizeof(double), cudaMemcpyDeviceToDevice, c->s));
    });
}

void seam_merge(ibmg_group* g, int r, ibmg_ctx* c, int l) {
    const size_t n = size_t(g->plan.n[l]), nn = n * n;
    double* row = c->lev[l].w + nn + size_t(g->plan.y0(r, l)) * n;
    LAUNCH(c, k_seam_merge, nblk(n), 256, 0, row, (const double*)pr(g, r).seam_in[l],
           (const double*)pr(g, r).seam_old[l], int(n));
}

// NCCL transport of exchange(): per plane, the last kHalo rows go to the next
// slab and the first kHalo rows to the previous one.  Messages between one
// pair are matched in posting order, so sends post "to next" before "to
// previous" and receives "from previous" before "from next" (P = 2: both
// neighbours are the same rank).
void exchange_nccl(ibmg_group* g, int r, ibmg_ctx* c, int l, int which, bool seam) {
    const int P = g->plan.P, n = g->plan.n[l];
    const size_t nn = size_t(n) * n, hn = size_t(kHalo) * n;
    const int pv = (r + P - 1) % P, nx = (r + 1) % P;
    const int y0 = g->plan.y0(r, l), y1 = g->plan.y1(r, l);
    if (seam) {
        NC(nccl().GroupStart());
        NC(nccl().Send(c->lev[l].w + nn + size_t(y1 % n) * n, size_t(n), ncclDouble, nx, g->comm, c->s));
        NC(nccl().Recv(pr(g, r).seam_in[l], size_t(n), ncclDouble, pv, g->comm, c->s));
        NC(nccl().GroupEnd());
        seam_merge(g, r, c, l);
    }
    double* v = lvec(g, r, l, which);
    NC(nccl().GroupStart());
    for (int f = 0; f < 3; ++f) {
        double* pl = v + size_t(f) * nn;
        NC(nccl().Send(pl + size_t(y1 - kHalo) * n, hn, ncclDouble, nx, g->comm, c->s));
        NC(nccl().Send(pl + size_t(y0) * n, hn, ncclDouble, pv, g->comm, c->s));
        NC(nccl().Recv(pl + size_t((y0 - kHalo + n) % n) * n, hn, ncclDouble, pv, g->comm, c->s));
        NC(nccl().Recv(pl + size_t(y1 % n) * n, hn, ncclDouble, nx, g->comm, c->s));
    }
    NC(nccl().GroupEnd());
}

// seam merge (after a colour pass) and halo push of a distributed level's vector
void exchange(ibmg_group* g, int l, int which, bool seam) {
    const int P = g->plan.P, n = g->plan.n[l];
    const size_t nn = size_t(n) * n;
    ++g->exchanges;
    if (g->comm) {
        each(g, [&](int r, ibmg_ctx* c) { exchange_nccl(g, r, c, l, which, seam); });
        return;
    }
    if (seam) {
        each(g, [&](int r, ibmg_ctx* c) {
            const int nx = (r + 1) % P;
            const double* row = c->lev[l].w + nn + size_t(g->plan.y1(r, l) % n) * n;
            CK(cudaMemcpyAsync(pr(g, nx).seam_in[l], row, n * sizeof(double), cudaMemcpyDefault, c->s));
            CK(cudaEventRecord(pr(g, r).ea, c->s));
        });
        each(g, [&](int r, ibmg_ctx* c) {
            CK(cudaStreamWaitEvent(c->s, pr(g, (r + P - 1) % P).ea, 0));
            seam_merge(g, r, c, l);
        });
    }
    each(g, [&](int r, ibmg_ctx* c) {
        const int y0 = g->plan.y0(r, l), y1 = g->plan.y1(r, l);
        copy_rows(g, (r + P - 1) % P, r, l, which, y0, kHalo);
        copy_rows(g, (r + 1) % P, r, l, which, y1 - kHalo, kHalo);
        CK(cudaEventRecord(pr(g, r).eb, c->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaStreamWaitEvent(c->s, pr(g, (r + P - 1) % P).eb, 0));
        CK(cudaStreamWaitEvent(c->s, pr(g, (r + 1) % P).eb, 0));
    });
}

// every slab's rows [r cnt, (r+1) cnt) of the 3 planes of an n x n vector
// (vec(r) on slab r) to every other slab: the agglomeration onto all slabs
template <class VecFn>
void allgather_rows(ibmg_group* g, int n, int cnt, VecFn&& vec) {
    const int P = g->plan.P;
    const size_t nn = size_t(n) * n, cn = size_t(cnt) * n;
    ++g->exchanges;
    if (g->comm) {
        each(g, [&](int r, ibmg_ctx* c) {
            double* v = vec(r);
            NC(nccl().GroupStart());
            for (int f = 0; f < 3; ++f)
                NC(nccl().AllGather(v + f * nn + size_t(r) * cn, v + f * nn, cn, ncclDouble, g->comm, c->s));
            NC(nccl().GroupEnd());
        });
        return;
    }
    each(g, [&](int r, ibmg_ctx* c) {
        for (int d = 0; d < P; ++d)
            if (d != r)
                CK(cudaMemcpy2DAsync(vec(d) + size_t(r) * cn, nn * sizeof(double), vec(r) + size_t(r) * cn,
                                     nn * sizeof(double), cn * sizeof(double), 3, cudaMemcpyDefault, c->s));
        CK(cudaEventRecord(pr(g, r).eb, c->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        for (int d = 0; d < P; ++d)
            if (d != r) CK(cudaStreamWaitEvent(c->s, pr(g, d).eb, 0));
    });
}

void allgather_level(ibmg_group* g, int l, int which, int rows_of) {
    const int cnt = (g->plan.n[rows_of] / g->plan.P) >> (l - rows_of);
    allgather_rows(g, g->plan.n[l], cnt, [&](int r) { return lvec(g, r, l, which); });
}

// make level 0's vector valid where the next consumer reads it
void sync0(ibmg_group* g, int which) {
    if (g->plan.la > 0) exchange(g, 0, which, false);
    else allgather_level(g, 0, which, 0);
}

// dh[off, off + len) of every slab <- sum over slabs
void allreduce(ibmg_group* g, int off, int len) {
    const int P = g->plan.P;
    if (len > kStash) throw InvalidArg("allreduce: too many values");
    if (g->comm) {
        each(g, [&](int, ibmg_ctx* c) {
            NC(nccl().AllReduce(c->dh + off, c->dh + off, size_t(len), ncclDouble, ncclSum, g->comm, c->s));
        });
        return;
    }
    // in-process: every slab sums the stashed partials in rank order; the
    // stash is double-buffered, so a slab may run one allreduce ahead
    const int p = int(g->red_seq++ & 1u);
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaMemcpyAsync(pr(g, r).stash + p * kStash, c->dh + off, len * sizeof(double), cudaMemcpyDeviceToDevice,
                           c->s));
        CK(cudaEventRecord(pr(g, r).ea, c->s));
    });
    each(g, [&](int r, ibmg_ctx* c) {
        RankPtrs rp{};
        for (int d = 0; d < P; ++d) {
            if (d != r) CK(cudaStreamWaitEvent(c->s, pr(g, d).ea, 0));
            rp.p[d] = pr(g, d).stash + p * kStash;
        }
        LAUNCH(c, k_sum_ranks, 1, 64, 0, rp, P, len, c->dh + off);
    });
}

// compact (owned fine rows) <-> whole-level level-0 vector
void pack(ibmg_group* g, int r, const double* full, double* compact) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    CK(cudaMemcpy2DAsync(compact, w * sizeof(double), full + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double),
                         w * sizeof(double), 3, cudaMemcpyDeviceToDevice, cx(g, r)->s));
}
void unpack(ibmg_group* g, int r, const double* compact, double* full) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    CK(cudaMemcpy2DAsync(full + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double), compact, w * sizeof(double),
                         w * sizeof(double), 3, cudaMemcpyDeviceToDevice, cx(g, r)->s));
}

// owned blocks of colour `col` on level l: list positions [lo, hi) (ids ascend
// within a colour, id = bx + by nbk, so a slab's rows are one range)
std::pair<int, int> owned_blocks(ibmg_group* g, int r, int l, int col) {
    const LevelBuf& lb = cx(g, r)->lev[l];
    const int nbk = g->plan.n[l] / 4;
    const int* a = lb.h_ids.data() + lb.coff[col];
    const int* e = lb.h_ids.data() + lb.coff[col + 1];
    const int lo = int(std::lower_bound(a, e, (g->plan.y0(r, l) / 4) * nbk) - lb.h_ids.data());
    const int hi = int(std::lower_bound(a, e, (g->plan.y1(r, l) / 4) * nbk) - lb.h_ids.data());
    return {lo, hi};
}

// In-process groups fuse the exchange into the colour passes: a pass kernel
// mirrors every write of its boundary rows (and of the next slab's seam row)
// into the neighbours' copies with peer stores (common.cuh Mirror), so a pass
// is followed only by an event barrier with the two neighbours.  NCCL groups
// (no peer pointers) snapshot the seam row and exchange after the pass.
bool fused_exchange(ibmg_group* g) { return !g->comm && g->plan.P > 1; }

Mirror mirror(ibmg_group* g, int r, int l) {
    if (!fused_exchange(g)) return Mirror{};
    const int P = g->plan.P;
    Mirror M;
    M.prv = lvec(g, (r + P - 1) % P, l, VW);
    M.nxt = lvec(g, (r + 1) % P, l, VW);
    M.y0 = g->plan.y0(r, l);
    M.y1 = g->plan.y1(r, l);
    return M;
}

// every slab's stream waits for its neighbours' work so far
void neighbour_barrier(ibmg_group* g) {
    const int P = g->plan.P;
    ++g->exchanges;
    each(g, [&](int r, ibmg_ctx* c) { CK(cudaEventRecord(pr(g, r).ea, c->s)); });
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaStreamWaitEvent(c->s, pr(g, (r + P - 1) % P).ea, 0));
        CK(cudaStreamWaitEvent(c->s, pr(g, (r + 1) % P).ea, 0));
    });
}

void before_pass(ibmg_group* g, int l) {
    if (!fused_exchange(g)) seam_snapshot(g, l);
}
void after_pass(ibmg_group* g, int l) {
    if (fused_exchange(g)) neighbour_barrier(g);
    else exchange(g, l, VW, true);
}

// one multicolour sweep of a distributed level: the single-GPU pass order
// (4 tile colours, then the big-block colours), each pass over the slab's own
// tiles / blocks, each followed by the exchange with the neighbour slabs
void sweep_group(ibmg_group* g, int l) {
    const int n = g->plan.n[l], half = (n / kTile) / 2;
    const int rows = n / g->plan.P;
    for (int tc = 0; tc < 4; ++tc) {
        before_pass(g, l);
        each(g, [&](int r, ibmg_ctx* c) {
            LevelBuf& lb = c->lev[l];
            plain_pass(c, lb, tc, lb.b, lb.w, g->plan.y0(r, l) / kTile, half * (rows / (2 * kTile)), mirror(g, r, l));
        });
        after_pass(g, l);
    }
    // every slab holds the same colouring (redundant setup), so the colour
    // count and the skip decision below are identical on all ranks
    const LevelBuf& l0 = g->c[0]->lev[l];
    for (int col = 0; col < l0.ncol; ++col) {
        if (l0.coff[col + 1] == l0.coff[col]) continue;
        before_pass(g, l);
        each(g, [&](int r, ibmg_ctx* c) {
            const std::pair<int, int> q = owned_blocks(g, r, l, col);
            if (q.second <= q.first) return;
            LevelBuf& lb = c->lev[l];
            BigColours BC{};
            BC.ncol = 1;
            BC.off[0] = q.first;
            BC.off[1] = q.second;
            const BigDeps DP{nullptr, nullptr, nullptr, 0u};
            const int grid = std::min(q.second - q.first, c->big_grid_max);
            if (c->prof) prof_begin(c, "k_big_phase");
            launch_k(c, k_big_phase, dim3(grid), dim3(kBigThreads), kBigSmem, true, lb.L, slabs(lb), BC, DP,
                     (const double*)lb.b, lb.w, mirror(g, r, l));
            if (c->prof) prof_end(c);
            ++c->launches;
        });
        after_pass(g, l);
    }
}

// coarse b (owned coarse rows) = R (b - A w) of distributed level l; coarse w = 0
void restrict_group(ibmg_group* g, int l) {
    each(g, [&](int r, ibmg_ctx* c) {
        LevelBuf& lb = c->lev[l];
        LevelBuf& nx = c->lev[l + 1];
        const int yc0 = g->plan.y0(r, l) / 2, yc1 = g->plan.y1(r, l) / 2;
        residual_restrict(c, l, lb.b, lb.w, nullptr, yc0, yc1, true);
        CK(cudaMemsetAsync(nx.w, 0, sizeof(double) * 3 * size_t(nx.L.nn), c->s));
    });
    if (l + 1 < g->plan.la) exchange(g, l + 1, VB, false);
    else allgather_level(g, l + 1, VB, l);
}

// out (owned rows of level 0) = A w, w valid on the owned rows + halo
void apply_owned(ibmg_group* g, int r, const double* w, double* out) {
    apply_rows(cx(g, r), 0, w, out, g->plan.y0(r, 0), g->plan.y1(r, 0), true);
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
        residual_restrict(c, l, lb.b, lb.w, nx.w, 0, nx.L.n, false);
    }
    coarse_cycle(c, c->lev[c->lc].b, c->lev[c->lc].w, c->lev[c->lc - 1].w);
    for (int l = c->lc - 1; l >= la; --l) {
        LevelBuf& lb = c->lev[l];
        if (l < c->lc - 1)
            LAUNCH(c, k_prolong_add, nblk(lb.L.nn), 256, 0, lb.L.n, (const double*)c->lev[l + 1].w, lb.w, 0, lb.L.nn);
        for (int s = 0; s < c->prm.nu2; ++s) sweep_level(c, l, lb.b, lb.w);
    }
}

// per-slab pointer lists (local slabs, indexed by rank)
struct Vecs {
    ibmg_group* g;
    std::vector<double*> v;
    double* operator[](int r) const { return v[size_t(r - g->r0)]; }
};
template <class Fn>
Vecs per_slab(ibmg_group* g, Fn&& fn) {
    Vecs V{g, {}};
    for (size_t i = 0; i < g->c.size(); ++i) V.v.push_back(fn(g->r0 + int(i)));
    return V;
}

// z (compact) = V(nu1, nu2)(0, b (compact)), no mean projection (as inside FGMRES)
void vcycle_group(ibmg_group* g, const Vecs& kb, const Vecs& kz) {
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

// dh[off] of every slab = global a . b (compact vectors of length len)
void gdot(ibmg_group* g, const Vecs& a, const Vecs& b, size_t len, int off) {
    each(g, [&](int r, ibmg_ctx* c) {
        LAUNCH(c, k_multidot_partial, dim3(kRedBlocks, 1), kRedThreads, 0, (const double*)a[r], len,
               (const double*)b[r], len, c->partial);
        LAUNCH(c, k_finish_dots, 1, 32, 0, (const double*)c->partial, kRedBlocks, c->dh + off, 0);
    });
    allreduce(g, off, 1);
}

// host copy of dh[off] of the first local slab (identical on every slab)
double read0(ibmg_group* g, int off) {
    ibmg_ctx* c = g->c[0];
    CK(cudaSetDevice(g->dev[0]));
    CK(cudaMemcpyAsync(c->hpin, c->dh + off, sizeof(double), cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return c->hpin[0];
}

// mean-zero pressure of the compact vectors x (project_pressure_mean, fields.cpp:78-85)
void pressure_mean_zero_group(ibmg_group* g, const Vecs& x) {
    const size_t cnt = size_t(g->rows) * g->prm.N, tot = size_t(g->prm.N) * g->prm.N;
    const int off = 2 * (g->prm.restart + 2);
    const Vecs p = per_slab(g, [&](int r) { return x[r] + 2 * cnt; });
    const Vecs ones = per_slab(g, [&](int r) { return cx(g, r)->ones; });
    gdot(g, p, ones, cnt, off);
    each(g, [&](int r, ibmg_ctx* c) {
        LAUNCH(c, k_sub_mean, nblk(cnt), 256, 0, p[r], cnt, tot, (const double*)c->dh + off);
    });
}

// r (compact) = b - A x (compact), returns ||r||^2 (global)
double true_residual(ibmg_group* g, const Vecs& x, const Vecs& b, const Vecs& res) {
    each(g, [&](int r, ibmg_ctx* c) { unpack(g, r, x[r], c->lev[0].w); });
    sync0(g, VW);
    each(g, [&](int r, ibmg_ctx* c) {
        apply_owned(g, r, c->lev[0].w, c->wv);
        pack(g, r, c->wv, res[r]);
        LAUNCH(c, k_b_minus, nblk(g->Mk), 256, 0, (const double*)b[r], res[r], g->Mk);
    });
    gdot(g, res, res, g->Mk, 0);
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
    const Vecs kb = per_slab(g, [&](int r) { return pr(g, r).kb; });
    const Vecs kx = per_slab(g, [&](int r) { return pr(g, r).kx; });
    const Vecs kr = per_slab(g, [&](int r) { return pr(g, r).kr; });
    const Vecs w = per_slab(g, [&](int r) { return cx(g, r)->stage_a; });
    each(g, [&](int r, ibmg_ctx* c) { CK(cudaMemsetAsync(kx[r], 0, sizeof(double) * Mk, c->s)); });
    gdot(g, kb, kb, Mk, hoff);
    const double bnorm = std::sqrt(read0(g, hoff));
    if (bnorm == 0.0) {
        st->converged = 1;
        return IBMG_OK;
    }
    const double tol = g->prm.rtol * bnorm;
    double beta = bnorm;
    const Vecs* rvec = &kb;
    int it = 0, restarts = 0;
    ibmg_ctx* c0 = g->c[0];
    while (true) {
        each(g, [&](int r, ibmg_ctx* c) {
            LAUNCH(c, k_scale_by_norm, nblk(Mk), 256, 0, (const double*)(*rvec)[r], c->V, Mk, (const double*)nullptr,
                   beta, (double*)nullptr);
        });
        std::fill(gv.begin(), gv.end(), 0.0);
        gv[0] = beta;
        int kdim = 0;
        for (int j = 0; j < m; ++j) {
            const Vecs Vj = per_slab(g, [&](int r) { return cx(g, r)->V + cx(g, r)->Mst * j; });
            const Vecs Zj = per_slab(g, [&](int r) { return cx(g, r)->Z + cx(g, r)->Mst * j; });
            vcycle_group(g, Vj, Zj);
            // w = A z_j from the V-cycle's level-0 w (owned rows + halo valid)
            each(g, [&](int r, ibmg_ctx* c) {
                apply_owned(g, r, c->lev[0].w, c->wv);
                pack(g, r, c->wv, w[r]);
            });
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
            CK(cudaStreamSynchronize(c->s));  // this slab's hpin is free
            std::copy(y.begin(), y.begin() + kdim, c->hpin);
            CK(cudaMemcpyAsync(c->dh + h2off, c->hpin, sizeof(double) * kdim, cudaMemcpyHostToDevice, c->s));
            LAUNCH(c, k_multi_axpy_add, nblk(Mk), 256, 0, (const double*)c->Z, c->Mst, kdim,
                   (const double*)(c->dh + h2off), kx[r], Mk);
        });
        beta = std::sqrt(true_residual(g, kx, kb, kr));
        rvec = &kr;
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

// FGMRES(m) over the slabs with the two-pass lagged CGS2 of fgmres2():
// per Arnoldi step every slab runs pass 1 on its rows and leaves the 2k raw sums in
// dh, one reduction over the slabs sums them, k_ortho_finish forms the coefficients
// (identically on every slab), pass 2 updates the slab's rows, and |w1|^2 is reduced:
// two passes over the basis and two small reductions per step, against three passes
// and three reductions in fgmres_group().  Host logic as fgmres2().
int fgmres_group2(ibmg_group* g, ibmg_stats* st) {
    const int m = g->prm.restart, ld = m + 2;
    const int SC = 5 * ld, RAW = 2 * ld, bslot = 6 * ld + 2;
    const size_t Mk = g->Mk;
    std::vector<double> Hx(size_t(m + 1) * m, 0.0), Ha(size_t(m + 1) * m, 0.0), cs(m), sn(m), gv(m + 1), y(m);
    st->iters = st->restarts = st->converged = 0;
    st->relres = 0.0;
    const Vecs kb = per_slab(g, [&](int r) { return pr(g, r).kb; });
    const Vecs kx = per_slab(g, [&](int r) { return pr(g, r).kx; });
    const Vecs kr = per_slab(g, [&](int r) { return pr(g, r).kr; });
    const Vecs w = per_slab(g, [&](int r) { return cx(g, r)->stage_a; });
    each(g, [&](int r, ibmg_ctx* c) { CK(cudaMemsetAsync(kx[r], 0, sizeof(double) * Mk, c->s)); });
    gdot(g, kb, kb, Mk, bslot);
    const double bnorm = std::sqrt(read0(g, bslot));
    if (bnorm == 0.0) {
        st->converged = 1;
        return IBMG_OK;
    }
    const double tol = g->prm.rtol * bnorm;
    double beta = bnorm;
    const Vecs* rvec = &kb;
    int it = 0, restarts = 0;
    ibmg_ctx* c0 = g->c[0];
    while (true) {
        each(g, [&](int r, ibmg_ctx* c) {
            LAUNCH(c, k_scale_by_norm, nblk(Mk), 256, 0, (const double*)(*rvec)[r], c->V, Mk, (const double*)nullptr,
                   beta, (double*)nullptr);
        });
        std::fill(gv.begin(), gv.end(), 0.0);
        std::fill(Hx.begin(), Hx.end(), 0.0);
        gv[0] = beta;
        int kdim = 0;
        double nu0 = 1.0;
        for (int j = 0; j < m; ++j) {
            const Vecs Vj = per_slab(g, [&](int r) { return cx(g, r)->V + cx(g, r)->Mst * j; });
            const Vecs Zj = per_slab(g, [&](int r) { return cx(g, r)->Z + cx(g, r)->Mst * j; });
            vcycle_group(g, Vj, Zj);
            each(g, [&](int r, ibmg_ctx* c) {
                apply_owned(g, r, c->lev[0].w, c->wv);
                pack(g, r, c->wv, w[r]);
                ortho_dots_raw(c, j + 1, w[r]);
            });
            allreduce(g, RAW, 2 * (j + 1));
            const bool more = j + 1 < m;
            each(g, [&](int r, ibmg_ctx* c) {
                LAUNCH(c, k_ortho_finish, 1, 64, 0, j + 1, c->dh, ld);
                ortho_update(c, j + 1, w[r], more ? c->V + c->Mst * (j + 1) : kr[r], nullptr);
            });
            allreduce(g, SC + 4, 1);
            CK(cudaSetDevice(g->dev[0]));
            CK(cudaMemcpyAsync(c0->hpin, c0->dh, sizeof(double) * (SC + 5), cudaMemcpyDeviceToHost, c0->s));
            CK(cudaEventRecord(c0->ev_dots, c0->s));
            CK(cudaEventSynchronize(c0->ev_dots));
            const double* hp = c0->hpin;
            const double nu = hp[SC + 2], h = hp[SC + 3], bnext = std::sqrt(hp[SC + 4]);
            if (j > 0 && !(nu > 0.0)) {  // breakdown: the space is invariant (fgmres2)
                for (int i = 0; i < j; ++i) Hx[size_t(i) * m + j - 1] += hp[ld + i];
                Hx[size_t(j) * m + j - 1] = 0.0;
                break;
            }
            if (j == 0) {
                nu0 = nu;
            } else {  // exact column j-1: q_j = sum a_i V_i + nu v_j
                for (int i = 0; i < j; ++i) Hx[size_t(i) * m + j - 1] += hp[ld + i];
                Hx[size_t(j) * m + j - 1] = nu;
            }
            for (int i = 0; i < j; ++i) Hx[size_t(i) * m + j] = hp[i];
            Hx[size_t(j) * m + j] = h;
            Hx[size_t(j + 1) * m + j] = bnext;
            for (int i = 0; i <= j + 1; ++i) Ha[size_t(i) * m + j] = Hx[size_t(i) * m + j];
            for (int i = 0; i < j; ++i) {
                const double a = Ha[size_t(i) * m + j], cc = Ha[size_t(i + 1) * m + j];
                Ha[size_t(i) * m + j] = cs[i] * a + sn[i] * cc;
                Ha[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * cc;
            }
            const double a = Ha[size_t(j) * m + j], cc = Ha[size_t(j + 1) * m + j];
            const double den = std::hypot(a, cc);
            cs[j] = a / den;
            sn[j] = cc / den;
            gv[j + 1] = -sn[j] * gv[j];
            gv[j] = cs[j] * gv[j];
            ++it;
            kdim = j + 1;
            if (!std::isfinite(gv[j + 1])) throw CudaError("FGMRES: non-finite residual estimate");
            if (std::fabs(gv[j + 1]) <= tol || it >= g->prm.max_iters || bnext == 0.0) break;
        }
        hessenberg_lsq(Hx, m, kdim, beta * nu0, y);  // r = beta q_0 = beta nu0 v_0
        each(g, [&](int r, ibmg_ctx* c) {
            CK(cudaStreamSynchronize(c->s));  // this slab's hpin is free
            std::copy(y.begin(), y.begin() + kdim, c->hpin);
            CK(cudaMemcpyAsync(c->dh + 4 * ld, c->hpin, sizeof(double) * kdim, cudaMemcpyHostToDevice, c->s));
            LAUNCH(c, k_multi_axpy_add, nblk(Mk), 256, 0, (const double*)c->Z, c->Mst, kdim,
                   (const double*)(c->dh + 4 * ld), kx[r], Mk);
        });
        beta = std::sqrt(true_residual(g, kx, kb, kr));
        rvec = &kr;
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

// the group's Krylov solver: two-pass lagged CGS2 unless IBMG_CGS2=1 (three sweeps)
int fgmres_slabs(ibmg_group* g, ibmg_stats* st) { return g->c[0]->ortho2 ? fgmres_group2(g, st) : fgmres_group(g, st); }

// host whole-grid vector (3 planes) -> each local slab's compact rows
void scatter_host(ibmg_group* g, const double* h, const Vecs& k) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    each(g, [&](int r, ibmg_ctx* c) {
        CK(cudaMemcpy2DAsync(k[r], w * sizeof(double), h + size_t(g->plan.y0(r, 0)) * N, nn * sizeof(double),
                             w * sizeof(double), 3, cudaMemcpyHostToDevice, c->s));
    });
}

// compact rows of every slab -> host whole-grid arrays (u: planes 0..1 or
// 0..2 at h; p plane at h_p when given).  NCCL group: the rows are first
// allgathered into each rank's whole-level buffer, so every rank returns the
// whole vector.
void gather_host(ibmg_group* g, const Vecs& k, double* h, int planes = 3, double* h_p = nullptr) {
    const size_t N = size_t(g->prm.N), nn = N * N, w = size_t(g->rows) * N;
    if (g->comm) {
        each(g, [&](int r, ibmg_ctx* c) { unpack(g, r, k[r], c->xv); });
        allgather_rows(g, g->prm.N, g->rows, [&](int r) { return cx(g, r)->xv; });
        each(g, [&](int, ibmg_ctx* c) {
            CK(cudaMemcpyAsync(h, c->xv, planes * nn * sizeof(double), cudaMemcpyDeviceToHost, c->s));
            if (h_p) CK(cudaMemcpyAsync(h_p, c->xv + 2 * nn, nn * sizeof(double), cudaMemcpyDeviceToHost, c->s));
            CK(cudaStreamSynchronize(c->s));
        });
        return;
    }
    each(g, [&](int r, ibmg_ctx* c) {
        const size_t o = size_t(g->plan.y0(r, 0)) * N;
        CK(cudaMemcpy2DAsync(h + o, nn * sizeof(double), k[r], w * sizeof(double), w * sizeof(double), planes,
                             cudaMemcpyDeviceToHost, c->s));
        if (h_p) CK(cudaMemcpyAsync(h_p + o, k[r] + 2 * w, w * sizeof(double), cudaMemcpyDeviceToHost, c->s));
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
        each(g, [&](int, ibmg_ctx* c) { CK(cudaStreamSynchronize(c->s)); });
        return rc;
    } catch (const std::invalid_argument& e) {
        return gfail(g, e, IBMG_INVALID);
    } catch (const NcclError& e) {
        return gfail(g, e, IBMG_NCCL);
    } catch (const std::exception& e) {
        return gfail(g, e, IBMG_CUDA);
    }
}

// the local slabs' contexts and scratch; peer access between distinct devices
void group_alloc(ibmg_group* g, const ibmg_params* p, int nlocal) {
    for (int i = 0; i < nlocal; ++i) {
        ibmg_params q = *p;
        q.device = g->dev[size_t(i)];
        ibmg_ctx* c = nullptr;
        const int rc = create_ctx(&q, g->rows, &c);
        if (rc != IBMG_OK) throw CudaError("slab context creation failed (status " + std::to_string(rc) + ")");
        for (int l = 0; l < g->plan.la; ++l) {  // box inverses of its own blocks only
            c->own_y0.push_back(g->plan.y0(g->r0 + i, l));
            c->own_y1.push_back(g->plan.y1(g->r0 + i, l));
        }
        g->c.push_back(c);
    }
    for (int i = 0; i < nlocal; ++i)
        for (int d = 0; d < nlocal; ++d)
            if (g->dev[size_t(i)] != g->dev[size_t(d)]) {
                CK(cudaSetDevice(g->dev[size_t(i)]));
                const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[size_t(d)], 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                cudaGetLastError();
            }
    g->Mk = g->c[0]->Mk;
    g->s.resize(size_t(nlocal));
    for (int i = 0; i < nlocal; ++i) {
        CK(cudaSetDevice(g->dev[size_t(i)]));
        auto& P = g->s[size_t(i)];
        P.kb = dalloc<double>(g->Mk);
        P.kx = dalloc<double>(g->Mk);
        P.kr = dalloc<double>(g->Mk);
        P.stash = dalloc<double>(2 * kStash);
        CK(cudaMemset(P.stash, 0, sizeof(double) * 2 * kStash));
        for (int l = 0; l < g->plan.la; ++l) {
            P.seam_in.push_back(dalloc<double>(size_t(g->plan.n[l])));
            P.seam_old.push_back(dalloc<double>(size_t(g->plan.n[l])));
        }
        CK(cudaEventCreateWithFlags(&P.ea, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P.eb, cudaEventDisableTiming));
    }
}

bool group_params_ok(const ibmg_params* p, int nslabs) {
    return p && nslabs >= 1 && nslabs <= kMaxSlabs && p->N >= 8 && !(p->N & (p->N - 1)) && p->N % nslabs == 0 &&
           p->restart >= 1 && p->restart + 1 <= kStash;
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
    for (size_t i = 0; i < g->c.size(); ++i) {
        cudaSetDevice(g->dev[i]);
        if (g->c[i]) cudaStreamSynchronize(g->c[i]->s);
        if (i < g->s.size()) {
            auto& P = g->s[i];
            dfree(P.kb);
            dfree(P.kx);
            dfree(P.kr);
            dfree(P.stash);
            for (auto& p : P.seam_in) dfree(p);
            for (auto& p : P.seam_old) dfree(p);
            if (P.ea) cudaEventDestroy(P.ea);
            if (P.eb) cudaEventDestroy(P.eb);
        }
        ibmg_destroy(g->c[i]);
    }
    if (g->comm) nccl_api()->CommDestroy(g->comm);
    delete g;
}

int ibmg_group_create(const ibmg_params* p, int nslabs, const int* devices, int min_rows, long min_cells,
                      ibmg_group** out) {
    if (!out) return IBMG_INVALID;
    *out = nullptr;
    if (!group_params_ok(p, nslabs)) return IBMG_INVALID;
    ibmg_group* g = new ibmg_group;
    g->prm = *p;
    g->plan = make_plan(p->N, p->coarsest_n, nslabs, min_rows, min_cells);
    g->rows = p->N / nslabs;
    for (int r = 0; r < nslabs; ++r) g->dev.push_back(devices ? devices[r] : p->device);
    try {
        group_alloc(g, p, nslabs);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ibmg_group_create: %s\n", e.what());
        ibmg_group_destroy(g);
        return IBMG_CUDA;
    }
    *out = g;
    return IBMG_OK;
}

int ibmg_nccl_unique_id(void* id_out) {
    if (!id_out) return IBMG_INVALID;
    const NcclApi* a = nccl_api();
    ncclUniqueId id;
    if (!a || a->GetUniqueId(&id) != ncclSuccess) return IBMG_NCCL;
    std::memcpy(id_out, &id, sizeof(id));
    return IBMG_OK;
}

int ibmg_group_create_nccl(const ibmg_params* p, int rank, int nranks, const void* nccl_id, int min_rows,
                           long min_cells, ibmg_group** out) {
    if (!out) return IBMG_INVALID;
    *out = nullptr;
    if (!group_params_ok(p, nranks) || !nccl_id || rank < 0 || rank >= nranks) return IBMG_INVALID;
    ibmg_group* g = new ibmg_group;
    g->prm = *p;
    g->plan = make_plan(p->N, p->coarsest_n, nranks, min_rows, min_cells);
    g->rows = p->N / nranks;
    g->r0 = rank;
    g->dev.push_back(p->device);
    try {
        group_alloc(g, p, 1);
        CK(cudaSetDevice(p->device));
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        NC(nccl().CommInitRank(&g->comm, nranks, id, rank));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ibmg_group_create_nccl: %s\n", e.what());
        ibmg_group_destroy(g);
        return IBMG_NCCL;
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
        const size_t n = size_t(g->plan.n[level]), nn = n * n, m = 3 * nn;
        each(g, [&](int, ibmg_ctx* c) {
            CK(cudaMemcpyAsync(c->lev[level].b, b, m * sizeof(double), cudaMemcpyHostToDevice, c->s));
            CK(cudaMemcpyAsync(c->lev[level].w, w, m * sizeof(double), cudaMemcpyHostToDevice, c->s));
        });
        sweep_group(g, level);
        if (g->comm) {  // every rank returns the whole level
            allgather_level(g, level, VW, level);
            each(g, [&](int, ibmg_ctx* c) {
                CK(cudaMemcpyAsync(w, c->lev[level].w, m * sizeof(double), cudaMemcpyDeviceToHost, c->s));
            });
            return IBMG_OK;
        }
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
        const Vecs kb = per_slab(g, [&](int r) { return pr(g, r).kb; });
        const Vecs kx = per_slab(g, [&](int r) { return pr(g, r).kx; });
        scatter_host(g, b, kb);
        vcycle_group(g, kb, kx);
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
        scatter_host(g, b, per_slab(g, [&](int r) { return pr(g, r).kb; }));
        const int rc = fgmres_slabs(g, st);
        gather_host(g, per_slab(g, [&](int r) { return pr(g, r).kx; }), x);
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
            pack(g, r, c->bv, pr(g, r).kb);
        });
        each(g, [&](int, ibmg_ctx* c) { CK(cudaStreamSynchronize(c->s)); });
        const double t1 = now_ms();
        const int rc = fgmres_slabs(g, st);
        gather_host(g, per_slab(g, [&](int r) { return pr(g, r).kx; }), u, 2, p);
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
