// cluster_kernel.cuh — the bottom of the V-cycle (every level with n <= 128)
// in ONE thread-block cluster of 16 CTAs, its level data resident in
// distributed shared memory (DSMEM).  Replaces, for those levels, the
// per-sweep dataflow launches (k_sweep_df, whose colour handoffs go through
// L2 flags at ~1-2 us each), the residual/restriction and prolongation
// launches between them, and the single-CTA coarse kernel (k_coarse_cycle):
// a colour handoff here is one cluster barrier (~0.2 us) and the neighbours'
// data is one DSMEM load away.  Algorithm 1 on the same
// schedule as the oracle (DESIGN.md §3 D12; oracle build_schedule):
//
// * "P-levels" (n >= 64, partitioned): CTA r = rx + 4 ry owns the cells
//   [rx n/4, (rx+1) n/4) x [ry n/4, (ry+1) n/4) of w and b.  Plain phase: the
//   16x16 tiles in their 2x2 tile colours, one colour per cluster step; a
//   tile is staged (local + DSMEM) into one warp's shared buffers, relaxed by
//   the 8 conflict-free cell colours (i + 2j) mod 8 (plain_cell, the same
//   arithmetic as k_sweep_df) and written back to the owners.  Big phase: the
//   big 4x4 blocks in colour order, spread over the cluster's 32 groups of
//   128 threads, stencil and E' columns read through the distributed view.
// * "Q-levels" (n <= 32, replicated): every CTA holds the whole level and runs
//   the plain phase redundantly (identical arithmetic in every copy); the big
//   blocks of a colour are spread over the 32 groups of the cluster and each
//   correction is stored into all 16 copies.  The E' rows of the residual are
//   spread over the cluster likewise; the coarsest bordered solve is
//   redundant.
//
// Every phase that reads what another CTA wrote is preceded by a cluster
// barrier (barrier.cluster.arrive.release / wait.acquire).  Same-colour tiles
// and blocks never touch each other's DOFs (the colouring), so the stores of
// one phase never race.
#pragma once
#include "coarse_kernel.cuh"

namespace ibmg {

constexpr int kClCX = 4, kClCY = 4, kCl = kClCX * kClCY;  // cluster = 4 x 4 regions
constexpr int kClThreads = 256;
constexpr int kClWarps = kClThreads / 32;
constexpr int kClGroups = kClThreads / kGroup;  // big-block groups of 128 threads per CTA
constexpr int kClMaxN = 128;                    // finest level the cluster holds
constexpr int kClMaxLev = 6;                    // 128 .. 4
constexpr int kClMaxColours = 32;               // = ibmg.cu kMaxColours

__device__ __forceinline__ unsigned cl_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// debug timeline (ibmg_debug_cluster_trace): CTA 0 thread 0 stamps
// (globaltimer, tag) after each cluster barrier; cl_tr == nullptr in production
__shared__ unsigned long long* cl_tr;
__shared__ int cl_nm;
__device__ __forceinline__ void cl_mark(int tag) {
    if (cl_tr && threadIdx.x == 0) {
        if (cl_nm < 2000) {
            cl_tr[2 * cl_nm] = gtimer();
            cl_tr[2 * cl_nm + 1] = (unsigned long long)tag;
        }
        ++cl_nm;
    }
}
// tag: level * 10000 + phase * 100 + index (see tools/trace_cluster.py)
__device__ __forceinline__ void cl_sync(int tag = 0) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (tag) cl_mark(tag);
}
// generic address of the same shared-memory location in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ T* cl_map(T* p, unsigned rank) {
    unsigned long long a;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(a) : "l"(p), "r"(rank));
    return reinterpret_cast<T*>(a);
}

// One field (w, b or a residual) of a level in cluster shared memory.
// part = 1: partitioned (this CTA holds its region, region-local layout
// f Rx Ry + (i mod Rx) + (j mod Ry) Rx); part = 0: replicated (full level,
// f nn + i + j n in every CTA).  The same offset holds the same field in every
// CTA (identical layouts), so a remote element is mapa of the local address.
struct DView {
    double* loc;
    int n, nn, lg;
    int part, Rx, Ry, lgRx, lgRy;
    unsigned me;
    __device__ __forceinline__ unsigned owner(int i, int j) const { return (i >> lgRx) + kClCX * (j >> lgRy); }
    __device__ __forceinline__ int loff(int f, int i, int j) const {  // i, j wrapped
        return part ? f * (Rx * Ry) + (i & (Rx - 1)) + (j & (Ry - 1)) * Rx : f * nn + i + j * n;
    }
    __device__ __forceinline__ double get(int f, int i, int j) const {  // wrapped coordinates
        const int k = loff(f, i, j);
        if (!part) return in_smem(loc)[k];
        // one generic load through mapa, local or remote (no divergent branch:
        // a warp's loads issue back to back)
        return *cl_map(loc + k, owner(i, j));
    }
    __device__ __forceinline__ double operator()(int f, int i, int j) const { return get(f, wr(i, n), wr(j, n)); }
    __device__ __forceinline__ double operator[](int flat) const {  // flat = f nn + i + j n
        const int f = flat >> (2 * lg), rem = flat & (nn - 1);
        return get(f, rem & (n - 1), rem >> lg);
    }
    // P: store to the owner; Q: store to every copy (the whole cluster)
    __device__ __forceinline__ void put(int f, int i, int j, double v) const {  // wrapped coordinates
        const int k = loff(f, i, j);
        if (part) {
            const unsigned o = owner(i, j);
            if (o == me) in_smem(loc)[k] = v;
            else *cl_map(loc + k, o) = v;
        } else {
#pragma unroll 4
            for (unsigned r = 0; r < (unsigned)kCl; ++r) *cl_map(loc + k, r) = v;
        }
    }
};

// One level of the cluster kernel (host-built, ibmg.cu cluster_args).
struct ClLev {
    Lev L;
    FaceList FL;
    EMat E;
    Slabs SL;
    const uint8_t* big;
    int nbig, ncol, part, Rx, Ry, lgRx, lgRy;
    int coff[kClMaxColours + 1];
    int w_off, b_off;  // shared-memory offsets (doubles) of w and b (this CTA's part or copy)
};

struct ClArgs {
    int nl, nu1, nu2;
    ClLev lv[kClMaxLev];
    const double* Acoarse;  // bordered inverse of the coarsest level, col-major (3nn+1)^2
    const double* b_in;     // b of the first cluster level (global)
    double* w_out;          // its correction (global)
    double* w_fine;         // optional: w of the next finer level += P w_out
    int u_off;              // union region (doubles): 2 E' slots | tile buffers, residual, E' dots
    unsigned long long* trace;  // debug timeline (nullptr in production)
};

// union region layout (doubles)
constexpr int kClSlotD = int(sizeof(ESlot) / sizeof(double));
constexpr int kClTileW = 3 * kRegP, kClTileB = 3 * 289;
constexpr int kClTileD = (kClTileW + kClTileB + 1) / 2 * 2;
constexpr int kClResD = 3 * 32 * 32;   // a P-level region residual (Rx Ry <= 1024 cells) or a replicated n = 32 level
constexpr int kClEDots = 2 * 32 * 32;  // E' row dots of a replicated level (faces <= 2 nn)
constexpr int kClUnionD = (kClGroups * kClSlotD > kClTileD + kClResD + kClEDots) ? kClGroups * kClSlotD
                                                                                    : kClTileD + kClResD + kClEDots;

__device__ __forceinline__ DView cl_view(const ClLev& C, double* base, int off, unsigned me) {
    return DView{base + off, C.L.n, C.L.nn, C.L.lg, C.part, C.Rx, C.Ry, C.lgRx, C.lgRy, me};
}

// ---- plain phase of a P-level: the tile colours in order, one cluster step each
__device__ void cl_plain_p(const ClLev& C, const DView& W, const DView& B, double* un, unsigned me) {
    const Lev& L = C.L;
    const int n = L.n, nbk = n >> 2, t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int rx = me % kClCX, ry = me / kClCX, X0 = rx * C.Rx, Y0 = ry * C.Ry;
    const int ntx = C.Rx / kTile, nty = C.Ry / kTile;
    double* sw = in_smem(un);
    double* sb = in_smem(un + kClTileW);
    for (int tc = 0; tc < 4; ++tc) {
        // this region's tiles of colour tc (tile colour (tx & 1) + 2 (ty & 1))
        for (int ty = 0; ty < nty; ++ty)
            for (int tx = 0; tx < ntx; ++tx) {
                const int gx = X0 / kTile + tx, gy = Y0 / kTile + ty;
                if ((gx & 1) + 2 * (gy & 1) != tc) continue;
                const int x0 = gx * kTile, y0 = gy * kTile;
                // stage the w region (2-cell halo) and the b region: local or
                // DSMEM; every thread's loads are issued before its stores
                constexpr int NW = (3 * kReg * kReg + kClThreads - 1) / kClThreads;
                constexpr int NB = (3 * 289 + kClThreads - 1) / kClThreads;
                double vw[NW], vb[NB];
#pragma unroll
                for (int u = 0; u < NW; ++u) {
                    const int q = t + u * kClThreads;
                    const int f = q / (kReg * kReg), rem = q - f * kReg * kReg, bb = rem / kReg, a = rem - bb * kReg;
                    vw[u] = q < 3 * kReg * kReg ? W.get(f, wr(x0 - 2 + a, n), wr(y0 - 2 + bb, n)) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const int q = t + u * kClThreads;
                    const int f = q / 289, rem = q - f * 289, bb = rem / 17, a = rem - bb * 17;
                    vb[u] = q < 3 * 289 ? B.get(f, wr(x0 + a, n), wr(y0 + bb, n)) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < NW; ++u) {
                    const int q = t + u * kClThreads;
                    const int f = q / (kReg * kReg), rem = q - f * kReg * kReg, bb = rem / kReg, a = rem - bb * kReg;
                    if (q < 3 * kReg * kReg) sw[f * kRegP + bb * kRegS + a] = vw[u];
                }
#pragma unroll
                for (int u = 0; u < NB; ++u) {
                    const int q = t + u * kClThreads;
                    if (q < 3 * 289) sb[q] = vb[u];
                }
                __syncthreads();
                if (wid == 0) {  // the 8 conflict-free colours on the staged tile (as df_plain_tile)
                    const bool isbig = lane < 16 && C.big[(x0 >> 2) + (lane & 3) + ((y0 >> 2) + (lane >> 2)) * nbk];
                    const unsigned bigmask = __ballot_sync(0xffffffffu, isbig);
                    TileW Wt{sw};
                    TileB Bt{sb};
                    for (int pc = 0; pc < 8; ++pc) {
                        const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
                        if (!((bigmask >> ((li >> 2) + 4 * (lj >> 2))) & 1)) plain_cell(L, Wt, Bt, li, lj);
                        __syncwarp();
                    }
                }
                __syncthreads();
                // write set: u faces i in [x0, x0+16], v faces j in [y0, y0+16], p cells
                TileW Wt{sw};
                for (int q = t; q < 17 * 17; q += kClThreads) {
                    const int a = q % 17, bb = q / 17, i = wr(x0 + a, n), j = wr(y0 + bb, n);
                    if (bb < 16) W.put(0, i, j, Wt(0, a, bb));
                    if (a < 16) W.put(1, i, j, Wt(1, a, bb));
                    if (a < 16 && bb < 16) W.put(2, i, j, Wt(2, a, bb));
                }
                __syncthreads();
            }
        cl_sync(C.L.lg * 10000 + 100 + tc);
    }
}

// ---- plain phase of a Q-level: the whole level in the 8 colours (i + 2j) mod 8
// (oracle build_schedule: one tile when n <= 32), redundantly in every CTA
__device__ void cl_plain_q(const ClLev& C, double* w, const double* b) {
    const Lev& L = C.L;
    const int n = L.n, nbk = n >> 2, t = threadIdx.x;
    SW W{in_smem(w), n, L.nn};
    SW Bq{const_cast<double*>(in_smem(b)), n, L.nn};
    const int per = L.nn >> 3, row = n >> 3;
    for (int pc = 0; pc < 8; ++pc) {
        for (int idx = t; idx < per; idx += kClThreads) {
            const int j = idx / row, i = ((pc - 2 * j) & 7) + 8 * (idx % row);
            if (!C.big[(i >> 2) + (j >> 2) * nbk]) plain_cell(L, W, Bq, i, j);
        }
        __syncthreads();
    }
}

// ---- big phase (P or Q): colour classes in order, one cluster step each.
// Block k of a colour goes to group k mod 32 of the cluster.  A group's next
// block (in the same or a later colour) has its E' rows refilled into the
// group's slot as soon as the current block's rows are consumed, and its
// inverse loaded into registers right after the current block's matvec.
__device__ void cl_big(const ClLev& C, const DView& W, const DView& B, double* un, BigScratch* S, unsigned me) {
    if (C.nbig == 0) return;
    const Lev& L = C.L;
    const int t = threadIdx.x, g = t / kGroup, gt = t % kGroup, nbk = L.n >> 2;
    ESlot* slot = reinterpret_cast<ESlot*>(in_smem(un)) + g;
    const int gid = int(me) * kClGroups + g;  // Q: this group's rank in the cluster
    // k-th item of this group in colour c (or -1): a list position.  Block m of
    // a colour goes to group m mod 32 of the cluster (P-levels too: DSMEM
    // makes every region reachable, and owner-computes left most groups idle
    // where the structure crosses few regions)
    auto item = [&](int c, int k) -> int {
        const int q = C.coff[c] + gid + kCl * kClGroups * k;
        return q < C.coff[c + 1] ? q : -1;
    };
    // this group's enumeration: (colour, k) -> the next item
    auto advance = [&](int& c, int& k, int& q) {
        ++k;
        q = item(c, k);
        while (q < 0 && ++c < C.ncol) {
            k = 0;
            q = item(c, 0);
        }
    };
    int c = 0, k = -1, q = -1;
    advance(c, k, q);
    double av[28];  // this thread's part of the group's next inverse, loaded a block ahead
    if (c < C.ncol) {
        eslot_issue(*slot, C.SL, q, gt, kGroup);
        load_inverse_part(av, C.SL.Ainv + (size_t)q * 3136, gt);
    }
    cp_async_commit();
    auto gsync = [g] { asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kGroup)); };
    for (int colour = 0; colour < C.ncol; ++colour) {
        while (c == colour) {
            int nc = c, nk = k, nq = q;
            advance(nc, nk, nq);
            cp_async_wait<0>();
            gsync();
            const int Bk = slot->rp[47];
            big_block_es<0>(L, *slot, nullptr, 4 * (Bk % nbk), 4 * (Bk / nbk), W, W, B,
                            [&](int f, int i, int j, double old, double d) { W.put(f, i, j, old + d); }, S[g], gt,
                            gsync,
                            [&] {
                                if (nc < C.ncol) eslot_issue(*slot, C.SL, nq, gt, kGroup);
                                cp_async_commit();
                            },
                            av, nc < C.ncol ? C.SL.Ainv + (size_t)nq * 3136 : nullptr, SlabTail{&C.SL, q});
            gsync();
            c = nc;
            k = nk;
            q = nq;
        }
        cl_sync(C.L.lg * 10000 + 300 + colour);
    }
    cp_async_wait<0>();
}

__device__ __forceinline__ void cl_sweep(const ClLev& C, double* sm, double* un, BigScratch* S, unsigned me) {
    const DView W = cl_view(C, sm, C.w_off, me), B = cl_view(C, sm, C.b_off, me);
    if (C.part) {
        cl_plain_p(C, W, B, un, me);
    } else {
        cl_plain_q(C, sm + C.w_off, sm + C.b_off);
        cl_sync(C.L.lg * 10000 + 200);  // every copy's plain phase reads the pre-big-phase values
    }
    cl_big(C, W, B, un, S, me);
}

// Fine residual r = b - A w of level C (stencil, then + E' w from the assembled
// rows, elasticity.cpp:88-107 / the coarse kernel's order), then coarse
// b = R r (transfers.cpp:107-134) into level D, coarse w = 0.
__device__ void cl_restrict(const ClLev& C, const ClLev& D, double* sm, double* un, unsigned me) {
    const Lev& L = C.L;
    const int n = L.n, nn = L.nn, t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const DView W = cl_view(C, sm, C.w_off, me), B = cl_view(C, sm, C.b_off, me);
    double* rs = in_smem(un + kClTileD);
    DView R = W;
    R.loc = rs;
    if (C.part) {
        const int rx = me % kClCX, ry = me / kClCX, X0 = rx * C.Rx, Y0 = ry * C.Ry, RR = C.Rx * C.Ry;
        for (int q = t; q < RR; q += kClThreads) {
            const int i = X0 + (q & (C.Rx - 1)), j = Y0 + (q >> C.lgRx);
            double ru, rv, rp;
            stokes_rows(L, W, i, j, ru, rv, rp);
            rs[q] = B.get(0, i, j) - ru;
            rs[RR + q] = B.get(1, i, j) - rv;
            rs[2 * RR + q] = B.get(2, i, j) - rp;
        }
        __syncthreads();
        // E' rows of the faces this CTA owns: a warp reads 32 faces at once,
        // ballots the owned ones and sums each of their rows (lanes over the
        // entries, fixed-order xor tree)
        for (int base = wid * 32; base < C.FL.nf; base += kClWarps * 32) {
            const int fq = base + lane;
            const int face = fq < C.FL.nf ? __ldg(C.FL.face + fq) : 0, rem = face & (nn - 1);
            const bool mine = fq < C.FL.nf && W.owner(rem & (n - 1), rem >> L.lg) == me;
            unsigned m = __ballot_sync(0xffffffffu, mine);
            while (m) {
                const int bl = __ffs(m) - 1;
                m &= m - 1;
                const int fr = base + bl, fc = __shfl_sync(0xffffffffu, face, bl);
                const int f = fc >> (2 * L.lg), rr = fc & (nn - 1);
                double s = 0.0;
                for (int e = __ldg(C.E.rp + fr) + lane; e < __ldg(C.E.rp + fr + 1); e += 32)
                    s += __ldg(C.E.val + e) * W[__ldg(C.E.col + e)];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) rs[R.loff(f, rr & (n - 1), rr >> L.lg)] += s;
            }
        }
        cl_sync(C.L.lg * 10000 + 400);  // every region's residual is complete
    } else {
        double* ed = in_smem(un + kClTileD + kClResD);
        SW Wl{in_smem(sm + C.w_off), n, nn};
        const double* bl = in_smem(sm + C.b_off);
        for (int q = t; q < nn; q += kClThreads) {
            double ru, rv, rp;
            stokes_rows(L, Wl, q & (n - 1), q >> L.lg, ru, rv, rp);
            rs[q] = bl[q] - ru;
            rs[nn + q] = bl[nn + q] - rv;
            rs[2 * nn + q] = bl[2 * nn + q] - rp;
        }
        // E' row dots spread over the cluster's warps, each stored into every copy
        for (int fq = int(me) * kClWarps + wid; fq < C.FL.nf; fq += kCl * kClWarps) {
            double s = 0.0;
            for (int e = __ldg(C.E.rp + fq) + lane; e < __ldg(C.E.rp + fq + 1); e += 32)
                s += __ldg(C.E.val + e) * Wl.s[__ldg(C.E.col + e)];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane < kCl) *cl_map(ed + fq, lane) = s;
        }
        cl_sync(C.L.lg * 10000 + 500);  // every copy holds every row's dot
        for (int fq = t; fq < C.FL.nf; fq += kClThreads) rs[__ldg(C.FL.face + fq)] += ed[fq];
        __syncthreads();
        R.part = 0;
    }
    // coarse b = R r, coarse w = 0 (D's cells of this CTA: its region, or all)
    const Lev& Lc = D.L;
    const int nc = Lc.n, nnc = Lc.nn;
    const DView Bc = cl_view(D, sm, D.b_off, me);
    double* wc = in_smem(sm + D.w_off);
    const int cells = D.part ? D.Rx * D.Ry : (C.part ? nnc / kCl : nnc);
    const int cx0 = D.part ? (me % kClCX) * D.Rx : 0, cy0 = D.part ? (me / kClCX) * D.Ry : 0;
    for (int q = t; q < cells; q += kClThreads) {
        int I, J;
        if (D.part) {
            I = cx0 + (q & (D.Rx - 1));
            J = cy0 + (q >> D.lgRx);
        } else {
            const int qq = C.part ? int(me) * cells + q : q;  // P -> Q: a slice per CTA, broadcast
            I = qq & (nc - 1);
            J = qq >> Lc.lg;
        }
        const int i = 2 * I, j = 2 * J;
        const double bu = 0.125 * (R(0, i - 1, j) + 2.0 * R(0, i, j) + R(0, i + 1, j) + R(0, i - 1, j + 1) +
                                   2.0 * R(0, i, j + 1) + R(0, i + 1, j + 1));
        const double bv = 0.125 * (R(1, i, j - 1) + 2.0 * R(1, i, j) + R(1, i, j + 1) + R(1, i + 1, j - 1) +
                                   2.0 * R(1, i + 1, j) + R(1, i + 1, j + 1));
        const double bp = 0.25 * (R(2, i, j) + R(2, i + 1, j) + R(2, i, j + 1) + R(2, i + 1, j + 1));
        if (!D.part && !C.part) {  // Q -> Q: redundant, this copy only
            double* bl = in_smem(sm + D.b_off);
            bl[I + J * nc] = bu;
            bl[nnc + I + J * nc] = bv;
            bl[2 * nnc + I + J * nc] = bp;
        } else {  // P -> P: an owned cell (local store); P -> Q: this CTA's slice, into every copy
            Bc.put(0, I, J, bu);
            Bc.put(1, I, J, bv);
            Bc.put(2, I, J, bp);
        }
    }
    const int wcount = 3 * (D.part ? D.Rx * D.Ry : nnc);
    for (int q = t; q < wcount; q += kClThreads) wc[q] = 0.0;
    cl_sync(C.L.lg * 10000 + 600);  // the coarse level is complete everywhere
}

// Level C += P (level D's w) on C's cells of this CTA (its region, or all).
__device__ void cl_prolong(const ClLev& C, const ClLev& D, double* sm, unsigned me) {
    const int n = C.L.n, t = threadIdx.x;
    const DView Ec = cl_view(D, sm, D.w_off, me);
    double* w = in_smem(sm + C.w_off);
    if (C.part) {
        const int X0 = (me % kClCX) * C.Rx, Y0 = (me / kClCX) * C.Ry, RR = C.Rx * C.Ry;
        for (int q = t; q < RR; q += kClThreads) {
            const int i = X0 + (q & (C.Rx - 1)), j = Y0 + (q >> C.lgRx);
            double du, dv, dp;
            prolong_rows(n, Ec, i, j, du, dv, dp);
            w[q] += du;
            w[RR + q] += dv;
            w[2 * RR + q] += dp;
        }
    } else {
        const int nn = C.L.nn;
        for (int q = t; q < nn; q += kClThreads) {
            double du, dv, dp;
            prolong_rows(n, Ec, q & (n - 1), q >> C.L.lg, du, dv, dp);
            w[q] += du;
            w[nn + q] += dv;
            w[2 * nn + q] += dp;
        }
    }
    if (C.part) cl_sync(C.L.lg * 10000 + 700);  // the next sweep stages neighbours' regions
    else __syncthreads();
}

__global__ void __launch_bounds__(kClThreads, 1) k_cluster_cycle(ClArgs A) {
    pdl_enter();
    extern __shared__ __align__(16) double csm[];
    __shared__ BigScratch S[kClGroups];
    const unsigned me = cl_rank();
    if (threadIdx.x == 0) {
        cl_tr = me == 0 ? A.trace : nullptr;
        cl_nm = 0;
    }
    __syncthreads();
    cl_mark(1);
    double* sm = csm;
    double* un = csm + A.u_off;
    const int t = threadIdx.x;
    // entry: b of the first level (global) into this CTA's part, w = 0
    {
        const ClLev& C = A.lv[0];
        const DView B = cl_view(C, sm, C.b_off, me);
        double* w = in_smem(sm + C.w_off);
        const int n = C.L.n, nn = C.L.nn;
        if (C.part) {
            const int X0 = (me % kClCX) * C.Rx, Y0 = (me / kClCX) * C.Ry, RR = C.Rx * C.Ry;
            for (int q = t; q < 3 * RR; q += kClThreads) {
                const int f = q / RR, r = q - f * RR, i = X0 + (r & (C.Rx - 1)), j = Y0 + (r >> C.lgRx);
                in_smem(B.loc)[q] = A.b_in[(size_t)f * nn + i + (size_t)j * n];
                w[q] = 0.0;
            }
        } else {
            for (int q = t; q < 3 * nn; q += kClThreads) {
                in_smem(B.loc)[q] = A.b_in[q];
                w[q] = 0.0;
            }
        }
        cl_sync(800);
    }
    for (int l = 0; l + 1 < A.nl; ++l) {
        for (int s = 0; s < A.nu1; ++s) cl_sweep(A.lv[l], sm, un, S, me);
        cl_restrict(A.lv[l], A.lv[l + 1], sm, un, me);
    }
    {  // coarsest: bordered inverse (mean-zero pressure), redundantly in every CTA
        const ClLev& C = A.lv[A.nl - 1];
        const int nn = C.L.nn, m = 3 * nn + 1;
        const double* b = in_smem(sm + C.b_off);
        double* w = in_smem(sm + C.w_off);
        for (int q = t; q < 3 * nn; q += kClThreads) {
            double s = 0.0;
            for (int cc = 0; cc < 3 * nn; ++cc) s += __ldg(A.Acoarse + (size_t)cc * m + q) * b[cc];
            w[q] = s;
        }
        __syncthreads();
        cl_mark(1000);
    }
    for (int l = A.nl - 2; l >= 0; --l) {
        cl_prolong(A.lv[l], A.lv[l + 1], sm, me);
        for (int s = 0; s < A.nu2; ++s) cl_sweep(A.lv[l], sm, un, S, me);
    }
    // exit: w of the first level to global (owned cells / CTA 0), then the
    // prolongation-add into the next finer level (spread over the cluster)
    const ClLev& C = A.lv[0];
    const int n = C.L.n, nn = C.L.nn;
    const DView W = cl_view(C, sm, C.w_off, me);
    if (C.part) {
        const int X0 = (me % kClCX) * C.Rx, Y0 = (me / kClCX) * C.Ry, RR = C.Rx * C.Ry;
        for (int q = t; q < 3 * RR; q += kClThreads) {
            const int f = q / RR, r = q - f * RR, i = X0 + (r & (C.Rx - 1)), j = Y0 + (r >> C.lgRx);
            A.w_out[(size_t)f * nn + i + (size_t)j * n] = in_smem(W.loc)[q];
        }
    } else if (me == 0) {
        for (int q = t; q < 3 * nn; q += kClThreads) A.w_out[q] = in_smem(W.loc)[q];
    }
    if (A.w_fine) {
        const int nf = 2 * n, nnf = nf * nf;
        for (int q = int(me) * kClThreads + t; q < nnf; q += kCl * kClThreads) {
            double du, dv, dp;
            prolong_rows(nf, W, q & (nf - 1), q / nf, du, dv, dp);
            A.w_fine[q] += du;
            A.w_fine[nnf + q] += dv;
            A.w_fine[2 * nnf + q] += dp;
        }
    }
    cl_sync(900);  // no CTA exits while others may still read its shared memory
}

}  // namespace ibmg
