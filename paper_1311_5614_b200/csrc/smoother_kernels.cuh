// smoother_kernels.cuh — multicolour box relaxation (the paper's generalised
// Vanka / big-box smoother) and the coarse-level kernels.
//
// Schedule (mirrored exactly by oracle/ibmg_oracle.cpp
// build_schedule): plain phase = 16x16-cell tiles coloured 2x2 (one launch per
// tile colour, one warp per tile, the 8 conflict-free colours (i+2j) mod 8 run
// in shared memory); big phase = big 4x4 blocks in 16 level-wide colours
// (bx mod 4, by mod 4), one CTA per block, dense 56x56 inverse applied.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>

#include "common.cuh"
#include "grid_kernels.cuh"

namespace cg = cooperative_groups;

namespace ibmg {

// Exact 5x5 Vanka solve of one plain cell (§5 "5-by-5 system") in
// closed form for the constant-coefficient periodic stencil, then the
// immediate correction (multiplicative sweep).
template <class WA, class BA>
__device__ __forceinline__ void plain_cell(const Lev& L, WA& W, const BA& B, int i, int j) {
    const double d = L.d, c = L.c, g = L.g;
    const double uW = W(0, i, j), uE = W(0, i + 1, j), vS = W(1, i, j), vN = W(1, i, j + 1), pC = W(2, i, j);
    const double r_uW =
        B(0, i, j) - (d * uW - c * (W(0, i - 1, j) + uE + W(0, i, j - 1) + W(0, i, j + 1)) + g * (pC - W(2, i - 1, j)));
    const double r_uE = B(0, i + 1, j) -
                        (d * uE - c * (uW + W(0, i + 2, j) + W(0, i + 1, j - 1) + W(0, i + 1, j + 1)) +
                         g * (W(2, i + 1, j) - pC));
    const double r_vS =
        B(1, i, j) - (d * vS - c * (W(1, i, j - 1) + vN + W(1, i - 1, j) + W(1, i + 1, j)) + g * (pC - W(2, i, j - 1)));
    const double r_vN = B(1, i, j + 1) -
                        (d * vN - c * (vS + W(1, i, j + 2) + W(1, i - 1, j + 1) + W(1, i + 1, j + 1)) +
                         g * (W(2, i, j + 1) - pC));
    const double r_p = B(2, i, j) - (-g * (uE - uW) - g * (vN - vS));
    const double dp = ((r_uW - r_uE + r_vS - r_vN) - L.dpc_g * r_p) * L.i4g;
    const double s = (r_uW - r_uE - 2.0 * g * dp) * L.idpc;
    const double t = (r_vS - r_vN - 2.0 * g * dp) * L.idpc;
    const double a = (r_uW + r_uE) * L.idmc, e = (r_vS + r_vN) * L.idmc;
    W(0, i, j) = uW + 0.5 * (a + s);
    W(0, i + 1, j) = uE + 0.5 * (a - s);
    W(1, i, j) = vS + 0.5 * (e + t);
    W(1, i, j + 1) = vN + 0.5 * (e - t);
    W(2, i, j) = pC + dp;
}

// Asynchronous global->shared copies (LDGSTS): the whole tile is in flight at
// once instead of one load round trip per loop iteration.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- plain phase, multi-tile levels (n >= 32): one warp per 16x16 tile.
constexpr int kTile = 16, kReg = kTile + 4;  // region with a 2-cell halo
// Row stride of the staged w region.  An odd stride would halve the shared-
// memory wavefronts of the passes (the 32 cells of a colour pass all have
// one word parity at an even stride: 4 wavefronts per fp64 access instead of
// 2), but needs 8-byte staging copies; measured on B200 that is slower
// (C4 plain phase 123 -> 160 ms, C2 step 7.77 -> 8.02 ms), so rows stay
// 16-byte aligned.
#ifndef IBMG_REG_STRIDE
#define IBMG_REG_STRIDE 20
#endif
constexpr int kRegS = IBMG_REG_STRIDE, kRegP = kReg * kRegS;  // (odd: 8-byte staging, 2-way passes)

struct TileW {
    double* s;  // [3][kReg][kRegS], local coords li, lj in [-2, 18)
    __device__ __forceinline__ double& operator()(int f, int i, int j) const {
        return s[f * kRegP + (j + 2) * kRegS + (i + 2)];
    }
};
// Optional working layout of the dataflow tiles (df_plain_tile, compile with
// -DIBMG_RELAYOUT=1): the region is staged with 16-byte copies / tensor copies at the
// even row stride kRegS, then moved in place to the odd row stride kRegS + 1, where
// the 32 cells of a colour pass (all of one column parity) spread over all 16 bank
// pairs: 2 shared-memory wavefronts per fp64 access (the minimum) instead of 4.
// Bitwise the same sweep; measured on B200 it does not pay (C4 plain phase 12.91 ->
// 12.73 ms per 24 launches, C3 sweeps 1.298 -> 1.308 ms, C2 step 7.22 -> 7.31 ms, C5
// 0.677 -> 0.691 ms per problem): the tile chain is bound by instruction latency at
// one warp per tile, not by the shared-memory pipe.  Default off.
#ifndef IBMG_RELAYOUT
#define IBMG_RELAYOUT 0
#endif
constexpr int kRegSW = IBMG_RELAYOUT ? kRegS + 1 : kRegS, kRegPW = kReg * kRegSW;
constexpr int kDfWDoubles = 3 * kRegPW;  // w region of a dataflow tile buffer; the b region follows
struct TileWW {
    double* s;  // [3][kReg][kRegSW]
    __device__ __forceinline__ double& operator()(int f, int i, int j) const {
        return s[f * kRegPW + (j + 2) * kRegSW + (i + 2)];
    }
};
// In-place move of the staged region [3][kReg][kRegS] to [3][kReg][kRegSW] (one warp):
// planes from the last to the first, a whole plane through registers, so no source
// is overwritten before it is read (destinations only move up).
__device__ __forceinline__ void relayout_region(double* sw, int lane) {
    if (kRegSW == kRegS) return;
    constexpr int kPer = (kReg * kReg + 31) / 32;
#pragma unroll
    for (int f = 2; f >= 0; --f) {
        double v[kPer];
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int e = lane + 32 * t;
            v[t] = e < kReg * kReg ? sw[f * kRegP + (e / kReg) * kRegS + e % kReg] : 0.0;
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int e = lane + 32 * t;
            if (e < kReg * kReg) sw[f * kRegPW + (e / kReg) * kRegSW + e % kReg] = v[t];
        }
        __syncwarp();
    }
}

// w region of a tile (2-cell halo, 3 planes) into the TileW layout with
// 16-byte cp.async (L1-allocating: w is not written by the launch).
__device__ __forceinline__ void stage_w_region(double* sw, const double* __restrict__ w, int n, int nn, int x0, int y0,
                                               int lane) {
    if (kRegS % 2) {  // odd stride: 8-byte copies
        for (int q = lane; q < 3 * kReg * kReg; q += 32) {
            const int f = q / (kReg * kReg), r = q - f * (kReg * kReg), bb = r / kReg, a = r - bb * kReg;
            cp_async8(&sw[f * kRegP + bb * kRegS + a], w + (size_t)f * nn + wr(x0 - 2 + a, n) + (size_t)wr(y0 - 2 + bb, n) * n);
        }
        return;
    }
    if (lane < 30) {  // 16-byte pairs: lane -> (pair lane % 10, rows lane / 10 + 3 k)
        const int a2 = lane % 10, r0 = lane / 10;
        const int xg = wr(x0 - 2 + 2 * a2, n);
        for (int row = r0; row < 3 * kReg; row += 3) {  // row = f * kReg + bb
            const int f = row / kReg, bb = row - f * kReg;
            cp_async16(&sw[f * kRegP + bb * kRegS + 2 * a2], w + (size_t)f * nn + xg + (size_t)wr(y0 - 2 + bb, n) * n);
        }
    }
}

struct TileB {
    const double* s;  // [3][17][17], local coords in [0, 17)
    __device__ __forceinline__ double operator()(int f, int i, int j) const { return s[f * 289 + j * 17 + i]; }
};

struct TileBG {  // b read through L1 (read-only in the kernel): local coords of the tile
    const double* b;
    int n, nn, x0, y0;
    __device__ __forceinline__ double operator()(int f, int i, int j) const {
        return __ldg(b + (size_t)f * nn + wr(x0 + i, n) + (size_t)wr(y0 + j, n) * n);
    }
};

// Plain phase of one tile colour on a large level (n > 512, bandwidth regime):
// one warp per 16x16 tile; only the w region (2-cell halo) is staged in shared
// memory (9.6 KB per warp -> ~23 resident warps per SM), b is read through L1.
// ty0 (even): first tile row of the launch (a slab's first tile row; 0 for
// the whole level).
__global__ void __launch_bounds__(32) k_plain_tiles(Lev L, int tc, const double* __restrict__ b,
                                                     double* __restrict__ w, const uint8_t* __restrict__ big, int ty0,
                                                     Mirror M) {
    pdl_enter();
    __shared__ __align__(16) double sw[3 * kRegP];
    const int n = L.n, nn = L.nn, lane = threadIdx.x;
    const int half = (n / kTile) >> 1;
    const int tx = 2 * (blockIdx.x % half) + (tc & 1), ty = ty0 + 2 * (blockIdx.x / half) + (tc >> 1);
    const int x0 = tx * kTile, y0 = ty * kTile;
    stage_w_region(sw, w, n, nn, x0, y0, lane);
    cp_async_commit();
    const bool isbig = lane < 16 && big[(x0 >> 2) + (lane & 3) + ((y0 >> 2) + (lane >> 2)) * (n >> 2)];
    const unsigned bigmask = __ballot_sync(0xffffffffu, isbig);
    cp_async_wait<0>();
    __syncwarp();
    TileW W{sw};
    TileBG B{b, n, nn, x0, y0};
    for (int pc = 0; pc < 8; ++pc) {
        const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
        if (!((bigmask >> ((li >> 2) + 4 * (lj >> 2))) & 1)) plain_cell(L, W, B, li, lj);
        __syncwarp();
    }
    // write set: u faces i in [x0, x0+16], v faces j in [y0, y0+16], p cells
    for (int q = lane; q < 17 * 17; q += 32) {
        const int a = q % 17, bb = q / 17, j = wr(y0 + bb, n);
        const size_t gi = wr(x0 + a, n) + (size_t)j * n;
        if (bb < 16) {
            w[gi] = W(0, a, bb);
            M.store(gi, j, n, W(0, a, bb));
        }
        if (a < 16) {
            w[nn + gi] = W(1, a, bb);
            M.store(nn + gi, j, n, W(1, a, bb));
        }
        if (a < 16 && bb < 16) {
            w[2 * nn + gi] = W(2, a, bb);
            M.store(2 * nn + gi, j, n, W(2, a, bb));
        }
    }
}

// Persistent, double-buffered plain phase (bandwidth regime): each one-warp
// CTA walks the tiles of the colour with a grid stride and stages BOTH the w
// region (2-cell halo) and the b region of the NEXT tile with cp.async while
// it relaxes the current one, so every resident warp keeps a tile's loads in
// flight and the 8 passes run on shared memory only.  Per tile the arithmetic
// is plain_cell on the same values as k_plain_tiles (bitwise identical).
constexpr int kPPBw = 3 * kRegP;           // w region doubles
constexpr int kPPBb = 3 * 289;              // b region doubles (17 x 17, odd stride)
constexpr int kPPBuf = (kPPBw + kPPBb + 1) / 2 * 2;  // even: both buffers 16-byte aligned
constexpr size_t kPPSmem = 2 * kPPBuf * sizeof(double);
__device__ __forceinline__ void pp_issue(double* buf, const double* __restrict__ w, const double* __restrict__ b, int n,
                                         int nn, int x0, int y0, int lane) {
    stage_w_region(buf, w, n, nn, x0, y0, lane);
    if (lane < 17) {  // b region 17 x 17: lane = column, one row per step
        const int xb = wr(x0 + lane, n);
        for (int bb = 0; bb < 17; ++bb) {
            const size_t gi = xb + (size_t)wr(y0 + bb, n) * n;
            const int sq = bb * 17 + lane;
            cp_async8(&buf[kPPBw + sq], b + gi);
            cp_async8(&buf[kPPBw + 289 + sq], b + nn + gi);
            cp_async8(&buf[kPPBw + 578 + sq], b + 2 * nn + gi);
        }
    }
}

__global__ void __launch_bounds__(32) k_plain_tiles_pp(Lev L, int tc, const double* __restrict__ b,
                                                        double* __restrict__ w, const uint8_t* __restrict__ big,
                                                        int ty0, int ntiles, Mirror M) {
    pdl_enter();
    extern __shared__ __align__(16) double pps[];
    const int n = L.n, nn = L.nn, lane = threadIdx.x;
    const int half = (n / kTile) >> 1;
    auto origin = [&](int t, int& x0, int& y0) {
        x0 = (2 * (t % half) + (tc & 1)) * kTile;
        y0 = (ty0 + 2 * (t / half) + (tc >> 1)) * kTile;
    };
    int t = blockIdx.x;
    if (t >= ntiles) return;
    int x0, y0;
    origin(t, x0, y0);
    pp_issue(pps, w, b, n, nn, x0, y0, lane);
    cp_async_commit();
    // big-block flags of a tile: loaded one tile ahead (their latency hides
    // behind the current tile instead of stalling the ballot)
    auto flag = [&](int xa, int ya) {
        return lane < 16 ? big[(xa >> 2) + (lane & 3) + ((ya >> 2) + (lane >> 2)) * (n >> 2)] : (uint8_t)0;
    };
    uint8_t fcur = flag(x0, y0);
    for (int k = 0; t < ntiles; t += gridDim.x, ++k) {
        const int tn = t + gridDim.x;
        int xn = 0, yn = 0;
        uint8_t fnext = 0;
        if (tn < ntiles) {
            origin(tn, xn, yn);
            pp_issue(pps + ((k + 1) & 1) * kPPBuf, w, b, n, nn, xn, yn, lane);
            fnext = flag(xn, yn);
        }
        cp_async_commit();
        const unsigned bigmask = __ballot_sync(0xffffffffu, fcur != 0);
        cp_async_wait<1>();
        __syncwarp();
        double* buf = pps + (k & 1) * kPPBuf;
        TileW W{buf};
        TileB B{buf + kPPBw};
        for (int pc = 0; pc < 8; ++pc) {
            const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
            if (!((bigmask >> ((li >> 2) + 4 * (lj >> 2))) & 1)) plain_cell(L, W, B, li, lj);
            __syncwarp();
        }
        {  // write set (as k_plain_tiles): half-warps take alternate rows, lane & 15
           // the column; lanes 0..15 then store the u column x0 + 16
            const int a = lane & 15, h = lane >> 4;
            const int xa = wr(x0 + a, n);
            for (int bb = h; bb < 17; bb += 2) {
                const int j = wr(y0 + bb, n);
                const size_t gi = xa + (size_t)j * n;
                if (bb < 16) {
                    w[gi] = W(0, a, bb);
                    M.store(gi, j, n, W(0, a, bb));
                    w[2 * nn + gi] = W(2, a, bb);
                    M.store(2 * nn + gi, j, n, W(2, a, bb));
                }
                w[nn + gi] = W(1, a, bb);
                M.store(nn + gi, j, n, W(1, a, bb));
            }
            if (lane < 16) {
                const int j = wr(y0 + lane, n);
                const size_t gi = wr(x0 + 16, n) + (size_t)j * n;
                w[gi] = W(0, 16, lane);
                M.store(gi, j, n, W(0, 16, lane));
            }
        }
        __syncwarp();  // this buffer is refilled two tiles later
        x0 = xn;
        y0 = yn;
        fcur = fnext;
    }
    cp_async_wait<0>();
}

// Global accessor for plain loads (no __ldg: the big phase writes w in-kernel).
struct GAccRW {
    const double* w;
    int n, nn;
    __device__ __forceinline__ double operator()(int comp, int i, int j) const {
        return w[(size_t)comp * nn + i + (size_t)j * n];
    }
};

// Residual of block DOF t (0..55) of the block at (bi, bj): b - A w including
// the -E' part from the assembled rows (row fi of the level's EMat, -1 if the
// face has no E' row).
template <class Acc, class BAcc, class WAcc>
__device__ __forceinline__ double block_residual(const Lev& L, const EMat& E, const Acc& acc, const BAcc& bacc,
                                                 const WAcc& flat, int fi, int t, int bi, int bj) {
    int f, i, j;
    block_dof(t, bi, bj, f, i, j);
    i = wr(i, L.n);
    j = wr(j, L.n);
    double ru, rv, rp;
    stokes_rows(L, acc, i, j, ru, rv, rp);
    double r = bacc(f, i, j) - (f == 0 ? ru : f == 1 ? rv : rp);
    if (fi >= 0) {
        double s = 0.0;
        for (int e = E.rp[fi]; e < E.rp[fi + 1]; ++e) s += E.val[e] * flat(E.col[e]);
        r += s;
    }
    return r;
}

struct FlatG {
    const double* w;
    __device__ __forceinline__ double operator()(int idx) const { return w[idx]; }
};

constexpr int kGroup = 128;
struct BigScratch {
    double sr[56], se[40], part[2][56], epart[3][40], wold[56];
};

// ---- per-block "slab": all w-independent data of one big block, packed at
// setup so it can be streamed into shared memory with cp.async ahead of use:
// the 56x56 inverse (col-major), the 40 E' row pointers (relative, padded to
// 48 ints) and the rows' (col, val) entries with columns pre-encoded as
// shared-memory indices (>= 0) or global flat indices (-(flat+1)).
constexpr int kSlabCap = 2560;  // entries per block held in shared memory
struct SlabSlot {
    double A[3136];
    double val[kSlabCap];
    int col[kSlabCap];
    int rp[48];
};
static_assert(sizeof(SlabSlot) % 16 == 0, "slot alignment");

struct Slabs {
    const double* Ainv;  // [nbig][3136]
    const int* rp;       // [nbig][48]
    const int* off;      // [nbig+1] entry offsets (multiples of 4)
    const int* col;
    const double* val;
};

// The E' entries of block q past kSlabCap (structures denser than ~h/3
// point spacing give blocks more entries than a shared-memory slot holds)
// stay in the slab arrays in global memory: a thread whose row runs past the
// slot adds them after its slot entries, in its own stride class and
// ascending order (blocks within the slot keep their exact summation order).
struct SlabTail {
    const Slabs* SL;  // nullptr: every entry is in the slot
    int q;
    template <class LocA>
    __device__ __forceinline__ double sum(int e0, int e1, int stride, const LocA& wloc) const {
        double s = 0.0;
        if (SL == nullptr || e1 <= kSlabCap) return s;
        const int o = __ldg(SL->off + q);
        int e = e0;
        if (e < kSlabCap) e += (kSlabCap - e + stride - 1) / stride * stride;
        for (; e < e1; e += stride) s += __ldg(SL->val + o + e) * wloc[__ldg(SL->col + o + e)];
        return s;
    }
};


__device__ __forceinline__ void slab_issue(SlabSlot& slot, const Slabs& SL, int q, int t, int nt) {
    const char* A = reinterpret_cast<const char*>(SL.Ainv + (size_t)q * 3136);
    char* dA = reinterpret_cast<char*>(slot.A);
    for (int c = t; c < 3136 * 8 / 16; c += nt) cp_async16(dA + 16 * c, A + 16 * c);
    if (t < 12) cp_async16(reinterpret_cast<char*>(slot.rp) + 16 * t, reinterpret_cast<const char*>(SL.rp + (size_t)q * 48) + 16 * t);
    // entries past kSlabCap stay in global memory (slab_entry)
    const int o = SL.off[q], cnt = min(SL.off[q + 1] - o, kSlabCap);
    const char* cv = reinterpret_cast<const char*>(SL.val + o);
    const char* cc = reinterpret_cast<const char*>(SL.col + o);
    for (int c = t; c < cnt / 2; c += nt) cp_async16(reinterpret_cast<char*>(slot.val) + 16 * c, cv + 16 * c);
    for (int c = t; c < cnt / 4; c += nt) cp_async16(reinterpret_cast<char*>(slot.col) + 16 * c, cc + 16 * c);
}

// One big-block relaxation from a shared-memory slab by 128 threads (flat
// column encoding: every E' column is indexed through `wloc`): Stokes
// residual of the 56 DOFs + E' row dots (3 threads per row) -> 56x56 inverse
// (2 column halves) -> correction.  Only shared-memory traffic except E'
// columns outside the staged region (global, not modified by this launch).
template <class WA, class LocA, class GlobA, class BA, class WAdd>
__device__ __forceinline__ void big_block_slab(const Lev& L, const SlabSlot& slot, int bi, int bj, const WA& W,
                                               const LocA& wloc, const GlobA& wglob, const BA& Bv, WAdd&& wadd,
                                               BigScratch& S, int gt, unsigned long long* dbg = nullptr,
                                               SlabTail tail = SlabTail{nullptr, 0}) {
    // stencil row and E' row dots are computed into registers first and
    // stored after both, so their global gathers are in flight together (one
    // L2 round trip for the residual instead of two)
    double sres = 0.0, wcur = 0.0, s0 = 0.0;
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        i = wr(i, L.n);
        j = wr(j, L.n);
        sres = Bv(f, i, j) - stokes_row(L, W, f, i, j);
        wcur = W(f, i, j);  // current value, reused for the correction (no re-read)
    }
    // E' row dots: 3 threads per row (strided entries), up to 24 column
    // gathers in flight per thread, fixed-order combine
    if (gt < 120) {
        const int r = gt % 40, p = gt / 40;
        const int e1 = min(slot.rp[r + 1], kSlabCap);
        for (int e = slot.rp[r] + p; e < e1; e += 72) {  // one round of up to 24 gathers per thread
            int cc[24];
            double vv[24], xx[24];
#pragma unroll
            for (int m = 0; m < 24; ++m) {  // branch-free: clamp the index, mask the value
                const int em = e + 3 * m;
                const bool ok = em < e1;
                cc[m] = slot.col[ok ? em : e];
                vv[m] = ok ? slot.val[em] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < 24; ++m) xx[m] = wloc[cc[m]];
#pragma unroll
            for (int m = 0; m < 24; ++m) s0 += vv[m] * xx[m];
        }
        s0 += tail.sum(slot.rp[r] + p, slot.rp[r + 1], 3, wloc);
    }
    if (gt < 56) {
        S.sr[gt] = sres;
        S.wold[gt] = wcur;
    }
    if (gt < 120) S.epart[gt / 40][gt % 40] = s0;
    if (dbg && gt == 0) dbg[0] = gtimer();
    __syncthreads();
    if (dbg && gt == 0) dbg[1] = gtimer();
    if (gt < 40) S.sr[gt] += (S.epart[0][gt] + S.epart[1][gt]) + S.epart[2][gt];  // combined residual
    __syncthreads();
    if (gt < 112) {
        const int row = gt % 56, cg = gt / 56;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < 28; c += 2) {
            const int cc = 28 * cg + c;
            s0 += slot.A[cc * 56 + row] * S.sr[cc];
            s1 += slot.A[(cc + 1) * 56 + row] * S.sr[cc + 1];
        }
        S.part[cg][row] = s0 + s1;
    }
    __syncthreads();
    if (dbg && gt == 0) dbg[2] = gtimer();
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        wadd(f, wr(i, L.n), wr(j, L.n), S.wold[gt], S.part[0][gt] + S.part[1][gt]);
    }
}

// E'-row part of a slab only (the coarse kernel keeps 4 of these in shared
// memory, one per 128-thread group; the inverse is read from L2 into registers).
struct ESlot {
    double val[kSlabCap];
    int col[kSlabCap];
    int rp[48];
};
static_assert(sizeof(ESlot) % 16 == 0, "slot alignment");

__device__ __forceinline__ void eslot_issue(ESlot& slot, const Slabs& SL, int q, int t, int nt) {
    if (t < 12) cp_async16(reinterpret_cast<char*>(slot.rp) + 16 * t, reinterpret_cast<const char*>(SL.rp + (size_t)q * 48) + 16 * t);
    // entries past kSlabCap stay in global memory (slab_entry)
    const int o = SL.off[q], cnt = min(SL.off[q + 1] - o, kSlabCap);
    const char* cv = reinterpret_cast<const char*>(SL.val + o);
    const char* cc = reinterpret_cast<const char*>(SL.col + o);
    for (int c = t; c < cnt / 2; c += nt) cp_async16(reinterpret_cast<char*>(slot.val) + 16 * c, cv + 16 * c);
    for (int c = t; c < cnt / 4; c += nt) cp_async16(reinterpret_cast<char*>(slot.col) + 16 * c, cc + 16 * c);
}

// big_block_slab with the E' rows from an ESlot and the inverse streamed from
// global memory straight into registers (issued first, overlapping the
// residual).  `gsync` is the group barrier.
struct NoOp {
    __device__ __forceinline__ void operator()() const {}
};

// `after_rows` runs right after the first group barrier, when the slot's E'
// rows have been consumed (callers refill the slot with the next block there).
__device__ __forceinline__ void load_inverse_part(double (&av)[28], const double* __restrict__ A_q, int gt) {
    if (gt < 112) {
        const double* A = A_q + (size_t)(28 * (gt / 56)) * 56 + gt % 56;
#pragma unroll
        for (int c = 0; c < 28; ++c) av[c] = __ldg(A + c * 56);
    }
}

// The inverse arrives in `av` (this thread's 28 entries): loaded here when
// A_q != nullptr, else preloaded by the caller; A_next != nullptr prefetches
// the next block's part into `av` after the apply, hiding its L2 latency
// behind the write-back and the colour barrier.
// EDOT 0: E' row dots by 3 threads per row, 24 gathers in flight per thread
// (latency: one block per CTA, long fine-level rows).  EDOT 1: one thread per
// row (threads 64..103, a warp apart from the stencil rows), 8 at a time —
// fewer instructions where several groups share an SM (coarse kernel).
template <int EDOT = 0, class WA, class LocA, class BA, class WAdd, class Sync, class After = NoOp>
__device__ __forceinline__ void big_block_es(const Lev& L, const ESlot& slot, const double* __restrict__ A_q, int bi,
                                             int bj, const WA& W, const LocA& wloc, const BA& Bv, WAdd&& wadd,
                                             BigScratch& S, int gt, Sync&& gsync, After after_rows = After{},
                                             double* avp = nullptr, const double* __restrict__ A_next = nullptr,
                                             SlabTail tail = SlabTail{nullptr, 0}) {
    double avl[28];
    double (&av)[28] = avp ? *reinterpret_cast<double(*)[28]>(avp) : avl;
    const int row = gt % 56, cg = gt / 56;
    if (A_q) load_inverse_part(av, A_q, gt);
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        i = wr(i, L.n);
        j = wr(j, L.n);
        S.sr[gt] = Bv(f, i, j) - stokes_row(L, W, f, i, j);
        S.wold[gt] = W(f, i, j);  // current value, reused for the correction (no re-read)
    }
    if (EDOT == 0 && gt < 120) {  // E' row dots: 3 threads per row, 24 gathers per round
        const int r = gt % 40, p = gt / 40;
        const int e1 = min(slot.rp[r + 1], kSlabCap);
        double s0 = 0.0;
        for (int e = slot.rp[r] + p; e < e1; e += 72) {  // one round of up to 24 gathers per thread
            double vv[24], xx[24];
#pragma unroll
            for (int m = 0; m < 24; ++m) {
                const int em = e + 3 * m;
                vv[m] = em < e1 ? slot.val[em] : 0.0;
                xx[m] = em < e1 ? wloc[slot.col[em]] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < 24; ++m) s0 += vv[m] * xx[m];
        }
        S.epart[p][r] = s0 + tail.sum(slot.rp[r] + p, slot.rp[r + 1], 3, wloc);
    }
    if (EDOT == 1 && gt >= 64 && gt < 104) {  // E' row dots: one thread per row
        const int r = gt - 64;
        const int e1 = min(slot.rp[r + 1], kSlabCap);
        double s0 = 0.0, s1 = 0.0;
        for (int e = slot.rp[r]; e < e1; e += 8) {
            double vv[8], xx[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int em = e + m;
                vv[m] = em < e1 ? slot.val[em] : 0.0;
                xx[m] = em < e1 ? wloc[slot.col[em]] : 0.0;
            }
#pragma unroll
            for (int m = 0; m < 8; m += 2) {
                s0 += vv[m] * xx[m];
                s1 += vv[m + 1] * xx[m + 1];
            }
        }
        S.epart[0][r] = (s0 + s1) + tail.sum(slot.rp[r], slot.rp[r + 1], 1, wloc);
    }
    gsync();
    after_rows();
    if (gt < 40)  // combined residual
        S.sr[gt] += EDOT == 0 ? (S.epart[0][gt] + S.epart[1][gt]) + S.epart[2][gt] : S.epart[0][gt];
    gsync();
    if (gt < 112) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int c = 0; c < 28; c += 2) {
            const int cc = 28 * cg + c;
            s0 += av[c] * S.sr[cc];
            s1 += av[c + 1] * S.sr[cc + 1];
        }
        S.part[cg][row] = s0 + s1;
    }
    if (A_next) load_inverse_part(av, A_next, gt);
    gsync();
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        wadd(f, wr(i, L.n), wr(j, L.n), S.wold[gt], S.part[0][gt] + S.part[1][gt]);
    }
}

// Global accessors that bypass L1 (ld.global.cg): the big phase reads values
// other CTAs wrote before the last grid barrier.
struct GAccCG {
    const double* w;
    int n, nn;
    __device__ __forceinline__ double operator()(int comp, int i, int j) const {
        return __ldcg(w + (size_t)comp * nn + i + (size_t)j * n);
    }
};
struct GAccB {
    const double* b;
    int n, nn;
    __device__ __forceinline__ double operator()(int comp, int i, int j) const {
        return __ldg(b + (size_t)comp * nn + i + (size_t)j * n);
    }
};
struct FlatCG {
    const double* w;
    __device__ __forceinline__ double operator[](int idx) const { return __ldcg(w + idx); }
};

struct BigColours {
    int ncol;
    int off[33];
};

struct BigDeps {
    const int* pred;   // predecessor list positions (CSR by block)
    const int* poff;
    unsigned* flags;   // completion epoch per block
    unsigned epoch;    // this launch's epoch (monotone per level)
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The big phase of one sweep on a level as ONE cooperative persistent kernel
// without grid barriers: each CTA takes its blocks in colour order; a block
// waits (acquire) until its predecessors — the conflicting big blocks of
// smaller colour — have published this epoch (release), so the result is
// exactly the colour-ordered Gauss-Seidel schedule while blocks that do not
// depend on each other run ahead.  The cooperative launch makes all CTAs
// co-resident, and dependencies only point to smaller colours, so the waits
// cannot deadlock.  The E' rows of a block go through one 31 KB shared-memory
// slot, refilled with the next block's rows once they are consumed (4 CTAs/SM,
// register-limited); the 25 KB inverse streams straight into registers at the
// start of each block.
constexpr int kBigThreads = 128;
constexpr size_t kBigSmem = sizeof(ESlot);
__global__ void __launch_bounds__(kBigThreads) k_big_phase(Lev L, Slabs SL, BigColours BC, BigDeps DP,
                                                            const double* __restrict__ b, double* w, Mirror M) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char dsm[];
    ESlot* slot = reinterpret_cast<ESlot*>(dsm);
    __shared__ BigScratch S;
    const int t = threadIdx.x, G = gridDim.x, nbk = L.n >> 2;
    auto next_item = [&](int c, int q, int& nc, int& nq) {
        // the item after (c, q) for this CTA; c = -1 starts the enumeration
        nq = (c < 0) ? -1 : q + G;
        nc = (c < 0) ? 0 : c;
        while (nc < BC.ncol) {
            if (nq < 0) nq = BC.off[nc] + (int)blockIdx.x;
            if (nq < BC.off[nc + 1]) return;
            ++nc;
            nq = -1;
        }
    };
    int c, q;
    next_item(-1, 0, c, q);
    if (c < BC.ncol) eslot_issue(slot[0], SL, q, t, kBigThreads);
    cp_async_commit();
    GAccCG W{w, L.n, L.nn};
    GAccB B{b, L.n, L.nn};
    int k = 0;
    while (c < BC.ncol) {
        int nc, nq;
        next_item(c, q, nc, nq);
        // wait for the predecessors of block q (one thread per predecessor);
        // poff == nullptr: one colour per launch (slab mode), nothing to wait for
        if (DP.poff)
            for (int e = DP.poff[q] + t; e < DP.poff[q + 1]; e += kBigThreads)
                while (ld_acquire(DP.flags + DP.pred[e]) != DP.epoch) __nanosleep(8);
        cp_async_wait<0>();
        __syncthreads();
        const ESlot& sl = slot[0];
        const int Bk = sl.rp[47];
        // one E'-row slot: refilled with the next block's rows as soon as this
        // block's rows are consumed (overlapping the matvec, the write-back,
        // the publish and the next dependency wait); one slot keeps 4 CTAs
        // per SM resident instead of 3
        big_block_es(L, sl, SL.Ainv + (size_t)q * 3136, 4 * (Bk % nbk), 4 * (Bk / nbk), W, FlatCG{w}, B,
                     [&](int f, int i, int j, double old, double d) {
                         const size_t off = (size_t)f * L.nn + i + (size_t)j * L.n;
                         __stcg(w + off, old + d);
                         M.store(off, j, L.n, old + d);
                     },
                     S, t, [] { __syncthreads(); },
                     [&] {
                         if (nc < BC.ncol) eslot_issue(slot[0], SL, nq, t, kBigThreads);
                         cp_async_commit();
                     },
                     nullptr, nullptr, SlabTail{&SL, q});
        __syncthreads();
        if (t == 0 && DP.flags) {  // bar.sync + st.release.gpu order the CTA's w stores before the flag
            st_release(DP.flags + q, DP.epoch);
        }
        ++k;
        c = nc;
        q = nq;
    }
    cp_async_wait<0>();
}


// ---- dataflow sweep (latency regime, 64 <= n <= 512) ------------------------
// One sweep of a level as ONE cooperative persistent kernel executing a task
// DAG: the plain tiles (warp tasks, tile-colour-major order),
// then the big blocks (CTA tasks, colour order).  A tile waits for its adjacent
// tiles of smaller tile colour; a big block waits for its conflicting big
// blocks of smaller colour and for every plain tile within 8 cells of it (its
// E' reach + stencil).  Each waiter polls completion epochs with acquire loads;
// each finisher publishes with a release store.  Every dependency points to an
// earlier task and all CTAs are co-resident, so the DAG cannot deadlock, and
// the result is exactly the colour-ordered schedule of the oracle.
constexpr int kDfWarps = 4;
struct DfArgs {
    Lev L;
    Slabs SL;
    BigColours BC;
    BigDeps DP;
    unsigned* tflags;        // per-tile completion epochs
    const uint8_t* big;
    const double* b;
    double* w;
    unsigned long long* trace;  // debug: per-task globaltimer stamps (nullptr in production)
};
constexpr size_t kDfTileBytes = (kDfWDoubles + 3 * 289) * sizeof(double);
constexpr size_t kDfSmem = 2 * sizeof(SlabSlot) + kDfWarps * ((kDfTileBytes + 15) / 16 * 16);

__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// ---- TMA staging of a tile's w region (Blackwell tensor memory accelerator)
// One 2-D tensor map per plane of the level's w (rows of n doubles, box 20 x 20
// = the tile plus its 2-cell halo, landing in the TileW layout, row stride 20):
// an interior tile's w region is three cp.async.bulk.tensor copies issued by one
// lane and completed on an mbarrier, instead of 20 16-byte cp.async per lane.
// Tiles whose region wraps the periodic edge keep the cp.async path (TMA
// fills out-of-bound boxes with zeros, not the periodic image).
struct TmaPlanes {
    CUtensorMap m[3];
    int use;  // 0: no tensor maps (cp.async staging everywhere)
};
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(mb)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, unsigned long long* mb) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(mb))
        : "memory");
}

// One plain tile task of a dataflow sweep (one warp): stage b and the
// big-block flags, wait for the adjacent tiles of smaller tile colour, stage
// the w region (L2 only: neighbours were written by other SMs), run the 8
// colour passes in shared memory, write back with L2 stores and publish the
// tile's epoch.  sw / sb: the warp's w region and b region buffers.
// trace: debug timeline slot of the task (nullptr in production).
__device__ __forceinline__ void df_plain_tile(const Lev& L, const double* __restrict__ b, double* __restrict__ w,
                                              const uint8_t* __restrict__ big, unsigned* tflags, unsigned epoch,
                                              int tx, int ty, int tc, double* sw, double* sb,
                                              unsigned long long* trace, const TmaPlanes* tm = nullptr,
                                              unsigned long long* mbar = nullptr, unsigned* mphase = nullptr) {
    const int n = L.n, nn = L.nn, lane = threadIdx.x & 31, nt = n / kTile, nbk = n >> 2;
    const int x0 = tx * kTile, y0 = ty * kTile;
    const unsigned long long t_a = trace ? gtimer() : 0;
    // b and the big-block flags are read-only in the sweep: staged before the
    // dependency wait (off the critical path of the tile-colour chain)
    for (int qq = lane; qq < 289; qq += 32) {
        const int a = qq % 17, bb = qq / 17;
        const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
        cp_async8(&sb[qq], b + gi);
        cp_async8(&sb[289 + qq], b + nn + gi);
        cp_async8(&sb[578 + qq], b + 2 * nn + gi);
    }
    cp_async_commit();
    const bool isbig = lane < 16 && big[(x0 >> 2) + (lane & 3) + ((y0 >> 2) + (lane >> 2)) * nbk];
    if (lane < 8) {  // adjacent tiles of smaller tile colour
        const int d = lane < 4 ? lane : lane + 1;  // skip the centre of the 3x3
        const int ax = wr(tx + d % 3 - 1, nt), ay = wr(ty + d / 3 - 1, nt);
        const int ac = (ax & 1) + 2 * (ay & 1);
        if (ac < tc)
            while (ld_acquire(tflags + ax + ay * nt) != epoch) __nanosleep(8);
    }
    __syncwarp();
    const unsigned long long t_b = trace ? gtimer() : 0;
    const bool tma = tm && kRegS == kReg && x0 >= 2 && y0 >= 2 && x0 + kTile + 2 <= n && y0 + kTile + 2 <= n;
    if (tma) {  // interior tile: three tensor copies (see TmaPlanes)
        if (lane == 0) {
            // the neighbours' stores (generic proxy, acquired above) before the
            // async-proxy reads; this warp's last reads of sw before its writes
            asm volatile("fence.proxy.async.global;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(mbar, 3u * kRegP * 8u);
#pragma unroll
            for (int f = 0; f < 3; ++f) tma_load_2d(sw + f * kRegP, &tm->m[f], x0 - 2, y0 - 2, mbar);
        }
    } else if (kRegS % 2) {  // odd stride: 8-byte copies (L2 only)
        for (int q = lane; q < 3 * kReg * kReg; q += 32) {
            const int f = q / (kReg * kReg), r = q - f * (kReg * kReg), bb = r / kReg, a = r - bb * kReg;
            const unsigned sa = (unsigned)__cvta_generic_to_shared(&sw[f * kRegP + bb * kRegS + a]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa),
                         "l"(w + (size_t)f * nn + wr(x0 - 2 + a, n) + (size_t)wr(y0 - 2 + bb, n) * n));
        }
    } else if (lane < 30) {  // 16-byte pairs, L2 only: lane -> (pair lane % 10, rows lane / 10 + 3 k)
        const int a2 = lane % 10, r0 = lane / 10;
        const int xg = wr(x0 - 2 + 2 * a2, n);
        for (int row = r0; row < 3 * kReg; row += 3) {  // row = f * kReg + bb
            const int f = row / kReg, bb = row - f * kReg;
            const size_t gi = xg + (size_t)wr(y0 - 2 + bb, n) * n;
            cp_async16_cg(&sw[f * kRegP + bb * kRegS + 2 * a2], w + (size_t)f * nn + gi);
        }
    }
    cp_async_commit();
    const unsigned bigmask = __ballot_sync(0xffffffffu, isbig);
    cp_async_wait<0>();
    if (tma) {
        mbar_wait(mbar, *mphase);
        *mphase ^= 1u;
    }
    __syncwarp();
    relayout_region(sw, lane);
    const unsigned long long t_s = trace ? gtimer() : 0;
    TileWW W{sw};
    TileB B{sb};
    for (int pc = 0; pc < 8; ++pc) {
        const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
        if (!((bigmask >> ((li >> 2) + 4 * (lj >> 2))) & 1)) plain_cell(L, W, B, li, lj);
        __syncwarp();
    }
    const unsigned long long t_p = trace ? gtimer() : 0;
    {  // write set: u faces i in [x0, x0+16], v faces j in [y0, y0+16], p cells.
       // Half-warps take alternate rows, lane & 15 the column (few index
       // operations: one warp per scheduler here, every instruction's latency
       // is on the tile chain); lanes 0..15 then store the u column x0 + 16.
        const int a = lane & 15, h = lane >> 4;
        const int xa = wr(x0 + a, n);
        for (int bb = h; bb < 17; bb += 2) {
            const size_t gi = xa + (size_t)wr(y0 + bb, n) * n;
            if (bb < 16) {
                __stcg(w + gi, W(0, a, bb));
                __stcg(w + 2 * nn + gi, W(2, a, bb));
            }
            __stcg(w + nn + gi, W(1, a, bb));
        }
        if (lane < 16) __stcg(w + wr(x0 + 16, n) + (size_t)wr(y0 + lane, n) * n, W(0, 16, lane));
    }
    __syncwarp();
    if (lane == 0) {  // warp-synchronous stores + st.release.gpu (cumulative) publish the tile
        st_release(tflags + tx + ty * nt, epoch);
        if (trace) {
            unsigned long long* r = trace;
            r[0] = t_a;
            r[1] = t_b;
            r[2] = gtimer();
            r[3] = blockIdx.x;
            r[4] = t_s;
            r[5] = t_p;
        }
    }
}

// ---- plain phase of a large level (n > 512) as one band-major dataflow launch
// The same tile tasks and dependencies as k_sweep_df's plain part (so the
// result is the oracle's tile-colour-ordered schedule), but the tasks run in
// skewed tile-row bands (ibmg.cu plain_df_order: seg[] maps each half row of
// tasks to its tile row and colour) instead of colour by colour.  Every
// tile's smaller-colour neighbours come earlier in that order, so it is a
// valid task order for the DAG.  The live rows are a few bands, mostly
// L2-resident: a tile's halo was written recently by its neighbours, and w
// and b cross HBM about once per sweep instead of once per tile colour plus
// halos (4 separate tile-colour launches).  One-warp CTAs, one w and one b
// region per warp; cooperative launch (all CTAs co-resident) => no deadlock.
constexpr size_t kPdfSmem = (kDfTileBytes + 127) / 128 * 128;
__global__ void __launch_bounds__(32) k_plain_df(Lev L, const double* __restrict__ b, double* __restrict__ w,
                                                  const uint8_t* __restrict__ big, unsigned* tflags, unsigned epoch,
                                                  const int* __restrict__ seg, const __grid_constant__ TmaPlanes tm) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char pdm[];
    __shared__ __align__(8) unsigned long long mbar;
    double* sw = reinterpret_cast<double*>(pdm);
    double* sb = sw + kDfWDoubles;
    const int nt = L.n / kTile, half = nt >> 1, ntiles = nt * nt;
    unsigned phase = 0;
    if (tm.use) {
        if (threadIdx.x == 0) mbar_init(&mbar, 1);
        __syncwarp();
    }
    for (int task = blockIdx.x; task < ntiles; task += gridDim.x) {
        const int s = task / half, i = task - s * half;
        const int sg = __ldg(seg + s), ty = sg >> 2, tc = sg & 3;
        df_plain_tile(L, b, w, big, tflags, epoch, 2 * i + (tc & 1), ty, tc, sw, sb, nullptr,
                      tm.use ? &tm : nullptr, &mbar, &phase);
    }
}

// ---- warp-specialised band-major plain phase (k_plain_df2, opt-in IBMG_PDF2=1) ----
// Same tasks, order and arithmetic as k_plain_df, two warps per CTA: the LOADER warp
// stages tile t + 1 (b region, dependency waits, w region by tensor copies or cp.async)
// into the second buffer while the COMPUTE warp runs the 8 colour passes, the write-back
// and the publish of tile t.  full[s] / empty[s] mbarriers hand the buffers over.
__device__ __forceinline__ void mbar_arrive(unsigned long long* mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
}
// arrive on mb once all cp.async copies this thread has issued so far have landed (no wait here)
__device__ __forceinline__ void cp_async_arrive(unsigned long long* mb) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(mb)) : "memory");
}
#ifndef IBMG_PDF2_NC
#define IBMG_PDF2_NC 3
#endif
#ifndef IBMG_PDF2_NL
#define IBMG_PDF2_NL 1
#endif
constexpr int kPdf2NC = IBMG_PDF2_NC;        // compute warps per CTA
constexpr int kPdf2NL = IBMG_PDF2_NL;        // loader warps per CTA (a loader stages ~1 tile per us: 81 8-byte b copies per lane)
constexpr int kPdf2NB = kPdf2NC + kPdf2NL;   // tile buffers per CTA
constexpr size_t kPdf2Buf = (kDfTileBytes + 127) / 128 * 128;
constexpr size_t kPdf2Smem = kPdf2NB * kPdf2Buf;
__global__ void __launch_bounds__(32 * kPdf2NB)
    k_plain_df2(Lev L, const double* __restrict__ b, double* __restrict__ w, const uint8_t* __restrict__ big,
                unsigned* tflags, unsigned epoch, const int* __restrict__ seg, const __grid_constant__ TmaPlanes tm) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char pdm[];
    __shared__ __align__(8) unsigned long long full[kPdf2NB], empty[kPdf2NB];
    const int n = L.n, nn = L.nn, lane = threadIdx.x & 31, role = threadIdx.x >> 5;  // roles < NL: loaders
    const int nt = n / kTile, half = nt >> 1, ntiles = nt * nt, nbk = n >> 2;
    if (threadIdx.x == 0) {
        for (int q = 0; q < kPdf2NB; ++q) {
            mbar_init(&full[q], 33);  // 32 lanes' cp.async completions + lane 0's arrival (with the tensor bytes)
            mbar_init(&empty[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int it = 0;
    for (int task = blockIdx.x; task < ntiles; task += gridDim.x, ++it) {
        // loader it % NL stages the CTA's it-th tile, compute warp it % NC relaxes it
        if (role < kPdf2NL ? role != it % kPdf2NL : role - kPdf2NL != it % kPdf2NC) continue;
        const int sl = it % kPdf2NB;
        const unsigned ph = (it / kPdf2NB) & 1;
        double* sw = reinterpret_cast<double*>(pdm + sl * kPdf2Buf);
        double* sb = sw + kDfWDoubles;
        const int sI = task / half, i = task - sI * half;
        const int sg = __ldg(seg + sI), ty = sg >> 2, tc = sg & 3, tx = 2 * i + (tc & 1);
        const int x0 = tx * kTile, y0 = ty * kTile;
        if (role < kPdf2NL) {
            // ---------------- loader ----------------
            if (it >= kPdf2NB) mbar_wait(&empty[sl], ph ^ 1u);  // its previous tile's compute warp is done with it
            for (int qq = lane; qq < 289; qq += 32) {
                const int a = qq % 17, bb = qq / 17;
                const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
                cp_async8(&sb[qq], b + gi);
                cp_async8(&sb[289 + qq], b + nn + gi);
                cp_async8(&sb[578 + qq], b + 2 * nn + gi);
            }
            if (lane < 8) {  // adjacent tiles of smaller tile colour
                const int d = lane < 4 ? lane : lane + 1;
                const int ax = wr(tx + d % 3 - 1, nt), ay = wr(ty + d / 3 - 1, nt);
                const int ac = (ax & 1) + 2 * (ay & 1);
                if (ac < tc)
                    while (ld_acquire(tflags + ax + ay * nt) != epoch) __nanosleep(8);
            }
            __syncwarp();
            // nothing below waits for a copy: the lanes' cp.async completions and the tensor bytes
            // arrive on full[sl] by themselves, and the loader moves on to the next tile
            const bool tma = tm.use && x0 >= 2 && y0 >= 2 && x0 + kTile + 2 <= n && y0 + kTile + 2 <= n;
            if (!tma && lane < 30) {
                const int a2 = lane % 10, r0 = lane / 10;
                const int xg = wr(x0 - 2 + 2 * a2, n);
                for (int row = r0; row < 3 * kReg; row += 3) {
                    const int f = row / kReg, bb = row - f * kReg;
                    const size_t gi = xg + (size_t)wr(y0 - 2 + bb, n) * n;
                    cp_async16_cg(&sw[f * kRegP + bb * kRegS + 2 * a2], w + (size_t)f * nn + gi);
                }
            }
            cp_async_arrive(&full[sl]);
            if (lane == 0) {
                if (tma) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&full[sl], 3u * kRegP * 8u);
#pragma unroll
                    for (int f = 0; f < 3; ++f) tma_load_2d(sw + f * kRegP, &tm.m[f], x0 - 2, y0 - 2, &full[sl]);
                } else {
                    mbar_arrive(&full[sl]);
                }
            }
        } else {
            // ---------------- compute ----------------
            const bool isbig = lane < 16 && big[(x0 >> 2) + (lane & 3) + ((y0 >> 2) + (lane >> 2)) * nbk];
            const unsigned bigmask = __ballot_sync(0xffffffffu, isbig);
            mbar_wait(&full[sl], ph);
            relayout_region(sw, lane);  // (-DIBMG_RELAYOUT=1: to the odd row stride; else nothing)
            TileWW W{sw};
            TileB B{sb};
            for (int pc = 0; pc < 8; ++pc) {
                const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
                if (!((bigmask >> ((li >> 2) + 4 * (lj >> 2))) & 1)) plain_cell(L, W, B, li, lj);
                __syncwarp();
            }
            {
                const int a = lane & 15, h = lane >> 4;
                const int xa = wr(x0 + a, n);
                for (int bb = h; bb < 17; bb += 2) {
                    const size_t gi = xa + (size_t)wr(y0 + bb, n) * n;
                    if (bb < 16) {
                        __stcg(w + gi, W(0, a, bb));
                        __stcg(w + 2 * nn + gi, W(2, a, bb));
                    }
                    __stcg(w + nn + gi, W(1, a, bb));
                }
                if (lane < 16) __stcg(w + wr(x0 + 16, n) + (size_t)wr(y0 + lane, n) * n, W(0, 16, lane));
            }
            __syncwarp();
            if (lane == 0) {
                st_release(tflags + tx + ty * nt, epoch);
                mbar_arrive(&empty[sl]);
            }
        }
    }
}

// ES = false: the double-buffered SlabSlot variant (inverse staged in shared
// memory, 1 CTA per SM).  ES = true: one E'-row slot refilled as soon as a
// block's rows are consumed and the 25 KB inverse streamed from L2 into
// registers (k_big_phase's scheme): 97 KB per CTA, 2 CTAs (two big blocks and
// 8 tile warps in flight) per SM.  Same arithmetic, bitwise identical results.
constexpr size_t kDfTileStride = (kDfTileBytes + 15) / 16 * 16;
constexpr size_t kDfSmemES = sizeof(ESlot) + kDfWarps * kDfTileStride;
template <bool ES>
__global__ void __launch_bounds__(32 * kDfWarps, ES ? 2 : 1) k_sweep_df(DfArgs A) {
    pdl_enter();
    extern __shared__ __align__(16) unsigned char dsm[];
    SlabSlot* slot = reinterpret_cast<SlabSlot*>(dsm);
    ESlot* eslot = reinterpret_cast<ESlot*>(dsm);
    __shared__ BigScratch S;
    const Lev& L = A.L;
    const int n = L.n, nn = L.nn, t = threadIdx.x, wid = t >> 5, G = gridDim.x;
    const int nt = n / kTile, ntiles = nt * nt, per = ntiles / 4, half = nt >> 1, nbk = n >> 2;
    double* sw = reinterpret_cast<double*>(dsm + (ES ? sizeof(ESlot) : 2 * sizeof(SlabSlot)) + wid * kDfTileStride);
    double* sb = sw + kDfWDoubles;
    const unsigned epoch = A.DP.epoch;
    // first big slab streams in while the plain tasks run
    int c = 0, q = -1;
    auto next_item = [&](int cc, int qq, int& nc, int& nq) {
        nq = (cc < 0) ? -1 : qq + G;
        nc = (cc < 0) ? 0 : cc;
        while (nc < A.BC.ncol) {
            if (nq < 0) nq = A.BC.off[nc] + (int)blockIdx.x;
            if (nq < A.BC.off[nc + 1]) return;
            ++nc;
            nq = -1;
        }
    };
    next_item(-1, 0, c, q);
    if (c < A.BC.ncol) {
        if (ES) eslot_issue(*eslot, A.SL, q, t, 32 * kDfWarps);
        else slab_issue(slot[0], A.SL, q, t, 32 * kDfWarps);
    }
    cp_async_commit();
    // ---- plain tasks: warp per tile, tile-colour-major order
    for (int task = blockIdx.x * kDfWarps + wid; task < ntiles; task += G * kDfWarps) {
        const int tc = task / per, i = task % per;
        df_plain_tile(L, A.b, A.w, A.big, A.tflags, epoch, 2 * (i % half) + (tc & 1), 2 * (i / half) + (tc >> 1), tc,
                      sw, sb, A.trace ? A.trace + 6 * task : nullptr);
    }
    __syncthreads();
    // ---- big tasks: CTA per block, colour order
    GAccCG Wg{A.w, n, nn};
    GAccB Bg{A.b, n, nn};
    int k = 0;
    while (c < A.BC.ncol) {
        int nc, nq;
        next_item(c, q, nc, nq);
        if (!ES) {
            if (nc < A.BC.ncol) slab_issue(slot[(k + 1) & 1], A.SL, nq, t, 32 * kDfWarps);
            cp_async_commit();
        }
        const int Bk = A.SL.rp[(size_t)q * 48 + 47];
        const int bi = 4 * (Bk % nbk), bj = 4 * (Bk / nbk);
        const unsigned long long t_a = A.trace ? gtimer() : 0;
        for (int e = A.DP.poff[q] + t; e < A.DP.poff[q + 1]; e += 32 * kDfWarps)
            while (ld_acquire(A.DP.flags + A.DP.pred[e]) != epoch) __nanosleep(8);
        if (t < 9) {  // plain tiles within 8 cells of the block
            const int tx0 = (bi - 8) >> 4, ty0 = (bj - 8) >> 4;
            const int tx = tx0 + t % 3, ty = ty0 + t / 3;
            if (tx * kTile <= bi + 11 && ty * kTile <= bj + 11)
                while (ld_acquire(A.tflags + wr(tx, nt) + wr(ty, nt) * nt) != epoch) __nanosleep(8);
        }
        __syncthreads();
        const unsigned long long t_b = A.trace ? gtimer() : 0;
        if (ES) cp_async_wait<0>();
        else cp_async_wait<1>();
        __syncthreads();
        const unsigned long long t_c = A.trace ? gtimer() : 0;
        auto wadd = [&](int f, int i, int j, double old, double d) {
            __stcg(A.w + (size_t)f * nn + i + (size_t)j * n, old + d);
        };
        if (ES) {
            big_block_es<0>(L, *eslot, A.SL.Ainv + (size_t)q * 3136, bi, bj, Wg, FlatCG{A.w}, Bg, wadd, S, t,
                            [] { __syncthreads(); },
                            [&] {
                                if (nc < A.BC.ncol) eslot_issue(*eslot, A.SL, nq, t, 32 * kDfWarps);
                                cp_async_commit();
                            },
                            nullptr, nullptr, SlabTail{&A.SL, q});
        } else {
            unsigned long long* dbgp = A.trace ? A.trace + 6 * ntiles + 9 * q + 6 : nullptr;
            big_block_slab(L, slot[k & 1], bi, bj, Wg, FlatCG{A.w}, FlatCG{A.w}, Bg, wadd, S, t, dbgp,
                           SlabTail{&A.SL, q});
        }
        __syncthreads();
        if (t == 0) {  // bar.sync + st.release.gpu order the CTA's w stores before the flag
            st_release(A.DP.flags + q, epoch);
            if (A.trace) {
                unsigned long long* r = A.trace + 6 * ntiles + 9 * q;
                r[0] = t_a;
                r[1] = t_b;
                r[2] = t_c;
                r[3] = gtimer();
                r[4] = c;
                r[5] = blockIdx.x;
            }
        }
        ++k;
        c = nc;
        q = nq;
    }
    cp_async_wait<0>();
}

// ---- setup: dense local matrices and their inverses --------------------------

// Dense local inverses: the m x m matrix is assembled in shared memory (row
// stride m + 1, odd: a warp's per-row accesses hit distinct banks) and
// inverted by gauss_jordan below.
__host__ __device__ constexpr int gj_ld(int m) { return m + 1; }

__device__ void gauss_jordan(const double* __restrict__ M, int m, double* __restrict__ out, int* err) {
    // Gauss-Jordan with partial pivoting on [A | I], register-resident: thread
    // (row r = t & 63, quarter cq = t >> 6) holds columns [cq Q, cq Q + Q) of
    // row r, Q = ceil(2m / 4) <= 28.  Rows are not swapped: step k takes the
    // unused row with the largest |a_rk| (lowest index on ties) as pivot row,
    // scales it by the reciprocal and eliminates column k from every other row
    // (the arithmetic of the row-swapping variant); the inverse's row k is row
    // piv(k) of the right half.  Per step only column k and the pivot row pass
    // through shared memory, double-buffered by step parity: 3 barriers.
    // M: the assembled A (row stride gj_ld(m)); out: inverse, column-major.
    // Requires blockDim = 256, m <= 56.
    constexpr int QMAX = 28;
    __shared__ double colk[2][64];
    __shared__ double prow[2][4 * QMAX];
    __shared__ int used[64], stepof[64];
    __shared__ int sp;
    __shared__ double spv;
    const int ld = gj_ld(m), t = threadIdx.x, r = t & 63, cq = t >> 6;
    const int Q = (2 * m + 3) / 4, c0 = cq * Q;
    const bool active = r < m;
    double a[QMAX];
#pragma unroll
    for (int j = 0; j < QMAX; ++j) {
        const int c = c0 + j;
        a[j] = (!active || j >= Q || c >= 2 * m) ? 0.0 : (c < m ? M[r * ld + c] : (c - m == r ? 1.0 : 0.0));
    }
    if (t < 64) used[t] = 0;
    __syncthreads();
    for (int k = 0; k < m; ++k) {
        const int b = k & 1, kq = k / Q, kj = k - kq * Q;
        if (active && cq == kq) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < QMAX; ++j)
                if (j == kj) v = a[j];
            colk[b][r] = v;
        }
        __syncthreads();
        if (t < 32) {
            double best = -1.0;
            int bi = 64;
            for (int i = t; i < m; i += 32) {
                const double v = fabs(colk[b][i]);
                if (!used[i] && v > best) {
                    best = v;
                    bi = i;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) {
                    best = ob;
                    bi = oi;
                }
            }
            if (t == 0) {
                sp = bi;
                spv = bi < m ? colk[b][bi] : 0.0;
                if (bi < m) {
                    used[bi] = 1;
                    stepof[bi] = k;
                }
            }
        }
        __syncthreads();
        const int p = sp;
        const double pv = spv;
        if (pv == 0.0) {
            if (t == 0) atomicOr(err, 2);
            return;
        }
        if (active && r == p) {
            const double ipv = 1.0 / pv;
#pragma unroll
            for (int j = 0; j < QMAX; ++j) {
                a[j] *= ipv;
                if (j < Q) prow[b][c0 + j] = a[j];
            }
        }
        __syncthreads();
        if (active && r != p) {
            const double f = colk[b][r];
#pragma unroll
            for (int j = 0; j < QMAX; ++j)
                if (j < Q) a[j] -= f * prow[b][c0 + j];
        }
    }
    if (active) {
        const int k = stepof[r];
#pragma unroll
        for (int j = 0; j < QMAX; ++j) {
            const int c = c0 + j;
            if (j < Q && c >= m && c < 2 * m) out[(size_t)(c - m) * m + k] = a[j];
        }
    }
}

// Stokes entries of row r of a box, emitted as (field, da, db, value) with da,
// db the column offset relative to the row's own (i, j).
template <class Emit>
__device__ __forceinline__ void stokes_row_entries(const Lev& L, int field, Emit&& emit) {
    const double d = L.d, c = L.c, g = L.g;
    if (field == 0) {
        emit(0, 0, 0, d); emit(0, -1, 0, -c); emit(0, 1, 0, -c); emit(0, 0, -1, -c); emit(0, 0, 1, -c);
        emit(2, 0, 0, g); emit(2, -1, 0, -g);
    } else if (field == 1) {
        emit(1, 0, 0, d); emit(1, 0, -1, -c); emit(1, 0, 1, -c); emit(1, -1, 0, -c); emit(1, 1, 0, -c);
        emit(2, 0, 0, g); emit(2, 0, -1, -g);
    } else {
        emit(0, 1, 0, -g); emit(0, 0, 0, g); emit(1, 0, 1, -g); emit(1, 0, 0, g);
    }
}

// One CTA per big block: assemble the 56x56 principal submatrix of A_l on the
// block DOFs, invert it, store the inverse column-major.
struct BInvLevels {
    Lev L[20];
    EMat E[20];
    const int* blk_ids[20];
    const int2* rr[20];
    double* Ainv[20];
    int start[21];
    int nlev;
    int bylo[20], byhi[20];  // block rows to invert (a slab's own rows; 0, n/4 = all)
};

// In-place Gauss-Jordan with partial pivoting, register-resident: 64 threads,
// thread t < 56 holds row t of the 56 x 56 matrix.  Step k takes the unused
// row with the largest |a_rk| (to 14 mantissa bits; lowest index on ties) as
// pivot row p, scales it
// (a_pk <- 1 / a_pk) and eliminates column k from every other row
// (a_rk <- -a_rk / a_pk): the in-place inversion of the row-permuted matrix,
// with no row moved.  Steps run in rounds of 8 with the pivot column at a
// static register index, and the register row rotates by 8 columns per round
// (no dynamic register indexing, a short loop): after 56 steps every column
// is back in place.  Per step: a warp argmax, two 64-thread barriers, the
// unscaled pivot row through shared memory (every thread scales its own
// update by f / a_pk); the pivot search is one warp max-reduce (redux) of a
// packed magnitude / row key per warp.
// 2 warps and ~150 registers per matrix: ~7 matrices in flight per SM, where
// the 256-thread [A | I] form (gauss_jordan) is barrier-bound at 3.
// M: the assembled A (row stride gj_ld(56)); out: inverse, column-major.
// mo <= 56: the matrix is the leading mo x mo block of M, padded with the
// identity (block-diagonal: the padding never pivots for the first mo columns
// and stays apart); out gets the mo x mo inverse, column-major with ld mo.
__device__ __forceinline__ void gauss_jordan56_regs(const double* __restrict__ M, double* __restrict__ out, int* err,
                                                    int mo = 56) {
    constexpr int m = 56, LD = gj_ld(56);
    __shared__ double prow[m];  // the pivot row, unscaled
    __shared__ double pinv;
    __shared__ int cand_i[2];
    __shared__ int stepof[64], pivrow[m];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const bool act = t < m;
    double a[m];
#pragma unroll
    for (int c = 0; c < m; ++c) a[c] = !act ? 0.0 : (t < mo && c < mo) ? M[t * LD + c] : (c == t ? 1.0 : 0.0);
    bool used = !act;
    // 7 rounds of 8 steps: inside a round the pivot column is a[s] (static),
    // after it the row rotates by 8 columns
    for (int k8 = 0; k8 < m / 8; ++k8) {
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            // pivot key: the high word of |a_rk| (sign, exponent, 20 mantissa bits:
            // monotone in |a_rk|) with its 6 low bits replaced by 63 - row, so
            // one integer max picks the largest magnitude (to 14 mantissa bits)
            // and the lowest row on ties; used rows bid 0
            const unsigned hi = (unsigned)(__double_as_longlong(fabs(a[s])) >> 32);
            const unsigned key = used ? 0u : ((hi & ~63u) | unsigned(63 - t));
            const unsigned wmax = __reduce_max_sync(0xffffffffu, key);
            if (lane == 0) cand_i[wid] = (int)wmax;
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const unsigned best = max((unsigned)cand_i[0], (unsigned)cand_i[1]);
            const int p = 63 - int(best & 63u);
            if ((best >> 6) == 0u) {  // no nonzero pivot left: singular
                if (t == 0) atomicOr(err, 2);
                return;
            }
            if (t == p) {
#pragma unroll
                for (int c = 0; c < m; ++c) prow[c] = a[c];
                pinv = 1.0 / a[s];
                used = true;
                stepof[t] = 8 * k8 + s;
                pivrow[8 * k8 + s] = t;
            }
            asm volatile("bar.sync 1, 64;" ::: "memory");
            const double inv = pinv;
            if (t == p) {
#pragma unroll
                for (int c = 0; c < m; ++c)
                    if (c != s) a[c] *= inv;
                a[s] = inv;
            } else if (act) {
                const double g = a[s] * inv;
#pragma unroll
                for (int c = 0; c < m; ++c)
                    if (c != s) a[c] -= g * prow[c];
                a[s] = -g;
            }
        }
        double r8[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) r8[c] = a[c];
#pragma unroll
        for (int c = 0; c + 8 < m; ++c) a[c] = a[c + 8];
#pragma unroll
        for (int c = 0; c < 8; ++c) a[m - 8 + c] = r8[c];
    }
    asm volatile("bar.sync 1, 64;" ::: "memory");
    // A^{-1}[r][c] = X[pivrow[r]][stepof[c]]: the thread of physical row q
    // (r = stepof[q]) writes column pivrow[j] of the inverse from its a[j]
    if (act) {
        const int r = stepof[t];
        if (r < mo) {
#pragma unroll
            for (int j = 0; j < m; ++j)
                if (j < mo) out[(size_t)pivrow[j] * mo + r] = a[j];
        }
    }
}

// Assemble the 56x56 box matrix of block B into M (shared, row stride
// gj_ld(56)) from the Stokes rows and the E' rows (rr40: the 40 velocity rows'
// ranges in E); any block size (64 threads for the register inverse).
__device__ __forceinline__ void box_assemble(const Lev& L, const EMat& E, const int2* __restrict__ rr40, int B,
                                             double* M) {
    const int t = threadIdx.x, nt = blockDim.x, n = L.n, nbk = n >> 2;
    const int bi = 4 * (B % nbk), bj = 4 * (B / nbk);
    constexpr int LD = gj_ld(56);
    for (int idx = t; idx < 56 * LD; idx += nt) M[idx] = 0.0;
    __syncthreads();
    if (t < 56) {
        int f, i, j;
        block_dof(t, bi, bj, f, i, j);
        const int a = i - bi, bb = j - bj;
        stokes_row_entries(L, f, [&](int f2, int da, int db, double v) {
            const int c = block_local(f2, a + da, bb + db);
            if (c >= 0) M[t * LD + c] += v;
        });
    }
    __syncthreads();
    // E' rows: the 40 rows' entries as one flattened range (row starts in
    // shared memory), 8 independent loads in flight per thread (the entries of
    // a row map to distinct local columns: every M element has one writer)
    __shared__ int rs[41];
    __shared__ int2 rrs[40];
    if (t < 40) rrs[t] = rr40[t];
    __syncthreads();
    if (t == 0) {
        int acc = 0;
        for (int r = 0; r < 40; ++r) {
            rs[r] = acc;
            acc += rrs[r].y - rrs[r].x;
        }
        rs[40] = acc;
    }
    __syncthreads();
    const int tot = rs[40];
    for (int e0 = t; e0 < tot; e0 += 8 * nt) {
        int row[8], idx[8], cidx[8];
        double val[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * nt;
            int lo = 0, hi = 40;  // last row with rs[row] <= e
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (rs[mid] <= e) lo = mid; else hi = mid;
            }
            row[u] = e < tot ? lo : -1;
            idx[u] = e < tot ? rrs[lo].x + (e - rs[lo]) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            cidx[u] = row[u] >= 0 ? __ldg(E.col + idx[u]) : 0;
            val[u] = row[u] >= 0 ? __ldg(E.val + idx[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (row[u] < 0) continue;
            const int comp = cidx[u] >= L.nn, f2 = cidx[u] - comp * L.nn;
            const int c = block_local(comp, wr((f2 & (n - 1)) - bi, n), wr(f2 / n - bj, n));
            if (c >= 0) M[row[u] * LD + c] -= val[u];
        }
    }
    __syncthreads();
}

// Assemble the 56x56 box matrix of block B (cell-block index, n/4 per row)
// from the Stokes rows and the E' rows (rr40: the 40 velocity rows' ranges in
// E) into M, and invert it into out (column-major).  256 threads.
__device__ __forceinline__ void box_inverse(const Lev& L, const EMat& E, const int2* __restrict__ rr40, int B,
                                            double* __restrict__ out, int* err, double* M) {
    const int t = threadIdx.x, nt = blockDim.x, n = L.n, nbk = n >> 2;
    const int bi = 4 * (B % nbk), bj = 4 * (B / nbk);
    constexpr int LD = gj_ld(56);
    for (int idx = t; idx < 56 * LD; idx += nt) M[idx] = 0.0;
    __syncthreads();
    if (t < 56) {
        int f, i, j;
        block_dof(t, bi, bj, f, i, j);
        const int a = i - bi, bb = j - bj;
        stokes_row_entries(L, f, [&](int f2, int da, int db, double v) {
            const int c = block_local(f2, a + da, bb + db);
            if (c >= 0) M[t * LD + c] += v;
        });
    }
    __syncthreads();
    // E' rows: one warp per row, the lanes over its entries (the entries of a
    // row map to distinct local columns, so every M element has one writer);
    // a thread-per-row loop made the box build latency-bound on the row length
    for (int row = t >> 5; row < 40; row += nt >> 5) {
        const int2 r = rr40[row];
        for (int e = r.x + (t & 31); e < r.y; e += 32) {
            const int cidx = E.col[e], comp = cidx >= L.nn, f2 = cidx - comp * L.nn;
            const int c = block_local(comp, wr((f2 & (n - 1)) - bi, n), wr(f2 / n - bj, n));
            if (c >= 0) M[row * LD + c] -= E.val[e];
        }
    }
    __syncthreads();
    gauss_jordan(M, 56, out, err);
    __syncthreads();
}

// RG = true: 64-thread CTAs, register Gauss-Jordan (default); false: 256
// threads, gauss_jordan (IBMG_GJ256=1).
template <bool RG>
__global__ void __launch_bounds__(RG ? 64 : 256, RG ? 4 : 1) k_block_inverse(BInvLevels BL, int* err) {
    pdl_enter();
    extern __shared__ double M[];  // 56 x gj_ld(56)
    int lv = 0;
    while (lv + 1 < BL.nlev && (int)blockIdx.x >= BL.start[lv + 1]) ++lv;
    const int q = blockIdx.x - BL.start[lv], nbk = BL.L[lv].n >> 2;
    const int B = BL.blk_ids[lv][q];
    if (B / nbk < BL.bylo[lv] || B / nbk >= BL.byhi[lv]) return;  // another slab's block
    if (RG) {
        box_assemble(BL.L[lv], BL.E[lv], BL.rr[lv] + (size_t)q * 40, B, M);
        gauss_jordan56_regs(M, BL.Ainv[lv] + (size_t)q * 3136, err);
    } else {
        box_inverse(BL.L[lv], BL.E[lv], BL.rr[lv] + (size_t)q * 40, B, BL.Ainv[lv] + (size_t)q * 3136, err, M);
    }
}

// Coarsest level (n = 4): dense bordered operator [A e; e^T 0] (mean-zero
// pressure constraint), 49 x 49, inverted; stored col-major.
template <bool RG>
__global__ void __launch_bounds__(RG ? 64 : 256) k_coarse_inverse(Lev L, FaceList FL, EMat E, double* __restrict__ Ainv,
                                                                   int* err) {
    pdl_enter();
    extern __shared__ double M[];
    const int n = L.n, nn = L.nn, m = 3 * nn + 1, ld = RG ? gj_ld(56) : gj_ld(m), t = threadIdx.x, nt = blockDim.x;
    for (int idx = t; idx < m * ld; idx += nt) M[idx] = 0.0;
    __syncthreads();
    if (t < 3 * nn) {
        const int f = t / nn, i = (t % nn) % n, j = (t % nn) / n;
        stokes_row_entries(L, f, [&](int f2, int da, int db, double v) {
            M[t * ld + f2 * nn + wr(i + da, n) + wr(j + db, n) * n] += v;
        });
        if (f == 2) {
            M[t * ld + 3 * nn] = 1.0;
            M[3 * nn * ld + t] = 1.0;
        }
    }
    __syncthreads();
    for (int q = t; q < FL.nf; q += nt) {
        const int r = FL.face[q];
        for (int e = E.rp[q]; e < E.rp[q + 1]; ++e) M[r * ld + E.col[e]] -= E.val[e];
    }
    __syncthreads();
    if (RG) gauss_jordan56_regs(M, Ainv, err, m);  // m = 49 <= 56: identity-padded
    else gauss_jordan(M, m, Ainv, err);
}

// E' row range (begin, end) of each of the 40 velocity DOFs of every big block
// ((0, 0) if the face has no E' row), and the block -> list position map bq.
// Big-block setup for every level with big blocks in one launch each
// (DESIGN.md §3.4): blocks are numbered level-major, start[] the prefix.
constexpr int kBSLevels = 16;
struct BSetup {
    int nlev;
    int lev[kBSLevels];  // level index (counters)
    Lev L[kBSLevels];
    FaceList FL[kBSLevels];
    EMat E[kBSLevels];
    const int* blk_ids[kBSLevels];
    int2* rr[kBSLevels];
    int* bq[kBSLevels];
    int* sl_rp[kBSLevels];
    int start[kBSLevels + 1];
};
__device__ __forceinline__ int bs_level(const BSetup& S, int qg) {
    int k = 0;
    while (qg >= S.start[k + 1]) ++k;
    return k;
}

// E' row range of velocity DOF t (0..39) of block B (binary search of the
// face list; (0, 0) for faces without an E' row).
__device__ __forceinline__ int2 block_row_range(const Lev& L, const FaceList& FL, const EMat& E, int B, int t) {
    const int n = L.n, nbk = n >> 2;
    int f, i, j;
    block_dof(t, 4 * (B % nbk), 4 * (B / nbk), f, i, j);
    const int key = f * L.nn + wr(i, n) + wr(j, n) * n;
    int lo = 0, hi = FL.nf;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (FL.face[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < FL.nf && FL.face[lo] == key) ? make_int2(E.rp[lo], E.rp[lo + 1]) : make_int2(0, 0);
}

// E' row ranges of the 40 velocity DOFs of every block.
__global__ void k_block_rows(BSetup S) {
    pdl_enter();
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= S.start[S.nlev] * 40) return;
    const int qg = idx / 40, t = idx % 40, k = bs_level(S, qg), q = qg - S.start[k];
    const int B = S.blk_ids[k][q];
    if (t == 0) S.bq[k][B] = q;
    S.rr[k][(size_t)q * 40 + t] = block_row_range(S.L[k], S.FL[k], S.E[k], B, t);
}

// ---- box inverses in canonical (block-id) order, before the colouring -------
// The inverse of a big block does not depend on its colour: the canonical
// pass numbers the big blocks of all levels in level-major block-id order
// (a scan of the conflict masks; the colouring's vertex order), assembles
// their E' row ranges and inverts them while the host colours the blocks.
// k_ainv_permute then moves each inverse to its colour-sorted list position.
struct CanonInv {
    int nlev;        // levels with blocks (all but the coarsest)
    int boff[21];    // level offsets in the level-major block numbering
    Lev L[20];
    FaceList FL[20];
    EMat E[20];
    const int* ids;    // canonical index -> level-major block index
    const int* total;  // device: number of big blocks, all levels
    int2* rr;          // [cap][40]
    double* Ainv;      // [cap][3136]
    int cap;
};
__device__ __forceinline__ int canon_level(const CanonInv& C, int e) {
    int l = 0;
    while (l + 1 < C.nlev && e >= C.boff[l + 1]) ++l;
    return l;
}
__global__ void k_canon_flags(const unsigned* __restrict__ cm, int nb, int* __restrict__ flag) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nb) flag[i] = cm[i] != 0u;
}
__global__ void k_canon_list(const unsigned* __restrict__ cm, int nb, const int* __restrict__ rank,
                             int* __restrict__ ids, int* __restrict__ total) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb) return;
    if (cm[i]) ids[rank[i]] = i;
    if (i == nb - 1) *total = rank[i] + (cm[i] != 0u);
}
__global__ void k_canon_rows(CanonInv C) {
    pdl_enter();
    const long tot = (long)min(*C.total, C.cap) * 40;
    for (long idx = (long)blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += (long)gridDim.x * blockDim.x) {
        const int g = int(idx / 40), t = int(idx % 40), e = C.ids[g], l = canon_level(C, e);
        C.rr[idx] = block_row_range(C.L[l], C.FL[l], C.E[l], e - C.boff[l], t);
    }
}
// one CTA per canonical block; the grid is the buffer capacity (>= the block
// count of the previous step), CTAs past the current count exit
template <bool RG>
__global__ void __launch_bounds__(RG ? 64 : 256, RG ? 4 : 1) k_canon_inverse(CanonInv C, int* err) {
    pdl_enter();
    extern __shared__ double M[];
    const int g = blockIdx.x;
    if (g >= min(*C.total, C.cap)) return;
    const int e = C.ids[g], l = canon_level(C, e);
    if (RG) {
        box_assemble(C.L[l], C.E[l], C.rr + (size_t)g * 40, e - C.boff[l], M);
        gauss_jordan56_regs(M, C.Ainv + (size_t)g * 3136, err);
    } else {
        box_inverse(C.L[l], C.E[l], C.rr + (size_t)g * 40, e - C.boff[l], C.Ainv + (size_t)g * 3136, err, M);
    }
}
struct APerm {
    int nlev;
    int boff[kBSLevels];  // level-major offset of each listed level
    const int* blk_ids[kBSLevels];
    double* Ainv[kBSLevels];
    int start[kBSLevels + 1];
};
// Ainv[level][q] = canonical inverse of list position q's block (256 threads
// per inverse, 16-byte copies).
__global__ void k_ainv_permute(APerm P, const int* __restrict__ rank, const double* __restrict__ Ac) {
    pdl_enter();
    for (int qg = blockIdx.x; qg < P.start[P.nlev]; qg += gridDim.x) {
        int k = 0;
        while (qg >= P.start[k + 1]) ++k;
        const int q = qg - P.start[k];
        const int g = rank[P.boff[k] + P.blk_ids[k][q]];
        const double2* src = reinterpret_cast<const double2*>(Ac + (size_t)g * 3136);
        double2* dst = reinterpret_cast<double2*>(P.Ainv[k] + (size_t)q * 3136);
        for (int i = threadIdx.x; i < 3136 / 2; i += blockDim.x) dst[i] = __ldcs(src + i);
    }
}

// Slab packing: row pointers + padded entry counts (cnt, level-major), the
// owner block id in rp[47]; the longest slab per level into counter 19.
__global__ void k_slab_count(BSetup S, int* __restrict__ cnt, int* __restrict__ counters, int ctr_stride) {
    pdl_enter();
    const int qg = blockIdx.x * blockDim.x + threadIdx.x;
    if (qg >= S.start[S.nlev]) return;
    const int k = bs_level(S, qg), q = qg - S.start[k];
    const int2* rr = S.rr[k];
    int* rp = S.sl_rp[k];
    int rel = 0;
    for (int t = 0; t < 40; ++t) {
        rp[(size_t)q * 48 + t] = rel;
        const int2 r = rr[(size_t)q * 40 + t];
        rel += r.y - r.x;
    }
    for (int t = 40; t < 47; ++t) rp[(size_t)q * 48 + t] = rel;
    rp[(size_t)q * 48 + 47] = S.blk_ids[k][q];  // owner block id (used by the coarse kernel)
    cnt[qg] = (rel + 3) & ~3;
    atomicMax(counters + S.lev[k] * ctr_stride + 19, rel);
}

// The entries, at off[qg] (level-major offsets), columns as flat indices: one
// warp per (block, row), the lanes over the row's entries (coalesced; rows of
// the coarse Galerkin levels run to hundreds of entries).
__global__ void k_slab_fill(BSetup S, const int* __restrict__ off, int* __restrict__ col, double* __restrict__ val) {
    pdl_enter();
    const long idx = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (idx >= (long)S.start[S.nlev] * 40) return;
    const int qg = int(idx / 40), t = int(idx % 40), k = bs_level(S, qg), q = qg - S.start[k];
    const int2 r = S.rr[k][idx - (long)S.start[k] * 40];
    const EMat& E = S.E[k];
    const int o = off[qg] + S.sl_rp[k][(size_t)q * 48 + t] - r.x;
    for (int e = r.x + lane; e < r.y; e += 32) {
        col[o + e] = E.col[e];
        val[o + e] = E.val[e];
    }
}

}  // namespace ibmg
