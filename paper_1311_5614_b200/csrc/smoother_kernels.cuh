// smoother_kernels.cuh — multicolour box relaxation (the paper's generalised
// Vanka / big-box smoother) and the coarse-level kernels.
//
// Schedule (mirrored exactly by oracle/ibmg_oracle.cpp
// build_schedule): plain phase = 16x16-cell tiles coloured 2x2 (one launch per
// tile colour, one warp per tile, the 8 conflict-free colours (i+2j) mod 8 run
// in shared memory); big phase = big 4x4 blocks in 16 level-wide colours
// (bx mod 4, by mod 4), one CTA per block, dense 56x56 inverse applied.
#pragma once
#include "common.cuh"
#include "grid_kernels.cuh"

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

// ---- plain phase, multi-tile levels (n >= 32): one warp per 16x16 tile.
constexpr int kTile = 16, kReg = kTile + 4;  // region with a 2-cell halo

struct TileW {
    double* s;  // [3][kReg][kReg], local coords li, lj in [-2, 18)
    __device__ __forceinline__ double& operator()(int f, int i, int j) const {
        return s[f * kReg * kReg + (j + 2) * kReg + (i + 2)];
    }
};
struct TileB {
    const double* s;  // [3][17][17], local coords in [0, 17)
    __device__ __forceinline__ double operator()(int f, int i, int j) const { return s[f * 289 + j * 17 + i]; }
};

__global__ void __launch_bounds__(32) k_plain_tiles(Lev L, int tc, const double* __restrict__ b,
                                                     double* __restrict__ w, const uint8_t* __restrict__ big) {
    __shared__ double sw[3 * kReg * kReg];
    __shared__ double sb[3 * 289];
    __shared__ uint8_t sbig[16];
    const int n = L.n, nn = L.nn, lane = threadIdx.x;
    const int half = (n / kTile) >> 1;
    const int tx = 2 * (blockIdx.x % half) + (tc & 1), ty = 2 * (blockIdx.x / half) + (tc >> 1);
    const int x0 = tx * kTile, y0 = ty * kTile;
    for (int q = lane; q < kReg * kReg; q += 32) {
        const int a = q % kReg, bb = q / kReg;
        const size_t gi = wr(x0 - 2 + a, n) + (size_t)wr(y0 - 2 + bb, n) * n;
        cp_async8(&sw[q], w + gi);
        cp_async8(&sw[kReg * kReg + q], w + nn + gi);
        cp_async8(&sw[2 * kReg * kReg + q], w + 2 * nn + gi);
    }
    for (int q = lane; q < 289; q += 32) {
        const int a = q % 17, bb = q / 17;
        const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
        cp_async8(&sb[q], b + gi);
        cp_async8(&sb[289 + q], b + nn + gi);
        cp_async8(&sb[578 + q], b + 2 * nn + gi);
    }
    if (lane < 16) sbig[lane] = big[(x0 >> 2) + (lane & 3) + ((y0 >> 2) + (lane >> 2)) * (n >> 2)];
    cp_async_wait_all();
    __syncwarp();
    TileW W{sw};
    TileB B{sb};
    for (int pc = 0; pc < 8; ++pc) {
        const int lj = lane >> 1, li = ((pc - 2 * lj) & 7) + 8 * (lane & 1);
        if (!sbig[(li >> 2) + 4 * (lj >> 2)]) plain_cell(L, W, B, li, lj);
        __syncwarp();
    }
    // write set: u faces i in [x0, x0+16], v faces j in [y0, y0+16], p cells
    for (int q = lane; q < 17 * 17; q += 32) {
        const int a = q % 17, bb = q / 17;
        const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
        if (bb < 16) w[gi] = W(0, a, bb);
        if (a < 16) w[nn + gi] = W(1, a, bb);
        if (a < 16 && bb < 16) w[2 * nn + gi] = W(2, a, bb);
    }
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

// One big-block relaxation by a group of 128 threads (4 warps).  Latency
// structure (the routine is a handful of dependent memory rounds):
//  (1) Stokes residual of the 56 DOFs and, in parallel, the E' row dots of the
//      40 velocity DOFs (warp per row, lanes over nonzeros; all (col, val)
//      loads of 5 rows issued before the dependent w gathers);
//  (2) the 56x56 inverse applied by 112 threads (2 column halves, loads
//      prefetched 14 at a time), reduced in a fixed order (deterministic).
// `gsync` is the group barrier (__syncthreads or a named barrier).
constexpr int kGroup = 128;
struct BigScratch {
    double sr[56], se[40], part[2][56];
};

template <class Acc, class Flat, class BAcc, class WAdd, class Sync>
__device__ __forceinline__ void big_block_group(const Lev& L, const EMat& E, const int2* __restrict__ rr_q,
                                                const double* __restrict__ A_q, int bi, int bj, const Acc& acc,
                                                const Flat& flat, const BAcc& bacc, WAdd&& wadd, BigScratch& S,
                                                int gt, Sync&& gsync) {
    const int wid = gt >> 5, lane = gt & 31;
    // inverse columns of this thread, issued first (independent of w)
    double av[28];
    const int row = gt % 56, cg = gt / 56;
    if (gt < 112) {
        const double* A = A_q + (size_t)(28 * cg) * 56 + row;
#pragma unroll
        for (int c = 0; c < 28; ++c) av[c] = A[c * 56];
    }
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        i = wr(i, L.n);
        j = wr(j, L.n);
        double ru, rv, rp;
        stokes_rows(L, acc, i, j, ru, rv, rp);
        S.sr[gt] = bacc(f, i, j) - (f == 0 ? ru : f == 1 ? rv : rp);
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        int beg[5], end[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const int2 r = rr_q[wid + 4 * (5 * half + k)];
            beg[k] = r.x;
            end[k] = r.y;
        }
        int cl[5][2];
        double vl[5][2];
#pragma unroll
        for (int k = 0; k < 5; ++k)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = beg[k] + lane + 32 * h;
                const bool ok = e < end[k];
                cl[k][h] = ok ? E.col[e] : -1;
                vl[k][h] = ok ? E.val[e] : 0.0;
            }
        double ps[5];
#pragma unroll
        for (int k = 0; k < 5; ++k)
            ps[k] = (cl[k][0] >= 0 ? vl[k][0] * flat(cl[k][0]) : 0.0) + (cl[k][1] >= 0 ? vl[k][1] * flat(cl[k][1]) : 0.0);
#pragma unroll
        for (int k = 0; k < 5; ++k)
            for (int e = beg[k] + lane + 64; e < end[k]; e += 32) ps[k] += E.val[e] * flat(E.col[e]);
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            const double v = warp_sum(ps[k]);
            if (lane == 0) S.se[wid + 4 * (5 * half + k)] = v;
        }
    }
    gsync();
    if (gt < 112) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < 28; ++c) {
            const int cc = 28 * cg + c;
            s += av[c] * (cc < 40 ? S.sr[cc] + S.se[cc] : S.sr[cc]);
        }
        S.part[cg][row] = s;
    }
    gsync();
    if (gt < 56) {
        int f, i, j;
        block_dof(gt, bi, bj, f, i, j);
        wadd(f, i, j, S.part[0][gt] + S.part[1][gt]);
    }
}

// One sweep phase of a multi-tile level (n >= 64): one 128-thread CTA per tile
// of tile colour tc.  The 20x20 region (2-cell halo) of w and the tile's b are
// staged in shared memory with cp.async; warp 0 runs the 8 plain colour
// passes; then the whole CTA relaxes the tile's big blocks one by one in local
// order (tile-local big phase); the write set goes back once.
struct TileFlat {  // flat velocity index -> shared region if inside, else global
    const double* s;
    const double* g;
    int n, nn, x0, y0;
    __device__ __forceinline__ double operator()(int idx) const {
        const int comp = idx >= nn, f = idx - comp * nn;
        const int li = wr((f & (n - 1)) - x0 + 2, n), lj = wr(f / n - y0 + 2, n);
        if (li < kReg && lj < kReg) return s[comp * kReg * kReg + lj * kReg + li];
        return g[idx];
    }
};
struct TileGW {  // wrapped global coords -> shared region (all stencil reads are inside)
    double* s;
    int n, x0, y0;
    __device__ __forceinline__ double& operator()(int f, int i, int j) const {
        return s[f * kReg * kReg + wr(j - y0 + 2, n) * kReg + wr(i - x0 + 2, n)];
    }
};
struct TileGB {
    const double* s;
    int n, x0, y0;
    __device__ __forceinline__ double operator()(int f, int i, int j) const {
        return s[f * 289 + wr(j - y0, n) * 17 + wr(i - x0, n)];
    }
};

constexpr int kTileThreads = 128;
__global__ void __launch_bounds__(kTileThreads) k_tile_sweep(Lev L, int tc, const double* __restrict__ b,
                                                              double* __restrict__ w, const uint8_t* __restrict__ big,
                                                              const int* __restrict__ bq, EMat E,
                                                              const int2* __restrict__ rr,
                                                              const double* __restrict__ Ainv) {
    __shared__ double sw[3 * kReg * kReg];
    __shared__ double sb[3 * 289];
    __shared__ int sq[16];
    __shared__ BigScratch S;
    const int n = L.n, nn = L.nn, t = threadIdx.x;
    const int half = (n / kTile) >> 1;
    const int tx = 2 * (blockIdx.x % half) + (tc & 1), ty = 2 * (blockIdx.x / half) + (tc >> 1);
    const int x0 = tx * kTile, y0 = ty * kTile, nbk = n >> 2;
    for (int q = t; q < kReg * kReg; q += kTileThreads) {
        const int a = q % kReg, bb = q / kReg;
        const size_t gi = wr(x0 - 2 + a, n) + (size_t)wr(y0 - 2 + bb, n) * n;
        cp_async8(&sw[q], w + gi);
        cp_async8(&sw[kReg * kReg + q], w + nn + gi);
        cp_async8(&sw[2 * kReg * kReg + q], w + 2 * nn + gi);
    }
    for (int q = t; q < 289; q += kTileThreads) {
        const int a = q % 17, bb = q / 17;
        const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
        cp_async8(&sb[q], b + gi);
        cp_async8(&sb[289 + q], b + nn + gi);
        cp_async8(&sb[578 + q], b + 2 * nn + gi);
    }
    if (t < 16) {
        const int B = (x0 >> 2) + (t & 3) + ((y0 >> 2) + (t >> 2)) * nbk;
        sq[t] = big[B] ? bq[B] : -1;
    }
    cp_async_wait_all();
    __syncthreads();
    if (t < 32) {
        TileW W{sw};
        TileB B{sb};
        for (int pc = 0; pc < 8; ++pc) {
            const int lj = t >> 1, li = ((pc - 2 * lj) & 7) + 8 * (t & 1);
            if (sq[(li >> 2) + 4 * (lj >> 2)] < 0) plain_cell(L, W, B, li, lj);
            __syncwarp();
        }
    }
    __syncthreads();
    TileGW GW{sw, n, x0, y0};
    TileGB GB{sb, n, x0, y0};
    TileFlat FL{sw, w, n, nn, x0, y0};
    for (int lb = 0; lb < 16; ++lb) {
        const int q = sq[lb];
        if (q < 0) continue;
        big_block_group(L, E, rr + (size_t)q * 40, Ainv + (size_t)q * 3136, x0 + 4 * (lb & 3), y0 + 4 * (lb >> 2), GW,
                        FL, GB, [&](int f, int i, int j, double d) { GW(f, i, j) += d; }, S, t,
                        [] { __syncthreads(); });
        __syncthreads();
    }
    for (int q = t; q < 17 * 17; q += kTileThreads) {
        const int a = q % 17, bb = q / 17;
        const size_t gi = wr(x0 + a, n) + (size_t)wr(y0 + bb, n) * n;
        TileW W{sw};
        if (bb < 16) w[gi] = W(0, a, bb);
        if (a < 16) w[nn + gi] = W(1, a, bb);
        if (a < 16 && bb < 16) w[2 * nn + gi] = W(2, a, bb);
    }
}

// ---- setup: dense local matrices and their inverses --------------------------

// Gauss-Jordan with partial pivoting on an m x 2m augmented matrix in shared
// memory (row-major, ld = 2m).  Ties in the pivot search go to the lowest row.
__device__ void gauss_jordan(double* M, int m, double* col, int* err) {
    const int ld = 2 * m, t = threadIdx.x, nt = blockDim.x;
    __shared__ int piv;
    for (int k = 0; k < m; ++k) {
        if (t < 32) {
            double best = -1.0;
            int bi = k;
            for (int i = k + t; i < m; i += 32) {
                const double v = fabs(M[i * ld + k]);
                if (v > best) { best = v; bi = i; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (t == 0) piv = bi;
        }
        __syncthreads();
        const int p = piv;
        if (p != k)
            for (int j = t; j < ld; j += nt) {
                const double a = M[k * ld + j];
                M[k * ld + j] = M[p * ld + j];
                M[p * ld + j] = a;
            }
        __syncthreads();
        const double pv = M[k * ld + k];
        if (pv == 0.0) {
            if (t == 0) atomicOr(err, 2);
            return;
        }
        __syncthreads();
        for (int j = t; j < ld; j += nt) M[k * ld + j] /= pv;
        for (int i = t; i < m; i += nt) col[i] = M[i * ld + k];
        __syncthreads();
        for (int idx = t; idx < m * ld; idx += nt) {
            const int i = idx / ld, j = idx - i * ld;
            if (i != k) M[idx] -= col[i] * M[k * ld + j];
        }
        __syncthreads();
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
__global__ void k_block_inverse(Lev L, EMat E, const int* __restrict__ blk_ids, const int2* __restrict__ rr,
                                double* __restrict__ Ainv, int* err) {
    extern __shared__ double M[];  // 56 x 112
    __shared__ double col[56];
    const int q = blockIdx.x, t = threadIdx.x, nt = blockDim.x, n = L.n;
    const int B = blk_ids[q], nbk = n >> 2;
    const int bi = 4 * (B % nbk), bj = 4 * (B / nbk);
    for (int idx = t; idx < 56 * 112; idx += nt) {
        const int i = idx / 112, j = idx % 112;
        M[idx] = (j == 56 + i) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (t < 56) {
        int f, i, j;
        block_dof(t, bi, bj, f, i, j);
        const int a = i - bi, bb = j - bj;
        stokes_row_entries(L, f, [&](int f2, int da, int db, double v) {
            const int c = block_local(f2, a + da, bb + db);
            if (c >= 0) M[t * 112 + c] += v;
        });
    }
    __syncthreads();
    if (t < 40) {
        const int2 r = rr[(size_t)q * 40 + t];
        for (int e = r.x; e < r.y; ++e) {
                const int cidx = E.col[e], comp = cidx >= L.nn, f2 = cidx - comp * L.nn;
            const int c = block_local(comp, wr((f2 & (n - 1)) - bi, n), wr(f2 / n - bj, n));
            if (c >= 0) M[t * 112 + c] -= E.val[e];
        }
    }
    __syncthreads();
    gauss_jordan(M, 56, col, err);
    for (int idx = t; idx < 56 * 56; idx += nt) {
        const int c = idx / 56, r = idx % 56;
        Ainv[(size_t)q * 3136 + idx] = M[r * 112 + 56 + c];
    }
}

// Coarsest level (n = 4): dense bordered operator [A e; e^T 0] (mean-zero
// pressure constraint), 49 x 49, inverted; stored col-major.
__global__ void k_coarse_inverse(Lev L, FaceList FL, EMat E, double* __restrict__ Ainv, int* err) {
    extern __shared__ double M[];
    __shared__ double col[64];
    const int n = L.n, nn = L.nn, m = 3 * nn + 1, ld = 2 * m, t = threadIdx.x, nt = blockDim.x;
    for (int idx = t; idx < m * ld; idx += nt) {
        const int i = idx / ld, j = idx % ld;
        M[idx] = (j == m + i) ? 1.0 : 0.0;
    }
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
    gauss_jordan(M, m, col, err);
    for (int idx = t; idx < m * m; idx += nt) {
        const int c = idx / m, r = idx % m;
        Ainv[idx] = M[r * ld + m + c];
    }
}

// E' row range (begin, end) of each of the 40 velocity DOFs of every big block
// ((0, 0) if the face has no E' row), and the block -> list position map bq.
__global__ void k_block_rows(Lev L, FaceList FL, EMat E, const int* __restrict__ blk_ids, int nbig,
                             int2* __restrict__ rr, int* __restrict__ bq) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nbig * 40) return;
    const int q = idx / 40, t = idx % 40, n = L.n, nbk = n >> 2;
    const int B = blk_ids[q];
    if (t == 0) bq[B] = q;
    int f, i, j;
    block_dof(t, 4 * (B % nbk), 4 * (B / nbk), f, i, j);
    const int key = f * L.nn + wr(i, n) + wr(j, n) * n;
    int lo = 0, hi = FL.nf;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (FL.face[mid] < key) lo = mid + 1; else hi = mid;
    }
    rr[idx] = (lo < FL.nf && FL.face[lo] == key) ? make_int2(E.rp[lo], E.rp[lo + 1]) : make_int2(0, 0);
}

// Block sort keys: colour (bx mod 4) + 4 (by mod 4) for big blocks, 16 otherwise.
__global__ void k_block_keys(int nbk, const uint8_t* __restrict__ big, int* keys, int* vals, int* counts) {
    const int B = blockIdx.x * blockDim.x + threadIdx.x;
    if (B >= nbk * nbk) return;
    const int bx = B % nbk, by = B / nbk;
    const int key = big[B] ? (bx & 3) + 4 * (by & 3) : 16;
    keys[B] = key;
    vals[B] = B;
    atomicAdd(&counts[key], 1);
}

}  // namespace ibmg
