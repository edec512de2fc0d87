// grid_kernels.cuh — periodic MAC stencils (operator apply, residual+restrict,
// prolong+add) and the Krylov vector kernels (deterministic reductions).
#pragma once
#include "common.cuh"

namespace ibmg {

// Stokes rows of cell (i, j) against an accessor: returns the u(i,j), v(i,j)
// and p(i,j) rows of S w (negated laplacian_hom + gradient_hom + divergence_hom,
// stokes_ops.cpp:78-130, plus rho/dt; periodic wrap replaces the wall branches).
template <class Acc>
__device__ __forceinline__ void stokes_rows(const Lev& L, const Acc& w, int i, int j, double& ru, double& rv,
                                            double& rp) {
    const int n = L.n;
    const int im = wr(i - 1, n), ip = wr(i + 1, n), jm = wr(j - 1, n), jp = wr(j + 1, n);
    const double uc = w(0, i, j), vc = w(1, i, j), pc = w(2, i, j);
    ru = L.d * uc - L.c * (w(0, im, j) + w(0, ip, j) + w(0, i, jm) + w(0, i, jp)) + L.g * (pc - w(2, im, j));
    rv = L.d * vc - L.c * (w(1, i, jm) + w(1, i, jp) + w(1, im, j) + w(1, ip, j)) + L.g * (pc - w(2, i, jm));
    rp = -L.g * (w(0, ip, j) - uc) - L.g * (w(1, i, jp) - vc);
}

// One Stokes row (field f of cell (i, j)) only: the loads of the other two rows
// are not issued (the box solves need one row per DOF).
template <class Acc>
__device__ __forceinline__ double stokes_row(const Lev& L, const Acc& w, int f, int i, int j) {
    const int n = L.n;
    const int im = wr(i - 1, n), ip = wr(i + 1, n), jm = wr(j - 1, n), jp = wr(j + 1, n);
    if (f == 0)
        return L.d * w(0, i, j) - L.c * (w(0, im, j) + w(0, ip, j) + w(0, i, jm) + w(0, i, jp)) +
               L.g * (w(2, i, j) - w(2, im, j));
    if (f == 1)
        return L.d * w(1, i, j) - L.c * (w(1, i, jm) + w(1, i, jp) + w(1, im, j) + w(1, ip, j)) +
               L.g * (w(2, i, j) - w(2, i, jm));
    return -L.g * (w(0, ip, j) - w(0, i, j)) - L.g * (w(1, i, jp) - w(1, i, j));
}

// Point-force + face-gather CTAs of a grid launch.  A launch
// of K1/K2 is [pf.nblk point CTAs | grid CTAs | G.nblk gather CTAs]:
//  * point CTAs compute F_k = cE_k (U_{k-1} - 2 U_k + U_{k+1}), U_k = R_k . w
//    (elasticity.cpp:62-84 in window form), one warp per point: lane
//    comp * 16 + tap loads one window weight and one field value for each of
//    k-1, k, k+1, then fixed xor-tree sums over the 16 taps (deterministic);
//  * grid CTAs write the stencil part of the output;
//  * gather CTAs wait until every earlier CTA of the launch has signalled a
//    monotone counter (CTAs are dispatched in index order, so waiting only on
//    lower indices always makes progress) and add sign * L_k F_k per face.
// nblk = 0: no point / gather CTAs.
struct PForce {
    Win W;
    Pts P;
    int n;
    const double* w;
    double* F;
    int nblk;
};
struct Gather {
    FaceList FL;
    Win W;
    const double* F;
    double* out;
    int nn;
    double sign;
    int nblk;
    unsigned long long* cnt;    // monotone per-context counter
    unsigned long long target;  // its value once this launch's producers are done
    // slab mode: only faces in rows [jlo, jhi) of the level are
    // gathered (the owned rows of a slab); lg = log2(n)
    int lg = 0, jlo = 0, jhi = 1 << 30;
    int sub = 32;  // lanes per face (8 when every list of the level is <= 32 entries)
    // gather-first launches (fused_launch_gf): the gather CTAs wait for the
    // point-force CTAs only (target_pf) and write sign * sum into `out`, a
    // face scratch; the grid CTAs add it after `target` (all gathers done)
    unsigned long long target_pf = 0;
};
constexpr int kPfPerCta = 8;  // 256-thread CTAs: 8 warps
// Latency-bound chains (origin -> weights / field values -> sum) need several in
// flight per warp: a warp takes kPfPts consecutive points, an 8-lane group of a
// gather CTA kGaFaces consecutive faces, every load of the batch issued before the
// first use (the fused kernels carry the tiles' 30 KB of shared memory and 64
// registers, so only 32 warps per SM are resident: at one chain per warp the C4
// fine level's 222k points and 1.1M faces cost 0.10 + 0.31 ms per apply).
constexpr int kPfPts = 4;
constexpr int kGaFaces = 4;
__host__ __device__ inline int pf_points_per_cta() { return kPfPerCta * kPfPts; }
__host__ __device__ inline int gather_faces_per_cta(int sub) { return sub == 8 ? kPfPerCta * 4 * kGaFaces : kPfPerCta; }

__device__ __forceinline__ void point_force_warp(const PForce& pf, int bid) {
    const int k0 = (bid * kPfPerCta + (threadIdx.x >> 5)) * kPfPts;
    if (k0 >= pf.P.n) return;
    const int lane = threadIdx.x & 31, comp = lane >> 4, e = lane & 15;
    const int n = pf.n;
    const double* wc = pf.w + (size_t)comp * n * n;
    double u[kPfPts][3];
#pragma unroll
    for (int q = 0; q < kPfPts; ++q) {
        const int k = k0 + q < pf.P.n ? k0 + q : pf.P.n - 1;  // clamped: the tail repeats the last point (not stored)
        const int ks[3] = {pf.P.kprev[k], k, pf.P.knext[k]};
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            const int kk = ks[t];
            const int4 o = pf.W.orgR[kk];
            const int i0 = comp ? o.z : o.x, j0 = comp ? o.w : o.y;
            u[q][t] = pf.W.w[(size_t)kk * 64 + (2 + comp) * 16 + e] *
                      __ldg(wc + wr(i0 + (e & 3), n) + (size_t)wr(j0 + (e >> 2), n) * n);
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int q = 0; q < kPfPts; ++q)
#pragma unroll
            for (int t = 0; t < 3; ++t) u[q][t] += __shfl_xor_sync(0xffffffffu, u[q][t], o);
    if (e == 0)
#pragma unroll
        for (int q = 0; q < kPfPts; ++q)
            if (k0 + q < pf.P.n) pf.F[2 * (k0 + q) + comp] = pf.P.cE[k0 + q] * (u[q][0] - 2.0 * u[q][1] + u[q][2]);
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Dispatch of a fused launch; `grid(b)` runs grid CTA b.  bid: this CTA's
// index in the launch (blockIdx.x; the batched kernels pass their own).
template <class GridFn>
__device__ __forceinline__ void fused_launch_at(const PForce& pf, const Gather& G, int ngrid, int bid, GridFn&& grid) {
    if (bid >= pf.nblk + ngrid) {  // gather CTA
        if (threadIdx.x == 0)
            while (ld_acquire_u64(G.cnt) < G.target) __nanosleep(32);
        __syncthreads();
        const int lane = threadIdx.x & 31;
        if (G.sub == 8) {
            const int q = (((bid - pf.nblk - ngrid) * kPfPerCta + (threadIdx.x >> 5)) * 4 + (lane >> 3)) * kGaFaces;
            face_gather_multi<kGaFaces>(G.FL, G.W, G.F, G.out, G.nn, G.sign, q, lane & 7, false, G.lg, G.jlo, G.jhi);
            return;
        }
        const int q = (bid - pf.nblk - ngrid) * kPfPerCta + (threadIdx.x >> 5);
        bool active = q < G.FL.nf;
        if (active && (G.jlo > 0 || G.jhi < (1 << 30))) {
            const int row = (G.FL.face[q] & (G.nn - 1)) >> G.lg;
            active = row >= G.jlo && row < G.jhi;
        }
        face_gather_sub<32>(G.FL, G.W, G.F, G.out, G.nn, G.sign, q, active, lane);
        return;
    }
    if (bid < pf.nblk) point_force_warp(pf, bid);
    else grid(bid - pf.nblk);
    if (G.nblk) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(G.cnt, 1ull);
        }
    }
}
template <class GridFn>
__device__ __forceinline__ void fused_launch(const PForce& pf, const Gather& G, int ngrid, GridFn&& grid) {
    fused_launch_at(pf, G, ngrid, (int)blockIdx.x, grid);
}

// Gather-first dispatch: [point-force CTAs | gather CTAs | grid CTAs].  The
// gathers wait for the point forces only and write sign * L F into the face
// scratch G.out (zero off the face list); the grid CTAs stream their cells
// and, just before storing, wait until every gather has signalled
// (G.target) and add the scratch.  The grid's bandwidth-bound work no longer
// waits for a tail of gathers; every wait is on lower-index CTAs (dispatched
// first), so it always makes progress.  Same values as fused_launch:
// v + sign * s either way.
template <class GridFn>
__device__ __forceinline__ void fused_launch_gf(const PForce& pf, const Gather& G, int ngrid, int bid, GridFn&& grid) {
    if (bid < pf.nblk) {
        point_force_warp(pf, bid);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(G.cnt, 1ull);
        }
        return;
    }
    if (bid < pf.nblk + G.nblk) {
        if (threadIdx.x == 0)
            while (ld_acquire_u64(G.cnt) < G.target_pf) __nanosleep(32);
        __syncthreads();
        const int lane = threadIdx.x & 31;
        if (G.sub == 8) {
            const int q = (((bid - pf.nblk) * kPfPerCta + (threadIdx.x >> 5)) * 4 + (lane >> 3)) * kGaFaces;
            face_gather_multi<kGaFaces>(G.FL, G.W, G.F, G.out, G.nn, G.sign, q, lane & 7, true, 0, 0, 1 << 30);
        } else {
            const int q = (bid - pf.nblk) * kPfPerCta + (threadIdx.x >> 5);
            face_gather_sub<32>(G.FL, G.W, G.F, G.out, G.nn, G.sign, q, q < G.FL.nf, lane, true);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(G.cnt, 1ull);
        }
        return;
    }
    grid(bid - pf.nblk - G.nblk);
}

// A grid thread's wait for every gather of a gather-first launch.
__device__ __forceinline__ void wait_gathers(const Gather& G) {
    if (G.nblk)
        while (ld_acquire_u64(G.cnt) < G.target) __nanosleep(20);
}

// out = S w (E' part added by k_face_gather). K1 of DESIGN.md §4.
// Grid CTAs cover cells [q0, q1) (a slab's owned rows; 0, nn for the level).
__global__ void k_stokes_apply(Lev L, const double* __restrict__ w, double* __restrict__ out, PForce pf, Gather G,
                               int ngrid, int q0, int q1) {
    pdl_enter();
    fused_launch(pf, G, ngrid, [&](int b) {
        const int q = q0 + b * blockDim.x + threadIdx.x;
        if (q >= q1) return;
        const int i = q & (L.n - 1), j = q >> L.lg;
        GAcc acc{w, L.n, L.nn};
        double ru, rv, rp;
        stokes_rows(L, acc, i, j, ru, rv, rp);
        out[q] = ru;
        out[L.nn + q] = rv;
        out[2 * L.nn + q] = rp;
    });
}

__device__ __forceinline__ void rr_cp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// Tiled operator apply for levels with n >= 64 (bandwidth regime; the same
// expressions and term order as stokes_rows).  A grid CTA owns 64 x 16 cells:
// the w region [x0-2, x0+66) x [y0-1, y0+17) of all three fields is staged in
// shared memory with 16-byte cp.async, and each thread forms the 2 x 2 cells
// (x0+2I.., y0+2J..) from double2 shared loads and writes them as double2
// rows (coalesced).  Rows past q1 (slab ends) are skipped.
constexpr int kApTx = 64, kApTy = 16;
constexpr int kApW = kApTx + 4, kApH = kApTy + 2;
struct ApSmem {
    double s[3][kApH][kApW];
};
__device__ __forceinline__ void apply_tile(const Lev& L, const double* __restrict__ w, double* __restrict__ out,
                                           int blk, int q0, int q1, ApSmem& S, const Gather* gf = nullptr) {
    const int n = L.n, nn = L.nn;
    const int ntx = n / kApTx, jb = q0 / n, je = q1 / n;
    const int ty = blk / ntx, tx = blk - ty * ntx;
    const int x0 = tx * kApTx, y0 = jb + ty * kApTy;
    constexpr int kPairs = kApW / 2;
    for (int e = threadIdx.x; e < 3 * kApH * kPairs; e += blockDim.x) {
        const int f = e / (kApH * kPairs), rem = e - f * (kApH * kPairs);
        const int r = rem / kPairs, pc = rem - r * kPairs;
        rr_cp16(&S.s[f][r][2 * pc], w + (size_t)f * nn + wr(x0 - 2 + 2 * pc, n) + (size_t)wr(y0 - 1 + r, n) * n);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    const int I = threadIdx.x & 31, J = threadIdx.x >> 5;
    const int x = x0 + 2 * I, y = y0 + 2 * J;
    if (y >= je) return;
    const double d = L.d, cc = L.c, g = L.g;
    auto ld2 = [&](int f, int r, int c) { return *reinterpret_cast<const double2*>(&S.s[f][r][c]); };
    const int c0 = 2 * I;  // smem column of x - 2; smem row 2J of y - 1
    double u[4][6], p[3][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            const double2 t = ld2(0, 2 * J + k, c0 + 2 * h);
            u[k][2 * h] = t.x;
            u[k][2 * h + 1] = t.y;
        }
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 t = ld2(2, 2 * J + k, c0 + 2 * h);
            p[k][2 * h] = t.x;
            p[k][2 * h + 1] = t.y;
        }
    // cells (ci, k) = (x - 2 + ci, y - 1 + k), ci in 2..3, k in 1..2
    double ru[2][2], rpu[2][2];
#pragma unroll
    for (int k = 1; k <= 2; ++k)
#pragma unroll
        for (int ci = 2; ci <= 3; ++ci) {
            ru[k - 1][ci - 2] = d * u[k][ci] - cc * (u[k][ci - 1] + u[k][ci + 1] + u[k - 1][ci] + u[k + 1][ci]) +
                                g * (p[k][ci] - p[k][ci - 1]);
            rpu[k - 1][ci - 2] = -g * (u[k][ci + 1] - u[k][ci]);
        }
    double v[4][6];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            const double2 t = ld2(1, 2 * J + k, c0 + 2 * h);
            v[k][2 * h] = t.x;
            v[k][2 * h + 1] = t.y;
        }
#pragma unroll
    for (int k = 1; k <= 2; ++k) {
        const int yy = y + k - 1;
        if (yy >= je) break;
        double rv[2], rp[2];
#pragma unroll
        for (int ci = 2; ci <= 3; ++ci) {
            rv[ci - 2] = d * v[k][ci] - cc * (v[k - 1][ci] + v[k + 1][ci] + v[k][ci - 1] + v[k][ci + 1]) +
                         g * (p[k][ci] - p[k - 1][ci]);
            rp[ci - 2] = rpu[k - 1][ci - 2] - g * (v[k + 1][ci] - v[k][ci]);
        }
        const size_t o = x + (size_t)yy * n;
        double2 ou = make_double2(ru[k - 1][0], ru[k - 1][1]), ov = make_double2(rv[0], rv[1]);
        if (gf && gf->nblk) {  // gather-first: + sign * L F from the face scratch
            if (k == 1) wait_gathers(*gf);
            const double2 eu = __ldcg(reinterpret_cast<const double2*>(gf->out + o));
            const double2 ev = __ldcg(reinterpret_cast<const double2*>(gf->out + nn + o));
            ou.x += eu.x;
            ou.y += eu.y;
            ov.x += ev.x;
            ov.y += ev.y;
        }
        *reinterpret_cast<double2*>(out + o) = ou;
        *reinterpret_cast<double2*>(out + nn + o) = ov;
        *reinterpret_cast<double2*>(out + 2 * (size_t)nn + o) = make_double2(rp[0], rp[1]);
    }
}

__global__ void __launch_bounds__(256) k_stokes_apply_t(Lev L, const double* __restrict__ w, double* __restrict__ out,
                                                        PForce pf, Gather G, int ngrid, int q0, int q1) {
    __shared__ __align__(16) ApSmem S;
    pdl_enter();
    fused_launch(pf, G, ngrid, [&](int blk) { apply_tile(L, w, out, blk, q0, q1, S); });
}
// gather-first variant: G.out is the level's face scratch, out the result
__global__ void __launch_bounds__(256) k_stokes_apply_gf(Lev L, const double* __restrict__ w, double* __restrict__ out,
                                                         PForce pf, Gather G, int ngrid) {
    __shared__ __align__(16) ApSmem S;
    pdl_enter();
    fused_launch_gf(pf, G, ngrid, (int)blockIdx.x, [&](int blk) { apply_tile(L, w, out, blk, 0, L.nn, S, &G); });
}

// r = b - S w (E' part added by k_face_gather with sign +1).
__global__ void k_stokes_residual(Lev L, const double* __restrict__ b, const double* __restrict__ w,
                                  double* __restrict__ r, PForce pf, Gather G, int ngrid, int q0, int q1) {
    pdl_enter();
    fused_launch(pf, G, ngrid, [&](int blk) {
        const int q = q0 + blk * blockDim.x + threadIdx.x;
        if (q >= q1) return;
        const int i = q & (L.n - 1), j = q >> L.lg;
        GAcc acc{w, L.n, L.nn};
        double ru, rv, rp;
        stokes_rows(L, acc, i, j, ru, rv, rp);
        r[q] = b[q] - ru;
        r[L.nn + q] = b[L.nn + q] - rv;
        r[2 * L.nn + q] = b[2 * L.nn + q] - rp;
    });
}

// Fused residual + restriction (K2): coarse b = R (b - S w) per coarse cell
// (restrict_saddle, transfers.cpp:107-134; periodic).  The E' part of the
// restricted residual, R E' w = sum_k L^{l+1}_k F_k, is added afterwards by
// the launch's face-gather CTAs on the coarse face list.  One thread per
// (coarse cell, component): the 6 (u, v) or 4 (p) fine residual rows of one
// component (stokes_row, the same expressions as stokes_rows), ~3x fewer
// registers than a thread per cell with all 16 (occupancy-bound otherwise).
__device__ __forceinline__ void residual_restrict_comp(const Lev& F, const double* __restrict__ b,
                                                       const double* __restrict__ w, double* __restrict__ bc,
                                                       double* __restrict__ wc_zero, int q, int q1, int comp) {
    const int nc = F.n >> 1, nnc = nc * nc;
    if (q >= q1) return;
    if (wc_zero) wc_zero[(size_t)comp * nnc + q] = 0.0;  // the coarse level's zero initial guess
    const int I = q % nc, J = q / nc;
    const int i = 2 * I, j = 2 * J, n = F.n, nn = F.nn;
    GAcc acc{w, n, nn};
    auto r_at = [&](int f, int a, int bb) {
        a = wr(a, n);
        bb = wr(bb, n);
        return b[(size_t)f * nn + a + bb * n] - stokes_row(F, acc, f, a, bb);
    };
    if (comp == 0)
        bc[q] = 0.125 * (r_at(0, i - 1, j) + 2.0 * r_at(0, i, j) + r_at(0, i + 1, j) + r_at(0, i - 1, j + 1) +
                         2.0 * r_at(0, i, j + 1) + r_at(0, i + 1, j + 1));
    else if (comp == 1)
        bc[nnc + q] = 0.125 * (r_at(1, i, j - 1) + 2.0 * r_at(1, i, j) + r_at(1, i, j + 1) + r_at(1, i + 1, j - 1) +
                               2.0 * r_at(1, i + 1, j) + r_at(1, i + 1, j + 1));
    else
        bc[2 * nnc + q] = 0.25 * (r_at(2, i, j) + r_at(2, i + 1, j) + r_at(2, i, j + 1) + r_at(2, i + 1, j + 1));
}

// Grid CTAs: ngrid = 3 x CTAs-per-component over coarse cells [q0, q1).
__global__ void k_residual_restrict(Lev F, const double* __restrict__ b, const double* __restrict__ w,
                                    double* __restrict__ bc, double* __restrict__ wc_zero, PForce pf, Gather G,
                                    int ngrid, int q0, int q1) {
    pdl_enter();
    fused_launch(pf, G, ngrid, [&](int blk) {
        const int nbc = ngrid / 3, comp = blk / nbc;
        residual_restrict_comp(F, b, w, bc, wc_zero, q0 + (blk - comp * nbc) * blockDim.x + threadIdx.x, q1, comp);
    });
}

// Tiled residual + restriction for levels whose coarse side is >= 32 (the
// bandwidth regime; same arithmetic, term order and results as
// residual_restrict_comp).  A grid CTA owns a 32 x 8 tile of coarse cells: it
// stages the fine w region [x0-2, x0+66) x [y0-2, y0+17) of all three fields
// into shared memory with 16-byte cp.async (every fine value crosses HBM once
// per launch, up to the 2-cell halo), loads its b values straight from
// global, and each thread then forms the 16 fine residual rows of one coarse
// cell from double2 shared loads (lane I reads columns 2I.., 16 B apart: no
// bank conflicts).  Tiles with rows past q1 (slab ends) skip those rows.
constexpr int kRrTx = 32, kRrTy = 8;
constexpr int kRrW = 2 * kRrTx + 4, kRrH = 2 * kRrTy + 3;
struct RrSmem {
    double s[3][kRrH][kRrW];
};


// e (optional): E'_l w on the level's velocity faces (dense, zero off the
// E-active faces; k_residual_restrict_e), added to b in the residual rows.
__device__ __forceinline__ void residual_restrict_tile(const Lev& F, const double* __restrict__ b,
                                                       const double* __restrict__ w, double* __restrict__ bc,
                                                       double* __restrict__ wc_zero, int blk, int q0, int q1,
                                                       RrSmem& S, const double* __restrict__ e = nullptr,
                                                       const Gather* gf = nullptr) {
    const int n = F.n, nn = F.nn, nc = n >> 1, nnc = nc * nc;
    const int ntx = nc / kRrTx, Jb = q0 / nc, Je = q1 / nc;
    const int ty = blk / ntx, tx = blk - ty * ntx;
    const int x0 = 2 * tx * kRrTx, y0 = 2 * (Jb + ty * kRrTy);
    constexpr int kPairs = kRrW / 2;
    for (int e = threadIdx.x; e < 3 * kRrH * kPairs; e += blockDim.x) {
        const int f = e / (kRrH * kPairs), rem = e - f * (kRrH * kPairs);
        const int r = rem / kPairs, pc = rem - r * kPairs;
        rr_cp16(&S.s[f][r][2 * pc], w + (size_t)f * nn + wr(x0 - 2 + 2 * pc, n) + (size_t)wr(y0 - 2 + r, n) * n);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int I = threadIdx.x & 31, J = threadIdx.x >> 5;
    const int Ic = tx * kRrTx + I, Jc = Jb + ty * kRrTy + J;
    const bool act = Jc < Je;
    const int q = Ic + Jc * nc;
    // b values of the cell's residual rows (fine x 2Ic-2.., rows as below)
    double2 bu[2][2], bv[3], bp[2];
    if (act) {
        const int xm = wr(2 * Ic - 2, n), xc = 2 * Ic;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const size_t row = (size_t)(2 * Jc + k) * n;
            bu[k][0] = __ldg(reinterpret_cast<const double2*>(b + row + xm));
            bu[k][1] = __ldg(reinterpret_cast<const double2*>(b + row + xc));
            bp[k] = __ldg(reinterpret_cast<const double2*>(b + 2 * (size_t)nn + row + xc));
        }
#pragma unroll
        for (int k = 0; k < 3; ++k)
            bv[k] = __ldg(reinterpret_cast<const double2*>(b + nn + (size_t)wr(2 * Jc - 1 + k, n) * n + xc));
        if (e) {  // b + E'w on the u and v rows (e is written by this launch: L2 loads)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const size_t row = (size_t)(2 * Jc + k) * n;
                const double2 e0 = __ldcg(reinterpret_cast<const double2*>(e + row + xm));
                const double2 e1 = __ldcg(reinterpret_cast<const double2*>(e + row + xc));
                bu[k][0].x += e0.x;
                bu[k][0].y += e0.y;
                bu[k][1].x += e1.x;
                bu[k][1].y += e1.y;
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2 ev =
                    __ldcg(reinterpret_cast<const double2*>(e + nn + (size_t)wr(2 * Jc - 1 + k, n) * n + xc));
                bv[k].x += ev.x;
                bv[k].y += ev.y;
            }
        }
        if (wc_zero) {
            wc_zero[q] = 0.0;
            wc_zero[nnc + q] = 0.0;
            wc_zero[2 * nnc + q] = 0.0;
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (!act) return;
    const double d = F.d, cc = F.c, g = F.g;
    auto ld2 = [&](int f, int r, int c) { return *reinterpret_cast<const double2*>(&S.s[f][r][c]); };
    const int c0 = 2 * I;  // smem column of fine x = 2Ic - 2
    // ---- u: smem rows 2J+1 .. 2J+4 (fine y 2Jc-1 .. 2Jc+2), columns c0 .. c0+5
    double u[4][6];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            const double2 t = ld2(0, 2 * J + 1 + k, c0 + 2 * h);
            u[k][2 * h] = t.x;
            u[k][2 * h + 1] = t.y;
        }
    double pu[2][4];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 t = ld2(2, 2 * J + 2 + k, c0 + 2 * h);
            pu[k][2 * h] = t.x;
            pu[k][2 * h + 1] = t.y;
        }
    // u residual at fine (2Ic - 2 + ci, 2Jc + k - 1), ci in 1..3, k in 1..2
    auto ru = [&](int k, int ci) {
        const double bb = (ci & 1) ? ((ci == 1) ? bu[k - 1][0].y : bu[k - 1][1].y) : bu[k - 1][1].x;
        return bb - (d * u[k][ci] - cc * (u[k][ci - 1] + u[k][ci + 1] + u[k - 1][ci] + u[k + 1][ci]) +
                     g * (pu[k - 1][ci] - pu[k - 1][ci - 1]));
    };
    double ecu = 0.0, ecv = 0.0;
    const bool gfa = gf && gf->nblk;
    if (gfa) {  // gather-first: R E' w on the coarse faces, from the face scratch
        wait_gathers(*gf);
        ecu = __ldcg(gf->out + q);
        ecv = __ldcg(gf->out + nnc + q);
    }
    {
        const double v = 0.125 * (ru(1, 1) + 2.0 * ru(1, 2) + ru(1, 3) + ru(2, 1) + 2.0 * ru(2, 2) + ru(2, 3));
        bc[q] = gfa ? v + ecu : v;
    }
    // ---- p rows: u(x+1, y) - u(x, y) and v(x, y+1) - v(x, y), fine (2Ic + a, 2Jc + bb)
    double v[5][6];
#pragma unroll
    for (int k = 0; k < 5; ++k)
#pragma unroll
        for (int h = 0; h < 3; ++h) {
            const double2 t = ld2(1, 2 * J + k, c0 + 2 * h);
            v[k][2 * h] = t.x;
            v[k][2 * h + 1] = t.y;
        }
    auto rp = [&](int a, int bb) {
        const double2 t = bp[bb];
        const double bval = a ? t.y : t.x;
        return bval - (-g * (u[1 + bb][3 + a] - u[1 + bb][2 + a]) - g * (v[3 + bb][2 + a] - v[2 + bb][2 + a]));
    };
    bc[2 * nnc + q] = 0.25 * (rp(0, 0) + rp(1, 0) + rp(0, 1) + rp(1, 1));
    // ---- v: smem rows 2J .. 2J+4 (fine y 2Jc-2 .. 2Jc+2); residual rows k in 1..3
    double pv[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double2 t = ld2(2, 2 * J + k, c0 + 2);
        pv[k][0] = t.x;
        pv[k][1] = t.y;
    }
    auto rv = [&](int k, int ci) {
        const double bb = (ci == 2) ? bv[k - 1].x : bv[k - 1].y;
        return bb - (d * v[k][ci] - cc * (v[k - 1][ci] + v[k + 1][ci] + v[k][ci - 1] + v[k][ci + 1]) +
                     g * (pv[k][ci - 2] - pv[k - 1][ci - 2]));
    };
    {
        const double v = 0.125 * (rv(1, 2) + 2.0 * rv(2, 2) + rv(3, 2) + rv(1, 3) + 2.0 * rv(2, 3) + rv(3, 3));
        bc[nnc + q] = gfa ? v + ecv : v;
    }
}

// gather-first variant (whole coarse level): G.out is the coarse level's face scratch
__global__ void __launch_bounds__(256) k_residual_restrict_gf(Lev F, const double* __restrict__ b,
                                                              const double* __restrict__ w, double* __restrict__ bc,
                                                              double* __restrict__ wc_zero, PForce pf, Gather G,
                                                              int ngrid) {
    __shared__ __align__(16) RrSmem S;
    pdl_enter();
    const int nnc = F.nn >> 2;
    fused_launch_gf(pf, G, ngrid, (int)blockIdx.x, [&](int blk) {
        residual_restrict_tile(F, b, w, bc, wc_zero, blk, 0, nnc, S, nullptr, &G);
    });
}

// Grid CTAs: ngrid = (nc / 32) x ceil(rows / 8) tiles over coarse rows
// [q0 / nc, q1 / nc) (q0, q1 whole coarse rows; nc >= 32).
__global__ void __launch_bounds__(256) k_residual_restrict_t(Lev F, const double* __restrict__ b,
                                                             const double* __restrict__ w, double* __restrict__ bc,
                                                             double* __restrict__ wc_zero, PForce pf, Gather G,
                                                             int ngrid, int q0, int q1) {
    __shared__ __align__(16) RrSmem S;
    pdl_enter();
    fused_launch(pf, G, ngrid,
                 [&](int blk) { residual_restrict_tile(F, b, w, bc, wc_zero, blk, q0, q1, S); });
}

// Variant for levels where the Lagrangian points far outnumber the E-active
// faces (coarse levels of many-structure grids): the E' part of the residual
// comes from the level's assembled rows (E'_l w, CSR, elasticity.cpp:88-107
// restated per level) instead of the factored point forces + coarse face
// gather, whose cost scales with the points.  Launch = [R.nblk row CTAs: a
// warp per E' row (lane-strided sum + fixed xor tree: deterministic) writing
// e[face] | tile CTAs: wait until every row CTA has signalled, then the tiled
// residual + restriction with b + e].  Row CTAs come first in dispatch order,
// so the waiting tiles never block them.
__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
struct ERes {
    FaceList FL;
    EMat E;
    double* e;                  // dense level vector (velocity part), zero off the face list
    int nblk;                   // row CTAs (8 rows each)
    unsigned long long* cnt;    // monotone per-context counter
    unsigned long long target;  // its value once this launch's row CTAs are done
};
__device__ __forceinline__ void residual_restrict_e_at(const Lev& F, const double* __restrict__ b,
                                                       const double* __restrict__ w, double* __restrict__ bc,
                                                       double* __restrict__ wc_zero, const ERes& R, int q0, int q1,
                                                       int bid, RrSmem& S) {
    if (bid < R.nblk) {
        const int row = bid * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
        if (row < R.FL.nf) {
            double s = 0.0;
            for (int k = R.E.rp[row] + lane; k < R.E.rp[row + 1]; k += 32) s += R.E.val[k] * w[R.E.col[k]];
            s = warp_sum_xor(s);
            if (lane == 0) __stcg(R.e + R.FL.face[row], s);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(R.cnt, 1ull);
        }
        return;
    }
    if (threadIdx.x == 0)
        while (ld_acquire_u64(R.cnt) < R.target) __nanosleep(32);
    __syncthreads();
    residual_restrict_tile(F, b, w, bc, wc_zero, bid - R.nblk, q0, q1, S, R.e);
}
__global__ void __launch_bounds__(256) k_residual_restrict_e(Lev F, const double* __restrict__ b,
                                                             const double* __restrict__ w, double* __restrict__ bc,
                                                             double* __restrict__ wc_zero, ERes R, int q0, int q1) {
    __shared__ __align__(16) RrSmem S;
    pdl_enter();
    residual_restrict_e_at(F, b, w, bc, wc_zero, R, q0, q1, (int)blockIdx.x, S);
}

// Plain restriction of a vector (ibmg_restrict).
__global__ void k_restrict(int nf, const double* __restrict__ rf, double* __restrict__ rc) {
    pdl_enter();
    const int nc = nf >> 1, nnc = nc * nc, nnf = nf * nf;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nnc) return;
    const int I = q % nc, J = q / nc, i = 2 * I, j = 2 * J;
    auto U = [&](int a, int bb) { return rf[wr(a, nf) + wr(bb, nf) * nf]; };
    auto V = [&](int a, int bb) { return rf[nnf + wr(a, nf) + wr(bb, nf) * nf]; };
    auto P = [&](int a, int bb) { return rf[2 * nnf + wr(a, nf) + wr(bb, nf) * nf]; };
    rc[q] = 0.125 * (U(i - 1, j) + 2.0 * U(i, j) + U(i + 1, j) + U(i - 1, j + 1) + 2.0 * U(i, j + 1) + U(i + 1, j + 1));
    rc[nnc + q] = 0.125 * (V(i, j - 1) + 2.0 * V(i, j) + V(i, j + 1) + V(i + 1, j - 1) + 2.0 * V(i + 1, j) + V(i + 1, j + 1));
    rc[2 * nnc + q] = 0.25 * (P(i, j) + P(i + 1, j) + P(i, j + 1) + P(i + 1, j + 1));
}

// Prolongation + add (K3): bilinear u/v (transfers.cpp:141-205 with the correct
// v weight ys[b].w, not line 202's xs[a].w), constant p.
template <class Acc>
__device__ __forceinline__ void prolong_rows(int nf, const Acc& ec, int i, int j, double& du, double& dv,
                                             double& dp) {
    const int nc = nf >> 1;
    // u: x face direction, y cell direction
    {
        int I[2], J[2];
        double wi[2], wj[2];
        int ni;
        if ((i & 1) == 0) { I[0] = i >> 1; wi[0] = 1.0; ni = 1; }
        else { I[0] = (i - 1) >> 1; wi[0] = 0.5; I[1] = (i + 1) >> 1; wi[1] = 0.5; ni = 2; }
        J[0] = j >> 1; wj[0] = 0.75; J[1] = (j & 1) ? (j >> 1) + 1 : (j >> 1) - 1; wj[1] = 0.25;
        double acc = 0.0;
        for (int a = 0; a < ni; ++a)
            for (int b = 0; b < 2; ++b) acc += wi[a] * wj[b] * ec(0, wr(I[a], nc), wr(J[b], nc));
        du = acc;
    }
    {
        int I[2], J[2];
        double wi[2], wj[2];
        int nj;
        if ((j & 1) == 0) { J[0] = j >> 1; wj[0] = 1.0; nj = 1; }
        else { J[0] = (j - 1) >> 1; wj[0] = 0.5; J[1] = (j + 1) >> 1; wj[1] = 0.5; nj = 2; }
        I[0] = i >> 1; wi[0] = 0.75; I[1] = (i & 1) ? (i >> 1) + 1 : (i >> 1) - 1; wi[1] = 0.25;
        double acc = 0.0;
        for (int b = 0; b < nj; ++b)
            for (int a = 0; a < 2; ++a) acc += wj[b] * wi[a] * ec(1, wr(I[a], nc), wr(J[b], nc));
        dv = acc;
    }
    dp = ec(2, i >> 1, j >> 1);
}

__global__ void k_prolong_add(int nf, const double* __restrict__ ec, double* __restrict__ wf, int q0, int q1) {
    pdl_enter();
    const int nnf = nf * nf;
    const int q = q0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= q1) return;
    const int i = q % nf, j = q / nf;
    GAcc acc{ec, nf >> 1, (nf >> 1) * (nf >> 1)};
    double du, dv, dp;
    prolong_rows(nf, acc, i, j, du, dv, dp);
    wf[q] += du;
    wf[nnf + q] += dv;
    wf[2 * nnf + q] += dp;
}

// ---------------- Krylov vector kernels ----------------
constexpr int kRedBlocks = 296;  // 2 x 148 SMs; fixed => reduction order fixed
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// partial[y * kRedBlocks + x] = sum over block x's strided range of V_y . w
// (y = blockIdx.y indexes the vector; V vectors are `stride` doubles apart).
__global__ void k_multidot_partial(const double* __restrict__ V, size_t stride, const double* __restrict__ w,
                                   size_t m, double* __restrict__ partial) {
    pdl_enter();
    const double* v = V + stride * blockIdx.y;
    double s = 0.0;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x)
        s += v[q] * w[q];
    __shared__ double red[kRedThreads / 32];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

// out[y] (+)= sum_x partial[y][x]; mode 0: store, 1: accumulate (CGS2 second pass).
__global__ void k_finish_dots(const double* __restrict__ partial, int nblk, double* __restrict__ out, int accumulate) {
    pdl_enter();
    double s = 0.0;
    for (int x = threadIdx.x; x < nblk; x += 32) s += partial[blockIdx.x * nblk + x];
    s = warp_sum(s);
    if (threadIdx.x == 0) out[blockIdx.x] = accumulate ? out[blockIdx.x] + s : s;
}

// Fused CGS2 sweeps over the Krylov basis (one read of w and of each V_i per
// sweep; K accumulators in registers):
//   MODE 0: partial[i] = V_i . w
//   MODE 1: w -= sum_i h[i] V_i, then partial[i] = V_i . w_new
//   MODE 2: w -= sum_i h[i] V_i, then partial[0] = w_new . w_new
// Per-block partial sums are reduced in a fixed order (warp butterfly, then
// the warps in index order), so the dots are deterministic.
constexpr int kCgsBlocks = 592;  // 4 per SM; fixed => reduction order fixed
inline int ortho_update_grid(size_t m, int per_cta) {
    if (per_cta <= 0) return kCgsBlocks;
    const int b = int(m / size_t(per_cta));
    return b < 16 ? 16 : (b > kCgsBlocks ? kCgsBlocks : b);
}
template <int MODE, int KMAX>
__global__ void __launch_bounds__(kRedThreads, (MODE == 1 ? 2 : 4) / (KMAX > 16 ? 2 : 1))
    k_cgs_sweep(const double* __restrict__ V, size_t stride, int k, const double* __restrict__ h,
                double* __restrict__ w, size_t m, double* __restrict__ partial, double* __restrict__ out,
                unsigned* __restrict__ ticket) {
    pdl_enter();
    constexpr int NACC = MODE == 2 ? 1 : KMAX;
    __shared__ double hs[KMAX];
    __shared__ double red[kRedThreads / 32][NACC];
    if (MODE > 0 && threadIdx.x < KMAX) hs[threadIdx.x] = threadIdx.x < k ? h[threadIdx.x] : 0.0;
    __syncthreads();
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = 0.0;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        double x = w[q];
        if (MODE == 0) {
            // batches of 8 independent loads issued back to back, then the FMAs
#pragma unroll
            for (int i0 = 0; i0 < KMAX; i0 += 8) {
                double v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = (i0 + i < k) ? __ldcs(V + stride * (i0 + i) + q) : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i0 + i] += v[i] * x;
            }
        } else {
            double v[KMAX];
#pragma unroll
            for (int i = 0; i < KMAX; ++i) v[i] = (i < k) ? __ldcs(V + stride * i + q) : 0.0;
#pragma unroll
            for (int i = 0; i < KMAX; ++i) x -= hs[i] * v[i];
            w[q] = x;
            if (MODE == 2) {
                acc[0] += x * x;
            } else {
#pragma unroll
                for (int i = 0; i < NACC; ++i) acc[i] += v[i] * x;
            }
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
        const double t = warp_sum(acc[i]);
        if (lane == 0) red[wid][i] = t;
    }
    __syncthreads();
    const int kk = MODE == 2 ? 1 : k;
    for (int i = threadIdx.x; i < kk; i += blockDim.x) {
        double t = 0.0;
        for (int ww = 0; ww < kRedThreads / 32; ++ww) t += red[ww][i];
        partial[(size_t)i * gridDim.x + blockIdx.x] = t;
    }
    // the last CTA to finish sums the partials in the fixed k_finish_dots
    // order (lane-strided, then a warp butterfly), one warp per dot
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = wid; i < kk; i += kRedThreads / 32) {
        double t = 0.0;
        for (int x = lane; x < (int)gridDim.x; x += 32) t += __ldcg(partial + (size_t)i * gridDim.x + x);
        t = warp_sum(t);
        if (lane == 0) out[i] = t;
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// ---- two-pass (lagged) CGS2 orthogonalisation of FGMRES ----
// At Arnoldi step j the basis slot V_j holds q, orthogonalised once against
// V_0..V_{j-1} (unnormalised: the previous update pass writes w1 there); w = A M q.  Pass 1 (k_ortho_dots) reads
// V_0..V_j and w once: b_i = V_i.w, a_i = V_i.q (i < j), gamma = q.w,
// delta = q.q; its last CTA forms nu = sqrt(delta - |a|^2) (q's norm after
// the second orthogonalisation), h = (gamma - a.b) / nu (= v_j.w),
// s = h / nu and c_i = b_i - a_i s.  Pass 2 (k_ortho_update) reads
// V_0..V_j and w once more and writes v_j = (q - sum a_i V_i) / nu into V_j
// (q's re-orthogonalisation, lagged by one step) and w1 = w - sum c_i V_i - s q
// (w projected once against V_0..V_j), plus |w1|^2.  Two passes over the
// basis per step instead of CGS2's three; in exact arithmetic the same
// Arnoldi basis.  dh layout (ld = restart + 2): [b | gamma] at 0,
// [a | delta] at ld, c at 4 ld, scalars at 5 ld: 1/nu, s, nu, h, |w1|^2.
// 3 CTAs per SM (2 for KMAX 32) of 256 threads: room for the unrolled loads
template <int KMAX>
constexpr int ortho_dots_blocks() { return KMAX > 16 ? 2 * 148 : 3 * 148; }
// CTAs of the two passes for Krylov vectors of m doubles: the counts above
// (kCgsBlocks for the update) on large vectors, about per_cta doubles per CTA
// on small ones (C2 / C5: 96 CTAs with many loads in flight each, instead of
// hundreds of CTAs doing one load round each).  A function of m only, so a
// problem's reduction order is the same in a batch and in its own context.
template <int KMAX>
inline int ortho_dots_grid(size_t m, int per_cta) {
    if (per_cta <= 0) return ortho_dots_blocks<KMAX>();
    const int b = int(m / size_t(per_cta));
    return b < 16 ? 16 : (b > ortho_dots_blocks<KMAX>() ? ortho_dots_blocks<KMAX>() : b);
}
// bid / nb: this CTA's index and the CTA count of the pass (bid and
// nb; the batched kernel passes its own)
// The coefficients of the update pass from the summed dots of pass 1 (bw: b_i and
// gamma, aqd: a_i and delta, k entries each): run by the last CTA of k_ortho_dots, or
// by k_ortho_finish once the slabs' sums are reduced (slab groups).  One CTA.
__device__ __forceinline__ void ortho_finish(const double* bw, const double* aqd, int k, double* __restrict__ dh,
                                             int ld, double* s_coef) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid == 0) {
        double na = 0.0, ab = 0.0;
        for (int i = lane; i < k - 1; i += 32) {
            na += aqd[i] * aqd[i];
            ab += aqd[i] * bw[i];
        }
        na = warp_sum(na);
        ab = warp_sum(ab);
        if (lane == 0) {
            // |q - V a|^2 = delta - |a|^2, clamped: near a Krylov breakdown the
            // difference can round below zero.  nu <= 1e-14 |q| is a breakdown
            // (q in span V): nu = 0 is published (v_j = 0, w projected on
            // V_{<j} only) and fgmres2 ends the cycle at the previous column.
            const double delta = aqd[k - 1], nu2 = fmax(delta - na, 0.0);
            const bool brk = !(nu2 > 1e-28 * delta);
            const double nu = brk ? 0.0 : sqrt(nu2), h = brk ? 0.0 : (bw[k - 1] - ab) / nu;
            dh[5 * ld] = brk ? 0.0 : 1.0 / nu;
            dh[5 * ld + 1] = brk ? 0.0 : h / nu;
            dh[5 * ld + 2] = nu;
            dh[5 * ld + 3] = h;
            *s_coef = brk ? 0.0 : h / nu;  // s for the coefficients below
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        dh[i] = bw[i];
        dh[ld + i] = aqd[i];
        if (i < k - 1) dh[4 * ld + i] = bw[i] - aqd[i] * *s_coef;
    }
}
// Slab groups: the 2k raw sums of pass 1 live at dh[2 ld ..) (k_ortho_dots<KMAX, true>),
// are summed over the slabs there, and this kernel forms the coefficients.
__global__ void k_ortho_finish(int k, double* __restrict__ dh, int ld) {
    pdl_enter();
    __shared__ double fin[64];
    __shared__ double s_coef;
    for (int d = threadIdx.x; d < 2 * k; d += blockDim.x) fin[d] = dh[2 * ld + d];
    __syncthreads();
    ortho_finish(fin, fin + k, k, dh, ld, &s_coef);
}

// FLAT (k <= KMAX / 2, chosen for k <= 4): no split of the basis range over the two
// thread halves — every thread takes all k vectors of its own elements, so at small k
// all 256 threads stream (the split leaves half of them idle at k = 1: 2.5 TB/s at C4).
template <int KMAX, bool RAW = false, bool FLAT = false>
__device__ __forceinline__ void ortho_dots_at(const double* __restrict__ V, size_t stride, int k,
                                              const double* __restrict__ w, size_t m, double* __restrict__ partial,
                                              double* __restrict__ dh, int ld, unsigned* __restrict__ ticket, int bid,
                                              int nb) {
    constexpr int KH = KMAX / 2;  // i-range per thread half
    constexpr int TPE = FLAT ? kRedThreads : 128;  // threads over distinct elements
    __shared__ double red[kRedThreads / 32][2 * KH];
    __shared__ double fin[2 * KMAX];
    __shared__ double s_coef;
    const int th = FLAT ? (int)threadIdx.x : (int)(threadIdx.x & 127), half = FLAT ? 0 : (int)(threadIdx.x >> 7);
    const int kh = FLAT ? k : (k + 1) >> 1, i0 = half * kh, ni = min(kh, k - i0);
    const double* qv_ptr = V + stride * (k - 1);
    // few basis vectors per thread => several elements per iteration, so
    // every thread keeps enough loads in flight at small k
    constexpr int UNR = KH <= 4 ? 4 : 1;
    constexpr int BAT = KH < 8 ? KH : 8;
    double aw[KH], aq[KH];
#pragma unroll
    for (int i = 0; i < KH; ++i) aw[i] = aq[i] = 0.0;
    const size_t step = (size_t)nb * TPE;
    for (size_t q0 = (size_t)bid * TPE + th; q0 < m; q0 += step * UNR) {
        double x[UNR], qq[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const size_t q = q0 + u * step;
            x[u] = q < m ? w[q] : 0.0;
            qq[u] = q < m ? qv_ptr[q] : 0.0;
        }
#pragma unroll
        for (int b0 = 0; b0 < KH; b0 += BAT) {
            double v[BAT][UNR];
#pragma unroll
            for (int i = 0; i < BAT; ++i)
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const size_t q = q0 + u * step;
                    v[i][u] = (b0 + i < ni && q < m) ? __ldcs(V + stride * (i0 + b0 + i) + q) : 0.0;
                }
#pragma unroll
            for (int i = 0; i < BAT; ++i)
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    aw[b0 + i] += v[i][u] * x[u];
                    aq[b0 + i] += v[i][u] * qq[u];
                }
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < KH; ++i) {
        const double tw = warp_sum(aw[i]), tq = warp_sum(aq[i]);
        if (lane == 0) {
            red[wid][i] = tw;
            red[wid][KH + i] = tq;
        }
    }
    __syncthreads();
    // dot d: which = d / k (0: with w, 1: with q), index i = d % k
    for (int d = threadIdx.x; d < 2 * k; d += blockDim.x) {
        const int which = d / k, i = d - which * k, hh = FLAT ? 0 : i / kh, sl = i - hh * kh;
        double t = 0.0;
        for (int ww = FLAT ? 0 : 4 * hh; ww < (FLAT ? kRedThreads / 32 : 4 * hh + 4); ++ww) t += red[ww][which * KH + sl];
        partial[(size_t)d * nb + bid] = t;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == nb - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int d = wid; d < 2 * k; d += kRedThreads / 32) {
        double t = 0.0;
        for (int x = lane; x < (int)nb; x += 32) t += __ldcg(partial + (size_t)d * nb + x);
        t = warp_sum(t);
        if (lane == 0) fin[d] = t;
    }
    __syncthreads();
    if (RAW) {  // slab groups: the raw sums, reduced over the slabs before k_ortho_finish
        for (int d = threadIdx.x; d < 2 * k; d += blockDim.x) dh[2 * ld + d] = fin[d];
    } else {
        ortho_finish(fin, fin + k, k, dh, ld, &s_coef);
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

template <int KMAX, bool RAW = false, bool FLAT = false>
__global__ void __launch_bounds__(kRedThreads, KMAX > 16 ? 2 : 3)
    k_ortho_dots(const double* __restrict__ V, size_t stride, int k, const double* __restrict__ w, size_t m,
                 double* __restrict__ partial, double* __restrict__ dh, int ld, unsigned* __restrict__ ticket) {
    pdl_enter();
    ortho_dots_at<KMAX, RAW, FLAT>(V, stride, k, w, m, partial, dh, ld, ticket, (int)blockIdx.x, (int)gridDim.x);
}
constexpr int kOrthoFlatK = 4;  // k <= this: the FLAT pass 1 (single context, batch and slab groups alike)

template <int KMAX>
__device__ __forceinline__ void ortho_update_at(double* __restrict__ V, size_t stride, int k,
                                                const double* __restrict__ w, double* __restrict__ w1out,
                                                double* __restrict__ zero, size_t m, double* __restrict__ partial,
                                                double* __restrict__ dh, int ld, unsigned* __restrict__ ticket, int bid,
                                                int nb) {
    __shared__ double as[KMAX], cs[KMAX];
    __shared__ double red[kRedThreads / 32];
    if (threadIdx.x < KMAX) {
        const bool on = (int)threadIdx.x < k - 1;
        as[threadIdx.x] = on ? dh[ld + threadIdx.x] : 0.0;
        cs[threadIdx.x] = on ? dh[4 * ld + threadIdx.x] : 0.0;
    }
    __syncthreads();
    const double inu = dh[5 * ld], sq = dh[5 * ld + 1];
    double* qv_ptr = V + stride * (k - 1);
    double acc = 0.0;
    for (size_t q = (size_t)bid * blockDim.x + threadIdx.x; q < m; q += (size_t)nb * blockDim.x) {
        double v[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; ++i) v[i] = (i < k - 1) ? __ldcs(V + stride * i + q) : 0.0;
        const double qq = qv_ptr[q];
        double x = w[q], t = qq;
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
            t -= as[i] * v[i];
            x -= cs[i] * v[i];
        }
        x -= sq * qq;
        qv_ptr[q] = t * inu;
        w1out[q] = x;
        if (zero) zero[q] = 0.0;
        acc += x * x;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    acc = warp_sum(acc);
    if (lane == 0) red[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int ww = 0; ww < kRedThreads / 32; ++ww) t += red[ww];
        partial[bid] = t;
    }
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == nb - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (wid == 0) {
        double t = 0.0;
        for (int x = lane; x < (int)nb; x += 32) t += __ldcg(partial + x);
        t = warp_sum(t);
        if (lane == 0) dh[5 * ld + 4] = t;
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

template <int KMAX>
__global__ void __launch_bounds__(kRedThreads, 4 / (KMAX > 16 ? 2 : 1))
    k_ortho_update(double* __restrict__ V, size_t stride, int k, const double* __restrict__ w,
                   double* __restrict__ w1out, double* __restrict__ zero, size_t m, double* __restrict__ partial,
                   double* __restrict__ dh, int ld, unsigned* __restrict__ ticket) {
    pdl_enter();
    ortho_update_at<KMAX>(V, stride, k, w, w1out, zero, m, partial, dh, ld, ticket, (int)blockIdx.x, (int)gridDim.x);
}

// w -= sum_{i<k} h[i] V_i   (one pass over w and the V's).
__global__ void k_multi_axpy_sub(const double* __restrict__ V, size_t stride, int k, const double* __restrict__ h,
                                 double* __restrict__ w, size_t m) {
    pdl_enter();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        double s = w[q];
        for (int i = 0; i < k; ++i) s -= h[i] * V[stride * i + q];
        w[q] = s;
    }
}

// x += sum_{i<k} y[i] Z_i
__global__ void k_multi_axpy_add(const double* __restrict__ Z, size_t stride, int k, const double* __restrict__ y,
                                 double* __restrict__ x, size_t m) {
    pdl_enter();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        double s = x[q];
        for (int i = 0; i < k; ++i) s += y[i] * Z[stride * i + q];
        x[q] = s;
    }
}

// dst = src * (1 / sqrt(*nrm2))  or  src / scalar when nrm2 == nullptr
// dst = src / s (s = sqrt(*nrm2) or scalar); zero[] (optional, same length)
// is cleared in the same pass (the next V-cycle's zero initial guess).
__global__ void k_scale_by_norm(const double* __restrict__ src, double* __restrict__ dst, size_t m,
                                const double* __restrict__ nrm2, double scalar, double* __restrict__ zero) {
    pdl_enter();
    const double s = nrm2 ? sqrt(*nrm2) : scalar;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x) {
        dst[q] = src[q] / s;
        if (zero) zero[q] = 0.0;
    }
}

// p -= mean(p)  (project_pressure_mean, fields.cpp:78-85); sum over all
// `total` cells precomputed in *sum; this launch covers `count` of them.
__global__ void k_sub_mean(double* __restrict__ p, size_t count, size_t total, const double* __restrict__ sum) {
    pdl_enter();
    const double mean = *sum / (double)total;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (size_t)gridDim.x * blockDim.x)
        p[q] -= mean;
}

// b = [(rho/dt) u ; 0]
__global__ void k_rhs_mass(const double* __restrict__ u, double* __restrict__ b, size_t nn, double rho_dt) {
    pdl_enter();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < 3 * nn; q += (size_t)gridDim.x * blockDim.x)
        b[q] = q < 2 * nn ? rho_dt * u[q] : 0.0;
}

// r = b - r  (residual from an applied operator)
__global__ void k_b_minus(const double* __restrict__ b, double* __restrict__ r, size_t m) {
    pdl_enter();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (size_t)gridDim.x * blockDim.x)
        r[q] = b[q] - r[q];
}

// ---------------- slab partition ----------------
constexpr int kMaxSlabs = 8;
struct RankPtrs {
    const double* p[kMaxSlabs];
};

// out[i] = sum_r src.p[r][i] in rank order (the allreduce of the per-slab
// partial dots: every slab sums the same values in the same order, so all
// slabs hold bitwise identical results).
__global__ void k_sum_ranks(RankPtrs src, int nranks, int len, double* __restrict__ out) {
    pdl_enter();
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += src.p[r][i];
        out[i] = s;
    }
}

// Seam row merge: the v faces of a slab's first row are also box DOFs of the
// boxes just below it (the neighbour slab's top cells).  After a colour pass,
// the entries the neighbour changed (its copy differs from the snapshot taken
// before the pass) replace ours; same-colour boxes never share a DOF, so
// each entry was written by at most one side.
__global__ void k_seam_merge(double* __restrict__ row, const double* __restrict__ theirs,
                             const double* __restrict__ old, int n) {
    pdl_enter();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double t = theirs[i];
    if (t != old[i]) row[i] = t;
}

}  // namespace ibmg
