// coarse_kernel.cuh — the bottom of the V-cycle (levels with n <= 32) in ONE
// CTA, entirely in shared memory: sweeps (same schedule as the oracle), the
// residual with the E' part, restriction, the dense bordered coarsest solve,
// prolongation.  Removes the latency-bound tail of Algorithm 1
// from the launch stream.  The big phase runs its colour
// classes in order, the blocks of a class one after another (a valid order of
// an independent set), their slabs double-buffered into shared memory.
#pragma once
#include "common.cuh"
#include "grid_kernels.cuh"
#include "smoother_kernels.cuh"

namespace ibmg {

constexpr int kCoarseMaxN = 32;
constexpr int kCoarseThreads = 384;  // 3 groups of 128 for the big phase (170 regs per thread)

struct CLev {
    Lev L;
    FaceList FL;
    EMat E;
    const uint8_t* big;
    Slabs SL;
    int nbig, ncol;
    int coff[33];
};

struct CoarseArgs {
    int nl, nu1, nu2;
    unsigned long long* trace;  // debug: phase stamps by thread 0 (nullptr in production)
    CLev lv[4];
    const double* Acoarse;   // bordered inverse, col-major (3nn+1)^2
    const double* b_in;
    double* w_out;
    double* w_fine;  // optional: w of the next finer level (n = 2 * lv[0].L.n) += P w_out
};

struct SW {
    double* s;
    int n, nn;
    __device__ __forceinline__ double& operator()(int f, int i, int j) const {
        return s[f * nn + wr(i, n) + wr(j, n) * n];
    }
};

// Pointers into the dynamic shared memory lose their address space when kept
// in local arrays or passed to a non-inlined function; asserting it again lets
// the compiler emit LDS/STS (short scoreboard) instead of generic LD/ST.
template <class T>
__device__ __forceinline__ T* in_smem(T* p) {
    __builtin_assume(__isShared(p));
    return p;
}

__device__ __forceinline__ void cmark(unsigned long long* tr, int& n) {
    if (tr && threadIdx.x == 0) tr[n] = gtimer();
    ++n;
}

__device__ void coarse_sweep(const CLev& C, double* w, const double* b, ESlot* slot, BigScratch* S,
                             unsigned long long* tr, int& nm) {
    w = in_smem(w);
    b = in_smem(b);
    slot = in_smem(slot);
    S = in_smem(S);
    const Lev& L = C.L;
    const int n = L.n, t = threadIdx.x, nt = blockDim.x, nbk = n >> 2;
    SW W{w, n, L.nn};
    SW B{const_cast<double*>(b), n, L.nn};
    // plain phase: the whole periodic level in the 8 colours (i + 2j) mod 8
    // (oracle build_schedule: one tile when n <= 32), n^2/8 cells per pass
    const int per = L.nn >> 3, row = n >> 3;
    for (int pc = 0; pc < 8; ++pc) {
        for (int idx = t; idx < per; idx += nt) {
            const int j = idx / row, i = ((pc - 2 * j) & 7) + 8 * (idx % row);
            if (!C.big[(i >> 2) + (j >> 2) * nbk]) plain_cell(L, W, B, i, j);
        }
        __syncthreads();
    }
    cmark(tr, nm);  // plain phase done
    // big phase: colour classes in order; the blocks of a class (independent)
    // are shared by 4 groups of 128 threads, each with its own E'-row slot.  A
    // group refills its slot with its next block (possibly of a later colour)
    // as soon as the current block's rows are consumed, so the load overlaps
    // the rest of the solve and the colour barrier.
    const int g = t / kGroup, gt = t % kGroup, G = nt / kGroup;
    auto next_of = [&](int c, int q, int& nc, int& nq) {  // this group's item after (c, q); c < 0 starts
        nq = (c < 0) ? -1 : q + G;
        nc = (c < 0) ? 0 : c;
        while (nc < C.ncol) {
            if (nq < 0) nq = C.coff[nc] + g;
            if (nq < C.coff[nc + 1]) return;
            ++nc;
            nq = -1;
        }
    };
    int cc, qq;
    next_of(-1, 0, cc, qq);
    if (cc < C.ncol) eslot_issue(slot[g], C.SL, qq, gt, kGroup);
    cp_async_commit();
    double av[28];  // this thread's part of the group's next inverse (prefetched)
    if (cc < C.ncol) load_inverse_part(av, C.SL.Ainv + (size_t)qq * 3136, gt);
    for (int colour = 0; colour < C.ncol; ++colour) {
        const int cnt = C.coff[colour + 1] - C.coff[colour];
        for (int base = 0; base < cnt; base += G) {
            if (cc == colour && qq == C.coff[colour] + base + g) {
                cp_async_wait<0>();
                asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kGroup));
                const int Bk = slot[g].rp[47];
                int nc, nq;
                next_of(cc, qq, nc, nq);
                big_block_es<1>(L, slot[g], nullptr, 4 * (Bk % nbk), 4 * (Bk / nbk), W,
                             (const double*)w, B,
                             [&](int f, int i, int j, double old, double d) { W(f, i, j) = old + d; }, S[g], gt,
                             [g] { asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kGroup)); },
                             [&] {
                                 if (nc < C.ncol) eslot_issue(slot[g], C.SL, nq, gt, kGroup);
                                 cp_async_commit();
                             },
                             av, nc < C.ncol ? C.SL.Ainv + (size_t)nq * 3136 : nullptr, SlabTail{&C.SL, qq});
                cc = nc;
                qq = nq;
            }
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    cmark(tr, nm);  // big phase done
}

// The body of one coarse cycle (A in parameter space, or one problem's
// arguments in global memory for the batched kernel, batch.cuh).
__device__ __forceinline__ void coarse_cycle_body(const CoarseArgs& A, double* w_fine) {
    extern __shared__ __align__(16) unsigned char dsm[];
    ESlot* slot = reinterpret_cast<ESlot*>(dsm);
    double* sm = reinterpret_cast<double*>(dsm + (kCoarseThreads / kGroup) * sizeof(ESlot));
    __shared__ BigScratch S[kCoarseThreads / kGroup];
    double* wl[4];
    double* bl[4];
    size_t off = 0;
    for (int l = 0; l < A.nl; ++l) {
        const int m = 3 * A.lv[l].L.nn;
        wl[l] = sm + off;
        off += m;
        bl[l] = sm + off;
        off += m;
    }
    double* r = sm + off;
    const int t = threadIdx.x, nt = blockDim.x;
    int nm = 0;
    cmark(A.trace, nm);
    for (int q = t; q < 3 * A.lv[0].L.nn; q += nt) bl[0][q] = A.b_in[q];
    __syncthreads();
    for (int l = 0; l + 1 < A.nl; ++l) {
        const CLev& C = A.lv[l];
        const Lev& L = C.L;
        const int n = L.n, nn = L.nn;
        for (int q = t; q < 3 * nn; q += nt) wl[l][q] = 0.0;
        __syncthreads();
        for (int s = 0; s < A.nu1; ++s) coarse_sweep(C, wl[l], bl[l], slot, S, A.trace, nm);
        // residual r = b - A w (stencil, then + E' w from the assembled rows)
        SW W{wl[l], n, nn};
        for (int q = t; q < nn; q += nt) {
            double ru, rv, rp;
            stokes_rows(L, W, q % n, q / n, ru, rv, rp);
            r[q] = bl[l][q] - ru;
            r[nn + q] = bl[l][nn + q] - rv;
            r[2 * nn + q] = bl[l][2 * nn + q] - rp;
        }
        __syncthreads();
        for (int fq = t; fq < C.FL.nf; fq += nt) {
            double s = 0.0;
            for (int e = C.E.rp[fq]; e < C.E.rp[fq + 1]; ++e) s += C.E.val[e] * wl[l][C.E.col[e]];
            r[C.FL.face[fq]] += s;
        }
        __syncthreads();
        const int nc = n >> 1, nnc = nc * nc;
        for (int q = t; q < nnc; q += nt) {
            const int I = q % nc, J = q / nc, i = 2 * I, j = 2 * J;
            SW R{r, n, nn};
            bl[l + 1][q] = 0.125 * (R(0, i - 1, j) + 2.0 * R(0, i, j) + R(0, i + 1, j) + R(0, i - 1, j + 1) +
                                    2.0 * R(0, i, j + 1) + R(0, i + 1, j + 1));
            bl[l + 1][nnc + q] = 0.125 * (R(1, i, j - 1) + 2.0 * R(1, i, j) + R(1, i, j + 1) + R(1, i + 1, j - 1) +
                                          2.0 * R(1, i + 1, j) + R(1, i + 1, j + 1));
            bl[l + 1][2 * nnc + q] = 0.25 * (R(2, i, j) + R(2, i + 1, j) + R(2, i, j + 1) + R(2, i + 1, j + 1));
        }
        __syncthreads();
        cmark(A.trace, nm);  // residual + restriction done
    }
    {
        const int l = A.nl - 1, nn = A.lv[l].L.nn, m = 3 * nn + 1;
        for (int q = t; q < 3 * nn; q += nt) {
            double s = 0.0;
            for (int c = 0; c < 3 * nn; ++c) s += A.Acoarse[(size_t)c * m + q] * bl[l][c];
            wl[l][q] = s;
        }
        __syncthreads();
        cmark(A.trace, nm);  // coarsest solve done
    }
    for (int l = A.nl - 2; l >= 0; --l) {
        const CLev& C = A.lv[l];
        const int n = C.L.n, nn = C.L.nn;
        SW E{wl[l + 1], n >> 1, nn >> 2};
        for (int q = t; q < nn; q += nt) {
            double du, dv, dp;
            prolong_rows(n, E, q % n, q / n, du, dv, dp);
            wl[l][q] += du;
            wl[l][nn + q] += dv;
            wl[l][2 * nn + q] += dp;
        }
        __syncthreads();
        cmark(A.trace, nm);  // prolongation done
        for (int s = 0; s < A.nu2; ++s) coarse_sweep(C, wl[l], bl[l], slot, S, A.trace, nm);
    }
    for (int q = t; q < 3 * A.lv[0].L.nn; q += nt) A.w_out[q] = wl[0][q];
    if (w_fine) {  // prolongation-add to the finer level (K3) from shared memory
        const int nf = 2 * A.lv[0].L.n, nnf = nf * nf;
        SW E{wl[0], A.lv[0].L.n, A.lv[0].L.nn};
        for (int q = t; q < nnf; q += nt) {
            double du, dv, dp;
            prolong_rows(nf, E, q % nf, q / nf, du, dv, dp);
            w_fine[q] += du;
            w_fine[nnf + q] += dv;
            w_fine[2 * nnf + q] += dp;
        }
    }
    cmark(A.trace, nm);
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse_cycle(CoarseArgs A) {
    pdl_enter();
    coarse_cycle_body(A, A.w_fine);
}

}  // namespace ibmg
