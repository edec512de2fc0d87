// paper_mode.cu — the paper-reproduction mode on B200 (C ABI include/ibmg_paper.h).
//
// Dirichlet cavity, thick fiber mesh, b x b box relaxation in lexicographic order
// (SPEC.md:390-457), V(nu1,nu2), stand-alone multigrid and
// right-preconditioned GMRES, in the reference's packed interior ordering
// (geometry.hpp:54-76) and sign convention (saddle.cpp:19-38).  Everything that
// touches grid data runs in the kernels below; the host sequences launches and does
// the (m+1) x m Hessenberg algebra.  There is no CPU fallback.
//
//  * E (elasticity.cpp:62-107) is assembled on the device: one thread per triplet
//    scale * rw * coef * cw, a stable radix sort by (row, col) and a sequential sum of
//    each run, so duplicates add in the reference's emission order.
//  * Coarse E = R E P (transfers.cpp:286-293): every fine entry expands into its <= 2
//    restriction rows x <= 4 prolongation columns (wall-reflected weights,
//    transfers.cpp:141-205 with line 202's v weight corrected); same sort + run sum.
//  * Box matrices: principal submatrices of the level operator, assembled and inverted
//    per box by an in-place Gauss-Jordan with partial pivoting; a box
//    that covers its level is bordered by the pressure mean.
//  * k_sweep runs the LEXICOGRAPHIC Gauss-Seidel order exactly, as a dataflow
//    pipeline: a CTA draws the next box from a ticket counter, waits (acquire) until
//    the boxes before it within the level's coupling reach have published, relaxes its
//    box, and publishes (release) its row's progress.  Boxes further apart than the
//    reach commute, so the result equals the sequential sweep; parallelism is the
//    skewed wavefront nb / (reach + 1).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ibmg_paper.h"

namespace pm {

constexpr double kPi = 3.14159265358979323846;
using u64 = unsigned long long;
constexpr u64 kNoKey = ~0ULL;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#define PM_CUDA(x)                                                                                      \
    do {                                                                                                \
        cudaError_t e_ = (x);                                                                           \
        if (e_ != cudaSuccess)                                                                          \
            throw pm::CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" +   \
                                std::to_string(__LINE__) + ")");                                        \
    } while (0)

// ---- level geometry and the packed interior ordering (geometry.hpp:54-76) ----
struct Geo {
    int n, nu, nvel, ntot;
    double h, ih, ih2;
};
inline Geo make_geo(int n) {
    Geo g;
    g.n = n;
    g.nu = (n - 1) * n;
    g.nvel = 2 * g.nu;
    g.ntot = g.nvel + n * n;
    g.h = 1.0 / n;
    g.ih = 1.0 / g.h;
    g.ih2 = 1.0 / (g.h * g.h);
    return g;
}
struct Dof {
    int t, i, j;  // t: 0 u, 1 v, 2 p
};
__device__ __forceinline__ int du(const Geo& g, int i, int j) { return (i - 1) + j * (g.n - 1); }
__device__ __forceinline__ int dv(const Geo& g, int i, int j) { return g.nu + i + (j - 1) * g.n; }
__device__ __forceinline__ int dp(const Geo& g, int i, int j) { return g.nvel + i + j * g.n; }
__device__ __forceinline__ Dof decode(const Geo& g, int d) {
    if (d < g.nu) return {0, d % (g.n - 1) + 1, d / (g.n - 1)};
    d -= g.nu;
    if (d < g.nu) return {1, d % g.n, d / g.n + 1};
    d -= g.nu;
    return {2, d % g.n, d / g.n};
}

// Row of the Stokes part (stokes_ops.cpp:78-130, saddle.cpp:19-38) applied to w:
// momentum Lap u - grad p with the tangential wall ghost -c, continuity div u.
template <bool CG>
__device__ __forceinline__ double ldw(const double* w, int k) {
    return CG ? __ldcg(w + k) : w[k];
}
template <bool CG>
__device__ double stokes_row(const Geo& g, Dof q, const double* __restrict__ w) {
    const int n = g.n, i = q.i, j = q.j;
    if (q.t == 0) {
        const double c = ldw<CG>(w, du(g, i, j));
        double acc = -4.0 * c;
        if (i > 1) acc += ldw<CG>(w, du(g, i - 1, j));
        if (i < n - 1) acc += ldw<CG>(w, du(g, i + 1, j));
        acc += (j > 0) ? ldw<CG>(w, du(g, i, j - 1)) : -c;
        acc += (j < n - 1) ? ldw<CG>(w, du(g, i, j + 1)) : -c;
        return acc * g.ih2 - (ldw<CG>(w, dp(g, i, j)) - ldw<CG>(w, dp(g, i - 1, j))) * g.ih;
    }
    if (q.t == 1) {
        const double c = ldw<CG>(w, dv(g, i, j));
        double acc = -4.0 * c;
        if (j > 1) acc += ldw<CG>(w, dv(g, i, j - 1));
        if (j < n - 1) acc += ldw<CG>(w, dv(g, i, j + 1));
        acc += (i > 0) ? ldw<CG>(w, dv(g, i - 1, j)) : -c;
        acc += (i < n - 1) ? ldw<CG>(w, dv(g, i + 1, j)) : -c;
        return acc * g.ih2 - (ldw<CG>(w, dp(g, i, j)) - ldw<CG>(w, dp(g, i, j - 1))) * g.ih;
    }
    double acc = 0.0;
    if (i + 1 <= n - 1) acc += ldw<CG>(w, du(g, i + 1, j));
    if (i >= 1) acc -= ldw<CG>(w, du(g, i, j));
    if (j + 1 <= n - 1) acc += ldw<CG>(w, dv(g, i, j + 1));
    if (j >= 1) acc -= ldw<CG>(w, dv(g, i, j));
    return acc * g.ih;
}

// The same row as (column, value) entries (assembly.cpp:13-50); returns the count (<= 7).
__device__ int stokes_entries(const Geo& g, Dof q, int* col, double* val) {
    const int n = g.n, i = q.i, j = q.j;
    int k = 0;
    if (q.t == 0) {
        double diag = -4.0;
        if (i > 1) col[k] = du(g, i - 1, j), val[k++] = g.ih2;
        if (i < n - 1) col[k] = du(g, i + 1, j), val[k++] = g.ih2;
        if (j > 0) col[k] = du(g, i, j - 1), val[k++] = g.ih2; else diag -= 1.0;
        if (j < n - 1) col[k] = du(g, i, j + 1), val[k++] = g.ih2; else diag -= 1.0;
        col[k] = du(g, i, j), val[k++] = diag * g.ih2;
        col[k] = dp(g, i, j), val[k++] = -g.ih;
        col[k] = dp(g, i - 1, j), val[k++] = g.ih;
    } else if (q.t == 1) {
        double diag = -4.0;
        if (j > 1) col[k] = dv(g, i, j - 1), val[k++] = g.ih2;
        if (j < n - 1) col[k] = dv(g, i, j + 1), val[k++] = g.ih2;
        if (i > 0) col[k] = dv(g, i - 1, j), val[k++] = g.ih2; else diag -= 1.0;
        if (i < n - 1) col[k] = dv(g, i + 1, j), val[k++] = g.ih2; else diag -= 1.0;
        col[k] = dv(g, i, j), val[k++] = diag * g.ih2;
        col[k] = dp(g, i, j), val[k++] = -g.ih;
        col[k] = dp(g, i, j - 1), val[k++] = g.ih;
    } else {
        if (i + 1 <= n - 1) col[k] = du(g, i + 1, j), val[k++] = g.ih;
        if (i >= 1) col[k] = du(g, i, j), val[k++] = -g.ih;
        if (j + 1 <= n - 1) col[k] = dv(g, i, j + 1), val[k++] = g.ih;
        if (j >= 1) col[k] = dv(g, i, j), val[k++] = -g.ih;
    }
    return k;
}

// E of a level (velocity block, alpha-free), CSR with the row of every entry kept.
struct Csr {
    int* rp = nullptr;
    int* row = nullptr;
    int* ci = nullptr;
    double* v = nullptr;
    long nnz = 0;
};
template <bool CG>
__device__ __forceinline__ double e_row(const Csr& E, int r, const double* __restrict__ w) {
    double s = 0.0;
    for (int k = E.rp[r]; k < E.rp[r + 1]; ++k) s += E.v[k] * ldw<CG>(w, E.ci[k]);
    return s;
}

// out = A w, or out = b - A w (saddle.cpp:19-54); one thread per DOF.
__global__ void k_apply(Geo g, Csr E, double alpha, const double* __restrict__ w, const double* __restrict__ b,
                        double* __restrict__ out) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= g.ntot) return;
    double a = stokes_row<false>(g, decode(g, d), w);
    if (alpha > 0.0 && d < g.nvel) a += alpha * e_row<false>(E, d, w);
    out[d] = b ? b[d] - a : a;
}

// restrict_saddle (transfers.cpp:107-134): one thread per coarse DOF.
__global__ void k_restrict(Geo f, Geo c, const double* __restrict__ rf, double* __restrict__ rc) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= c.ntot) return;
    const Dof q = decode(c, d);
    const int i = 2 * q.i, j = 2 * q.j;
    if (q.t == 0)
        rc[d] = 0.125 * (rf[du(f, i - 1, j)] + 2.0 * rf[du(f, i, j)] + rf[du(f, i + 1, j)] + rf[du(f, i - 1, j + 1)] +
                         2.0 * rf[du(f, i, j + 1)] + rf[du(f, i + 1, j + 1)]);
    else if (q.t == 1)
        rc[d] = 0.125 * (rf[dv(f, i, j - 1)] + 2.0 * rf[dv(f, i, j)] + rf[dv(f, i, j + 1)] + rf[dv(f, i + 1, j - 1)] +
                         2.0 * rf[dv(f, i + 1, j)] + rf[dv(f, i + 1, j + 1)]);
    else
        rc[d] = 0.25 * (rf[dp(f, i, j)] + rf[dp(f, i + 1, j)] + rf[dp(f, i, j + 1)] + rf[dp(f, i + 1, j + 1)]);
}

// Bilinear weights with homogeneous walls (transfers.cpp:141-205): the normal index
// takes 1 or 1/2, 1/2 and drops boundary faces, the tangential index 3/4, 1/4 and
// reflects through the wall with a negative weight.
struct W2 {
    int I;
    double w;
};
__device__ __forceinline__ int normal_w(int i, int nc, W2* o) {
    int m = 0;
    if (i % 2 == 0) {
        if (i / 2 >= 1 && i / 2 <= nc - 1) o[m++] = {i / 2, 1.0};
    } else {
        if ((i - 1) / 2 >= 1) o[m++] = {(i - 1) / 2, 0.5};
        if ((i + 1) / 2 <= nc - 1) o[m++] = {(i + 1) / 2, 0.5};
    }
    return m;
}
__device__ __forceinline__ void tangential_w(int j, int nc, W2* o) {
    const int J = j / 2;
    o[0] = {J, 0.75};
    o[1] = {(j % 2 == 0) ? J - 1 : J + 1, 0.25};
    if (o[1].I < 0) o[1] = {0, -0.25};
    else if (o[1].I > nc - 1) o[1] = {nc - 1, -0.25};
}
// Prolongation row of a fine velocity DOF: coarse DOFs and weights (<= 4).
__device__ int prolong_row(const Geo& f, const Geo& c, Dof q, int* col, double* wt) {
    W2 xs[2], ys[2];
    int k = 0;
    if (q.t == 0) {
        const int nx = normal_w(q.i, c.n, xs);
        tangential_w(q.j, c.n, ys);
        for (int a = 0; a < nx; ++a)
            for (int b = 0; b < 2; ++b) col[k] = du(c, xs[a].I, ys[b].I), wt[k++] = xs[a].w * ys[b].w;
    } else {
        const int ny = normal_w(q.j, c.n, ys);
        tangential_w(q.i, c.n, xs);
        for (int b = 0; b < ny; ++b)
            for (int a = 0; a < 2; ++a) col[k] = dv(c, xs[a].I, ys[b].I), wt[k++] = xs[a].w * ys[b].w;
    }
    return k;
}
// Restriction column of a fine velocity DOF: the coarse rows whose stencil holds it (<= 2).
__device__ int restrict_col(const Geo& c, Dof q, int* row, double* wt) {
    int k = 0;
    if (q.t == 0) {
        const int J = q.j / 2;
        if (q.i % 2 == 0) {
            if (q.i / 2 >= 1 && q.i / 2 <= c.n - 1) row[k] = du(c, q.i / 2, J), wt[k++] = 0.25;
        } else {
            if ((q.i - 1) / 2 >= 1) row[k] = du(c, (q.i - 1) / 2, J), wt[k++] = 0.125;
            if ((q.i + 1) / 2 <= c.n - 1) row[k] = du(c, (q.i + 1) / 2, J), wt[k++] = 0.125;
        }
    } else {
        const int I = q.i / 2;
        if (q.j % 2 == 0) {
            if (q.j / 2 >= 1 && q.j / 2 <= c.n - 1) row[k] = dv(c, I, q.j / 2), wt[k++] = 0.25;
        } else {
            if ((q.j - 1) / 2 >= 1) row[k] = dv(c, I, (q.j - 1) / 2), wt[k++] = 0.125;
            if ((q.j + 1) / 2 <= c.n - 1) row[k] = dv(c, I, (q.j + 1) / 2), wt[k++] = 0.125;
        }
    }
    return k;
}

// prolong_saddle_add (transfers.cpp:209-232): one thread per fine DOF.
__global__ void k_prolong_add(Geo f, Geo c, const double* __restrict__ ec, double* __restrict__ wf) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= f.ntot) return;
    const Dof q = decode(f, d);
    if (q.t == 2) {
        wf[d] += ec[dp(c, q.i / 2, q.j / 2)];
        return;
    }
    int col[4];
    double wt[4];
    const int k = prolong_row(f, c, q, col, wt);
    double acc = 0.0;
    for (int a = 0; a < k; ++a) acc += wt[a] * ec[col[a]];
    wf[d] += acc;
}

// ---- Lagrangian side (fiber.cpp:12-16, 58-87) ----
__device__ __forceinline__ double delta_1d(double r, double h) {
    const double a = fabs(r);
    if (a >= 2.0 * h) return 0.0;
    return (1.0 + cos(kPi * r / (2.0 * h))) / (4.0 * h);
}
struct NodeW {
    int ux0, uy0, vx0, vy0;
    double ux[4], uy[4], vx[4], vy[4];
};
__global__ void k_node_weights(int nn, const double* __restrict__ X, double h, NodeW* __restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nn) return;
    const double x = X[2 * q], y = X[2 * q + 1];
    NodeW w;
    double s = x / h;
    w.ux0 = (int)ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) w.ux[a] = delta_1d((w.ux0 + a) * h - x, h);
    s = y / h - 0.5;
    w.uy0 = (int)ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) w.uy[a] = delta_1d((w.uy0 + a + 0.5) * h - y, h);
    s = x / h - 0.5;
    w.vx0 = (int)ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) w.vx[a] = delta_1d((w.vx0 + a + 0.5) * h - x, h);
    s = y / h;
    w.vy0 = (int)ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) w.vy[a] = delta_1d((w.vy0 + a) * h - y, h);
    out[q] = w;
}
// Entry e (= b*4 + a) of node weights of component comp: the packed DOF (or -1) and weight.
__device__ __forceinline__ int node_entry(const Geo& g, const NodeW& w, int comp, int e, double* wt) {
    const int a = e & 3, b = e >> 2;
    if (comp == 0) {
        const int i = w.ux0 + a, j = w.uy0 + b;
        *wt = w.ux[a] * w.uy[b];
        if (*wt == 0.0 || i < 1 || i > g.n - 1 || j < 0 || j > g.n - 1) return -1;
        return du(g, i, j);
    }
    const int i = w.vx0 + a, j = w.vy0 + b;
    *wt = w.vx[a] * w.vy[b];
    if (*wt == 0.0 || j < 1 || j > g.n - 1 || i < 0 || i > g.n - 1) return -1;
    return dv(g, i, j);
}

// assemble_elasticity's triplets (elasticity.cpp:62-107): thread = (node, comp, row entry,
// neighbour, column entry), in the reference's emission order within a (row, col) key.
__global__ void k_e_emit(Geo g, int m1, int m2, double ds, const NodeW* __restrict__ nw, u64* __restrict__ key,
                         double* __restrict__ val) {
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)m1 * m2 * 1536;
    if (idx >= total) return;
    const int e = idx & 15, c = (idx >> 4) % 3, a = (idx / 48) & 15, comp = (idx / 768) & 1;
    const int q = int(idx / 1536), k = q % m1, l = q / m1;
    const int kc = (c == 1) ? k : (c == 0 ? (k == 0 ? m1 - 1 : k - 1) : (k == m1 - 1 ? 0 : k + 1));
    const double ids2 = 1.0 / (ds * ds), scale = ds * ds * g.h * g.h;
    const double coef = (c == 1) ? -2.0 * ids2 : ids2;
    double rw, cw;
    const int r = node_entry(g, nw[q], comp, a, &rw);
    const int cc = node_entry(g, nw[kc + l * m1], comp, e, &cw);
    if (r < 0 || cc < 0) {
        key[idx] = kNoKey;
        val[idx] = 0.0;
        return;
    }
    key[idx] = (u64)r * g.nvel + cc;
    val[idx] = scale * rw * coef * cw;
}

// Galerkin expansion (transfers.cpp:286-293): fine entry -> <= 2 x 4 coarse entries.
__global__ void k_galerkin_emit(Geo f, Geo c, Csr E, u64* __restrict__ key, double* __restrict__ val) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= E.nnz) return;
    int rr[2], cc[4];
    double rw[2], cw[4];
    const int nr = restrict_col(c, decode(f, E.row[k]), rr, rw);
    const int nc = prolong_row(f, c, decode(f, E.ci[k]), cc, cw);
    const double v = E.v[k];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 4; ++b) {
            const long o = k * 8 + a * 4 + b;
            if (a < nr && b < nc) {
                key[o] = (u64)rr[a] * c.nvel + cc[b];
                val[o] = rw[a] * v * cw[b];
            } else {
                key[o] = kNoKey;
                val[o] = 0.0;
            }
        }
}

__global__ void k_heads(const u64* __restrict__ key, long n, int* __restrict__ head) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) head[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}
// Sum of each run of equal keys, sequentially in sorted (= emission) order.
__global__ void k_run_sums(const u64* __restrict__ key, const double* __restrict__ val, const int* __restrict__ head,
                           const int* __restrict__ seg, long n, u64* __restrict__ ukey, double* __restrict__ usum) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !head[i]) return;
    const u64 k = key[i];
    double s = 0.0;
    for (long j = i; j < n && key[j] == k; ++j) s += val[j];
    ukey[seg[i]] = k;
    usum[seg[i]] = s;
}
__global__ void k_csr_fill(const u64* __restrict__ ukey, const double* __restrict__ usum, long nnz, int nvel, Csr E) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nnz) {
        E.row[k] = int(ukey[k] / nvel);
        E.ci[k] = int(ukey[k] % nvel);
        E.v[k] = usum[k];
    }
    if (k <= nvel) {  // rp[r] = first entry with key >= r * nvel
        const u64 t = (u64)k * nvel;
        long lo = 0, hi = nnz;
        while (lo < hi) {
            const long mid = (lo + hi) / 2;
            if (ukey[mid] < t) lo = mid + 1; else hi = mid;
        }
        E.rp[k] = int(lo);
    }
}

// ---- boxes ----
struct Box {
    int i0, j0, b, ulo, uhi, cu, vlo, vhi, cv, mu, mv, m;
};
__host__ __device__ inline Box box_geo(int n, int b, int bx, int by) {
    Box B;
    B.i0 = bx * b;
    B.j0 = by * b;
    B.b = b;
    B.ulo = B.i0 > 1 ? B.i0 : 1;
    B.uhi = B.i0 + b < n - 1 ? B.i0 + b : n - 1;
    B.cu = B.uhi - B.ulo + 1;
    B.mu = b * B.cu;
    B.vlo = B.j0 > 1 ? B.j0 : 1;
    B.vhi = B.j0 + b < n - 1 ? B.j0 + b : n - 1;
    B.cv = B.vhi - B.vlo + 1;
    B.mv = b * B.cv;
    B.m = B.mu + B.mv + b * b;
    return B;
}
__device__ __forceinline__ int box_dof(const Geo& g, const Box& B, int a) {
    if (a < B.mu) return du(g, B.ulo + a % B.cu, B.j0 + a / B.cu);
    a -= B.mu;
    if (a < B.mv) return dv(g, B.i0 + a % B.b, B.vlo + a / B.b);
    a -= B.mv;
    return dp(g, B.i0 + a % B.b, B.j0 + a / B.b);
}
__device__ __forceinline__ int box_local(const Box& B, Dof q) {
    if (q.t == 0) {
        if (q.j < B.j0 || q.j >= B.j0 + B.b || q.i < B.ulo || q.i > B.uhi) return -1;
        return (q.j - B.j0) * B.cu + (q.i - B.ulo);
    }
    if (q.t == 1) {
        if (q.i < B.i0 || q.i >= B.i0 + B.b || q.j < B.vlo || q.j > B.vhi) return -1;
        return B.mu + (q.j - B.vlo) * B.b + (q.i - B.i0);
    }
    if (q.i < B.i0 || q.i >= B.i0 + B.b || q.j < B.j0 || q.j >= B.j0 + B.b) return -1;
    return B.mu + B.mv + (q.j - B.j0) * B.b + (q.i - B.i0);
}

// Principal submatrix of the level operator on a box (row-major mc x mc, identity
// padded past the box's own m; a whole-level box is bordered by the pressure mean).
__global__ void k_box_assemble(Geo g, Csr E, double alpha, int b, int nb, int mc, int whole, double* __restrict__ M) {
    const int bx = blockIdx.x % nb, by = blockIdx.x / nb;
    const Box B = box_geo(g.n, b, bx, by);
    double* A = M + (size_t)blockIdx.x * mc * mc;
    for (int a = threadIdx.x; a < mc; a += blockDim.x) {
        double* row = A + (size_t)a * mc;
        for (int c = 0; c < mc; ++c) row[c] = 0.0;
        if (a >= B.m) {
            if (whole && a == B.m) {
                for (int c = B.mu + B.mv; c < B.m; ++c) row[c] = 1.0;
            } else {
                row[a] = 1.0;
            }
            continue;
        }
        const int d = box_dof(g, B, a);
        const Dof q = decode(g, d);
        int col[7];
        double val[7];
        const int k = stokes_entries(g, q, col, val);
        for (int e = 0; e < k; ++e) {
            const int lc = box_local(B, decode(g, col[e]));
            if (lc >= 0) row[lc] += val[e];
        }
        if (alpha > 0.0 && d < g.nvel)
            for (int e = E.rp[d]; e < E.rp[d + 1]; ++e) {
                const int lc = box_local(B, decode(g, E.ci[e]));
                if (lc >= 0) row[lc] += alpha * E.v[e];
            }
        if (whole && q.t == 2) row[B.m] = 1.0;
    }
}

// In-place Gauss-Jordan inverse with partial pivoting, one CTA per box; the result is
// written transposed (column-major) so that the sweep's matvec reads it coalesced.
__global__ void k_box_invert(int mc, double* __restrict__ M, double* __restrict__ Tinv, int* __restrict__ fail) {
    extern __shared__ double sm[];
    double* rowk = sm;                          // mc
    double* redv = sm + mc;                     // blockDim.x / 32
    int* redi = (int*)(redv + 32);              // 32
    int* piv = redi + 32;                       // mc
    __shared__ int s_p;
    double* A = M + (size_t)blockIdx.x * mc * mc;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int k = 0; k < mc; ++k) {
        double best = -1.0;
        int bi = mc;
        for (int i = k + tid; i < mc; i += nt) {
            const double v = fabs(A[(size_t)i * mc + k]);
            if (v > best) best = v, bi = i;
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(~0u, best, o);
            const int oi = __shfl_xor_sync(~0u, bi, o);
            if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
        }
        if (lane == 0) redv[warp] = best, redi[warp] = bi;
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nw; ++w)
                if (redv[w] > best || (redv[w] == best && redi[w] < bi)) best = redv[w], bi = redi[w];
            s_p = bi;
            piv[k] = bi;
            if (!(best > 0.0)) *fail = 1;
        }
        __syncthreads();
        const int p = s_p;
        if (p >= mc) return;
        // swap rows k and p, scale the pivot row (A[k][k] <- 1 first), keep it in shared memory
        const double d = 1.0 / A[(size_t)p * mc + k];
        __syncthreads();
        for (int j = tid; j < mc; j += nt) {
            const double xp = A[(size_t)p * mc + j], xk = A[(size_t)k * mc + j];
            if (p != k) A[(size_t)p * mc + j] = xk;
            const double v = ((j == k) ? 1.0 : xp) * d;
            A[(size_t)k * mc + j] = v;
            rowk[j] = v;
        }
        __syncthreads();
        for (int i = warp; i < mc; i += nw) {
            if (i == k) continue;
            const double f = A[(size_t)i * mc + k];
            __syncwarp();
            if (f != 0.0)
                for (int j = lane; j < mc; j += 32) {
                    const double x = (j == k) ? 0.0 : A[(size_t)i * mc + j];
                    A[(size_t)i * mc + j] = x - f * rowk[j];
                }
            __syncwarp();
        }
        __syncthreads();
    }
    for (int k = mc - 1; k >= 0; --k) {  // undo the row swaps as column swaps
        const int p = piv[k];
        if (p != k)
            for (int i = tid; i < mc; i += nt) {
                const double x = A[(size_t)i * mc + k];
                A[(size_t)i * mc + k] = A[(size_t)i * mc + p];
                A[(size_t)i * mc + p] = x;
            }
        __syncthreads();
    }
    double* T = Tinv + (size_t)blockIdx.x * mc * mc;
    for (int e = tid; e < mc * mc; e += nt) {
        const int c = e / mc, a = e % mc;
        T[e] = A[(size_t)a * mc + c];
    }
}

// Coupling reach of E in boxes: a velocity DOF lies on the faces of up to two cells.
__global__ void k_reach(Geo g, Csr E, int b, int* __restrict__ reach) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= E.nnz || E.v[k] == 0.0) return;
    const Dof r = decode(g, E.row[k]), c = decode(g, E.ci[k]);
    auto span = [&](Dof q, int& xlo, int& xhi, int& ylo, int& yhi) {
        if (q.t == 0) xlo = (q.i - 1) / b, xhi = q.i / b, ylo = yhi = q.j / b;
        else xlo = xhi = q.i / b, ylo = (q.j - 1) / b, yhi = q.j / b;
    };
    int rxl, rxh, ryl, ryh, cxl, cxh, cyl, cyh;
    span(r, rxl, rxh, ryl, ryh);
    span(c, cxl, cxh, cyl, cyh);
    const int dx = max(abs(rxl - cxh), abs(rxh - cxl)), dy = max(abs(ryl - cyh), abs(ryh - cyl));
    atomicMax(reach, max(dx, dy));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Relaxation of box t: residual rows of the box (matrix-free Stokes part
// + E rows, read through L2: other CTAs wrote them), dense inverse, immediate correction.
// r: mc doubles of shared memory.  Small boxes (blockDim = 32 mc): one warp per row, the
// lanes share the E row (fixed xor-tree sum).
__device__ __forceinline__ void box_relax(const Geo& g, const Csr& E, double alpha, int b, int nb, int mc, int t,
                                          const double* __restrict__ Tinv, const double* __restrict__ rhs,
                                          double* __restrict__ w, double* r) {
    const int tid = threadIdx.x, bx = t % nb, by = t / nb;
    const Box B = box_geo(g.n, b, bx, by);
    const int d = tid < B.m ? box_dof(g, B, tid) : -1;
    if (blockDim.x == 32 * mc) {
        const int a = tid >> 5, lane = tid & 31;
        if (a < B.m) {
            const int da = box_dof(g, B, a);
            double part = 0.0;
            if (alpha > 0.0 && da < g.nvel)
                for (int k = E.rp[da] + lane; k < E.rp[da + 1]; k += 32) part += E.v[k] * __ldcg(w + E.ci[k]);
            for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(~0u, part, o);
            if (lane == 0) r[a] = rhs[da] - (stokes_row<true>(g, decode(g, da), w) + alpha * part);
        } else if (lane == 0) {
            r[a] = 0.0;
        }
    } else if (tid < B.m) {
        double a = stokes_row<true>(g, decode(g, d), w);
        if (alpha > 0.0 && d < g.nvel) a += alpha * e_row<true>(E, d, w);
        r[tid] = rhs[d] - a;
    } else if (tid < mc) {
        r[tid] = 0.0;
    }
    __syncthreads();
    if (tid < B.m) {
        const double* T = Tinv + (size_t)t * mc * mc + tid;
        double s = 0.0;
        for (int c = 0; c < B.m; ++c) s += T[(size_t)c * mc] * r[c];  // (a whole-level box: the border column multiplies 0)
        w[d] = __ldcg(w + d) + s;
    }
}

// One lexicographic box sweep as a dataflow pipeline; see the header.
// sync[0] is the ticket counter, sync[1 + by] the number of boxes of row by published.
__global__ void k_sweep(Geo g, Csr E, double alpha, int b, int nb, int mc, int reach, const double* __restrict__ Tinv,
                        const double* __restrict__ rhs, double* __restrict__ w, int* __restrict__ sync) {
    extern __shared__ double r[];  // mc
    __shared__ int s_t;
    const int tid = threadIdx.x;
    if (tid == 0) {
        const int t = atomicAdd(sync, 1);
        s_t = t;
        const int bx = t % nb, by = t / nb;
        if (bx > 0)
            while (ld_acquire(sync + 1 + by) < bx) {}
        if (by > 0) {
            const int need = min(nb, bx + reach + 1);
            while (ld_acquire(sync + by) < need) {}
        }
    }
    __syncthreads();
    const int t = s_t;
    box_relax(g, E, alpha, b, nb, mc, t, Tinv, rhs, w, r);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        st_release(sync + 1 + t / nb, t % nb + 1);
    }
}

// One colour of the multicolour ordering (opt-in): the boxes (cx + per ix,
// cy + per iy), per = reach + 1, are further apart than the coupling reach, so they
// relax independently; the colours follow each other in stream order.
__global__ void k_sweep_colour(Geo g, Csr E, double alpha, int b, int nb, int mc, int per, int cx, int cy, int ncx,
                               const double* __restrict__ Tinv, const double* __restrict__ rhs, double* __restrict__ w) {
    extern __shared__ double r[];  // mc
    const int ix = blockIdx.x % ncx, iy = blockIdx.x / ncx;
    box_relax(g, E, alpha, b, nb, mc, (cx + per * ix) + (cy + per * iy) * nb, Tinv, rhs, w, r);
}

// ---- vectors ----
__global__ void k_multi_dot(const double* __restrict__ V, size_t stride, const double* __restrict__ w, int n,
                            double* __restrict__ out) {
    __shared__ double red[32];
    const double* v = V + stride * blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i] * w[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (blockDim.x >> 5); ++k) t += red[k];
        out[blockIdx.x] = t;
    }
}
// w += sign * sum_i h[i] V_i
__global__ void k_multi_axpy(const double* __restrict__ V, size_t stride, int k, const double* __restrict__ h,
                             double sign, double* __restrict__ w, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int q = 0; q < k; ++q) s += h[q] * V[stride * q + i];
    w[i] += sign * s;
}
// dst = src / sqrt(*nrm2)   (or dst = src * scale when nrm2 == nullptr)
__global__ void k_scale(const double* src, const double* __restrict__ nrm2, double scale, double* dst, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = nrm2 ? src[i] / sqrt(*nrm2) : src[i] * scale;
}
// project_pressure_mean (fields.cpp:78-85): one CTA, fixed summation order.
__global__ void k_pressure_mean(double* __restrict__ p, int np) {
    __shared__ double red[32];
    __shared__ double mean;
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) s += p[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (blockDim.x >> 5); ++k) t += red[k];
        mean = t / np;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < np; i += blockDim.x) p[i] -= mean;
}

// fiber_second_difference (fiber.cpp:34-55), closed fibers.
__global__ void k_second_difference(int m1, int m2, double ds, double gamma, const double* __restrict__ f,
                                    double* __restrict__ out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m1 * m2) return;
    const int k = q % m1, l = q / m1;
    const int a = (k == 0 ? m1 - 1 : k - 1) + l * m1, c = (k == m1 - 1 ? 0 : k + 1) + l * m1;
    const double ids2 = 1.0 / (ds * ds);
    for (int x = 0; x < 2; ++x) out[2 * q + x] = gamma * ((f[2 * a + x] + f[2 * c + x] - f[2 * q + x] * 2.0) * ids2);
}
// spread (fiber.cpp:89-114) as (face, value) pairs in node order; summed by sort + run sums.
__global__ void k_spread_emit(Geo g, int nn, double ds, const NodeW* __restrict__ nw, const double* __restrict__ F,
                              u64* __restrict__ key, double* __restrict__ val) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nn * 32) return;
    const int e = idx & 15, comp = (idx >> 4) & 1, q = idx >> 5;
    double wt;
    const int d = node_entry(g, nw[q], comp, e, &wt);
    key[idx] = d < 0 ? kNoKey : (u64)d;
    val[idx] = d < 0 ? 0.0 : F[2 * q + comp] * wt * (ds * ds);
}
__global__ void k_scatter_runs(const u64* __restrict__ ukey, const double* __restrict__ usum, long n, double sign,
                               double* __restrict__ out) {
    const long k = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n && ukey[k] != kNoKey) out[ukey[k]] += sign * usum[k];
}
// interpolate (fiber.cpp:116-140): one thread per node and component.
__global__ void k_interp(Geo g, int nn, const NodeW* __restrict__ nw, const double* __restrict__ vel,
                         double* __restrict__ U) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nn * 2) return;
    const int comp = idx & 1, q = idx >> 1;
    double s = 0.0;
    for (int e = 0; e < 16; ++e) {
        double wt;
        const int d = node_entry(g, nw[q], comp, e, &wt);
        if (d >= 0) s += vel[d] * wt;
    }
    U[idx] = s * (g.h * g.h);
}
// boundary_fold (saddle.cpp:56-94) for the lid data: only the top wall's tangential velocity is nonzero.
__global__ void k_lid_fold(Geo g, double* __restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (i > g.n - 1) return;
    const double ulid = (1.0 - cos(2.0 * kPi * (i * g.h))) / 2.0;
    b[du(g, i, g.n - 1)] -= 2.0 * ulid * g.ih2;
}

// ---- host side ----
struct Level {
    Geo g{};
    Csr E;
    int b = 1, nb = 1, mc = 0, whole = 0, reach = 1;
    double* Tinv = nullptr;
    double *w = nullptr, *rhs = nullptr, *r = nullptr;
    int* sync = nullptr;
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    void need(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        PM_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
        cap = n;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

struct Ctx {
    ibmg_paper_params P{};
    cudaStream_t s = nullptr;
    std::vector<Level> lev;
    int m1 = 0, m2 = 0;
    double ds = 0;
    std::vector<double> Xh;
    double* X = nullptr;
    NodeW* nw = nullptr;
    DevBuf<u64> k0, k1, uk;
    DevBuf<double> v0, v1, us;
    DevBuf<int> head, seg;
    DevBuf<char> cubtmp;
    DevBuf<double> V, Z, hd, va, vb, vc, lagF, lagU;
    int* fail = nullptr;
    long long launches = 0;
    std::string err;
    Ctx* stokes = nullptr;  // alpha = 0 twin for alpha_exp
    ~Ctx();
};

inline int nblk(long n, int t = 256) { return int((n + t - 1) / t); }
#define PM_LAUNCH(c, kern, grid, block, smem, ...)               \
    do {                                                         \
        kern<<<(grid), (block), (smem), (c)->s>>>(__VA_ARGS__);  \
        PM_CUDA(cudaGetLastError());                             \
        ++(c)->launches;                                         \
    } while (0)

void free_csr(Csr& E) {
    for (void* p : {(void*)E.rp, (void*)E.row, (void*)E.ci, (void*)E.v})
        if (p) cudaFree(p);
    E = Csr{};
}
void free_levels(Ctx* c) {
    for (Level& L : c->lev) {
        free_csr(L.E);
        for (void* p : {(void*)L.Tinv, (void*)L.w, (void*)L.rhs, (void*)L.r, (void*)L.sync})
            if (p) cudaFree(p);
    }
    c->lev.clear();
}
Ctx::~Ctx() {
    delete stokes;
    cudaSetDevice(P.device);
    free_levels(this);
    for (void* p : {(void*)X, (void*)nw, (void*)fail})
        if (p) cudaFree(p);
    if (s) cudaStreamDestroy(s);
}

// Stable sort of (key, value) pairs and run sums; returns the number of distinct real keys
// (c->uk / c->us hold them, sorted).
long sort_reduce(Ctx* c, long n) {
    if (n == 0) return 0;
    c->k1.need(n);
    c->v1.need(n);
    c->head.need(n);
    c->seg.need(n);
    c->uk.need(n);
    c->us.need(n);
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, c->k0.p, c->k1.p, c->v0.p, c->v1.p, n, 0, 64, c->s);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, c->head.p, c->seg.p, n, c->s);
    c->cubtmp.need(std::max(t1, t2));
    size_t tb = c->cubtmp.cap;
    PM_CUDA(cub::DeviceRadixSort::SortPairs(c->cubtmp.p, tb, c->k0.p, c->k1.p, c->v0.p, c->v1.p, n, 0, 64, c->s));
    PM_LAUNCH(c, k_heads, nblk(n), 256, 0, c->k1.p, n, c->head.p);
    tb = c->cubtmp.cap;
    PM_CUDA(cub::DeviceScan::ExclusiveSum(c->cubtmp.p, tb, c->head.p, c->seg.p, n, c->s));
    PM_LAUNCH(c, k_run_sums, nblk(n), 256, 0, c->k1.p, c->v1.p, c->head.p, c->seg.p, n, c->uk.p, c->us.p);
    int lastseg = 0, lasthead = 0;
    u64 lastkey = 0;
    PM_CUDA(cudaMemcpyAsync(&lastseg, c->seg.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    PM_CUDA(cudaMemcpyAsync(&lasthead, c->head.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, c->s));
    PM_CUDA(cudaMemcpyAsync(&lastkey, c->k1.p + n - 1, sizeof(u64), cudaMemcpyDeviceToHost, c->s));
    PM_CUDA(cudaStreamSynchronize(c->s));
    long cnt = lastseg + lasthead;  // exclusive scan of the heads + the last head
    if (lastkey == kNoKey) --cnt;  // the padding run sorts last
    return cnt;
}

void csr_from_runs(Ctx* c, const Geo& g, long nnz, Csr& E) {
    free_csr(E);
    E.nnz = nnz;
    PM_CUDA(cudaMalloc(&E.rp, sizeof(int) * (g.nvel + 1)));
    PM_CUDA(cudaMalloc(&E.row, sizeof(int) * std::max<long>(nnz, 1)));
    PM_CUDA(cudaMalloc(&E.ci, sizeof(int) * std::max<long>(nnz, 1)));
    PM_CUDA(cudaMalloc(&E.v, sizeof(double) * std::max<long>(nnz, 1)));
    PM_LAUNCH(c, k_csr_fill, nblk(std::max<long>(nnz, g.nvel + 1)), 256, 0, c->uk.p, c->us.p, nnz, g.nvel, E);
}

void require_supports_interior(const Ctx* c) {  // fiber.cpp:18-32
    const double rad = 2.0 / c->P.N;
    for (int q = 0; q < c->m1 * c->m2; ++q) {
        const double x = c->Xh[2 * q], y = c->Xh[2 * q + 1];
        if (x - rad < 0.0 || x + rad > 1.0 || y - rad < 0.0 || y + rad > 1.0)
            throw std::invalid_argument("fiber node " + std::to_string(q) +
                                        " has kernel support crossing the domain boundary");
    }
}

void build(Ctx* c) {
    const int N = c->P.N, cn = c->P.coarsest_n;
    if (N < 2 * cn || (N & (N - 1)) || cn < 2 || (cn & (cn - 1)))
        throw std::invalid_argument("N and coarsest_n must be powers of two with N >= 2 coarsest_n");
    if (c->P.box < 1 || (c->P.box & (c->P.box - 1)) || c->P.box > 16)
        throw std::invalid_argument("box must be 1, 2, 4, 8 or 16");
    if (c->P.alpha < 0) throw std::invalid_argument("SaddleSystem: alpha must be >= 0");
    if (c->P.nu1 < 0 || c->P.nu2 < 0 || c->P.nu1 + c->P.nu2 < 1) throw std::invalid_argument("nu1 + nu2 must be >= 1");
    if (c->P.order != 0 && c->P.order != 1) throw std::invalid_argument("order must be 0 (lexicographic) or 1 (multicolour)");
    PM_CUDA(cudaSetDevice(c->P.device));
    if (!c->s) PM_CUDA(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
    if (!c->fail) PM_CUDA(cudaMalloc(&c->fail, sizeof(int)));
    free_levels(c);
    const bool has_e = c->m1 > 0;
    const int nn = c->m1 * c->m2;
    if (has_e) {
        require_supports_interior(c);
        if (c->X) cudaFree(c->X);
        if (c->nw) cudaFree(c->nw);
        PM_CUDA(cudaMalloc(&c->X, sizeof(double) * 2 * nn));
        PM_CUDA(cudaMalloc(&c->nw, sizeof(NodeW) * nn));
        PM_CUDA(cudaMemcpyAsync(c->X, c->Xh.data(), sizeof(double) * 2 * nn, cudaMemcpyHostToDevice, c->s));
        PM_LAUNCH(c, k_node_weights, nblk(nn, 128), 128, 0, nn, c->X, 1.0 / N, c->nw);
    }
    for (int n = N; n >= cn; n /= 2) {
        Level L;
        L.g = make_geo(n);
        c->lev.push_back(L);
    }
    PM_CUDA(cudaMemsetAsync(c->fail, 0, sizeof(int), c->s));
    for (size_t l = 0; l < c->lev.size(); ++l) {
        Level& L = c->lev[l];
        const Geo& g = L.g;
        if (has_e) {
            long cnt;
            if (l == 0) {
                const long tot = (long)nn * 1536;
                c->k0.need(tot);
                c->v0.need(tot);
                PM_LAUNCH(c, k_e_emit, nblk(tot), 256, 0, g, c->m1, c->m2, c->ds, c->nw, c->k0.p, c->v0.p);
                cnt = sort_reduce(c, tot);
            } else {
                const Csr& F = c->lev[l - 1].E;
                const long tot = F.nnz * 8;
                c->k0.need(tot);
                c->v0.need(tot);
                if (tot) PM_LAUNCH(c, k_galerkin_emit, nblk(F.nnz), 256, 0, c->lev[l - 1].g, g, F, c->k0.p, c->v0.p);
                cnt = sort_reduce(c, tot);
            }
            csr_from_runs(c, g, cnt, L.E);
        } else {
            csr_from_runs(c, g, 0, L.E);
        }
        const int n = g.n;
        L.b = std::min(c->P.box, n);
        if (l + 1 == c->lev.size()) L.b = n;  // coarsest level: direct solve
        L.nb = n / L.b;
        L.whole = (L.nb == 1);
        L.mc = 2 * L.b * (L.b + 1) + L.b * L.b;
        if (L.whole) L.mc = box_geo(n, L.b, 0, 0).m + 1;
        const size_t nbox = (size_t)L.nb * L.nb, msz = nbox * L.mc * L.mc;
        PM_CUDA(cudaMalloc(&L.Tinv, sizeof(double) * msz));
        PM_CUDA(cudaMalloc(&L.w, sizeof(double) * g.ntot));
        PM_CUDA(cudaMalloc(&L.rhs, sizeof(double) * g.ntot));
        PM_CUDA(cudaMalloc(&L.r, sizeof(double) * g.ntot));
        PM_CUDA(cudaMalloc(&L.sync, sizeof(int) * (L.nb + 1)));
        double* M = nullptr;
        PM_CUDA(cudaMalloc(&M, sizeof(double) * msz));
        const double alpha = has_e ? c->P.alpha : 0.0;
        PM_LAUNCH(c, k_box_assemble, (int)nbox, 128, 0, g, L.E, alpha, L.b, L.nb, L.mc, L.whole, M);
        const int nt = std::min(1024, std::max(32, (L.mc * 4 + 31) / 32 * 32));
        const size_t sm = sizeof(double) * (L.mc + 32) + sizeof(int) * (32 + L.mc);
        PM_LAUNCH(c, k_box_invert, (int)nbox, nt, sm, L.mc, M, L.Tinv, c->fail);
        // coupling reach: the stencil reaches the box after next for single-cell boxes
        int reach = (L.b == 1) ? 2 : 1;
        if (has_e && alpha > 0.0 && L.E.nnz) {
            int* dr = L.sync;  // scratch
            PM_CUDA(cudaMemsetAsync(dr, 0, sizeof(int), c->s));
            PM_LAUNCH(c, k_reach, nblk(L.E.nnz), 256, 0, g, L.E, L.b, dr);
            int er = 0;
            PM_CUDA(cudaMemcpyAsync(&er, dr, sizeof(int), cudaMemcpyDeviceToHost, c->s));
            PM_CUDA(cudaStreamSynchronize(c->s));
            reach = std::max(reach, er);
        }
        L.reach = reach;
        PM_CUDA(cudaStreamSynchronize(c->s));
        cudaFree(M);
    }
    int fail = 0;
    PM_CUDA(cudaMemcpy(&fail, c->fail, sizeof(int), cudaMemcpyDeviceToHost));
    if (fail) throw std::runtime_error("singular box matrix");
    delete c->stokes;
    c->stokes = nullptr;
}

void apply(Ctx* c, int l, const double* w, const double* b, double* out) {
    Level& L = c->lev[l];
    const double alpha = c->m1 > 0 ? c->P.alpha : 0.0;
    PM_LAUNCH(c, k_apply, nblk(L.g.ntot), 256, 0, L.g, L.E, alpha, w, b, out);
}
void sweep(Ctx* c, int l, const double* rhs, double* w) {
    Level& L = c->lev[l];
    const double alpha = c->m1 > 0 ? c->P.alpha : 0.0;
    const int nt = (L.mc <= 16 && alpha > 0.0) ? 32 * L.mc : (L.mc + 31) / 32 * 32;
    if (c->P.order == 1 && !L.whole) {  // multicolour: (reach + 1)^2 launches
        const int per = L.reach + 1;
        for (int cy = 0; cy < per && cy < L.nb; ++cy)
            for (int cx = 0; cx < per && cx < L.nb; ++cx) {
                const int ncx = (L.nb - cx + per - 1) / per, ncy = (L.nb - cy + per - 1) / per;
                PM_LAUNCH(c, k_sweep_colour, ncx * ncy, nt, sizeof(double) * L.mc, L.g, L.E, alpha, L.b, L.nb, L.mc, per,
                          cx, cy, ncx, L.Tinv, rhs, w);
            }
        return;
    }
    PM_CUDA(cudaMemsetAsync(L.sync, 0, sizeof(int) * (L.nb + 1), c->s));
    PM_LAUNCH(c, k_sweep, L.nb * L.nb, nt, sizeof(double) * L.mc, L.g, L.E, alpha, L.b, L.nb, L.mc, L.reach, L.Tinv, rhs,
              w, L.sync);
}
void restrict_to(Ctx* c, int l, const double* rf, double* rc) {
    PM_LAUNCH(c, k_restrict, nblk(c->lev[l + 1].g.ntot), 256, 0, c->lev[l].g, c->lev[l + 1].g, rf, rc);
}
void prolong_add(Ctx* c, int l, const double* ec, double* wf) {
    PM_LAUNCH(c, k_prolong_add, nblk(c->lev[l].g.ntot), 256, 0, c->lev[l].g, c->lev[l + 1].g, ec, wf);
}
void pressure_mean(Ctx* c, int l, double* x) {
    const Geo& g = c->lev[l].g;
    PM_LAUNCH(c, k_pressure_mean, 1, 1024, 0, x + g.nvel, g.n * g.n);
}

// Algorithm 1.
void vcycle_rec(Ctx* c, int l) {
    Level& L = c->lev[l];
    if (L.whole) {
        sweep(c, l, L.rhs, L.w);
        return;
    }
    for (int s = 0; s < c->P.nu1; ++s) sweep(c, l, L.rhs, L.w);
    apply(c, l, L.w, L.rhs, L.r);
    Level& K = c->lev[l + 1];
    restrict_to(c, l, L.r, K.rhs);
    PM_CUDA(cudaMemsetAsync(K.w, 0, sizeof(double) * K.g.ntot, c->s));
    vcycle_rec(c, l + 1);
    prolong_add(c, l, K.w, L.w);
    for (int s = 0; s < c->P.nu2; ++s) sweep(c, l, L.rhs, L.w);
}
// z = V(0, b) on device vectors, mean-zero pressure.
void vcycle(Ctx* c, const double* b, double* z) {
    Level& L = c->lev[0];
    PM_CUDA(cudaMemcpyAsync(L.rhs, b, sizeof(double) * L.g.ntot, cudaMemcpyDeviceToDevice, c->s));
    PM_CUDA(cudaMemsetAsync(L.w, 0, sizeof(double) * L.g.ntot, c->s));
    vcycle_rec(c, 0);
    pressure_mean(c, 0, L.w);
    PM_CUDA(cudaMemcpyAsync(z, L.w, sizeof(double) * L.g.ntot, cudaMemcpyDeviceToDevice, c->s));
}

double dev_norm(Ctx* c, const double* x, int n) {
    c->hd.need(256);
    PM_LAUNCH(c, k_multi_dot, 1, 1024, 0, x, (size_t)0, x, n, c->hd.p);
    double s = 0.0;
    PM_CUDA(cudaMemcpyAsync(&s, c->hd.p, sizeof(double), cudaMemcpyDeviceToHost, c->s));
    PM_CUDA(cudaStreamSynchronize(c->s));
    return std::sqrt(s);
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// mg_solve on device vectors b, x.
void mg_solve(Ctx* c, const double* b, double* x, double rtol, int max_iter, ibmg_paper_stats* st, double* hist,
              int hl) {
    const int n = c->lev[0].g.ntot;
    c->va.need(n);
    c->vb.need(n);
    double* r = c->va.p;
    double* z = c->vb.p;
    PM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->s));
    PM_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, c->s));
    const double bn = dev_norm(c, b, n);
    if (hist && hl > 0) hist[0] = 1.0;
    if (bn == 0.0) {
        st->converged = 1;
        return;
    }
    c->hd.need(256);
    double prev = bn;
    int grow = 0;
    const double one = 1.0;
    PM_CUDA(cudaMemcpyAsync(c->hd.p + 8, &one, sizeof(double), cudaMemcpyHostToDevice, c->s));
    for (int it = 1; it <= max_iter; ++it) {
        vcycle(c, r, z);
        PM_LAUNCH(c, k_multi_axpy, nblk(n), 256, 0, z, (size_t)0, 1, c->hd.p + 8, 1.0, x, n);
        apply(c, 0, x, b, r);
        const double rn = dev_norm(c, r, n);
        st->iters = it;
        st->relres = rn / bn;
        if (hist && it < hl) hist[it] = rn / bn;
        if (rn <= rtol * bn) {
            st->converged = 1;
            break;
        }
        grow = (rn > prev) ? grow + 1 : 0;
        prev = rn;
        if (grow >= 5 || !std::isfinite(rn)) {
            st->diverged = 1;
            break;
        }
    }
    pressure_mean(c, 0, x);
}

// gmres_solve: right-preconditioned, unrestarted, x0 = 0, CGS2; the
// Givens estimate is confirmed on the true residual.  Same control flow
// as the oracle's (oracle/paper_oracle.cpp gmres_solve).
void gmres_solve(Ctx* c, const double* b, double* x, double rtol, int max_iter, ibmg_paper_stats* st, double* hist,
                 int hl) {
    const int n = c->lev[0].g.ntot, m = max_iter;
    const size_t stride = (size_t)n;
    c->V.need(stride * (m + 1));
    c->Z.need(stride * m);
    c->va.need(n);
    c->vb.need(n);
    c->hd.need(std::max<size_t>(256, 2 * (size_t)(m + 2) + 16));  // dev_norm's slot included: no regrowth below
    double* w = c->va.p;
    double* r = c->vb.p;
    double* h1d = c->hd.p;
    double* h2d = c->hd.p + (m + 2);
    double* nd = c->hd.p + 2 * (m + 2);
    PM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->s));
    const double bn = dev_norm(c, b, n);
    if (hist && hl > 0) hist[0] = 1.0;
    if (bn == 0.0) {
        st->converged = 1;
        return;
    }
    PM_LAUNCH(c, k_scale, nblk(n), 256, 0, b, (const double*)nullptr, 1.0 / bn, c->V.p, n);
    std::vector<double> H(size_t(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0), y(m), hh(2 * (m + 2) + 1);
    g[0] = bn;
    auto form_x = [&](int k) {
        for (int i = k - 1; i >= 0; --i) {
            double s = g[i];
            for (int j = i + 1; j < k; ++j) s -= H[size_t(i) * m + j] * y[j];
            y[i] = s / H[size_t(i) * m + i];
        }
        PM_CUDA(cudaMemcpyAsync(h1d, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c->s));
        PM_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, c->s));
        PM_LAUNCH(c, k_multi_axpy, nblk(n), 256, 0, c->Z.p, stride, k, h1d, 1.0, x, n);
    };
    for (int j = 0; j < m; ++j) {
        double* vj = c->V.p + stride * j;
        double* zj = c->Z.p + stride * j;
        vcycle(c, vj, zj);
        apply(c, 0, zj, nullptr, w);
        PM_LAUNCH(c, k_multi_dot, j + 1, 256, 0, c->V.p, stride, w, n, h1d);
        PM_LAUNCH(c, k_multi_axpy, nblk(n), 256, 0, c->V.p, stride, j + 1, h1d, -1.0, w, n);
        PM_LAUNCH(c, k_multi_dot, j + 1, 256, 0, c->V.p, stride, w, n, h2d);
        PM_LAUNCH(c, k_multi_axpy, nblk(n), 256, 0, c->V.p, stride, j + 1, h2d, -1.0, w, n);
        PM_LAUNCH(c, k_multi_dot, 1, 1024, 0, w, (size_t)0, w, n, nd);
        PM_CUDA(cudaMemcpyAsync(hh.data(), c->hd.p, sizeof(double) * (2 * (m + 2) + 1), cudaMemcpyDeviceToHost, c->s));
        PM_CUDA(cudaStreamSynchronize(c->s));
        const double hn = std::sqrt(hh[2 * (m + 2)]);
        for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = hh[i] + hh[m + 2 + i];
        for (int i = 0; i < j; ++i) {
            const double a = H[size_t(i) * m + j], d = H[size_t(i + 1) * m + j];
            H[size_t(i) * m + j] = cs[i] * a + sn[i] * d;
            H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * d;
        }
        const double a = H[size_t(j) * m + j], d = std::hypot(a, hn);
        cs[j] = a / d;
        sn[j] = hn / d;
        H[size_t(j) * m + j] = d;
        g[j + 1] = -sn[j] * g[j];
        g[j] = cs[j] * g[j];
        st->iters = j + 1;
        const double est = std::fabs(g[j + 1]) / bn;
        if (hist && j + 1 < hl) hist[j + 1] = est;
        const bool last = (j + 1 == m) || hn == 0.0;
        if (est <= rtol || last) {
            form_x(j + 1);
            apply(c, 0, x, b, r);
            st->relres = dev_norm(c, r, n) / bn;
            if (st->relres <= rtol) st->converged = 1;
            if (st->converged || last) break;
        }
        PM_LAUNCH(c, k_scale, nblk(n), 256, 0, (const double*)w, (const double*)nd, 1.0, c->V.p + stride * (j + 1), n);
    }
    pressure_mean(c, 0, x);
}

// Lagrangian helpers on device arrays.
void spread_dev(Ctx* c, const double* F, double sign, double* f_vel) {  // f_vel += sign * S F
    const int nn = c->m1 * c->m2;
    c->k0.need((size_t)nn * 32);
    c->v0.need((size_t)nn * 32);
    PM_LAUNCH(c, k_spread_emit, nblk((long)nn * 32), 256, 0, c->lev[0].g, nn, c->ds, c->nw, F, c->k0.p, c->v0.p);
    const long cnt = sort_reduce(c, (long)nn * 32);
    if (cnt) PM_LAUNCH(c, k_scatter_runs, nblk(cnt), 256, 0, c->uk.p, c->us.p, cnt, sign, f_vel);
}

struct HostVec {  // device copy of a host vector
    double* p = nullptr;
    size_t n = 0;
    HostVec(Ctx* c, const double* h, size_t n_) : n(n_) {
        PM_CUDA(cudaMalloc(&p, sizeof(double) * std::max<size_t>(n, 1)));
        if (h) PM_CUDA(cudaMemcpyAsync(p, h, sizeof(double) * n, cudaMemcpyHostToDevice, c->s));
    }
    void to_host(Ctx* c, double* h) {
        PM_CUDA(cudaMemcpyAsync(h, p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->s));
        PM_CUDA(cudaStreamSynchronize(c->s));
    }
    ~HostVec() {
        if (p) cudaFree(p);
    }
};

}  // namespace pm

struct ibmg_paper : pm::Ctx {};

#define PM_TRY(ctx, ...)                                 \
    if (!(ctx)) return 1;                                \
    try {                                                \
        PM_CUDA(cudaSetDevice((ctx)->P.device));         \
        __VA_ARGS__;                                     \
        return 0;                                        \
    } catch (const std::invalid_argument& e) {           \
        (ctx)->err = e.what();                           \
        return 1;                                        \
    } catch (const std::exception& e) {                  \
        (ctx)->err = e.what();                           \
        return 3;                                        \
    }

static void need_level(ibmg_paper* c, int l, bool has_coarser = false) {
    if (l < 0 || l + (has_coarser ? 1 : 0) >= (int)c->lev.size()) throw std::invalid_argument("level out of range");
}

extern "C" {

int ibmg_paper_create(const ibmg_paper_params* params, ibmg_paper** out) {
    if (!params || !out) return 1;
    ibmg_paper* c = new ibmg_paper;
    c->P = *params;
    try {
        pm::build(c);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "ibmg_paper_create: %s\n", e.what());
        delete c;
        *out = nullptr;
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ibmg_paper_create: %s\n", e.what());
        delete c;
        *out = nullptr;
        return 3;
    }
    *out = c;
    return 0;
}
void ibmg_paper_destroy(ibmg_paper* c) { delete c; }
const char* ibmg_paper_last_error(const ibmg_paper* c) { return c ? c->err.c_str() : "null context"; }

int ibmg_paper_set_mesh(ibmg_paper* c, int m1, int m2, double ds, const double* X) {
    PM_TRY(c, {
        if (m1 != 0 && (m1 < 3 || m2 < 1 || !(ds > 0.0) || !X))
            throw std::invalid_argument("FiberMesh: m1 >= 3, m2 >= 1, ds > 0");
        c->m1 = m1;
        c->m2 = m1 ? m2 : 0;
        c->ds = ds;
        c->Xh.assign(X, X + (m1 ? size_t(2) * m1 * m2 : 0));
        pm::build(c);
    });
}
int ibmg_paper_num_levels(const ibmg_paper* c) { return c ? (int)c->lev.size() : -1; }
static bool has_level(const ibmg_paper* c, int l) { return c && l >= 0 && l < (int)c->lev.size(); }
int ibmg_paper_level_n(const ibmg_paper* c, int l) { return has_level(c, l) ? c->lev[l].g.n : -1; }
int ibmg_paper_level_dofs(const ibmg_paper* c, int l) { return has_level(c, l) ? c->lev[l].g.ntot : -1; }
int ibmg_paper_level_boxes(const ibmg_paper* c, int l) { return has_level(c, l) ? c->lev[l].nb : -1; }
int ibmg_paper_level_reach(const ibmg_paper* c, int l) { return has_level(c, l) ? c->lev[l].reach : -1; }
long long ibmg_paper_kernel_launches(const ibmg_paper* c) { return c ? c->launches : -1; }

int ibmg_paper_apply(ibmg_paper* c, int l, const double* w, double* out) {
    PM_TRY(c, {
        need_level(c, l);
        const int n = c->lev[l].g.ntot;
        pm::HostVec dw(c, w, n), dout(c, nullptr, n);
        pm::apply(c, l, dw.p, nullptr, dout.p);
        dout.to_host(c, out);
    });
}
int ibmg_paper_residual(ibmg_paper* c, int l, const double* b, const double* w, double* r, double* norm) {
    PM_TRY(c, {
        need_level(c, l);
        const int n = c->lev[l].g.ntot;
        pm::HostVec dw(c, w, n), db(c, b, n), dr(c, nullptr, n);
        pm::apply(c, l, dw.p, db.p, dr.p);
        if (norm) *norm = pm::dev_norm(c, dr.p, n);
        dr.to_host(c, r);
    });
}
int ibmg_paper_restrict(ibmg_paper* c, int l, const double* rf, double* rc) {
    PM_TRY(c, {
        need_level(c, l, true);
        pm::HostVec df(c, rf, c->lev[l].g.ntot), dc(c, nullptr, c->lev[l + 1].g.ntot);
        pm::restrict_to(c, l, df.p, dc.p);
        dc.to_host(c, rc);
    });
}
int ibmg_paper_prolong_add(ibmg_paper* c, int l, const double* ec, double* wf) {
    PM_TRY(c, {
        need_level(c, l, true);
        pm::HostVec dc(c, ec, c->lev[l + 1].g.ntot), df(c, wf, c->lev[l].g.ntot);
        pm::prolong_add(c, l, dc.p, df.p);
        df.to_host(c, wf);
    });
}
int ibmg_paper_sweep(ibmg_paper* c, int l, const double* b, double* w) {
    PM_TRY(c, {
        need_level(c, l);
        const int n = c->lev[l].g.ntot;
        pm::HostVec db(c, b, n), dw(c, w, n);
        pm::sweep(c, l, db.p, dw.p);
        dw.to_host(c, w);
    });
}
int ibmg_paper_vcycle(ibmg_paper* c, const double* b, double* z) {
    PM_TRY(c, {
        const int n = c->lev[0].g.ntot;
        pm::HostVec db(c, b, n), dz(c, nullptr, n);
        pm::vcycle(c, db.p, dz.p);
        dz.to_host(c, z);
    });
}
long ibmg_paper_elasticity_triplets(ibmg_paper* c, int l, int* rows, int* cols, double* vals, long cap) {
    if (!c) return -1;
    try {
        PM_CUDA(cudaSetDevice(c->P.device));
        need_level(c, l);
        const pm::Csr& E = c->lev[l].E;
        if (!rows) return E.nnz;
        const long k = std::min(cap, E.nnz);
        PM_CUDA(cudaMemcpy(rows, E.row, sizeof(int) * k, cudaMemcpyDeviceToHost));
        PM_CUDA(cudaMemcpy(cols, E.ci, sizeof(int) * k, cudaMemcpyDeviceToHost));
        PM_CUDA(cudaMemcpy(vals, E.v, sizeof(double) * k, cudaMemcpyDeviceToHost));
        return E.nnz;
    } catch (const std::exception& e) {
        c->err = e.what();
        return -1;
    }
}

int ibmg_paper_build_rhs(ibmg_paper* c, int lid, double gamma, double* b) {
    PM_TRY(c, {
        const pm::Geo& g = c->lev[0].g;
        pm::HostVec db(c, nullptr, g.ntot);
        PM_CUDA(cudaMemsetAsync(db.p, 0, sizeof(double) * g.ntot, c->s));
        if (lid) PM_LAUNCH(c, pm::k_lid_fold, pm::nblk(g.n - 1, 128), 128, 0, g, db.p);
        if (c->m1 > 0 && gamma != 0.0) {
            const int nn = c->m1 * c->m2;
            c->lagF.need(2 * (size_t)nn);
            PM_LAUNCH(c, pm::k_second_difference, pm::nblk(nn, 128), 128, 0, c->m1, c->m2, c->ds, gamma,
                      (const double*)c->X, c->lagF.p);
            pm::spread_dev(c, c->lagF.p, -1.0, db.p);
        }
        db.to_host(c, b);
    });
}
int ibmg_paper_spread(ibmg_paper* c, const double* F, double* f_vel) {
    PM_TRY(c, {
        if (c->m1 == 0) throw std::invalid_argument("spread: no fiber mesh");
        const pm::Geo& g = c->lev[0].g;
        pm::HostVec dF(c, F, 2 * (size_t)c->m1 * c->m2), df(c, nullptr, g.nvel);
        PM_CUDA(cudaMemsetAsync(df.p, 0, sizeof(double) * g.nvel, c->s));
        pm::spread_dev(c, dF.p, 1.0, df.p);
        df.to_host(c, f_vel);
    });
}
int ibmg_paper_interpolate(ibmg_paper* c, const double* vel, double* U) {
    PM_TRY(c, {
        if (c->m1 == 0) throw std::invalid_argument("interpolate: no fiber mesh");
        const pm::Geo& g = c->lev[0].g;
        const int nn = c->m1 * c->m2;
        pm::HostVec dv(c, vel, g.nvel), dU(c, nullptr, 2 * (size_t)nn);
        PM_LAUNCH(c, pm::k_interp, pm::nblk(2 * nn, 128), 128, 0, g, nn, c->nw, (const double*)dv.p, dU.p);
        dU.to_host(c, U);
    });
}

static int solve(ibmg_paper* c, bool gmres, const double* b, double* x, double rtol, int max_iter,
                 ibmg_paper_stats* st, double* hist, int hl) {
    PM_TRY(c, {
        if (!(rtol > 0.0 && rtol < 1.0) || max_iter < 1 || !st) throw std::invalid_argument("0 < rtol < 1, max_iter >= 1");
        const int n = c->lev[0].g.ntot;
        *st = ibmg_paper_stats{0, 0, 0, 0.0, 0.0, 0.0};
        pm::HostVec db(c, b, n), dx(c, nullptr, n);
        const double t0 = pm::now_ms();
        if (gmres) pm::gmres_solve(c, db.p, dx.p, rtol, max_iter, st, hist, hl);
        else pm::mg_solve(c, db.p, dx.p, rtol, max_iter, st, hist, hl);
        dx.to_host(c, x);
        st->solve_ms = pm::now_ms() - t0;
    });
}
int ibmg_paper_mg_solve(ibmg_paper* c, const double* b, double* x, double rtol, int max_iter, ibmg_paper_stats* st,
                        double* hist, int hl) {
    return solve(c, false, b, x, rtol, max_iter, st, hist, hl);
}
int ibmg_paper_gmres_solve(ibmg_paper* c, const double* b, double* x, double rtol, int max_iter, ibmg_paper_stats* st,
                           double* hist, int hl) {
    return solve(c, true, b, x, rtol, max_iter, st, hist, hl);
}

// w = a - w (elementwise)
__global__ void pm_k_a_minus(const double* __restrict__ a, double* __restrict__ w, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] = a[i] - w[i];
}

int ibmg_paper_vcycle_spectrum(ibmg_paper* c, int m, unsigned long long seed, double* H, int* m_done) {
    PM_TRY(c, {
        if (m < 2 || !H) throw std::invalid_argument("SpectrumProbe: m >= 2");
        const int n = c->lev[0].g.ntot;
        const size_t stride = (size_t)n;
        c->V.need(stride * (m + 1));
        c->va.need(n);
        c->vb.need(n);
        c->hd.need(std::max<size_t>(256, 2 * (size_t)(m + 2) + 16));
        double* a = c->va.p;
        double* w = c->vb.p;
        double* h1d = c->hd.p;
        double* h2d = c->hd.p + (m + 2);
        double* nd = c->hd.p + 2 * (m + 2);
        std::vector<double> x0(n), hh(2 * (m + 2) + 1);
        unsigned long long z = seed;
        for (double& v : x0) {
            z += 0x9E3779B97F4A7C15ull;
            unsigned long long t = z;
            t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
            t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
            t ^= t >> 31;
            v = double(t >> 11) * (2.0 / 9007199254740992.0) - 1.0;
        }
        PM_CUDA(cudaMemcpyAsync(w, x0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->s));
        pm::pressure_mean(c, 0, w);
        PM_LAUNCH(c, pm::k_multi_dot, 1, 1024, 0, (const double*)w, (size_t)0, (const double*)w, n, nd);
        PM_LAUNCH(c, pm::k_scale, pm::nblk(n), 256, 0, (const double*)w, (const double*)nd, 1.0, c->V.p, n);
        std::fill(H, H + size_t(m + 1) * m, 0.0);
        int done = 0;
        for (int j = 0; j < m; ++j) {
            const double* vj = c->V.p + stride * j;
            pm::apply(c, 0, vj, nullptr, a);
            pm::vcycle(c, a, w);                                        // w = V(0, A v_j), mean-zero p
            PM_LAUNCH(c, pm_k_a_minus, pm::nblk(n), 256, 0, vj, w, n);  // w = v_j - w
            pm::pressure_mean(c, 0, w);
            PM_LAUNCH(c, pm::k_multi_dot, j + 1, 256, 0, (const double*)c->V.p, stride, (const double*)w, n, h1d);
            PM_LAUNCH(c, pm::k_multi_axpy, pm::nblk(n), 256, 0, (const double*)c->V.p, stride, j + 1, (const double*)h1d,
                      -1.0, w, n);
            PM_LAUNCH(c, pm::k_multi_dot, j + 1, 256, 0, (const double*)c->V.p, stride, (const double*)w, n, h2d);
            PM_LAUNCH(c, pm::k_multi_axpy, pm::nblk(n), 256, 0, (const double*)c->V.p, stride, j + 1, (const double*)h2d,
                      -1.0, w, n);
            PM_LAUNCH(c, pm::k_multi_dot, 1, 1024, 0, (const double*)w, (size_t)0, (const double*)w, n, nd);
            PM_CUDA(cudaMemcpyAsync(hh.data(), c->hd.p, sizeof(double) * (2 * (m + 2) + 1), cudaMemcpyDeviceToHost, c->s));
            PM_CUDA(cudaStreamSynchronize(c->s));
            const double hn = std::sqrt(hh[2 * (m + 2)]);
            for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = hh[i] + hh[m + 2 + i];
            H[size_t(j + 1) * m + j] = hn;
            done = j + 1;
            if (!(hn > 1e-300)) break;
            PM_LAUNCH(c, pm::k_scale, pm::nblk(n), 256, 0, (const double*)w, (const double*)nd, 1.0,
                      c->V.p + stride * (j + 1), n);
        }
        if (m_done) *m_done = done;
    });
}

// power iteration on M X = S* L^-1 S A_f X, u = L^-1 f
// solving Lap u - grad p = -f, div u = 0 with homogeneous walls (MG-GMRES at 1e-10 on the
// alpha = 0 twin of this context).  The iteration vector lives on the device.
int ibmg_paper_alpha_exp(ibmg_paper* c, double tol, int max_steps, double* alpha_exp, int* steps) {
    PM_TRY(c, {
        if (c->m1 == 0) throw std::invalid_argument("alpha_exp needs a fiber mesh");
        if (!c->stokes) {
            pm::Ctx* s = new pm::Ctx;
            s->P = c->P;
            s->P.alpha = 0.0;
            s->m1 = c->m1;
            s->m2 = c->m2;
            s->ds = c->ds;
            s->Xh = c->Xh;
            c->stokes = s;
            pm::build(s);
        }
        pm::Ctx* s = c->stokes;
        const pm::Geo& g = s->lev[0].g;
        const int nn = s->m1 * s->m2, nx = 2 * nn;
        std::vector<double> xh(nx);
        unsigned long long seed = 12345;
        for (double& v : xh) {
            seed = seed * 6364136223846793005ULL + 1442695040888963407ULL;
            v = double(seed >> 11) / 9007199254740992.0 - 0.5;
        }
        pm::HostVec x(s, xh.data(), nx), y(s, nullptr, nx), F(s, nullptr, nx), b(s, nullptr, g.ntot), w(s, nullptr, g.ntot);
        s->hd.need(256);
        double lam = 0.0, prev = 0.0;
        int it = 0;
        for (it = 1; it <= max_steps; ++it) {
            const double xn = pm::dev_norm(s, x.p, nx);
            PM_LAUNCH(s, pm::k_scale, pm::nblk(nx), 256, 0, (const double*)x.p, (const double*)nullptr, 1.0 / xn, x.p, nx);
            PM_LAUNCH(s, pm::k_second_difference, pm::nblk(nn, 128), 128, 0, s->m1, s->m2, s->ds, 1.0,
                      (const double*)x.p, F.p);
            PM_CUDA(cudaMemsetAsync(b.p, 0, sizeof(double) * g.ntot, s->s));
            pm::spread_dev(s, F.p, -1.0, b.p);
            ibmg_paper_stats st{};
            pm::gmres_solve(s, b.p, w.p, 1e-10, 100, &st, nullptr, 0);
            PM_LAUNCH(s, pm::k_interp, pm::nblk(2 * nn, 128), 128, 0, g, nn, s->nw, (const double*)w.p, y.p);
            PM_LAUNCH(s, pm::k_multi_dot, 1, 1024, 0, (const double*)x.p, (size_t)0, (const double*)y.p, nx, s->hd.p);
            PM_CUDA(cudaMemcpyAsync(&lam, s->hd.p, sizeof(double), cudaMemcpyDeviceToHost, s->s));
            PM_CUDA(cudaStreamSynchronize(s->s));
            if (it > 1 && std::fabs(lam - prev) <= tol * std::fabs(lam)) break;
            prev = lam;
            PM_CUDA(cudaMemcpyAsync(x.p, y.p, sizeof(double) * nx, cudaMemcpyDeviceToDevice, s->s));
        }
        c->launches += s->launches;
        s->launches = 0;
        if (it > max_steps) throw std::runtime_error("power iteration did not converge");
        *alpha_exp = 2.0 / std::fabs(lam);
        if (steps) *steps = it;
    });
}

}  // extern "C"
