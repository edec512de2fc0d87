// common.cuh — shared device types and helpers for the periodic MAC-grid kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ibmg {

// One multigrid level of the periodic n x n MAC grid (n a power of two).
// d, c, g are the stencil coefficients of the negated, mass-augmented Stokes
// rows (reference rows assembly.cpp:13-50):
//   u row: d u_C - c (u_W + u_E + u_S + u_N) + g (p_C - p_W)
//   p row: -g (u_E - u_C) - g (v_N - v_C)
struct Lev {
    int n, nn, lg;   // cells per side, n*n, log2(n)
    double h, d, c, g;
    // closed-form 5x5 Vanka constants: 1/(d+c), 1/(d-c), (d+c)/g, 1/(4g)
    double idpc, idmc, dpc_g, i4g;
};

// Per-level Lagrangian windows: for every point four 4x4
// patches with unwrapped integer origins: Lu, Lv (left = R...R W^T) and Ru, Rv
// (right = W P...P).  On the fine level left == right == the 4-point kernel
// weights W (elasticity.cpp:16-58).
struct Win {
    int4* orgL;   // {Lu.i0, Lu.j0, Lv.i0, Lv.j0}
    int4* orgR;   // {Ru.i0, Ru.j0, Rv.i0, Rv.j0}
    double* w;    // [pt][4][16]: Lu, Lv, Ru, Rv patches, entry b*4 + a at (i0+a, j0+b)
};

// CSR of E-active faces of a level: for each unique face (sorted flat
// velocity index) the (point, left weight) entries in ascending point order.
struct FaceList {
    int nf = 0;          // unique faces
    int* face = nullptr; // [nf] flat index comp*nn + i + j*n
    int* off = nullptr;  // [nf+1]
    int* ent = nullptr;  // entries: pt*32 + comp*16 + e (window slot of Lu/Lv)
};

// Assembled E'_l rows on the E-active faces of a level (row q <-> FaceList
// face q): CSR with flat velocity column indices.  Built from the factored
// windows (E'_l = sum_k L_k c_k (R_{k-1} - 2 R_k + R_{k+1})), i.e. the
// reference's assembled Galerkin elasticity (elasticity.cpp:88-107,
// transfers.cpp:286-293) restricted to its nonzero rows.
struct EMat {
    int* rp = nullptr;     // [nf+1]
    int* col = nullptr;    // [nnz]
    double* val = nullptr; // [nnz]
};

// Lagrangian point data.
struct Pts {
    int n = 0;
    int* kprev = nullptr;
    int* knext = nullptr;
    double* cE = nullptr;    // dt * kappa_m * h0^2  (E' coefficient, ds^2 cancels)
    double* kap = nullptr;   // kappa_m
    double* ids2 = nullptr;  // 1 / ds_m^2
    double* dsq = nullptr;   // ds_m^2 (spread quadrature, fiber.cpp:93)
};

__host__ __device__ __forceinline__ int wr(int i, int n) { return i & (n - 1); }

// Slab partition (slab_group.cuh): halo depth in rows, and the
// neighbour copies a colour pass mirrors its boundary writes into (peer
// stores over NVLink, or plain stores when the slabs share a GPU).  A write of
// row j (wrapped) also goes to the previous slab when j is among the first
// kHaloRows owned rows, and to the next slab when j is among the last
// kHaloRows owned rows or is row y1 (the next slab's first v row, a face of
// this slab's top boxes).  prv == nullptr: no mirroring (one context).
constexpr int kHaloRows = 24;
struct Mirror {
    double* prv = nullptr;
    double* nxt = nullptr;
    int y0 = 0, y1 = 0;
    __device__ __forceinline__ void store(size_t off, int j, int n, double v) const {
        if (prv == nullptr) return;
        if (wr(j - y0, n) < kHaloRows) __stcg(prv + off, v);
        if (wr(j - (y1 - kHaloRows), n) <= kHaloRows) __stcg(nxt + off, v);
    }
};

// Programmatic dependent launch: every kernel of the library is launched with
// programmatic stream serialization (ibmg.cu launch_k), lets the next kernel
// in the stream be scheduled at once, and waits for the previous kernel's
// completion (and memory flush) before touching any data.  The dependent's
// CTAs are resident when its prerequisite finishes: no launch gap.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// Enumerate the 56 DOFs of a 4x4 big block at cell origin (bi, bj):
// u faces (a in 0..4, b in 0..3), v faces (a in 0..3, b in 0..4), p (4x4).
__device__ __forceinline__ void block_dof(int t, int bi, int bj, int& field, int& i, int& j) {
    if (t < 20) {
        field = 0;
        i = bi + t % 5;
        j = bj + t / 5;
    } else if (t < 40) {
        t -= 20;
        field = 1;
        i = bi + t % 4;
        j = bj + t / 4;
    } else {
        t -= 40;
        field = 2;
        i = bi + t % 4;
        j = bj + t / 4;
    }
}

// Local index inside a block of a (field, i, j) DOF with unwrapped-relative
// coordinates (a, b) = (i - bi, j - bj) taken mod n; -1 if outside.
__device__ __forceinline__ int block_local(int field, int a, int b) {
    if (field == 0) return (a >= 0 && a <= 4 && b >= 0 && b <= 3) ? a + 5 * b : -1;
    if (field == 1) return (a >= 0 && a <= 3 && b >= 0 && b <= 4) ? 20 + a + 4 * b : -1;
    return (a >= 0 && a <= 3 && b >= 0 && b <= 3) ? 40 + a + 4 * b : -1;
}

// Window value of patch slot s (0 Lu, 1 Lv, 2 Ru, 3 Rv) of point k at the
// wrapped face (i, j), 0 if outside the 4x4 support.
__device__ __forceinline__ double win_at(const Win& W, int k, int s, int n, int i, int j) {
    const int4 o = (s < 2) ? W.orgL[k] : W.orgR[k];
    const int i0 = (s & 1) ? o.z : o.x;
    const int j0 = (s & 1) ? o.w : o.y;
    const int a = wr(i - i0, n), b = wr(j - j0, n);
    if (a >= 4 || b >= 4) return 0.0;
    return W.w[(size_t)k * 64 + s * 16 + b * 4 + a];
}

// U_k = R_k . w for component comp (0 u, 1 v) against a field accessor.
template <class Acc>
__device__ __forceinline__ double win_dot_R(const Win& W, int k, int comp, int n, const Acc& acc) {
    const int4 o = W.orgR[k];
    const int i0 = comp ? o.z : o.x, j0 = comp ? o.w : o.y;
    const double* p = W.w + (size_t)k * 64 + (2 + comp) * 16;
    double s = 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int a = 0; a < 4; ++a) s += p[b * 4 + a] * acc(comp, wr(i0 + a, n), wr(j0 + b, n));
    return s;
}

// Global-memory field accessor: comp 0 u, 1 v, 2 p.
struct GAcc {
    const double* w;
    int n, nn;
    __device__ __forceinline__ double operator()(int comp, int i, int j) const {
        return __ldg(w + (size_t)comp * nn + i + (size_t)j * n);
    }
};

// out[face q] += sign * sum_{(k, l) in list(q)} l * F[k][comp]: a group of SUB
// lanes per face (SUB = 32 on coarse levels, whose lists run to thousands of
// entries; SUB = 8 where every list is <= 32 entries), lanes strided over the
// entries, then a fixed xor-tree over the group (deterministic spread: no
// atomics).  All 32 lanes must call it (inactive groups pass active = false).
template <int SUB>
__device__ __forceinline__ void face_gather_sub(const FaceList& FL, const Win& W, const double* __restrict__ F,
                                                double* __restrict__ out, int nn, double sign, int q, bool active,
                                                int gl, bool assign = false) {
    double s = 0.0;
    int face = 0;
    if (active) {
        face = FL.face[q];
        const int comp = face >= nn;
        const int e1 = FL.off[q + 1];
        int e = FL.off[q] + gl;
        // 4 entries per lane in flight (the per-lane summation order is unchanged)
        for (; e + 3 * SUB < e1; e += 4 * SUB) {
            int v[4];
            double a[4], f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = FL.ent[e + SUB * u];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = v[u] >> 5;
                a[u] = W.w[(size_t)k * 64 + (v[u] & 31)];
                f[u] = F[2 * k + comp];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) s += a[u] * f[u];
        }
        for (; e < e1; e += SUB) {
            const int v = FL.ent[e];
            const int k = v >> 5;
            s += W.w[(size_t)k * 64 + (v & 31)] * F[2 * k + comp];
        }
    }
#pragma unroll
    for (int o = SUB / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (active && gl == 0) {
        if (assign) out[face] = sign * s;  // into a face scratch the grid CTAs add (gather-first launches)
        else out[face] += sign * s;
    }
}

// NF consecutive faces per 8-lane group, the loads of all NF chains issued together
// (face -> offsets -> entries -> weights and forces).  Per face the arithmetic is
// face_gather_sub<8>'s: lane gl adds entries off + gl, off + gl + 8, ... in order, then
// the xor tree over the 8 lanes; lane f of the group updates face f.  Rows outside
// [jlo, jhi) are skipped (slab mode).  All 32 lanes must call it.
template <int NF>
__device__ __forceinline__ void face_gather_multi(const FaceList& FL, const Win& W, const double* __restrict__ F,
                                                  double* __restrict__ out, int nn, double sign, int q0, int gl,
                                                  bool assign, int lg, int jlo, int jhi) {
    double s[NF];
    int face[NF], e[NF], e1[NF], comp[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        s[f] = 0.0;
        face[f] = -1;
        e[f] = e1[f] = 0;
        comp[f] = 0;
        if (q0 + f < FL.nf) {
            face[f] = FL.face[q0 + f];
            e[f] = FL.off[q0 + f] + gl;
            e1[f] = FL.off[q0 + f + 1];
        }
    }
#pragma unroll
    for (int f = 0; f < NF; ++f)
        if (face[f] >= 0) {
            comp[f] = face[f] >= nn;
            if (jlo > 0 || jhi < (1 << 30)) {
                const int row = (face[f] & (nn - 1)) >> lg;
                if (row < jlo || row >= jhi) face[f] = -1, e1[f] = 0;
            }
        }
    while (true) {
        int v[NF];
        bool on[NF], any = false;
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            on[f] = e[f] < e1[f];
            any |= on[f];
            v[f] = on[f] ? FL.ent[e[f]] : 0;
        }
        if (!any) break;
        double a[NF], ff[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            const int k = v[f] >> 5;
            a[f] = on[f] ? W.w[(size_t)k * 64 + (v[f] & 31)] : 0.0;
            ff[f] = on[f] ? F[2 * k + comp[f]] : 0.0;
        }
#pragma unroll
        for (int f = 0; f < NF; ++f)
            if (on[f]) {
                s[f] += a[f] * ff[f];
                e[f] += 8;
            }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1)
#pragma unroll
        for (int f = 0; f < NF; ++f) s[f] += __shfl_xor_sync(0xffffffffu, s[f], o);
#pragma unroll
    for (int f = 0; f < NF; ++f)
        if (gl == f && face[f] >= 0) {
            if (assign) out[face[f]] = sign * s[f];
            else out[face[f]] += sign * s[f];
        }
}

// one warp per face (k_face_gather: RHS forces, spread)
__device__ __forceinline__ void face_gather_warp(const FaceList& FL, const Win& W, const double* __restrict__ F,
                                                 double* __restrict__ out, int nn, double sign, int q, int lane) {
    face_gather_sub<32>(FL, W, F, out, nn, sign, q, q < FL.nf, lane);
}

}  // namespace ibmg
