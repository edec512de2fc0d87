// ib_kernels.cuh — Lagrangian-structure kernels: 4-point kernel windows on every
// level, E-active face lists, point forces, deterministic spread (gather over
// face lists: no float atomics), interpolation and the X update.
#pragma once
#include "common.cuh"

namespace ibmg {

constexpr double kPi = 3.14159265358979323846;

// delta_1d (fiber.cpp:12-16): (1 + cos(pi r / 2h)) / 4h for |r| < 2h.
__device__ __forceinline__ double delta_1d(double r, double h) {
    const double a = fabs(r);
    if (a >= 2.0 * h) return 0.0;
    return (1.0 + cos(kPi * r / (2.0 * h))) / (4.0 * h);
}
// kernel_line_faces / kernel_line_centers (fiber.cpp:58-87), periodic (no clip).
__device__ __forceinline__ int line_faces(double X, double h, double* w) {
    const int first = (int)ceil(X / h - 2.0);
    for (int a = 0; a < 4; ++a) w[a] = delta_1d((double)(first + a) * h - X, h);
    return first;
}
__device__ __forceinline__ int line_centers(double X, double h, double* w) {
    const int first = (int)ceil((X / h - 0.5) - 2.0);
    for (int a = 0; a < 4; ++a) w[a] = delta_1d(((double)(first + a) + 0.5) * h - X, h);
    return first;
}

struct WinLevels {
    Win win[20];
    int n[20];
    int nlev;
};

__device__ __forceinline__ void patch_add(double* dst, int a, int b, double v, int* err) {
    if (a < 0 || a >= 4 || b < 0 || b >= 4) {
        atomicOr(err, 1);
        return;
    }
    dst[b * 4 + a] += v;
}

// Face-direction restriction weights {1/8, 1/4, 1/8} (transfers.cpp:117-127):
// fine face index f feeds coarse F = f/2 (1/4) when even, (f-1)/2 and (f+1)/2 (1/8) when odd.
// Cell-direction restriction: coarse C = c>>1 with weight 1.
// Face-direction prolongation: coarse f/2 (1) or (f-1)/2,(f+1)/2 (1/2).
// Cell-direction prolongation: C = c>>1 (3/4) and C-1 (c even) / C+1 (c odd) (1/4).
__device__ __forceinline__ int face_restrict(int f, int* I, double* w) {
    if ((f & 1) == 0) { I[0] = f >> 1; w[0] = 0.25; return 1; }
    I[0] = (f - 1) >> 1; w[0] = 0.125; I[1] = (f + 1) >> 1; w[1] = 0.125; return 2;
}
__device__ __forceinline__ int face_prolong(int f, int* I, double* w) {
    if ((f & 1) == 0) { I[0] = f >> 1; w[0] = 1.0; return 1; }
    I[0] = (f - 1) >> 1; w[0] = 0.5; I[1] = (f + 1) >> 1; w[1] = 0.5; return 2;
}
__device__ __forceinline__ int cell_prolong(int c, int* J, double* w) {
    J[0] = c >> 1; w[0] = 0.75; J[1] = (c & 1) ? (c >> 1) + 1 : (c >> 1) - 1; w[1] = 0.25; return 2;
}

// Weight of fine index fi in coarse index ci for a 1-D transfer kind:
// 0 face-restrict {1/8, 1/4, 1/8}, 1 cell-restrict (1), 2 face-prolong
// (1 or 1/2, 1/2), 3 cell-prolong (3/4, 1/4); see face_restrict etc. above.
__device__ __forceinline__ double transfer_weight(int kind, int fi, int ci) {
    const int h = fi >> 1;
    const bool odd = fi & 1;
    if (kind == 1) return ci == h ? 1.0 : 0.0;
    if (kind == 3) return ci == h ? 0.75 : (ci == (odd ? h + 1 : h - 1) ? 0.25 : 0.0);
    const double w_even = kind == 0 ? 0.25 : 1.0, w_odd = kind == 0 ? 0.125 : 0.5;
    if (!odd) return ci == h ? w_even : 0.0;
    return (ci == h || ci == h + 1) ? w_odd : 0.0;  // (fi - 1) / 2 = h, (fi + 1) / 2 = h + 1
}
__device__ __forceinline__ double transfer_total(int kind) { return kind == 0 ? 0.25 : 1.0; }

// Windows of every point on every level, one thread per point.  Level l+1's
// left window is R applied to level l's (R*...*R*W^T), the right window is
// level l's times P (W*P*...*P) — the factored form of the reference's
// recursive Galerkin R*E*P (transfers.cpp:286-293, PAPER Eq. 20).
__global__ void k_windows(int npts, const double* __restrict__ X, WinLevels WL, double h0, int* err) {
    pdl_enter();
    // one thread per (point, patch s): s = 0 Lu, 1 Lv, 2 Ru, 3 Rv; the 16-entry
    // patch and its origin stay in registers from level to level
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= 4 * npts) return;
    const int k = idx >> 2, s = idx & 3, comp = s & 1;
    const double x = X[2 * k], y = X[2 * k + 1];
    double wx[4], wy[4], cur[16];
    int ox, oy;
    if (comp == 0) {
        ox = line_faces(x, h0, wx);
        oy = line_centers(y, h0, wy);
    } else {
        ox = line_centers(x, h0, wx);
        oy = line_faces(y, h0, wy);
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int a = 0; a < 4; ++a) cur[b * 4 + a] = wx[a] * wy[b];
    for (int l = 0;; ++l) {
        Win& W = WL.win[l];
        double* p = W.w + (size_t)k * 64 + s * 16;
#pragma unroll
        for (int e = 0; e < 16; ++e) p[e] = cur[e];
        int* org = reinterpret_cast<int*>(s < 2 ? &W.orgL[k] : &W.orgR[k]) + 2 * comp;
        org[0] = ox;
        org[1] = oy;
        if (l + 1 >= WL.nlev) break;
        // next patch = Wx^T cur Wy with the separable 1-D transfer weights
        // (gather form: static register indexing, no scatter into a local
        // array).  kind: 0 face-restrict, 1 cell-restrict, 2 face-prolong,
        // 3 cell-prolong; x and y kinds per patch type as in the reference's
        // R (transfers.cpp:117-127) and P (transfers.cpp:141-205).
        const int kx = s == 0 ? 0 : s == 1 ? 1 : s == 2 ? 2 : 3;
        const int ky = s == 0 ? 1 : s == 1 ? 0 : s == 2 ? 3 : 2;
        int nx, ny;
        if (s == 0) { nx = ox >> 1; ny = oy >> 1; }             // left u: face-restrict x, cell-restrict y
        else if (s == 1) { nx = ox >> 1; ny = oy >> 1; }        // left v: cell-restrict x, face-restrict y
        else if (s == 2) { nx = ox >> 1; ny = (oy - 1) >> 1; }  // right u: face-prolong x, cell-prolong y
        else { nx = (ox - 1) >> 1; ny = oy >> 1; }              // right v: cell-prolong x, face-prolong y
        double tx[4][4], ty[4][4];
        bool bad = false;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            double cs = 0.0, rs = 0.0, sx = 0.0, sy = 0.0;
#pragma unroll
            for (int A = 0; A < 4; ++A) {
                tx[a][A] = transfer_weight(kx, ox + a, nx + A);
                ty[a][A] = transfer_weight(ky, oy + a, ny + A);
                sx += tx[a][A];
                sy += ty[a][A];
                cs += fabs(cur[A * 4 + a]);  // column a
                rs += fabs(cur[a * 4 + A]);  // row a
            }
            bad |= (cs != 0.0 && sx != transfer_total(kx)) || (rs != 0.0 && sy != transfer_total(ky));
        }
        if (bad) atomicOr(err, 1);  // a weight falls outside the 4x4 patch
        double nxt[16];
#pragma unroll
        for (int B = 0; B < 4; ++B)
#pragma unroll
            for (int A = 0; A < 4; ++A) {
                double acc = 0.0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    double t = 0.0;
#pragma unroll
                    for (int a = 0; a < 4; ++a) t += tx[a][A] * cur[b * 4 + a];
                    acc += ty[b][B] * t;
                }
                nxt[B * 4 + A] = acc;
            }
#pragma unroll
        for (int e = 0; e < 16; ++e) cur[e] = nxt[e];
        ox = nx;
        oy = ny;
    }
}

// Face lists of every level in one sort: level-major face
// numbering key = base[l] + face (face < 2 n_l^2; 2 n_l^2 is the level's
// sentinel for zero window weights), value = entry pt*32 + comp*16 + e.
struct FaceBase {
    int nlev;
    unsigned base[21];
    int n[20];
};
__global__ void k_face_keys(int npts, WinLevels WL, FaceBase FB, unsigned* keys, int* vals) {
    pdl_enter();
    const long items = (long)npts * 32;
    const long q = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= items * FB.nlev) return;
    const int l = int(q / items), r = int(q - l * items);
    const int k = r >> 5, s = (r >> 4) & 1, e = r & 15, n = FB.n[l];
    const Win& W = WL.win[l];
    const double v = W.w[(size_t)k * 64 + s * 16 + e];
    const int4 o = W.orgL[k];
    const int i0 = s ? o.z : o.x, j0 = s ? o.w : o.y;
    const int i = wr(i0 + (e & 3), n), j = wr(j0 + (e >> 2), n);
    keys[q] = FB.base[l] + unsigned((v != 0.0) ? s * n * n + i + j * n : 2 * n * n);
    vals[q] = r;
}

// Per run of the sorted keys: the level-local face index, the level's first
// run (counter 20), its number of faces (17) and longest list (29); the
// sentinel run of a level is not a face.
__global__ void k_face_levels(const unsigned* __restrict__ ukeys, const int* __restrict__ nruns,
                              const int* __restrict__ off, FaceBase FB, int* __restrict__ face,
                              int* __restrict__ counters, int ctr_stride) {
    pdl_enter();
    const int nr = *nruns;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nr; q += gridDim.x * blockDim.x) {
        const unsigned key = ukeys[q];
        int l = 0;
        while (l + 1 < FB.nlev && key >= FB.base[l + 1]) ++l;
        const int loc = int(key - FB.base[l]), n = FB.n[l];
        face[q] = loc;
        int* ctr = counters + l * ctr_stride;
        if (q == 0 || ukeys[q - 1] < FB.base[l]) ctr[20] = q;
        if (loc != 2 * n * n) {
            atomicAdd(ctr + 17, 1);
            atomicMax(ctr + 29, off[q + 1] - off[q]);
        }
    }
}

// Per-level block arrays (flags, conflict masks) of the levels with big
// blocks, contiguous and level-major: level l's blocks start at boff[l].
struct BlkLevels {
    int nlev;  // levels 0 .. nlev-1 (all but the coarsest)
    int n[20];
    int boff[21];
};

// Big-block marking: a 4x4 block is big when any face of it
// lies in the support of any point's left or right window on the level.
// Thread per (level, point, window slot, tap).
__global__ void k_mark_big(int npts, WinLevels WL, BlkLevels BK, uint8_t* __restrict__ flags_all) {
    pdl_enter();
    const long per = (long)npts * 64;
    const long qq = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (qq >= per * BK.nlev) return;
    const int l = int(qq / per), q = int(qq - l * per);
    const Win& W = WL.win[l];
    const int n = BK.n[l];
    uint8_t* flags = flags_all + BK.boff[l];
    const int k = q >> 6, s = (q >> 4) & 3, e = q & 15;
    if (W.w[(size_t)k * 64 + s * 16 + e] == 0.0) return;
    const int4 o = (s < 2) ? W.orgL[k] : W.orgR[k];
    const int comp = s & 1;
    const int i0 = comp ? o.z : o.x, j0 = comp ? o.w : o.y;
    const int i = wr(i0 + (e & 3), n), j = wr(j0 + (e >> 2), n);
    const int nbk = n >> 2;
    flags[(i >> 2) + (j >> 2) * nbk] = 1;
    if (comp == 0) {
        const int i2 = wr(i - 1, n);
        flags[(i2 >> 2) + (j >> 2) * nbk] = 1;
    } else {
        const int j2 = wr(j - 1, n);
        flags[(i >> 2) + (j2 >> 2) * nbk] = 1;
    }
}

// Nonzero support of window slot s of point k: unwrapped extent (for the
// E' reach) and its owner blocks (a face belongs to the cell on its high side
// and the one below/left) as a 2x2 occupancy over the unwrapped base block
// (bx0, by0): the owners of a 4x4 patch span at most 5 cells per axis, i.e.
// at most two blocks.
struct WinSupport {
    int bx0, by0;
    unsigned occ;  // bit dx + 2 dy
};
__device__ __forceinline__ WinSupport window_support(const Win& W, int k, int s, int& lo_i, int& hi_i, int& lo_j,
                                                     int& hi_j) {
    const int4 o = (s < 2) ? W.orgL[k] : W.orgR[k];
    const int comp = s & 1;
    const int i0 = comp ? o.z : o.x, j0 = comp ? o.w : o.y;
    WinSupport r{(i0 - (comp ? 0 : 1)) >> 2, (j0 - comp) >> 2, 0u};
    const double* p = W.w + (size_t)k * 64 + s * 16;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        if (p[e] == 0.0) continue;
        const int i = i0 + (e & 3), j = j0 + (e >> 2);
        lo_i = min(lo_i, i);
        hi_i = max(hi_i, i);
        lo_j = min(lo_j, j);
        hi_j = max(hi_j, j);
        const int i2 = comp ? i : i - 1, j2 = comp ? j - 1 : j;
        r.occ |= 1u << (((i >> 2) - r.bx0) + 2 * ((j >> 2) - r.by0));
        r.occ |= 1u << (((i2 >> 2) - r.bx0) + 2 * ((j2 >> 2) - r.by0));
    }
    return r;
}

__device__ __forceinline__ int canon_off(int d, int nbk) { return wr(d + nbk / 2, nbk) - nbk / 2; }

// Per point k and component comp (oracle block_pair_masks):
//  * the length-2 couplings of the big-block conflict graph: every pair (A, B)
//    of boxes with A owning a nonzero left-window entry of k and B a nonzero
//    right-window entry of k-1, k or k+1 at canonical Chebyshev offset 2 sets
//    bit (dx+2) + 5 (dy+2) in mask[A] and the mirrored bit in mask[B];
//  * the E' reach: the extent (face index units) of the union of the L_k and
//    R_{k-1}, R_k, R_{k+1} supports, max into *reach (same-colour blocks are
//    >= 8 cells apart only when it is <= 7, checked at setup).
__global__ void k_block_pairs(int npts, WinLevels WL, BlkLevels BK, Pts P, unsigned* __restrict__ mask_all,
                              int* __restrict__ counters, int ctr_stride) {
    pdl_enter();
    const int qq = blockIdx.x * blockDim.x + threadIdx.x;
    if (qq >= npts * 2 * BK.nlev) return;
    const int l = qq / (npts * 2), q = qq - l * npts * 2;
    const Win& W = WL.win[l];
    const int n = BK.n[l];
    unsigned* mask = mask_all + BK.boff[l];
    int* reach = counters + l * ctr_stride + 18;
    const int k = q >> 1, comp = q & 1, nbk = n >> 2;
    int lo_i = 1 << 30, hi_i = -(1 << 30), lo_j = 1 << 30, hi_j = -(1 << 30);
    const WinSupport Ls = window_support(W, k, comp, lo_i, hi_i, lo_j, hi_j);
    const WinSupport Rs[3] = {window_support(W, P.kprev[k], 2 + comp, lo_i, hi_i, lo_j, hi_j),
                              window_support(W, k, 2 + comp, lo_i, hi_i, lo_j, hi_j),
                              window_support(W, P.knext[k], 2 + comp, lo_i, hi_i, lo_j, hi_j)};
    if (hi_i >= lo_i) atomicMax(reach, max(hi_i - lo_i, hi_j - lo_j));
    for (int x = 0; x < 4; ++x) {
        if (!(Ls.occ >> x & 1u)) continue;
        const int ax = Ls.bx0 + (x & 1), ay = Ls.by0 + (x >> 1);
        const int A = wr(ax, nbk) + wr(ay, nbk) * nbk;
        for (int r = 0; r < 3; ++r)
            for (int y = 0; y < 4; ++y) {
                if (!(Rs[r].occ >> y & 1u)) continue;
                const int bx = Rs[r].bx0 + (y & 1), by = Rs[r].by0 + (y >> 1);
                const int dx = canon_off(bx - ax, nbk), dy = canon_off(by - ay, nbk);
                if (max(abs(dx), abs(dy)) != 2) continue;
                const int B = wr(bx, nbk) + wr(by, nbk) * nbk;
                const int ex = canon_off(ax - bx, nbk), ey = canon_off(ay - by, nbk);
                atomicOr(mask + A, 1u << ((dx + 2) + 5 * (dy + 2)));
                atomicOr(mask + B, 1u << ((ex + 2) + 5 * (ey + 2)));
            }
    }
}

// Conflict masks of the big blocks (oracle colour_blocks),
// in place over the k_block_pairs output: for a big block A, bit
// (dx+2) + 5 (dy+2) for every offset (dx, dy) != 0 in [-2, 2]^2 whose block
// B = A + (dx, dy) (periodic) is big, is not A itself, and conflicts with A —
// canonical Chebyshev offset 1, or 2 with the pair bit set — and bit 12
// (the zero offset) marking A big; 0 for blocks that are not big.
__global__ void k_block_conflicts(BlkLevels BK, const uint8_t* __restrict__ big_all, unsigned* __restrict__ mask_all) {
    pdl_enter();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= BK.boff[BK.nlev]) return;
    int l = 0;
    while (g >= BK.boff[l + 1]) ++l;
    const int nbk = BK.n[l] >> 2, A = g - BK.boff[l];
    const uint8_t* big = big_all + BK.boff[l];
    unsigned* mask = mask_all + BK.boff[l];
    if (!big[A]) {
        mask[A] = 0u;
        return;
    }
    const unsigned pairs = mask[A];
    const int ax = A % nbk, ay = A / nbk;
    unsigned m = 1u << 12;
    for (int dy = -2; dy <= 2; ++dy)
        for (int dx = -2; dx <= 2; ++dx) {
            const int B = wr(ax + dx, nbk) + wr(ay + dy, nbk) * nbk;
            if (B == A || !big[B]) continue;
            const int cx = canon_off(dx, nbk), cy = canon_off(dy, nbk);
            const int len = max(abs(cx), abs(cy));
            if (len > 2 || (len == 2 && !(pairs >> ((cx + 2) + 5 * (cy + 2)) & 1u))) continue;
            m |= 1u << ((dx + 2) + 5 * (dy + 2));
        }
    mask[A] = m;
}

// Stand-alone face gather (spread of given forces): face_gather_warp per warp.
__global__ void k_face_gather(FaceList FL, Win W, const double* __restrict__ F, double* __restrict__ out,
                              int nn, double sign) {
    pdl_enter();
    face_gather_warp(FL, W, F, out, nn, sign, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31);
}

// Assembly of E'_l rows for the face lists of all levels in
// one launch: a row is the run q of the batched face lists (k_face_keys);
// entry pairs accumulate into a 16x16 shared-memory patch of column offsets
// (slot = wr(col - row + 8, n); the E' reach is <= 7, checked at setup) in a
// fixed order (entry pairs ascending in point, windows k-1, k, k+1, lower
// half-warp first): deterministic.  pass 0 writes the row's nonzero count,
// pass 1 the (col, val) pairs at rp[q].  Levels whose face lists run long
// (coarse levels: a face there collects many points) take a CTA per row, the
// 16 warps on interleaved entry pairs with private patches summed in warp
// order; the others a warp per row.
constexpr int kEWarps = 16;
struct ERows {
    int nlev;
    Win W[20];
    int n[20];
    int start[21];   // first run of each level; start[nlev] = total runs
    int islong[20];  // CTA per row on this level
    int lstart[21];  // prefix over the long levels' run counts (CTA part)
    int nwarp_cta;   // CTAs of the warp part
};

// Accumulate entry pairs e0, e0 + stride, ... of a row into the patch pt.
__device__ __forceinline__ void erow_accumulate(double* pt, const int* __restrict__ ent, int e_begin, int e_end,
                                                int stride, const Win& W, const Pts& P, int n, int comp, int di,
                                                int dj, int lane) {
    const int half = lane >> 4, e16 = lane & 15;
    for (int e0 = e_begin; e0 < e_end; e0 += stride) {
        const int e = e0 + half;
        const bool act = e < e_end;
        const int v = act ? ent[e] : 0;
        const int k = v >> 5;
        const double lc = act ? W.w[(size_t)k * 64 + (v & 31)] * P.cE[k] : 0.0;
        const int ks[3] = {P.kprev[k], k, P.knext[k]};
        const double coef[3] = {1.0, -2.0, 1.0};
        for (int t = 0; t < 3; ++t) {
            int slot = -1;
            double add = 0.0;
            if (act) {
                const int kk = ks[t];
                const double r = W.w[(size_t)kk * 64 + (2 + comp) * 16 + e16];
                if (r != 0.0) {
                    const int4 o = W.orgR[kk];
                    const int i0 = comp ? o.z : o.x, j0 = comp ? o.w : o.y;
                    const int sx = wr(i0 + (e16 & 3) - di + 8, n), sy = wr(j0 + (e16 >> 2) - dj + 8, n);
                    slot = (sx < 16 && sy < 16) ? sy * 16 + sx : -1;
                    add = lc * coef[t] * r;
                }
            }
            if (half == 0 && slot >= 0) pt[slot] += add;
            __syncwarp();
            if (half == 1 && slot >= 0) pt[slot] += add;
            __syncwarp();
        }
    }
}

// Compact a finished patch (one warp): count (pass 0) or (col, val) pairs.
__device__ __forceinline__ void erow_emit(const double* pt, int q, int pass, int n, int comp, int di, int dj,
                                          int* __restrict__ cnt, const int* __restrict__ rp, int* __restrict__ col,
                                          double* __restrict__ val, int lane) {
    const int nn = n * n;
    int base = pass ? rp[q] : 0;
    for (int y = 0; y < 8; ++y) {
        const int s = y * 32 + lane;
        const double v = pt[s];
        const unsigned m = __ballot_sync(0xffffffffu, v != 0.0);
        if (pass && v != 0.0) {
            const int pos = base + __popc(m & ((1u << lane) - 1u));
            col[pos] = comp * nn + wr(di - 8 + (s & 15), n) + wr(dj - 8 + (s >> 4), n) * n;
            val[pos] = v;
        }
        base += __popc(m);
    }
    if (!pass && lane == 0) cnt[q] = base;
}

__global__ void __launch_bounds__(32 * kEWarps) k_erows(ERows R, const int* __restrict__ face,
                                                         const int* __restrict__ off, const int* __restrict__ ent,
                                                         Pts P, int pass, int* __restrict__ cnt,
                                                         const int* __restrict__ rp, int* __restrict__ col,
                                                         double* __restrict__ val) {
    pdl_enter();
    __shared__ double patch[kEWarps][256];
    __shared__ double fin[256];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool cta_row = (int)blockIdx.x >= R.nwarp_cta;
    int q, l = 0;
    if (!cta_row) {
        q = blockIdx.x * kEWarps + wid;
        if (q >= R.start[R.nlev]) return;
        while (q >= R.start[l + 1]) ++l;
        if (R.islong[l]) return;
    } else {
        const int cq = blockIdx.x - R.nwarp_cta;
        while (cq >= R.lstart[l + 1]) ++l;
        q = R.start[l] + (cq - R.lstart[l]);
    }
    const int n = R.n[l], nn = n * n, fc = face[q];
    if (fc == 2 * nn) {  // the level's sentinel run (zero window weights): no row
        if (!pass && lane == 0 && (!cta_row || wid == 0)) cnt[q] = 0;
        return;
    }
    const int comp = fc >= nn, f = fc - comp * nn, di = f & (n - 1), dj = f / n;
    double* pt = patch[wid];
    for (int s = lane; s < 256; s += 32) pt[s] = 0.0;
    __syncwarp();
    if (!cta_row) {
        erow_accumulate(pt, ent, off[q], off[q + 1], 2, R.W[l], P, n, comp, di, dj, lane);
        erow_emit(pt, q, pass, n, comp, di, dj, cnt, rp, col, val, lane);
        return;
    }
    erow_accumulate(pt, ent, off[q] + 2 * wid, off[q + 1], 2 * kEWarps, R.W[l], P, n, comp, di, dj, lane);
    __syncthreads();
    if (threadIdx.x < 256) {
        double s = 0.0;
        for (int w = 0; w < kEWarps; ++w) s += patch[w][threadIdx.x];
        fin[threadIdx.x] = s;
    }
    __syncthreads();
    if (wid == 0) erow_emit(fin, q, pass, n, comp, di, dj, cnt, rp, col, val, lane);
}

// Fiber force density of the RHS times the spread quadrature:
// F_k ds^2 = kappa (X_{k-1} + X_{k+1} - 2 X_k)/ds^2 * ds^2  (fiber.cpp:34-55, 93).
__global__ void k_rhs_force(Pts P, const double* __restrict__ X, double* __restrict__ F) {
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P.n) return;
    const int km = P.kprev[k], kp = P.knext[k];
    for (int c = 0; c < 2; ++c) {
        const double d = X[2 * km + c] + X[2 * kp + c] - X[2 * k + c] * 2.0;
        F[2 * k + c] = ((d * P.ids2[k]) * P.kap[k]) * P.dsq[k];
    }
}

// Plain spread input scaling: F_k ds_m^2 (ds^2 quadrature, fiber.cpp:93).
__global__ void k_scale_dsq(Pts P, const double* __restrict__ Fin, double* __restrict__ F) {
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= P.n) return;
    F[2 * k] = Fin[2 * k] * P.dsq[k];
    F[2 * k + 1] = Fin[2 * k + 1] * P.dsq[k];
}

// interpolate (fiber.cpp:116-140): U_k = h^2 sum W u; optionally X += dt U.
__global__ void k_interp(Win W, int npts, int n, double h, const double* __restrict__ u, double* __restrict__ U,
                         double* __restrict__ X, double dt) {
    pdl_enter();
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= npts) return;
    GAcc acc{u, n, n * n};
    const double w0 = h * h;
    // fine level: left == right windows; use the right-window dot
    const double Uu = win_dot_R(W, k, 0, n, acc) * w0;
    const double Vv = win_dot_R(W, k, 1, n, acc) * w0;
    if (U) {
        U[2 * k] = Uu;
        U[2 * k + 1] = Vv;
    }
    if (X) {
        X[2 * k] += dt * Uu;
        X[2 * k + 1] += dt * Vv;
    }
}

}  // namespace ibmg
