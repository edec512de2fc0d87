// ibmg_oracle.cpp — CPU oracle (TEST INFRASTRUCTURE ONLY; see ibmg_oracle.h).
//
// Periodic, backward-Euler restatement of the reference solver path.  Every
// routine cites the reference file:line (under /root/reference/proj/core/src
// or /root/reference/SPEC.md) whose semantics it follows.  Sign convention is
// rows are -1 x the reference's, plus rho/dt on the momentum
// diagonal, so the momentum block (rho/dt - mu L - E') is SPD.
#include "ibmg_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle_common.h"

namespace orc {

struct Line {
    long first;
    double w[4];
};
Line line_faces(double X, double h) {
    Line l;
    const double s = X / h;
    l.first = (long)std::ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) l.w[a] = delta_1d(double(l.first + a) * h - X, h);
    return l;
}
Line line_centers(double X, double h) {
    Line l;
    const double s = X / h - 0.5;
    l.first = (long)std::ceil(s - 2.0);
    for (int a = 0; a < 4; ++a) l.w[a] = delta_1d((double(l.first + a) + 0.5) * h - X, h);
    return l;
}

using SpVec = std::vector<std::pair<int, double>>;  // (flat velocity index, weight)

// Node weight tables (elasticity.cpp:16-58), periodic: every face is a DOF.
void node_windows(double X, double Y, int n, double h, SpVec& wu, SpVec& wv) {
    const int nn = n * n;
    wu.clear();
    wv.clear();
    Line lx = line_faces(X, h), ly = line_centers(Y, h);
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
            const double w = lx.w[a] * ly.w[b];
            if (w == 0.0) continue;
            wu.emplace_back(wrap(lx.first + a, n) + wrap(ly.first + b, n) * n, w);
        }
    lx = line_centers(X, h);
    ly = line_faces(Y, h);
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) {
            const double w = lx.w[a] * ly.w[b];
            if (w == 0.0) continue;
            wv.emplace_back(nn + wrap(lx.first + a, n) + wrap(ly.first + b, n) * n, w);
        }
}

// ---- transfers, periodic (transfers.cpp:107-134, 141-232 with the v-weight
// fixed: line 202 emits xs[a].w*w; the correct bilinear weight is ys[b].w*w).
void restrict_saddle(int nf, const double* rf, double* rc) {
    const int nc = nf / 2, nnf = nf * nf, nnc = nc * nc;
    auto fu = [&](long i, long j) { return rf[wrap(i, nf) + wrap(j, nf) * nf]; };
    auto fv = [&](long i, long j) { return rf[nnf + wrap(i, nf) + wrap(j, nf) * nf]; };
    auto fp = [&](long i, long j) { return rf[2 * nnf + wrap(i, nf) + wrap(j, nf) * nf]; };
    for (int J = 0; J < nc; ++J)
        for (int I = 0; I < nc; ++I) {
            const long i = 2 * I, j = 2 * J;
            rc[I + J * nc] = 0.125 * (fu(i - 1, j) + 2.0 * fu(i, j) + fu(i + 1, j) + fu(i - 1, j + 1) +
                                      2.0 * fu(i, j + 1) + fu(i + 1, j + 1));
            rc[nnc + I + J * nc] = 0.125 * (fv(i, j - 1) + 2.0 * fv(i, j) + fv(i, j + 1) +
                                            fv(i + 1, j - 1) + 2.0 * fv(i + 1, j) + fv(i + 1, j + 1));
            rc[2 * nnc + I + J * nc] =
                0.25 * (fp(i, j) + fp(i + 1, j) + fp(i, j + 1) + fp(i + 1, j + 1));
        }
}

struct W2 {
    long I;
    double w;
};
// Bilinear weights of fine face-normal index i (1 or 1/2,1/2) and of the
// tangential index j (3/4,1/4), for_each_u_weight transfers.cpp:141-172.
inline int normal_weights(long i, W2* xs) {
    if (i % 2 == 0) {
        xs[0] = {i / 2, 1.0};
        return 1;
    }
    xs[0] = {(i - 1) / 2, 0.5};
    xs[1] = {(i + 1) / 2, 0.5};
    return 2;
}
inline void tangential_weights(long j, W2* ys) {
    const long J = j / 2;
    ys[0] = {J, 0.75};
    ys[1] = {(j % 2 == 0) ? J - 1 : J + 1, 0.25};
}

void prolong_add(int nf, const double* ec, double* wf) {
    const int nc = nf / 2, nnf = nf * nf, nnc = nc * nc;
    W2 xs[2], ys[2];
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) {
            double acc = 0.0;
            const int nx = normal_weights(i, xs);
            tangential_weights(j, ys);
            for (int a = 0; a < nx; ++a)
                for (int b = 0; b < 2; ++b)
                    acc += xs[a].w * ys[b].w * ec[wrap(xs[a].I, nc) + wrap(ys[b].I, nc) * nc];
            wf[i + j * nf] += acc;
        }
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) {
            double acc = 0.0;
            const int ny = normal_weights(j, ys);
            tangential_weights(i, xs);
            for (int b = 0; b < ny; ++b)
                for (int a = 0; a < 2; ++a)
                    acc += ys[b].w * xs[a].w * ec[nnc + wrap(xs[a].I, nc) + wrap(ys[b].I, nc) * nc];
            wf[nnf + i + j * nf] += acc;
        }
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) wf[2 * nnf + i + j * nf] += ec[2 * nnc + (i / 2) + (j / 2) * nc];
}

// Velocity R and P as matrices (transfers.cpp:234-284), periodic.
Csr velocity_restriction_matrix(int nf) {
    const int nc = nf / 2, nnf = nf * nf, nnc = nc * nc;
    std::vector<Trip> t;
    for (int J = 0; J < nc; ++J)
        for (int I = 0; I < nc; ++I) {
            const long i = 2 * I, j = 2 * J;
            const int r = I + J * nc;
            auto U = [&](long a, long b) { return wrap(a, nf) + wrap(b, nf) * nf; };
            t.push_back({r, U(i - 1, j), 0.125});
            t.push_back({r, U(i, j), 0.25});
            t.push_back({r, U(i + 1, j), 0.125});
            t.push_back({r, U(i - 1, j + 1), 0.125});
            t.push_back({r, U(i, j + 1), 0.25});
            t.push_back({r, U(i + 1, j + 1), 0.125});
            const int rv = nnc + r;
            auto V = [&](long a, long b) { return nnf + wrap(a, nf) + wrap(b, nf) * nf; };
            t.push_back({rv, V(i, j - 1), 0.125});
            t.push_back({rv, V(i, j), 0.25});
            t.push_back({rv, V(i, j + 1), 0.125});
            t.push_back({rv, V(i + 1, j - 1), 0.125});
            t.push_back({rv, V(i + 1, j), 0.25});
            t.push_back({rv, V(i + 1, j + 1), 0.125});
        }
    return Csr::from_trips(2 * nnc, 2 * nnf, t, false);
}
Csr velocity_prolongation_matrix(int nf) {
    const int nc = nf / 2, nnf = nf * nf, nnc = nc * nc;
    std::vector<Trip> t;
    W2 xs[2], ys[2];
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) {
            const int nx = normal_weights(i, xs);
            tangential_weights(j, ys);
            for (int a = 0; a < nx; ++a)
                for (int b = 0; b < 2; ++b)
                    t.push_back({i + j * nf, wrap(xs[a].I, nc) + wrap(ys[b].I, nc) * nc, xs[a].w * ys[b].w});
        }
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) {
            const int ny = normal_weights(j, ys);
            tangential_weights(i, xs);
            for (int b = 0; b < ny; ++b)
                for (int a = 0; a < 2; ++a)
                    t.push_back({nnf + i + j * nf, nnc + wrap(xs[a].I, nc) + wrap(ys[b].I, nc) * nc,
                                 ys[b].w * xs[a].w});
        }
    return Csr::from_trips(2 * nnf, 2 * nnc, t, false);
}

// ---- periodic, negated, mass-augmented Stokes rows (assembly.cpp:13-50).
void stokes_trips(int n, double h, double rho_dt, double mu, std::vector<Trip>& t) {
    const int nn = n * n;
    const double c = mu / (h * h), d = rho_dt + 4.0 * c, g = 1.0 / h;
    auto U = [&](long i, long j) { return wrap(i, n) + wrap(j, n) * n; };
    auto V = [&](long i, long j) { return nn + wrap(i, n) + wrap(j, n) * n; };
    auto P = [&](long i, long j) { return 2 * nn + wrap(i, n) + wrap(j, n) * n; };
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            int r = U(i, j);
            t.push_back({r, r, d});
            t.push_back({r, U(i - 1, j), -c});
            t.push_back({r, U(i + 1, j), -c});
            t.push_back({r, U(i, j - 1), -c});
            t.push_back({r, U(i, j + 1), -c});
            t.push_back({r, P(i, j), g});
            t.push_back({r, P(i - 1, j), -g});
            r = V(i, j);
            t.push_back({r, r, d});
            t.push_back({r, V(i, j - 1), -c});
            t.push_back({r, V(i, j + 1), -c});
            t.push_back({r, V(i - 1, j), -c});
            t.push_back({r, V(i + 1, j), -c});
            t.push_back({r, P(i, j), g});
            t.push_back({r, P(i, j - 1), -g});
            r = P(i, j);
            t.push_back({r, U(i + 1, j), -g});
            t.push_back({r, U(i, j), g});
            t.push_back({r, V(i, j + 1), -g});
            t.push_back({r, V(i, j), g});
        }
}

struct Pass {
    bool big = false;
    std::vector<int> items;  // cell index i + j n, or block index bx + by (n/4)
};

struct Level {
    int n = 0;
    double h = 0.0;
    Csr A;  // full saddle, 3n^2
    Csr E;  // velocity E' (2n^2)
    std::vector<SpVec> Lu, Lv, Ru, Rv;  // per-point left/right windows
    std::vector<char> big;              // per 4x4 block
    std::vector<Pass> passes;
    std::vector<DenseLu> blk;               // factors per block (big only)
    // plain-cell 5x5 factors, cached per level per step: the
    // level's common matrix (constant-coefficient stencil) factored once; a
    // plain cell whose extracted matrix differs in any bit keeps its own
    DenseLu plain_lu;
    std::map<int, DenseLu> plain_own;
    DenseLu coarse;                         // coarsest bordered LU
    std::vector<double> w, b, r;
};

struct Ctx {
    orc_params prm{};
    std::string err;
    std::vector<Level> lev;
    // structures
    std::vector<int> nb, off;
    std::vector<double> kappa, ds, X;
    int npts = 0;
    bool have_structs = false;
};

int box_dofs(const Level& L, bool big, int item, int* d) {
    const int n = L.n, nn = n * n;
    if (!big) {
        const int i = item % n, j = item / n;
        d[0] = i + j * n;
        d[1] = wrap(i + 1, n) + j * n;
        d[2] = nn + i + j * n;
        d[3] = nn + i + wrap(j + 1, n) * n;
        d[4] = 2 * nn + i + j * n;
        return 5;
    }
    const int nbk = n / 4;
    const int bi = 4 * (item % nbk), bj = 4 * (item / nbk);
    int m = 0;
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 5; ++a) d[m++] = wrap(bi + a, n) + wrap(bj + b, n) * n;
    for (int b = 0; b < 5; ++b)
        for (int a = 0; a < 4; ++a) d[m++] = nn + wrap(bi + a, n) + wrap(bj + b, n) * n;
    for (int b = 0; b < 4; ++b)
        for (int a = 0; a < 4; ++a) d[m++] = 2 * nn + (bi + a) + (bj + b) * n;
    return m;  // 56
}

void extract(const Csr& A, const int* d, int m, DenseLu& lu) {
    lu.m = m;
    lu.a.assign(size_t(m) * m, 0.0);
    for (int r = 0; r < m; ++r)
        for (int c = 0; c < m; ++c) lu.a[size_t(r) * m + c] = A.at(d[r], d[c]);
}

// Canonical periodic block offset in [-nbk/2, nbk/2).
inline int canon(int d, int nbk) { return wrap(d + nbk / 2, nbk) - nbk / 2; }

// Big-block conflict graph.  Two big blocks conflict (may
// not share a colour, and the later waits for the earlier) when their
// canonical periodic offset has Chebyshev length 1 (shared faces, stencil
// coupling), or length 2 and E'_l couples their boxes: some point k has a
// nonzero left-window entry on a face of one box and one of k-1, k, k+1 a
// nonzero right-window entry of the same component on a face of the other
// (E'_l = sum_k L_k c_k (R_{k-1} - 2 R_k + R_{k+1}); the E' reach <= 7
// excludes length >= 3).  The length-2 couplings are bit (dx+2) + 5 (dy+2) of
// mask[A]; mirrored by k_block_pairs + colour_big_blocks on the GPU.
std::vector<unsigned> block_pair_masks(const Level& L, const std::vector<int>& kprev, const std::vector<int>& knext) {
    const int n = L.n, nn = n * n, nbk = n / 4;
    std::vector<unsigned> mask(size_t(nbk) * nbk, 0u);
    auto owners = [&](const SpVec& win, std::vector<int>& out) {
        for (auto& e : win) {
            const int f = e.first % nn, i = f % n, j = f / n;
            const bool is_u = e.first < nn;
            const int i2 = is_u ? wrap(i - 1, n) : i, j2 = is_u ? j : wrap(j - 1, n);
            out.push_back((i / 4) + (j / 4) * nbk);
            out.push_back((i2 / 4) + (j2 / 4) * nbk);
        }
    };
    const int npts = int(L.Lu.size());
    std::vector<int> la, ra;
    for (int k = 0; k < npts; ++k)
        for (int comp = 0; comp < 2; ++comp) {
            la.clear();
            ra.clear();
            owners(comp ? L.Lv[k] : L.Lu[k], la);
            for (int kk : {kprev[k], k, knext[k]}) owners(comp ? L.Rv[kk] : L.Ru[kk], ra);
            for (int A : la)
                for (int B : ra) {
                    const int dx = canon(B % nbk - A % nbk, nbk), dy = canon(B / nbk - A / nbk, nbk);
                    if (std::max(std::abs(dx), std::abs(dy)) != 2) continue;
                    const int ex = canon(A % nbk - B % nbk, nbk), ey = canon(A / nbk - B / nbk, nbk);
                    mask[A] |= 1u << ((dx + 2) + 5 * (dy + 2));
                    mask[B] |= 1u << ((ex + 2) + 5 * (ey + 2));
                }
        }
    return mask;
}

// Deterministic colouring of the big blocks over the conflict graph above
// (neighbours listed in offset order dy, dx ascending): DSatur — the block
// with the most distinct neighbour colours, then the highest conflict degree,
// then the most recently queued, takes its smallest free colour — when the
// level has <= kDsaturMax big blocks, else greedy in ascending block id.
// Mirrored exactly by the GPU host (paper_1311_5614_b200/csrc/ibmg.cu).
constexpr int kDsaturMax = 4096;
std::vector<int> colour_blocks(const std::vector<char>& big, const std::vector<unsigned>& mask, int nbk, int* ncol) {
    std::vector<int> ids, pos(big.size(), -1);
    for (int q = 0; q < int(big.size()); ++q)
        if (big[q]) {
            pos[q] = int(ids.size());
            ids.push_back(q);
        }
    const int nb = int(ids.size());
    std::vector<std::vector<int>> adj(nb);
    for (int v = 0; v < nb; ++v) {
        const int A = ids[v], ax = A % nbk, ay = A / nbk;
        for (int dy = -2; dy <= 2; ++dy)
            for (int dx = -2; dx <= 2; ++dx) {
                const int B = wrap(ax + dx, nbk) + wrap(ay + dy, nbk) * nbk;
                if (B == A || !big[B]) continue;
                const int cx = canon(B % nbk - ax, nbk), cy = canon(B / nbk - ay, nbk);
                const int len = std::max(std::abs(cx), std::abs(cy));
                if (len > 2 || (len == 2 && !(mask[A] >> ((cx + 2) + 5 * (cy + 2)) & 1u))) continue;
                if (std::find(adj[v].begin(), adj[v].end(), pos[B]) == adj[v].end()) adj[v].push_back(pos[B]);
            }
    }
    std::vector<int> col(big.size(), -1), cv(nb, -1);
    std::vector<unsigned long long> used(nb, 0ull);
    *ncol = 0;
    auto take = [&](int v) {
        int k = 0;
        while (used[v] >> k & 1ull) ++k;
        cv[v] = k;
        col[ids[v]] = k;
        *ncol = std::max(*ncol, k + 1);
        return k;
    };
    if (nb > kDsaturMax) {
        for (int v = 0; v < nb; ++v) {
            const int k = take(v);
            for (int u : adj[v]) used[u] |= 1ull << k;
        }
        return col;
    }
    // bucket queue on saturation * 32 + degree, last pushed first within a
    // bucket (stale entries skipped), as the GPU host
    std::vector<int> sat(nb, 0);
    std::vector<std::vector<int>> bucket(32 * 32);
    auto key = [&](int v) { return sat[v] * 32 + int(adj[v].size()); };
    for (int v = 0; v < nb; ++v) bucket[key(v)].push_back(v);
    for (int done = 0; done < nb;) {
        int top = 32 * 32 - 1;
        while (bucket[top].empty()) --top;
        const int v = bucket[top].back();
        bucket[top].pop_back();
        if (cv[v] >= 0 || key(v) != top) continue;
        const int k = take(v);
        ++done;
        for (int u : adj[v]) {
            if (cv[u] >= 0 || (used[u] >> k & 1ull)) continue;
            used[u] |= 1ull << k;
            ++sat[u];
            bucket[key(u)].push_back(u);
        }
    }
    return col;
}

// Fixed multicolour schedule.  Plain phase: 16x16-cell
// tiles coloured 2x2 (one tile, periodic, when n <= 32); inside each tile the
// 8 conflict-free colours (i + 2j) mod 8 of local coordinates over cells
// outside big blocks.  Big phase: the greedy colour classes of the big blocks
// in colour order.  Boxes within one pass are mutually independent, so each
// pass is exactly a Gauss-Seidel pass in any order (SPEC.md:427-431
// semantics) and the GPU runs it in parallel.
void build_schedule(Level& L, const std::vector<int>& kprev, const std::vector<int>& knext) {
    // levels n <= 32 (one CTA on the GPU) colour the whole periodic level
    // (i + 2j) mod 8 — valid across the seam since 8 | n — instead of tiling
    const int n = L.n, T = n <= 32 ? n : 16, nt = n / T, nbk = n / 4;
    L.passes.clear();
    const int ntc = nt >= 2 ? 4 : 1;
    for (int tc = 0; tc < ntc; ++tc) {
        auto tile_ok = [&](int tx, int ty) { return ntc == 1 || ((tx % 2) + 2 * (ty % 2)) == tc; };
        for (int pc = 0; pc < 8; ++pc) {
            Pass p;
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    if (!tile_ok(i / T, j / T)) continue;
                    const int li = i % T, lj = j % T;
                    if ((li + 2 * lj) % 8 != pc) continue;
                    if (L.big[(i / 4) + (j / 4) * nbk]) continue;
                    p.items.push_back(i + j * n);
                }
            if (!p.items.empty()) L.passes.push_back(std::move(p));
        }
    }
    int ncol = 0;
    const std::vector<int> col = colour_blocks(L.big, block_pair_masks(L, kprev, knext), nbk, &ncol);
    for (int bc = 0; bc < ncol; ++bc) {
        Pass p;
        p.big = true;
        for (int q = 0; q < nbk * nbk; ++q)
            if (col[q] == bc) p.items.push_back(q);
        if (!p.items.empty()) L.passes.push_back(std::move(p));
    }
}

void mark_big(Level& L, int npts) {
    const int n = L.n, nn = n * n, nbk = n / 4;
    L.big.assign(size_t(nbk) * nbk, 0);
    auto mark_face = [&](int idx) {
        const int f = idx % nn;
        const int i = f % n, j = f / n;
        // a face belongs to the cell on its high side and the one below/left
        const bool is_u = idx < nn;
        const int i2 = is_u ? wrap(i - 1, n) : i, j2 = is_u ? j : wrap(j - 1, n);
        L.big[(i / 4) + (j / 4) * nbk] = 1;
        L.big[(i2 / 4) + (j2 / 4) * nbk] = 1;
    };
    for (int k = 0; k < npts; ++k) {
        for (auto& e : L.Lu[k]) mark_face(e.first);
        for (auto& e : L.Lv[k]) mark_face(e.first);
        for (auto& e : L.Ru[k]) mark_face(e.first);
        for (auto& e : L.Rv[k]) mark_face(e.first);
    }
}

SpVec sp_apply_rows(const Csr& M, const SpVec& x) {  // y = M^T-style scatter: y[c] += x[r]*M(r,c)
    std::map<int, double> acc;
    for (auto& e : x)
        for (long k = M.rp[e.first]; k < M.rp[e.first + 1]; ++k) acc[M.ci[k]] += e.second * M.v[k];
    SpVec y;
    for (auto& a : acc)
        if (a.second != 0.0) y.emplace_back(a.first, a.second);
    return y;
}

Csr transpose(const Csr& M) {
    std::vector<Trip> t;
    for (int r = 0; r < M.nr; ++r)
        for (long k = M.rp[r]; k < M.rp[r + 1]; ++k) t.push_back({M.ci[k], r, M.v[k]});
    return Csr::from_trips(M.nc, M.nr, t, false);
}

void build(Ctx& C) {
    const orc_params& p = C.prm;
    const double rho_dt = p.rho / p.dt;
    C.lev.clear();
    int n = p.N;
    while (true) {
        Level L;
        L.n = n;
        L.h = 1.0 / n;
        L.w.assign(size_t(3) * n * n, 0.0);
        L.b = L.w;
        L.r = L.w;
        C.lev.push_back(std::move(L));
        if (n <= p.coarsest_n) break;
        n /= 2;
    }
    const int nl = int(C.lev.size());
    const int npts = C.npts;
    // closed-curve neighbours of every point (membrane-local, periodic in s1)
    std::vector<int> kprev(npts), knext(npts);
    for (size_t m = 0; m < C.nb.size(); ++m)
        for (int k = 0; k < C.nb[m]; ++k) {
            kprev[C.off[m] + k] = C.off[m] + (k == 0 ? C.nb[m] - 1 : k - 1);
            knext[C.off[m] + k] = C.off[m] + (k == C.nb[m] - 1 ? 0 : k + 1);
        }
    // fine windows + E' (elasticity.cpp:62-107, with per-membrane kappa and dt)
    {
        Level& L = C.lev[0];
        const int nn = L.n * L.n;
        L.Lu.resize(npts);
        L.Lv.resize(npts);
        for (int k = 0; k < npts; ++k) node_windows(C.X[2 * k], C.X[2 * k + 1], L.n, L.h, L.Lu[k], L.Lv[k]);
        L.Ru = L.Lu;
        L.Rv = L.Lv;
        std::vector<Trip> t;
        for (size_t m = 0; m < C.nb.size(); ++m) {
            const int nbm = C.nb[m], o = C.off[m];
            const double ids2 = 1.0 / (C.ds[m] * C.ds[m]);
            const double scale = p.dt * C.kappa[m] * C.ds[m] * C.ds[m] * L.h * L.h;
            const double coef[3] = {ids2, -2.0 * ids2, ids2};
            for (int comp = 0; comp < 2; ++comp) {
                const std::vector<SpVec>& W = comp == 0 ? L.Lu : L.Lv;
                for (int k = 0; k < nbm; ++k) {
                    const int km = o + (k == 0 ? nbm - 1 : k - 1), kc = o + k,
                              kp = o + (k == nbm - 1 ? 0 : k + 1);
                    const SpVec* cols[3] = {&W[km], &W[kc], &W[kp]};
                    for (auto& [ri, rw] : W[kc])
                        for (int c = 0; c < 3; ++c)
                            for (auto& [cj, cw] : *cols[c]) t.push_back({ri, cj, scale * rw * coef[c] * cw});
                }
            }
        }
        L.E = Csr::from_trips(2 * nn, 2 * nn, t, false);
    }
    // coarse windows and Galerkin E' (transfers.cpp:286-293; PAPER Eq. 20)
    for (int l = 0; l + 1 < nl; ++l) {
        Level& F = C.lev[l];
        Level& G = C.lev[l + 1];
        Csr R = velocity_restriction_matrix(F.n);
        Csr P = velocity_prolongation_matrix(F.n);
        Csr Rt = transpose(R);
        G.Lu.resize(npts);
        G.Lv.resize(npts);
        G.Ru.resize(npts);
        G.Rv.resize(npts);
        for (int k = 0; k < npts; ++k) {
            G.Lu[k] = sp_apply_rows(Rt, F.Lu[k]);
            G.Lv[k] = sp_apply_rows(Rt, F.Lv[k]);
            G.Ru[k] = sp_apply_rows(P, F.Ru[k]);
            G.Rv[k] = sp_apply_rows(P, F.Rv[k]);
        }
        Csr RE = spgemm(R, F.E);
        G.E = spgemm(RE, P);
    }
    // assembled level operators, marking, schedule, factors
    for (int l = 0; l < nl; ++l) {
        Level& L = C.lev[l];
        const int nn = L.n * L.n;
        std::vector<Trip> t;
        stokes_trips(L.n, L.h, rho_dt, p.mu, t);
        for (int r = 0; r < L.E.nr; ++r)
            for (long k = L.E.rp[r]; k < L.E.rp[r + 1]; ++k) t.push_back({r, L.E.ci[k], -L.E.v[k]});
        L.A = Csr::from_trips(3 * nn, 3 * nn, t, false);
        if (l == nl - 1) {
            // bordered dense LU with the mean-zero pressure constraint
            const int m = 3 * nn + 1;
            L.coarse.m = m;
            L.coarse.a.assign(size_t(m) * m, 0.0);
            for (int r = 0; r < 3 * nn; ++r)
                for (long k = L.A.rp[r]; k < L.A.rp[r + 1]; ++k) L.coarse.a[size_t(r) * m + L.A.ci[k]] = L.A.v[k];
            for (int q = 0; q < nn; ++q) {
                L.coarse.a[size_t(2 * nn + q) * m + 3 * nn] = 1.0;
                L.coarse.a[size_t(3 * nn) * m + 2 * nn + q] = 1.0;
            }
            if (!L.coarse.factor()) throw std::runtime_error("coarsest operator singular");
            continue;
        }
        mark_big(L, npts);
        build_schedule(L, kprev, knext);
        L.blk.assign(L.big.size(), DenseLu{});
        // independent per block / per cell: OpenMP (each factor is the same
        // sequential arithmetic whichever thread runs it)
        int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
        for (long bkk = 0; bkk < long(L.big.size()); ++bkk) {
            if (!L.big[bkk]) continue;
            int d[56];
            const int m = box_dofs(L, true, int(bkk), d);
            extract(L.A, d, m, L.blk[bkk]);
            if (!L.blk[bkk].factor()) bad |= 1;
        }
        if (bad) throw std::runtime_error("big-box local matrix singular");
        L.plain_own.clear();
        L.plain_lu = DenseLu{};
        std::vector<int> plain;
        for (const Pass& ps : L.passes)
            if (!ps.big) plain.insert(plain.end(), ps.items.begin(), ps.items.end());
        if (!plain.empty()) {
            int d[56];
            const int m = box_dofs(L, false, plain[0], d);
            extract(L.A, d, m, L.plain_lu);
            L.plain_lu.a0 = L.plain_lu.a;
            if (!L.plain_lu.factor()) throw std::runtime_error("plain-cell local matrix singular");
        }
#pragma omp parallel for schedule(static) reduction(| : bad)
        for (long t = 1; t < long(plain.size()); ++t) {
            int d[56];
            const int m = box_dofs(L, false, plain[t], d);
            DenseLu lu;
            extract(L.A, d, m, lu);
            if (std::memcmp(lu.a.data(), L.plain_lu.a0.data(), sizeof(double) * 25) != 0) {
                if (!lu.factor()) bad |= 1;
#pragma omp critical(plain_own)
                L.plain_own.emplace(plain[t], std::move(lu));
            }
        }
        if (bad) throw std::runtime_error("plain-cell local matrix singular");
    }
}

void apply_level(const Level& L, const double* w, double* out) {
    const int m = L.A.nr;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < m; ++r) out[r] = L.A.row_dot(r, w);
}
void residual_level(const Level& L, const double* b, const double* w, double* r) {
    const int m = L.A.nr;
#pragma omp parallel for schedule(static)
    for (int q = 0; q < m; ++q) r[q] = b[q] - L.A.row_dot(q, w);
}

// One multiplicative box sweep: residual rows of the box,
// exact local solve, immediate correction.
void sweep(const Level& L, const double* b, double* w) {
    for (const Pass& ps : L.passes) {
        const int cnt = int(ps.items.size());
#pragma omp parallel for schedule(static)
        for (int t = 0; t < cnt; ++t) {
            int d[56];
            double rr[56];
            const int item = ps.items[t];
            const int m = box_dofs(L, ps.big, item, d);
            for (int a = 0; a < m; ++a) rr[a] = b[d[a]] - L.A.row_dot(d[a], w);
            if (ps.big) {
                L.blk[item].solve(rr);
            } else {  // the cached factors (identical arithmetic to factoring here)
                auto it = L.plain_own.find(item);
                (it == L.plain_own.end() ? L.plain_lu : it->second).solve(rr);
            }
            for (int a = 0; a < m; ++a) w[d[a]] += rr[a];
        }
    }
}

void coarse_solve(const Level& L, const double* b, double* x) {
    const int m = L.coarse.m;
    std::vector<double> y(m, 0.0);
    for (int q = 0; q < m - 1; ++q) y[q] = b[q];
    L.coarse.solve(y.data());
    for (int q = 0; q < m - 1; ++q) x[q] = y[q];
}

void project_pressure_mean(double* x, int n) {  // fields.cpp:78-85
    const int nn = n * n;
    double mean = 0.0;
    for (int k = 0; k < nn; ++k) mean += x[2 * nn + k];
    mean /= nn;
    for (int k = 0; k < nn; ++k) x[2 * nn + k] -= mean;
}

// Algorithm 1, zero initial guess.
void vcycle_rec(Ctx& C, int l) {
    Level& L = C.lev[l];
    const int nl = int(C.lev.size());
    if (l == nl - 1) {
        coarse_solve(L, L.b.data(), L.w.data());
        return;
    }
    std::fill(L.w.begin(), L.w.end(), 0.0);
    for (int s = 0; s < C.prm.nu1; ++s) sweep(L, L.b.data(), L.w.data());
    residual_level(L, L.b.data(), L.w.data(), L.r.data());
    restrict_saddle(L.n, L.r.data(), C.lev[l + 1].b.data());
    vcycle_rec(C, l + 1);
    prolong_add(L.n, C.lev[l + 1].w.data(), L.w.data());
    for (int s = 0; s < C.prm.nu2; ++s) sweep(L, L.b.data(), L.w.data());
}

// project = false inside FGMRES: a constant pressure is in the null space of
// the periodic operator (G 1 = 0; E' and the mass term act on velocity), so
// A z does not see z's pressure mean and the solution's mean is removed once
// at the end.  The stand-alone V-cycle projects.
void vcycle(Ctx& C, const double* b, double* z, bool project = true) {
    Level& L = C.lev[0];
    std::copy(b, b + L.b.size(), L.b.begin());
    vcycle_rec(C, 0);
    std::copy(L.w.begin(), L.w.end(), z);
    if (project) project_pressure_mean(z, L.n);
}

double dotv(const std::vector<double>& a, const std::vector<double>& b) {  // fields.cpp:87-92
    double s = 0.0;
    for (size_t k = 0; k < a.size(); ++k) s += a[k] * b[k];
    return s;
}

// FGMRES(m), right preconditioned, x0 = 0, classical Gram-Schmidt with one
// full reorthogonalisation pass (CGS2, SPEC.md:510 allows MGS or CGS2),
// convergence on the true residual.
int fgmres(Ctx& C, const double* bptr, double* xptr, orc_stats* st, double* hist, int hist_len) {
    Level& L = C.lev[0];
    const size_t M = L.b.size();
    const int m = C.prm.restart;
    std::vector<double> b(bptr, bptr + M), x(M, 0.0), r(M), w(M);
    // basis vectors allocated on first use: a solve that converges in k steps
    // touches k + 1 V and k Z vectors (C4: 35 of 61 x 1.6 GB)
    std::vector<std::vector<double>> V(m + 1), Z(m);
    std::vector<double> H(size_t(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), h1(m + 1);
    const double bnorm = std::sqrt(dotv(b, b));
    int it = 0, restarts = 0, hn = 0;
    st->iters = 0;
    st->restarts = 0;
    st->converged = 0;
    st->relres = 0.0;
    if (bnorm == 0.0) {
        std::fill(xptr, xptr + M, 0.0);
        st->converged = 1;
        return 0;
    }
    r = b;
    double beta = bnorm;
    const double tol = C.prm.rtol * bnorm;
    while (true) {
        V[0].resize(M);
        for (size_t q = 0; q < M; ++q) V[0][q] = r[q] / beta;
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int j = 0, kdim = 0;
        for (; j < m; ++j) {
            Z[j].resize(M);
            vcycle(C, V[j].data(), Z[j].data(), false);
            apply_level(L, Z[j].data(), w.data());
            for (int pass = 0; pass < 2; ++pass) {
                for (int i = 0; i <= j; ++i) h1[i] = dotv(V[i], w);
                for (int i = 0; i <= j; ++i) {
                    const double hi = h1[i];
                    for (size_t q = 0; q < M; ++q) w[q] -= hi * V[i][q];
                }
                for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = (pass == 0 ? 0.0 : H[size_t(i) * m + j]) + h1[i];
            }
            const double hnext = std::sqrt(dotv(w, w));
            H[size_t(j + 1) * m + j] = hnext;
            for (int i = 0; i < j; ++i) {
                const double a = H[size_t(i) * m + j], c = H[size_t(i + 1) * m + j];
                H[size_t(i) * m + j] = cs[i] * a + sn[i] * c;
                H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
            }
            const double a = H[size_t(j) * m + j], c = H[size_t(j + 1) * m + j];
            const double den = std::hypot(a, c);
            cs[j] = a / den;
            sn[j] = c / den;
            H[size_t(j) * m + j] = den;
            H[size_t(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            ++it;
            kdim = j + 1;
            if (hist && hn < hist_len) hist[hn++] = std::fabs(g[j + 1]) / bnorm;
            if (std::fabs(g[j + 1]) <= tol || it >= C.prm.max_iters || hnext == 0.0) break;
            V[j + 1].resize(M);
            for (size_t q = 0; q < M; ++q) V[j + 1][q] = w[q] / hnext;
        }
        for (int i = kdim - 1; i >= 0; --i) {
            double s = g[i];
            for (int k = i + 1; k < kdim; ++k) s -= H[size_t(i) * m + k] * y[k];
            y[i] = s / H[size_t(i) * m + i];
        }
        for (int i = 0; i < kdim; ++i)
            for (size_t q = 0; q < M; ++q) x[q] += y[i] * Z[i][q];
        residual_level(L, b.data(), x.data(), r.data());
        beta = std::sqrt(dotv(r, r));
        if (beta <= tol) {
            st->converged = 1;
            break;
        }
        if (it >= C.prm.max_iters) break;
        ++restarts;
    }
    project_pressure_mean(x.data(), L.n);
    std::copy(x.begin(), x.end(), xptr);
    st->iters = it;
    st->restarts = restarts;
    st->relres = beta / bnorm;
    return st->converged ? 0 : 2;
}

// fiber_force + spread (fiber.cpp:34-55, 89-114), periodic, ds^2 quadrature.
void spread_fine(const Ctx& C, const double* F, double* f) {
    const Level& L = C.lev[0];
    const int n = L.n, nn = n * n;
    std::fill(f, f + 2 * nn, 0.0);
    for (size_t m = 0; m < C.nb.size(); ++m) {
        const double w0 = C.ds[m] * C.ds[m];
        for (int k = C.off[m]; k < C.off[m] + C.nb[m]; ++k) {
            const double X = C.X[2 * k], Y = C.X[2 * k + 1];
            Line ux = line_faces(X, L.h), uy = line_centers(Y, L.h);
            for (int b = 0; b < 4; ++b)
                for (int a = 0; a < 4; ++a)
                    f[wrap(ux.first + a, n) + wrap(uy.first + b, n) * n] += F[2 * k] * ux.w[a] * uy.w[b] * w0;
            Line vx = line_centers(X, L.h), vy = line_faces(Y, L.h);
            for (int b = 0; b < 4; ++b)
                for (int a = 0; a < 4; ++a)
                    f[nn + wrap(vx.first + a, n) + wrap(vy.first + b, n) * n] +=
                        F[2 * k + 1] * vx.w[a] * vy.w[b] * w0;
        }
    }
}

void interp_fine(const Ctx& C, const double* u, double* U) {  // fiber.cpp:116-140
    const Level& L = C.lev[0];
    const int n = L.n, nn = n * n;
    const double w0 = L.h * L.h;
    for (int k = 0; k < C.npts; ++k) {
        const double X = C.X[2 * k], Y = C.X[2 * k + 1];
        Line ux = line_faces(X, L.h), uy = line_centers(Y, L.h);
        double Uu = 0.0;
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a) Uu += u[wrap(ux.first + a, n) + wrap(uy.first + b, n) * n] * ux.w[a] * uy.w[b];
        Line vx = line_centers(X, L.h), vy = line_faces(Y, L.h);
        double Vv = 0.0;
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a)
                Vv += u[nn + wrap(vx.first + a, n) + wrap(vy.first + b, n) * n] * vx.w[a] * vy.w[b];
        U[2 * k] = Uu * w0;
        U[2 * k + 1] = Vv * w0;
    }
}

void fiber_force(const Ctx& C, double* F) {
    for (size_t m = 0; m < C.nb.size(); ++m) {
        const int nbm = C.nb[m], o = C.off[m];
        const double ids2 = 1.0 / (C.ds[m] * C.ds[m]);
        for (int k = 0; k < nbm; ++k) {
            const int km = o + (k == 0 ? nbm - 1 : k - 1), kc = o + k, kp = o + (k == nbm - 1 ? 0 : k + 1);
            for (int c = 0; c < 2; ++c) {
                const double d = C.X[2 * km + c] + C.X[2 * kp + c] - C.X[2 * kc + c] * 2.0;
                F[2 * kc + c] = (d * ids2) * C.kappa[m];
            }
        }
    }
}

void rhs(const Ctx& C, const double* u_n, double* b) {
    const Level& L = C.lev[0];
    const int nn = L.n * L.n;
    std::vector<double> F(2 * size_t(C.npts)), f(2 * size_t(nn));
    fiber_force(C, F.data());
    spread_fine(C, F.data(), f.data());
    const double rho_dt = C.prm.rho / C.prm.dt;
    for (int q = 0; q < 2 * nn; ++q) b[q] = rho_dt * u_n[q] + f[q];
    for (int q = 0; q < nn; ++q) b[2 * nn + q] = 0.0;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace orc

using namespace orc;

#define ORC_TRY(ctx, body)                       \
    try {                                        \
        body;                                    \
        return 0;                                \
    } catch (const std::exception& e) {          \
        static_cast<Ctx*>(ctx)->err = e.what();  \
        return 1;                                \
    }

extern "C" {

void* orc_create(const orc_params* p, char* err, int errlen) {
    auto fail = [&](const char* m) -> void* {
        if (err && errlen > 0) std::snprintf(err, errlen, "%s", m);
        return nullptr;
    };
    if (!p) return fail("null params");
    if (p->N < 8 || (p->N & (p->N - 1))) return fail("N must be a power of two >= 8");
    if (!(p->rho > 0 && p->mu > 0 && p->dt > 0)) return fail("rho, mu, dt must be positive");
    if (p->coarsest_n != 4) return fail("coarsest_n must be 4");
    if (p->restart < 1 || p->max_iters < 1 || !(p->rtol > 0 && p->rtol < 1)) return fail("bad Krylov params");
    Ctx* C = new Ctx;
    C->prm = *p;
#ifdef _OPENMP
    omp_set_num_threads(std::max(1, p->threads));
#endif
    try {
        build(*C);
    } catch (const std::exception& e) {
        delete C;
        return fail(e.what());
    }
    return C;
}

void orc_destroy(void* ctx) { delete static_cast<Ctx*>(ctx); }
const char* orc_last_error(void* ctx) { return static_cast<Ctx*>(ctx)->err.c_str(); }

int orc_set_structures(void* ctx, int n_mem, const int* nb, const double* kappa, const double* ds,
                       const double* X) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    ORC_TRY(ctx, {
        C.nb.assign(nb, nb + n_mem);
        C.kappa.assign(kappa, kappa + n_mem);
        C.ds.assign(ds, ds + n_mem);
        C.off.assign(n_mem, 0);
        int tot = 0;
        for (int m = 0; m < n_mem; ++m) {
            if (nb[m] < 3) throw std::invalid_argument("membrane needs >= 3 points");
            if (!(ds[m] > 0)) throw std::invalid_argument("ds must be positive");
            if (kappa[m] < 0) throw std::invalid_argument("kappa must be >= 0");
            C.off[m] = tot;
            tot += nb[m];
        }
        C.npts = tot;
        C.X.assign(X, X + 2 * size_t(tot));
        build(C);
        C.have_structs = true;
    });
}

int orc_num_levels(void* ctx) { return int(static_cast<Ctx*>(ctx)->lev.size()); }
int orc_level_n(void* ctx, int l) { return static_cast<Ctx*>(ctx)->lev.at(l).n; }

int orc_apply(void* ctx, int level, const double* w, double* out) {
    ORC_TRY(ctx, apply_level(static_cast<Ctx*>(ctx)->lev.at(level), w, out));
}
int orc_residual(void* ctx, int level, const double* b, const double* w, double* r) {
    ORC_TRY(ctx, residual_level(static_cast<Ctx*>(ctx)->lev.at(level), b, w, r));
}
int orc_sweep(void* ctx, int level, const double* b, double* w) {
    ORC_TRY(ctx, {
        Ctx& C = *static_cast<Ctx*>(ctx);
        if (level >= int(C.lev.size()) - 1) throw std::invalid_argument("no sweep on the coarsest level");
        sweep(C.lev[level], b, w);
    });
}
int orc_vcycle(void* ctx, const double* b, double* z) { ORC_TRY(ctx, vcycle(*static_cast<Ctx*>(ctx), b, z)); }
int orc_coarse_solve(void* ctx, const double* b, double* x) {
    ORC_TRY(ctx, coarse_solve(static_cast<Ctx*>(ctx)->lev.back(), b, x));
}
int orc_restrict(int nf, const double* rf, double* rc) {
    if (nf < 2 || nf % 2) return 1;
    restrict_saddle(nf, rf, rc);
    return 0;
}
int orc_prolong_add(int nf, const double* ec, double* wf) {
    if (nf < 2 || nf % 2) return 1;
    prolong_add(nf, ec, wf);
    return 0;
}

long orc_elasticity_triplets(void* ctx, int level, int* rows, int* cols, double* vals, long cap) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    const Csr& E = C.lev.at(level).E;
    long q = 0;
    for (int r = 0; r < E.nr; ++r)
        for (long k = E.rp[r]; k < E.rp[r + 1]; ++k, ++q)
            if (q < cap) {
                rows[q] = r;
                cols[q] = E.ci[k];
                vals[q] = E.v[k];
            }
    return q;
}

int orc_big_blocks(void* ctx, int level, int* flags) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    const Level& L = C.lev.at(level);
    int c = 0;
    for (size_t q = 0; q < L.big.size(); ++q) {
        if (flags) flags[q] = L.big[q];
        c += L.big[q];
    }
    return c;
}

int orc_rhs(void* ctx, const double* u_n, double* b) { ORC_TRY(ctx, rhs(*static_cast<Ctx*>(ctx), u_n, b)); }
int orc_interp(void* ctx, const double* u, double* U) { ORC_TRY(ctx, interp_fine(*static_cast<Ctx*>(ctx), u, U)); }
int orc_spread(void* ctx, const double* F, double* f) { ORC_TRY(ctx, spread_fine(*static_cast<Ctx*>(ctx), F, f)); }

int orc_solve(void* ctx, const double* b, double* x, orc_stats* st, double* hist, int hist_len) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    orc_stats local{};
    if (!st) st = &local;
    try {
        const double t0 = now_ms();
        const int rc = fgmres(C, b, x, st, hist, hist_len);
        st->solve_ms = now_ms() - t0;
        return rc;
    } catch (const std::exception& e) {
        C.err = e.what();
        return 1;
    }
}

// step_implicit: operators lagged at X^n, X^{n+1} = X^n + dt S* u^{n+1}.
int orc_step(void* ctx, double* u, double* p, double* X, orc_stats* st) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    orc_stats local{};
    if (!st) st = &local;
    try {
        const double t0 = now_ms();
        std::copy(X, X + 2 * size_t(C.npts), C.X.begin());
        build(C);
        const int N = C.prm.N, nn = N * N;
        std::vector<double> b(3 * size_t(nn)), x(3 * size_t(nn)), U(2 * size_t(C.npts));
        rhs(C, u, b.data());
        const double t1 = now_ms();
        const int rc = fgmres(C, b.data(), x.data(), st, nullptr, 0);
        const double t2 = now_ms();
        std::copy(x.begin(), x.begin() + 2 * nn, u);
        std::copy(x.begin() + 2 * nn, x.end(), p);
        interp_fine(C, u, U.data());
        for (int k = 0; k < 2 * C.npts; ++k) X[k] += C.prm.dt * U[k];
        st->setup_ms = t1 - t0;
        st->solve_ms = t2 - t1;
        st->total_ms = now_ms() - t0;
        return rc;
    } catch (const std::exception& e) {
        C.err = e.what();
        return 1;
    }
}

}  // extern "C"
