// paper_oracle.cpp — CPU oracle of the Dirichlet paper-reproduction mode (TEST
// INFRASTRUCTURE ONLY; see paper_oracle.h).  Every routine cites the reference
// file:line (under /root/reference/proj/core/src, or SPEC.md / PAPER.md) whose
// semantics it restates.  Sign convention and DOF ordering are the reference's.
#include "paper_oracle.h"

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "oracle_common.h"

namespace porc {

using orc::Csr;
using orc::DenseLu;
using orc::Trip;

// geometry.hpp:54-76: interior u faces, interior v faces, cells; x fastest.
struct Dof {
    int n = 0;
    int nu() const { return (n - 1) * n; }
    int nv() const { return n * (n - 1); }
    int np() const { return n * n; }
    int nvel() const { return nu() + nv(); }
    int ntot() const { return nvel() + np(); }
    int u(int i, int j) const { return (i - 1) + j * (n - 1); }      // i in [1, n-1], j in [0, n)
    int v(int i, int j) const { return nu() + i + (j - 1) * n; }     // i in [0, n), j in [1, n-1]
    int p(int i, int j) const { return nvel() + i + j * n; }
};

// fiber.cpp:58-87: kernel lines clipped to the grid's index range.
struct Line {
    int first = 0, count = 0;
    double w[4] = {0, 0, 0, 0};
};
Line line_faces(double X, double h, int n) {
    Line l;
    const double s = X / h;
    int lo = (int)std::ceil(s - 2.0), hi = (int)std::floor(s + 2.0);
    lo = std::max(lo, 0);
    hi = std::min(hi, n);
    l.first = lo;
    for (int idx = lo; idx <= hi && l.count < 4; ++idx) l.w[l.count++] = orc::delta_1d(idx * h - X, h);
    return l;
}
Line line_centers(double X, double h, int n) {
    Line l;
    const double s = X / h - 0.5;
    int lo = (int)std::ceil(s - 2.0), hi = (int)std::floor(s + 2.0);
    lo = std::max(lo, 0);
    hi = std::min(hi, n - 1);
    l.first = lo;
    for (int idx = lo; idx <= hi && l.count < 4; ++idx) l.w[l.count++] = orc::delta_1d((idx + 0.5) * h - X, h);
    return l;
}

using SpVec = std::vector<std::pair<int, double>>;

// elasticity.cpp:16-58 (collect_u_weights / collect_v_weights).
void node_weights(double X, double Y, const Dof& d, double h, SpVec& wu, SpVec& wv) {
    wu.clear();
    wv.clear();
    Line lx = line_faces(X, h, d.n), ly = line_centers(Y, h, d.n);
    for (int b = 0; b < ly.count; ++b)
        for (int a = 0; a < lx.count; ++a) {
            const int i = lx.first + a;
            const double w = lx.w[a] * ly.w[b];
            if (w == 0.0 || i < 1 || i > d.n - 1) continue;
            wu.emplace_back(d.u(i, ly.first + b), w);
        }
    lx = line_centers(X, h, d.n);
    ly = line_faces(Y, h, d.n);
    for (int b = 0; b < ly.count; ++b)
        for (int a = 0; a < lx.count; ++a) {
            const int j = ly.first + b;
            const double w = lx.w[a] * ly.w[b];
            if (w == 0.0 || j < 1 || j > d.n - 1) continue;
            wv.emplace_back(d.v(lx.first + a, j), w);
        }
}

// assembly.cpp:13-50: the Stokes rows with homogeneous walls.
void stokes_trips(const Dof& d, double h, std::vector<Trip>& t) {
    const int n = d.n;
    const double ih2 = 1.0 / (h * h), ih = 1.0 / h;
    for (int j = 0; j < n; ++j)
        for (int i = 1; i <= n - 1; ++i) {
            const int r = d.u(i, j);
            double diag = -4.0;
            if (i > 1) t.push_back({r, d.u(i - 1, j), ih2});
            if (i < n - 1) t.push_back({r, d.u(i + 1, j), ih2});
            if (j > 0) t.push_back({r, d.u(i, j - 1), ih2}); else diag -= 1.0;
            if (j < n - 1) t.push_back({r, d.u(i, j + 1), ih2}); else diag -= 1.0;
            t.push_back({r, r, diag * ih2});
            t.push_back({r, d.p(i, j), -ih});
            t.push_back({r, d.p(i - 1, j), ih});
        }
    for (int j = 1; j <= n - 1; ++j)
        for (int i = 0; i < n; ++i) {
            const int r = d.v(i, j);
            double diag = -4.0;
            if (j > 1) t.push_back({r, d.v(i, j - 1), ih2});
            if (j < n - 1) t.push_back({r, d.v(i, j + 1), ih2});
            if (i > 0) t.push_back({r, d.v(i - 1, j), ih2}); else diag -= 1.0;
            if (i < n - 1) t.push_back({r, d.v(i + 1, j), ih2}); else diag -= 1.0;
            t.push_back({r, r, diag * ih2});
            t.push_back({r, d.p(i, j), -ih});
            t.push_back({r, d.p(i, j - 1), ih});
        }
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int r = d.p(i, j);
            if (i + 1 <= n - 1) t.push_back({r, d.u(i + 1, j), ih});
            if (i >= 1) t.push_back({r, d.u(i, j), -ih});
            if (j + 1 <= n - 1) t.push_back({r, d.v(i, j + 1), ih});
            if (j >= 1) t.push_back({r, d.v(i, j), -ih});
        }
}

// transfers.cpp:107-134.
void restrict_saddle(int nf, const double* rf, double* rc) {
    Dof f{nf}, c{nf / 2};
    const int nc = nf / 2;
    for (int J = 0; J < nc; ++J)
        for (int I = 1; I <= nc - 1; ++I) {
            const int i = 2 * I, j = 2 * J;
            rc[c.u(I, J)] = 0.125 * (rf[f.u(i - 1, j)] + 2.0 * rf[f.u(i, j)] + rf[f.u(i + 1, j)] +
                                     rf[f.u(i - 1, j + 1)] + 2.0 * rf[f.u(i, j + 1)] + rf[f.u(i + 1, j + 1)]);
        }
    for (int J = 1; J <= nc - 1; ++J)
        for (int I = 0; I < nc; ++I) {
            const int i = 2 * I, j = 2 * J;
            rc[c.v(I, J)] = 0.125 * (rf[f.v(i, j - 1)] + 2.0 * rf[f.v(i, j)] + rf[f.v(i, j + 1)] +
                                     rf[f.v(i + 1, j - 1)] + 2.0 * rf[f.v(i + 1, j)] + rf[f.v(i + 1, j + 1)]);
        }
    for (int J = 0; J < nc; ++J)
        for (int I = 0; I < nc; ++I)
            rc[c.p(I, J)] = 0.25 * (rf[f.p(2 * I, 2 * J)] + rf[f.p(2 * I + 1, 2 * J)] + rf[f.p(2 * I, 2 * J + 1)] +
                                    rf[f.p(2 * I + 1, 2 * J + 1)]);
}

// Bilinear weights with homogeneous walls (transfers.cpp:141-205): the normal
// index takes weight 1 or 1/2, 1/2 and drops boundary faces, the tangential
// index 3/4, 1/4 and reflects through the wall with a negative weight.  The v
// weight is the correct xs.w * ys.w product (line 202 squares the x weight).
struct W2 {
    int I;
    double w;
};
inline int normal_w(int i, int nc, W2* o) {  // coarse normal faces 1 .. nc-1
    int k = 0;
    if (i % 2 == 0) {
        o[k++] = {i / 2, 1.0};
    } else {
        o[k++] = {(i - 1) / 2, 0.5};
        o[k++] = {(i + 1) / 2, 0.5};
    }
    int m = 0;
    for (int a = 0; a < k; ++a)
        if (o[a].I >= 1 && o[a].I <= nc - 1) o[m++] = o[a];
    return m;
}
inline void tangential_w(int j, int nc, W2* o) {
    const int J = j / 2;
    o[0] = {J, 0.75};
    o[1] = {(j % 2 == 0) ? J - 1 : J + 1, 0.25};
    if (o[1].I < 0) o[1] = {0, -0.25};
    else if (o[1].I > nc - 1) o[1] = {nc - 1, -0.25};
}

template <typename F>
void for_each_prolong_weight(int nf, F&& emit) {  // emit(fine vel dof, coarse vel dof, weight)
    Dof f{nf}, c{nf / 2};
    const int nc = nf / 2;
    W2 xs[2], ys[2];
    for (int j = 0; j < nf; ++j)
        for (int i = 1; i <= nf - 1; ++i) {
            const int nx = normal_w(i, nc, xs);
            tangential_w(j, nc, ys);
            for (int a = 0; a < nx; ++a)
                for (int b = 0; b < 2; ++b) emit(f.u(i, j), c.u(xs[a].I, ys[b].I), xs[a].w * ys[b].w);
        }
    for (int j = 1; j <= nf - 1; ++j)
        for (int i = 0; i < nf; ++i) {
            const int ny = normal_w(j, nc, ys);
            tangential_w(i, nc, xs);
            for (int b = 0; b < ny; ++b)
                for (int a = 0; a < 2; ++a) emit(f.v(i, j), c.v(xs[a].I, ys[b].I), xs[a].w * ys[b].w);
        }
}

// transfers.cpp:209-232.
void prolong_add(int nf, const double* ec, double* wf) {
    Dof f{nf}, c{nf / 2};
    for_each_prolong_weight(nf, [&](int r, int col, double w) { wf[r] += w * ec[col]; });
    for (int j = 0; j < nf; ++j)
        for (int i = 0; i < nf; ++i) wf[f.p(i, j)] += ec[c.p(i / 2, j / 2)];
}

// transfers.cpp:234-284.
Csr velocity_restriction_matrix(int nf) {
    Dof f{nf}, c{nf / 2};
    const int nc = nf / 2;
    std::vector<Trip> t;
    for (int J = 0; J < nc; ++J)
        for (int I = 1; I <= nc - 1; ++I) {
            const int i = 2 * I, j = 2 * J, r = c.u(I, J);
            t.push_back({r, f.u(i - 1, j), 0.125});
            t.push_back({r, f.u(i, j), 0.25});
            t.push_back({r, f.u(i + 1, j), 0.125});
            t.push_back({r, f.u(i - 1, j + 1), 0.125});
            t.push_back({r, f.u(i, j + 1), 0.25});
            t.push_back({r, f.u(i + 1, j + 1), 0.125});
        }
    for (int J = 1; J <= nc - 1; ++J)
        for (int I = 0; I < nc; ++I) {
            const int i = 2 * I, j = 2 * J, r = c.v(I, J);
            t.push_back({r, f.v(i, j - 1), 0.125});
            t.push_back({r, f.v(i, j), 0.25});
            t.push_back({r, f.v(i, j + 1), 0.125});
            t.push_back({r, f.v(i + 1, j - 1), 0.125});
            t.push_back({r, f.v(i + 1, j), 0.25});
            t.push_back({r, f.v(i + 1, j + 1), 0.125});
        }
    return Csr::from_trips(c.nvel(), f.nvel(), t, false);
}
Csr velocity_prolongation_matrix(int nf) {
    Dof f{nf}, c{nf / 2};
    std::vector<Trip> t;
    for_each_prolong_weight(nf, [&](int r, int col, double w) { t.push_back({r, col, w}); });
    return Csr::from_trips(f.nvel(), c.nvel(), t, false);
}

struct Box {
    std::vector<int> dofs;  // u faces (j major), v faces, cells
    DenseLu lu;             // principal submatrix, bordered by the pressure mean when the box is the level
};

struct Level {
    Dof d;
    double h = 0;
    Csr S, E, A;  // Stokes rows, elasticity (velocity block, alpha-free), S + alpha E
    int b = 1, nb = 1, reach = 1;
    bool whole = false;
    std::vector<Box> boxes;
    std::vector<int> order;  // box visiting order of a sweep
    std::vector<double> w, rhs, r;
};

struct Ctx {
    porc_params P{};
    int m1 = 0, m2 = 0;
    double ds = 0;
    std::vector<double> X;
    std::vector<Level> lev;
    std::string err;
};

// elasticity.cpp:62-107: scale * W^T T W with the per-fiber second difference.
Csr assemble_elasticity(const Ctx& C, const Dof& d, double h) {
    const int m1 = C.m1, m2 = C.m2;
    std::vector<SpVec> wu(size_t(m1) * m2), wv(size_t(m1) * m2);
    for (int q = 0; q < m1 * m2; ++q) node_weights(C.X[2 * q], C.X[2 * q + 1], d, h, wu[q], wv[q]);
    const double scale = C.ds * C.ds * h * h, ids2 = 1.0 / (C.ds * C.ds);
    std::vector<Trip> t;
    for (const std::vector<SpVec>* w : {&wu, &wv})
        for (int l = 0; l < m2; ++l)
            for (int k = 0; k < m1; ++k) {
                const int km = (k == 0) ? m1 - 1 : k - 1, kp = (k == m1 - 1) ? 0 : k + 1;
                const SpVec& row = (*w)[k + size_t(l) * m1];
                const SpVec* cols[3] = {&(*w)[km + size_t(l) * m1], &row, &(*w)[kp + size_t(l) * m1]};
                const double coef[3] = {ids2, -2.0 * ids2, ids2};
                for (const auto& [ri, rw] : row)
                    for (int c = 0; c < 3; ++c)
                        for (const auto& [ci, cw] : *cols[c]) t.push_back({ri, ci, scale * rw * coef[c] * cw});
            }
    return Csr::from_trips(d.nvel(), d.nvel(), t, false);
}

// fiber.cpp:18-32.
void require_supports_interior(const Ctx& C) {
    const double rad = 2.0 / C.P.N;
    for (int q = 0; q < C.m1 * C.m2; ++q) {
        const double x = C.X[2 * q], y = C.X[2 * q + 1];
        if (x - rad < 0.0 || x + rad > 1.0 || y - rad < 0.0 || y + rad > 1.0)
            throw std::invalid_argument("fiber node " + std::to_string(q) + " has kernel support crossing the domain boundary");
    }
}

// SPEC.md:409-417 (build_partition): all faces of the member cells, Dirichlet faces excluded.
void box_dofs(const Dof& d, int b, int bx, int by, std::vector<int>& out) {
    out.clear();
    const int i0 = bx * b, j0 = by * b, n = d.n;
    for (int j = j0; j < j0 + b; ++j)
        for (int i = i0; i <= i0 + b; ++i)
            if (i >= 1 && i <= n - 1) out.push_back(d.u(i, j));
    for (int j = j0; j <= j0 + b; ++j)
        for (int i = i0; i < i0 + b; ++i)
            if (j >= 1 && j <= n - 1) out.push_back(d.v(i, j));
    for (int j = j0; j < j0 + b; ++j)
        for (int i = i0; i < i0 + b; ++i) out.push_back(d.p(i, j));
}

void build(Ctx& C) {
    const int N = C.P.N;
    if (N < 2 * C.P.coarsest_n || (N & (N - 1)) || C.P.coarsest_n < 2 || (C.P.coarsest_n & (C.P.coarsest_n - 1)))
        throw std::invalid_argument("N and coarsest_n must be powers of two with N >= 2 coarsest_n");
    if (C.P.box < 1 || (C.P.box & (C.P.box - 1))) throw std::invalid_argument("box must be a power of two");
    if (C.P.alpha < 0) throw std::invalid_argument("alpha must be >= 0");
    if (C.P.order != 0 && C.P.order != 1) throw std::invalid_argument("order must be 0 (lexicographic) or 1 (multicolour)");
    C.lev.clear();
    for (int n = N; n >= C.P.coarsest_n; n /= 2) {
        Level L;
        L.d = Dof{n};
        L.h = 1.0 / n;
        C.lev.push_back(std::move(L));
    }
    const bool has_e = C.m1 > 0;
    if (has_e) require_supports_interior(C);
    for (size_t l = 0; l < C.lev.size(); ++l) {
        Level& L = C.lev[l];
        std::vector<Trip> t;
        stokes_trips(L.d, L.h, t);
        L.S = Csr::from_trips(L.d.ntot(), L.d.ntot(), t, false);
        if (has_e) {
            if (l == 0) {
                L.E = assemble_elasticity(C, L.d, L.h);
            } else {  // transfers.cpp:286-293
                const int nf = C.lev[l - 1].d.n;
                L.E = orc::spgemm(orc::spgemm(velocity_restriction_matrix(nf), C.lev[l - 1].E),
                                  velocity_prolongation_matrix(nf));
            }
        }
        // assembly.cpp:52-60: alpha * E into the velocity block
        std::vector<Trip> ta;
        for (int r = 0; r < L.S.nr; ++r)
            for (long k = L.S.rp[r]; k < L.S.rp[r + 1]; ++k) ta.push_back({r, L.S.ci[k], L.S.v[k]});
        if (has_e && C.P.alpha > 0)
            for (int r = 0; r < L.E.nr; ++r)
                for (long k = L.E.rp[r]; k < L.E.rp[r + 1]; ++k) ta.push_back({r, L.E.ci[k], C.P.alpha * L.E.v[k]});
        L.A = Csr::from_trips(L.d.ntot(), L.d.ntot(), ta, false);
        const int n = L.d.n;
        L.b = std::min(C.P.box, n);
        if (int(l) + 1 == int(C.lev.size())) L.b = n;  // coarsest level: direct solve
        L.nb = n / L.b;
        L.whole = (L.nb == 1);
        L.boxes.resize(size_t(L.nb) * L.nb);
        L.w.assign(L.d.ntot(), 0.0);
        L.rhs.assign(L.d.ntot(), 0.0);
        L.r.assign(L.d.ntot(), 0.0);
        // coupling reach in boxes: the largest Chebyshev distance between a box owning a row's DOF and
        // a box owning one of its columns (a velocity lies on the faces of up to two cells)
        {
            auto span = [&](int dof, int* lo, int* hi) {  // box index ranges (x, y) of the cells touching dof
                const int nu = L.d.nu(), nvel = L.d.nvel(), nn = L.d.n;
                if (dof < nu) {
                    const int i = dof % (nn - 1) + 1, j = dof / (nn - 1);
                    lo[0] = (i - 1) / L.b, hi[0] = i / L.b, lo[1] = hi[1] = j / L.b;
                } else if (dof < nvel) {
                    const int i = (dof - nu) % nn, j = (dof - nu) / nn + 1;
                    lo[0] = hi[0] = i / L.b, lo[1] = (j - 1) / L.b, hi[1] = j / L.b;
                } else {
                    lo[0] = hi[0] = ((dof - nvel) % nn) / L.b, lo[1] = hi[1] = ((dof - nvel) / nn) / L.b;
                }
            };
            int reach = 0;
            for (int r = 0; r < L.A.nr; ++r)
                for (long k = L.A.rp[r]; k < L.A.rp[r + 1]; ++k) {
                    if (L.A.v[k] == 0.0) continue;
                    int rl[2], rh[2], cl[2], ch[2];
                    span(r, rl, rh);
                    span(L.A.ci[k], cl, ch);
                    for (int x = 0; x < 2; ++x)
                        reach = std::max(reach, std::max(std::abs(rl[x] - ch[x]), std::abs(rh[x] - cl[x])));
                }
            L.reach = std::max(reach, 1);
        }
        L.order.clear();
        if (C.P.order == 1 && !L.whole) {
            const int per = L.reach + 1;
            for (int cy = 0; cy < per; ++cy)
                for (int cx = 0; cx < per; ++cx)
                    for (int by = cy; by < L.nb; by += per)
                        for (int bx = cx; bx < L.nb; bx += per) L.order.push_back(bx + by * L.nb);
        } else {
            for (int q = 0; q < L.nb * L.nb; ++q) L.order.push_back(q);
        }
        for (int by = 0; by < L.nb; ++by)
            for (int bx = 0; bx < L.nb; ++bx) {
                Box& B = L.boxes[bx + size_t(by) * L.nb];
                box_dofs(L.d, L.b, bx, by, B.dofs);
                const int m = int(B.dofs.size()), mm = m + (L.whole ? 1 : 0);
                B.lu.m = mm;
                B.lu.a.assign(size_t(mm) * mm, 0.0);
                for (int a = 0; a < m; ++a)
                    for (int c = 0; c < m; ++c) B.lu.a[size_t(a) * mm + c] = L.A.at(B.dofs[a], B.dofs[c]);
                if (L.whole)  // mean-zero pressure border
                    for (int a = 0; a < m; ++a)
                        if (B.dofs[a] >= L.d.nvel()) B.lu.a[size_t(a) * mm + m] = B.lu.a[size_t(m) * mm + a] = 1.0;
                if (!B.lu.factor()) throw std::runtime_error("singular box matrix");
            }
    }
}

void residual_level(const Level& L, const double* b, const double* w, double* r) {  // saddle.cpp:48-54
    for (int i = 0; i < L.A.nr; ++i) r[i] = b[i] - L.A.row_dot(i, w);
}

// boxes in lexicographic order (x fastest), residual rows of
// the box, exact local solve, immediate correction.
void sweep(const Level& L, const double* b, double* w) {
    std::vector<double> x;
    for (int q : L.order) {
        const Box& B = L.boxes[q];
        const int m = int(B.dofs.size());
        x.assign(B.lu.m, 0.0);
        for (int a = 0; a < m; ++a) x[a] = b[B.dofs[a]] - L.A.row_dot(B.dofs[a], w);
        B.lu.solve(x.data());
        for (int a = 0; a < m; ++a) w[B.dofs[a]] += x[a];
    }
}

void project_pressure_mean(const Dof& d, double* x) {  // fields.cpp:78-85
    double s = 0.0;
    for (int k = 0; k < d.np(); ++k) s += x[d.nvel() + k];
    s /= d.np();
    for (int k = 0; k < d.np(); ++k) x[d.nvel() + k] -= s;
}

// Algorithm 1 on level l: L.w is the
// iterate (in/out), L.rhs the right-hand side.
void vcycle_rec(Ctx& C, int l) {
    Level& L = C.lev[l];
    if (L.whole) {  // one box = exact solve
        sweep(L, L.rhs.data(), L.w.data());
        return;
    }
    for (int s = 0; s < C.P.nu1; ++s) sweep(L, L.rhs.data(), L.w.data());
    residual_level(L, L.rhs.data(), L.w.data(), L.r.data());
    Level& K = C.lev[l + 1];
    restrict_saddle(L.d.n, L.r.data(), K.rhs.data());
    std::fill(K.w.begin(), K.w.end(), 0.0);
    vcycle_rec(C, l + 1);
    prolong_add(L.d.n, K.w.data(), L.w.data());
    for (int s = 0; s < C.P.nu2; ++s) sweep(L, L.rhs.data(), L.w.data());
}

void vcycle(Ctx& C, const double* b, double* z) {  // zero initial guess
    Level& L = C.lev[0];
    std::copy(b, b + L.d.ntot(), L.rhs.begin());
    std::fill(L.w.begin(), L.w.end(), 0.0);
    vcycle_rec(C, 0);
    project_pressure_mean(L.d, L.w.data());
    std::copy(L.w.begin(), L.w.end(), z);
}

double dotv(const double* a, const double* b, int n) {  // fields.cpp:87-92
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

// mg_solve: w <- w + V(b - A w) from w = 0; a cycle is
// linear in (w, b), so the correction form is Algorithm 1 with initial guess w.
void mg_solve(Ctx& C, const double* b, double* x, double rtol, int max_iter, porc_stats* st, double* hist, int hl) {
    const Level& L = C.lev[0];
    const int n = L.d.ntot();
    std::vector<double> r(b, b + n), z(n);
    std::fill(x, x + n, 0.0);
    const double bn = std::sqrt(dotv(b, b, n));
    *st = porc_stats{0, 0, 0, 0.0};
    if (hist && hl > 0) hist[0] = 1.0;
    if (bn == 0.0) {
        st->converged = 1;
        return;
    }
    double prev = bn;
    int grow = 0;
    for (int it = 1; it <= max_iter; ++it) {
        vcycle(C, r.data(), z.data());
        for (int i = 0; i < n; ++i) x[i] += z[i];
        residual_level(L, b, x, r.data());
        const double rn = std::sqrt(dotv(r.data(), r.data(), n));
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
    project_pressure_mean(L.d, x);
}

// gmres_solve: right-preconditioned, unrestarted, x0 = 0,
// classical Gram-Schmidt with one reorthogonalisation pass (SPEC.md:510 allows
// MGS or CGS2), Givens residual estimate confirmed on the true residual
// (SPEC.md:511); z_j = M v_j kept so that x = sum y_j z_j.
void gmres_solve(Ctx& C, const double* b, double* x, double rtol, int max_iter, porc_stats* st, double* hist,
                 int hl) {
    const Level& L = C.lev[0];
    const int n = L.d.ntot(), m = max_iter;
    *st = porc_stats{0, 0, 0, 0.0};
    std::fill(x, x + n, 0.0);
    const double bn = std::sqrt(dotv(b, b, n));
    if (hist && hl > 0) hist[0] = 1.0;
    if (bn == 0.0) {
        st->converged = 1;
        return;
    }
    std::vector<std::vector<double>> V(1, std::vector<double>(b, b + n)), Z;
    for (double& v : V[0]) v /= bn;
    std::vector<double> H(size_t(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0), w(n), y(m), r(n), h1(m + 1), h2(m + 1);
    g[0] = bn;
    auto form_x = [&](int k) {
        for (int i = k - 1; i >= 0; --i) {
            double s = g[i];
            for (int j = i + 1; j < k; ++j) s -= H[size_t(i) * m + j] * y[j];
            y[i] = s / H[size_t(i) * m + i];
        }
        std::fill(x, x + n, 0.0);
        for (int j = 0; j < k; ++j)
            for (int i = 0; i < n; ++i) x[i] += y[j] * Z[j][i];
    };
    for (int j = 0; j < m; ++j) {
        Z.emplace_back(n);
        vcycle(C, V[j].data(), Z[j].data());
        for (int i = 0; i < n; ++i) w[i] = L.A.row_dot(i, Z[j].data());
        for (int i = 0; i <= j; ++i) h1[i] = dotv(V[i].data(), w.data(), n);
        for (int i = 0; i <= j; ++i)
            for (int q = 0; q < n; ++q) w[q] -= h1[i] * V[i][q];
        for (int i = 0; i <= j; ++i) h2[i] = dotv(V[i].data(), w.data(), n);
        for (int i = 0; i <= j; ++i)
            for (int q = 0; q < n; ++q) w[q] -= h2[i] * V[i][q];
        const double hn = std::sqrt(dotv(w.data(), w.data(), n));
        for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = h1[i] + h2[i];
        for (int i = 0; i < j; ++i) {  // earlier rotations on the new column
            const double a = H[size_t(i) * m + j], c = H[size_t(i + 1) * m + j];
            H[size_t(i) * m + j] = cs[i] * a + sn[i] * c;
            H[size_t(i + 1) * m + j] = -sn[i] * a + cs[i] * c;
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
            residual_level(L, b, x, r.data());
            st->relres = std::sqrt(dotv(r.data(), r.data(), n)) / bn;
            if (st->relres <= rtol) st->converged = 1;
            if (st->converged || last) break;
        }
        V.emplace_back(w);
        for (double& v : V[j + 1]) v /= hn;
    }
    project_pressure_mean(L.d, x);
}

// fiber.cpp:34-55, 89-114, 116-140 on the packed interior velocity ordering
// (supports are interior, so boundary faces carry zero weight).
void fiber_second_difference(const Ctx& C, const double* f, double* out) {
    const double ids2 = 1.0 / (C.ds * C.ds);
    for (int l = 0; l < C.m2; ++l)
        for (int k = 0; k < C.m1; ++k) {
            const int km = (k == 0) ? C.m1 - 1 : k - 1, kp = (k == C.m1 - 1) ? 0 : k + 1;
            const size_t q = k + size_t(l) * C.m1, a = km + size_t(l) * C.m1, c = kp + size_t(l) * C.m1;
            for (int x = 0; x < 2; ++x) out[2 * q + x] = (f[2 * a + x] + f[2 * c + x] - f[2 * q + x] * 2.0) * ids2;
        }
}
void spread(const Ctx& C, const double* F, double* f) {
    const Level& L = C.lev[0];
    std::fill(f, f + L.d.nvel(), 0.0);
    const double w0 = C.ds * C.ds;
    SpVec wu, wv;
    for (int q = 0; q < C.m1 * C.m2; ++q) {
        node_weights(C.X[2 * q], C.X[2 * q + 1], L.d, L.h, wu, wv);
        for (const auto& [i, w] : wu) f[i] += F[2 * q] * w * w0;
        for (const auto& [i, w] : wv) f[i] += F[2 * q + 1] * w * w0;
    }
}
void interp(const Ctx& C, const double* vel, double* U) {
    const Level& L = C.lev[0];
    const double w0 = L.h * L.h;
    SpVec wu, wv;
    for (int q = 0; q < C.m1 * C.m2; ++q) {
        node_weights(C.X[2 * q], C.X[2 * q + 1], L.d, L.h, wu, wv);
        double a = 0.0, b = 0.0;
        for (const auto& [i, w] : wu) a += vel[i] * w;
        for (const auto& [i, w] : wv) b += vel[i] * w;
        U[2 * q] = a * w0;
        U[2 * q + 1] = b * w0;
    }
}

// saddle.cpp:56-104 with the lid data of PAPER.md:612-613 (only the top wall's
// tangential velocity is nonzero, so only the u rows of the top cell row fold).
void rhs(const Ctx& C, int lid, double gamma, double* b) {
    const Level& L = C.lev[0];
    const int n = L.d.n;
    std::fill(b, b + L.d.ntot(), 0.0);
    if (lid)
        for (int i = 1; i <= n - 1; ++i) {
            const double ulid = (1.0 - std::cos(2.0 * orc::kPi * (i * L.h))) / 2.0;
            b[L.d.u(i, n - 1)] -= 2.0 * ulid / (L.h * L.h);
        }
    if (C.m1 > 0 && gamma != 0.0) {
        std::vector<double> F(C.X.size()), f(L.d.nvel());
        fiber_second_difference(C, C.X.data(), F.data());
        for (double& v : F) v *= gamma;
        spread(C, F.data(), f.data());
        for (int k = 0; k < L.d.nvel(); ++k) b[k] -= f[k];
    }
}

}  // namespace porc

using porc::Ctx;

#define PORC_TRY(ctx, ...)                                    \
    try {                                                     \
        __VA_ARGS__;                                          \
        return 0;                                             \
    } catch (const std::exception& e) {                       \
        static_cast<Ctx*>(ctx)->err = e.what();               \
        return 1;                                             \
    }

extern "C" {

void* porc_create(const porc_params* p, char* err, int errlen) {
    Ctx* C = new Ctx;
    C->P = *p;
    try {
        porc::build(*C);
    } catch (const std::exception& e) {
        if (err && errlen > 0) std::snprintf(err, errlen, "%s", e.what());
        delete C;
        return nullptr;
    }
    return C;
}
void porc_destroy(void* ctx) { delete static_cast<Ctx*>(ctx); }
const char* porc_last_error(void* ctx) { return static_cast<Ctx*>(ctx)->err.c_str(); }

int porc_set_mesh(void* ctx, int m1, int m2, double ds, const double* X) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    PORC_TRY(ctx, {
        if (m1 != 0 && (m1 < 3 || m2 < 1 || !(ds > 0.0))) throw std::invalid_argument("FiberMesh: m1 >= 3, m2 >= 1, ds > 0");
        C.m1 = m1;
        C.m2 = m1 ? m2 : 0;
        C.ds = ds;
        C.X.assign(X, X + size_t(2) * C.m1 * C.m2);
        porc::build(C);
    });
}
int porc_num_levels(void* ctx) { return int(static_cast<Ctx*>(ctx)->lev.size()); }
int porc_level_n(void* ctx, int l) { return static_cast<Ctx*>(ctx)->lev.at(l).d.n; }
int porc_level_dofs(void* ctx, int l) { return static_cast<Ctx*>(ctx)->lev.at(l).d.ntot(); }
int porc_level_boxes(void* ctx, int l) { return static_cast<Ctx*>(ctx)->lev.at(l).nb; }
int porc_level_reach(void* ctx, int l) { return static_cast<Ctx*>(ctx)->lev.at(l).reach; }

int porc_apply(void* ctx, int l, const double* w, double* out) {
    PORC_TRY(ctx, {
        const porc::Level& L = static_cast<Ctx*>(ctx)->lev.at(l);
        for (int i = 0; i < L.A.nr; ++i) out[i] = L.A.row_dot(i, w);
    });
}
int porc_residual(void* ctx, int l, const double* b, const double* w, double* r) {
    PORC_TRY(ctx, porc::residual_level(static_cast<Ctx*>(ctx)->lev.at(l), b, w, r));
}
int porc_sweep(void* ctx, int l, const double* b, double* w) {
    PORC_TRY(ctx, porc::sweep(static_cast<Ctx*>(ctx)->lev.at(l), b, w));
}
int porc_vcycle(void* ctx, const double* b, double* z) { PORC_TRY(ctx, porc::vcycle(*static_cast<Ctx*>(ctx), b, z)); }
int porc_restrict(int nf, const double* rf, double* rc) {
    porc::restrict_saddle(nf, rf, rc);
    return 0;
}
int porc_prolong_add(int nf, const double* ec, double* wf) {
    porc::prolong_add(nf, ec, wf);
    return 0;
}
static long dump(const orc::Csr& M, int* rows, int* cols, double* vals, long cap) {
    long q = 0;
    for (int r = 0; r < M.nr; ++r)
        for (long k = M.rp[r]; k < M.rp[r + 1]; ++k, ++q)
            if (rows && q < cap) {
                rows[q] = r;
                cols[q] = M.ci[k];
                vals[q] = M.v[k];
            }
    return q;
}
long porc_elasticity_triplets(void* ctx, int l, int* rows, int* cols, double* vals, long cap) {
    return dump(static_cast<Ctx*>(ctx)->lev.at(l).E, rows, cols, vals, cap);
}
long porc_saddle_triplets(void* ctx, int l, int* rows, int* cols, double* vals, long cap) {
    return dump(static_cast<Ctx*>(ctx)->lev.at(l).A, rows, cols, vals, cap);
}
int porc_rhs(void* ctx, int lid, double gamma, double* b) { PORC_TRY(ctx, porc::rhs(*static_cast<Ctx*>(ctx), lid, gamma, b)); }
int porc_spread(void* ctx, const double* F, double* f) { PORC_TRY(ctx, porc::spread(*static_cast<Ctx*>(ctx), F, f)); }
int porc_interp(void* ctx, const double* vel, double* U) { PORC_TRY(ctx, porc::interp(*static_cast<Ctx*>(ctx), vel, U)); }

int porc_mg_solve(void* ctx, const double* b, double* x, double rtol, int max_iter, porc_stats* st, double* hist,
                  int hist_len) {
    PORC_TRY(ctx, porc::mg_solve(*static_cast<Ctx*>(ctx), b, x, rtol, max_iter, st, hist, hist_len));
}
int porc_gmres_solve(void* ctx, const double* b, double* x, double rtol, int max_iter, porc_stats* st, double* hist,
                     int hist_len) {
    PORC_TRY(ctx, porc::gmres_solve(*static_cast<Ctx*>(ctx), b, x, rtol, max_iter, st, hist, hist_len));
}

int porc_vcycle_spectrum(void* ctx, int m, unsigned long long seed, double* H, int* m_done) {
    Ctx& C = *static_cast<Ctx*>(ctx);
    PORC_TRY(ctx, {
        if (m < 2) throw std::invalid_argument("SpectrumProbe: m >= 2");
        const porc::Level& L = C.lev[0];
        const int n = L.d.ntot();
        std::vector<std::vector<double>> V(1, std::vector<double>(n));
        unsigned long long z = seed;
        for (double& v : V[0]) {  // splitmix64 -> U[-1, 1), as the GPU probe
            z += 0x9E3779B97F4A7C15ull;
            unsigned long long t = z;
            t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
            t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
            t ^= t >> 31;
            v = double(t >> 11) * (2.0 / 9007199254740992.0) - 1.0;
        }
        porc::project_pressure_mean(L.d, V[0].data());
        const double n0 = std::sqrt(porc::dotv(V[0].data(), V[0].data(), n));
        for (double& v : V[0]) v /= n0;
        std::fill(H, H + size_t(m + 1) * m, 0.0);
        std::vector<double> a(n), w(n), h1(m + 1), h2(m + 1);
        int done = 0;
        for (int j = 0; j < m; ++j) {
            for (int i = 0; i < n; ++i) a[i] = L.A.row_dot(i, V[j].data());
            porc::vcycle(C, a.data(), w.data());
            for (int i = 0; i < n; ++i) w[i] = V[j][i] - w[i];
            porc::project_pressure_mean(L.d, w.data());
            for (int i = 0; i <= j; ++i) h1[i] = porc::dotv(V[i].data(), w.data(), n);
            for (int i = 0; i <= j; ++i)
                for (int q = 0; q < n; ++q) w[q] -= h1[i] * V[i][q];
            for (int i = 0; i <= j; ++i) h2[i] = porc::dotv(V[i].data(), w.data(), n);
            for (int i = 0; i <= j; ++i)
                for (int q = 0; q < n; ++q) w[q] -= h2[i] * V[i][q];
            const double hn = std::sqrt(porc::dotv(w.data(), w.data(), n));
            for (int i = 0; i <= j; ++i) H[size_t(i) * m + j] = h1[i] + h2[i];
            H[size_t(j + 1) * m + j] = hn;
            done = j + 1;
            if (!(hn > 1e-300)) break;
            V.emplace_back(w);
            for (double& v : V[j + 1]) v /= hn;
        }
        if (m_done) *m_done = done;
    });
}

// power iteration on M X = S* L^-1 S A_f X,
// where u = L^-1 f solves Lap u - grad p = -f, div u = 0 with homogeneous walls.
int porc_alpha_exp(void* ctx, double tol, int max_steps, double* alpha_exp, int* steps) {
    Ctx& C0 = *static_cast<Ctx*>(ctx);
    PORC_TRY(ctx, {
        if (C0.m1 == 0) throw std::invalid_argument("alpha_exp needs a fiber mesh");
        Ctx S;  // the same hierarchy with alpha = 0
        S.P = C0.P;
        S.P.alpha = 0.0;
        S.m1 = C0.m1;
        S.m2 = C0.m2;
        S.ds = C0.ds;
        S.X = C0.X;
        porc::build(S);
        const porc::Level& L = S.lev[0];
        const size_t nx = S.X.size();
        std::vector<double> x(nx), y(nx), F(nx), b(L.d.ntot()), w(L.d.ntot());
        unsigned long long s = 12345;
        for (double& v : x) {
            s = s * 6364136223846793005ULL + 1442695040888963407ULL;
            v = double(s >> 11) / 9007199254740992.0 - 0.5;
        }
        double lam = 0.0, prev = 0.0;
        int it = 0;
        for (it = 1; it <= max_steps; ++it) {
            const double xn = std::sqrt(porc::dotv(x.data(), x.data(), int(nx)));
            for (double& v : x) v /= xn;
            porc::fiber_second_difference(S, x.data(), F.data());
            std::fill(b.begin(), b.end(), 0.0);
            std::vector<double> f(L.d.nvel());
            porc::spread(S, F.data(), f.data());
            for (int k = 0; k < L.d.nvel(); ++k) b[k] = -f[k];
            porc_stats st;
            porc::gmres_solve(S, b.data(), w.data(), 1e-10, 100, &st, nullptr, 0);
            porc::interp(S, w.data(), y.data());
            lam = porc::dotv(x.data(), y.data(), int(nx));  // Rayleigh quotient, |x| = 1
            if (it > 1 && std::fabs(lam - prev) <= tol * std::fabs(lam)) break;
            prev = lam;
            x = y;
        }
        if (it > max_steps) throw std::runtime_error("power iteration did not converge");
        *alpha_exp = 2.0 / std::fabs(lam);
        if (steps) *steps = it;
    });
}

}  // extern "C"
