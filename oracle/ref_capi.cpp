// ref_capi.cpp — C entry points over the REFERENCE's own operator sources
// (/root/reference/proj/core/src/*.cpp, compiled in place by Makefile.ref with
// the test-only Eigen shim) for pinning the oracle (TEST INFRASTRUCTURE ONLY).
// Geometry is the reference's Dirichlet unit square: nx = ny = n, h = 1/n,
// origin 0; vectors use the reference's packed interior ordering
// (geometry.hpp:54-72); one closed fiber (m2 = 1, periodic_s1).
#include <cmath>
#include <cstring>
#include <exception>
#include <vector>

#include "ibmg/assembly.hpp"
#include "ibmg/elasticity.hpp"
#include "ibmg/fiber.hpp"
#include "ibmg/saddle.hpp"
#include "ibmg/stokes_ops.hpp"
#include "ibmg/transfers.hpp"

using namespace ibmg;

namespace {
GridGeometry geom(int n) { return GridGeometry(n, n, 1.0 / n); }
FiberMesh mesh(int m1, double ds, const double* X) {
    FiberMesh M(m1, 1, ds, true);
    for (int k = 0; k < m1; ++k) M.X.at(k, 0) = Vec2{X[2 * k], X[2 * k + 1]};
    return M;
}
long dump(const SparseOperator& A, int* rows, int* cols, double* vals, long cap) {
    long q = 0;
    for (long r = 0; r < A.outerSize(); ++r)
        for (SparseOperator::InnerIterator it(A, r); it; ++it, ++q)
            if (rows && q < cap) {
                rows[q] = int(it.row());
                cols[q] = int(it.col());
                vals[q] = it.value();
            }
    return q;
}
}  // namespace

extern "C" {

int ref_sizes(int n, int* nu, int* nv, int* np) {
    DofMap dm(geom(n));
    *nu = dm.nu();
    *nv = dm.nv();
    *np = dm.np();
    return 0;
}

int ref_laplacian_hom(int n, const double* vel, double* out) {
    try {
        DofMap dm(geom(n));
        laplacian_hom(geom(n), std::span<const double>(vel, dm.n_vel()), std::span<double>(out, dm.n_vel()));
        return 0;
    } catch (const std::exception&) { return 1; }
}
int ref_gradient_hom(int n, const double* p, double* out) {
    try {
        DofMap dm(geom(n));
        gradient_hom(geom(n), std::span<const double>(p, dm.np()), std::span<double>(out, dm.n_vel()));
        return 0;
    } catch (const std::exception&) { return 1; }
}
int ref_divergence_hom(int n, const double* vel, double* out) {
    try {
        DofMap dm(geom(n));
        divergence_hom(geom(n), std::span<const double>(vel, dm.n_vel()), std::span<double>(out, dm.np()));
        return 0;
    } catch (const std::exception&) { return 1; }
}
double ref_delta_1d(double r, double h) { return delta_1d(r, h); }
double ref_adjointness_check(int n, int trials, unsigned long long seed) {
    return adjointness_check(geom(n), trials, seed);
}

int ref_fiber_force(int m1, double ds, double gamma, const double* X, double* F) {
    try {
        FiberMesh M = mesh(m1, ds, X);
        LagrangianField f = fiber_force(M, gamma);
        for (int k = 0; k < m1; ++k) {
            F[2 * k] = f.at(k, 0).x;
            F[2 * k + 1] = f.at(k, 0).y;
        }
        return 0;
    } catch (const std::exception&) { return 1; }
}

int ref_spread(int n, int m1, double ds, const double* X, const double* F, double* f_vel) {
    try {
        FiberMesh M = mesh(m1, ds, X);
        LagrangianField L(m1, 1);
        for (int k = 0; k < m1; ++k) L.at(k, 0) = Vec2{F[2 * k], F[2 * k + 1]};
        std::vector<double> p = pack_velocity(spread(M, L, geom(n)));
        std::memcpy(f_vel, p.data(), p.size() * sizeof(double));
        return 0;
    } catch (const std::exception&) { return 1; }
}

int ref_interpolate(int n, int m1, double ds, const double* X, const double* vel, double* U) {
    try {
        FiberMesh M = mesh(m1, ds, X);
        DofMap dm(geom(n));
        VelocityField v = unpack_velocity(geom(n), std::span<const double>(vel, dm.n_vel()));
        LagrangianField L = interpolate(M, v);
        for (int k = 0; k < m1; ++k) {
            U[2 * k] = L.at(k, 0).x;
            U[2 * k + 1] = L.at(k, 0).y;
        }
        return 0;
    } catch (const std::exception&) { return 1; }
}

long ref_assemble_elasticity(int n, int m1, double ds, const double* X, double gamma, int* rows, int* cols,
                             double* vals, long cap) {
    try {
        return dump(assemble_elasticity(mesh(m1, ds, X), geom(n), gamma).matrix, rows, cols, vals, cap);
    } catch (const std::exception&) { return -1; }
}

long ref_galerkin_elasticity(int n, int m1, double ds, const double* X, double gamma, int levels, int* rows,
                             int* cols, double* vals, long cap) {
    try {
        GridGeometry g = geom(n);
        SparseOperator E = assemble_elasticity(mesh(m1, ds, X), g, gamma).matrix;
        for (int l = 0; l < levels; ++l) {
            E = galerkin_coarsen_elasticity(E, g);
            g = g.coarsened();
        }
        return dump(E, rows, cols, vals, cap);
    } catch (const std::exception&) { return -1; }
}

// R * E * P with P assembled column by column from the reference's correct
// field-level prolong_velocity (transfers.cpp:67-105) instead of the packed
// velocity_prolongation_matrix, whose v weight is wrong (transfers.cpp:202).
long ref_galerkin_elasticity_fixed_p(int n, int m1, double ds, const double* X, double gamma, int* rows, int* cols,
                                     double* vals, long cap) {
    try {
        GridGeometry g = geom(n), gc = g.coarsened();
        DofMap df(g), dc(gc);
        SparseOperator E = assemble_elasticity(mesh(m1, ds, X), g, gamma).matrix;
        std::vector<Triplet> t;
        std::vector<double> e(dc.n_vel(), 0.0);
        for (int col = 0; col < dc.n_vel(); ++col) {
            e[col] = 1.0;
            std::vector<double> f = pack_velocity(prolong_velocity(unpack_velocity(gc, e), g));
            e[col] = 0.0;
            for (int r = 0; r < df.n_vel(); ++r)
                if (f[r] != 0.0) t.emplace_back(r, col, f[r]);
        }
        SparseOperator P(df.n_vel(), dc.n_vel());
        P.setFromTriplets(t.begin(), t.end());
        SparseOperator C = (velocity_restriction_matrix(g) * E * P).pruned();
        return dump(C, rows, cols, vals, cap);
    } catch (const std::exception&) { return -1; }
}

// Field-level bilinear prolongation (transfers.cpp:67-105, correct weights).
int ref_prolong_velocity(int n, const double* ec_vel, double* wf_vel) {
    try {
        GridGeometry g = geom(n), gc = g.coarsened();
        DofMap dc(gc);
        std::vector<double> f =
            pack_velocity(prolong_velocity(unpack_velocity(gc, std::span<const double>(ec_vel, dc.n_vel())), g));
        std::memcpy(wf_vel, f.data(), f.size() * sizeof(double));
        return 0;
    } catch (const std::exception&) { return 1; }
}

int ref_elasticity_apply_matrix_free(int n, int m1, double ds, const double* X, const double* vel, double* out) {
    try {
        DofMap dm(geom(n));
        elasticity_apply_matrix_free(mesh(m1, ds, X), geom(n), std::span<const double>(vel, dm.n_vel()),
                                     std::span<double>(out, dm.n_vel()));
        return 0;
    } catch (const std::exception&) { return 1; }
}

int ref_restrict_saddle(int n, const double* rf, double* rc) {
    try {
        DofMap df(geom(n)), dc(geom(n).coarsened());
        restrict_saddle(geom(n), std::span<const double>(rf, df.n_total()), std::span<double>(rc, dc.n_total()));
        return 0;
    } catch (const std::exception&) { return 1; }
}
int ref_prolong_saddle_add(int n, const double* ec, double* wf) {
    try {
        DofMap df(geom(n)), dc(geom(n).coarsened());
        prolong_saddle_add(geom(n), std::span<const double>(ec, dc.n_total()), std::span<double>(wf, df.n_total()));
        return 0;
    } catch (const std::exception&) { return 1; }
}

// SaddleSystem::apply (saddle.cpp:19-38) with alpha*E (E from assemble_elasticity).
int ref_saddle_apply(int n, int m1, double ds, const double* X, double gamma, double alpha, const double* w,
                     double* out) {
    try {
        GridGeometry g = geom(n);
        ElasticityOperator E = (alpha > 0) ? assemble_elasticity(mesh(m1, ds, X), g, gamma) : ElasticityOperator{};
        SaddleSystem S(g, VelocityBC::zero(), alpha, std::move(E));
        DofMap dm(g);
        S.apply(std::span<const double>(w, dm.n_total()), std::span<double>(out, dm.n_total()));
        return 0;
    } catch (const std::exception&) { return 1; }
}

// ---- Dirichlet paper-mode pins (thick m1 x m2 mesh, walls included) -------
namespace {
FiberMesh mesh2(int m1, int m2, double ds, const double* X) {
    FiberMesh M(m1, m2, ds, true);
    for (int l = 0; l < m2; ++l)
        for (int k = 0; k < m1; ++k) M.X.at(k, l) = Vec2{X[2 * (k + size_t(l) * m1)], X[2 * (k + size_t(l) * m1) + 1]};
    return M;
}
VelocityBC lid_bc() {
    return VelocityBC{[](double x, double y) { return y >= 1.0 ? (1.0 - std::cos(2.0 * 3.14159265358979323846 * x)) / 2.0 : 0.0; },
                      [](double, double) { return 0.0; }};
}
}  // namespace

// assemble_saddle_matrix (assembly.cpp:5-65) of SaddleSystem(g, bc, alpha, assemble_elasticity(mesh, g, 1)).
long ref_assemble_saddle_m2(int n, int m1, int m2, double ds, const double* X, double alpha, int* rows, int* cols,
                            double* vals, long cap) {
    try {
        GridGeometry g = geom(n);
        ElasticityOperator E = (alpha > 0) ? assemble_elasticity(mesh2(m1, m2, ds, X), g, 1.0) : ElasticityOperator{};
        SaddleSystem S(g, VelocityBC::zero(), alpha, std::move(E));
        return dump(assemble_saddle_matrix(S), rows, cols, vals, cap);
    } catch (const std::exception&) { return -1; }
}

// Galerkin-coarsened elasticity (transfers.cpp:286-293) `levels` times.  The v block
// goes through the packed prolongation's wrong weight (transfers.cpp:202); the u block is exact.
long ref_galerkin_elasticity_m2(int n, int m1, int m2, double ds, const double* X, int levels, int* rows, int* cols,
                                double* vals, long cap) {
    try {
        GridGeometry g = geom(n);
        SparseOperator E = assemble_elasticity(mesh2(m1, m2, ds, X), g, 1.0).matrix;
        for (int l = 0; l < levels; ++l) {
            E = galerkin_coarsen_elasticity(E, g);
            g = g.coarsened();
        }
        return dump(E, rows, cols, vals, cap);
    } catch (const std::exception&) { return -1; }
}

// build_rhs (saddle.cpp:96-104) with the lid-driven cavity data.
int ref_build_rhs_lid(int n, int m1, int m2, double ds, const double* X, double gamma, double* out) {
    try {
        GridGeometry g = geom(n);
        SaddleSystem S(g, lid_bc(), 0.0, ElasticityOperator{});
        FiberMesh M = mesh2(m1, m2, ds, X);
        std::vector<double> b = build_rhs(S, &M, gamma);
        std::memcpy(out, b.data(), b.size() * sizeof(double));
        return 0;
    } catch (const std::exception&) { return 1; }
}

// spread / interpolate on the thick mesh (fiber.cpp:89-140), packed velocities.
int ref_spread_m2(int n, int m1, int m2, double ds, const double* X, const double* F, double* f_vel) {
    try {
        FiberMesh M = mesh2(m1, m2, ds, X);
        LagrangianField L(m1, m2);
        for (size_t q = 0; q < size_t(m1) * m2; ++q) L.val[q] = Vec2{F[2 * q], F[2 * q + 1]};
        std::vector<double> f = pack_velocity(spread(M, L, geom(n)));
        std::memcpy(f_vel, f.data(), f.size() * sizeof(double));
        return 0;
    } catch (const std::exception&) { return 1; }
}
int ref_interpolate_m2(int n, int m1, int m2, double ds, const double* X, const double* vel, double* U) {
    try {
        DofMap dm(geom(n));
        FiberMesh M = mesh2(m1, m2, ds, X);
        LagrangianField L = interpolate(M, unpack_velocity(geom(n), std::span<const double>(vel, dm.n_vel())));
        for (size_t q = 0; q < size_t(m1) * m2; ++q) {
            U[2 * q] = L.val[q].x;
            U[2 * q + 1] = L.val[q].y;
        }
        return 0;
    } catch (const std::exception&) { return 1; }
}

}  // extern "C"

// Mesh text IO through the reference's own writer/reader (fiber.cpp:142-166).
#include <sstream>
#include <string>
extern "C" {
long ref_write_fiber_mesh(int m1, double ds, const double* X, char* buf, long cap) {
    try {
        std::ostringstream os;
        write_fiber_mesh(os, mesh(m1, ds, X));
        const std::string s = os.str();
        if (buf && cap > long(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
        return long(s.size());
    } catch (const std::exception&) {
        return -1;
    }
}
int ref_read_fiber_mesh(const char* text, int* m1, double* ds, double* X, int cap) {
    try {
        std::istringstream is(text);
        const FiberMesh M = read_fiber_mesh(is);
        *m1 = M.m1;
        *ds = M.ds;
        for (int k = 0; k < M.m1 && k < cap; ++k) {
            X[2 * k] = M.X.at(k, 0).x;
            X[2 * k + 1] = M.X.at(k, 0).y;
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}
}
