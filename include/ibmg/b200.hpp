// ibmg/b200.hpp — C++ facade over the C ABI (include/ibmg_gpu.h), mirroring the
// reference's ibmg:: solver interface (proj/core/include/ibmg/*.hpp) so that a
// reference user switches by changing includes and the SaddleSystem
// constructor.  Same names, span conventions and error behaviour:
//   * SaddleSystem::apply(span w, span out)      saddle.hpp:32, saddle.cpp:19-38
//   * SaddleSystem::residual(span w, double* n)  saddle.hpp:38, saddle.cpp:48-54
//   * restrict_saddle / prolong_saddle_add        transfers.hpp:25-28
//   * spread / interpolate                        fiber.hpp:80-83 (flat arrays)
//   * build_rhs                                   saddle.hpp:46
//   * v_cycle / gmres_solve / step_implicit
// Status 1 -> std::invalid_argument (the reference's validation errors),
// 3/4 -> std::runtime_error; non-convergence is a flag in SolveStats
// (SPEC.md:478), not an exception.
//
// Periodic geometry, rho/dt, mu and per-membrane kappa are the SURVEY §9
// extensions (D1-D3); the packed vectors are [u | v | p] on the periodic grid.
#pragma once

#include <istream>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ibmg_gpu.h"

namespace ibmg::b200 {

struct Membrane {
    int nb = 0;           // points (closed curve, periodic in s1)
    double kappa = 0.0;   // stiffness
    double ds = 0.0;      // Lagrangian spacing (ds^2 quadrature)
};

struct SolveStats {
    int iterations = 0;
    int restarts = 0;
    bool converged = false;
    double relres = 0.0;
    double setup_ms = 0.0, solve_ms = 0.0, total_ms = 0.0;
};

inline void check(int rc, const ibmg_ctx* ctx) {
    if (rc == IBMG_OK || rc == IBMG_NOT_CONVERGED) return;
    const std::string msg = ibmg_last_error(ctx);
    if (rc == IBMG_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

class SaddleSystem {
   public:
    struct Params {
        int N = 64;
        double rho = 1.0, mu = 1.0, dt = 1e-2;
        int nu1 = 1, nu2 = 1, restart = 30, max_iters = 600;
        double rtol = 1e-10;
        int device = 0;
    };

    explicit SaddleSystem(const Params& p) : N_(p.N) {
        ibmg_params q{p.N, p.rho, p.mu, p.dt, p.nu1, p.nu2, p.restart, p.max_iters, p.rtol, 4, p.device};
        const int rc = ibmg_create(&q, &ctx_);
        if (rc == IBMG_INVALID) throw std::invalid_argument("SaddleSystem: invalid parameters");
        if (rc != IBMG_OK) throw std::runtime_error("SaddleSystem: CUDA initialisation failed");
    }
    ~SaddleSystem() { ibmg_destroy(ctx_); }
    SaddleSystem(const SaddleSystem&) = delete;
    SaddleSystem& operator=(const SaddleSystem&) = delete;

    int N() const { return N_; }
    int n_total() const { return 3 * N_ * N_; }
    int n_vel() const { return 2 * N_ * N_; }
    int num_levels() const { return ibmg_num_levels(ctx_); }

    // FiberMesh + assemble_elasticity + Galerkin hierarchy (X: 2*sum(nb), (x, y) interleaved)
    void set_structures(std::span<const Membrane> mem, std::span<const double> X) {
        std::vector<int> nb;
        std::vector<double> k, ds;
        size_t tot = 0;
        for (const Membrane& m : mem) {
            nb.push_back(m.nb);
            k.push_back(m.kappa);
            ds.push_back(m.ds);
            tot += size_t(m.nb);
        }
        if (X.size() != 2 * tot) throw std::invalid_argument("set_structures: X size mismatch");
        check(ibmg_set_structures(ctx_, int(mem.size()), nb.data(), k.data(), ds.data(), X.data(), IBMG_PTR_HOST),
              ctx_);
        npts_ = tot;
    }

    void apply(std::span<const double> w, std::span<double> out) const {
        if (int(w.size()) != n_total() || int(out.size()) != n_total())
            throw std::invalid_argument("SaddleSystem::apply: size mismatch");
        check(ibmg_apply(ctx_, 0, w.data(), out.data(), IBMG_PTR_HOST), ctx_);
    }

    std::vector<double> residual(std::span<const double> b, std::span<const double> w, double* norm = nullptr) const {
        if (int(w.size()) != n_total() || int(b.size()) != n_total())
            throw std::invalid_argument("SaddleSystem::residual: size mismatch");
        std::vector<double> r(static_cast<size_t>(n_total()));
        check(ibmg_residual(ctx_, 0, b.data(), w.data(), r.data(), norm, IBMG_PTR_HOST), ctx_);
        return r;
    }

    std::vector<double> build_rhs(std::span<const double> u_n) const {
        if (int(u_n.size()) != n_vel()) throw std::invalid_argument("build_rhs: size mismatch");
        std::vector<double> b(static_cast<size_t>(n_total()));
        check(ibmg_build_rhs(ctx_, u_n.data(), b.data(), IBMG_PTR_HOST), ctx_);
        return b;
    }

    std::vector<double> v_cycle(std::span<const double> b) const {
        std::vector<double> z(static_cast<size_t>(n_total()));
        check(ibmg_vcycle(ctx_, b.data(), z.data(), IBMG_PTR_HOST), ctx_);
        return z;
    }

    std::vector<double> gmres_solve(std::span<const double> b, SolveStats* st = nullptr) const {
        std::vector<double> x(static_cast<size_t>(n_total()));
        ibmg_stats s{};
        check(ibmg_solve(ctx_, b.data(), x.data(), &s, IBMG_PTR_HOST), ctx_);
        if (st) *st = {s.iters, s.restarts, s.converged != 0, s.relres, s.setup_ms, s.solve_ms, s.total_ms};
        return x;
    }

    // iteration_matrix_spectrum: Arnoldi Hessenberg matrix of
    // E = I - V(0, A .) on mean-zero pressure, (m_done + 1) x m_done row-major
    // (leading block of the (m+1) x m buffer); its eigenvalues are the Ritz values.
    std::vector<double> iteration_matrix_hessenberg(int m, unsigned long long seed, int* m_done) const {
        std::vector<double> H(size_t(m + 1) * m);
        int done = 0;
        check(ibmg_vcycle_spectrum(ctx_, m, seed, H.data(), &done), ctx_);
        if (m_done) *m_done = done;
        return H;
    }

    // run_simulation: n_steps consecutive steps, the state resident on the device
    // between them; returns the per-step stats of the steps taken (stops at a non-converged step)
    std::vector<SolveStats> run_simulation(int n_steps, std::span<double> u, std::span<double> p, std::span<double> X) {
        if ((int)u.size() != n_vel() || (int)p.size() != N_ * N_)
            throw std::invalid_argument("run_simulation: size mismatch");
        std::vector<ibmg_stats> st(n_steps > 0 ? n_steps : 1);
        int done = 0;
        check(ibmg_run_simulation(ctx_, n_steps, u.data(), p.data(), X.data(), st.data(), &done, IBMG_PTR_HOST), ctx_);
        std::vector<SolveStats> out;
        for (int k = 0; k < done; ++k)
            out.push_back(SolveStats{st[k].iters, st[k].restarts, st[k].converged != 0, st[k].relres, st[k].setup_ms,
                                     st[k].solve_ms, st[k].total_ms});
        return out;
    }
    // step_implicit: u (2N^2) in/out, p (N^2) out, X in/out
    SolveStats step_implicit(std::span<double> u, std::span<double> p, std::span<double> X) {
        if (int(u.size()) != n_vel() || int(p.size()) != N_ * N_ || X.size() != 2 * npts_)
            throw std::invalid_argument("step_implicit: size mismatch");
        ibmg_stats s{};
        check(ibmg_step(ctx_, u.data(), p.data(), X.data(), &s, IBMG_PTR_HOST), ctx_);
        return {s.iters, s.restarts, s.converged != 0, s.relres, s.setup_ms, s.solve_ms, s.total_ms};
    }

    std::vector<double> interpolate(std::span<const double> u) const {
        std::vector<double> U(2 * npts_);
        check(ibmg_interpolate(ctx_, u.data(), U.data(), IBMG_PTR_HOST), ctx_);
        return U;
    }
    std::vector<double> spread(std::span<const double> F) const {
        std::vector<double> f(static_cast<size_t>(n_vel()));
        check(ibmg_spread(ctx_, F.data(), f.data(), IBMG_PTR_HOST), ctx_);
        return f;
    }

    ibmg_ctx* handle() const { return ctx_; }

   private:
    ibmg_ctx* ctx_ = nullptr;
    int N_ = 0;
    size_t npts_ = 0;
};

// transfers.hpp:25-28 equivalents on a system's level `level` -> level+1
inline std::vector<double> restrict_saddle(const SaddleSystem& s, int level, std::span<const double> rf) {
    const int nc = ibmg_level_n(s.handle(), level + 1);
    std::vector<double> rc(3 * size_t(nc) * nc);
    check(ibmg_restrict(s.handle(), level, rf.data(), rc.data(), IBMG_PTR_HOST), s.handle());
    return rc;
}
inline void prolong_saddle_add(const SaddleSystem& s, int level, std::span<const double> ec, std::span<double> wf) {
    check(ibmg_prolong_add(s.handle(), level, ec.data(), wf.data(), IBMG_PTR_HOST), s.handle());
}

// Mesh text format of the reference (write_fiber_mesh / read_fiber_mesh,
// fiber.cpp:142-166): header "m1 m2 ds periodic_s1", then "k l x y" per node at
// 17 significant digits.  A structure set is one block per closed membrane.
inline void write_fiber_mesh(std::ostream& os, std::span<const double> X, double ds, bool periodic = true) {
    const size_t m1 = X.size() / 2;
    const auto prec = os.precision(17);
    os << m1 << ' ' << 1 << ' ' << ds << ' ' << (periodic ? 1 : 0) << '\n';
    for (size_t k = 0; k < m1; ++k) os << k << ' ' << 0 << ' ' << X[2 * k] << ' ' << X[2 * k + 1] << '\n';
    os.precision(prec);
}

struct MeshBlock {
    int m1 = 0, m2 = 0;
    double ds = 0.0;
    bool periodic = true;
    std::vector<double> X;  // (x, y) interleaved, l-major
};

// Next block of the stream; false at end of input.  Errors as the reference's
// reader (std::runtime_error).
inline bool read_fiber_mesh(std::istream& is, MeshBlock& out) {
    int m1 = 0, m2 = 0, per = 0;
    double ds = 0.0;
    if (!(is >> m1)) return false;
    if (!(is >> m2 >> ds >> per)) throw std::runtime_error("read_fiber_mesh: bad header");
    out = MeshBlock{m1, m2, ds, per != 0, std::vector<double>(2 * size_t(m1) * m2)};
    for (long q = 0; q < long(m1) * m2; ++q) {
        int k = 0, l = 0;
        double x = 0.0, y = 0.0;
        if (!(is >> k >> l >> x >> y)) throw std::runtime_error("read_fiber_mesh: bad node line");
        if (k < 0 || k >= m1 || l < 0 || l >= m2) throw std::runtime_error("read_fiber_mesh: node index out of range");
        out.X[2 * (size_t(l) * m1 + k)] = x;
        out.X[2 * (size_t(l) * m1 + k) + 1] = y;
    }
    return true;
}

}  // namespace ibmg::b200
