// ibmg/b200_paper.hpp — C++ facade over include/ibmg_paper.h: the reference's own
// Dirichlet SaddleSystem interface (proj/core/include/ibmg/*.hpp) on B200, with the
// SPEC-only solver modules behind it.  Vectors are the reference's packed interior
// ordering (DofMap, geometry.hpp:54-76), so a reference caller passes its arrays
// unchanged:
//   * DofMap                                            geometry.hpp:54-76
//   * FiberMesh (m1 x m2 nodes, closed in s1)           fiber.hpp:36-50
//   * SaddleSystem::apply / residual                    saddle.hpp:32-38, saddle.cpp:19-54
//   * build_rhs (lid-driven cavity or homogeneous)      saddle.hpp:46, saddle.cpp:56-104
//   * restrict_saddle / prolong_saddle_add              transfers.hpp:25-28
//   * spread / interpolate                              fiber.hpp:80-83
//   * sweep, v_cycle, mg_solve, gmres_solve
//   * estimate_alpha_exp
// Status 1 -> std::invalid_argument, 3 -> std::runtime_error; unconverged / diverged
// solves are flags.
#pragma once

#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ibmg_paper.h"

namespace ibmg::b200 {

struct DofMap {  // geometry.hpp:54-76 with nx = ny = n
    int n = 0;
    int nu() const { return (n - 1) * n; }
    int nv() const { return n * (n - 1); }
    int np() const { return n * n; }
    int n_vel() const { return nu() + nv(); }
    int n_total() const { return nu() + nv() + np(); }
    int u(int i, int j) const { return (i - 1) + j * (n - 1); }
    int v(int i, int j) const { return nu() + i + (j - 1) * n; }
    int p(int i, int j) const { return n_vel() + i + j * n; }
};

struct FiberMesh {  // fiber.hpp:36-50; X[2 (k + l m1)] = (x, y) of node (k, l)
    int m1 = 0, m2 = 0;
    double ds = 0.0;
    std::vector<double> X;
};

struct PaperStats {
    int iterations = 0;
    bool converged = false, diverged = false;
    double relres = 0.0, solve_ms = 0.0;
};

class CavitySystem {
   public:
    struct Params {
        int N = 32, box = 1, nu1 = 1, nu2 = 1;
        double alpha = 0.0;
        int device = 0;
        int order = 0;  // 0 lexicographic (the paper), 1 multicolour (opt-in)
    };
    explicit CavitySystem(const Params& p) : dm_{p.N} {
        ibmg_paper_params q{p.N, p.box, p.nu1, p.nu2, 4, p.alpha, p.device, p.order};
        const int rc = ibmg_paper_create(&q, &ctx_);
        if (rc == 1) throw std::invalid_argument("CavitySystem: invalid parameters");
        if (rc != 0) throw std::runtime_error("CavitySystem: CUDA initialisation failed");
    }
    ~CavitySystem() { ibmg_paper_destroy(ctx_); }
    CavitySystem(const CavitySystem&) = delete;
    CavitySystem& operator=(const CavitySystem&) = delete;

    const DofMap& dm() const { return dm_; }
    int num_levels() const { return ibmg_paper_num_levels(ctx_); }
    long long kernel_launches() const { return ibmg_paper_kernel_launches(ctx_); }

    void set_mesh(const FiberMesh& m) {
        if (m.X.size() != size_t(2) * m.m1 * m.m2) throw std::invalid_argument("FiberMesh: X size mismatch");
        check(ibmg_paper_set_mesh(ctx_, m.m1, m.m2, m.ds, m.X.data()));
        nodes_ = m.m1 * m.m2;
    }
    void apply(std::span<const double> w, std::span<double> out) const {
        if ((int)w.size() != dm_.n_total() || (int)out.size() != dm_.n_total())
            throw std::invalid_argument("SaddleSystem::apply: size mismatch");
        check(ibmg_paper_apply(ctx_, 0, w.data(), out.data()));
    }
    std::vector<double> residual(std::span<const double> rhs, std::span<const double> w, double* norm = nullptr) const {
        if ((int)w.size() != dm_.n_total() || (int)rhs.size() != dm_.n_total())
            throw std::invalid_argument("SaddleSystem::residual: size mismatch");
        std::vector<double> r(dm_.n_total());
        check(ibmg_paper_residual(ctx_, 0, rhs.data(), w.data(), r.data(), norm));
        return r;
    }
    std::vector<double> build_rhs(bool lid, double gamma) const {
        std::vector<double> b(dm_.n_total());
        check(ibmg_paper_build_rhs(ctx_, lid ? 1 : 0, gamma, b.data()));
        return b;
    }
    void sweep(std::span<const double> b, std::span<double> w) const {
        need(b.size(), w.size());
        check(ibmg_paper_sweep(ctx_, 0, b.data(), w.data()));
    }
    std::vector<double> v_cycle(std::span<const double> b) const {
        need(b.size(), b.size());
        std::vector<double> z(dm_.n_total());
        check(ibmg_paper_vcycle(ctx_, b.data(), z.data()));
        return z;
    }
    std::vector<double> mg_solve(std::span<const double> b, PaperStats& st, double rtol = 1e-6, int max_iter = 100) const {
        return solve(false, b, st, rtol, max_iter);
    }
    std::vector<double> gmres_solve(std::span<const double> b, PaperStats& st, double rtol = 1e-6,
                                    int max_iter = 100) const {
        return solve(true, b, st, rtol, max_iter);
    }
    std::vector<double> spread(std::span<const double> F) const {
        if ((int)F.size() != 2 * nodes_) throw std::invalid_argument("spread: field shape mismatch");
        std::vector<double> f(dm_.n_vel());
        check(ibmg_paper_spread(ctx_, F.data(), f.data()));
        return f;
    }
    std::vector<double> interpolate(std::span<const double> vel) const {
        if ((int)vel.size() != dm_.n_vel()) throw std::invalid_argument("interpolate: size mismatch");
        std::vector<double> U(2 * size_t(nodes_));
        check(ibmg_paper_interpolate(ctx_, vel.data(), U.data()));
        return U;
    }
    // iteration_matrix_spectrum: the (m+1) x m Hessenberg matrix of m Arnoldi steps
    // on the V-cycle's error propagator; rho = max |eig(H[:done, :done])|
    std::vector<double> iteration_matrix_hessenberg(int m, unsigned long long seed, int* done = nullptr) const {
        std::vector<double> H(size_t(m + 1) * m);
        check(ibmg_paper_vcycle_spectrum(ctx_, m, seed, H.data(), done));
        return H;
    }
    double estimate_alpha_exp(double tol = 1e-4, int max_steps = 1000, int* steps = nullptr) const {
        double a = 0.0;
        check(ibmg_paper_alpha_exp(ctx_, tol, max_steps, &a, steps));
        return a;
    }

   private:
    void check(int rc) const {
        if (rc == 0) return;
        const std::string msg = ibmg_paper_last_error(ctx_);
        if (rc == 1) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    void need(size_t a, size_t b) const {
        if ((int)a != dm_.n_total() || (int)b != dm_.n_total()) throw std::invalid_argument("size mismatch");
    }
    std::vector<double> solve(bool gmres, std::span<const double> b, PaperStats& st, double rtol, int max_iter) const {
        need(b.size(), b.size());
        std::vector<double> x(dm_.n_total());
        ibmg_paper_stats s{};
        check((gmres ? ibmg_paper_gmres_solve : ibmg_paper_mg_solve)(ctx_, b.data(), x.data(), rtol, max_iter, &s,
                                                                     nullptr, 0));
        st = PaperStats{s.iters, s.converged != 0, s.diverged != 0, s.relres, s.solve_ms};
        return x;
    }
    DofMap dm_;
    ibmg_paper* ctx_ = nullptr;
    int nodes_ = 0;
};

// transfers.hpp:25-28 on the hierarchy of a system (level -> level + 1 and back)
inline void restrict_saddle(ibmg_paper* ctx, int level, std::span<const double> rf, std::span<double> rc) {
    if (ibmg_paper_restrict(ctx, level, rf.data(), rc.data())) throw std::invalid_argument("restrict_saddle: size mismatch");
}

}  // namespace ibmg::b200
