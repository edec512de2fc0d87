// C++ user of the ibmg::b200 facade, written like a reference-side caller of
// SaddleSystem / step_implicit.  Prints one JSON line with the
// step's stats and checksums; tests/test_facade.py compares it with the oracle.
#include <cmath>
#include <cstdio>
#include <vector>

#include "ibmg/b200.hpp"

int main(int argc, char** argv) {
    using namespace ibmg::b200;
    const int N = 64, nb = 128;
    // ellipse (0.5, 0.5), semi-axes 0.3 / 0.15, points at equal parameter spacing
    // (the arclength placement is exercised from Python; here any closed curve works)
    std::vector<double> X(2 * nb);
    const double pi = 3.14159265358979323846;
    double L = 0.0;
    for (int k = 0; k < nb; ++k) {
        const double t = 2 * pi * k / nb;
        X[2 * k] = 0.5 + 0.3 * std::cos(t);
        X[2 * k + 1] = 0.5 + 0.15 * std::sin(t);
    }
    for (int k = 0; k < nb; ++k) {
        const int q = (k + 1) % nb;
        L += std::hypot(X[2 * q] - X[2 * k], X[2 * q + 1] - X[2 * k + 1]);
    }
    SaddleSystem::Params p;
    p.N = N;
    p.dt = 1e-2;
    SaddleSystem sys(p);
    Membrane m{nb, 1e2, L / nb};
    sys.set_structures(std::span<const Membrane>(&m, 1), X);
    std::vector<double> u(2 * N * N, 0.0), pr(N * N, 0.0);
    const SolveStats st = sys.step_implicit(u, pr, X);
    double su = 0, sp = 0, sx = 0;
    for (double v : u) su += v * v;
    for (double v : pr) sp += v * v;
    for (double v : X) sx += v;
    // invalid argument path: mismatched sizes throw std::invalid_argument like the reference
    bool threw = false;
    try {
        std::vector<double> bad(5);
        sys.apply(bad, bad);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    std::printf("{\"iters\": %d, \"converged\": %d, \"relres\": %.3e, \"u2\": %.17g, \"p2\": %.17g, \"xsum\": %.17g, "
                "\"ds\": %.17g, \"threw\": %d}\n",
                st.iterations, st.converged ? 1 : 0, st.relres, su, sp, sx, L / nb, threw ? 1 : 0);
    return st.converged ? 0 : 2;
}
