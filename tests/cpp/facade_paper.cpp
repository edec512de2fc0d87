// Compiled C++ caller of the paper-mode facade (include/ibmg/b200_paper.hpp): the
// Table 2 cell b = 4, V(1,1), relative stiffness 100 at h = 2^-6 (11 iterations in
// PAPER.md:1069-1083) through the reference's SaddleSystem-style interface.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "ibmg/b200_paper.hpp"

int main() {
    using namespace ibmg::b200;
    const int N = 64;
    FiberMesh m;
    m.m1 = 19 * N / 8;
    m.m2 = 3 * N / 32 + 1;
    const double r = 0.25, w = 1.0 / 16;
    m.ds = 2 * std::numbers::pi * r / m.m1;
    m.X.resize(size_t(2) * m.m1 * m.m2);
    for (int l = 0; l < m.m2; ++l)
        for (int k = 0; k < m.m1; ++k) {
            const double rad = r + l * (w / (m.m2 - 1)), th = k * m.ds / r;
            m.X[2 * (k + size_t(l) * m.m1)] = 0.5 + rad * std::cos(th);
            m.X[2 * (k + size_t(l) * m.m1) + 1] = 0.5 + rad * std::sin(th);
        }
    const double alpha = 100 * 3.93;
    CavitySystem sys({N, 4, 1, 1, alpha, 0});
    sys.set_mesh(m);
    std::vector<double> b = sys.build_rhs(true, alpha);
    PaperStats st;
    std::vector<double> x = sys.gmres_solve(b, st);
    double nrm = 0.0;
    sys.residual(b, x, &nrm);
    double bn = 0.0;
    for (double v : b) bn += v * v;
    bool threw = false;
    try {
        std::vector<double> bad(7);
        sys.apply(bad, bad);
    } catch (const std::invalid_argument&) { threw = true; }
    std::printf("iters %d converged %d relres %.3e true %.3e threw %d launches %lld\n", st.iterations, int(st.converged),
                st.relres, nrm / std::sqrt(bn), int(threw), sys.kernel_launches());
    return (st.converged && threw) ? 0 : 1;
}
