// oracle_common.h — sparse/dense helpers shared by the CPU oracles (TEST
// INFRASTRUCTURE ONLY; see ibmg_oracle.h): the periodic backward-Euler oracle
// (ibmg_oracle.cpp) and the Dirichlet paper-mode oracle (paper_oracle.cpp).
#ifndef IBMG_ORACLE_COMMON_H
#define IBMG_ORACLE_COMMON_H

#include <algorithm>
#include <cmath>
#include <vector>

namespace orc {

constexpr double kPi = 3.14159265358979323846;

inline int wrap(long i, int n) {
    long r = i % n;
    return int(r < 0 ? r + n : r);
}

struct Trip {
    int r, c;
    double v;
};

// Row-major compressed sparse matrix (the role of ibmg::SparseOperator,
// linalg.hpp:10).  from_trips sums duplicates like Eigen::setFromTriplets.
struct Csr {
    int nr = 0, nc = 0;
    std::vector<long> rp;
    std::vector<int> ci;
    std::vector<double> v;

    static Csr from_trips(int nr, int nc, std::vector<Trip>& t, bool prune_zeros) {
        std::stable_sort(t.begin(), t.end(), [](const Trip& a, const Trip& b) {
            return a.r < b.r || (a.r == b.r && a.c < b.c);
        });
        Csr m;
        m.nr = nr;
        m.nc = nc;
        m.rp.assign(size_t(nr) + 1, 0);
        for (size_t k = 0; k < t.size();) {
            size_t e = k;
            double s = 0.0;
            while (e < t.size() && t[e].r == t[k].r && t[e].c == t[k].c) s += t[e++].v;
            if (!(prune_zeros && s == 0.0)) {
                m.ci.push_back(t[k].c);
                m.v.push_back(s);
                m.rp[size_t(t[k].r) + 1]++;
            }
            k = e;
        }
        for (int i = 0; i < nr; ++i) m.rp[i + 1] += m.rp[i];
        return m;
    }
    double row_dot(int r, const double* x) const {
        double s = 0.0;
        for (long k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * x[ci[k]];
        return s;
    }
    double at(int r, int c) const {
        auto b = ci.begin() + rp[r], e = ci.begin() + rp[r + 1];
        auto it = std::lower_bound(b, e, c);
        return (it != e && *it == c) ? v[it - ci.begin()] : 0.0;
    }
};

// C = A * B with a dense accumulator per row (Eigen's sparse product role in
// transfers.cpp:290).  Exact zeros pruned, like .pruned().
inline Csr spgemm(const Csr& A, const Csr& B) {
    Csr C;
    C.nr = A.nr;
    C.nc = B.nc;
    C.rp.assign(size_t(A.nr) + 1, 0);
    std::vector<double> acc(B.nc, 0.0);
    std::vector<char> mark(B.nc, 0);
    std::vector<int> cols;
    for (int i = 0; i < A.nr; ++i) {
        cols.clear();
        for (long ka = A.rp[i]; ka < A.rp[i + 1]; ++ka) {
            const int k = A.ci[ka];
            const double a = A.v[ka];
            for (long kb = B.rp[k]; kb < B.rp[k + 1]; ++kb) {
                const int j = B.ci[kb];
                if (!mark[j]) {
                    mark[j] = 1;
                    cols.push_back(j);
                }
                acc[j] += a * B.v[kb];
            }
        }
        std::sort(cols.begin(), cols.end());
        for (int j : cols) {
            if (acc[j] != 0.0) {
                C.ci.push_back(j);
                C.v.push_back(acc[j]);
            }
            acc[j] = 0.0;
            mark[j] = 0;
        }
        C.rp[i + 1] = long(C.ci.size());
    }
    return C;
}

// ---- dense LU with partial pivoting ("LU with partial pivoting")
struct DenseLu {
    int m = 0;
    std::vector<double> a;  // row-major m x m, factors in place
    std::vector<double> a0; // (plain-cell cache) the matrix before factoring
    std::vector<int> piv;
    bool factor() {
        piv.resize(m);
        for (int k = 0; k < m; ++k) {
            int p = k;
            double best = std::fabs(a[size_t(k) * m + k]);
            for (int i = k + 1; i < m; ++i) {
                const double v = std::fabs(a[size_t(i) * m + k]);
                if (v > best) {
                    best = v;
                    p = i;
                }
            }
            if (best == 0.0) return false;
            piv[k] = p;
            if (p != k)
                for (int j = 0; j < m; ++j) std::swap(a[size_t(k) * m + j], a[size_t(p) * m + j]);
            const double inv = 1.0 / a[size_t(k) * m + k];
            for (int i = k + 1; i < m; ++i) {
                double& l = a[size_t(i) * m + k];
                l *= inv;
                if (l != 0.0)
                    for (int j = k + 1; j < m; ++j) a[size_t(i) * m + j] -= l * a[size_t(k) * m + j];
            }
        }
        return true;
    }
    void solve(double* x) const {
        for (int k = 0; k < m; ++k)
            if (piv[k] != k) std::swap(x[k], x[piv[k]]);
        for (int i = 0; i < m; ++i) {
            double s = x[i];
            for (int j = 0; j < i; ++j) s -= a[size_t(i) * m + j] * x[j];
            x[i] = s;
        }
        for (int i = m - 1; i >= 0; --i) {
            double s = x[i];
            for (int j = i + 1; j < m; ++j) s -= a[size_t(i) * m + j] * x[j];
            x[i] = s / a[size_t(i) * m + i];
        }
    }
};

// ---- IB kernel (fiber.cpp:12-16, 58-87), periodic: no clipping, the first
// index is left unwrapped and wrapped at use.
inline double delta_1d(double r, double h) {
    const double a = std::fabs(r);
    if (a >= 2.0 * h) return 0.0;
    return (1.0 + std::cos(kPi * r / (2.0 * h))) / (4.0 * h);
}

}  // namespace orc
#endif
