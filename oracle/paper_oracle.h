/*
 * paper_oracle.h — CPU oracle of the paper-reproduction mode (TEST INFRASTRUCTURE).
 *
 * The Dirichlet (lid-driven cavity), steady Stokes-IB model problem of
 * arXiv 1311.5614 §4-§6 in the reference's own conventions: unknowns in the
 * reference's packed interior ordering (geometry.hpp:54-76), rows
 *   (Lap + alpha E) u - grad p = f,   div u = g         (saddle.cpp:19-38)
 * with the wall data folded into the right-hand side (saddle.cpp:56-94), a
 * thick fiber mesh of m1 x m2 nodes (fiber.hpp:36-50), the wall-reflected
 * transfers (transfers.cpp:107-232, v weight of line 202 corrected) and the
 * Galerkin R E P elasticity (transfers.cpp:234-293).  The solver modules exist
 * only in SPEC.md and are restated from it: n x n box relaxation in
 * lexicographic order, V(nu1,nu2)
 * (SPEC.md:349-352), the coarsest solve, the stand-alone
 * multigrid iteration and right-preconditioned GMRES and
 * the alpha_exp power iteration.
 *
 * Like ibmg_oracle.h this library is the parity checker, never the product.
 */
#ifndef IBMG_PAPER_ORACLE_H
#define IBMG_PAPER_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int N;          /* fine cells per side, power of two >= 2 * coarsest_n */
    int box;        /* box edge in cells (1, 2, 4, 8, 16); a level with n <= box is one box */
    int nu1, nu2;   /* pre / post sweeps */
    int coarsest_n; /* direct solve at this size (4) */
    double alpha;   /* gamma * dt, multiplies E in the momentum rows */
    int order;      /* 0: lexicographic (the paper's smoother); 1: multicolour (SPEC.md:452 opt-in extension):
                       colour (bx mod (R+1)) + (R+1) (by mod (R+1)) with R the level's coupling reach in boxes,
                       colours in ascending order, lexicographic inside a colour */
} porc_params;

typedef struct {
    int iters;      /* V-cycles (mg) or Arnoldi steps (gmres) */
    int converged;  /* relative residual <= rtol */
    int diverged;   /* mg: residual grew for 5 consecutive cycles */
    double relres;  /* true ||b - A x|| / ||b|| at exit */
} porc_stats;

void* porc_create(const porc_params* p, char* err, int errlen);
void porc_destroy(void* ctx);
const char* porc_last_error(void* ctx);

/* Fiber mesh: node (k, l) at X[2 (k + l m1)], closed in s1 (periodic_s1).  Builds
 * E per level (fine assembly + Galerkin), the assembled level operators, the
 * box partition and its factors.  m1 = 0 clears the structure (pure Stokes). */
int porc_set_mesh(void* ctx, int m1, int m2, double ds, const double* X);

int porc_num_levels(void* ctx);
int porc_level_n(void* ctx, int level);
int porc_level_dofs(void* ctx, int level);       /* (n-1) n + n (n-1) + n^2 */
int porc_level_boxes(void* ctx, int level);      /* boxes per side */
int porc_level_reach(void* ctx, int level);      /* coupling reach of the level operator in boxes */

int porc_apply(void* ctx, int level, const double* w, double* out);
int porc_residual(void* ctx, int level, const double* b, const double* w, double* r);
int porc_sweep(void* ctx, int level, const double* b, double* w);
int porc_vcycle(void* ctx, const double* b, double* z);   /* zero initial guess, mean-zero p */
int porc_restrict(int nf, const double* rf, double* rc);
int porc_prolong_add(int nf, const double* ec, double* wf);
long porc_elasticity_triplets(void* ctx, int level, int* rows, int* cols, double* vals, long cap);
long porc_saddle_triplets(void* ctx, int level, int* rows, int* cols, double* vals, long cap);

/* build_rhs (saddle.cpp:96-104) for the lid-driven cavity u(x,1) = (1 - cos 2 pi x)/2
 * (lid = 0 gives homogeneous walls): boundary_fold - spread(gamma A_f X). */
int porc_rhs(void* ctx, int lid, double gamma, double* b);
int porc_spread(void* ctx, const double* F, double* f_vel);   /* fiber.cpp:89-114 */
int porc_interp(void* ctx, const double* vel, double* U);     /* fiber.cpp:116-140 */

/* Stationary multigrid iteration w <- w + V(b - A w) from w = 0. */
int porc_mg_solve(void* ctx, const double* b, double* x, double rtol, int max_iter, porc_stats* st,
                  double* hist, int hist_len);
/* Full (unrestarted) right-preconditioned GMRES, CGS2, x0 = 0. */
int porc_gmres_solve(void* ctx, const double* b, double* x, double rtol, int max_iter, porc_stats* st,
                     double* hist, int hist_len);

/* alpha_exp = 2 / rho(S* L^-1 S A_f) by power iteration on the node positions
 * (PAPER.md:640-659); the Stokes solves use this context's hierarchy with
 * alpha = 0 and MG-GMRES at rtol 1e-10. */
int porc_alpha_exp(void* ctx, double tol, int max_steps, double* alpha_exp, int* steps);

/* iteration_matrix_spectrum: m Arnoldi steps (CGS2) on the error
 * propagator E x = x - V(0, A x) restricted to mean-zero pressure, from the splitmix64 start vector
 * of `seed`; H is the (m+1) x m Hessenberg matrix, row-major.  rho = max |eig(H[:m_done, :m_done])|. */
int porc_vcycle_spectrum(void* ctx, int m, unsigned long long seed, double* H, int* m_done);

#ifdef __cplusplus
}
#endif
#endif
