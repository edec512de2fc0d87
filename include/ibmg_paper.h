/*
 * ibmg_paper.h — C ABI of the paper-reproduction mode on B200.
 *
 * The model problem of arXiv 1311.5614 §4-§6 in the reference's own conventions:
 * the lid-driven cavity on the unit square (Dirichlet walls, geometry.hpp:17-18),
 * unknowns in the reference's packed interior ordering (geometry.hpp:54-76)
 *   x = [u (n-1) n | v n (n-1) | p n n],  u(i,j) -> (i-1) + j (n-1),  v(i,j) -> nu + i + (j-1) n,
 * rows exactly SaddleSystem::apply's (saddle.cpp:19-38)
 *   momentum:   (Lap + alpha E) u - grad p,   E = S A_f S* (elasticity.cpp:88-107, ds^2 h^2 scaling)
 *   continuity: div u
 * a thick fiber mesh of m1 x m2 nodes closed in s1 (fiber.hpp:36-50), wall-reflected
 * transfers (transfers.cpp:107-232, the v weight of line 202 corrected) and Galerkin
 * coarse elasticity R E P (transfers.cpp:286-293).  The smoother is the paper's n x n
 * box relaxation in LEXICOGRAPHIC order
 * for any power-of-two box edge; the GPU runs the lexicographic Gauss-Seidel order
 * exactly as a dataflow pipeline (a box waits for the earlier boxes it is coupled to).
 *
 * All vectors are host arrays; calls are synchronous.  Status codes as ibmg_gpu.h:
 * 0 OK, 1 INVALID (std::invalid_argument in the reference), 3 CUDA.  Unconverged and
 * diverged solves are flags in the stats, not errors.
 */
#ifndef IBMG_PAPER_H
#define IBMG_PAPER_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ibmg_paper ibmg_paper;

typedef struct {
    int N;          /* fine cells per side, power of two >= 2 * coarsest_n (GridGeometry nx = ny) */
    int box;        /* box edge in cells: 1, 2, 4, 8, 16 (BoxPartition.n) */
    int nu1, nu2;   /* CyclePolicy */
    int coarsest_n; /* direct solve at this size (4) */
    double alpha;   /* gamma dt (SaddleSystem::alpha, saddle.hpp:23) */
    int device;     /* CUDA device ordinal */
    int order;      /* 0: lexicographic sweep, the paper's smoother (dataflow pipeline); 1: multicolour ordering
                       (the opt-in extension of SPEC.md:452): colour (bx mod (R+1)) + (R+1) (by mod (R+1)), R the
                       level's coupling reach in boxes, one launch per colour */
} ibmg_paper_params;

typedef struct {
    int iters;      /* V-cycles (mg) or Arnoldi steps (gmres) */
    int converged;
    int diverged;   /* mg only: the residual grew in 5 consecutive cycles */
    double relres;  /* true ||b - A x|| / ||b|| */
    double setup_ms, solve_ms;
} ibmg_paper_stats;

/* Replaces SaddleSystem + build_hierarchy + build_partition/build_local_solvers
 * (saddle.cpp:7-13). */
int ibmg_paper_create(const ibmg_paper_params* params, ibmg_paper** out);
void ibmg_paper_destroy(ibmg_paper* ctx);
const char* ibmg_paper_last_error(const ibmg_paper* ctx);

/* Replaces FiberMesh + assemble_elasticity + galerkin_coarsen_elasticity
 * (fiber.hpp:36-50, elasticity.cpp:88-107, transfers.cpp:286-293): node (k, l) at
 * X[2 (k + l m1)]; m1 = 0 clears the structure.  Rebuilds every level's E, box
 * inverses and coupling reach.  INVALID when a node's kernel support crosses the
 * walls (require_supports_interior, fiber.cpp:18-32). */
int ibmg_paper_set_mesh(ibmg_paper* ctx, int m1, int m2, double ds, const double* X);

int ibmg_paper_num_levels(const ibmg_paper* ctx);
int ibmg_paper_level_n(const ibmg_paper* ctx, int level);
int ibmg_paper_level_dofs(const ibmg_paper* ctx, int level);
int ibmg_paper_level_boxes(const ibmg_paper* ctx, int level);  /* boxes per side */
int ibmg_paper_level_reach(const ibmg_paper* ctx, int level);  /* coupling reach in boxes (pipeline skew - 1) */

/* SaddleSystem::apply / residual (saddle.cpp:19-54) on a level. */
int ibmg_paper_apply(ibmg_paper* ctx, int level, const double* w, double* out);
int ibmg_paper_residual(ibmg_paper* ctx, int level, const double* b, const double* w, double* r, double* norm);
/* restrict_saddle / prolong_saddle_add (transfers.cpp:107-134, 209-232): level -> level + 1 and back. */
int ibmg_paper_restrict(ibmg_paper* ctx, int level, const double* rf, double* rc);
int ibmg_paper_prolong_add(ibmg_paper* ctx, int level, const double* ec, double* wf);
/* sweep: one lexicographic box sweep in place. */
int ibmg_paper_sweep(ibmg_paper* ctx, int level, const double* b, double* w);
/* v_cycle from a zero initial guess, mean-zero pressure. */
int ibmg_paper_vcycle(ibmg_paper* ctx, const double* b, double* z);
/* E of a level (alpha-free) as host triplets; returns nnz (rows == NULL sizes). */
long ibmg_paper_elasticity_triplets(ibmg_paper* ctx, int level, int* rows, int* cols, double* vals, long cap);

/* build_rhs (saddle.cpp:96-104) with the lid data u(x,1) = (1 - cos 2 pi x)/2 (lid != 0)
 * or homogeneous walls: boundary_fold - spread(gamma A_f X). */
int ibmg_paper_build_rhs(ibmg_paper* ctx, int lid, double gamma, double* b);
/* spread / interpolate (fiber.cpp:89-140) on packed velocities; F, U interleaved per node. */
int ibmg_paper_spread(ibmg_paper* ctx, const double* F, double* f_vel);
int ibmg_paper_interpolate(ibmg_paper* ctx, const double* vel, double* U);

/* mg_solve / gmres_solve: x0 = 0, relative residual rtol, cap
 * max_iter; hist (optional, hist_len doubles) receives the relative residuals. */
int ibmg_paper_mg_solve(ibmg_paper* ctx, const double* b, double* x, double rtol, int max_iter,
                        ibmg_paper_stats* stats, double* hist, int hist_len);
int ibmg_paper_gmres_solve(ibmg_paper* ctx, const double* b, double* x, double rtol, int max_iter,
                           ibmg_paper_stats* stats, double* hist, int hist_len);
/* estimate_alpha_exp: power iteration on S* L^-1 S A_f. */
int ibmg_paper_alpha_exp(ibmg_paper* ctx, double tol, int max_steps, double* alpha_exp, int* steps);

/* iteration_matrix_spectrum: m Arnoldi steps (CGS2) on the error
 * propagator E x = x - v_cycle(0, A x) restricted to mean-zero pressure, from the splitmix64 start
 * vector of `seed`; H receives the (m+1) x m Hessenberg matrix (row-major), m_done the steps taken.
 * The spectral radius estimate is max |eig(H[:m_done, :m_done])|. */
int ibmg_paper_vcycle_spectrum(ibmg_paper* ctx, int m, unsigned long long seed, double* H, int* m_done);

long long ibmg_paper_kernel_launches(const ibmg_paper* ctx);

#ifdef __cplusplus
}
#endif
#endif
