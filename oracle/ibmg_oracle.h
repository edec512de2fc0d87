/*
 * ibmg_oracle.h — CPU oracle for the implicit-IB MG-FGMRES step (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker, never the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it.  The GPU product path (libibmg_b200.so) never links or calls it.
 *
 * It restates, on a 2D periodic MAC grid with the backward-Euler mass term, the
 * reference's operator semantics (/root/reference/proj/core/src/ *.cpp) and the
 * SPEC-only solver modules (SPEC.md smoothers 390-457, multigrid 278-388,
 * krylov 459-521, timestepper 523-595), with the decisions of SURVEY.md §9 and
 * DESIGN.md §3.  It is written in the reference's own style: explicit sparse
 * assembly (assembly.cpp:5-65), triplet elasticity (elasticity.cpp:62-107),
 * Galerkin R*E*P by sparse products (transfers.cpp:286-293), dense LU box
 * solves — an independent formulation from the GPU's
 * matrix-free window kernels.
 *
 * DOF layout of one level with n x n cells: x = [u | v | p], each n*n doubles,
 * index i + j*n (x fastest).  u(i,j) sits at (i h, (j+1/2) h), v(i,j) at
 * ((i+1/2) h, j h), p(i,j) at the cell centre.
 */
#ifndef IBMG_ORACLE_H
#define IBMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int N;            /* fine cells per side (power of two >= 8) */
    double rho, mu, dt;
    int nu1, nu2;     /* pre/post sweeps (V(1,1) default) */
    int restart;      /* FGMRES restart length (30) */
    int max_iters;    /* total Arnoldi steps cap */
    double rtol;      /* relative residual (1e-10) */
    int coarsest_n;   /* 4 */
    int threads;      /* OpenMP threads for box passes (1 = sequential) */
} orc_params;

typedef struct {
    int iters;        /* Arnoldi steps == V-cycles */
    int restarts;
    int converged;
    double relres;    /* true ||b - Ax|| / ||b|| at exit */
    double setup_ms, solve_ms, total_ms;
} orc_stats;

void* orc_create(const orc_params* p, char* err, int errlen);
void orc_destroy(void* ctx);
const char* orc_last_error(void* ctx);

/* Membranes: n_mem closed curves; nb[m] points each; X interleaved (x,y),
 * concatenated membrane-major.  Builds E' = dt*S*K*S^T per level (Galerkin),
 * assembled level operators, box marking, box factors and the coarse LU. */
int orc_set_structures(void* ctx, int n_mem, const int* nb, const double* kappa,
                       const double* ds, const double* X);

int orc_num_levels(void* ctx);
int orc_level_n(void* ctx, int level);

/* Level operator A_l (full saddle incl. -E'_l) applied to w. */
int orc_apply(void* ctx, int level, const double* w, double* out);
/* r = b - A_l w */
int orc_residual(void* ctx, int level, const double* b, const double* w, double* r);
/* One relaxation sweep (the fixed multicolour schedule) on level l, in place on w. */
int orc_sweep(void* ctx, int level, const double* b, double* w);
/* z = one V(nu1,nu2) cycle from zero initial guess applied to b (fine level). */
int orc_vcycle(void* ctx, const double* b, double* z);
/* Direct bordered solve on the coarsest level. */
int orc_coarse_solve(void* ctx, const double* b, double* x);
/* Periodic transfers on a fine level with nf cells per side. */
int orc_restrict(int nf, const double* rf, double* rc);
int orc_prolong_add(int nf, const double* ec, double* wf);

/* Velocity E'_l as triplets (row, col, val) of the velocity block: returns nnz;
 * writes at most cap entries. */
long orc_elasticity_triplets(void* ctx, int level, int* rows, int* cols, double* vals, long cap);
/* Big-block flags of level l (n/4 x n/4, bx fastest); returns count of big blocks. */
int orc_big_blocks(void* ctx, int level, int* flags);

/* RHS b = [(rho/dt) u^n + S F(X^n) ; 0] (F = kappa D2 X / ds^2, ds^2 quadrature). */
int orc_rhs(void* ctx, const double* u_n, double* b);
/* Fine-level interpolation U_k = sum u delta delta h^2 (points of the structures). */
int orc_interp(void* ctx, const double* u, double* U);
/* Fine-level spread f = sum F_k delta delta ds_m^2. */
int orc_spread(void* ctx, const double* F, double* f);

/* FGMRES(restart) right-preconditioned by one V-cycle, x0 = 0. hist (optional)
 * receives the true/estimated residual history (length hist_len). */
int orc_solve(void* ctx, const double* b, double* x, orc_stats* st, double* hist, int hist_len);

/* One backward-Euler implicit step: rebuild at X^n (lagged), solve, X update.
 * u: 2N^2 in/out, p: N^2 out, X: 2*Nb_total in/out. */
int orc_step(void* ctx, double* u, double* p, double* X, orc_stats* st);

#ifdef __cplusplus
}
#endif
#endif
