/*
 * ibmg_gpu.h — C ABI of the B200-native implicit-IB MG-FGMRES solver.
 *
 * Drop-in boundary for the reference's solver interface.
 * Every entry point names the reference function it replaces; plain pointers
 * and sizes only.  `ptr_kind` says whether the caller's arrays are host
 * (IBMG_PTR_HOST, copies are made inside the call) or device memory on the
 * context's GPU (IBMG_PTR_DEVICE).  All calls are synchronous with respect
 * to the caller's pointers on return; work is ordered on the context's own
 * CUDA stream.  One context per host thread.
 *
 * DOF layout of a level with n x n cells (periodic, h = 1/n):
 *   x = [u | v | p], each n*n doubles, index i + j*n (x fastest);
 *   u(i,j) at (i h, (j+1/2) h), v(i,j) at ((i+1/2) h, j h), p(i,j) at the cell centre.
 * This is the reference's packed ordering (fields.hpp:53-56, geometry.hpp:67-72)
 * specialised to periodic boundaries, where every face is an unknown.
 *
 * Operator (sign convention SURVEY.md §9-D3):
 *   momentum:   (rho/dt - mu L) u + G p - E' u,  E' = dt * S K S^T (ds^2 quadrature)
 *   continuity: -D u
 * which is -1 x the reference's SaddleSystem rows (saddle.hpp:11-18) plus the
 * backward-Euler mass term.
 *
 * Status codes: 0 OK, 1 INVALID (std::invalid_argument in the reference),
 * 2 NOT_CONVERGED (stats still filled; SPEC.md:478 flag), 3 CUDA, 4 NCCL.
 */
#ifndef IBMG_GPU_H
#define IBMG_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

enum { IBMG_OK = 0, IBMG_INVALID = 1, IBMG_NOT_CONVERGED = 2, IBMG_CUDA = 3, IBMG_NCCL = 4 };
enum { IBMG_PTR_HOST = 0, IBMG_PTR_DEVICE = 1 };

typedef struct ibmg_ctx ibmg_ctx;

typedef struct {
    int N;            /* fine cells per side, power of two >= 8 (GridGeometry nx = ny, geometry.hpp:19-31) */
    double rho, mu, dt;
    int nu1, nu2;     /* V(nu1,nu2) (CyclePolicy) */
    int restart;      /* FGMRES restart length (30) */
    int max_iters;    /* total Arnoldi-step cap (GmresConfig.max_iter) */
    double rtol;      /* relative residual threshold (1e-10) */
    int coarsest_n;   /* 4 (SPEC.md "Coarsest level at 4x4 cells") */
    int device;       /* CUDA device ordinal */
} ibmg_params;

typedef struct {
    int iters;        /* Arnoldi steps == V-cycles applied */
    int restarts;
    int converged;
    double relres;    /* true ||b - A x|| / ||b|| */
    double setup_ms;  /* structure rebuild at X^n (windows, lists, box inverses) */
    double solve_ms;  /* FGMRES */
    double total_ms;  /* whole step */
} ibmg_stats;

/* Replaces SaddleSystem construction + build_hierarchy (saddle.cpp:7-13). */
int ibmg_create(const ibmg_params* params, ibmg_ctx** out);
void ibmg_destroy(ibmg_ctx* ctx);
const char* ibmg_last_error(const ibmg_ctx* ctx);

/* Replaces FiberMesh + assemble_elasticity + galerkin_coarsen_elasticity
 * (fiber.hpp:36-50, elasticity.cpp:88-107, transfers.cpp:286-293): n_mem closed
 * membranes, nb[m] points each, stiffness kappa[m], spacing ds[m]; X interleaved
 * (x, y), membrane-major, 2*sum(nb) doubles.  Rebuilds all per-level data. */
int ibmg_set_structures(ibmg_ctx* ctx, int n_mem, const int* nb, const double* kappa,
                        const double* ds, const double* X, int ptr_kind);

int ibmg_num_levels(const ibmg_ctx* ctx);
int ibmg_level_n(const ibmg_ctx* ctx, int level);

/* Time scheme of the IB coupling: implicit = 1 (default) puts
 * E' = dt S K S^T on the left (step_implicit); implicit = 0 drops it (E' = 0 on
 * every level, pure Stokes + mass solve) while ibmg_step / ibmg_build_rhs keep
 * the spread spring forces S F(X^n) on the right: step_explicit (Eqs. 9-12). */
int ibmg_set_scheme(ibmg_ctx* ctx, int implicit);

/* Replaces SaddleSystem::apply (saddle.cpp:19-38) on level `level` (0 = fine). */
int ibmg_apply(ibmg_ctx* ctx, int level, const double* w, double* out, int ptr_kind);
/* Replaces SaddleSystem::residual (saddle.cpp:48-54): r = b - A w, norm optional. */
int ibmg_residual(ibmg_ctx* ctx, int level, const double* b, const double* w, double* r,
                  double* norm, int ptr_kind);
/* Replaces restrict_saddle (transfers.cpp:107-134): level -> level+1. */
int ibmg_restrict(ibmg_ctx* ctx, int level, const double* rf, double* rc, int ptr_kind);
/* Replaces prolong_saddle_add (transfers.cpp:209-232, v weights corrected): wf += P ec. */
int ibmg_prolong_add(ibmg_ctx* ctx, int level, const double* ec, double* wf, int ptr_kind);
/* Replaces the SPEC smoother `sweep`: one multicolour box sweep in place. */
int ibmg_sweep(ibmg_ctx* ctx, int level, const double* b, double* w, int ptr_kind);
/* Replaces `v_cycle`: z = V(nu1,nu2)(0, b), mean-zero pressure. */
int ibmg_vcycle(ibmg_ctx* ctx, const double* b, double* z, int ptr_kind);
/* Replaces `coarsest_solve` on the coarsest level. */
int ibmg_coarse_solve(ibmg_ctx* ctx, const double* b, double* x, int ptr_kind);
/* Big-block flags of a level ((n/4)^2 ints, host); returns the count or -1. */
int ibmg_big_blocks(ibmg_ctx* ctx, int level, int* flags_host);

/* Assembled E'_level (velocity block, E' = dt S K S^T Galerkin-coarsened) as host
 * triplets: returns nnz (call with rows == NULL to size); the role of
 * assemble_elasticity / galerkin_coarsen_elasticity's matrices
 * (elasticity.cpp:88-107, transfers.cpp:286-293). */
long ibmg_elasticity_triplets(ibmg_ctx* ctx, int level, int* rows, int* cols, double* vals, long cap);

/* Debug only (not the solver path): one dataflow sweep on a multi-tile level with
 * per-task globaltimer stamps (device b, w); returns the trace length in words. */
long ibmg_debug_sweep_trace(ibmg_ctx* ctx, int level, const double* b, double* w, unsigned long long* out, long cap);

/* Debug only: one cluster-kernel launch (device b, w at the first cluster level)
 * with (globaltimer, tag) stamps of CTA 0 after each cluster barrier; returns the
 * stamp count. */
long ibmg_debug_cluster_trace(ibmg_ctx* ctx, const double* b, double* w, unsigned long long* out, long cap);
/* First level of the 16-CTA cluster kernel (levels n <= 128), or -1 when the
 * cluster path is off (IBMG_CLUSTER=0 or no cluster launch on the device). */
int ibmg_cluster_level(const ibmg_ctx* ctx);

/* Debug only: one coarse-cycle launch (device b, w at the first coarse-kernel
 * level) with thread-0 globaltimer phase stamps; returns the stamp count. */
long ibmg_debug_coarse_trace(ibmg_ctx* ctx, const double* b, double* w, unsigned long long* out, long cap);

/* Replaces build_rhs (saddle.cpp:96-104): b = [(rho/dt) u^n + S F(X^n); 0]. */
int ibmg_build_rhs(ibmg_ctx* ctx, const double* u_n, double* b, int ptr_kind);
/* Replaces interpolate (fiber.cpp:116-140): U = S^T u (h^2 weights), 2*npts. */
int ibmg_interpolate(ibmg_ctx* ctx, const double* u, double* U, int ptr_kind);
/* Replaces spread (fiber.cpp:89-114): f = S F (ds^2 weights), 2*N^2. */
int ibmg_spread(ibmg_ctx* ctx, const double* F, double* f, int ptr_kind);

/* Replaces gmres_solve re-specified as FGMRES(restart) with
 * one V-cycle as right preconditioner, x0 = 0. */
int ibmg_solve(ibmg_ctx* ctx, const double* b, double* x, ibmg_stats* stats, int ptr_kind);

/* Replaces iteration_matrix_spectrum (§5.2): Arnoldi of
 * dimension m (<= restart) on the multigrid error-propagation operator
 * E x = x - V(0, A x), restricted to mean-zero pressure, from a seeded random
 * start.  H: host (m+1) x m row-major Hessenberg matrix (its eigenvalues are
 * the Ritz values; rho = max modulus); *m_done = steps completed. */
int ibmg_vcycle_spectrum(ibmg_ctx* ctx, int m, unsigned long long seed, double* H, int* m_done);

/* Replaces step_implicit: rebuild at X^n, RHS, solve,
 * X^{n+1} = X^n + dt S^T u^{n+1}.  u: 2N^2 in/out, p: N^2 out, X in/out. */
int ibmg_step(ibmg_ctx* ctx, double* u, double* p, double* X, ibmg_stats* stats, int ptr_kind);
/* Replaces run_simulation: n_steps consecutive implicit (or, after
 * ibmg_set_scheme(ctx, 0), explicit) steps with the state resident on the device between
 * them — host arrays are uploaded once and read back once.  stats (optional) receives
 * n_steps records, *steps_done the steps taken; the run stops at the first step that
 * does not converge (status 2).  The results equal n_steps calls of ibmg_step bit for bit. */
int ibmg_run_simulation(ibmg_ctx* ctx, int n_steps, double* u, double* p, double* X, ibmg_stats* stats,
                        int* steps_done, int ptr_kind);

/* Number of kernels this context has launched (evidence for bench's gpu_launches). */
long long ibmg_kernel_launches(const ibmg_ctx* ctx);
/* Cap the grid of the persistent cooperative kernels (0 = all SMs).  For many
 * concurrent contexts on one GPU (batches of independent problems, C5) a cap of
 * ~SMs/contexts lets their sweeps run side by side instead of serialising.  A
 * cap > 0 also turns programmatic dependent launch off for the context (its
 * early-resident waiting CTAs would take SMs from the other contexts), and the
 * latency-hiding extras whose discarded work costs the other contexts
 * throughput: the speculative V-cycle behind the FGMRES dots and the
 * canonical-order box inverses. */
int ibmg_set_grid_limit(ibmg_ctx* ctx, int max_ctas);
/* Per-kernel CUDA-event timing on the context stream (bench roofline evidence):
 * enable=1 starts (and clears) the accumulation; report writes JSON
 * {"kernel": [total_ms, launches], ...} and returns its length. */
int ibmg_profile(ibmg_ctx* ctx, int enable);
int ibmg_profile_report(ibmg_ctx* ctx, char* buf, int cap);
/* The context's CUDA stream (cudaStream_t), for callers timing with events. */
void* ibmg_stream(const ibmg_ctx* ctx);
/* Stream ordering of device-pointer inputs: every call given IBMG_PTR_DEVICE
 * arrays first makes the context's stream wait on an event recorded on this
 * caller stream (cudaStream_t; NULL = the legacy default stream, the default),
 * so inputs still being produced there are read only after their producers.
 * Outputs are complete when a call returns (the context stream is
 * synchronised), so no ordering is needed on the way out. */
int ibmg_set_input_stream(ibmg_ctx* ctx, void* stream);

/* ---- Slab partition of one problem (BASELINE north_star: large
 * fine grids slab-partitioned across 2/4/8 GPUs with NVLink halo exchange per
 * smoothing sweep and coarse-level agglomeration).  No reference counterpart:
 * the reference is single-threaded CPU code; the group takes the
 * same calls as a context (SPEC.md:349 v_cycle, :474 gmres_solve, :548
 * step_implicit) on host whole-grid vectors.
 *
 * nslabs y-slabs of the fine grid, slab r on devices[r] (slabs may share a
 * GPU; distinct GPUs need peer access).  A level is distributed while each
 * slab has >= max(min_rows, 24) rows, a multiple of 32, and >= min_cells
 * cells; coarser levels are agglomerated (every slab runs them on the whole
 * level).  Every colour pass on a distributed level is followed by a seam
 * merge and a 24-row halo push between neighbouring slabs; FGMRES dots are
 * summed over the slabs in rank order. */
typedef struct ibmg_group ibmg_group;

/* Host-only plan (no GPU needed): returns the number of distributed levels
 * (-1 on invalid arguments) and, if rows_out != NULL, the owned rows
 * rows_out[(r * nlev + l) * 2 + {0, 1}] = [y0, y1) of slab r on level l. */
int ibmg_slab_plan(int N, int coarsest_n, int nslabs, int min_rows, long min_cells, int* rows_out);
/* In-process group: all nslabs slabs in this process, slab r on devices[r]
 * (NULL: params->device); exchanges are peer copies ordered by CUDA events.
 * min_rows < 0 is a test mode that distributes levels even for one slab. */
int ibmg_group_create(const ibmg_params* params, int nslabs, const int* devices, int min_rows, long min_cells,
                      ibmg_group** out);
/* NCCL group: one slab per process (torchrun, one rank per GPU on
 * params->device); halos / seams by ncclSend/ncclRecv, dots by ncclAllReduce,
 * agglomeration by ncclAllGather, stream-ordered.  nccl_id: the 128-byte
 * ncclUniqueId from ibmg_nccl_unique_id on rank 0, broadcast by the caller.
 * Host outputs (vcycle/solve/step/sweep) are whole on every rank. */
int ibmg_nccl_unique_id(void* id_out);
int ibmg_group_create_nccl(const ibmg_params* params, int rank, int nranks, const void* nccl_id, int min_rows,
                           long min_cells, ibmg_group** out);
void ibmg_group_destroy(ibmg_group* group);
const char* ibmg_group_last_error(const ibmg_group* group);
int ibmg_group_distributed_levels(const ibmg_group* group);
long long ibmg_group_kernel_launches(const ibmg_group* group);
/* Number of halo exchanges / allgathers issued (evidence for tests and bench). */
long long ibmg_group_exchanges(const ibmg_group* group);
/* As ibmg_set_structures, on every slab (host arrays). */
int ibmg_group_set_structures(ibmg_group* group, int n_mem, const int* nb, const double* kappa, const double* ds,
                              const double* X);
/* One distributed sweep on a distributed level (host whole-level b, w; w in place). */
int ibmg_group_sweep(ibmg_group* group, int level, const double* b, double* w);
/* As ibmg_vcycle / ibmg_solve / ibmg_step with host whole-grid vectors. */
int ibmg_group_vcycle(ibmg_group* group, const double* b, double* z);
int ibmg_group_solve(ibmg_group* group, const double* b, double* x, ibmg_stats* stats);
int ibmg_group_step(ibmg_group* group, double* u, double* p, double* X, ibmg_stats* stats);

/* ---- Batch of independent problems stepped in lockstep (C5).
 * No reference counterpart (the reference solves one system per call): the
 * batch takes the reference's step_implicit for `count`
 * problems at once.  nslots contexts of one grid size (64 <= N <= 512); every
 * slot gets its own structures; ibmg_batch_step runs the rebuilds per slot
 * and then ONE launch per smoother / transfer / Krylov phase for all slots
 * (tile and block tasks of all problems in one dataflow DAG, the problem index
 * in the grid), FGMRES advancing every unconverged problem one Arnoldi step
 * per round.  Results equal the single-context step's (same arithmetic per
 * problem). */
typedef struct ibmg_batch ibmg_batch;
int ibmg_batch_create(const ibmg_params* params, int nslots, ibmg_batch** out);
void ibmg_batch_destroy(ibmg_batch* batch);
const char* ibmg_batch_last_error(const ibmg_batch* batch);
long long ibmg_batch_kernel_launches(const ibmg_batch* batch);
void* ibmg_batch_stream(const ibmg_batch* batch);
/* As ibmg_set_structures for slot `slot` (host arrays; the rebuild happens in the step). */
int ibmg_batch_set_structures(ibmg_batch* batch, int slot, int n_mem, const int* nb, const double* kappa,
                              const double* ds, const double* X);
/* One implicit step of slots 0..count-1: u[k] (2N^2 in/out), p[k] (N^2 out), X[k]
 * (in/out), host or device pointers; stats[k] per problem (may be NULL). */
int ibmg_batch_step(ibmg_batch* batch, int count, double* const* u, double* const* p, double* const* X,
                    ibmg_stats* stats, int ptr_kind);
/* ibmg_batch_step in two phases, so that one thread can prepare (upload,
 * rebuild at X^n, RHS: host colouring + setup kernels) the next batch while
 * another solves this one: prepare(count, u, X) then solve(count, u, p, X). */
int ibmg_batch_prepare(ibmg_batch* batch, int count, double* const* u, double* const* X, int ptr_kind);
int ibmg_batch_solve(ibmg_batch* batch, int count, double* const* u, double* const* p, double* const* X,
                     ibmg_stats* stats, int ptr_kind);

#ifdef __cplusplus
}
#endif
#endif
