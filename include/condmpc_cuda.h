/* condmpc_cuda.h — C ABI of the B200 condensed-space IPM hot path.
 *
 * Drop-in boundary for the per-iteration body of condmpc::ipm::solve
 * (/root/reference/proj/src/ipm.cpp:160-268). All matrices are FP64, column-major
 * with leading dimension = rows (Eigen::MatrixXd layout,
 * proj/include/condmpc/types.hpp:10-11). Pointers are borrowed for the call.
 * Return codes: 0 ok, 1 not positive definite (pivot reported), <0 error (message in
 * cmpc_last_error(), thread-local). One context = one QP = one CUDA stream; contexts
 * are independent, so concurrent solves on different threads are safe
 * (proj/src/verify.cpp:104-111 runs ipm::solve concurrently).
 */
#ifndef CONDMPC_CUDA_H
#define CONDMPC_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMPC_OK 0
#define CMPC_NOT_PD 1
#define CMPC_ERR_DIM (-1)
#define CMPC_ERR_ARG (-2)
#define CMPC_ERR_CUDA (-3)

typedef struct cmpc_ctx cmpc_ctx;

int cmpc_abi_version(void);
const char* cmpc_last_error(void);
/* kernels launched by this thread so far (all entry points) */
long long cmpc_launch_count(void);

/* context = the device-resident DenseQp + IpmState of one solve */
int cmpc_ctx_create(cmpc_ctx** out, int device);
void cmpc_ctx_destroy(cmpc_ctx* ctx);
/* Per-context options (no process-wide switches): "jtl_recurrence" 1 (default) carries J'lambda
 * across a step, 0 recomputes it by a pass over J as compute_residuals does (ipm.cpp:46-70);
 * "rhs_pass" 0/1 (default) fuses J'(r2 - sigma r3) into the condensation, 2 runs it as its own
 * pass; "graphs" 1 (default) replays the per-iteration segments as CUDA graphs, 0 launches them
 * eagerly; "small_path" 1 (default) runs the whole solve in one CTA (every decision on the
 * device, the log hook replayed afterwards) for QPs with n <= 32 whose J fits in shared memory
 * when no inspect hook is given, 0 never; "speculate" 1 (default) enqueues the step update and
 * the next residual pass behind the factor/step segment before the host has seen the step,
 * gated on the device's own evaluation of line-search trial 0 (the host re-checks it and
 * finishes the line search itself when trial 0 is refused), 0 waits for the host's decision.
 * "markov" 1 (default) reads the SYRK prototypes of a QP built by cmpc_build_qp from the
 * Markov table (G_k = A_K^k B per state, never materialising P) when every prototype is a
 * state row and the materialised P would exceed 64 MB, 2 whenever every prototype is a state
 * row, 0 always materialises P (takes effect at the next cmpc_build_qp).
 * Unknown keys or values: CMPC_ERR_DIM. Takes effect at the next solve. */
int cmpc_ctx_set_option(cmpc_ctx* ctx, const char* key, int64_t value);

/* Load DenseQp{H, h, h0, J, d} (proj/include/condmpc/reduction.hpp:25-33).
 * on_device = 0: host pointers (copied H2D); 1: device pointers (copied D2D).
 * Runs the exact structure analysis of J (distinct rows up to sign, prefix widths). */
int cmpc_load_qp(cmpc_ctx* ctx, int64_t n, int64_t m, const double* H, const double* h, double h0,
                 const double* J, const double* d, int on_device);

/* The structured LQ-MPC problem (LqProblemData, proj/include/condmpc/problem.hpp:22-45).
 * Matrices column-major (Eigen's layout, layout = 0) or row-major (layout = 1, e.g. C-ordered
 * numpy arrays: transposed on the device instead of on the host); w is T x n_x stage-major (w[t * n_x + i]); bounds
 * may hold +-inf (rows of infinite bounds are skipped, as in reduction.cpp:191-251); S, K,
 * E, F, w may be NULL when zero / n_c == 0. */
typedef struct cmpc_lq_problem {
  int64_t nx, nu, nc, T;
  const double *A, *B, *Q, *Qf, *R, *S, *E, *F;
  const double *gl, *gu, *xl, *xu, *ul, *uu;
  const double *w, *x_bar, *K;
  int64_t layout;
} cmpc_lq_problem;
/* build_dense_qp (proj/src/reduction.cpp:255-268) on the device, then load it like
 * cmpc_load_qp without the dense J ever crossing PCIe; the problem stays resident for the
 * two calls below. Replaces the reference's host build + upload. */
int cmpc_build_qp(cmpc_ctx* ctx, const cmpc_lq_problem* problem);
/* refresh_initial_state (reduction.cpp:270-280) on a device-built QP: new x_bar -> free
 * response, h, h0, d recomputed on the device; H, J and the analysed structure are kept. */
int cmpc_refresh_initial_state(cmpc_ctx* ctx, const double* x_bar);
/* The loaded QP's H (n x n), h, h0, d (host pointers, each nullable; tests and hooks) */
int cmpc_get_qp(cmpc_ctx* ctx, double* H, double* h, double* h0, double* d);
/* recover_trajectory (reduction.cpp:282-314) on the device: x ((T+1) x n_x stage-major),
 * u (T x n_u), Eq. (1a) objective; v NULL = the last solve's iterate on the device. */
int cmpc_recover_trajectory(cmpc_ctx* ctx, const double* v, double* x, double* u, double* objective);
/* A new context (own stream and iterate buffers) holding a device copy of ctx's loaded QP
 * and its structure: instances that share H and J and differ in h, h0, d (the
 * refresh_initial_state case, config 5's batch) are cloned and then updated with
 * cmpc_update_qp_affine instead of re-uploading and re-analysing J. */
int cmpc_ctx_clone(cmpc_ctx* src, cmpc_ctx** out);
/* Solve `count` loaded contexts concurrently: a pool of `threads` host threads, each driving
 * its contexts' own streams (the GPU overlaps the instances). v_out: count x n (nullable),
 * scal_out: count x 14 (cmpc_solve's out_scalars per instance). */
int cmpc_solve_batch(cmpc_ctx** ctxs, int64_t count, const double* opts, int64_t max_iter,
                     double* v_out, double* scal_out, int threads);
/* Solve `count` instances sharing H and J (config 5): h_all count x n, h0_all count,
 * d_all count x m (host, row per instance); `nctx` loaded worker contexts (clones of one
 * analysed QP), one host thread each, take instances in turn. v_out / scal_out as above. */
int cmpc_solve_batch_affine(cmpc_ctx** ctxs, int nctx, int64_t count, const double* h_all,
                            const double* h0_all, const double* d_all, const double* opts,
                            int64_t max_iter, double* v_out, double* scal_out);
/* Lockstep batch (config 5, refresh_initial_state semantics): `count` instances sharing the
 * loaded H and J of `base` (kept alive by the caller) and differing in (h, h0, d), solved by
 * ONE host loop whose kernels each cover every active instance (the reference solves them one
 * by one: proj/src/verify.cpp:104-111 over proj/src/ipm.cpp:160-268 per instance). n <= 160.
 * set_affine: h_all count x n, h0_all count, d_all count x m (host, row per instance).
 * solve: v_out count x n (nullable), scal_out count x 14 (cmpc_solve's out_scalars: status,
 * iterations, kkt, objective), stats (nullable) 10: batch iterations, device seconds, wall
 * seconds, kernel launches, host syncs, device rounds, the condensation kernel's device seconds,
 * its launches, the instances it covered (summed over launches), its algorithmic FLOPs per
 * instance (sum over the SYRK rows of hi (hi + 1)). */
typedef struct cmpc_batch cmpc_batch;
/* In-process loopback communicator (tests): `nranks` contexts on one device, each driven by
 * its own host thread, behave like the ranks of an NCCL communicator in the row-sharded solve
 * (every allreduce is reduced in rank order on the device). attach: as cmpc_ctx_attach_comm. */
int cmpc_loop_create(int nranks, int device, void** group);
void cmpc_loop_destroy(void* group);
int cmpc_ctx_attach_loop(cmpc_ctx* ctx, void* group, int rank, int64_t m_total);
int cmpc_batch_create(cmpc_ctx* base, int64_t count, cmpc_batch** out);
int cmpc_batch_set_affine(cmpc_batch* b, const double* h_all, const double* h0_all, const double* d_all);
int cmpc_batch_solve(cmpc_batch* b, const double* opts, int64_t max_iter, double* v_out, double* scal_out,
                     double* stats);
/* The batch's condensation step alone (assemble_condensed + the right-hand side's J'w,
 * proj/src/ipm.cpp:72-103, for every instance): sigma_all, w_all count x m (host); M_out
 * count x n x n (lower triangle of H + J' diag(sigma_b) J, column-major), tq_out count x n
 * (J' w_b). Leaves the batch's iterates untouched. */
int cmpc_batch_condense(cmpc_batch* b, const double* sigma_all, const double* w_all, double* M_out,
                        double* tq_out);
void cmpc_batch_destroy(cmpc_batch* b);
/* Page-lock / release a host buffer (cudaHostRegister) used for repeated uploads */
int cmpc_host_register(void* p, int64_t bytes);
int cmpc_host_unregister(void* p);
/* out[8] = n, m, prototypes, SYRK prototypes, singleton prototypes, SYRK work units,
 * algorithmic SYRK flops per condensation (sum over prototypes of hi (hi + 1)),
 * algorithmic bytes of one pass over P (8 x nonzeros) */
int cmpc_qp_info(cmpc_ctx* ctx, int64_t* out);
/* out[4] = Markov table in use (1: the prototypes of a built QP are read from the table of
 * B-responses, P is never stored), its rows, its columns, bytes of the stored prototype
 * source (the table, or P) */
int cmpc_qp_layout(cmpc_ctx* ctx, int64_t* out);
/* Diagnostics: run the condensation once and record a per-CTA timeline; out (cap x 4):
 * {start us, end us, SM id, planned weighted k-steps}; *nctas = CTAs of the launch */
int cmpc_debug_syrk_timeline(cmpc_ctx* ctx, double* out, int64_t cap, int64_t* nctas);
/* Replace h, h0, d of a loaded QP (refresh_initial_state, proj/src/reduction.cpp:270-280) */
int cmpc_update_qp_affine(cmpc_ctx* ctx, const double* h, double h0, const double* d, int on_device);

/* IpmState (proj/include/condmpc/ipm.hpp:18-25); host pointers, any may be NULL on get */
int cmpc_set_state(cmpc_ctx* ctx, const double* v, const double* s, const double* lambda,
                   const double* z, double mu);
int cmpc_get_state(cmpc_ctx* ctx, double* v, double* s, double* lambda, double* z);

/* compute_residuals (ipm.cpp:46-70): r1 (n), r2, r3 (m), kkt error; outputs nullable */
int cmpc_compute_residuals(cmpc_ctx* ctx, double* r1, double* r2, double* r3, double* kkt);
int cmpc_set_residuals(cmpc_ctx* ctx, const double* r1, const double* r2, const double* r3);
/* assemble_condensed (ipm.cpp:72-77): M = H + J' diag(sigma) J (full symmetric, n x n).
 * sigma NULL = z./s of the current state. M may be NULL (keeps it on the device). */
int cmpc_assemble_condensed(cmpc_ctx* ctx, const double* sigma, double* M);
/* factorize the device M + delta I (ReferenceBackend::factorize, dense_linalg.cpp:59-77);
 * returns CMPC_NOT_PD with *pivot = first failing pivot (0-based) */
int cmpc_factorize_condensed(cmpc_ctx* ctx, double delta, int64_t* pivot);
int cmpc_get_factor(cmpc_ctx* ctx, double* L);
int cmpc_set_factor(cmpc_ctx* ctx, const double* L);
/* step_directions (ipm.cpp:79-103) with the current factor, then fraction_to_boundary
 * (ipm.cpp:105-116): alpha[2] = {alpha_max, alpha_z}. Outputs nullable. */
int cmpc_step_directions(cmpc_ctx* ctx, double tau, double* pv, double* ps, double* plambda,
                         double* pz, double* alpha);
int cmpc_set_directions(cmpc_ctx* ctx, const double* pv, const double* ps, const double* plambda,
                        const double* pz);
/* line_search (ipm.cpp:118-144) on the current directions; *trial = accepted j or -1 */
int cmpc_line_search(cmpc_ctx* ctx, double alpha_max, double armijo_eta, double* alpha, int* trial);
/* merit (ipm.cpp:25-32) at (v + alpha pv, s + alpha ps) */
int cmpc_merit(cmpc_ctx* ctx, double alpha, double rho, double* phi);
/* v, s, lambda += alpha p; z += alpha_z pz (ipm.cpp:240-243) */
int cmpc_apply_step(cmpc_ctx* ctx, double alpha, double alpha_z);
int cmpc_dense_objective(cmpc_ctx* ctx, double* obj);

/* ipm::solve (ipm.cpp:160-268) on the loaded QP.
 * opts[5] = tol, mu_init, kappa_mu, tau, armijo_eta.
 * out_scalars[14] = status (0 converged, 1 max_iter, 2 factorization_failure,
 *   3 line_search_failure), iter, kkt_error, objective, total_seconds, linalg_seconds,
 *   device_seconds, launches, syncs, trials, condensation (SYRK + reduce) seconds, Cholesky
 *   seconds, condensations, SYRK kernel seconds; the per-phase times are CUDA events on the
 *   solve's stream.
 * log(user, rec[8]) per accepted step: iter, mu, alpha, alpha_z, kkt_error, objective,
 *   delta, trial (IterationRecord, ipm.hpp:41-49, plus the shift and trial index).
 * inspect(...) per iteration before the line search (IterationInspection, ipm.hpp:53-58);
 *   pointers valid only during the callback. */
typedef void (*cmpc_log_fn)(void* user, const double* rec);
typedef void (*cmpc_inspect_fn)(void* user, const double* v, const double* s, const double* lambda,
                                const double* z, double mu, const double* r1, const double* r2,
                                const double* r3, double kkt, const double* pv, const double* ps,
                                const double* plambda, const double* pz, double delta);
int cmpc_solve(cmpc_ctx* ctx, const double* opts, int64_t max_iter, double* v, double* s,
               double* lambda, double* z, double* out_scalars, cmpc_log_fn log,
               cmpc_inspect_fn inspect, void* user);

/* Row-sharded solve, one process per GPU: each rank loads its own rows of
 * J and d (cmpc_load_qp with m = its row count) and the full H, h, h0; rank 0 creates the
 * NCCL unique id (128 bytes) and the host broadcasts it; every rank attaches with the total
 * row count. cmpc_solve then runs the same host loop on every rank: the per-row partial
 * sums (J_g' Sigma_g J_g, J_g' y_g, residual/merit sums and maxima, step-length minima) are
 * allreduced over NVLink on the solve's stream and the Cholesky + solve run redundantly on
 * the identical condensed matrix, so every rank takes identical decisions and returns the
 * same v (its own rows of s, lambda, z). Needs libnccl.so.2 at run time (dlopen). */
int cmpc_comm_unique_id(void* id128);
int cmpc_ctx_attach_comm(cmpc_ctx* ctx, const void* id128, int nranks, int rank, int64_t m_total);
int cmpc_ctx_detach_comm(cmpc_ctx* ctx);

/* Device time of one phase of the iteration on the current device state, averaged over
 * reps back-to-back launches (CUDA events): 0 sigma+condense, 1 condense, 2 Cholesky,
 * 3 triangular solves, 4 residuals, 5 step recovery, 6 line-search trial, 7 J x, 8 J' y,
 * 9 sigma/omega/rhs preparation, 10 Cholesky fused with both triangular solves. */
int cmpc_time_phase(cmpc_ctx* ctx, int what, int reps, double* ms_per_rep);

/* Stand-alone dense linear algebra (the reference's linalg plug point,
 * proj/include/condmpc/dense_linalg.hpp:37-59), host buffers in and out. */
int cmpc_gram_weighted(int device, int64_t m, int64_t n, const double* J, const double* sigma,
                       double* G);
int cmpc_cholesky(int device, int64_t n, const double* M, double* L, int64_t* pivot);
int cmpc_cholesky_solve(int device, int64_t n, const double* L, const double* b, double* x);
/* fraction_to_boundary (ipm.cpp:105-116) on host vectors: out[2] = {alpha, alpha_z} */
int cmpc_fraction_to_boundary(int device, int64_t m, const double* s, const double* ps,
                              const double* z, const double* pz, double tau, double* out);

#ifdef __cplusplus
}
#endif

#endif /* CONDMPC_CUDA_H */
