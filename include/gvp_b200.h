/*
 * gvp_b200 — C ABI of the B200-native P-GVIMP engine (libgvp_b200.so).
 *
 * Plain C: pointers, sizes, status codes. No torch or CUDA-runtime types
 * leak through the signatures except an opaque stream handle (void*) on the
 * *_dev entry points; 0 means the library's own stream.
 *
 * Two families of entry points:
 *
 *  1. Drop-in host entry points (gvp_factor_expectations, gvp_gbp_marginals,
 *     ...). Host pointers, blocking, one plan. Each one replaces one function
 *     of the reference package `gvplan` (/root/reference/pkg/src/gvplan) and
 *     keeps its argument meaning; the reference location is cited on each.
 *     Block-tridiagonal matrices are passed stacked: diag (nblocks, n, n),
 *     off (nblocks-1, n, n), C order — the reference's lists of blocks
 *     (blocktri.py:48-66) stacked with np.stack.
 *
 *  2. The batched engine (gvp_engine_*): B independent plans resident in HBM,
 *     the whole Algorithm-1 loop (optimizer.py:299-401) on device. Batched
 *     arrays are "plan-minor": element e of knot i of plan b is at
 *     [(i * E + e) * B + b] (E = n*n for blocks, n for vectors), so a warp of
 *     consecutive plans reads 256 contiguous bytes per element. For B = 1
 *     this is exactly the stacked layout of family 1.
 *
 * Status codes map to the reference's exceptions.
 */
#ifndef GVP_B200_H
#define GVP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define GVP_OK 0
#define GVP_ERR_NOT_SPD 1          /* NotPositiveDefiniteError (blocktri.py:20); where = knot */
#define GVP_ERR_NONFINITE 2        /* FactorEvaluationError (factors.py:34-37); where = factor index */
#define GVP_ERR_NO_FEASIBLE_STEP 3 /* RuntimeError "no feasible step size" (optimizer.py:217-221) */
#define GVP_ERR_SQRT 4             /* gaussian_sqrt's eigh root (quadrature.py:178-181) has a clipped
                                      eigenvalue: singular, numpy.linalg.LinAlgError in _moment_gradients */
#define GVP_ERR_ARG -1             /* bad argument (ValueError) */
#define GVP_ERR_UNSUPPORTED -2     /* block size n outside the supported range, or grid ndim not 2/3 */
#define GVP_ERR_CUDA -3            /* CUDA runtime failure; see gvp_last_error() */
#define GVP_ERR_NO_DEVICE -4       /* no CUDA device visible */

/* "where" sub-codes for GVP_ERR_NOT_SPD raised by the step machinery */
#define GVP_WHERE_MEAN_SOLVE_BIAS (1 << 30) /* pivot failed in the proximal mean solve */

/* Human-readable description of the last error on this thread. */
const char* gvp_last_error(void);
/* Library version string. */
const char* gvp_version(void);
/* Number of visible CUDA devices (0 if none); never fails. */
int gvp_device_count(void);

/* ------------------------------------------------- 1. drop-in host entry points */

/* Hinge-collision quadrature moments of every factor.
 * Replaces gvplan._kernels.factor_expectations (_kernels.pyx:132-177; numpy
 * twin _kernels_py.py:16-53). means (nfac, n), chols (nfac, n, n) (any square
 * root; the full n x n product L xi is formed like _kernels.pyx:107-112),
 * points (npts, n), weights (npts), grid of shape grid_shape[0..grid_ndim-1]
 * = (ny, nx) or (nz, ny, nx), x fastest. pos_dim is accepted and, like the
 * compiled reference kernel, the grid's ndim decides the position dims.
 * Outputs e0 (nfac), e1 (nfac, n), e2 (nfac, n, n), *oob = number of
 * border-clamped sigma points. */
int gvp_factor_expectations(const double* means, const double* chols, int64_t nfac, int32_t n,
                            const double* points, const double* weights, int64_t npts,
                            const double* grid, int32_t grid_ndim, const int64_t* grid_shape,
                            const double* origin, double cell_size, double radius_eps,
                            double sigma_obs, int32_t pos_dim, double* e0, double* e1,
                            double* e2, int64_t* oob);

/* Fused factor stage of one plan: per interior knot i = 1..nblocks-2, the
 * Cholesky root of covs[i] (with the 1e-10 jitter retry of
 * quadrature.py:164-177), the quadrature moments, and the moment-form
 * gradients of factors.py:95-104. Replaces the body of
 * gvplan.factors.evaluate_all_factors (factors.py:167-225) after the marginal
 * extraction. mean (nblocks, n), covs (nblocks, n, n). Outputs e_psi
 * (nblocks-2, clamped at 0 like factors.py:218-224), g_mu (nblocks-2, n),
 * g_sigma (nblocks-2, n, n), *oob. On GVP_ERR_NONFINITE *where is the
 * factor_index (= knot) of the first bad factor. */
int gvp_evaluate_factors(const double* mean, const double* covs, int64_t nblocks, int32_t n,
                         const double* points, const double* weights, int64_t npts,
                         const double* grid, int32_t grid_ndim, const int64_t* grid_shape,
                         const double* origin, double cell_size, double radius_eps,
                         double sigma_obs, double* e_psi, double* g_mu, double* g_sigma,
                         int64_t* oob, int64_t* where);

/* The block-chain drop-ins below (marginals, mean solve, log det, forward
 * Schur chols, proximal update, select_step_size) take 1 <= n <= 32: n <= 8
 * on the register-block kernels, 9 <= n <= 32 (e.g. the 7-DOF arm's n = 14)
 * on the warp-per-chain kernels of csrc/wide_kernels.cu. */

/* Marginal covariance blocks of an SPD block-tridiagonal precision by exact
 * chain GBP. Replaces gvplan.gbp.gbp_marginals (gbp.py:43-80). covs (nblocks,
 * n, n), crosses (nblocks-1, n, n). GVP_ERR_NOT_SPD: *where = knot whose
 * belief precision failed. */
int gvp_gbp_marginals(const double* diag, const double* off, int64_t nblocks, int32_t n,
                      double* covs, double* crosses, int64_t* where);

/* Solve Lambda mu = eta. Replaces gvplan.gbp.gbp_mean_solve (gbp.py:83-106).
 * GVP_ERR_NOT_SPD: *where = pivot block. */
int gvp_gbp_mean_solve(const double* diag, const double* off, const double* info,
                       int64_t nblocks, int32_t n, double* out, int64_t* where);

/* log det by forward Schur pivots. Replaces
 * gvplan.blocktri.logdet_block_tridiag (blocktri.py:151-174). */
int gvp_logdet_block_tridiag(const double* diag, const double* off, int64_t nblocks, int32_t n,
                             double* out, int64_t* where);
/* forward_schur_chols (blocktri.py:151-165): Cholesky factors (K, n, n, lower)
 * of the forward Schur pivots; GVP_ERR_NOT_SPD with *where = pivot block. */
int gvp_forward_schur_chols(const double* diag, const double* off, int64_t nblocks, int32_t n, double* chols,
                            int64_t* where);

/* One closed-form KL-proximal step. Replaces gvplan.optimizer.proximal_update
 * (optimizer.py:129-161). cur (mean, diag, off), prior (kdiag, koff, info),
 * gradients (g_mu, gdiag, goff). Outputs the next mean/diag/off (precision
 * symmetrised, not SPD-checked). GVP_ERR_NOT_SPD from the mean solve:
 * *where = pivot block. */
int gvp_proximal_update(const double* mean, const double* diag, const double* off,
                        const double* kdiag, const double* koff, const double* info,
                        const double* g_mu, const double* gdiag, const double* goff,
                        int64_t nblocks, int32_t n, double beta, double temp,
                        double* out_mean, double* out_diag, double* out_off, int64_t* where);

/* Largest feasible beta by bisection, whole search on device. Replaces
 * gvplan.optimizer.select_step_size (optimizer.py:188-231) including its
 * probe (proximal_update + gbp_marginals + kl_joint). Outputs beta, kl and
 * the accepted state with its marginals. probe_log (optional, may be NULL):
 * up to max_probes rows of (beta, feasible, kl); *nprobes = rows written. */
int gvp_select_step_size(const double* mean, const double* diag, const double* off,
                         const double* kdiag, const double* koff, const double* info,
                         const double* g_mu, const double* gdiag, const double* goff,
                         int64_t nblocks, int32_t n, double temp, double kl_bound,
                         double beta_min, double beta_max, double* beta, double* kl,
                         double* out_mean, double* out_diag, double* out_off, double* covs,
                         double* crosses, double* probe_log, int32_t max_probes,
                         int32_t* nprobes, int64_t* where);

/* The same, given the log det of the current precision (ld_cur; NaN: computed
 * here, as gvp_select_step_size does) and returning the accepted state's log
 * det (*ld_next; NaN where the path does not produce it): a host loop carries
 * one iteration's into the next (kl_joint's logdet_cur, entropy_of) instead of
 * two extra log det sweeps per iteration. */
int gvp_select_step_size_ld(const double* mean, const double* diag, const double* off,
                            const double* kdiag, const double* koff, const double* info,
                            const double* g_mu, const double* gdiag, const double* goff,
                            int64_t nblocks, int32_t n, double temp, double kl_bound,
                            double beta_min, double beta_max, double* beta, double* kl,
                            double* out_mean, double* out_diag, double* out_off, double* covs,
                            double* crosses, double* probe_log, int32_t max_probes,
                            int32_t* nprobes, int64_t* where, double ld_cur, double* ld_next);

/* Candidate lanes (1, 2, 4, 8, 16) gvp_select_step_size probes concurrently;
 * the beta sequence is the reference's for any value (default 16). */
int gvp_set_step_lanes(int32_t lanes);

/* -------------------------------------------------------- 2. batched engine */

typedef struct gvp_plan_config {
  double kl_bound;       /* OptimizerConfig (optimizer.py:72-87) */
  double beta_min;
  double beta_max;
  double temp_low;
  double temp_high;
  double collision_tol;  /* < 0 -> 1e-4 * N (optimizer.py:316-318) */
  double tol_mean;
  double tol_cost;
  double init_cov_scale;
  int32_t max_iters;
  int32_t spec_lanes;    /* candidate betas probed concurrently per plan: 0 = auto, else 1/2/4/8/16 */
} gvp_plan_config;

typedef struct gvp_engine gvp_engine;

/* nplans independent plans of nknots = N+1 knots, state size n, sharing one
 * SDF (grid values on host, copied once) and one quadrature rule. If
 * shared_prior != 0 every plan uses the same prior precision (one copy,
 * L2-resident); info and prior mean stay per plan. */
int gvp_engine_create(gvp_engine** out, int32_t nplans, int64_t nknots, int32_t n,
                      int32_t shared_prior, const double* grid, int32_t grid_ndim,
                      const int64_t* grid_shape, const double* origin, double cell_size,
                      double radius_eps, double sigma_obs, const double* points,
                      const double* weights, int64_t npts, const gvp_plan_config* cfg);
void gvp_engine_destroy(gvp_engine* e);

/* Upload the problem (host pointers, plan-minor layout): prior precision
 * kdiag/koff (one plan's blocks if shared_prior), info and prior mean
 * (nknots, n, nplans), initial joint mean (nknots, n, nplans). Resets all
 * per-plan state (initial_state, optimizer.py:280-296). */
int gvp_engine_load(gvp_engine* e, const double* kdiag, const double* koff, const double* info,
                    const double* prior_mean, const double* init_mean);
/* Same, from device pointers (no host traffic). */
int gvp_engine_load_dev(gvp_engine* e, const double* kdiag, const double* koff,
                        const double* info, const double* prior_mean, const double* init_mean);
/* A shared-prior batch by its boundary states (optimizer.batch_problem's
 * affine construction, expanded on the device): kdiag/koff as above, plan 0's
 * info and prior mean (nknots, n), the anchored-mean responses to unit start /
 * goal offsets resp0/respg (n, nknots, n), the anchor block (n, n), and every
 * plan's start and goal (nplans, n). Initial mean: initial_mean's straight
 * line (OptimizerConfig.init default). */
int gvp_engine_load_boundary(gvp_engine* e, const double* kdiag, const double* koff, const double* base_info,
                             const double* base_mean, const double* resp0, const double* respg,
                             const double* anchor, const double* x0s, const double* goals);

/* Run up to `iters` more iterations of Algorithm 1 for every active plan
 * (asynchronous on the engine stream unless sync != 0). */
int gvp_engine_step(gvp_engine* e, int32_t iters, int32_t sync);
/* Same as gvp_engine_step but kernel by kernel with CUDA events on the
 * engine stream; the device time of each stage summed over the iterations
 * goes to ms[0..3] = {bisection (residual + probes), commit, factor kernel,
 * eigh fix-up + control} (synchronous). */
int gvp_engine_step_profiled(gvp_engine* e, int32_t iters, double* ms);
/* Same with one bucket per kernel: ms[0..nms) of {residual, probes, commit,
 * factor kernel, eigh fix-up, control}. */
int gvp_engine_step_profiled_ex(gvp_engine* e, int32_t iters, double* ms, int32_t nms);
/* The engine's cudaStream_t (as void*), for events/interop. */
void* gvp_engine_stream(gvp_engine* e);
/* Block until the engine stream is idle. */
int gvp_engine_sync(gvp_engine* e);
/* Number of plans still active (not converged, not failed, below max_iters). */
int gvp_engine_active(gvp_engine* e, int32_t* nactive);

/* Copy results to host (plan-minor layouts):
 * mean (nknots, n, B); diag (nknots, n, n, B); off (nknots-1, n, n, B);
 * covs like diag; crosses like off; any pointer may be NULL. */
int gvp_engine_get_state(gvp_engine* e, double* mean, double* diag, double* off, double* covs,
                         double* crosses);
/* The same results without the host-side unpacking, straight into caller
 * (ideally pinned) buffers: mean (nknots, n, nplans) and the marginal
 * covariances packed lower-symmetric (nknots, n(n+1)/2, nplans), entry
 * r(r+1)/2 + c holding Sigma_ii[r][c], c <= r. Either pointer may be NULL. */
int gvp_engine_get_packed(gvp_engine* e, double* mean, double* covs_packed);
/* Per-plan summary: converged, iterations, switch_iteration (-1 = none),
 * status, where (each int32[B]). */
int gvp_engine_get_summary(gvp_engine* e, int32_t* converged, int32_t* iterations,
                           int32_t* switch_iteration, int32_t* status, int32_t* where);
/* Per-iteration records (max_iters, B, GVP_NREC): beta, temperature,
 * prior_cost, collision_cost, entropy_cost, total_cost, kl_step, mean_shift
 * (optimizer.py:366-379); rows past a plan's last iteration are NaN. */
#define GVP_NREC 8
int gvp_engine_get_records(gvp_engine* e, double* records);
/* Candidate lanes per plan the engine runs with (after auto selection). */
int32_t gvp_engine_lanes(gvp_engine* e);
/* Device pointers of the resident state, for zero-copy consumers. Layout:
 * plan-minor; diag and covs are packed lower-symmetric, (nknots, n(n+1)/2, B). */
int gvp_engine_device_state(gvp_engine* e, double** mean, double** diag, double** off,
                            double** covs, double** crosses);
/* Launch counters: kernels launched by this engine since create. */
int64_t gvp_engine_launches(gvp_engine* e);
/* Map bank: nmaps signed-distance maps with the engine's grid
 * geometry, plan b reading map plan_map[b] (nreal entries). set: host grids
 * (nmaps x row-major (ny,nx) / (nz,ny,nx)); raster: rasterised on the device
 * from primitive lists like rasterize (sdf.py:156-185) — map m owns primitives
 * [prim_off[m], prim_off[m+1]), kind 0 disc/sphere (center, radius, pad) or
 * 1 box (center, halfextents), 2*dim doubles each. Call before stepping. */
int gvp_engine_set_map_bank(gvp_engine* e, int32_t nmaps, const double* grids, const int32_t* plan_map);
int gvp_engine_raster_map_bank(gvp_engine* e, int32_t nmaps, const int32_t* prim_off, const int32_t* kinds,
                               const double* params, const int32_t* plan_map);
/* Drop-in rasterize (sdf.py:156-185), bit-identical values: counts per axis
 * (x, y[, z]) as the reference derives them from bounds, out row-major
 * (ny, nx) or (nz, ny, nx) in host memory. */
int gvp_rasterize(int32_t dim, const int64_t* counts, const double* origin, double cell_size, int32_t nprim,
                  const int32_t* kinds, const double* params, double* out);
/* Probe trace of the step-size search (optimizer.py:188-231 `trace`): per
 * plan the last iteration's probes as (beta, spd, kl) rows, at most
 * max_probes each. Enable before the first step. */
int gvp_engine_trace_probes(gvp_engine* e, int32_t max_probes);
int gvp_engine_get_probes(gvp_engine* e, double* log, int32_t* counts);
/* One iteration (synchronous) in which every plan with a finite beta[b]
 * (host, nplans entries; NaN = searched) takes that step size instead of the
 * searched one: proximal_update at a given beta (optimizer.py:129-161) inside
 * the engine. The search still runs and is traced, so a known step sequence
 * (e.g. the reference's) can be replayed while each search is compared. */
int gvp_engine_step_beta(gvp_engine* e, const double* beta);
/* Replace the iterate (mean, precision) of nsel selected plans and redo what
 * an iteration leaves for the next one (marginals, log det, Lambda mu, factor
 * stage); records and iteration counts are kept. Host, batch-major over the
 * selected plans: mean (nsel, nknots, n), diag (nsel, nknots, n, n), off
 * (nsel, nknots-1, n, n). E.g. restart from another implementation's state. */
int gvp_engine_set_state(gvp_engine* e, int32_t nsel, const int32_t* plans, const double* mean,
                         const double* diag, const double* off);
/* Per-plan count (int64[nplans]) of sigma points clamped at the SDF border
 * over every factor stage so far (sdf.py:53-56 note_oob). */
int gvp_engine_get_oob(gvp_engine* e, int64_t* oob);

/* ------------------------------------------------ iP-GVIMP on the device */
/* Statistical linearisation of the planar quadrotor (slr.py:69-92) for B
 * nominal trajectories: host arrays means (B,K,6), covs (B,K,6,6), rule points
 * (Q,6) / weights (Q), params = {1/mass, length/inertia, gravity}. Out: the
 * LTV triples A (B,K,6,6), a (B,K,6) (B_i is the constant input matrix).
 * status/where per plan: GVP_ERR_SQRT (covariance needs gaussian_sqrt's eigh
 * root), GVP_ERR_NONFINITE (euler_step non-finite), GVP_ERR_NOT_SPD (P_xx). */
int gvp_slr_quadrotor(int32_t nplans, int32_t K, const double* means, const double* covs, const double* points,
                      const double* weights, int32_t Q, double dt, const double* params, double* A, double* a,
                      int32_t* status, int32_t* where);
/* Anchored LTV prior assembly (prior.py:56-170, transition_kernel + grammian +
 * assemble_prior) for B plans of S steps, n = 6: A (B,S,6,6), a (B,S,6),
 * B (B,S,6,m), Gauss-Legendre nodes/weights on [-1,1]. Out: Phi (B,S,6,6),
 * offsets (B,S,6), Grammians (B,S,6,6), precision diag (B,S+1,6,6) / off
 * (B,S,6,6) and information (B,S+1,6). The anchored mean is gvp_gbp_mean_solve. */
int gvp_prior_assemble(int32_t nplans, int32_t S, int32_t n, int32_t m, const double* A, const double* a,
                       const double* B, double dt, double q_c, double sigma_b, const double* x0, const double* goal,
                       const double* gl_nodes, const double* gl_weights, int32_t nodes, double* phis, double* offs,
                       double* grams, double* diag, double* off, double* info, int32_t* status, int32_t* where);
/* The same with the robust-conditioning mode (NOT the reference's arithmetic):
 * every Grammian regularised to Q + grammian_reg tr(Q)/n I before its SPD
 * check and inverse (grammian_reg = 0: gvp_prior_assemble). */
int gvp_prior_assemble_reg(int32_t nplans, int32_t S, int32_t n, int32_t m, const double* A, const double* a,
                           const double* B, double dt, double q_c, double sigma_b, const double* x0,
                           const double* goal, const double* gl_nodes, const double* gl_weights, int32_t nodes,
                           double grammian_reg, double* phis, double* offs, double* grams, double* diag,
                           double* off, double* info, int32_t* status, int32_t* where);

/* ------------------------------------------------ 7-DOF sphere arm */
/* Factor moments (the factor_expectations contract, _kernels.pyx:132-177) for
 * a 7-joint standard-DH arm covered by spheres: psi(q) = sigma sum_s
 * max(r_s + eps - d(FK_s(q)), 0)^2, q = x[:7], n = 14. Host arrays: means
 * (F,14), chols (F,14,14) lower; the rule's joint-space projection tables proj
 * (NP,7), mom (NP,120) = [m0 | m1 (14) | m2 packed (105)], cnt (NP); 3D grid
 * (nz,ny,nx), origin (x,y,z), cell; dh (7,4) = (a, d, alpha, theta offset),
 * base (3); spheres: link (S, 0..7), geom (S,4) = (local xyz, radius).
 * Out: e0 (F), e1 (F,14), e2 (F,14,14), oob (sphere centres outside). */
int gvp_arm_factor_expectations(int64_t nfac, const double* means, const double* chols, int32_t nproj,
                                const double* proj, const double* mom, const int32_t* cnt, const double* grid,
                                const int64_t* shape, const double* origin, double cell, const double* dh,
                                const double* base, int32_t nspheres, const int32_t* sphere_link,
                                const double* sphere_geom, double radius_eps, double sigma_obs, double* e0,
                                double* e1, double* e2, int64_t* oob);

/* Device-resident arm collision model for the planner loop (the factor stage
 * of evaluate_all_factors, factors.py:167-225, for the arm): created once
 * with the grid, arm and the rule's projection tables (as above), then per
 * call: covariances -> gaussian_sqrt (quadrature.py:164-181, GVP_ERR_SQRT if
 * the eigh root would be needed) -> moments -> _moment_gradients
 * (factors.py:95-104). means (F,14), covs (F,14,14); out e_psi (F) =
 * max(e0, 0), g_mu (F,14), g_sigma (F,14,14), oob. GVP_ERR_NONFINITE /
 * GVP_ERR_SQRT: *where = position of the factor in the call. */
typedef struct gvp_arm gvp_arm;
int gvp_arm_create(gvp_arm** out, const double* grid, const int64_t* shape, const double* origin, double cell,
                   const double* dh, const double* base, int32_t nspheres, const int32_t* sphere_link,
                   const double* sphere_geom, double radius_eps, double sigma_obs, int32_t nproj,
                   const double* proj, const double* mom, const int32_t* cnt);
void gvp_arm_destroy(gvp_arm* h);
int gvp_arm_factor_grads(gvp_arm* h, int64_t nfac, const double* means, const double* covs, double* e_psi,
                         double* g_mu, double* g_sigma, int64_t* oob, int64_t* where);

/* ------------------------------------------------ batched device kernels (tests) */
/* All pointers device memory, plan-minor layout with nplans plans, async on
 * `stream` (a cudaStream_t; NULL = legacy default stream). */
int gvp_gbp_marginals_dev(int32_t nplans, int64_t nblocks, int32_t n, const double* diag,
                          const double* off, double* covs, double* crosses, double* logdet,
                          int32_t* status, int32_t* where, double* scratch, void* stream);
/* scratch size in doubles for gvp_gbp_marginals_dev / gvp_select_step_dev */
int64_t gvp_chain_scratch_doubles(int32_t nplans, int64_t nblocks, int32_t n, int32_t lanes);

#ifdef __cplusplus
}
#endif
#endif /* GVP_B200_H */
