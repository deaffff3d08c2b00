// Internal (C++) interfaces shared by the translation units of libgvp_b200.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/gvp_b200.h"
#include "gvp_block.cuh"

namespace gvp {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);
#define GVP_CUDA(call)                                         \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::gvp::cuda_fail(_e, #call); \
  } while (0)

// ------------------------------------------------------------------ SDF field
// Signed-distance grid resident in HBM in a "corner-packed" layout: cell
// (iz, iy, ix) stores its 4 (2D) or 8 (3D) corner values contiguously, so the
// bi/trilinear gather of one sigma point is a single 32 B / 64 B sector
// fetch instead of 4 / 8 scattered loads. Values are the reference's grid
// values bit for bit (sdf.py:23-56 layout: (ny, nx) / (nz, ny, nx), x
// fastest).
struct FieldDev {
  int ndim;
  int64_t nx, ny, nz;
  double ox, oy, oz, cell, inv_cell;
  const double* corners;  // device
  // map bank: plan b reads map plan_map[b] at corners + plan_map[b] * map_stride
  const int* plan_map;    // device, nullptr = one map for every plan
  int64_t map_stride;     // doubles per packed map
  // Lipschitz bound of the interpolated field (max |grid difference| / cell per
  // axis, combined in 2-norm; INFINITY = unknown): the fused factor kernel
  // skips the per-point gathers of a factor whose whole sigma-point cloud is
  // provably clear of every obstacle
  double lip;
};
// corner-pack raw grids on the device (nmaps maps of the geometry in f) into dst
int pack_field_maps(const FieldDev& f, int nmaps, const double* raw_dev, double* dst_dev, cudaStream_t s);
int64_t packed_field_doubles(const FieldDev& f);
// Lipschitz constant of the multilinear interpolant of nmaps row-major grids
// (nz, ny, nx) with spacing cell (the clear-cloud shortcut of the factor
// kernel); INFINITY if any node is non-finite
double field_lipschitz(const double* grids, int64_t nmaps, int ndim, int64_t nx, int64_t ny, int64_t nz,
                       double cell);
// rasterize primitive unions on the device (sdf.py:134-185): per map m the
// primitives [prim_off[m], prim_off[m+1]) of kinds (0 disc/sphere, 1 box) with
// params [center(dim) | radius or halfextents(dim)] (2*dim doubles each);
// raw row-major grids (nz, ny, nx) out
int rasterize_maps(int dim, const int64_t* counts, const double* origin, double cell, int nmaps,
                   const int* prim_off_dev, const int* kinds_dev, const double* params_dev, double* raw_dev,
                   cudaStream_t s);

struct Field {
  FieldDev dev{};
  double* d_corners = nullptr;
  int64_t bytes = 0;
  ~Field();
  int build(const double* grid_host, int ndim, const int64_t* shape, const double* origin,
            double cell, cudaStream_t s);
};

// ------------------------------------------------------------------ rule
// Quadrature rule plus its position-projection tables (DESIGN.md §kernel a):
// the hinge potential reads only x[:P] = mu[:P] + L[:P,:P] xi[:P] (L lower
// triangular), so sigma points sharing xi[:P] share psi. Per distinct
// projection j: coords xi_j[:P], point count, and the moments
// m0_j = sum w_l, m1_j = sum w_l xi_l (n), m2_j = sum w_l xi_l xi_l^T (packed).
struct RuleDev {
  int n, P;
  int64_t npts, nproj;
  const double* points;   // (npts, n)   exact-contract kernel
  const double* weights;  // (npts)
  const double* proj;     // (nproj, P)
  const double* mom;      // (nproj, 1 + n + n(n+1)/2)
  const int* cnt;         // (nproj)
  const void* host;       // the owning host Rule (projection tables for by-value launch)
  double proj_radius;     // max_j |proj_j| (2-norm): the sigma cloud lies within |L[:P,:P]|_F * this
};

struct Rule {
  RuleDev dev{};
  double* d_buf = nullptr;
  int* d_cnt = nullptr;
  // host copies of the projection tables (passed by value to the fused kernel)
  std::vector<double> h_proj, h_mom;
  std::vector<int> h_cnt;
  ~Rule();
  int build(const double* points, const double* weights, int64_t npts, int n, int P,
            cudaStream_t s);
};

// ------------------------------------------------------------------ launches
// factor kernels (factor_kernels.cu)
int launch_factor_moments(int64_t nfac, int n, const double* means, const double* chols,
                          const RuleDev& rule, const FieldDev& field, double radius_eps,
                          double sigma_obs, double* e0, double* e1, double* e2,
                          unsigned long long* oob, cudaStream_t s);

struct FactorOut {
  MutView e_psi;  // (F) per plan
  MutView g_mu;   // knot-indexed: entry for factor f at knot f+1 (view base at knot 0)
  MutView g_diag; // knot-indexed
  unsigned long long* oob;  // per plan
  int* status;              // per plan (0 ok, GVP_ERR_*)
  int* where;               // per plan (atomicMin'd factor index)
  // gaussian_sqrt's eigh fallback: [0] = count, then b * nfac + f of every factor
  // whose Cholesky (and jitter retry) failed, finished by the eigh fix-up kernel.
  // nullptr: report GVP_ERR_SQRT instead. Size 1 + nplans * nfac.
  int* eigh_list = nullptr;
  // bit 0: the factor kernel, bit 1: the eigh fix-up (callers that time the
  // factor kernel alone launch the two separately)
  int phases = 3;
  // zero eigh_list[0] before the factor kernel; the engine instead re-arms the
  // list itself once the fix-up has consumed it (outside the timed factor stage)
  bool reset_eigh = true;
};
int launch_factor_grads(int nplans, int64_t nknots, int n, const View& mean, const View& covs,
                        const RuleDev& rule, const FieldDev& field, double radius_eps,
                        double sigma_obs, const FactorOut& out, const int* active,
                        cudaStream_t s);

// chain kernels (chain_kernels.cu)
// GBP marginals by cyclic reduction (cr_kernels.cu): one CTA per plan, log-depth
int launch_cr_marginals(int nplans, int64_t K, int n, const View& D, const View& U, const MutView& cov,
                        const MutView& cross, double* ws, int* status, int* where, cudaStream_t s);
int64_t cr_workspace_doubles(int nplans, int64_t K, int n);
int launch_marginals(int nplans, int64_t K, int n, const View& diag, const View& off,
                     const MutView& covs, const MutView& crosses, double* logdet, int* status,
                     int* where, double* scratch, const int* active, cudaStream_t s);
int launch_mean_solve(int nplans, int64_t K, int n, const View& diag, const View& off,
                      const View& eta, const MutView& out, int* status, int* where,
                      double* scratch, cudaStream_t s);
// chols (nullable): the forward Schur pivots' Cholesky factors, (nplans, K, n, n) lower
int launch_logdet_fwd(int nplans, int64_t K, int n, const View& diag, const View& off,
                      double* out, int* status, int* where, double* chols, cudaStream_t s);

struct StepProblem {
  View mean, diag, off;      // current iterate
  View kdiag, koff, info;    // prior (kdiag/koff may be shared, sp = 0)
  View gmu, gdiag, goff;     // joint gradients (goff may be a zero view)
  bool has_goff;
  View pmean;                // prior mean (for the prior cost at commit)
  bool has_pmean;
};
struct StepOut {
  MutView mean, diag, off, covs, crosses;  // may alias the inputs (in-place commit)
  double* beta;        // per plan
  double* kl;          // per plan
  double* logdet_next; // per plan: log det of the accepted precision
  double* mean_shift;  // per plan: ||mu' - mu||
  double* prior_cost;  // per plan (optional): 1/2 d'K^{-1}d + 1/2 tr(K^{-1} Sigma') of the accepted state
  double* probe_log;   // optional (nplans, max_probes, 3)
  int max_probes;
  int* nprobes;        // optional per plan
  int* status;
  int* where;
};
struct StepParams {
  const double* temp;        // per plan
  const double* logdet_cur;  // per plan
  double kl_bound, beta_min, beta_max;
  int lanes;                 // speculative candidates per plan
  bool fixed_beta;           // proximal_update only (no bisection, no KL)
  const double* beta_fixed;  // per plan when fixed_beta
};
int launch_select_step(int nplans, int64_t K, int n, const StepProblem& pb, const StepParams& pr,
                       const StepOut& out, double* scratch, const int* active, cudaStream_t s);
int64_t chain_scratch_doubles(int nplans, int64_t K, int n, int lanes);

// ---- step kernel v2 (step_kernel.cu): plan-minor arrays with plan stride Bp,
// diagonal blocks packed lower-symmetric (n(n+1)/2 entries), off blocks full.
struct V2Launch {
  int nplans;
  int64_t K;
  int n;
  int64_t Bp;
  int lanes;
  bool fill;  // probes: spread the plans over every resident CTA slot (fewer plans per CTA, more lanes each)
  const double *ld, *lo, *kd, *ko, *gd, *g, *eta, *v, *mu, *pmean;
  bool kshared;
  double *o_mu, *o_ld, *o_lo, *o_cov, *o_cr, *o_v;
  double *beta, *kl, *ld_next, *shift, *prior_cost;
  const double* temp;
  const double* ld_cur;
  double kl_bound, beta_min, beta_max;
  int *status, *where;
  double* probe_log;
  int max_probes;
  int* nprobes;
  double* scratch;
  const int* active;
  // true: the search writes kl / ld_next (the accepted probe's KL and
  // forward-Schur log det); the commit overwrites them only where fixkl[b]
  bool search_kl;
  const int* fixkl;
  // recorded between the residual kernel and the probe kernel when set
  // (per-kernel timing, gvp_engine_step_profiled_ex); never inside a capture
  cudaEvent_t ev_residual_done;
};
// forward-Schur log det of packed precisions (plan-minor, stride Bp), the
// probes' own recursion: a bit-identical ld_cur for the next search. mask
// (nullable): only plans with mask[b] != 0.
int launch_logdet_fwd_packed(int nplans, int64_t K, int n, int64_t Bp, const double* ld, const double* lo,
                             double* logdet, const int* mask, int* status, int* where, cudaStream_t s);
// ---- wide blocks, 9 <= n <= 32 (wide_kernels.cu): one warp per chain, lanes over rows
struct WideStep {
  int nplans;
  int64_t K;
  int n;
  View mean, diag, off, kdiag, koff, info, gmu, gdiag, goff;  // full n x n blocks
  bool has_goff;
  MutView o_mean, o_diag, o_off, o_cov, o_cross;
  const int* active;
  int *status, *where, *nprobes;
  double *beta, *kl, *ld_next;  // beta: in = previous beta (NaN: none) / fixed beta, out = accepted
  const double *temp, *ld_cur;
  double kl_bound, beta_min, beta_max;
  double* probe_log;
  int max_probes;
  double* scratch;  // wide_scratch_doubles
  bool fixed;       // proximal_update only
};
int64_t wide_scratch_doubles(int nplans, int64_t K, int n);
int launch_wide_marginals(int nplans, int64_t K, int n, const View& D, const View& U, const MutView& cov,
                          const MutView& cross, double* logdet, double* scratch, int* status, int* where,
                          cudaStream_t s);
int launch_wide_mean_solve(int nplans, int64_t K, int n, const View& D, const View& U, const View& E,
                           const MutView& x, double* scratch, int* status, int* where, cudaStream_t s);
int launch_wide_logdet(int nplans, int64_t K, int n, const View& D, const View& U, double* logdet, double* chols,
                       int* status, int* where, cudaStream_t s);
int launch_wide_step(const WideStep& q, cudaStream_t s);
int launch_select_step_v2(const V2Launch& q, cudaStream_t s);
int launch_select_bisect(const V2Launch& q, cudaStream_t s);  // bisection only
int launch_select_commit(const V2Launch& q, cudaStream_t s);  // commit of q.beta
// even plan stride >= 2 required by the TMA-staged step kernel
int64_t step_plan_stride(int nplans);
int64_t step_scratch_doubles(int nplans, int64_t K, int n, int lanes);
// packed-layout helpers (step_kernel.cu)
int launch_marginals_packed(int nplans, int64_t K, int n, int64_t Bp, const double* ld,
                            const double* lo, double* cov, double* cr, double* logdet,
                            int* status, int* where, double* scratch, const int* active,
                            cudaStream_t s);
int launch_lam_mu(int nplans, int64_t K, int n, int64_t Bp, const double* ld, const double* lo,
                  const double* mu, double* v, cudaStream_t s);

}  // namespace gvp
