// Batched P-GVIMP engine: Algorithm 1 (optimizer.py:299-401) for B
// independent plans, all state resident in HBM, no host round trip inside an
// iteration. One iteration = 3 kernels on the engine stream:
//
//   select_step_v2_kernel  bisection (speculative lanes) + in-place commit of
//                          (mu, Lambda), the accepted marginals, KL, log det,
//                          prior cost and Lambda mu for the next rhs
//   factor_grads_kernel    collision factors at the accepted state (the cache
//                          the next iteration's step uses, optimizer.py:354-360)
//   control_kernel         cost_breakdown (optimizer.py:238-277), the record,
//                          convergence and temperature switch (optimizer.py:381-398)
//
// The iteration is captured once into a CUDA graph and replayed.
//
// Device layout: plan-minor with plan stride B; diagonal blocks (precision,
// prior precision, covariances, collision Hessian terms) packed lower
// symmetric, n(n+1)/2 entries; off-diagonal blocks full n x n.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "gvp_internal.cuh"

using namespace gvp;

namespace {
constexpr double kLog2Pi = 1.8378770664093453;  // log(2 pi), optimizer.py:38

struct PlanState {
  // logdet: forward-Schur log det of the current precision (the probes' ld_cur);
  // logdet_next: the accepted state's, written by the search (or the commit)
  double *temp, *logdet, *beta, *kl, *shift, *prior_cost, *prev_total, *prev_temp, *total, *logdet_next;
  int *active, *status, *where, *converged, *iters, *switch_it, *switched, *fstatus, *fwhere;
  int* fixkl;  // gvp_engine_step_beta: the pinned beta was not probed (commit supplies KL / log det)
  unsigned long long* oob;
  int* nactive;
};

__global__ void init_plans_kernel(int B, PlanState ps, double temp_low) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ps.temp[b] = temp_low;
  ps.beta[b] = NAN;        // no previous step: no speculation target in the first search
  ps.prev_total[b] = NAN;  // NaN encodes python None
  ps.prev_temp[b] = NAN;
  ps.active[b] = 1;
  ps.status[b] = 0;
  ps.where[b] = -1;
  ps.converged[b] = 0;
  ps.iters[b] = 0;
  ps.switch_it[b] = -1;
  ps.switched[b] = 0;
  ps.fstatus[b] = 0;
  ps.fwhere[b] = INT_MAX;
  ps.oob[b] = 0;
  ps.fixkl[b] = 0;
  ps.logdet_next[b] = NAN;
}

// full (K, n, n, sw) -> packed (K, T, dw) times `scale`; a shared prior
// (sw = 1) is written to both columns of its 2-wide copy (dw = 2)
__global__ void pack_sym_kernel(int64_t K, int n, int64_t sw, int64_t dw,
                                const double* __restrict__ src, double* __restrict__ dst,
                                double scale) {
  const int T = n * (n + 1) / 2;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * T * dw) return;
  const int64_t b = t % dw, q = (t / dw) % T, i = t / (dw * T);
  int r = 0;
  while ((r + 1) * (r + 2) / 2 <= q) ++r;
  const int c = (int)q - r * (r + 1) / 2;
  dst[t] = src[((i * n + r) * n + c) * sw + (sw == 1 ? 0 : b)] * scale;
}
// dst (rows, Bp) = src (rows, sw) times `scale`; sw = 2 (shared, column 0) or Bp
__global__ void scale_copy_kernel(int64_t count, int64_t Bp, const double* __restrict__ src,
                                  int64_t sw, double* __restrict__ dst, double scale) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int64_t row = t / Bp, b = t % Bp;
  dst[t] = src[row * sw + (sw == Bp ? b : 0)] * scale;
}

__global__ void control_kernel(int B, int64_t F, int n64dim, const double* __restrict__ epsi,
                               PlanState ps, double* __restrict__ records, int max_iters,
                               double temp_high, double tol_mean, double tol_cost, double ctol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  if (!ps.active[b]) return;
  if (ps.status[b] != 0 || ps.fstatus[b] != 0) {  // a kernel failed this plan
    if (ps.status[b] == 0) {
      ps.status[b] = ps.fstatus[b];
      ps.where[b] = ps.fwhere[b];
    }
    ps.active[b] = 0;
    return;
  }
  const int it = ps.iters[b] + 1;
  const double ld_new = ps.logdet_next[b];
  ps.logdet[b] = ld_new;  // the accepted state becomes the current one
  double coll = 0.0;  // sum(f.e_psi), ascending factor order (optimizer.py:274)
  {
    // The adds are one dependent chain (the reference's order), so the loads
    // must be far ahead of them: each thread streams its own plan's column
    // through a two-chunk shared-memory buffer with asynchronous copies
    // (per-thread completion, no barrier), C loads in flight per chunk.
    constexpr int C = 64;
    __shared__ double sbuf[2][C][32];
    const int l = threadIdx.x;  // one warp per CTA
    auto issue = [&](int buf, int64_t f0) {
      const int64_t m = F - f0 < C ? F - f0 : C;
      for (int k = 0; k < m; ++k) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&sbuf[buf][k][l]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(epsi + (f0 + k) * B + b)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (F > 0) issue(0, 0);
    for (int64_t f0 = 0, c = 0; f0 < F; f0 += C, ++c) {
      const int buf = (int)(c & 1);
      if (f0 + C < F) {
        issue(buf ^ 1, f0 + C);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      const int64_t m = F - f0 < C ? F - f0 : C;
      for (int k = 0; k < m; ++k) coll += sbuf[buf][k][l];
    }
  }
  const double temp = ps.temp[b];
  const double dim = (double)n64dim;
  const double entropy = 0.5 * (dim * (kLog2Pi + 1.0) - ld_new);  // optimizer.py:234-235
  const double ent_cost = -temp * entropy;
  const double prior = ps.prior_cost[b];
  const double total = prior + coll + ent_cost;
  const double shift = ps.shift[b];
  double* rec = records + ((int64_t)(it - 1) * B + b) * GVP_NREC;
  rec[0] = ps.beta[b];
  rec[1] = temp;
  rec[2] = prior;
  rec[3] = coll;
  rec[4] = ent_cost;
  rec[5] = total;
  rec[6] = ps.kl[b];
  rec[7] = shift;
  ps.iters[b] = it;
  ps.total[b] = total;
  const double prev_temp = ps.prev_temp[b], prev_total = ps.prev_total[b];
  const bool same_temp = !isnan(prev_temp) && prev_temp == temp;
  const double change = !isnan(prev_total) ? fabs(total - prev_total) : INFINITY;
  if (same_temp && shift < tol_mean && change < tol_cost) {
    ps.converged[b] = 1;
    ps.active[b] = 0;
    return;
  }
  ps.prev_total[b] = (same_temp || isnan(prev_temp)) ? total : NAN;
  ps.prev_temp[b] = temp;
  if (!ps.switched[b] && coll < ctol && temp != temp_high) {
    ps.temp[b] = temp_high;
    ps.switched[b] = 1;
    ps.switch_it[b] = it;
    ps.prev_total[b] = NAN;
  }
  if (it >= max_iters) {
    ps.active[b] = 0;
    return;
  }
}

__global__ void fill_kernel(double* p, int64_t count, double v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count) p[t] = v;
}

// plans with a finite entry take that step size instead of the searched one;
// fixkl marks those whose pinned step the search did not accept (its KL and
// log det then come from the commit and the forward log det kernel)
__global__ void pin_beta_kernel(int B, const double* __restrict__ pinned, const int* __restrict__ active,
                                double* __restrict__ beta, int* __restrict__ status, int* __restrict__ where,
                                int* __restrict__ fixkl) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || !active[b]) return;
  const double v = pinned[b];
  fixkl[b] = 0;
  if (isfinite(v)) {
    fixkl[b] = (status[b] != GVP_OK || beta[b] != v) ? 1 : 0;
    beta[b] = v;
    if (status[b] == GVP_ERR_NO_FEASIBLE_STEP) {  // the search found nothing; the pinned step is taken anyway
      status[b] = GVP_OK;
      where[b] = -1;
    }
  }
}

// dst (rows, B) column plans[s] <- src (nsel, rows) row s
__global__ void scatter_cols_kernel(int nsel, const int* __restrict__ plans, int64_t rows,
                                    const double* __restrict__ src, double* __restrict__ dst, int64_t B) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)nsel * rows) return;
  const int64_t sidx = t / rows, row = t % rows;
  dst[row * B + plans[sidx]] = src[t];
}

__global__ void count_active_kernel(int B, const int* active, int* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < B && active[b]) atomicAdd(out, 1);
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
// The per-plan problem of a batch sharing one system (optimizer.batch_problem,
// SURVEY §8e): information and anchored prior mean are affine in each plan's
// start / goal offset from plan 0's, the initial mean is initial_mean's
// straight line (optimizer.py:280-296). One thread per (knot, coordinate,
// plan), plan-minor outputs; plans >= nreal (padding) copy plan 0.
__global__ void expand_boundary_kernel(int B, int nreal, int64_t K, int n, const double* __restrict__ bnd,
                                       double* __restrict__ info, double* __restrict__ pmean,
                                       double* __restrict__ mean) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * n * B) return;
  const int b = (int)(t % B);
  const int64_t kr = t / B, k = kr / n;
  const int r = (int)(kr - k * n);
  const double* base_info = bnd;
  const double* base_mean = bnd + K * n;
  const double* resp0 = base_mean + K * n;           // (n, K, n)
  const double* respg = resp0 + (int64_t)n * K * n;  // (n, K, n)
  const double* anchor = respg + (int64_t)n * K * n; // (n, n)
  const double* x0s = anchor + n * n;                // (nreal, n) [B rows reserved]
  const double* goals = x0s + (int64_t)B * n;
  const int bs = b < nreal ? b : 0;
  const double* x0 = x0s + (int64_t)bs * n;
  const double* g = goals + (int64_t)bs * n;
  double inf = base_info[k * n + r];
  if (k == 0) {
    double t0 = 0.0;  // (d0 @ anchor.T)[r]
    for (int j = 0; j < n; ++j) t0 += (x0[j] - x0s[j]) * anchor[r * n + j];
    inf += t0;
  }
  if (k == K - 1) {
    double tg = 0.0;
    for (int j = 0; j < n; ++j) tg += (g[j] - goals[j]) * anchor[r * n + j];
    inf += tg;
  }
  double m0 = 0.0, mg = 0.0;  // sum_j d0_j resp0[j], sum_j dg_j respg[j]
  for (int j = 0; j < n; ++j) {
    m0 += (x0[j] - x0s[j]) * resp0[((int64_t)j * K + k) * n + r];
    mg += (g[j] - goals[j]) * respg[((int64_t)j * K + k) * n + r];
  }
  const double a = (double)k * (1.0 / (double)(K - 1 > 0 ? K - 1 : 1));  // np.linspace(0, 1, K)
  info[t] = inf;
  pmean[t] = (base_mean[k * n + r] + m0) + mg;
  mean[t] = (1.0 - a) * x0[r] + a * g[r];
}

}  // namespace

struct gvp_engine {
  int B = 0;        // plans on device (even: the step kernel's TMA boxes need a 16-B plan stride)
  int nreal = 0;    // plans of the caller; an odd count is padded with a copy of plan 0
  int64_t K = 0;
  int n = 0, T = 0;
  bool shared_prior = false;
  int lanes = 1;
  bool fill = false;  // auto lanes: the probe kernel fills every resident CTA slot
  cudaStream_t stream = nullptr;
  Field field;
  Rule rule;
  double radius_eps = 0, sigma_obs = 0;
  gvp_plan_config cfg{};
  // resident state (plan-minor; diag-type blocks packed)
  double *mean = nullptr, *diag = nullptr, *off = nullptr, *covs = nullptr, *crosses = nullptr;
  double *kdiag = nullptr, *koff = nullptr, *info = nullptr, *pmean = nullptr;
  double *gmu = nullptr, *gdiag = nullptr, *v = nullptr, *epsi = nullptr, *scratch = nullptr;
  double *kfull_d = nullptr;  // staging for full-block prior uploads
  double* bnd = nullptr;       // gvp_engine_load_boundary staging (bnd_doubles())
  int64_t bnd_doubles() const { return 2 * K * n + 2 * (int64_t)n * K * n + (int64_t)n * n + 2 * (int64_t)B * n; }
  double* records = nullptr;
  double* scal = nullptr;
  int* ints = nullptr;
  unsigned long long* oob = nullptr;
  PlanState ps{};
  cudaGraphExec_t graph = nullptr;
  // optional per-iteration probe trace (the reference's select_step trace)
  double* plog = nullptr;
  int* pcount = nullptr;
  double* pinned = nullptr;  // gvp_engine_step_beta: per-plan step sizes (NaN = searched)
  int* eigh_list = nullptr;  // FactorOut::eigh_list (gaussian_sqrt's eigh fallback)
  int max_probes = 0;
  int iters_launched = 0;
  int64_t launches = 0;
  std::vector<void*> allocs;

  template <class Tp>
  int alloc(Tp** p, size_t count) {
    void* q = nullptr;
    GVP_CUDA(cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(Tp)));
    allocs.push_back(q);
    *p = static_cast<Tp*>(q);
    return GVP_OK;
  }
  ~gvp_engine() {
    if (graph) cudaGraphExecDestroy(graph);
    for (void* p : allocs) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
  }
  int64_t kb() const { return shared_prior ? 2 : B; }  // prior columns (2-wide when shared)
  View vw(const double* p, int64_t E) const { return View{p, E * B, B, 1}; }
  MutView mvw(double* p, int64_t E) const { return MutView{p, E * B, B, 1}; }

  // phases: bit 0 the factor kernel, bit 1 the eigh fix-up, which then
  // re-arms the list (zeroed once at creation) for the next factor kernel
  int factors(int phases = 3) {
    FactorOut fo{mvw(epsi, 1), mvw(gmu, n), mvw(gdiag, T), ps.oob, ps.fstatus, ps.fwhere, eigh_list};
    fo.phases = phases;
    fo.reset_eigh = false;
    launches += ((phases & 1) + ((phases >> 1) & 1)) * (K > 2);  // factor_grads_kernel, eigh fix-up
    int r = launch_factor_grads(B, K, n, vw(mean, n), vw(covs, T), rule.dev, field.dev, radius_eps,
                                sigma_obs, fo, ps.active, stream);
    if (r) return r;
    if (phases & 2) GVP_CUDA(cudaMemsetAsync(eigh_list, 0, sizeof(int), stream));
    return GVP_OK;
  }

  V2Launch step_args() const {
    V2Launch q{};
    q.nplans = B;
    q.K = K;
    q.n = n;
    q.Bp = B;
    q.lanes = lanes;
    q.fill = fill;
    q.ld = diag; q.lo = off; q.kd = kdiag; q.ko = koff; q.gd = gdiag;
    q.g = gmu; q.eta = info; q.v = v; q.mu = mean; q.pmean = pmean;
    q.kshared = shared_prior;
    q.o_mu = mean; q.o_ld = diag; q.o_lo = off; q.o_cov = covs; q.o_cr = crosses; q.o_v = v;
    q.beta = ps.beta; q.kl = ps.kl; q.ld_next = ps.logdet_next; q.shift = ps.shift;
    q.prior_cost = ps.prior_cost;
    q.temp = ps.temp; q.ld_cur = ps.logdet;
    q.search_kl = true; q.fixkl = ps.fixkl;
    q.kl_bound = cfg.kl_bound; q.beta_min = cfg.beta_min; q.beta_max = cfg.beta_max;
    q.status = ps.status; q.where = ps.where;
    q.probe_log = plog; q.max_probes = max_probes; q.nprobes = pcount;
    q.scratch = scratch;
    q.active = ps.active;
    return q;
  }

  int control() {
    const double ctol = cfg.collision_tol >= 0 ? cfg.collision_tol : 1e-4 * (double)(K - 1);
    // one warp per CTA: the per-plan collision sum is a chain of dependent
    // loads (reference order), so spread the plans over as many SMs as possible
    control_kernel<<<nblk(B, 32), 32, 0, stream>>>(B, std::max<int64_t>(K - 2, 0), (int)(K * n),
                                                     epsi, ps, records, cfg.max_iters,
                                                     cfg.temp_high, cfg.tol_mean, cfg.tol_cost, ctol);
    ++launches;
    GVP_CUDA(cudaGetLastError());
    return GVP_OK;
  }

  int iteration_body() {
    int r = launch_select_step_v2(step_args(), stream);
    if (r) return r;
    launches += 3;  // residual + bisection probes + commit
    if ((r = factors())) return r;
    return control();
  }
};

static int pick_lanes(const gvp_plan_config* cfg, int B) {
  if (cfg->spec_lanes > 0) return cfg->spec_lanes;
  // A split-probe CTA's bisection time is its per-knot step latency times its
  // rounds, nearly independent of how many CTAs share its SM (B200, C5: 3552
  // and 4096 plans over 222 / 256 CTAs both 11.5 ms). So spread the plans over
  // all 2 x 148 resident CTAs (launch_probe's fill: ppc = ceil(B / 296), even)
  // and take the layout with the fewest plan columns P = 32 / L >= ppc: each
  // plan gets 32 / ppc speculative lanes, which cut its rounds. C5: 14 plans
  // per CTA, 11.1 ms vs 12.0 ms at 16 per CTA; 3000 plans: 11.9 -> see DESIGN.
  const int64_t slots = 2 * 148;
  int64_t need = (B + slots - 1) / slots;
  need = std::max<int64_t>(2, (need + 1) / 2 * 2);
  int P = 2;
  while (P < need && P < 32) P *= 2;
  return 32 / P;
}

extern "C" int gvp_engine_create(gvp_engine** out, int32_t nplans, int64_t nknots, int32_t n,
                                 int32_t shared_prior, const double* grid, int32_t grid_ndim,
                                 const int64_t* grid_shape, const double* origin,
                                 double cell_size, double radius_eps, double sigma_obs,
                                 const double* points, const double* weights, int64_t npts,
                                 const gvp_plan_config* cfg) {
  *out = nullptr;
  if (nplans < 1 || nknots < 2 || !cfg) {
    set_error("bad engine dimensions");
    return GVP_ERR_ARG;
  }
  if (n != 2 && n != 4 && n != 6) {
    set_error("engine supports state size n in {2, 4, 6}");
    return GVP_ERR_UNSUPPORTED;
  }
  if (cfg->max_iters < 1 || !(cfg->kl_bound > 0) ||
      !(0 < cfg->beta_min && cfg->beta_min < cfg->beta_max)) {
    set_error("invalid optimizer config (optimizer.py:89-99)");
    return GVP_ERR_ARG;
  }
  const int lanes = pick_lanes(cfg, nplans);
  if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16) {
    set_error("spec_lanes must be 0 (auto), 1, 2, 4, 8 or 16");
    return GVP_ERR_ARG;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error("no CUDA device visible");
    return GVP_ERR_NO_DEVICE;
  }
  auto* e = new gvp_engine();
  e->nreal = nplans;
  e->B = (int)step_plan_stride(nplans);
  e->K = nknots;
  e->n = n;
  e->T = n * (n + 1) / 2;
  e->lanes = lanes;
  e->fill = cfg->spec_lanes <= 0;
  e->shared_prior = shared_prior != 0;
  e->cfg = *cfg;
  e->radius_eps = radius_eps;
  e->sigma_obs = sigma_obs;
  int r = GVP_OK;
  auto fail = [&](int code) {
    delete e;
    return code;
  };
  if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(cuda_fail(cudaGetLastError(), "cudaStreamCreate"));
  if ((r = e->field.build(grid, grid_ndim, grid_shape, origin, cell_size, e->stream))) return fail(r);
  if (grid_ndim > n) return set_error("grid dim exceeds state dim"), fail(GVP_ERR_ARG);
  if ((r = e->rule.build(points, weights, npts, n, grid_ndim, e->stream))) return fail(r);
  const int64_t B = e->B, K = nknots, N2 = (int64_t)n * n, T = e->T, kb = e->kb();
  const int64_t scr = std::max(step_scratch_doubles(e->B, K, n, lanes), K * T * B);
  if ((r = e->alloc(&e->mean, K * n * B)) || (r = e->alloc(&e->diag, K * T * B)) ||
      (r = e->alloc(&e->off, (K - 1) * N2 * B)) || (r = e->alloc(&e->covs, K * T * B)) ||
      (r = e->alloc(&e->crosses, (K - 1) * N2 * B)) || (r = e->alloc(&e->kdiag, K * T * kb)) ||
      (r = e->alloc(&e->koff, (K - 1) * N2 * kb)) || (r = e->alloc(&e->info, K * n * B)) ||
      (r = e->alloc(&e->pmean, K * n * B)) || (r = e->alloc(&e->gmu, K * n * B)) ||
      (r = e->alloc(&e->gdiag, K * T * B)) || (r = e->alloc(&e->v, K * n * B)) ||
      (r = e->alloc(&e->epsi, std::max<int64_t>(K - 2, 1) * B)) ||
      (r = e->alloc(&e->kfull_d, K * N2 * kb)) || (r = e->alloc(&e->scratch, (size_t)scr)) ||
      (r = e->alloc(&e->records, (size_t)cfg->max_iters * B * GVP_NREC)) ||
      (r = e->alloc(&e->scal, 10 * B)) || (r = e->alloc(&e->ints, 10 * B + 1)) ||
      (r = e->alloc(&e->oob, B)) || (r = e->alloc(&e->bnd, (size_t)e->bnd_doubles())) ||
      (r = e->alloc(&e->eigh_list, (size_t)(1 + B * std::max<int64_t>(K - 2, 1)))))
    return fail(r);
  if (cudaMemset(e->eigh_list, 0, sizeof(int)) != cudaSuccess) return fail(GVP_ERR_CUDA);
  PlanState& ps = e->ps;
  double* s = e->scal;
  ps.temp = s; ps.logdet = s + B; ps.beta = s + 2 * B; ps.kl = s + 3 * B; ps.shift = s + 4 * B;
  ps.prior_cost = s + 5 * B; ps.prev_total = s + 6 * B; ps.prev_temp = s + 7 * B; ps.total = s + 8 * B;
  ps.logdet_next = s + 9 * B;
  int* q = e->ints;
  ps.active = q; ps.status = q + B; ps.where = q + 2 * B; ps.converged = q + 3 * B;
  ps.iters = q + 4 * B; ps.switch_it = q + 5 * B; ps.switched = q + 6 * B; ps.fstatus = q + 7 * B;
  ps.fwhere = q + 8 * B; ps.fixkl = q + 9 * B; ps.nactive = q + 10 * B;
  ps.oob = e->oob;
  *out = e;
  return GVP_OK;
}

extern "C" void gvp_engine_destroy(gvp_engine* e) { delete e; }

// after kfull_d (full prior diag blocks), koff, info, pmean, mean are on device
static int engine_reset(gvp_engine* e) {
  const int64_t B = e->B, K = e->K, T = e->T, N2 = (int64_t)e->n * e->n, kb = e->kb();
  cudaStream_t s = e->stream;
  // knots 0 and K-1 carry no factor: their gradient blocks stay zero
  GVP_CUDA(cudaMemsetAsync(e->gmu, 0, K * e->n * B * sizeof(double), s));
  GVP_CUDA(cudaMemsetAsync(e->gdiag, 0, K * T * B * sizeof(double), s));
  const int64_t cnt = (int64_t)e->cfg.max_iters * B * GVP_NREC;
  fill_kernel<<<nblk(cnt, 256), 256, 0, s>>>(e->records, cnt, NAN);
  init_plans_kernel<<<nblk(B, 128), 128, 0, s>>>((int)B, e->ps, e->cfg.temp_low);
  // prior precision diag -> packed; initial_state (optimizer.py:280-296):
  // Lambda_0 = K^{-1} / init_cov_scale, per plan
  pack_sym_kernel<<<nblk(K * T * kb, 256), 256, 0, s>>>(K, e->n, e->shared_prior ? 1 : B, kb,
                                                        e->kfull_d, e->kdiag, 1.0);
  const double inv_scale = 1.0 / e->cfg.init_cov_scale;
  scale_copy_kernel<<<nblk(K * T * B, 256), 256, 0, s>>>(K * T * B, B, e->kdiag, kb, e->diag,
                                                         inv_scale);
  scale_copy_kernel<<<nblk((K - 1) * N2 * B, 256), 256, 0, s>>>((K - 1) * N2 * B, B, e->koff, kb,
                                                                e->off, inv_scale);
  GVP_CUDA(cudaGetLastError());
  // result.marginals = gbp_marginals(cur.prec) (optimizer.py:329) + log det, v = Lambda mu
  int r = launch_marginals_packed((int)B, K, e->n, B, e->diag, e->off, e->covs, e->crosses,
                                  e->ps.logdet, e->ps.status, e->ps.where, e->scratch, nullptr, s);
  if (r) return r;
  // ld_cur of the first search: forward Schur, the probes' own recursion (the
  // backward-sweep value above differs by ~cond * eps, which the KL would see)
  if ((r = launch_logdet_fwd_packed((int)B, K, e->n, B, e->diag, e->off, e->ps.logdet, nullptr, e->ps.status,
                                    e->ps.where, s)))
    return r;
  if ((r = launch_lam_mu((int)B, K, e->n, B, e->diag, e->off, e->mean, e->v, s))) return r;
  // first factor sweep (optimizer.py:338-344)
  if ((r = e->factors())) return r;
  e->launches += 8;
  e->iters_launched = 0;
  if (e->graph) {
    cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
  }
  return GVP_OK;
}

static int engine_upload(gvp_engine* e, const double* kdiag, const double* koff,
                         const double* info, const double* pm, const double* m0,
                         cudaMemcpyKind kind) {
  const int64_t K = e->K, N2 = (int64_t)e->n * e->n;
  cudaStream_t s = e->stream;
  // caller layout (rows, nreal) -> device (rows, B); a padding column is a copy of plan 0
  auto put = [&](double* dst, const double* src, int64_t rows) -> int {
    const size_t sp = (size_t)e->nreal * 8, dp = (size_t)e->B * 8;
    GVP_CUDA(cudaMemcpy2DAsync(dst, dp, src, sp, sp, rows, kind, s));
    if (e->B > e->nreal) GVP_CUDA(cudaMemcpy2DAsync(dst + e->nreal, dp, src, sp, 8, rows, kind, s));
    return GVP_OK;
  };
  int r;
  if (e->shared_prior) {
    GVP_CUDA(cudaMemcpyAsync(e->kfull_d, kdiag, K * N2 * 8, kind, s));
    for (int col = 0; col < 2; ++col)  // 2-wide copy of the shared off blocks
      GVP_CUDA(cudaMemcpy2DAsync(e->koff + col, 16, koff, 8, 8, (K - 1) * N2, kind, s));
  } else {
    if ((r = put(e->kfull_d, kdiag, K * N2)) || (r = put(e->koff, koff, (K - 1) * N2))) return r;
  }
  if ((r = put(e->info, info, K * e->n)) || (r = put(e->pmean, pm, K * e->n)) ||
      (r = put(e->mean, m0, K * e->n)))
    return r;
  return engine_reset(e);
}

// device (rows, B) -> caller (rows, nreal)
static int get_cols(gvp_engine* e, double* dst, const double* src, int64_t rows) {
  const size_t sp = (size_t)e->B * 8, dp = (size_t)e->nreal * 8;
  GVP_CUDA(cudaMemcpy2DAsync(dst, dp, src, sp, dp, rows, cudaMemcpyDeviceToHost, e->stream));
  return GVP_OK;
}

extern "C" int gvp_engine_load(gvp_engine* e, const double* kdiag, const double* koff,
                               const double* info, const double* prior_mean,
                               const double* init_mean) {
  return engine_upload(e, kdiag, koff, info, prior_mean, init_mean, cudaMemcpyHostToDevice);
}

// Upload a shared-system batch by its boundary states (see expand_boundary_kernel):
// host pointers; kdiag / koff as for gvp_engine_load (one plan's blocks),
// base_info / base_mean (K, n) of plan 0's prior, resp0 / respg (n, K, n) the
// anchored-mean responses to unit start / goal offsets, anchor (n, n), x0s /
// goals (nplans, n). The initial mean is initial_mean's straight line.
extern "C" int gvp_engine_load_boundary(gvp_engine* e, const double* kdiag, const double* koff,
                                        const double* base_info, const double* base_mean, const double* resp0,
                                        const double* respg, const double* anchor, const double* x0s,
                                        const double* goals) {
  if (!e || !kdiag || !koff || !base_info || !base_mean || !resp0 || !respg || !anchor || !x0s || !goals)
    return GVP_ERR_ARG;
  if (!e->shared_prior) {
    set_error("gvp_engine_load_boundary needs a shared-prior engine");
    return GVP_ERR_ARG;
  }
  const int64_t K = e->K, n = e->n, N2 = n * n, Kn = K * n;
  cudaStream_t s = e->stream;
  GVP_CUDA(cudaMemcpyAsync(e->kfull_d, kdiag, K * N2 * 8, cudaMemcpyHostToDevice, s));
  for (int col = 0; col < 2; ++col)  // 2-wide copy of the shared off blocks
    GVP_CUDA(cudaMemcpy2DAsync(e->koff + col, 16, koff, 8, 8, (K - 1) * N2, cudaMemcpyHostToDevice, s));
  double* d = e->bnd;
  GVP_CUDA(cudaMemcpyAsync(d, base_info, Kn * 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(d + Kn, base_mean, Kn * 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(d + 2 * Kn, resp0, n * Kn * 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(d + 2 * Kn + n * Kn, respg, n * Kn * 8, cudaMemcpyHostToDevice, s));
  double* da = d + 2 * Kn + 2 * n * Kn;
  GVP_CUDA(cudaMemcpyAsync(da, anchor, N2 * 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(da + N2, x0s, (size_t)e->nreal * n * 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(da + N2 + (int64_t)e->B * n, goals, (size_t)e->nreal * n * 8, cudaMemcpyHostToDevice, s));
  const int64_t tot = K * n * e->B;
  expand_boundary_kernel<<<nblk(tot, 256), 256, 0, s>>>(e->B, e->nreal, K, (int)n, d, e->info, e->pmean, e->mean);
  GVP_CUDA(cudaGetLastError());
  ++e->launches;
  return engine_reset(e);
}

extern "C" int gvp_engine_load_dev(gvp_engine* e, const double* kdiag, const double* koff,
                                   const double* info, const double* prior_mean,
                                   const double* init_mean) {
  return engine_upload(e, kdiag, koff, info, prior_mean, init_mean, cudaMemcpyDeviceToDevice);
}

extern "C" int gvp_engine_step(gvp_engine* e, int32_t iters, int32_t sync) {
  cudaStream_t s = e->stream;
  static const bool no_graph = std::getenv("GVP_NO_GRAPH") != nullptr;
  for (int k = 0; k < iters && e->iters_launched < e->cfg.max_iters; ++k) {
    if (no_graph) {  // debugging aid: plain launches
      int r = e->iteration_body();
      if (r) return r;
      ++e->iters_launched;
      continue;
    }
    if (!e->graph) {
      cudaGraph_t g;
      GVP_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      const int64_t before = e->launches;
      int r = e->iteration_body();
      cudaError_t ce = cudaStreamEndCapture(s, &g);
      if (r) return r;
      if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
      GVP_CUDA(cudaGraphInstantiate(&e->graph, g, 0));
      cudaGraphDestroy(g);
      e->launches = before;  // counted per replay below
    }
    GVP_CUDA(cudaGraphLaunch(e->graph, s));
    e->launches += 4 + 2 * (e->K > 2);  // residual, probes, commit, [factors + eigh fix-up], control
    ++e->iters_launched;
  }
  if (sync) GVP_CUDA(cudaStreamSynchronize(s));
  return GVP_OK;
}

// Per-kernel device times of `iters` iterations (ungraphed, events between the
// kernels), summed into ms[0..nms): residual, probe (bisection), commit, factor
// kernel, eigh fix-up, control.
extern "C" int gvp_engine_step_profiled_ex(gvp_engine* e, int32_t iters, double* ms, int32_t nms) {
  if (!e || !ms || nms < 1) return GVP_ERR_ARG;
  constexpr int NB = 6;
  cudaStream_t s = e->stream;
  cudaEvent_t ev[NB + 1];
  for (auto& x : ev) GVP_CUDA(cudaEventCreate(&x));
  double acc[NB] = {0, 0, 0, 0, 0, 0};
  int r = GVP_OK;
  for (int k = 0; k < iters && e->iters_launched < e->cfg.max_iters; ++k) {
    GVP_CUDA(cudaEventRecord(ev[0], s));
    V2Launch q = e->step_args();
    q.ev_residual_done = ev[1];
    if ((r = launch_select_bisect(q, s))) break;
    GVP_CUDA(cudaEventRecord(ev[2], s));
    if ((r = launch_select_commit(e->step_args(), s))) break;
    e->launches += 3;  // residual + bisection probes + commit
    GVP_CUDA(cudaEventRecord(ev[3], s));
    if ((r = e->factors(1))) break;
    GVP_CUDA(cudaEventRecord(ev[4], s));
    if ((r = e->factors(2))) break;
    GVP_CUDA(cudaEventRecord(ev[5], s));
    if ((r = e->control())) break;
    GVP_CUDA(cudaEventRecord(ev[6], s));
    GVP_CUDA(cudaEventSynchronize(ev[6]));
    for (int j = 0; j < NB; ++j) {
      float t = 0.f;
      GVP_CUDA(cudaEventElapsedTime(&t, ev[j], ev[j + 1]));
      acc[j] += t;
    }
    ++e->iters_launched;
  }
  for (auto& x : ev) cudaEventDestroy(x);
  for (int j = 0; j < NB && j < nms; ++j) ms[j] = acc[j];
  return r;
}

// ms[0..4): bisection (residual + probes), commit, factor kernel, eigh fix-up + control
extern "C" int gvp_engine_step_profiled(gvp_engine* e, int32_t iters, double* ms) {
  double m[6];
  const int r = gvp_engine_step_profiled_ex(e, iters, m, 6);
  if (r) return r;
  ms[0] = m[0] + m[1];
  ms[1] = m[2];
  ms[2] = m[3];
  ms[3] = m[4] + m[5];
  return GVP_OK;
}

// One iteration in which every plan with a finite beta[b] (host, nplans
// entries) takes that step size instead of the searched one. The search still
// runs (and is traced): a caller can replay a known step sequence, e.g. the
// reference's, and compare each search's decisions against it.
extern "C" int gvp_engine_step_beta(gvp_engine* e, const double* beta) {
  if (!e || !beta) return GVP_ERR_ARG;
  if (e->iters_launched >= e->cfg.max_iters) return GVP_OK;
  cudaStream_t s = e->stream;
  int r;
  if (!e->pinned && (r = e->alloc(&e->pinned, (size_t)e->B))) return r;
  std::vector<double> h(e->B);
  for (int b = 0; b < e->B; ++b) h[b] = beta[b < e->nreal ? b : 0];
  GVP_CUDA(cudaMemcpyAsync(e->pinned, h.data(), sizeof(double) * e->B, cudaMemcpyHostToDevice, s));
  if ((r = launch_select_bisect(e->step_args(), s))) return r;
  pin_beta_kernel<<<nblk(e->B, 128), 128, 0, s>>>(e->B, e->pinned, e->ps.active, e->ps.beta, e->ps.status,
                                                  e->ps.where, e->ps.fixkl);
  GVP_CUDA(cudaGetLastError());
  if ((r = launch_select_commit(e->step_args(), s))) return r;
  if ((r = launch_logdet_fwd_packed(e->B, e->K, e->n, e->B, e->diag, e->off, e->ps.logdet_next, e->ps.fixkl,
                                    nullptr, nullptr, s)))
    return r;
  e->launches += 5;  // residual + bisection probes + pin + commit + log det
  if ((r = e->factors())) return r;
  if ((r = e->control())) return r;
  GVP_CUDA(cudaMemsetAsync(e->ps.fixkl, 0, sizeof(int) * e->B, s));
  ++e->iters_launched;
  GVP_CUDA(cudaStreamSynchronize(s));
  return GVP_OK;
}

// Replace the current iterate (mean, precision) of selected plans, e.g. with
// another implementation's state, and redo what an iteration leaves behind
// for the next one: marginals, forward log det, Lambda mu and the factor
// stage at the new state. Records, iteration counts and convergence state are
// kept. Host arrays, batch-major over the nsel selected plans: mean
// (nsel, K, n), diag (nsel, K, n, n), off (nsel, K-1, n, n).
extern "C" int gvp_engine_set_state(gvp_engine* e, int32_t nsel, const int32_t* plans, const double* mean,
                                    const double* diag, const double* off) {
  if (!e || nsel < 1 || !plans || !mean || !diag || !off) return GVP_ERR_ARG;
  const int64_t K = e->K, n = e->n, T = e->T, N2 = n * n, B = e->B;
  for (int s = 0; s < nsel; ++s)
    if (plans[s] < 0 || plans[s] >= e->nreal) {
      set_error("set_state: plan index out of range");
      return GVP_ERR_ARG;
    }
  cudaStream_t st = e->stream;
  // packed lower diag blocks, host side
  std::vector<double> dp((size_t)nsel * K * T);
  for (int64_t s = 0; s < nsel; ++s)
    for (int64_t i = 0; i < K; ++i)
      for (int64_t r = 0; r < n; ++r)
        for (int64_t c = 0; c <= r; ++c)
          dp[(s * K + i) * T + r * (r + 1) / 2 + c] = diag[((s * K + i) * n + r) * n + c];
  const int64_t rows_max = std::max({K * n, K * T, (K - 1) * N2});
  double* stage = nullptr;
  int* dplans = nullptr;
  GVP_CUDA(cudaMalloc(&stage, sizeof(double) * nsel * rows_max));
  GVP_CUDA(cudaMalloc(&dplans, sizeof(int) * nsel));
  int r = GVP_OK;
  auto put = [&](const double* src, int64_t rows, double* dst) -> int {
    GVP_CUDA(cudaMemcpyAsync(stage, src, sizeof(double) * nsel * rows, cudaMemcpyHostToDevice, st));
    scatter_cols_kernel<<<nblk(nsel * rows, 256), 256, 0, st>>>(nsel, dplans, rows, stage, dst, B);
    GVP_CUDA(cudaGetLastError());
    GVP_CUDA(cudaStreamSynchronize(st));  // the stage buffer is reused
    return GVP_OK;
  };
  cudaError_t ce = cudaMemcpyAsync(dplans, plans, sizeof(int) * nsel, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) r = cuda_fail(ce, "set_state upload");
  if (!r) r = put(mean, K * n, e->mean);
  if (!r) r = put(dp.data(), K * T, e->diag);
  if (!r && K > 1) r = put(off, (K - 1) * N2, e->off);
  cudaFree(stage);
  cudaFree(dplans);
  if (r) return r;
  if ((r = launch_marginals_packed((int)B, K, e->n, B, e->diag, e->off, e->covs, e->crosses, e->ps.logdet,
                                   e->ps.status, e->ps.where, e->scratch, e->ps.active, st)))
    return r;
  if ((r = launch_logdet_fwd_packed((int)B, K, e->n, B, e->diag, e->off, e->ps.logdet, nullptr, e->ps.status,
                                    e->ps.where, st)))
    return r;
  if ((r = launch_lam_mu((int)B, K, e->n, B, e->diag, e->off, e->mean, e->v, st))) return r;
  if ((r = e->factors())) return r;
  e->launches += 4;
  GVP_CUDA(cudaStreamSynchronize(st));
  return GVP_OK;
}

// Per-plan count of sigma points that left the SDF grid (clamped, sdf.py:53-56)
// over every factor stage so far.
extern "C" int gvp_engine_get_oob(gvp_engine* e, int64_t* oob) {
  if (!e || !oob) return GVP_ERR_ARG;
  GVP_CUDA(cudaMemcpyAsync(oob, e->ps.oob, sizeof(int64_t) * e->nreal, cudaMemcpyDeviceToHost, e->stream));
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  return GVP_OK;
}

extern "C" void* gvp_engine_stream(gvp_engine* e) { return (void*)e->stream; }

extern "C" int gvp_engine_sync(gvp_engine* e) {
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  return GVP_OK;
}

extern "C" int gvp_engine_active(gvp_engine* e, int32_t* nactive) {
  GVP_CUDA(cudaMemsetAsync(e->ps.nactive, 0, sizeof(int), e->stream));
  count_active_kernel<<<nblk(e->nreal, 128), 128, 0, e->stream>>>(e->nreal, e->ps.active, e->ps.nactive);
  GVP_CUDA(cudaGetLastError());
  GVP_CUDA(cudaMemcpyAsync(nactive, e->ps.nactive, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  if (e->iters_launched >= e->cfg.max_iters) *nactive = 0;
  return GVP_OK;
}

// packed (K, T, B) device -> full (K, n, n, B) host
static int fetch_sym(gvp_engine* e, double* host, const double* dev) {
  const int64_t B = e->nreal, K = e->K, T = e->T, n = e->n;
  std::vector<double> tmp((size_t)(K * T * B));
  int rr = get_cols(e, tmp.data(), dev, K * T);
  if (rr) return rr;
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  for (int64_t i = 0; i < K; ++i)
    for (int64_t r = 0; r < n; ++r)
      for (int64_t c = 0; c <= r; ++c) {
        const double* src = &tmp[(size_t)((i * T + r * (r + 1) / 2 + c) * B)];
        double* d1 = host + ((i * n + r) * n + c) * B;
        double* d2 = host + ((i * n + c) * n + r) * B;
        for (int64_t b = 0; b < B; ++b) d1[b] = d2[b] = src[b];
      }
  return GVP_OK;
}

extern "C" int gvp_engine_get_state(gvp_engine* e, double* mean, double* diag, double* off,
                                    double* covs, double* crosses) {
  const int64_t K = e->K, N2 = (int64_t)e->n * e->n;
  cudaStream_t s = e->stream;
  int r0;
  if (mean && (r0 = get_cols(e, mean, e->mean, K * e->n))) return r0;
  if (off && (r0 = get_cols(e, off, e->off, (K - 1) * N2))) return r0;
  if (crosses && (r0 = get_cols(e, crosses, e->crosses, (K - 1) * N2))) return r0;
  GVP_CUDA(cudaStreamSynchronize(s));
  if (diag) {
    int r = fetch_sym(e, diag, e->diag);
    if (r) return r;
  }
  if (covs) {
    int r = fetch_sym(e, covs, e->covs);
    if (r) return r;
  }
  return GVP_OK;
}

extern "C" int gvp_engine_get_packed(gvp_engine* e, double* mean, double* covs_packed) {
  if (!e) return GVP_ERR_ARG;
  int r;
  if (mean && (r = get_cols(e, mean, e->mean, e->K * e->n))) return r;
  if (covs_packed && (r = get_cols(e, covs_packed, e->covs, e->K * e->T))) return r;
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  return GVP_OK;
}

extern "C" int gvp_engine_get_summary(gvp_engine* e, int32_t* converged, int32_t* iterations,
                                      int32_t* switch_iteration, int32_t* status, int32_t* where) {
  cudaStream_t s = e->stream;
  const size_t bytes = e->nreal * sizeof(int);
  if (converged) GVP_CUDA(cudaMemcpyAsync(converged, e->ps.converged, bytes, cudaMemcpyDeviceToHost, s));
  if (iterations) GVP_CUDA(cudaMemcpyAsync(iterations, e->ps.iters, bytes, cudaMemcpyDeviceToHost, s));
  if (switch_iteration) GVP_CUDA(cudaMemcpyAsync(switch_iteration, e->ps.switch_it, bytes, cudaMemcpyDeviceToHost, s));
  if (status) GVP_CUDA(cudaMemcpyAsync(status, e->ps.status, bytes, cudaMemcpyDeviceToHost, s));
  if (where) GVP_CUDA(cudaMemcpyAsync(where, e->ps.where, bytes, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  return GVP_OK;
}

extern "C" int gvp_engine_get_records(gvp_engine* e, double* records) {
  const size_t sp = (size_t)e->B * GVP_NREC * 8, dp = (size_t)e->nreal * GVP_NREC * 8;
  GVP_CUDA(cudaMemcpy2DAsync(records, dp, e->records, sp, dp, e->cfg.max_iters,
                             cudaMemcpyDeviceToHost, e->stream));
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  return GVP_OK;
}

extern "C" int gvp_engine_device_state(gvp_engine* e, double** mean, double** diag, double** off,
                                       double** covs, double** crosses) {
  if (mean) *mean = e->mean;
  if (diag) *diag = e->diag;
  if (off) *off = e->off;
  if (covs) *covs = e->covs;
  if (crosses) *crosses = e->crosses;
  return GVP_OK;
}

extern "C" int64_t gvp_engine_launches(gvp_engine* e) { return e->launches; }

// Map bank: nmaps signed-distance maps with the engine's grid
// geometry; plan b reads map plan_map[b]. From host grids (nmaps x (ny, nx) or
// (nz, ny, nx), row-major) or rasterised on the device from primitive lists.
static int install_bank(gvp_engine* e, int nmaps, const double* raw_dev, const int32_t* plan_map, double lip) {
  for (int b = 0; b < e->nreal; ++b)
    if (plan_map[b] < 0 || plan_map[b] >= nmaps) {
      set_error("plan_map entry outside [0, nmaps)");
      return GVP_ERR_ARG;
    }
  FieldDev f = e->field.dev;
  const int64_t stride = packed_field_doubles(f);
  double* bank = nullptr;
  int* pm = nullptr;
  int r;
  if ((r = e->alloc(&bank, (size_t)stride * nmaps)) || (r = e->alloc(&pm, (size_t)e->B))) return r;
  if ((r = pack_field_maps(f, nmaps, raw_dev, bank, e->stream))) return r;
  std::vector<int> h(e->B);
  for (int b = 0; b < e->B; ++b) h[b] = plan_map[b < e->nreal ? b : 0];  // padding plan = plan 0
  GVP_CUDA(cudaMemcpyAsync(pm, h.data(), sizeof(int) * e->B, cudaMemcpyHostToDevice, e->stream));
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  f.corners = bank;
  f.plan_map = pm;
  f.map_stride = stride;
  f.lip = lip;
  e->field.dev = f;
  if (e->graph) {  // the captured factor launch holds the old field
    cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
  }
  return GVP_OK;
}

extern "C" int gvp_engine_set_map_bank(gvp_engine* e, int32_t nmaps, const double* grids,
                                       const int32_t* plan_map) {
  if (!e || nmaps < 1 || !grids || !plan_map) return GVP_ERR_ARG;
  const FieldDev& f = e->field.dev;
  const int64_t cells = f.nx * f.ny * f.nz;
  double* raw = nullptr;
  GVP_CUDA(cudaMalloc(&raw, sizeof(double) * cells * nmaps));
  cudaError_t ce = cudaMemcpyAsync(raw, grids, sizeof(double) * cells * nmaps, cudaMemcpyHostToDevice, e->stream);
  // Lipschitz bound over every map of the bank (the factor kernel's clear-cloud shortcut)
  const double lip = field_lipschitz(grids, nmaps, f.ndim, f.nx, f.ny, f.nz, f.cell);
  int r = ce == cudaSuccess ? install_bank(e, nmaps, raw, plan_map, lip) : GVP_ERR_CUDA;
  if (ce != cudaSuccess) set_error(cudaGetErrorString(ce));
  cudaStreamSynchronize(e->stream);
  cudaFree(raw);
  return r;
}

extern "C" int gvp_engine_raster_map_bank(gvp_engine* e, int32_t nmaps, const int32_t* prim_off,
                                          const int32_t* kinds, const double* params, const int32_t* plan_map) {
  if (!e || nmaps < 1 || !prim_off || !plan_map) return GVP_ERR_ARG;
  const FieldDev& f = e->field.dev;
  const int dim = f.ndim;
  const int nprim = prim_off[nmaps];
  for (int m = 0; m < nmaps; ++m)
    if (prim_off[m] > prim_off[m + 1] || prim_off[m] < 0) return GVP_ERR_ARG;
  if (nprim > 0 && (!kinds || !params)) return GVP_ERR_ARG;
  const int64_t cells = f.nx * f.ny * f.nz;
  const int64_t counts[3] = {f.nx, f.ny, f.nz};
  const double origin[3] = {f.ox, f.oy, f.oz};
  double *raw = nullptr, *par = nullptr;
  int *off = nullptr, *kd = nullptr;
  GVP_CUDA(cudaMalloc(&raw, sizeof(double) * cells * nmaps));
  GVP_CUDA(cudaMalloc(&par, sizeof(double) * (2 * dim * nprim + 1)));
  GVP_CUDA(cudaMalloc(&off, sizeof(int) * (nmaps + 1)));
  GVP_CUDA(cudaMalloc(&kd, sizeof(int) * (nprim + 1)));
  GVP_CUDA(cudaMemcpyAsync(off, prim_off, sizeof(int) * (nmaps + 1), cudaMemcpyHostToDevice, e->stream));
  if (nprim) {
    GVP_CUDA(cudaMemcpyAsync(kd, kinds, sizeof(int) * nprim, cudaMemcpyHostToDevice, e->stream));
    GVP_CUDA(cudaMemcpyAsync(par, params, sizeof(double) * 2 * dim * nprim, cudaMemcpyHostToDevice, e->stream));
  }
  int r = rasterize_maps(dim, counts, origin, f.cell, nmaps, off, kd, par, raw, e->stream);
  if (!r) r = install_bank(e, nmaps, raw, plan_map, INFINITY);  // no host copy: shortcut off
  cudaStreamSynchronize(e->stream);
  cudaFree(raw);
  cudaFree(par);
  cudaFree(off);
  cudaFree(kd);
  return r;
}

// Record every probe (beta, spd, kl) of each plan's step-size search; the log
// holds the last iteration. Must be enabled before the first step.
extern "C" int gvp_engine_trace_probes(gvp_engine* e, int32_t max_probes) {
  if (!e || max_probes <= 0) return GVP_ERR_ARG;
  if (e->iters_launched > 0) {
    set_error("enable the probe trace before the first step");
    return GVP_ERR_ARG;
  }
  int r;
  if ((r = e->alloc(&e->plog, (size_t)e->B * max_probes * 3)) || (r = e->alloc(&e->pcount, (size_t)e->B)))
    return r;
  GVP_CUDA(cudaMemsetAsync(e->pcount, 0, sizeof(int) * e->B, e->stream));
  e->max_probes = max_probes;
  if (e->graph) {
    cudaGraphExecDestroy(e->graph);
    e->graph = nullptr;
  }
  return GVP_OK;
}

extern "C" int gvp_engine_get_probes(gvp_engine* e, double* log, int32_t* counts) {
  if (!e || !e->plog) return GVP_ERR_ARG;
  GVP_CUDA(cudaMemcpyAsync(log, e->plog, sizeof(double) * e->nreal * e->max_probes * 3,
                           cudaMemcpyDeviceToHost, e->stream));
  GVP_CUDA(cudaMemcpyAsync(counts, e->pcount, sizeof(int) * e->nreal, cudaMemcpyDeviceToHost, e->stream));
  GVP_CUDA(cudaStreamSynchronize(e->stream));
  return GVP_OK;
}
extern "C" int32_t gvp_engine_lanes(gvp_engine* e) { return e->lanes; }
