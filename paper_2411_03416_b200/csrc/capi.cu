// C ABI of libgvp_b200: drop-in host entry points and the batched engine.
// See include/gvp_b200.h for the contract of every function.
#include <cuda_runtime.h>

#include <cstdlib>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gvp_internal.cuh"

namespace gvp {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int cuda_fail(cudaError_t err, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorString(err) + " in " + what;
  return err == cudaErrorNoDevice || err == cudaErrorInsufficientDriver ? GVP_ERR_NO_DEVICE
                                                                        : GVP_ERR_CUDA;
}

// plan-minor views over a batch of B plans
static View pview(const double* p, int64_t E, int64_t B) { return View{p, E * B, B, 1}; }
static MutView pmview(double* p, int64_t E, int64_t B) { return MutView{p, E * B, B, 1}; }
// a view shared by all plans (one copy)
static View sview(const double* p, int64_t E) { return View{p, E, 1, 0}; }

// --------------------------------------------------------------- device arena
// grow-only device buffers reused across drop-in calls (one per slot)
struct Arena {
  std::vector<void*> ptr;
  std::vector<size_t> cap;
  template <class T>
  int get(int slot, size_t count, T** out) {
    if ((int)ptr.size() <= slot) {
      ptr.resize(slot + 1, nullptr);
      cap.resize(slot + 1, 0);
    }
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (cap[slot] < bytes) {
      if (ptr[slot]) cudaFree(ptr[slot]);
      ptr[slot] = nullptr;
      cap[slot] = 0;
      GVP_CUDA(cudaMalloc(&ptr[slot], bytes));
      cap[slot] = bytes;
    }
    *out = static_cast<T*>(ptr[slot]);
    return GVP_OK;
  }
};

struct Context {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  Arena arena;
  Field field;
  Rule rule;
  // gvp_select_step_size_ld: a known log det of the current precision (NaN:
  // compute it) and the accepted state's log det, for the call in progress
  double ld_in = NAN, ld_out = NAN;
  int init() {
    if (stream) return GVP_OK;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      set_error("no CUDA device visible");
      return GVP_ERR_NO_DEVICE;
    }
    GVP_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    return GVP_OK;
  }
};
static Context& ctx() {
  static Context* c = new Context();  // leaked on purpose: no teardown-order issues at exit
  return *c;
}

#define GVP_TRY(expr)          \
  do {                         \
    int _r = (expr);           \
    if (_r != GVP_OK) return _r; \
  } while (0)

template <class T>
static int h2d(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (count) GVP_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return GVP_OK;
}
template <class T>
static int d2h(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (count) GVP_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  return GVP_OK;
}

// full (K, n, n) -> packed lower (K, n(n+1)/2) and back (host side of the C ABI)
static std::vector<double> pack_lower(const double* full, int64_t K, int n) {
  const int T = n * (n + 1) / 2;
  std::vector<double> out((size_t)(K * T));
  for (int64_t i = 0; i < K; ++i)
    for (int r = 0; r < n; ++r)
      for (int c = 0; c <= r; ++c) out[(size_t)(i * T + r * (r + 1) / 2 + c)] = full[(i * n + r) * n + c];
  return out;
}
static void unpack_sym(const double* packed, int64_t K, int n, double* full) {
  const int T = n * (n + 1) / 2;
  for (int64_t i = 0; i < K; ++i)
    for (int r = 0; r < n; ++r)
      for (int c = 0; c <= r; ++c) {
        const double v = packed[i * T + r * (r + 1) / 2 + c];
        full[(i * n + r) * n + c] = v;
        full[(i * n + c) * n + r] = v;
      }
}
static bool blocks_symmetric(const double* full, int64_t K, int n) {
  for (int64_t i = 0; i < K; ++i)
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < r; ++c)
        if (full[(i * n + r) * n + c] != full[(i * n + c) * n + r]) return false;
  return true;
}
static bool all_zero(const double* p, int64_t count) {
  if (!p) return true;
  for (int64_t k = 0; k < count; ++k)
    if (p[k] != 0.0) return false;
  return true;
}
static int g_step_lanes = 16;  // candidate lanes of the drop-in select_step_size (one plan)

static int check_n(int n) {
  if (n < 1 || n > 8) {
    set_error("block size n must be in 1..8");
    return GVP_ERR_UNSUPPORTED;
  }
  return GVP_OK;
}
// the block-chain drop-ins also take wide blocks (wide_kernels.cu)
constexpr int kWideMin = 9, kWideMax = 32;
static int check_chain_n(int n) {
  if (n < 1 || n > kWideMax) {
    set_error("block size n must be in 1..32");
    return GVP_ERR_UNSUPPORTED;
  }
  return GVP_OK;
}

}  // namespace gvp

using namespace gvp;

// =================================================================== misc
extern "C" const char* gvp_last_error(void) { return g_err.c_str(); }
extern "C" const char* gvp_version(void) { return "gvp_b200 0.1.0 (sm_100a)"; }
extern "C" int gvp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// =================================================================== drop-in host API
extern "C" int gvp_factor_expectations(const double* means, const double* chols, int64_t nfac,
                                       int32_t n, const double* points, const double* weights,
                                       int64_t npts, const double* grid, int32_t grid_ndim,
                                       const int64_t* grid_shape, const double* origin,
                                       double cell_size, double radius_eps, double sigma_obs,
                                       int32_t pos_dim, double* e0, double* e1, double* e2,
                                       int64_t* oob) {
  (void)pos_dim;  // like _kernels.pyx:142, the grid's ndim decides
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_n(n));
  if (nfac < 0 || npts < 0) return set_error("negative size"), GVP_ERR_ARG;
  cudaStream_t s = C.stream;
  GVP_TRY(C.field.build(grid, grid_ndim, grid_shape, origin, cell_size, s));
  GVP_TRY(C.rule.build(points, weights, npts, n, grid_ndim, s));
  double *d_means, *d_chols, *d_e0, *d_e1, *d_e2;
  unsigned long long* d_oob;
  GVP_TRY(C.arena.get(0, nfac * n, &d_means));
  GVP_TRY(C.arena.get(1, nfac * n * n, &d_chols));
  GVP_TRY(C.arena.get(2, nfac, &d_e0));
  GVP_TRY(C.arena.get(3, nfac * n, &d_e1));
  GVP_TRY(C.arena.get(4, nfac * n * n, &d_e2));
  GVP_TRY(C.arena.get(5, 1, &d_oob));
  GVP_TRY(h2d(d_means, means, nfac * n, s));
  GVP_TRY(h2d(d_chols, chols, nfac * n * n, s));
  GVP_CUDA(cudaMemsetAsync(d_oob, 0, sizeof(unsigned long long), s));
  GVP_TRY(launch_factor_moments(nfac, n, d_means, d_chols, C.rule.dev, C.field.dev, radius_eps,
                                sigma_obs, d_e0, d_e1, d_e2, d_oob, s));
  unsigned long long h_oob = 0;
  GVP_TRY(d2h(e0, d_e0, nfac, s));
  GVP_TRY(d2h(e1, d_e1, nfac * n, s));
  GVP_TRY(d2h(e2, d_e2, nfac * n * n, s));
  GVP_TRY(d2h(&h_oob, d_oob, 1, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  *oob = (int64_t)h_oob;
  return GVP_OK;
}

extern "C" int gvp_evaluate_factors(const double* mean, const double* covs, int64_t nblocks,
                                    int32_t n, const double* points, const double* weights,
                                    int64_t npts, const double* grid, int32_t grid_ndim,
                                    const int64_t* grid_shape, const double* origin,
                                    double cell_size, double radius_eps, double sigma_obs,
                                    double* e_psi, double* g_mu, double* g_sigma, int64_t* oob,
                                    int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_n(n));
  if (n < grid_ndim) return set_error("state dim below grid dim"), GVP_ERR_ARG;
  cudaStream_t s = C.stream;
  const int64_t K = nblocks, F = std::max<int64_t>(K - 2, 0);
  *oob = 0;
  *where = -1;
  if (F == 0) return GVP_OK;
  GVP_TRY(C.field.build(grid, grid_ndim, grid_shape, origin, cell_size, s));
  GVP_TRY(C.rule.build(points, weights, npts, n, grid_ndim, s));
  double *d_mean, *d_covs, *d_epsi, *d_gmu, *d_gd;
  unsigned long long* d_oob;
  int* d_st;
  const int T = n * (n + 1) / 2;
  GVP_TRY(C.arena.get(0, K * n, &d_mean));
  GVP_TRY(C.arena.get(1, K * T, &d_covs));
  GVP_TRY(C.arena.get(2, F, &d_epsi));
  GVP_TRY(C.arena.get(3, K * n, &d_gmu));
  GVP_TRY(C.arena.get(4, K * T, &d_gd));
  GVP_TRY(C.arena.get(5, 1, &d_oob));
  GVP_TRY(C.arena.get(6, 2, &d_st));
  int* d_eigh;  // gaussian_sqrt's eigh fallback list (FactorOut::eigh_list)
  GVP_TRY(C.arena.get(7, (size_t)std::max<int64_t>(F, 1) + 1, &d_eigh));
  // the kernel reads the lower triangle of each covariance block, like
  // np.linalg.cholesky does in gaussian_sqrt (quadrature.py:175)
  const std::vector<double> covs_p = pack_lower(covs, K, n);
  GVP_TRY(h2d(d_mean, mean, K * n, s));
  GVP_TRY(h2d(d_covs, covs_p.data(), K * T, s));
  GVP_CUDA(cudaMemsetAsync(d_oob, 0, sizeof(unsigned long long), s));
  const int init_st[2] = {0, INT_MAX};
  GVP_TRY(h2d(d_st, init_st, 2, s));
  FactorOut fo{pmview(d_epsi, 1, 1), pmview(d_gmu, n, 1), pmview(d_gd, T, 1), d_oob, d_st,
               d_st + 1, d_eigh};
  GVP_TRY(launch_factor_grads(1, K, n, pview(d_mean, n, 1), pview(d_covs, T, 1), C.rule.dev,
                              C.field.dev, radius_eps, sigma_obs, fo, nullptr, s));
  int st[2];
  unsigned long long h_oob;
  std::vector<double> gd_p((size_t)(F * T));
  GVP_TRY(d2h(st, d_st, 2, s));
  GVP_TRY(d2h(&h_oob, d_oob, 1, s));
  GVP_TRY(d2h(e_psi, d_epsi, F, s));
  GVP_TRY(d2h(g_mu, d_gmu + n, F * n, s));
  GVP_TRY(d2h(gd_p.data(), d_gd + T, F * T, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  unpack_sym(gd_p.data(), F, n, g_sigma);
  *oob = (int64_t)h_oob;
  if (st[0] != GVP_OK) {
    *where = st[1];
    set_error(st[0] == GVP_ERR_SQRT ? "Singular matrix (eigh root of gaussian_sqrt with a clipped eigenvalue)"
                                    : "non-finite expectation");
    return st[0];
  }
  return GVP_OK;
}

namespace {
struct ChainBufs {
  double *diag, *off, *scr;
  int* st;
};
int upload_bt(Context& C, const double* diag, const double* off, int64_t K, int n, ChainBufs& b,
              int scr_lanes = 1) {
  cudaStream_t s = C.stream;
  GVP_TRY(C.arena.get(10, K * n * n, &b.diag));
  GVP_TRY(C.arena.get(11, std::max<int64_t>(K - 1, 1) * n * n, &b.off));
  GVP_TRY(C.arena.get(12, (size_t)chain_scratch_doubles(1, K, n, scr_lanes), &b.scr));
  GVP_TRY(C.arena.get(13, 4, &b.st));
  GVP_TRY(h2d(b.diag, diag, K * n * n, s));
  GVP_TRY(h2d(b.off, off, (K - 1) * n * n, s));
  return GVP_OK;
}
int fetch_status(Context& C, const int* d_st, int64_t* where) {
  int st[2];
  GVP_TRY(d2h(st, d_st, 2, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  if (where) *where = st[1];
  return st[0];
}
}  // namespace

// cyclic reduction for short chains: its rounding grows faster with K than the
// sequential sweep's on ill-conditioned (anchored) chains (cr_kernels.cu)
constexpr int64_t kCrMaxKnots = 128;

extern "C" int gvp_gbp_marginals(const double* diag, const double* off, int64_t nblocks,
                                 int32_t n, double* covs, double* crosses, int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  if (nblocks < 1) return set_error("need at least one block"), GVP_ERR_ARG;
  const int64_t K = nblocks;
  if (n >= kWideMin) {
    double *d_d, *d_o, *d_cov, *d_cr, *d_scr;
    int* d_st;
    GVP_TRY(C.arena.get(10, K * n * n, &d_d));
    GVP_TRY(C.arena.get(11, std::max<int64_t>(K - 1, 1) * n * n, &d_o));
    GVP_TRY(C.arena.get(12, (size_t)wide_scratch_doubles(1, K, n), &d_scr));
    GVP_TRY(C.arena.get(13, 4, &d_st));
    GVP_TRY(C.arena.get(14, K * n * n, &d_cov));
    GVP_TRY(C.arena.get(15, std::max<int64_t>(K - 1, 1) * n * n, &d_cr));
    GVP_TRY(h2d(d_d, diag, K * n * n, C.stream));
    GVP_TRY(h2d(d_o, off, (K - 1) * n * n, C.stream));
    GVP_TRY(launch_wide_marginals(1, K, n, pview(d_d, n * n, 1), pview(d_o, n * n, 1), pmview(d_cov, n * n, 1),
                                  pmview(d_cr, n * n, 1), nullptr, d_scr, d_st, d_st + 1, C.stream));
    const int st = fetch_status(C, d_st, where);
    if (st != GVP_OK) {
      set_error("belief precision at knot " + std::to_string(*where) + " is not positive definite");
      return st;
    }
    GVP_TRY(d2h(covs, d_cov, K * n * n, C.stream));
    GVP_TRY(d2h(crosses, d_cr, (K - 1) * n * n, C.stream));
    GVP_CUDA(cudaStreamSynchronize(C.stream));
    return GVP_OK;
  }
  ChainBufs b;
  GVP_TRY(upload_bt(C, diag, off, K, n, b));
  double *d_cov, *d_cr;
  GVP_TRY(C.arena.get(14, K * n * n, &d_cov));
  GVP_TRY(C.arena.get(15, std::max<int64_t>(K - 1, 1) * n * n, &d_cr));
  // log-depth cyclic reduction (one plan: the sequential sweep would be pure latency);
  // on a non-SPD pivot the sequential sweep names the reference's knot
  static const int mode = [] {  // GVP_MARGINALS=seq|cr overrides the choice (A/B measurements)
    const char* ev = std::getenv("GVP_MARGINALS");
    return !ev ? 0 : (ev[0] == 's' ? 1 : 2);
  }();
  const bool use_cr = mode == 2 || (mode == 0 && K <= kCrMaxKnots);
  int st = GVP_ERR_NOT_SPD;
  if (use_cr) {
    double* d_ws;
    GVP_TRY(C.arena.get(16, (size_t)cr_workspace_doubles(1, K, n), &d_ws));
    GVP_TRY(launch_cr_marginals(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), pmview(d_cov, n * n, 1),
                                pmview(d_cr, n * n, 1), d_ws, b.st, b.st + 1, C.stream));
    st = fetch_status(C, b.st, where);
  }
  if (st != GVP_OK) {
    GVP_TRY(launch_marginals(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1),
                             pmview(d_cov, n * n, 1), pmview(d_cr, n * n, 1), nullptr, b.st,
                             b.st + 1, b.scr, nullptr, C.stream));
    st = fetch_status(C, b.st, where);
  }
  if (st != GVP_OK) {
    set_error("belief precision at knot " + std::to_string(*where) + " is not positive definite");
    return st;
  }
  GVP_TRY(d2h(covs, d_cov, K * n * n, C.stream));
  GVP_TRY(d2h(crosses, d_cr, (K - 1) * n * n, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  return GVP_OK;
}

extern "C" int gvp_gbp_mean_solve(const double* diag, const double* off, const double* info,
                                  int64_t nblocks, int32_t n, double* out, int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  if (nblocks < 1) return set_error("need at least one block"), GVP_ERR_ARG;
  const int64_t K = nblocks;
  ChainBufs b;
  if (n >= kWideMin) {
    GVP_TRY(C.arena.get(10, K * n * n, &b.diag));
    GVP_TRY(C.arena.get(11, std::max<int64_t>(K - 1, 1) * n * n, &b.off));
    GVP_TRY(C.arena.get(12, (size_t)wide_scratch_doubles(1, K, n), &b.scr));
    GVP_TRY(C.arena.get(13, 4, &b.st));
    GVP_TRY(h2d(b.diag, diag, K * n * n, C.stream));
    GVP_TRY(h2d(b.off, off, (K - 1) * n * n, C.stream));
  } else {
    GVP_TRY(upload_bt(C, diag, off, K, n, b));
  }
  double *d_eta, *d_out;
  GVP_TRY(C.arena.get(14, K * n, &d_eta));
  GVP_TRY(C.arena.get(15, K * n, &d_out));
  GVP_TRY(h2d(d_eta, info, K * n, C.stream));
  if (n >= kWideMin)
    GVP_TRY(launch_wide_mean_solve(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), pview(d_eta, n, 1),
                                   pmview(d_out, n, 1), b.scr, b.st, b.st + 1, C.stream));
  else
  GVP_TRY(launch_mean_solve(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1),
                            pview(d_eta, n, 1), pmview(d_out, n, 1), b.st, b.st + 1, b.scr,
                            C.stream));
  const int st = fetch_status(C, b.st, where);
  if (st != GVP_OK) {
    set_error("pivot block " + std::to_string(*where) + " is not positive definite");
    return st;
  }
  GVP_TRY(d2h(out, d_out, K * n, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  return GVP_OK;
}

extern "C" int gvp_logdet_block_tridiag(const double* diag, const double* off, int64_t nblocks,
                                        int32_t n, double* out, int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  if (nblocks < 1) return set_error("need at least one block"), GVP_ERR_ARG;
  const int64_t K = nblocks;
  ChainBufs b;
  GVP_TRY(upload_bt(C, diag, off, K, n, b, 0));
  double* d_out;
  GVP_TRY(C.arena.get(14, 1, &d_out));
  if (n >= kWideMin)
    GVP_TRY(launch_wide_logdet(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), d_out, nullptr, b.st,
                               b.st + 1, C.stream));
  else
  GVP_TRY(launch_logdet_fwd(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), d_out, b.st,
                            b.st + 1, nullptr, C.stream));
  const int st = fetch_status(C, b.st, where);
  if (st != GVP_OK) {
    set_error("pivot block " + std::to_string(*where) + " is not positive definite");
    return st;
  }
  GVP_TRY(d2h(out, d_out, 1, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  return GVP_OK;
}

// forward_schur_chols (blocktri.py:151-165): Cholesky factors of the forward
// Schur pivots S_0 = D_0, S_i = D_i - W'W, W = L_{i-1}^-1 U_{i-1}; chols (K, n, n)
extern "C" int gvp_forward_schur_chols(const double* diag, const double* off, int64_t nblocks, int32_t n,
                                       double* chols, int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  if (nblocks < 1 || !chols) return set_error("need at least one block"), GVP_ERR_ARG;
  const int64_t K = nblocks;
  ChainBufs b;
  GVP_TRY(upload_bt(C, diag, off, K, n, b, 0));
  double *d_out, *d_ch;
  GVP_TRY(C.arena.get(14, 1, &d_out));
  GVP_TRY(C.arena.get(15, (size_t)K * n * n, &d_ch));
  if (n >= kWideMin)
    GVP_TRY(launch_wide_logdet(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), d_out, d_ch, b.st,
                               b.st + 1, C.stream));
  else
  GVP_TRY(launch_logdet_fwd(1, K, n, pview(b.diag, n * n, 1), pview(b.off, n * n, 1), d_out, b.st,
                            b.st + 1, d_ch, C.stream));
  const int st = fetch_status(C, b.st, where);
  if (st != GVP_OK) {
    set_error("pivot block " + std::to_string(*where) + " is not positive definite");
    return st;
  }
  GVP_TRY(d2h(chols, d_ch, (size_t)K * n * n, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  return GVP_OK;
}

namespace {
// uploads of one plan's step problem; returns device StepProblem
struct StepBufs {
  double *mean, *diag, *off, *kdiag, *koff, *info, *gmu, *gdiag, *goff, *scr;
  double *omean, *odiag, *ooff, *covs, *crosses, *scal;  // scal: beta, kl, ld_next, shift, temp, ld_cur, beta_fixed
  double* plog;
  int *st, *np;
};
int upload_step(Context& C, const double* mean, const double* diag, const double* off,
                const double* kdiag, const double* koff, const double* info, const double* g_mu,
                const double* gdiag, const double* goff, int64_t K, int n, int max_probes,
                StepBufs& b, StepProblem& pb) {
  cudaStream_t s = C.stream;
  const int64_t B2 = (int64_t)n * n, K1 = std::max<int64_t>(K - 1, 1);
  GVP_TRY(C.arena.get(20, K * n, &b.mean));
  GVP_TRY(C.arena.get(21, K * B2, &b.diag));
  GVP_TRY(C.arena.get(22, K1 * B2, &b.off));
  GVP_TRY(C.arena.get(23, K * B2, &b.kdiag));
  GVP_TRY(C.arena.get(24, K1 * B2, &b.koff));
  GVP_TRY(C.arena.get(25, K * n, &b.info));
  GVP_TRY(C.arena.get(26, K * n, &b.gmu));
  GVP_TRY(C.arena.get(27, K * B2, &b.gdiag));
  GVP_TRY(C.arena.get(28, K1 * B2, &b.goff));
  GVP_TRY(C.arena.get(29, (size_t)chain_scratch_doubles(1, K, n, 1), &b.scr));
  GVP_TRY(C.arena.get(30, K * n, &b.omean));
  GVP_TRY(C.arena.get(31, K * B2, &b.odiag));
  GVP_TRY(C.arena.get(32, K1 * B2, &b.ooff));
  GVP_TRY(C.arena.get(33, K * B2, &b.covs));
  GVP_TRY(C.arena.get(34, K1 * B2, &b.crosses));
  GVP_TRY(C.arena.get(35, 16, &b.scal));
  GVP_TRY(C.arena.get(36, std::max(max_probes, 1) * 3, &b.plog));
  GVP_TRY(C.arena.get(37, 4, &b.st));
  b.np = b.st + 2;
  GVP_TRY(h2d(b.mean, mean, K * n, s));
  GVP_TRY(h2d(b.diag, diag, K * B2, s));
  GVP_TRY(h2d(b.off, off, (K - 1) * B2, s));
  GVP_TRY(h2d(b.kdiag, kdiag, K * B2, s));
  GVP_TRY(h2d(b.koff, koff, (K - 1) * B2, s));
  GVP_TRY(h2d(b.info, info, K * n, s));
  GVP_TRY(h2d(b.gmu, g_mu, K * n, s));
  GVP_TRY(h2d(b.gdiag, gdiag, K * B2, s));
  // unary factors leave the gradient's off blocks zero (factors.py:228-255): an
  // all-zero goff is neither uploaded nor read (the same bits: 0 * 2/T + x = x)
  const bool has_goff = goff && !all_zero(goff, (K - 1) * B2);
  if (has_goff) GVP_TRY(h2d(b.goff, goff, (K - 1) * B2, s));
  pb = StepProblem{pview(b.mean, n, 1),  pview(b.diag, B2, 1), pview(b.off, B2, 1),
                   pview(b.kdiag, B2, 1), pview(b.koff, B2, 1), pview(b.info, n, 1),
                   pview(b.gmu, n, 1),   pview(b.gdiag, B2, 1), pview(b.goff, B2, 1),
                   has_goff,             pview(b.mean, n, 1),   false};
  return GVP_OK;
}
}  // namespace

namespace {
// wide blocks (9 <= n <= 32): one CTA per plan, probe slots on warp pairs
// (wide_kernels.cu). fixed: proximal_update at beta; else select_step_size.
int wide_step_call(Context& C, const double* mean, const double* diag, const double* off, const double* kdiag,
                   const double* koff, const double* info, const double* g_mu, const double* gdiag,
                   const double* goff, int64_t K, int n, bool fixed, double beta_fixed, double temp,
                   double kl_bound, double beta_min, double beta_max, double* beta, double* kl, double* out_mean,
                   double* out_diag, double* out_off, double* covs, double* crosses, double* probe_log,
                   int max_probes, int* nprobes, int64_t* where) {
  const int64_t B2 = (int64_t)n * n;
  cudaStream_t s = C.stream;
  StepBufs b;
  StepProblem pb;
  GVP_TRY(upload_step(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, K, n,
                      probe_log ? max_probes : 0, b, pb));
  double* wscr;
  GVP_TRY(C.arena.get(60, (size_t)wide_scratch_doubles(1, K, n), &wscr));
  // scal: 0 beta (in: previous / fixed, out: accepted), 1 kl, 2 ld_next, 4 temp, 5 ld_cur
  const double init[6] = {fixed ? beta_fixed : NAN, 0.0, 0.0, 0.0, temp, std::isfinite(C.ld_in) ? C.ld_in : 0.0};
  GVP_TRY(h2d(b.scal, init, 6, s));
  if (!fixed && !std::isfinite(C.ld_in)) {  // log det of the current precision (kl_joint's logdet_cur)
    GVP_TRY(launch_wide_logdet(1, K, n, pb.diag, pb.off, b.scal + 5, nullptr, b.st, b.st + 1, s));
    int64_t w0 = -1;
    if (fetch_status(C, b.st, &w0) != GVP_OK) {
      if (where) *where = w0;
      set_error("pivot block " + std::to_string(w0) + " is not positive definite");
      return GVP_ERR_NOT_SPD;
    }
  }
  WideStep q{};
  q.nplans = 1; q.K = K; q.n = n;
  q.mean = pb.mean; q.diag = pb.diag; q.off = pb.off; q.kdiag = pb.kdiag; q.koff = pb.koff; q.info = pb.info;
  q.gmu = pb.gmu; q.gdiag = pb.gdiag; q.goff = pb.goff; q.has_goff = pb.has_goff;
  q.o_mean = pmview(b.omean, n, 1); q.o_diag = pmview(b.odiag, B2, 1); q.o_off = pmview(b.ooff, B2, 1);
  q.o_cov = pmview(b.covs, B2, 1); q.o_cross = pmview(b.crosses, B2, 1);
  q.active = nullptr; q.status = b.st; q.where = b.st + 1; q.nprobes = b.np;
  q.beta = b.scal; q.kl = b.scal + 1; q.ld_next = b.scal + 2; q.temp = b.scal + 4; q.ld_cur = b.scal + 5;
  q.kl_bound = kl_bound; q.beta_min = beta_min; q.beta_max = beta_max;
  q.probe_log = probe_log ? b.plog : nullptr; q.max_probes = max_probes;
  q.scratch = wscr; q.fixed = fixed;
  GVP_TRY(launch_wide_step(q, s));
  int stw[3];
  GVP_TRY(d2h(stw, b.st, 3, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  if (nprobes) *nprobes = fixed ? 0 : stw[2];
  if (probe_log && !fixed && stw[2] > 0) {
    GVP_TRY(d2h(probe_log, b.plog, (size_t)std::min(stw[2], max_probes) * 3, s));
    GVP_CUDA(cudaStreamSynchronize(s));
  }
  if (stw[0] != GVP_OK) {
    if (where) *where = stw[1];
    if (stw[0] == GVP_ERR_NO_FEASIBLE_STEP) {
      char msg[160];
      std::snprintf(msg, sizeof msg, "no feasible step size at beta_min=%g (KL bound %g)", beta_min, kl_bound);
      set_error(msg);
    } else {
      set_error("pivot block " + std::to_string(stw[1] & ~GVP_WHERE_MEAN_SOLVE_BIAS) + " is not positive definite");
    }
    return stw[0];
  }
  double sc[3];
  GVP_TRY(d2h(sc, b.scal, 3, s));
  GVP_TRY(d2h(out_mean, b.omean, K * n, s));
  GVP_TRY(d2h(out_diag, b.odiag, K * B2, s));
  GVP_TRY(d2h(out_off, b.ooff, (K - 1) * B2, s));
  if (covs) GVP_TRY(d2h(covs, b.covs, K * B2, s));
  if (crosses) GVP_TRY(d2h(crosses, b.crosses, (K - 1) * B2, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  if (beta) *beta = sc[0];
  if (kl) *kl = sc[1];
  if (!fixed) C.ld_out = sc[2];
  if (where) *where = -1;
  return GVP_OK;
}
}  // namespace

extern "C" int gvp_proximal_update(const double* mean, const double* diag, const double* off,
                                   const double* kdiag, const double* koff, const double* info,
                                   const double* g_mu, const double* gdiag, const double* goff,
                                   int64_t nblocks, int32_t n, double beta, double temp,
                                   double* out_mean, double* out_diag, double* out_off,
                                   int64_t* where) {
  if (!(beta > 0)) return set_error("beta must be positive"), GVP_ERR_ARG;
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  const int64_t K = nblocks, B2 = (int64_t)n * n;
  if (n >= kWideMin)
    return wide_step_call(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, K, n, true, beta, temp, 0.0,
                          0.0, 0.0, nullptr, nullptr, out_mean, out_diag, out_off, nullptr, nullptr, nullptr, 0,
                          nullptr, where);
  StepBufs b;
  StepProblem pb;
  GVP_TRY(upload_step(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, K, n, 0, b, pb));
  const double sc[2] = {temp, beta};
  GVP_TRY(h2d(b.scal + 4, sc, 2, C.stream));
  StepParams pr{b.scal + 4, nullptr, 0, 0, 0, 1, true, b.scal + 5};
  StepOut out{pmview(b.omean, n, 1), pmview(b.odiag, B2, 1), pmview(b.ooff, B2, 1),
              pmview(b.covs, B2, 1), pmview(b.crosses, B2, 1), nullptr, nullptr, nullptr,
              nullptr, nullptr, nullptr, 0, nullptr, b.st, b.st + 1};
  GVP_TRY(launch_select_step(1, K, n, pb, pr, out, b.scr, nullptr, C.stream));
  const int st = fetch_status(C, b.st, where);
  if (st != GVP_OK) {
    set_error("pivot block " + std::to_string(*where) + " is not positive definite");
    return st;
  }
  GVP_TRY(d2h(out_mean, b.omean, K * n, C.stream));
  GVP_TRY(d2h(out_diag, b.odiag, K * B2, C.stream));
  GVP_TRY(d2h(out_off, b.ooff, (K - 1) * B2, C.stream));
  GVP_CUDA(cudaStreamSynchronize(C.stream));
  return GVP_OK;
}

// general-layout fallback (full blocks, one thread, pairwise-factor off
// gradients and non-symmetric diagonal blocks allowed): chain_kernels.cu
static int select_step_size_v1(const double* mean, const double* diag, const double* off,
                               const double* kdiag, const double* koff, const double* info,
                               const double* g_mu, const double* gdiag, const double* goff,
                               int64_t nblocks, int32_t n, double temp, double kl_bound,
                               double beta_min, double beta_max, double* beta, double* kl,
                               double* out_mean, double* out_diag, double* out_off, double* covs,
                               double* crosses, double* probe_log, int32_t max_probes,
                               int32_t* nprobes, int64_t* where) {
  Context& C = ctx();
  const int64_t K = nblocks, B2 = (int64_t)n * n;
  StepBufs b;
  StepProblem pb;
  GVP_TRY(upload_step(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, K, n,
                      probe_log ? max_probes : 0, b, pb));
  cudaStream_t s = C.stream;
  // log det of the current precision, from the same backward Schur pivots the
  // probes use for the candidate (consistent KL)
  GVP_TRY(launch_marginals(1, K, n, pb.diag, pb.off, pmview(b.covs, B2, 1),
                           pmview(b.crosses, B2, 1), b.scal + 5, b.st, b.st + 1, b.scr, nullptr,
                           s));
  int64_t w0 = -1;
  int st = fetch_status(C, b.st, &w0);
  if (st != GVP_OK) {
    if (where) *where = w0;
    set_error("current precision is not positive definite at knot " + std::to_string(w0));
    return st;
  }
  GVP_TRY(h2d(b.scal + 4, &temp, 1, s));
  StepParams pr{b.scal + 4, b.scal + 5, kl_bound, beta_min, beta_max, 1, false, nullptr};
  StepOut out{pmview(b.omean, n, 1),
              pmview(b.odiag, B2, 1),
              pmview(b.ooff, B2, 1),
              pmview(b.covs, B2, 1),
              pmview(b.crosses, B2, 1),
              b.scal + 0,
              b.scal + 1,
              b.scal + 2,
              b.scal + 3,
              nullptr,
              probe_log ? b.plog : nullptr,
              max_probes,
              b.np,
              b.st,
              b.st + 1};
  GVP_TRY(launch_select_step(1, K, n, pb, pr, out, b.scr, nullptr, s));
  int stw[3];
  GVP_TRY(d2h(stw, b.st, 3, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  if (nprobes) *nprobes = stw[2];
  if (probe_log && stw[2] > 0)
    GVP_TRY(d2h(probe_log, b.plog, (size_t)std::min(stw[2], max_probes) * 3, s));
  if (stw[0] != GVP_OK) {
    if (where) *where = stw[1];
    GVP_CUDA(cudaStreamSynchronize(s));
    if (stw[0] == GVP_ERR_NO_FEASIBLE_STEP) {
      char msg[160];
      std::snprintf(msg, sizeof msg, "no feasible step size at beta_min=%g (KL bound %g)", beta_min,
                    kl_bound);
      set_error(msg);
    } else {
      set_error("pivot block " + std::to_string(stw[1] & ~GVP_WHERE_MEAN_SOLVE_BIAS) +
                " is not positive definite");
    }
    return stw[0];
  }
  double sc[3];
  GVP_TRY(d2h(sc, b.scal, 3, s));
  GVP_TRY(d2h(out_mean, b.omean, K * n, s));
  GVP_TRY(d2h(out_diag, b.odiag, K * B2, s));
  GVP_TRY(d2h(out_off, b.ooff, (K - 1) * B2, s));
  GVP_TRY(d2h(covs, b.covs, K * B2, s));
  GVP_TRY(d2h(crosses, b.crosses, (K - 1) * B2, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  *beta = sc[0];
  *kl = sc[1];
  if (where) *where = -1;
  return GVP_OK;
}

extern "C" int gvp_set_step_lanes(int32_t lanes) {
  if (lanes != 1 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16) {
    set_error("lanes must be 1, 2, 4, 8 or 16");
    return GVP_ERR_ARG;
  }
  g_step_lanes = lanes;
  return GVP_OK;
}

static int select_step_impl(Context& C, const double* mean, const double* diag, const double* off,
                            const double* kdiag, const double* koff, const double* info,
                            const double* g_mu, const double* gdiag, const double* goff,
                            int64_t nblocks, int32_t n, double temp, double kl_bound,
                            double beta_min, double beta_max, double* beta, double* kl,
                            double* out_mean, double* out_diag, double* out_off,
                            double* covs, double* crosses, double* probe_log,
                            int32_t max_probes, int32_t* nprobes, int64_t* where);

extern "C" int gvp_select_step_size(const double* mean, const double* diag, const double* off,
                                    const double* kdiag, const double* koff, const double* info,
                                    const double* g_mu, const double* gdiag, const double* goff,
                                    int64_t nblocks, int32_t n, double temp, double kl_bound,
                                    double beta_min, double beta_max, double* beta, double* kl,
                                    double* out_mean, double* out_diag, double* out_off,
                                    double* covs, double* crosses, double* probe_log,
                                    int32_t max_probes, int32_t* nprobes, int64_t* where) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  C.ld_in = NAN;
  return select_step_impl(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, nblocks, n, temp, kl_bound,
                          beta_min, beta_max, beta, kl, out_mean, out_diag, out_off, covs, crosses, probe_log,
                          max_probes, nprobes, where);
}

extern "C" int gvp_select_step_size_ld(const double* mean, const double* diag, const double* off,
                                       const double* kdiag, const double* koff, const double* info,
                                       const double* g_mu, const double* gdiag, const double* goff,
                                       int64_t nblocks, int32_t n, double temp, double kl_bound,
                                       double beta_min, double beta_max, double* beta, double* kl,
                                       double* out_mean, double* out_diag, double* out_off,
                                       double* covs, double* crosses, double* probe_log,
                                       int32_t max_probes, int32_t* nprobes, int64_t* where, double ld_cur,
                                       double* ld_next) {
  Context& C = ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  C.ld_in = ld_cur;
  C.ld_out = NAN;
  const int r = select_step_impl(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, nblocks, n, temp,
                                 kl_bound, beta_min, beta_max, beta, kl, out_mean, out_diag, out_off, covs, crosses,
                                 probe_log, max_probes, nprobes, where);
  C.ld_in = NAN;
  if (ld_next) *ld_next = C.ld_out;
  return r;
}

static int select_step_impl(Context& C, const double* mean, const double* diag, const double* off,
                            const double* kdiag, const double* koff, const double* info,
                            const double* g_mu, const double* gdiag, const double* goff,
                            int64_t nblocks, int32_t n, double temp, double kl_bound,
                            double beta_min, double beta_max, double* beta, double* kl,
                            double* out_mean, double* out_diag, double* out_off,
                            double* covs, double* crosses, double* probe_log,
                            int32_t max_probes, int32_t* nprobes, int64_t* where) {
  GVP_TRY(C.init());
  GVP_TRY(check_chain_n(n));
  if (n >= kWideMin)
    return wide_step_call(C, mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, nblocks, n, false, 0.0, temp,
                          kl_bound, beta_min, beta_max, beta, kl, out_mean, out_diag, out_off, covs, crosses,
                          probe_log, max_probes, nprobes, where);
  const int64_t K = nblocks, N2 = (int64_t)n * n, K1 = std::max<int64_t>(K - 1, 0);
  const bool v2_ok = (n == 2 || n == 4 || n == 6) && blocks_symmetric(diag, K, n) &&
                     blocks_symmetric(kdiag, K, n) && blocks_symmetric(gdiag, K, n) &&
                     all_zero(goff, K1 * N2);
  if (!v2_ok)
    return select_step_size_v1(mean, diag, off, kdiag, koff, info, g_mu, gdiag, goff, nblocks, n,
                               temp, kl_bound, beta_min, beta_max, beta, kl, out_mean, out_diag,
                               out_off, covs, crosses, probe_log, max_probes, nprobes, where);
  // ---- packed layout, TMA-staged probe + commit kernels (step_select.cu).
  // The step kernel wants an even plan stride: the plan goes in column 0 of
  // 2-wide arrays (column 1 is a copy), the prior is the 2-wide shared prior.
  cudaStream_t s = C.stream;
  const int T = n * (n + 1) / 2;
  const int L = g_step_lanes;
  auto wide = [](const double* src, int64_t rows) {
    std::vector<double> w((size_t)(2 * rows));
    for (int64_t r = 0; r < rows; ++r) w[2 * r] = w[2 * r + 1] = src[r];
    return w;
  };
  const std::vector<double> ld_p = pack_lower(diag, K, n), kd_p = pack_lower(kdiag, K, n),
                            gd_p = pack_lower(gdiag, K, n);
  double *ld, *lo, *kd, *ko, *gd, *g, *eta, *v, *mu, *omu, *old_, *olo, *ocov, *ocr, *ov, *scal,
      *plog, *scr;
  int* st;
  const int64_t K1a = std::max<int64_t>(K1, 1);
  GVP_TRY(C.arena.get(40, 2 * K * T, &ld));
  GVP_TRY(C.arena.get(41, 2 * K1a * N2, &lo));
  GVP_TRY(C.arena.get(42, 2 * K * T, &kd));
  GVP_TRY(C.arena.get(43, 2 * K1a * N2, &ko));
  GVP_TRY(C.arena.get(44, 2 * K * T, &gd));
  GVP_TRY(C.arena.get(45, 2 * K * n, &g));
  GVP_TRY(C.arena.get(46, 2 * K * n, &eta));
  GVP_TRY(C.arena.get(47, 2 * K * n, &v));
  GVP_TRY(C.arena.get(48, 2 * K * n, &mu));
  GVP_TRY(C.arena.get(49, 2 * K * n, &omu));
  GVP_TRY(C.arena.get(50, 2 * K * T, &old_));
  GVP_TRY(C.arena.get(51, 2 * K1a * N2, &olo));
  GVP_TRY(C.arena.get(52, 2 * K * T, &ocov));
  GVP_TRY(C.arena.get(53, 2 * K1a * N2, &ocr));
  GVP_TRY(C.arena.get(54, 2 * K * n, &ov));
  GVP_TRY(C.arena.get(55, 16, &scal));
  GVP_TRY(C.arena.get(56, std::max(max_probes, 1) * 3 * 2, &plog));
  GVP_TRY(C.arena.get(57, (size_t)std::max(step_scratch_doubles(2, K, n, L), 2 * K * T), &scr));
  GVP_TRY(C.arena.get(58, 8, &st));
  {
    const auto w_ld = wide(ld_p.data(), K * T), w_lo = wide(off, K1 * N2),
               w_kd = wide(kd_p.data(), K * T), w_ko = wide(koff, K1 * N2),
               w_gd = wide(gd_p.data(), K * T), w_g = wide(g_mu, K * n), w_eta = wide(info, K * n),
               w_mu = wide(mean, K * n);
    GVP_TRY(h2d(ld, w_ld.data(), w_ld.size(), s));
    GVP_TRY(h2d(lo, w_lo.data(), w_lo.size(), s));
    GVP_TRY(h2d(kd, w_kd.data(), w_kd.size(), s));
    GVP_TRY(h2d(ko, w_ko.data(), w_ko.size(), s));
    GVP_TRY(h2d(gd, w_gd.data(), w_gd.size(), s));
    GVP_TRY(h2d(g, w_g.data(), w_g.size(), s));
    GVP_TRY(h2d(eta, w_eta.data(), w_eta.size(), s));
    GVP_TRY(h2d(mu, w_mu.data(), w_mu.size(), s));
    const double tt[2] = {temp, temp};
    GVP_TRY(h2d(scal + 8, tt, 2, s));
    const double nan2[2] = {NAN, NAN};  // no previous beta to aim the speculation at
    GVP_TRY(h2d(scal, nan2, 2, s));
    GVP_CUDA(cudaStreamSynchronize(s));
  }
  // rhs piece Lambda mu; the current precision's SPD check (backward sweep) and
  // its log det by the probes' own forward Schur recursion (kl_joint's
  // logdet_cur: the KL is the difference of two nearby log dets, so both come
  // from the same recursion)
  GVP_TRY(launch_lam_mu(2, K, n, 2, ld, lo, mu, v, s));
  GVP_TRY(launch_marginals_packed(1, K, n, 2, ld, lo, ocov, ocr, scal + 10, st, st + 1, scr,
                                  nullptr, s));
  if (std::isfinite(C.ld_in)) {
    GVP_TRY(h2d(scal + 10, &C.ld_in, 1, s));
  } else {
    GVP_TRY(launch_logdet_fwd_packed(1, K, n, 2, ld, lo, scal + 10, nullptr, st, st + 1, s));
  }
  int64_t w0 = -1;
  if (fetch_status(C, st, &w0) != GVP_OK) {
    if (where) *where = w0;
    set_error("current precision is not positive definite at knot " + std::to_string(w0));
    return GVP_ERR_NOT_SPD;
  }
  V2Launch q{};
  q.nplans = 1; q.K = K; q.n = n; q.Bp = 2; q.lanes = L;
  q.ld = ld; q.lo = lo; q.kd = kd; q.ko = ko; q.gd = gd; q.g = g; q.eta = eta; q.v = v;
  q.mu = mu; q.pmean = mu; q.kshared = true;
  q.o_mu = omu; q.o_ld = old_; q.o_lo = olo; q.o_cov = ocov; q.o_cr = ocr; q.o_v = ov;
  q.beta = scal; q.kl = scal + 2; q.ld_next = scal + 4; q.shift = scal + 6; q.prior_cost = nullptr;
  q.temp = scal + 8; q.ld_cur = scal + 10;
  q.kl_bound = kl_bound; q.beta_min = beta_min; q.beta_max = beta_max;
  q.status = st; q.where = st + 2;
  q.probe_log = probe_log ? plog : nullptr; q.max_probes = max_probes; q.nprobes = st + 4;
  q.scratch = scr; q.active = nullptr;
  q.search_kl = true; q.fixkl = nullptr;  // step.kl: the accepted probe's KL
  GVP_TRY(launch_select_step_v2(q, s));
  int stv[5];
  GVP_TRY(d2h(stv, st, 5, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  const int stw[3] = {stv[0], stv[2], stv[4]};
  if (nprobes) *nprobes = stw[2];
  if (probe_log && stw[2] > 0) {
    GVP_TRY(d2h(probe_log, plog, (size_t)std::min(stw[2], max_probes) * 3, s));
    GVP_CUDA(cudaStreamSynchronize(s));
  }
  if (stw[0] != GVP_OK) {
    if (where) *where = stw[1];
    if (stw[0] == GVP_ERR_NO_FEASIBLE_STEP) {
      char msg[160];
      std::snprintf(msg, sizeof msg, "no feasible step size at beta_min=%g (KL bound %g)", beta_min,
                    kl_bound);
      set_error(msg);
    } else {
      set_error("pivot block " + std::to_string(stw[1] & ~GVP_WHERE_MEAN_SOLVE_BIAS) +
                " is not positive definite");
    }
    return stw[0];
  }
  double sc[5];
  std::vector<double> ldo((size_t)(K * T)), covo((size_t)(K * T));
  auto narrow = [&](double* dst, const double* src, int64_t rows) -> int {
    if (rows > 0)
      GVP_CUDA(cudaMemcpy2DAsync(dst, 8, src, 16, 8, rows, cudaMemcpyDeviceToHost, s));
    return GVP_OK;
  };
  GVP_TRY(d2h(sc, scal, 5, s));
  GVP_TRY(narrow(out_mean, omu, K * n));
  GVP_TRY(narrow(ldo.data(), old_, K * T));
  GVP_TRY(narrow(out_off, olo, K1 * N2));
  GVP_TRY(narrow(covo.data(), ocov, K * T));
  GVP_TRY(narrow(crosses, ocr, K1 * N2));
  GVP_CUDA(cudaStreamSynchronize(s));
  unpack_sym(ldo.data(), K, n, out_diag);
  unpack_sym(covo.data(), K, n, covs);
  *beta = sc[0];
  *kl = sc[2];
  C.ld_out = sc[4];
  if (where) *where = -1;
  return GVP_OK;
}

// =================================================================== batched device kernels
extern "C" int64_t gvp_chain_scratch_doubles(int32_t nplans, int64_t nblocks, int32_t n,
                                             int32_t lanes) {
  return chain_scratch_doubles(nplans, nblocks, n, lanes);
}

extern "C" int gvp_gbp_marginals_dev(int32_t nplans, int64_t nblocks, int32_t n,
                                     const double* diag, const double* off, double* covs,
                                     double* crosses, double* logdet, int32_t* status,
                                     int32_t* where, double* scratch, void* stream) {
  GVP_TRY(check_n(n));
  const int64_t B2 = (int64_t)n * n;
  return launch_marginals(nplans, nblocks, n, pview(diag, B2, nplans), pview(off, B2, nplans),
                          pmview(covs, B2, nplans), pmview(crosses, B2, nplans), logdet, status,
                          where, scratch, nullptr, (cudaStream_t)stream);
}
