// select_step_size (optimizer.py:188-231) for a batch of plans: the bisection
// (one-pass probes, step_probe.cu) followed by the commit of each plan's
// accepted beta (exact two-pass, commit.cu). Also the step scratch sizing.
#include <cuda_runtime.h>

#include <algorithm>

#include "gvp_internal.cuh"
#include "step_common.cuh"

namespace gvp {

int64_t step_plan_stride(int nplans) { return std::max<int64_t>(2, ((int64_t)nplans + 1) & ~1LL); }

// commit scratch (one column per plan: Phi^-1 | Li | y per knot) followed by
// the probe's residual e (K x n per plan); independent of the lane count
int64_t step_scratch_doubles(int nplans, int64_t K, int n, int lanes) {
  (void)lanes;
  return std::max<int64_t>(1, probe_residual_offset(nplans, K, n) + K * n * step_plan_stride(nplans));
}

// bisection (L candidate lanes per plan): the accepted beta of each plan -> q.beta
int launch_select_bisect(const V2Launch& q, cudaStream_t s) {
  if (q.nplans == 0 || q.K == 0) return GVP_OK;
  const int L = q.lanes;
  if (L != 1 && L != 2 && L != 4 && L != 8 && L != 16) {
    set_error("lanes must be 1, 2, 4, 8 or 16");
    return GVP_ERR_ARG;
  }
  if (q.Bp % 2 || q.Bp < 2) {
    set_error("plan stride must be even (step_plan_stride)");
    return GVP_ERR_ARG;
  }
  return launch_probe(q, L, s);
}

// the commit of the accepted beta: next iterate, marginals, KL, log det, costs
int launch_select_commit(const V2Launch& q, cudaStream_t s) {
  if (q.nplans == 0 || q.K == 0) return GVP_OK;
  return launch_commit_split(q, s);
}

int launch_select_step_v2(const V2Launch& q, cudaStream_t s) {
  int r = launch_select_bisect(q, s);
  if (r) return r;
  return launch_select_commit(q, s);
}

}  // namespace gvp
