// Shared pieces of the TMA-staged step kernels (step_probe.cu: one-pass
// bisection probes; commit.cu: two-pass commit): mbarrier/TMA
// helpers, packed Cholesky, the per-plan bisection state machine and the
// tensor-map encoder.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "gvp_internal.cuh"

namespace gvp {
namespace v3 {

// TMA ring depth: 8 stages when they fit in 96 KB, else 4. Each stage slot is
// consumed exactly once per step in step order, so the mbarrier phase parity
// of step s is (s / NS) & 1.
constexpr int ring_stages(int stage_doubles) { return stage_doubles * 8 <= 12288 ? 8 : 4; }
constexpr int kMaxStages = 8;

template <int N> constexpr int T_ = N * (N + 1) / 2;

GVP_DEV uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
GVP_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(bar)), "r"(count) : "memory");
}
GVP_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}
GVP_DEV bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(saddr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
GVP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
GVP_DEV void tma3(double* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          saddr(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar))
      : "memory");
}
GVP_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }

// row starts rounded so every TMA box lands on a 128-byte boundary
constexpr int cx_round(int x, int m) { return (x + m - 1) / m * m; }
constexpr int cx_gran(int w) { return w % 16 == 0 ? 1 : w % 8 == 0 ? 2 : w % 4 == 0 ? 4 : w % 2 == 0 ? 8 : 16; }

// ------------------------------------------------------------ packed algebra
template <int N>
GVP_DEV bool chol_inv(const double (&A)[T_<N>], double (&Li)[T_<N>], double& pivprod) {
  double L[T_<N>], inv[N];
  bool ok = true;
  pivprod = 1.0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double s = A[tri_idx(j, j)];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= L[tri_idx(j, k)] * L[tri_idx(j, k)];
    ok = ok && (s > 0.0);
    const double r = rsqrt_nb(s);
    const double d = s * r;
    ok = ok && (d > kPivotFloor);
    L[tri_idx(j, j)] = d;
    inv[j] = r;
    pivprod *= d;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double t = A[tri_idx(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[tri_idx(i, k)] * L[tri_idx(j, k)];
      L[tri_idx(i, j)] = t * r;
    }
  }
#pragma unroll
  for (int c = 0; c < N; ++c) {
    Li[tri_idx(c, c)] = inv[c];
#pragma unroll
    for (int r = c + 1; r < N; ++r) {
      double t = 0.0;
#pragma unroll
      for (int k = c; k < r; ++k) t += L[tri_idx(r, k)] * Li[tri_idx(k, c)];
      Li[tri_idx(r, c)] = -t * inv[r];
    }
  }
  return ok;
}
template <int N>
GVP_DEV double sym_at(const double (&A)[T_<N>], int r, int c) {
  return r >= c ? A[tri_idx(r, c)] : A[tri_idx(c, r)];
}

// bisection state of one plan, kept in shared memory: the CTA's lane slots
// are re-dealt among its still-searching plans every round
struct PlanSt {
  double lo, hi, best, kl_lo, kl_hi, prev, temp, ldc;
  int phase, nprobe;
  double ld_best;  // forward-Schur log det of Lambda'(best) (the probe's)
};
static_assert(sizeof(PlanSt) <= 80, "PlanSt must fit 10 doubles");

// ------------------------------------------------------------ bisection search
// (shared by the bisection kernels and the commit kernel). A CTA's 32 lane
// slots are re-dealt every round among its still-searching plans (k = 32 /
// n_active contiguous slots each, in plan order); each slot probes one
// candidate beta; afterwards one thread per plan replays the reference's
// sequential bisection (optimizer.py:188-231) over the round's probes.

// one thread per plan loads its state (phase 0 first round, 1 beta_min
// pending, 2 bisect, 3 commit, 4 done)
template <class A>
GVP_DEV void search_init(const A& a, PlanSt* pst, int P, int64_t b0, bool commit, int tid) {
  if (tid >= P) return;
  const int64_t bb = b0 + tid;
  const bool ok = (bb < a.B) && (!a.active || a.active[bb]) && (!commit || a.status[bb] == GVP_OK);
  PlanSt& S = pst[tid];
  S.phase = ok ? (commit ? 3 : 0) : 4;
  S.lo = a.beta_min;
  S.hi = a.beta_max;
  S.best = (commit && ok) ? a.beta[bb] : a.beta_max;
  S.kl_lo = 0.0;
  S.kl_hi = INFINITY;
  // the previous iteration's beta (a.beta on entry; NaN = none) aims the first round
  S.prev = (!commit && ok) ? a.beta[bb] : -1.0;
  S.temp = ok ? a.temp[bb] : 1.0;
  S.ldc = ok ? a.ld_cur[bb] : 0.0;
  S.nprobe = 0;
  S.ld_best = NAN;
}

struct Pick {
  int p;        // plan column this slot serves (0 for idle slots)
  int my_rank;  // rank among active plans of plan `tid` (tid < P), else -1
  int kl;       // slots of the plan this slot serves (0: every plan is done)
  int dbase, dkl;  // first slot / slot count of plan `tid` (my_rank >= 0)
  int phase;    // phase of the served plan (4: idle slot)
  bool on, write;
  double beta;
};

// slot assignment + candidate beta of this slot for the round; kl == 0: all done
template <class A>
GVP_DEV Pick search_pick(const A& a, const PlanSt* pst, int P, int LP, int lcol, int tid, bool commit) {
  Pick k;
  k.on = k.write = false;
  k.beta = 0.0;
  int nact = 0;
  for (int j = 0; j < P; ++j) nact += pst[j].phase < 4 ? 1 : 0;
  k.kl = 0;
  k.my_rank = -1;
  k.dbase = k.dkl = 0;
  k.p = 0;
  k.phase = 4;
  if (nact == 0) return k;
  // plan rank r owns slots [r LP / nact, (r + 1) LP / nact): all LP slots in use
  auto first = [&](int r) { return r * LP / nact; };
  const int my_idx = ((lcol + 1) * nact - 1) / LP, q = lcol - first(my_idx);
  k.kl = first(my_idx + 1) - first(my_idx);
  int pj = -1;
  for (int j = 0, c = 0; j < P; ++j)
    if (pst[j].phase < 4) {
      if (c == my_idx) pj = j;
      if (j == tid) k.my_rank = c;
      ++c;
    }
  if (k.my_rank >= 0) {
    k.dbase = first(k.my_rank);
    k.dkl = first(k.my_rank + 1) - k.dbase;
  }
  if (pj < 0) return k;
  k.p = pj;
  const PlanSt& S = pst[pj];
  k.phase = S.phase;
  int qs = -1, nslots = 0;  // speculative index / count
  double l = a.beta_min, h = a.beta_max, target = -1.0;
  if (S.phase == 0) {
    if (q == 0) {
      k.on = true;
      k.beta = a.beta_max;
    } else if (q == 1) {
      k.on = true;
      k.beta = a.beta_min;
    } else {
      qs = q - 2;
      nslots = k.kl - 2;
      target = S.prev;
    }
  } else if (S.phase == 1) {
    if (q == 0) {
      k.on = true;
      k.beta = a.beta_min;
    } else {
      qs = q - 1;
      nslots = k.kl - 1;
      target = S.prev;
    }
  } else if (S.phase == 2) {
    qs = q;
    nslots = k.kl;
    l = S.lo;
    h = S.hi;
    // predicted crossing beta* (KL(beta*) = bound): log-log interpolation
    // of the bracket's KL values
    if (S.kl_lo > 0.0 && isfinite(S.kl_hi) && S.kl_hi > S.kl_lo && S.kl_lo < a.kl_bound &&
        a.kl_bound < S.kl_hi) {
      const double t = (log(a.kl_bound) - log(S.kl_lo)) / (log(S.kl_hi) - log(S.kl_lo));
      target = exp(log(l) + t * (log(h) - log(l)));
    }
  } else if (commit && S.phase == 3 && q == 0) {
    k.on = true;
    k.write = true;
    k.beta = S.best;
  }
  if (qs >= 0) {
    // Speculative slots: a complete subtree of depth dt on (up to) half of
    // them — always resolves dt levels — and the rest follow the bisection
    // path towards the predicted crossing below it. Any choice is exact:
    // the walk only uses slots whose beta equals the reference's midpoint.
    int dt = 0;
    while ((2 << dt) - 1 <= nslots / 2) ++dt;
    const int ntree = (1 << dt) - 1;
    bool valid = true;
    if (qs >= ntree && target > l && target < h) {  // path node at depth dt + (qs - ntree)
      const int depth = dt + (qs - ntree);
      for (int s2 = 0;; ++s2) {
        if (!((h - l) > 1e-3 * h)) {
          valid = false;
          break;
        }
        const double mid = 0.5 * (l + h);
        if (s2 == depth) break;
        if (mid <= target) l = mid; else h = mid;
      }
    } else {  // BFS node qs + 1 of the subtree
      const int kk = qs + 1;
      const int depth = 31 - __clz(kk);
      for (int lev = depth - 1; lev >= 0 && valid; --lev) {
        if (!((h - l) > 1e-3 * h)) valid = false;
        const double mid = 0.5 * (l + h);
        if ((kk >> lev) & 1) l = mid; else h = mid;
      }
      valid = valid && ((h - l) > 1e-3 * h);
    }
    if (valid) {
      k.on = true;
      k.beta = 0.5 * (l + h);
    }
  }
  return k;
}

// Per-plan decision by thread `j` (= plan column) over the kl slots that served
// it (base = my_rank * kl): the reference's sequential logic.
template <class A>
GVP_DEV void search_decide(const A& a, PlanSt* pst, int j, int base, int kl, int64_t b0, bool commit,
                           const double* r_beta, const double* r_kl, const int* r_res,
                           const int* r_fail, const int* r_on, const double* r_ld = nullptr) {
  const int64_t bj = b0 + j;
  PlanSt D = pst[j];
  auto log_probe = [&](int q) {
    const bool spd = r_res[q] != 1;
    if (a.probe_log && D.nprobe < a.max_probes) {
      double* row = a.probe_log + (bj * a.max_probes + D.nprobe) * 3;
      row[0] = r_beta[q];
      row[1] = spd ? 1.0 : 0.0;
      row[2] = spd ? r_kl[q] : INFINITY;
    }
    ++D.nprobe;
  };
  auto feasible = [&](int q) { return r_res[q] == 0 && !(r_kl[q] > a.kl_bound); };
  auto fail = [&](int code, int w) {
    a.status[bj] = code;
    a.where[bj] = w;
    if (a.nprobes) a.nprobes[bj] = D.nprobe;
    D.phase = 4;
  };
  // Replay the reference's bisection (optimizer.py:223-230) as far as this
  // round's probes reach: at each step the reference evaluates
  // mid = 0.5 * (lo + hi); if some slot probed exactly that beta (bitwise),
  // take its verdict, otherwise stop and probe it next round.
  auto walk = [&]() -> bool {
    for (int lev = 0; lev <= kl; ++lev) {
      if (!((D.hi - D.lo) > 1e-3 * D.hi)) return true;
      const double mid = 0.5 * (D.lo + D.hi);
      int q = -1;
      for (int qq = base + kl - 1; qq >= base; --qq)
        if (r_on[qq] && r_beta[qq] == mid) q = qq;
      if (q < 0) return true;
      log_probe(q);
      if (r_res[q] == 2) {
        fail(GVP_ERR_NOT_SPD, r_fail[q] | GVP_WHERE_MEAN_SOLVE_BIAS);
        return false;
      }
      if (feasible(q)) {
        D.lo = mid;
        D.best = mid;
        D.kl_lo = r_kl[q];
        if (r_ld) D.ld_best = r_ld[q];
      } else {
        D.hi = mid;
        D.kl_hi = r_res[q] == 1 ? INFINITY : r_kl[q];
      }
    }
    return true;
  };
  const int q0 = base, q1 = base + 1;
  if (D.phase == 3) {
    D.phase = 4;
  } else if (D.phase == 0) {
    log_probe(q0);
    if (r_res[q0] == 2) {
      fail(GVP_ERR_NOT_SPD, r_fail[q0] | GVP_WHERE_MEAN_SOLVE_BIAS);
    } else if (feasible(q0)) {
      D.best = a.beta_max;
      D.kl_lo = r_kl[q0];
      if (r_ld) D.ld_best = r_ld[q0];
      D.phase = 3;
    } else if (kl == 1) {
      D.kl_hi = r_res[q0] == 1 ? INFINITY : r_kl[q0];
      D.phase = 1;
    } else {
      log_probe(q1);
      if (r_res[q1] == 2) {
        fail(GVP_ERR_NOT_SPD, r_fail[q1] | GVP_WHERE_MEAN_SOLVE_BIAS);
      } else if (!feasible(q1)) {
        fail(GVP_ERR_NO_FEASIBLE_STEP, -1);
      } else {
        D.best = a.beta_min;
        D.lo = a.beta_min;
        D.hi = a.beta_max;
        D.kl_lo = r_kl[q1];
        if (r_ld) D.ld_best = r_ld[q1];
        D.kl_hi = r_res[q0] == 1 ? INFINITY : r_kl[q0];
        if (walk()) D.phase = ((D.hi - D.lo) > 1e-3 * D.hi) ? 2 : 3;
      }
    }
  } else if (D.phase == 1) {
    log_probe(q0);
    if (r_res[q0] == 2) {
      fail(GVP_ERR_NOT_SPD, r_fail[q0] | GVP_WHERE_MEAN_SOLVE_BIAS);
    } else if (!feasible(q0)) {
      fail(GVP_ERR_NO_FEASIBLE_STEP, -1);
    } else {
      D.best = a.beta_min;
      D.lo = a.beta_min;
      D.hi = a.beta_max;
      D.kl_lo = r_kl[q0];
      if (r_ld) D.ld_best = r_ld[q0];
      if (walk()) D.phase = ((D.hi - D.lo) > 1e-3 * D.hi) ? 2 : 3;
    }
  } else if (D.phase == 2) {
    if (walk()) D.phase = ((D.hi - D.lo) > 1e-3 * D.hi) ? 2 : 3;
  }
  if (!commit && D.phase == 3) {  // search finished: hand beta to the commit kernel
    a.beta[bj] = D.best;
    if (r_ld) {  // the accepted probe's KL (kl_joint of step.kl) and forward-Schur log det
      a.kl[bj] = D.kl_lo;
      a.ld_next[bj] = D.ld_best;
    }
    a.status[bj] = GVP_OK;
    a.where[bj] = -1;
    if (a.nprobes) a.nprobes[bj] = D.nprobe;
    D.phase = 4;
  }
  pst[j] = D;
}

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 3D map over a plan-minor array [K][E][W] (W = plan stride), box [bw, rows, 1]
static inline int make_map(CUtensorMap* m, const double* base, int64_t W, int64_t E, int64_t K, int bw,
                    int rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return GVP_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)E, (cuuint64_t)std::max<int64_t>(K, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(W * 8), (cuuint64_t)(W * E * 8)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return GVP_ERR_CUDA;
  }
  return GVP_OK;
}

}  // namespace v3

// one-pass bisection (step_probe.cu); its residual buffer lives in the step scratch
int launch_probe(const V2Launch& q, int L, cudaStream_t s);
int64_t probe_residual_offset(int nplans, int64_t K, int n);
// commit with the output work split off the two recursion warps (commit.cu)
int launch_commit_split(const V2Launch& q, cudaStream_t s);
}  // namespace gvp
