// Kernel (b)+(c) v2: select_step_size (optimizer.py:188-231) for a batch of
// plans, block-synchronous, with speculative bisection lanes.
//
// Thread mapping: a CTA of TB threads owns P = TB / L plans; each plan has L
// lanes (consecutive threads). In a round every lane of a plan probes one
// candidate beta. The candidates are the nodes of the bisection tree the
// reference walks sequentially (BFS order, the same float operations that
// produce `mid = 0.5 * (lo + hi)`), so after a round the group replays the
// reference's decisions over d = floor(log2(L + 1)) tree levels at once and
// reproduces its beta sequence exactly; off-path nodes are discarded.
//
// Each probe = two passes over the chain (see chain_kernels.cu for the
// algebra): pass B (knot K-1 -> 0) fuses the GBP backward Schur sweep of the
// candidate precision (SPD test + log det) with a backward elimination of
// the mean system; pass F (0 -> K-1) fuses the forward substitution, the
// covariance sweep, tr(Lambda_k Sigma') and the Mahalanobis term.
// Triangular factors are kept as their inverses so the recurrences use only
// multiplications (one rsqrt per pivot).
//
// Memory: all plan data is plan-minor with packed-symmetric diagonal blocks
// (T = n(n+1)/2 entries). Each knot's inputs for the CTA are staged in
// shared memory by cp.async D stages ahead of the knot being computed, so
// the HBM/L2 latency overlaps the sequential block algebra. Per-lane sweep
// intermediates go to a lane-minor scratch array and come back the same way.
#include <cuda_runtime.h>

#include <cmath>

#include "gvp_internal.cuh"

namespace gvp {
namespace v2 {

constexpr int kStages = 3;

GVP_DEV void cp_async8(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
GVP_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NW>
GVP_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NW) : "memory"); }

template <int N> constexpr int T_ = N * (N + 1) / 2;

// ------------------------------------------------------------ packed algebra
// lower Cholesky of a packed SPD matrix -> inverse factor Li (packed lower);
// returns false on a non-SPD pivot (blocktri.py:24-32 predicate). Also
// returns the product of the pivots (for the log det).
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
    const double r = rsqrt(s);        // 1 / pivot
    const double d = s * r;           // pivot
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
  // triangular inverse, column by column: Li[r][c] = -(sum_{k=c}^{r-1} L[r][k] Li[k][c]) / L[r][r]
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

// W = Li U^T (Li packed lower, U full row-major): W[r][c] = sum_{k<=r} Li[r][k] U[c][k]
template <int N>
GVP_DEV void li_ut(const double (&Li)[T_<N>], const double (&U)[N * N], double (&W)[N * N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k <= r; ++k) t += Li[tri_idx(r, k)] * U[c * N + k];
      W[r * N + c] = t;
    }
}
// A -= W^T W (A packed symmetric)
template <int N>
GVP_DEV void sub_gram(double (&A)[T_<N>], const double (&W)[N * N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) t += W[k * N + r] * W[k * N + c];
      A[tri_idx(r, c)] -= t;
    }
}
// P = Li^T Li (packed symmetric inverse)
template <int N>
GVP_DEV void inv_from_li(const double (&Li)[T_<N>], double (&P)[T_<N>]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = r; k < N; ++k) t += Li[tri_idx(k, r)] * Li[tri_idx(k, c)];
      P[tri_idx(r, c)] = t;
    }
}
template <int N>
GVP_DEV double sym_at(const double (&A)[T_<N>], int r, int c) {
  return r >= c ? A[tri_idx(r, c)] : A[tri_idx(c, r)];
}

// ------------------------------------------------------------ arguments
struct Args {
  int B;            // plans
  int64_t K;        // knots
  int64_t Bp;       // plan stride of the plan-minor arrays (>= B)
  int TB;           // threads per CTA
  // inputs (plan-minor, packed diag blocks)
  const double *ld, *lo, *kd, *ko, *gd, *g, *eta, *v, *mu, *pmean;
  int64_t ksp;      // 1 = per-plan prior precision, 0 = shared
  // outputs of the commit (may alias mu/ld/lo/v)
  double *o_mu, *o_ld, *o_lo, *o_cov, *o_cr, *o_v;
  double *beta, *kl, *ld_next, *shift, *prior_cost;
  const double* temp;
  const double* ld_cur;
  double kl_bound, beta_min, beta_max;
  int *status, *where;
  double* probe_log;
  int max_probes;
  int* nprobes;
  double* scratch;  // [K][SE][BLp]
  int64_t BLp;      // lane stride of scratch (>= B * L)
  const int* active;
};

// smem row map of one stage. Pass B per plan: LD T | GD T | KD T | G N | ETA N | V N | LO N2 | KO N2
//                             Pass F per plan: LD T | KD T | GD T | MU N | PM N | LO N2 | KO N2
//                                    per lane: PHI T (knot i+1) | LIPSI T | Y N
template <int N>
struct Layout {
  static constexpr int T = T_<N>, N2 = N * N;
  static constexpr int B_LD = 0, B_GD = T, B_KD = 2 * T, B_G = 3 * T, B_ETA = 3 * T + N,
                       B_V = 3 * T + 2 * N, B_LO = 3 * T + 3 * N, B_KO = 3 * T + 3 * N + N2,
                       B_ROWS = 3 * T + 3 * N + 2 * N2;
  static constexpr int F_LD = 0, F_KD = T, F_GD = 2 * T, F_MU = 3 * T, F_PM = 3 * T + N,
                       F_LO = 3 * T + 2 * N, F_KO = 3 * T + 2 * N + N2,
                       F_PLAN_ROWS = 3 * T + 2 * N + 2 * N2;
  static constexpr int SE = 2 * T + N;  // scratch entries per knot per lane: PHIINV | LIPSI | Y
  static constexpr int S_PHI = 0, S_LIPSI = T, S_Y = 2 * T;
};

template <int N>
GVP_DEV int stage_doubles(int P, int TB) {
  using Ly = Layout<N>;
  const int b = Ly::B_ROWS * P;
  const int f = Ly::F_PLAN_ROWS * P + Ly::SE * TB;
  return b > f ? b : f;
}

// copy helpers: rows [r0, r0+E) of array `base` (entries per knot E, plan
// stride sp) for knot `i` and the CTA's plans into smem rows starting at `dst_row`
struct CopyCtx {
  double* sm;       // stage base
  int P, TB, tid;
  int64_t b0, B, Bp;
};
GVP_DEV void copy_plan_rows(const CopyCtx& c, int dst_row, const double* base, int E, int64_t i,
                            int64_t sp) {
  const int total = E * c.P;
  for (int idx = c.tid; idx < total; idx += c.TB) {
    const int e = idx / c.P, p = idx - e * c.P;
    const int64_t b = c.b0 + p;
    if (b < c.B)
      cp_async8(c.sm + (dst_row + e) * c.P + p, base + (i * E + e) * (sp ? c.Bp : 1) + (sp ? b : 0));
  }
}

// ------------------------------------------------------------ the kernel
template <int N, int L>
__global__ void __launch_bounds__(128)
select_step_v2_kernel(Args a) {
  using Ly = Layout<N>;
  constexpr int T = T_<N>, N2 = N * N;
  constexpr int SE = Ly::SE;
  extern __shared__ __align__(16) double smem[];
  const int TB = a.TB, P = TB / L;
  const int tid = threadIdx.x;
  const int p = tid / L, lane = tid % L;
  const int64_t b0 = (int64_t)blockIdx.x * P;
  const int64_t b = b0 + p;
  const int64_t K = a.K;
  const int SD = stage_doubles<N>(P, TB);
  const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << ((tid & 31) / L * L));

  // ---- per-plan bisection state (identical in all lanes of the group)
  bool plan_ok = (b < a.B) && (!a.active || a.active[b]);
  int phase = plan_ok ? 0 : 4;  // 0 first round, 1 beta_min (L==1), 2 bisect, 3 commit, 4 done
  double lo = a.beta_min, hi = a.beta_max, best = a.beta_max;
  const double temp = plan_ok ? a.temp[b] : 1.0;
  const double ldc = plan_ok ? a.ld_cur[b] : 0.0;
  int nprobe = 0;
  auto log_probe = [&](double bt, bool spd, double klv) {
    if (lane == 0 && a.probe_log && nprobe < a.max_probes) {
      double* row = a.probe_log + (b * a.max_probes + nprobe) * 3;
      row[0] = bt;
      row[1] = spd ? 1.0 : 0.0;
      row[2] = spd ? klv : INFINITY;
    }
    ++nprobe;
  };

  CopyCtx cc{nullptr, P, TB, tid, b0, a.B, a.Bp};
  const int64_t lane_idx = b0 * L + tid;  // this lane's scratch column
  double* scr = a.scratch;

  for (;;) {
    // ---------------- candidate of this lane for this round
    bool lane_on = false, write = false;
    double beta = 0.0;
    const bool tree_phase = (phase == 2) || (phase == 0 && L >= 2 && lane >= 2);
    if (phase == 0 && lane == 0) {
      lane_on = true;
      beta = a.beta_max;
    } else if (phase == 0 && L >= 2 && lane == 1) {
      lane_on = true;
      beta = a.beta_min;
    } else if (phase == 1 && lane == 0) {
      lane_on = true;
      beta = a.beta_min;
    } else if (phase == 3 && lane == 0) {
      lane_on = true;
      write = true;
      beta = best;
    } else if (tree_phase) {
      // BFS node k of the bisection subtree rooted at (l, h)
      const int k = (phase == 2) ? lane + 1 : lane - 1;
      double l = (phase == 2) ? lo : a.beta_min, h = (phase == 2) ? hi : a.beta_max;
      int depth = 31 - __clz(k);
      bool valid = true;
      for (int lev = depth - 1; lev >= 0 && valid; --lev) {
        if (!((h - l) > 1e-3 * h)) valid = false;
        const double mid = 0.5 * (l + h);
        if ((k >> lev) & 1) l = mid; else h = mid;
      }
      valid = valid && ((h - l) > 1e-3 * h);
      if (valid) {
        lane_on = true;
        beta = 0.5 * (l + h);
      }
    }
    const int any_work = __syncthreads_or(phase < 4);
    if (!any_work) break;

    // ---------------- probe (all threads walk the knots; inactive lanes skip math)
    const double inv_t = 1.0 / temp, two_t = 2.0 / temp;
    const double inv_b = lane_on ? 1.0 / beta : 0.0, c = lane_on ? beta / (beta + 1.0) : 0.0;
    int res = 0;  // 0 ok, 1 not spd (candidate infeasible), 2 mean-solve pivot failure
    int fail_knot = -1;
    double ld_sum = 0.0;

    // ===== pass B: knots K-1 .. 0
    double LiPhiN[T], LiPsiN[T], yN[N];
    auto issueB = [&](int64_t s) {
      const int64_t i = K - 1 - s;
      cc.sm = smem + (s % kStages) * SD;
      copy_plan_rows(cc, Ly::B_LD, a.ld, T, i, 1);
      copy_plan_rows(cc, Ly::B_GD, a.gd, T, i, 1);
      copy_plan_rows(cc, Ly::B_KD, a.kd, T, i, a.ksp);
      copy_plan_rows(cc, Ly::B_G, a.g, N, i, 1);
      copy_plan_rows(cc, Ly::B_ETA, a.eta, N, i, 1);
      copy_plan_rows(cc, Ly::B_V, a.v, N, i, 1);
      if (i < K - 1) {
        copy_plan_rows(cc, Ly::B_LO, a.lo, N2, i, 1);
        copy_plan_rows(cc, Ly::B_KO, a.ko, N2, i, a.ksp);
      }
    };
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < K) issueB(s);
      cp_commit();
    }
    for (int64_t s = 0; s < K; ++s) {
      cp_wait<kStages - 2>();
      __syncthreads();
      if (s + kStages - 1 < K) issueB(s + kStages - 1);
      cp_commit();
      const int64_t i = K - 1 - s;
      const double* st = smem + (s % kStages) * SD;
      if (lane_on && res == 0) {
        auto sv = [&](int row) { return st[row * P + p]; };
        double Phi[T], Psi[T], rhs[N];
#pragma unroll
        for (int q = 0; q < T; ++q) {
          const double ldq = sv(Ly::B_LD + q), kdq = sv(Ly::B_KD + q);
          Phi[q] = ((sv(Ly::B_GD + q) * two_t + kdq * inv_t) + ldq * inv_b) * c;
          Psi[q] = kdq * inv_t + ldq * inv_b;
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
          rhs[r] = ((-sv(Ly::B_G + r)) * inv_t + sv(Ly::B_ETA + r) * inv_t) + sv(Ly::B_V + r) * inv_b;
        if (i < K - 1) {
          double So[N2], W[N2];
#pragma unroll
          for (int q = 0; q < N2; ++q) So[q] = sv(Ly::B_KO + q) * inv_t + sv(Ly::B_LO + q) * inv_b;
          // candidate off block U' = c * S_off (no pairwise factors: G_off = 0)
          double Up[N2];
#pragma unroll
          for (int q = 0; q < N2; ++q) Up[q] = So[q] * c;
          li_ut<N>(LiPhiN, Up, W);
          sub_gram<N>(Phi, W);
          li_ut<N>(LiPsiN, So, W);
          sub_gram<N>(Psi, W);
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += W[q * N + r] * yN[q];
            rhs[r] -= t;
          }
        }
        double LiPhi[T], LiPsi[T], pp, pq;
        if (!chol_inv<N>(Phi, LiPhi, pp)) {
          res = 1;
          fail_knot = (int)i;
        } else if (!chol_inv<N>(Psi, LiPsi, pq)) {
          res = 2;
          fail_knot = (int)i;
        } else {
          ld_sum += 2.0 * log(pp);
          double PhiInv[T];
          inv_from_li<N>(LiPhi, PhiInv);
          double* sc = scr + i * SE * a.BLp + lane_idx;
#pragma unroll
          for (int q = 0; q < T; ++q) {
            sc[(Ly::S_PHI + q) * a.BLp] = PhiInv[q];
            sc[(Ly::S_LIPSI + q) * a.BLp] = LiPsi[q];
            LiPhiN[q] = LiPhi[q];
            LiPsiN[q] = LiPsi[q];
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 <= r; ++k2) t += LiPsi[tri_idx(r, k2)] * rhs[k2];
            yN[r] = t;
            sc[(Ly::S_Y + r) * a.BLp] = t;
          }
        }
      }
    }
    cp_wait<0>();
    __syncthreads();

    // ===== pass F: knots 0 .. K-1
    double Sig[T], So_prev[N2], Lo_prev[N2], m_prev[N], d_prev[N];
    double trace = 0.0, mahal = 0.0, sh2 = 0.0, pq_c = 0.0, ptr_c = 0.0;
    double dp_prev[N], Ko_prev[N2], part_prev[N], Up_prev[N2];
    const bool passF = lane_on && res == 0;
    auto issueF = [&](int64_t i) {
      cc.sm = smem + (i % kStages) * SD;
      copy_plan_rows(cc, Ly::F_LD, a.ld, T, i, 1);
      copy_plan_rows(cc, Ly::F_KD, a.kd, T, i, a.ksp);
      copy_plan_rows(cc, Ly::F_GD, a.gd, T, i, 1);
      copy_plan_rows(cc, Ly::F_MU, a.mu, N, i, 1);
      copy_plan_rows(cc, Ly::F_PM, a.pmean, N, i, 1);
      if (i < K - 1) {
        copy_plan_rows(cc, Ly::F_LO, a.lo, N2, i, 1);
        copy_plan_rows(cc, Ly::F_KO, a.ko, N2, i, a.ksp);
      }
      // per-lane scratch: PHIINV of knot i+1 (or knot 0 at i = 0 .. handled below), LIPSI/Y of knot i
      double* lane_rows = cc.sm + Ly::F_PLAN_ROWS * P;
      for (int idx = tid; idx < SE * TB; idx += TB) {
        const int e = idx / TB, t = idx - e * TB;
        int64_t knot = i;
        if (e < T) knot = (i + 1 < K) ? i + 1 : i;  // PHIINV of the next knot
        cp_async8(lane_rows + e * TB + t, scr + (knot * SE + e) * a.BLp + b0 * L + t);
      }
    };
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < K) issueF(s);
      cp_commit();
    }
    if (passF) {  // Sigma_00 = Phi_0^{-1}
      const double* sc = scr + lane_idx;
#pragma unroll
      for (int q = 0; q < T; ++q) Sig[q] = sc[(Ly::S_PHI + q) * a.BLp];
    }
    for (int64_t i = 0; i < K; ++i) {
      cp_wait<kStages - 2>();
      __syncthreads();
      if (i + kStages - 1 < K) issueF(i + kStages - 1);
      cp_commit();
      if (!passF) continue;
      const double* st = smem + (i % kStages) * SD;
      const double* lr = st + Ly::F_PLAN_ROWS * P;
      auto sv = [&](int row) { return st[row * P + p]; };
      auto lv = [&](int row) { return lr[row * TB + tid]; };
      double m[N], dl[N];
      {
        // mu'_i = LiPsi^T (y_i - LiPsi (S_{i-1,i}^T mu'_{i-1}))
        double z[N], w[N];
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
          if (i > 0) {
#pragma unroll
            for (int q = 0; q < N; ++q) t += So_prev[q * N + r] * m_prev[q];
          }
          z[r] = t;
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q <= r; ++q) t += lv(Ly::S_LIPSI + tri_idx(r, q)) * z[q];
          w[r] = lv(Ly::S_Y + r) - t;
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = r; q < N; ++q) t += lv(Ly::S_LIPSI + tri_idx(q, r)) * w[q];
          m[r] = t;
        }
      }
#pragma unroll
      for (int r = 0; r < N; ++r) {
        dl[r] = sv(Ly::F_MU + r) - m[r];
        sh2 += dl[r] * dl[r];
      }
      // tr(Lambda_ii Sigma_ii) and delta' Lambda_ii delta (packed symmetric)
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int q = 0; q <= r; ++q) {
          const double lam = sv(Ly::F_LD + tri_idx(r, q));
          const double f = (q == r) ? 1.0 : 2.0;
          trace += f * lam * Sig[tri_idx(r, q)];
          mahal += f * lam * dl[r] * dl[q];
        }
      if (i > 0) {
        double t = 0.0;
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) t += d_prev[r] * Lo_prev[r * N + q] * dl[q];
        mahal += 2.0 * t;
      }
      double dp[N];
      if (write) {
        double Pn[T];
#pragma unroll
        for (int q = 0; q < T; ++q)
          Pn[q] = ((sv(Ly::F_GD + q) * two_t + sv(Ly::F_KD + q) * inv_t) + sv(Ly::F_LD + q) * inv_b) * c;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          a.o_mu[(i * N + r) * a.Bp + b] = m[r];
          dp[r] = m[r] - sv(Ly::F_PM + r);
        }
#pragma unroll
        for (int q = 0; q < T; ++q) {
          a.o_ld[(i * T + q) * a.Bp + b] = Pn[q];
          a.o_cov[(i * T + q) * a.Bp + b] = Sig[q];
        }
        // prior cost pieces (optimizer.py:260-263): d' K d and tr(K Sigma)
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            const double kk = sv(Ly::F_KD + tri_idx(r, q));
            const double f = (q == r) ? 1.0 : 2.0;
            pq_c += f * kk * dp[r] * dp[q];
            ptr_c += f * kk * Sig[tri_idx(r, q)];
          }
        // v' = Lambda' mu' for the next iteration's rhs
        double part[N];
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) t += sym_at<N>(Pn, r, q) * m[q];
          if (i > 0) {
#pragma unroll
            for (int q = 0; q < N; ++q) t += Up_prev[q * N + r] * m_prev[q];
          }
          part[r] = t;
        }
        if (i > 0) {
          double t2 = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q < N; ++q) t2 += dp_prev[r] * Ko_prev[r * N + q] * dp[q];
          pq_c += 2.0 * t2;
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = part_prev[r];
#pragma unroll
            for (int q = 0; q < N; ++q) t += Up_prev[r * N + q] * m[q];
            a.o_v[((i - 1) * N + r) * a.Bp + b] = t;
          }
        }
#pragma unroll
        for (int r = 0; r < N; ++r) part_prev[r] = part[r];
        if (i == K - 1) {
#pragma unroll
          for (int r = 0; r < N; ++r) a.o_v[(i * N + r) * a.Bp + b] = part[r];
        }
      }
      if (i + 1 < K) {
        double Up[N2], Pi[T], A[N2], M[N2], Bm[N2];
#pragma unroll
        for (int q = 0; q < N2; ++q) {
          const double lo_q = sv(Ly::F_LO + q), ko_q = sv(Ly::F_KO + q);
          So_prev[q] = ko_q * inv_t + lo_q * inv_b;
          Up[q] = So_prev[q] * c;
          Lo_prev[q] = lo_q;
        }
#pragma unroll
        for (int q = 0; q < T; ++q) Pi[q] = lv(Ly::S_PHI + q);  // Phi_{i+1}^{-1}
        // A = Sigma_ii U', M = A Phi^{-1}, Bm = U' Phi^{-1}
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) t += sym_at<N>(Sig, r, k2) * Up[k2 * N + q];
            A[r * N + q] = t;
          }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double t = 0.0, u = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) {
              t += A[r * N + k2] * sym_at<N>(Pi, k2, q);
              u += Up[r * N + k2] * sym_at<N>(Pi, k2, q);
            }
            M[r * N + q] = t;
            Bm[r * N + q] = u;
          }
        double tc = 0.0;
#pragma unroll
        for (int q = 0; q < N2; ++q) tc += Lo_prev[q] * M[q];
        trace -= 2.0 * tc;
        if (write) {
          double tk = 0.0;
#pragma unroll
          for (int q = 0; q < N2; ++q) {
            a.o_cr[(i * N2 + q) * a.Bp + b] = -M[q];
            a.o_lo[(i * N2 + q) * a.Bp + b] = Up[q];
            Ko_prev[q] = sv(Ly::F_KO + q);
            tk += Ko_prev[q] * M[q];
            Up_prev[q] = Up[q];
          }
          ptr_c -= 2.0 * tk;
#pragma unroll
          for (int r = 0; r < N; ++r) dp_prev[r] = dp[r];
        }
        // Sigma_{i+1} = Phi^{-1} + Bm^T M (symmetric by construction)
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) t += Bm[k2 * N + r] * M[k2 * N + q];
            const double s1 = Pi[tri_idx(r, q)] + t;
            double t2 = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) t2 += Bm[k2 * N + q] * M[k2 * N + r];
            Sig[tri_idx(r, q)] = 0.5 * (s1 + (Pi[tri_idx(r, q)] + t2));
          }
      }
#pragma unroll
      for (int r = 0; r < N; ++r) {
        m_prev[r] = m[r];
        d_prev[r] = dl[r];
      }
    }
    cp_wait<0>();
    __syncthreads();

    double klv = 0.0;
    if (passF) {
      const double x = 0.5 * ((((trace + mahal) - (double)(K * N)) + ld_sum) - ldc);
      klv = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
    }

    // ---------------- group decision (replays the reference's sequential logic)
    if (phase < 4) {
      if (write) {  // lane 0 committed
        a.beta[b] = best;
        a.kl[b] = klv;
        a.ld_next[b] = ld_sum;
        a.shift[b] = sqrt(sh2);
        if (a.prior_cost) a.prior_cost[b] = 0.5 * pq_c + 0.5 * ptr_c;
        a.status[b] = GVP_OK;
        a.where[b] = -1;
        if (a.nprobes) a.nprobes[b] = nprobe;
      }
    }
    // results of all lanes in the group
    double r_kl[L];
    int r_res[L];
    bool r_on[L];
    double r_beta[L];
    int r_fail[L];
#pragma unroll
    for (int q = 0; q < L; ++q) {
      r_kl[q] = __shfl_sync(gmask, klv, q, L);
      r_res[q] = __shfl_sync(gmask, res, q, L);
      r_on[q] = __shfl_sync(gmask, (int)lane_on, q, L);
      r_beta[q] = __shfl_sync(gmask, beta, q, L);
      r_fail[q] = __shfl_sync(gmask, fail_knot, q, L);
    }
    if (phase >= 4) continue;
    auto feasible = [&](int q) { return r_res[q] == 0 && !(r_kl[q] > a.kl_bound); };
    auto fail = [&](int code, int w) {
      if (lane == 0) {
        a.status[b] = code;
        a.where[b] = w;
        if (a.nprobes) a.nprobes[b] = nprobe;
      }
      phase = 4;
    };
    // walk a subtree whose node k sits at lane (k - 1 + off); returns false on error
    auto walk = [&](int off, int depth_avail) -> bool {
      int k = 1;
      for (int lev = 0; lev < depth_avail; ++lev) {
        if (!((hi - lo) > 1e-3 * hi)) return true;
        const int q = k - 1 + off;
        if (q >= L || !r_on[q]) return true;  // not evaluated (should not happen on-path)
        log_probe(r_beta[q], r_res[q] != 1, r_kl[q]);
        if (r_res[q] == 2) {
          fail(GVP_ERR_NOT_SPD, r_fail[q] | GVP_WHERE_MEAN_SOLVE_BIAS);
          return false;
        }
        if (feasible(q)) {
          lo = r_beta[q];
          best = r_beta[q];
          k = 2 * k + 1;
        } else {
          hi = r_beta[q];
          k = 2 * k;
        }
      }
      return true;
    };
    auto tree_depth = [](int nodes) {  // complete levels available in `nodes` lanes
      int d = 0;
      while ((2 << d) - 1 <= nodes) ++d;
      return d;
    };
    if (phase == 3) {
      phase = 4;
    } else if (phase == 0) {
      log_probe(r_beta[0], r_res[0] != 1, r_kl[0]);
      if (r_res[0] == 2) {
        fail(GVP_ERR_NOT_SPD, r_fail[0] | GVP_WHERE_MEAN_SOLVE_BIAS);
      } else if (feasible(0)) {
        best = a.beta_max;
        phase = 3;
      } else if (L == 1) {
        phase = 1;
      } else {
        log_probe(r_beta[1], r_res[1] != 1, r_kl[1]);
        if (r_res[1] == 2) {
          fail(GVP_ERR_NOT_SPD, r_fail[1] | GVP_WHERE_MEAN_SOLVE_BIAS);
        } else if (!feasible(1)) {
          fail(GVP_ERR_NO_FEASIBLE_STEP, -1);
        } else {
          best = a.beta_min;
          lo = a.beta_min;
          hi = a.beta_max;
          if (walk(2, tree_depth(L - 2))) phase = ((hi - lo) > 1e-3 * hi) ? 2 : 3;
        }
      }
    } else if (phase == 1) {
      log_probe(r_beta[0], r_res[0] != 1, r_kl[0]);
      if (r_res[0] == 2) {
        fail(GVP_ERR_NOT_SPD, r_fail[0] | GVP_WHERE_MEAN_SOLVE_BIAS);
      } else if (!feasible(0)) {
        fail(GVP_ERR_NO_FEASIBLE_STEP, -1);
      } else {
        best = a.beta_min;
        lo = a.beta_min;
        hi = a.beta_max;
        phase = ((hi - lo) > 1e-3 * hi) ? 2 : 3;
      }
    } else if (phase == 2) {
      if (walk(0, tree_depth(L))) phase = ((hi - lo) > 1e-3 * hi) ? 2 : 3;
    }
  }
}

// GBP marginals (gbp.py:43-80) on the packed layout, one thread per plan;
// log det from the same per-knot pivot products the step kernel uses.
template <int N>
__global__ void __launch_bounds__(64)
marginals_packed_kernel(int nplans, int64_t K, int64_t Bp, const double* __restrict__ ld,
                        const double* __restrict__ lo, double* __restrict__ cov,
                        double* __restrict__ cr, double* __restrict__ logdet,
                        int* __restrict__ status, int* __restrict__ where,
                        double* __restrict__ scr, const int* __restrict__ active) {
  constexpr int T = T_<N>, N2 = N * N;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  if (active && !active[b]) return;
  double LiN[T], lds = 0.0;
  for (int64_t i = K - 1; i >= 0; --i) {
    double Phi[T];
#pragma unroll
    for (int q = 0; q < T; ++q) Phi[q] = ld[(i * T + q) * Bp + b];
    if (i < K - 1) {
      double U[N2], W[N2];
#pragma unroll
      for (int q = 0; q < N2; ++q) U[q] = lo[(i * N2 + q) * Bp + b];
      li_ut<N>(LiN, U, W);
      sub_gram<N>(Phi, W);
    }
    double Li[T], pp;
    if (!chol_inv<N>(Phi, Li, pp)) {
      status[b] = GVP_ERR_NOT_SPD;
      where[b] = (int)i;
      return;
    }
    lds += 2.0 * log(pp);
    double Pi[T];
    inv_from_li<N>(Li, Pi);
#pragma unroll
    for (int q = 0; q < T; ++q) {
      scr[(i * T + q) * Bp + b] = Pi[q];
      LiN[q] = Li[q];
    }
  }
  double Sig[T];
#pragma unroll
  for (int q = 0; q < T; ++q) {
    Sig[q] = scr[q * Bp + b];
    cov[q * Bp + b] = Sig[q];
  }
  for (int64_t i = 0; i + 1 < K; ++i) {
    double U[N2], Pi[T], A[N2], M[N2], Bm[N2];
#pragma unroll
    for (int q = 0; q < N2; ++q) U[q] = lo[(i * N2 + q) * Bp + b];
#pragma unroll
    for (int q = 0; q < T; ++q) Pi[q] = scr[((i + 1) * T + q) * Bp + b];
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) t += sym_at<N>(Sig, r, k) * U[k * N + c];
        A[r * N + c] = t;
      }
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double t = 0.0, u = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          t += A[r * N + k] * sym_at<N>(Pi, k, c);
          u += U[r * N + k] * sym_at<N>(Pi, k, c);
        }
        M[r * N + c] = t;
        Bm[r * N + c] = u;
      }
#pragma unroll
    for (int q = 0; q < N2; ++q) cr[(i * N2 + q) * Bp + b] = -M[q];
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) {
        double t = 0.0, t2 = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          t += Bm[k * N + r] * M[k * N + c];
          t2 += Bm[k * N + c] * M[k * N + r];
        }
        Sig[tri_idx(r, c)] = 0.5 * ((Pi[tri_idx(r, c)] + t) + (Pi[tri_idx(r, c)] + t2));
      }
#pragma unroll
    for (int q = 0; q < T; ++q) cov[((i + 1) * T + q) * Bp + b] = Sig[q];
  }
  if (logdet) logdet[b] = lds;
  status[b] = GVP_OK;
}

// v = Lambda mu for packed Lambda (the rhs piece of the proximal mean system)
template <int N>
__global__ void lam_mu_kernel(int nplans, int64_t K, int64_t Bp, const double* __restrict__ ld,
                              const double* __restrict__ lo, const double* __restrict__ mu,
                              double* __restrict__ v) {
  constexpr int T = T_<N>, N2 = N * N;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * nplans) return;
  const int64_t b = t % nplans, i = t / nplans;
  double out[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      const int q = r >= c ? tri_idx(r, c) : tri_idx(c, r);
      s += ld[(i * T + q) * Bp + b] * mu[(i * N + c) * Bp + b];
    }
    if (i > 0) {
#pragma unroll
      for (int c = 0; c < N; ++c) s += lo[((i - 1) * N2 + c * N + r) * Bp + b] * mu[((i - 1) * N + c) * Bp + b];
    }
    if (i + 1 < K) {
#pragma unroll
      for (int c = 0; c < N; ++c) s += lo[(i * N2 + r * N + c) * Bp + b] * mu[((i + 1) * N + c) * Bp + b];
    }
    out[r] = s;
  }
#pragma unroll
  for (int r = 0; r < N; ++r) v[(i * N + r) * Bp + b] = out[r];
}

}  // namespace v2

int launch_marginals_packed(int nplans, int64_t K, int n, int64_t Bp, const double* ld,
                            const double* lo, double* cov, double* cr, double* logdet,
                            int* status, int* where, double* scratch, const int* active,
                            cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  const unsigned grid = (unsigned)((nplans + 31) / 32);
  switch (n) {
    case 2: v2::marginals_packed_kernel<2><<<grid, 32, 0, s>>>(nplans, K, Bp, ld, lo, cov, cr, logdet, status, where, scratch, active); break;
    case 4: v2::marginals_packed_kernel<4><<<grid, 32, 0, s>>>(nplans, K, Bp, ld, lo, cov, cr, logdet, status, where, scratch, active); break;
    case 6: v2::marginals_packed_kernel<6><<<grid, 32, 0, s>>>(nplans, K, Bp, ld, lo, cov, cr, logdet, status, where, scratch, active); break;
    default:
      set_error("packed marginals support n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int launch_lam_mu(int nplans, int64_t K, int n, int64_t Bp, const double* ld, const double* lo,
                  const double* mu, double* v, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  const int64_t tot = K * nplans;
  const unsigned grid = (unsigned)((tot + 127) / 128);
  switch (n) {
    case 2: v2::lam_mu_kernel<2><<<grid, 128, 0, s>>>(nplans, K, Bp, ld, lo, mu, v); break;
    case 4: v2::lam_mu_kernel<4><<<grid, 128, 0, s>>>(nplans, K, Bp, ld, lo, mu, v); break;
    case 6: v2::lam_mu_kernel<6><<<grid, 128, 0, s>>>(nplans, K, Bp, ld, lo, mu, v); break;
    default:
      set_error("lam_mu supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

// ------------------------------------------------------------ launcher
int64_t step_scratch_doubles(int nplans, int64_t K, int n, int lanes) {
  const int64_t T = (int64_t)n * (n + 1) / 2;
  const int64_t BL = ((int64_t)nplans * lanes + 1) & ~1LL;
  return std::max<int64_t>(1, K * (2 * T + n) * BL);
}

int launch_select_step_v2(const V2Launch& q, cudaStream_t s) {
  if (q.nplans == 0 || q.K == 0) return GVP_OK;
  const int L = q.lanes;
  int TB = 64;
  // enough CTAs to cover the SMs: small batches use small CTAs
  if ((int64_t)q.nplans * L <= 148 * 32) TB = 32;
  if (L > TB) TB = L;
  const int P = TB / L;
  const unsigned grid = (unsigned)((q.nplans + P - 1) / P);
  v2::Args a{};
  a.B = q.nplans;
  a.K = q.K;
  a.Bp = q.Bp;
  a.TB = TB;
  a.ld = q.ld; a.lo = q.lo; a.kd = q.kd; a.ko = q.ko; a.gd = q.gd;
  a.g = q.g; a.eta = q.eta; a.v = q.v; a.mu = q.mu; a.pmean = q.pmean;
  a.ksp = q.kshared ? 0 : 1;
  a.o_mu = q.o_mu; a.o_ld = q.o_ld; a.o_lo = q.o_lo; a.o_cov = q.o_cov; a.o_cr = q.o_cr; a.o_v = q.o_v;
  a.beta = q.beta; a.kl = q.kl; a.ld_next = q.ld_next; a.shift = q.shift; a.prior_cost = q.prior_cost;
  a.temp = q.temp; a.ld_cur = q.ld_cur;
  a.kl_bound = q.kl_bound; a.beta_min = q.beta_min; a.beta_max = q.beta_max;
  a.status = q.status; a.where = q.where;
  a.probe_log = q.probe_log; a.max_probes = q.max_probes; a.nprobes = q.nprobes;
  a.scratch = q.scratch;
  a.BLp = ((int64_t)q.nplans * L + 1) & ~1LL;
  a.active = q.active;
#define GVP_V2(NN, LL)                                                                          \
  {                                                                                             \
    const int sd = v2::Layout<NN>::B_ROWS * P > v2::Layout<NN>::F_PLAN_ROWS * P +               \
                                                      v2::Layout<NN>::SE * TB                   \
                       ? v2::Layout<NN>::B_ROWS * P                                             \
                       : v2::Layout<NN>::F_PLAN_ROWS * P + v2::Layout<NN>::SE * TB;            \
    const size_t bytes = (size_t)sd * v2::kStages * sizeof(double);                             \
    GVP_CUDA(cudaFuncSetAttribute(v2::select_step_v2_kernel<NN, LL>,                           \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));    \
    v2::select_step_v2_kernel<NN, LL><<<grid, TB, bytes, s>>>(a);                               \
  }
#define GVP_V2_L(NN)                         \
  switch (L) {                               \
    case 1: GVP_V2(NN, 1) break;             \
    case 4: GVP_V2(NN, 4) break;             \
    case 8: GVP_V2(NN, 8) break;             \
    case 16: GVP_V2(NN, 16) break;           \
    case 32: GVP_V2(NN, 32) break;           \
    default:                                 \
      set_error("lanes must be 1, 4, 8, 16 or 32"); \
      return GVP_ERR_ARG;                    \
  }
  switch (q.n) {
    case 2: GVP_V2_L(2) break;
    case 4: GVP_V2_L(4) break;
    case 6: GVP_V2_L(6) break;
    default:
      set_error("step kernel v2 supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_V2_L
#undef GVP_V2
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp
