// Kernel (b)+(c) v3: select_step_size (optimizer.py:188-231) for a batch of
// plans — TMA-staged, two threads per probe lane, speculative bisection.
//
// Thread mapping. A CTA owns P plans; each plan has L candidate lanes
// (speculative bisection, see below) and each lane is a PAIR of threads:
//   role A: the candidate precision's GBP chain — backward Schur pivots
//           Phi_i (SPD test, log det), forward covariance sweep Sigma_ii,
//           Sigma_i,i+1 and tr(Lambda_k Sigma') (gbp.py:43-80, gbp.py:109-120)
//   role B: the proximal mean system (optimizer.py:155-159) — backward
//           elimination pivots Psi_i, forward substitution mu', the
//           Mahalanobis term of kl_joint (optimizer.py:164-177) and, on
//           commit, Lambda' mu' for the next iteration's rhs.
// The two chains only meet in the KL; role B also forms U' Phi^{-1} for role A.
//
// Speculation. In a round the L lanes of a plan probe the nodes of the
// bisection subtree the reference would walk next (BFS order, identical
// float operations for every mid point); after the round the group replays
// the reference's sequential decisions over floor(log2(L+1)) levels, so the
// beta sequence is the reference's bit for bit; off-path nodes are dropped.
//
// Staging. Every knot's inputs for the CTA are brought into shared memory by
// the Tensor Memory Accelerator: one elected thread issues one
// cp.async.bulk.tensor per array per knot (boxes of [plans x entries]) two
// knots ahead, completion tracked by mbarrier transaction counts; the
// per-lane sweep intermediates of pass B return for pass F the same way.
// All plan arrays are plan-minor with an even plan stride Bp; diagonal
// blocks are packed lower-symmetric; a prior precision shared by all plans is
// stored 2-wide (two identical plan columns) so its boxes meet TMA's 16-byte
// rule.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "gvp_internal.cuh"

namespace gvp {
namespace v3 {

constexpr int kStages = 4;  // prefetch distance 2; slot of knot i-1 stays valid during knot i
constexpr int kAhead = 2;

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
    const double r = rsqrt(s);
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

// ------------------------------------------------------------ stage layout
// rows per plan (pass B / pass F), and per lane (pass F scratch)
template <int N>
struct Ly {
  static constexpr int T = T_<N>, N2 = N * N;
  // pass B plan rows
  static constexpr int B_LD = 0, B_GD = T, B_G = 2 * T, B_ETA = 2 * T + N, B_V = 2 * T + 2 * N,
                       B_LO = 2 * T + 3 * N, B_PLAN = 2 * T + 3 * N + N2;
  // pass F plan rows
  static constexpr int F_LD = 0, F_GD = T, F_MU = 2 * T, F_PM = 2 * T + N, F_LO = 2 * T + 2 * N,
                       F_PLAN = 2 * T + 2 * N + N2;
  // prior rows (both passes): KD | KO
  static constexpr int K_KD = 0, K_KO = T, K_ROWS = T + N2;
  // scratch entries per knot per lane: PHIINV | LIPSI | Y
  static constexpr int SE = 2 * T + N, S_PHI = 0, S_LIPSI = T, S_Y = 2 * T;
};

// Compile-time shared-memory layout of one CTA (32 lane slots = P plans x L
// lanes, two warps). Every TMA box lands on a 128-byte boundary: row starts
// are rounded to a multiple of cx_gran(width) rows.
constexpr int cx_round(int x, int m) { return (x + m - 1) / m * m; }
constexpr int cx_gran(int w) { return w % 16 == 0 ? 1 : w % 8 == 0 ? 2 : w % 4 == 0 ? 4 : w % 2 == 0 ? 8 : 16; }
template <int N, int L, bool KS>
struct Lay {
  static constexpr int T = N * (N + 1) / 2, N2 = N * N;
  static constexpr int P = 32 / L, Pb = P, Kb = KS ? 2 : P, LPb = 32;
  static constexpr int gP = cx_gran(Pb), gK = cx_gran(Kb);
  // pass B plan rows: LD T | GD T | G N | ETA N | V N | LO N2
  static constexpr int B0 = 0, B1 = cx_round(B0 + T, gP), B2 = cx_round(B1 + T, gP),
                       B3 = cx_round(B2 + N, gP), B4 = cx_round(B3 + N, gP),
                       B5 = cx_round(B4 + N, gP), BR = cx_round(B5 + N2, gP);
  // pass F plan rows: LD T | GD T | MU N | PM N | LO N2
  static constexpr int F0 = 0, F1 = cx_round(F0 + T, gP), F2 = cx_round(F1 + T, gP),
                       F3 = cx_round(F2 + N, gP), F4 = cx_round(F3 + N, gP),
                       FR = cx_round(F4 + N2, gP);
  // prior rows: KD T | KO N2
  static constexpr int K0 = 0, K1 = cx_round(T, gK), KR = cx_round(K1 + N2, gK);
  static constexpr int OFF_PLAN = 0, OFF_PRIOR = cx_round((BR > FR ? BR : FR) * Pb, 16),
                       OFF_PHI = OFF_PRIOR + cx_round(KR * Kb, 16),
                       OFF_PSIY = OFF_PHI + cx_round(T * LPb, 16),
                       STAGE = OFF_PSIY + cx_round((T + N) * LPb, 16);
  static constexpr int XCH = kStages * STAGE, BAR = XCH + 8 * 32;
  static constexpr int PST = BAR + 16;        // per-plan bisection state (10 doubles x 32)
  static constexpr int RES = PST + 10 * 32;   // per-slot probe results (5 x 32)
  static constexpr size_t BYTES = (size_t)(RES + 5 * 32) * 8;
  static constexpr uint32_t TX_B = ((2 * T + 3 * N + N2) * Pb + (T + N2) * Kb) * 8;
  static constexpr uint32_t TX_F = ((2 * T + 2 * N + N2) * Pb + (T + N2) * Kb + (2 * T + N) * LPb) * 8;
};

// bisection state of one plan, kept in shared memory: the CTA's lane slots
// are re-dealt among its still-searching plans every round
struct PlanSt {
  double lo, hi, best, kl_lo, kl_hi, prev, temp, ldc;
  int phase, nprobe;
};
static_assert(sizeof(PlanSt) <= 80, "PlanSt must fit 10 doubles");

struct Args {
  CUtensorMap m_ld, m_lo, m_kd, m_ko, m_gd, m_g, m_eta, m_v, m_mu, m_pm, m_phi, m_psiy;
  int B;
  int64_t K, Bp;
  int P, Pbox, Kbox;   // plans per CTA, plan box width (even), prior box width (2 if shared)
  int ksp;             // 1 per-plan prior, 0 shared (2-wide)
  double *o_mu, *o_ld, *o_lo, *o_cov, *o_cr, *o_v;
  double *beta, *kl, *ld_next, *shift, *prior_cost;
  const double *temp, *ld_cur;
  double kl_bound, beta_min, beta_max;
  int *status, *where, *nprobes;
  double* probe_log;
  int max_probes;
  double* scratch;
  int64_t BLp;
  const int* active;
  // smem offsets (doubles) of the regions inside one stage; first row of each
  // array inside its region (every TMA box lands on a 128-byte boundary)
  int off_plan, off_prior, off_phi, off_psiy, stage_doubles, bm_off, bar_off;
  int rB[6], rF[5], rK[2];
  uint32_t bytes_B, bytes_F;
};

// COMMIT = false: the bisection; the accepted beta goes to a.beta[b].
// COMMIT = true (L = 1): one write-mode probe at a.beta[b] producing the next
// iterate, its marginals, KL, log det, prior cost and Lambda' mu'. Keeping the
// write path out of the bisection kernel keeps its loop bodies small enough
// for the instruction cache.
template <int N, int L, bool COMMIT, bool KS>
__global__ void __launch_bounds__(64)
select_step_v3_kernel(const __grid_constant__ Args a) {
  using Y = Ly<N>;
  using LO = Lay<N, L, KS>;
  constexpr int T = Y::T, N2 = Y::N2, SE = Y::SE;
  // dynamic shared memory only (no static __shared__): the window starts
  // 1 KB-aligned, so the compile-time layout keeps every TMA box 128-B aligned
  // and all stage reads are LDS with immediate offsets
  extern __shared__ __align__(1024) double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LO::BAR);
  const int tid = threadIdx.x;
  // warp-specialised roles: even warps run chain A, odd warps chain B for the
  // same 32 lane slots, so neither chain diverges inside a warp
  const int role = (tid >> 5) & 1;
  const int lcol = ((tid >> 6) << 5) | (tid & 31);  // lane slot in the CTA
  constexpr int P = LO::P, Pb = LO::Pb, Kb = LO::Kb;
  constexpr int LP = P * L;                   // lane slots per CTA (= 32)
  const int64_t b0 = (int64_t)blockIdx.x * P;
  const int64_t K = a.K;
  double* xch = smem + LO::XCH;              // per-slot exchange between the two roles
  PlanSt* pst = reinterpret_cast<PlanSt*>(smem + LO::PST);
  double* r_beta = smem + LO::RES;           // per-slot results of the round
  double* r_kl = r_beta + 32;
  int* r_res = reinterpret_cast<int*>(r_kl + 32);
  int* r_fail = r_res + 32;
  int* r_on = r_fail + 32;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < P) {  // one thread per plan loads its state
    const int64_t bb = b0 + tid;
    const bool ok = (bb < a.B) && (!a.active || a.active[bb]) && (!COMMIT || a.status[bb] == GVP_OK);
    PlanSt& S = pst[tid];
    S.phase = ok ? (COMMIT ? 3 : 0) : 4;  // 0 first round, 1 beta_min pending, 2 bisect, 3 commit, 4 done
    S.lo = a.beta_min;
    S.hi = a.beta_max;
    S.best = (COMMIT && ok) ? a.beta[bb] : a.beta_max;
    S.kl_lo = 0.0;
    S.kl_hi = INFINITY;
    // the previous iteration's beta (a.beta on entry; NaN = none) aims the first round
    S.prev = (!COMMIT && ok) ? a.beta[bb] : -1.0;
    S.temp = ok ? a.temp[bb] : 1.0;
    S.ldc = ok ? a.ld_cur[bb] : 0.0;
    S.nprobe = 0;
  }
  __syncthreads();
  uint32_t uses[kStages] = {0, 0, 0, 0};  // per-slot completed-phase counters (uniform)

  double* scr = a.scratch;
  const int64_t sc_col = b0 * L + lcol;  // global scratch column of this slot

  auto slot = [&](int64_t s) { return smem + (s % kStages) * LO::STAGE; };
  // issue the TMA loads of one knot of a pass into slot s % kStages
  auto issue = [&](int64_t s, int64_t i, bool passB) {
    double* st = slot(s);
    uint64_t* bar = &bars[s % kStages];
    mbar_expect_tx(bar, passB ? LO::TX_B : LO::TX_F);
    const int ck = KS ? 0 : (int)b0;
    double* pl = st + LO::OFF_PLAN;
    double* pr = st + LO::OFF_PRIOR;
    tma3(pr + LO::K0 * Kb, &a.m_kd, ck, 0, (int)i, bar);
    tma3(pr + LO::K1 * Kb, &a.m_ko, ck, 0, (int)i, bar);
    if (passB) {
      tma3(pl + LO::B0 * Pb, &a.m_ld, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::B1 * Pb, &a.m_gd, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::B2* Pb, &a.m_g, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::B3 * Pb, &a.m_eta, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::B4* Pb, &a.m_v, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::B5 * Pb, &a.m_lo, (int)b0, 0, (int)i, bar);
    } else {
      tma3(pl + LO::F0 * Pb, &a.m_ld, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::F1 * Pb, &a.m_gd, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::F2 * Pb, &a.m_mu, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::F3 * Pb, &a.m_pm, (int)b0, 0, (int)i, bar);
      tma3(pl + LO::F4 * Pb, &a.m_lo, (int)b0, 0, (int)i, bar);
      tma3(st + LO::OFF_PHI, &a.m_phi, (int)(b0 * L), 0, (int)(i + 1), bar);        // PHIINV of knot i+1
      tma3(st + LO::OFF_PSIY, &a.m_psiy, (int)(b0 * L), Y::S_LIPSI, (int)i, bar);  // LIPSI | Y of knot i
    }
  };
  auto wait_slot = [&](int64_t s) {
    const int k = (int)(s % kStages);
    mbar_wait(&bars[k], uses[k] & 1u);
    ++uses[k];
  };

  for (;;) {
    // ---------------- lane pool: the CTA's still-searching plans share its 32
    // slots (k each, contiguous, in plan order); idle slots after the last
    int nact = 0;
    for (int j = 0; j < P; ++j) nact += pst[j].phase < 4 ? 1 : 0;
    if (nact == 0) break;  // uniform: every thread read the same shared state
    const int kl = LP / nact;
    const int my_idx = lcol / kl, q = lcol % kl;
    int pj = -1, my_rank = -1;  // plan served by this slot; rank of plan `tid` if it decides
    for (int j = 0, c = 0; j < P; ++j)
      if (pst[j].phase < 4) {
        if (c == my_idx) pj = j;
        if (j == tid) my_rank = c;
        ++c;
      }
    const int p = pj < 0 ? 0 : pj;  // plan column this slot reads (idle slots: any)
    const int64_t b = b0 + p;
    const int kcol = KS ? 0 : p;
    const PlanSt S = pst[p];
    const int phase = pj < 0 ? 4 : S.phase;
    const double temp = S.temp, ldc = S.ldc;

    // ---------------- candidate beta of this slot
    bool lane_on = false, write = false;
    double beta = 0.0;
    int qs = -1, nslots = 0;  // speculative index / count
    double l = a.beta_min, h = a.beta_max, target = -1.0;
    if (phase == 0) {
      if (q == 0) {
        lane_on = true;
        beta = a.beta_max;
      } else if (q == 1) {
        lane_on = true;
        beta = a.beta_min;
      } else {
        qs = q - 2;
        nslots = kl - 2;
        target = S.prev;
      }
    } else if (phase == 1) {
      if (q == 0) {
        lane_on = true;
        beta = a.beta_min;
      } else {
        qs = q - 1;
        nslots = kl - 1;
        target = S.prev;
      }
    } else if (phase == 2) {
      qs = q;
      nslots = kl;
      l = S.lo;
      h = S.hi;
      // predicted crossing beta* (KL(beta*) = bound): log-log interpolation
      // of the bracket's KL values
      if (S.kl_lo > 0.0 && isfinite(S.kl_hi) && S.kl_hi > S.kl_lo && S.kl_lo < a.kl_bound &&
          a.kl_bound < S.kl_hi) {
        const double t = (log(a.kl_bound) - log(S.kl_lo)) / (log(S.kl_hi) - log(S.kl_lo));
        target = exp(log(l) + t * (log(h) - log(l)));
      }
    } else if (COMMIT && phase == 3 && q == 0) {
      lane_on = true;
      write = true;
      beta = S.best;
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
        lane_on = true;
        beta = 0.5 * (l + h);
      }
    }
    __syncthreads();  // everyone has read the shared plan state

    const double inv_t = 1.0 / temp, two_t = 2.0 / temp;
    const double inv_b = lane_on ? 1.0 / beta : 0.0, c = lane_on ? beta / (beta + 1.0) : 0.0;
    int res = 0;  // role A: 1 = Phi not SPD; role B: 2 = mean pivot not SPD
    int fail_knot = -1;
    double ld_sum = 0.0;

    // =============================== pass B: knots K-1 .. 0
    double LiN[T], yN[N];
    int64_t sbase = 0;
    if (tid == 0)
      for (int s = 0; s < kAhead && s < K; ++s) issue(s, K - 1 - s, true);
    for (int64_t s = 0; s < K; ++s) {
      wait_slot(s);
      __syncthreads();  // everyone past knot s-1: its slot may be refilled
      if (tid == 0 && s + kAhead < K) issue(s + kAhead, K - 1 - (s + kAhead), true);
      const int64_t i = K - 1 - s;
      if (!(lane_on && res == 0)) continue;
      const double* st = slot(s);
      const double* pl = st + LO::OFF_PLAN;
      const double* pr = st + LO::OFF_PRIOR;
      auto pv = [&](int row) { return pl[row * Pb + p]; };
      auto kv = [&](int row) { return pr[row * Kb + kcol]; };
      double A_[T];
      if (role == 0) {  // Lambda' diag block (optimizer.py:151-153), already symmetric
#pragma unroll
        for (int q = 0; q < T; ++q)
          A_[q] = ((pv(LO::B1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::B0 + q) * inv_b) * c;
      } else {          // S diag block (optimizer.py:155)
#pragma unroll
        for (int q = 0; q < T; ++q) A_[q] = kv(LO::K0 + q) * inv_t + pv(LO::B0 + q) * inv_b;
      }
      double rhs[N];
      if (role == 1) {
#pragma unroll
        for (int r = 0; r < N; ++r)
          rhs[r] = ((-pv(LO::B2+ r)) * inv_t + pv(LO::B3 + r) * inv_t) + pv(LO::B4+ r) * inv_b;
      }
      if (i < K - 1) {
        // off block: S_off = K_off/T + Lambda_off/beta; role A uses U' = c * S_off
        const double sc_ = role == 0 ? c : 1.0;
        double W[N2];  // W = Li_{i+1} X^T, X = sc_ * S_off
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 <= r; ++k2)
              t += LiN[tri_idx(r, k2)] * ((kv(LO::K1 + q * N + k2) * inv_t + pv(LO::B5 + q * N + k2) * inv_b) * sc_);
            W[r * N + q] = t;
          }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) t += W[k2 * N + r] * W[k2 * N + q];
            A_[tri_idx(r, q)] -= t;
          }
        if (role == 1) {
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < N; ++k2) t += W[k2 * N + r] * yN[k2];
            rhs[r] -= t;
          }
        }
      }
      double Li[T], pp;
      if (!chol_inv<N>(A_, Li, pp)) {
        res = role == 0 ? 1 : 2;
        fail_knot = (int)i;
        continue;
      }
      double* sc = scr + (i * SE) * a.BLp + sc_col;
      if (role == 0) {
        ld_sum += 2.0 * log(pp);
        // Phi^{-1} = Li^T Li -> scratch for the covariance sweep
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = r; k2 < N; ++k2) t += Li[tri_idx(k2, r)] * Li[tri_idx(k2, q)];
            sc[(Y::S_PHI + tri_idx(r, q)) * a.BLp] = t;
          }
      } else {
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int k2 = 0; k2 <= r; ++k2) t += Li[tri_idx(r, k2)] * rhs[k2];
          yN[r] = t;
          sc[(Y::S_Y + r) * a.BLp] = t;
        }
#pragma unroll
        for (int q = 0; q < T; ++q) sc[(Y::S_LIPSI + q) * a.BLp] = Li[q];
      }
#pragma unroll
      for (int q = 0; q < T; ++q) LiN[q] = Li[q];
    }
    sbase += K;
    fence_proxy_async();  // scratch stores (generic proxy) -> TMA reads (async proxy)
    __syncthreads();
    // both threads of a lane agree on the outcome (the mean solve fails first,
    // like proximal_update raising before gbp_marginals, optimizer.py:203-207)
    {
      int* xi = reinterpret_cast<int*>(xch);  // [role][slot] result codes, then fail knots
      xi[role * 32 + lcol] = res;  // 32 lane slots per warp pair
      xi[64 + role * 32 + lcol] = fail_knot;
      __syncthreads();
      const int other = xi[(1 - role) * 32 + lcol];
      const int otherk = xi[64 + (1 - role) * 32 + lcol];
      __syncthreads();
      const int rA = role == 0 ? res : other, rB = role == 0 ? other : res;
      const int kA = role == 0 ? fail_knot : otherk, kB = role == 0 ? otherk : fail_knot;
      res = rB ? 2 : (rA ? 1 : 0);
      fail_knot = rB ? kB : kA;
    }

    // =============================== pass F: knots 0 .. K-1
    const bool passF = lane_on && res == 0;
    double Sig[T], mprev[N], dprev[N], dpprev[N], part[N];
    double trace = 0.0, mahal = 0.0, sh2 = 0.0, pq_c = 0.0, ptr_c = 0.0;
    if (passF && role == 0) {
      const double* sc = scr + sc_col;  // Sigma_00 = Phi_0^{-1}
#pragma unroll
      for (int q = 0; q < T; ++q) Sig[q] = sc[(Y::S_PHI + q) * a.BLp];
    }
    if (tid == 0)
      for (int s = 0; s < kAhead && s < K; ++s) issue(sbase + s, s, false);
    for (int64_t i = 0; i < K; ++i) {
      const int64_t s = sbase + i;
      wait_slot(s);
      __syncthreads();
      if (tid == 0 && i + kAhead < K) issue(s + kAhead, i + kAhead, false);
      const double* st = slot(s);
      const double* pl = st + LO::OFF_PLAN;
      const double* pr = st + LO::OFF_PRIOR;
      const double* stp = slot(s - 1);  // knot i-1 (valid when i > 0)
      const double* plp = stp + LO::OFF_PLAN;
      const double* prp = stp + LO::OFF_PRIOR;
      auto pv = [&](int row) { return pl[row * Pb + p]; };
      auto kv = [&](int row) { return pr[row * Kb + kcol]; };
      auto pvp = [&](int row) { return plp[row * Pb + p]; };
      auto kvp = [&](int row) { return prp[row * Kb + kcol]; };
      auto phi = [&](int q) { return st[LO::OFF_PHI + q * LP + lcol]; };
      auto psi = [&](int q) { return st[LO::OFF_PSIY + q * LP + lcol]; };  // LIPSI rows then Y rows
      if (passF && role == 1) {
        // ---- mean: mu'_i = Li^T (y_i - Li S_{i-1,i}^T mu'_{i-1})
        double m[N];
        {
          double z[N], w[N];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
            if (i > 0) {
#pragma unroll
              for (int q = 0; q < N; ++q)
                t += (kvp(LO::K1 + q * N + r) * inv_t + pvp(LO::F4 + q * N + r) * inv_b) * mprev[q];
            }
            z[r] = t;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q <= r; ++q) t += psi(tri_idx(r, q)) * z[q];
            w[r] = psi(T + r) - t;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = r; q < N; ++q) t += psi(tri_idx(q, r)) * w[q];
            m[r] = t;
          }
        }
        double dl[N];
#pragma unroll
        for (int r = 0; r < N; ++r) {
          dl[r] = pv(LO::F2 + r) - m[r];  // delta = cur.mean - nxt.mean
          sh2 += dl[r] * dl[r];
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q)
            mahal += ((q == r) ? 1.0 : 2.0) * pv(LO::F0 + tri_idx(r, q)) * dl[r] * dl[q];
        if (i > 0) {
          double t = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q < N; ++q) t += dprev[r] * pvp(LO::F4 + r * N + q) * dl[q];
          mahal += 2.0 * t;
        }
        if (COMMIT && write) {
          double dp[N], Pn[T];
#pragma unroll
          for (int q = 0; q < T; ++q)
            Pn[q] = ((pv(LO::F1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::F0 + q) * inv_b) * c;
#pragma unroll
          for (int r = 0; r < N; ++r) {
            a.o_mu[(i * N + r) * a.Bp + b] = m[r];
            dp[r] = m[r] - pv(LO::F3 + r);
          }
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q)
              pq_c += ((q == r) ? 1.0 : 2.0) * kv(LO::K0 + tri_idx(r, q)) * dp[r] * dp[q];
          double pt[N];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += sym_at<N>(Pn, r, q) * m[q];
            if (i > 0) {
#pragma unroll
              for (int q = 0; q < N; ++q)
                t += ((kvp(LO::K1 + q * N + r) * inv_t + pvp(LO::F4 + q * N + r) * inv_b) * c) * mprev[q];
            }
            pt[r] = t;
          }
          if (i > 0) {
            double t2 = 0.0;
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q < N; ++q) t2 += dpprev[r] * kvp(LO::K1 + r * N + q) * dp[q];
            pq_c += 2.0 * t2;
#pragma unroll
            for (int r = 0; r < N; ++r) {
              double t = part[r];
#pragma unroll
              for (int q = 0; q < N; ++q)
                t += ((kvp(LO::K1 + r * N + q) * inv_t + pvp(LO::F4 + r * N + q) * inv_b) * c) * m[q];
              a.o_v[((i - 1) * N + r) * a.Bp + b] = t;
            }
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            part[r] = pt[r];
            dpprev[r] = dp[r];
          }
          if (i == K - 1) {
#pragma unroll
            for (int r = 0; r < N; ++r) a.o_v[(i * N + r) * a.Bp + b] = pt[r];
          }
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          mprev[r] = m[r];
          dprev[r] = dl[r];
        }
      }
      if (passF && role == 0) {
        // ---- tr(Lambda_ii Sigma_ii)
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q)
            trace += ((q == r) ? 1.0 : 2.0) * pv(LO::F0 + tri_idx(r, q)) * Sig[tri_idx(r, q)];
        if (COMMIT && write) {
#pragma unroll
          for (int q = 0; q < T; ++q) {
            a.o_ld[(i * T + q) * a.Bp + b] =
                ((pv(LO::F1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::F0 + q) * inv_b) * c;
            a.o_cov[(i * T + q) * a.Bp + b] = Sig[q];
          }
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q)
              ptr_c += ((q == r) ? 1.0 : 2.0) * kv(LO::K0 + tri_idx(r, q)) * Sig[tri_idx(r, q)];
        }
        if (i + 1 < K) {
          // M = Sigma_ii U' Phi^{-1} = -Sigma_{i,i+1};  Sigma_{i+1} = Phi^{-1} + (U' Phi^{-1})^T M
          double Up[N2], M[N2], bm[N2];
#pragma unroll
          for (int q = 0; q < N2; ++q) Up[q] = (kv(LO::K1 + q) * inv_t + pv(LO::F4 + q) * inv_b) * c;
          // U' Phi_{i+1}^{-1}
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q < N; ++q) {
              double t = 0.0;
#pragma unroll
              for (int k2 = 0; k2 < N; ++k2)
                t += Up[r * N + k2] * phi(k2 >= q ? tri_idx(k2, q) : tri_idx(q, k2));
              bm[r * N + q] = t;
            }
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q < N; ++q) {
              double t = 0.0;
#pragma unroll
              for (int k2 = 0; k2 < N; ++k2) t += sym_at<N>(Sig, r, k2) * bm[k2 * N + q];
              M[r * N + q] = t;
            }
          double tc = 0.0;
#pragma unroll
          for (int q = 0; q < N2; ++q) tc += pv(LO::F4 + q) * M[q];
          trace -= 2.0 * tc;  // 2 <Lambda_{i,i+1}, Sigma_{i,i+1}>
          if (COMMIT && write) {
            double tk = 0.0;
#pragma unroll
            for (int q = 0; q < N2; ++q) {
              a.o_cr[(i * N2 + q) * a.Bp + b] = -M[q];
              a.o_lo[(i * N2 + q) * a.Bp + b] = Up[q];
              tk += kv(LO::K1 + q) * M[q];
            }
            ptr_c -= 2.0 * tk;
          }
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q) {
              double t = 0.0;
#pragma unroll
              for (int k2 = 0; k2 < N; ++k2) t += bm[k2 * N + r] * M[k2 * N + q];
              Sig[tri_idx(r, q)] = phi(tri_idx(r, q)) + t;
            }
        }
      }
    }
    sbase += K;
    __syncthreads();

    // ---------------- KL of each lane: role A holds trace + log det, role B mahal + shift
    // each role publishes its quantities: A -> trace, ptr, log det; B -> mahal, pq, shift
    xch[(0 * 2 + role) * 32 + lcol] = role == 0 ? trace : mahal;
    xch[(1 * 2 + role) * 32 + lcol] = ld_sum;
    xch[(2 * 2 + role) * 32 + lcol] = sh2;
    xch[(3 * 2 + role) * 32 + lcol] = role == 0 ? ptr_c : pq_c;
    __syncthreads();
    const double o_trace_or_mahal = xch[(0 * 2 + 1 - role) * 32 + lcol];
    const double o_ld = xch[(1 * 2 + 1 - role) * 32 + lcol];
    const double o_sh = xch[(2 * 2 + 1 - role) * 32 + lcol];
    const double o_pq = xch[(3 * 2 + 1 - role) * 32 + lcol];
    __syncthreads();
    const double tr_ = role == 0 ? trace : o_trace_or_mahal;
    const double mh_ = role == 0 ? o_trace_or_mahal : mahal;
    const double ld_ = role == 0 ? ld_sum : o_ld;
    const double sh_ = role == 0 ? o_sh : sh2;
    const double ptr_ = role == 0 ? ptr_c : o_pq, pq_ = role == 0 ? o_pq : pq_c;
    double klv = 0.0;
    if (passF) {
      const double x = 0.5 * ((((tr_ + mh_) - (double)(K * N)) + ld_) - ldc);
      klv = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
    }
    if (COMMIT && write && role == 0) {
      a.beta[b] = beta;
      a.kl[b] = klv;
      a.ld_next[b] = ld_;
      a.shift[b] = sqrt(sh_);
      if (a.prior_cost) a.prior_cost[b] = 0.5 * pq_ + 0.5 * ptr_;
    }

    // ---------------- per-plan decision (the reference's sequential logic),
    // one thread per plan over the results of the slots that served it
    if (role == 0) {
      r_beta[lcol] = beta;
      r_kl[lcol] = klv;
      r_res[lcol] = res;
      r_fail[lcol] = fail_knot;
      r_on[lcol] = lane_on ? 1 : 0;
    }
    __syncthreads();
    if (my_rank >= 0) {
      const int j = tid;
      const int base = my_rank * kl;
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
          if (walk()) D.phase = ((D.hi - D.lo) > 1e-3 * D.hi) ? 2 : 3;
        }
      } else if (D.phase == 2) {
        if (walk()) D.phase = ((D.hi - D.lo) > 1e-3 * D.hi) ? 2 : 3;
      }
      if (!COMMIT && D.phase == 3) {  // search finished: hand beta to the commit kernel
        a.beta[bj] = D.best;
        a.status[bj] = GVP_OK;
        a.where[bj] = -1;
        if (a.nprobes) a.nprobes[bj] = D.nprobe;
        D.phase = 4;
      }
      pst[j] = D;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
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
static int make_map(CUtensorMap* m, const double* base, int64_t W, int64_t E, int64_t K, int bw,
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

int64_t step_scratch_doubles(int nplans, int64_t K, int n, int lanes) {
  const int64_t T = (int64_t)n * (n + 1) / 2;
  const int64_t BL = (((int64_t)nplans + 1) & ~1LL) * lanes + 64;  // padded columns
  return std::max<int64_t>(1, K * (2 * T + n) * BL);
}

int64_t step_plan_stride(int nplans) { return std::max<int64_t>(2, ((int64_t)nplans + 1) & ~1LL); }

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

static int launch_v3(const V2Launch& q, const int L, const bool commit, cudaStream_t s) {
  // two warps per 32 lane slots (warp-specialised roles); 32 / L plans per CTA
  // (even for L <= 16, so every TMA box starts on a 16-byte plan boundary)
  const int TB = 64;
  // Fill all 32 lane slots (B200, C5 at L = 1: 32 plans/CTA 47 ms vs 8 plans/CTA
  // 104 ms — the per-knot TMA issue + barrier cost is paid per CTA).
  const int P = 32 / L;
  const int Pb = round_up(P, 2);
  const int Kb = q.kshared ? 2 : Pb;
  const int n = q.n;
  const int T = n * (n + 1) / 2, N2 = n * n, SE = 2 * T + n;
  v3::Args a;
  std::memset(&a, 0, sizeof(a));
  a.B = q.nplans;
  a.K = q.K;
  a.Bp = q.Bp;
  a.P = P;
  a.Pbox = Pb;
  a.Kbox = Kb;
  a.ksp = q.kshared ? 0 : 1;
  const int64_t K = q.K, K1 = std::max<int64_t>(K - 1, 1);
  const int64_t KW = q.kshared ? 2 : q.Bp;
  const int64_t BLp = (q.Bp * L) + 64;
  int r;
  if ((r = v3::make_map(&a.m_ld, q.ld, q.Bp, T, K, Pb, T)) || (r = v3::make_map(&a.m_lo, q.lo, q.Bp, N2, K1, Pb, N2)) ||
      (r = v3::make_map(&a.m_kd, q.kd, KW, T, K, Kb, T)) || (r = v3::make_map(&a.m_ko, q.ko, KW, N2, K1, Kb, N2)) ||
      (r = v3::make_map(&a.m_gd, q.gd, q.Bp, T, K, Pb, T)) || (r = v3::make_map(&a.m_g, q.g, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_eta, q.eta, q.Bp, n, K, Pb, n)) || (r = v3::make_map(&a.m_v, q.v, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_mu, q.mu, q.Bp, n, K, Pb, n)) || (r = v3::make_map(&a.m_pm, q.pmean, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_phi, q.scratch, BLp, SE, K, P * L < 2 ? 2 : P * L, T)) ||
      (r = v3::make_map(&a.m_psiy, q.scratch, BLp, SE, K, P * L < 2 ? 2 : P * L, T + n)))
    return r;
  a.o_mu = q.o_mu; a.o_ld = q.o_ld; a.o_lo = q.o_lo; a.o_cov = q.o_cov; a.o_cr = q.o_cr; a.o_v = q.o_v;
  a.beta = q.beta; a.kl = q.kl; a.ld_next = q.ld_next; a.shift = q.shift; a.prior_cost = q.prior_cost;
  a.temp = q.temp; a.ld_cur = q.ld_cur;
  a.kl_bound = q.kl_bound; a.beta_min = q.beta_min; a.beta_max = q.beta_max;
  a.status = q.status; a.where = q.where; a.nprobes = q.nprobes;
  a.probe_log = q.probe_log; a.max_probes = q.max_probes;
  a.scratch = q.scratch;
  a.BLp = BLp;
  a.active = q.active;
  // one stage: plan rows | prior rows | PHI rows (lanes) | LIPSI+Y rows (lanes).
  // Every array's box starts on a 128-byte boundary (TMA destination rule):
  // row starts are rounded to a multiple of 16 / gcd(width, 16) rows.
  const int LPb = P * L < 2 ? 2 : P * L;
  auto gran = [](int width) {
    int g = 16;
    while (g > 1 && (width * g) % 16 == 0 && (width * (g / 2)) % 16 == 0) g /= 2;
    return g;
  };
  auto layout = [&](const int* sizes, int cnt, int width, int* starts) {
    const int g = gran(width);
    int row = 0;
    for (int k = 0; k < cnt; ++k) {
      starts[k] = row;
      row = round_up(row + sizes[k], g);
    }
    return row;
  };
  const int szB[6] = {T, T, n, n, n, N2}, szF[5] = {T, T, n, n, N2}, szK[2] = {T, N2};
  const int rowsB = layout(szB, 6, Pb, a.rB), rowsF = layout(szF, 5, Pb, a.rF);
  const int rowsK = layout(szK, 2, Kb, a.rK);
  a.off_plan = 0;
  a.off_prior = round_up(std::max(rowsB, rowsF) * Pb, 16);
  a.off_phi = a.off_prior + round_up(rowsK * Kb, 16);
  a.off_psiy = a.off_phi + round_up(T * LPb, 16);
  a.stage_doubles = a.off_psiy + round_up((T + n) * LPb, 16);
  a.bm_off = v3::kStages * a.stage_doubles;
  a.bar_off = a.bm_off + 8 * 32;  // role exchange: 4 doubles x 2 roles x 32 lane slots
  a.bytes_B = (uint32_t)(((2 * T + 3 * n + N2) * Pb + (T + N2) * Kb) * 8);
  a.bytes_F = (uint32_t)(((2 * T + 2 * n + N2) * Pb + (T + N2) * Kb + (2 * T + n) * LPb) * 8);
  (void)SE;
  const size_t bytes = (size_t)(a.bar_off + 2 * v3::kStages) * sizeof(double) + 1024;
  const unsigned grid = (unsigned)((q.nplans + P - 1) / P);
#define GVP_V3_KS(NN, LL, CC, KK)                                                               \
  {                                                                                             \
    using LOH = v3::Lay<NN, LL, KK>;                                                            \
    if (LOH::TX_B != a.bytes_B || LOH::TX_F != a.bytes_F || LOH::STAGE != a.stage_doubles) {   \
      set_error("internal: device/host stage layout mismatch");                                 \
      return GVP_ERR_ARG;                                                                       \
    }                                                                                           \
    GVP_CUDA(cudaFuncSetAttribute(v3::select_step_v3_kernel<NN, LL, CC, KK>,                    \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LOH::BYTES)); \
    v3::select_step_v3_kernel<NN, LL, CC, KK><<<grid, TB, LOH::BYTES, s>>>(a);                  \
  }
#define GVP_V3(NN, LL, CC)                                 \
  if (q.kshared) GVP_V3_KS(NN, LL, CC, true) else GVP_V3_KS(NN, LL, CC, false)
#define GVP_V3_L(NN)                           \
  if (commit) {                                \
    GVP_V3(NN, 1, true)                        \
  } else {                                     \
    switch (L) {                               \
      case 1: GVP_V3(NN, 1, false) break;      \
      case 4: GVP_V3(NN, 4, false) break;      \
      case 8: GVP_V3(NN, 8, false) break;      \
      default: GVP_V3(NN, 16, false) break;    \
    }                                          \
  }
  switch (n) {
    case 2: GVP_V3_L(2) break;
    case 4: GVP_V3_L(4) break;
    case 6: GVP_V3_L(6) break;
    default:
      set_error("step kernel supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_V3_L
#undef GVP_V3
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

// bisection (L candidate lanes per plan), then the commit of the accepted beta
int launch_select_step_v2(const V2Launch& q, cudaStream_t s) {
  if (q.nplans == 0 || q.K == 0) return GVP_OK;
  const int L = q.lanes;
  if (L != 1 && L != 4 && L != 8 && L != 16) {
    set_error("lanes must be 1, 4, 8 or 16");
    return GVP_ERR_ARG;
  }
  if (q.Bp % 2 || q.Bp < 2) {
    set_error("plan stride must be even (step_plan_stride)");
    return GVP_ERR_ARG;
  }
  int r = launch_v3(q, L, false, s);
  if (r) return r;
  return launch_v3(q, 1, true, s);
}

}  // namespace gvp
