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
#include <cstdlib>
#include <cstring>

#include "gvp_internal.cuh"
#include "step_common.cuh"

namespace gvp {
namespace v3 {

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
template <int N, int L, bool KS, bool CM>
struct Lay {
  static constexpr int T = N * (N + 1) / 2, N2 = N * N;
  // LPb: scratch columns per CTA — one per lane slot in the bisection, one per
  // plan in the commit (only its write slot runs)
  static constexpr int P = 32 / L, Pb = P, Kb = KS ? 2 : P, LPb = CM ? P : 32;
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
  static constexpr int NS = ring_stages(STAGE), AH = NS - 2;  // slot of knot i-1 stays valid at knot i
  static constexpr int XCH = NS * STAGE, BAR = XCH + 8 * 32;
  static constexpr int PST = BAR + 16;        // per-plan bisection state (10 doubles x 32)
  static constexpr int RES = PST + 10 * 32;   // per-slot probe results (5 x 32)
  static constexpr size_t BYTES = (size_t)(RES + 5 * 32) * 8;
  static constexpr uint32_t TX_B = ((2 * T + 3 * N + N2) * Pb + (T + N2) * Kb) * 8;
  static constexpr uint32_t TX_F = ((2 * T + 2 * N + N2) * Pb + (T + N2) * Kb + (2 * T + N) * LPb) * 8;
};

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
  using LO = Lay<N, L, KS, COMMIT>;
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
    for (int s = 0; s < LO::NS; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  search_init(a, pst, P, b0, COMMIT, tid);
  __syncthreads();

  double* scr = a.scratch;
  // global scratch column: per lane slot (bisection) / per plan (commit)
  auto sc_column = [&](int p_) -> int64_t { return COMMIT ? b0 + p_ : b0 * L + lcol; };

  auto slot = [&](int64_t s) { return smem + (s % LO::NS) * LO::STAGE; };
  // issue the TMA loads of one knot of a pass into slot s % NS
  auto issue = [&](int64_t s, int64_t i, bool passB) {
    double* st = slot(s);
    uint64_t* bar = &bars[s % LO::NS];
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
      const int sc0 = (int)(COMMIT ? b0 : b0 * L);
      tma3(st + LO::OFF_PHI, &a.m_phi, sc0, 0, (int)(i + 1), bar);        // PHIINV of knot i+1
      tma3(st + LO::OFF_PSIY, &a.m_psiy, sc0, Y::S_LIPSI, (int)i, bar);  // LIPSI | Y of knot i
    }
  };
  auto wait_slot = [&](int64_t s) {
    mbar_wait(&bars[s % LO::NS], (uint32_t)((s / LO::NS) & 1));
  };

  for (;;) {
    const Pick pk = search_pick(a, pst, P, LP, lcol, tid, COMMIT);
    if (pk.kl == 0) break;  // uniform: every thread read the same shared state
    const int p = pk.p, kl = pk.kl, my_rank = pk.my_rank;
    const int64_t b = b0 + p;
    const int kcol = KS ? 0 : p;
    const double temp = pst[p].temp, ldc = pst[p].ldc;
    const bool lane_on = pk.on, write = pk.on && pk.write;
    const double beta = pk.beta;
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
      for (int s = 0; s < LO::AH && s < K; ++s) issue(s, K - 1 - s, true);
    for (int64_t s = 0; s < K; ++s) {
      wait_slot(s);
      __syncthreads();  // everyone past knot s-1: its slot may be refilled
      if (tid == 0 && s + LO::AH < K) issue(s + LO::AH, K - 1 - (s + LO::AH), true);
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
      double* sc = scr + (i * SE) * a.BLp + sc_column(p);
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
      const double* sc = scr + sc_column(p);  // Sigma_00 = Phi_0^{-1}
#pragma unroll
      for (int q = 0; q < T; ++q) Sig[q] = sc[(Y::S_PHI + q) * a.BLp];
    }
    if (tid == 0)
      for (int s = 0; s < LO::AH && s < K; ++s) issue(sbase + s, s, false);
    for (int64_t i = 0; i < K; ++i) {
      const int64_t s = sbase + i;
      wait_slot(s);
      __syncthreads();
      if (tid == 0 && i + LO::AH < K) issue(s + LO::AH, i + LO::AH, false);
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
      const int scs = COMMIT ? p : lcol;  // this slot's scratch column in the stage
      auto phi = [&](int q) { return st[LO::OFF_PHI + q * LO::LPb + scs]; };
      auto psi = [&](int q) { return st[LO::OFF_PSIY + q * LO::LPb + scs]; };  // LIPSI rows then Y rows
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
    if (my_rank >= 0)
      search_decide(a, pst, tid, my_rank * kl, kl, b0, COMMIT, r_beta, r_kl, r_res, r_fail, r_on);
    __syncthreads();
  }
}

}  // namespace v3

int64_t step_scratch_doubles(int nplans, int64_t K, int n, int lanes) {
  const int64_t T = (int64_t)n * (n + 1) / 2;
  const int64_t BL = (((int64_t)nplans + 1) & ~1LL) * lanes + 64;  // padded columns
  // two-pass bisection scratch, or commit scratch + the one-pass probe's residual
  const int64_t two_pass = K * (2 * T + n) * BL;
  const int64_t one_pass = probe_residual_offset(nplans, K, n) + K * n * step_plan_stride(nplans);
  return std::max<int64_t>(1, std::max(two_pass, one_pass));
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
  // scratch columns: one per lane slot (bisection) or one per plan (commit)
  const int SW = commit ? Pb : (P * L < 2 ? 2 : P * L);
  const int64_t BLp = (commit ? q.Bp : q.Bp * L) + 64;
  int r;
  if ((r = v3::make_map(&a.m_ld, q.ld, q.Bp, T, K, Pb, T)) || (r = v3::make_map(&a.m_lo, q.lo, q.Bp, N2, K1, Pb, N2)) ||
      (r = v3::make_map(&a.m_kd, q.kd, KW, T, K, Kb, T)) || (r = v3::make_map(&a.m_ko, q.ko, KW, N2, K1, Kb, N2)) ||
      (r = v3::make_map(&a.m_gd, q.gd, q.Bp, T, K, Pb, T)) || (r = v3::make_map(&a.m_g, q.g, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_eta, q.eta, q.Bp, n, K, Pb, n)) || (r = v3::make_map(&a.m_v, q.v, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_mu, q.mu, q.Bp, n, K, Pb, n)) || (r = v3::make_map(&a.m_pm, q.pmean, q.Bp, n, K, Pb, n)) ||
      (r = v3::make_map(&a.m_phi, q.scratch, BLp, SE, K, SW, T)) ||
      (r = v3::make_map(&a.m_psiy, q.scratch, BLp, SE, K, SW, T + n)))
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
  const int LPb = SW;
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
  a.bm_off = 0;
  a.bar_off = a.bm_off + 8 * 32;  // role exchange: 4 doubles x 2 roles x 32 lane slots
  a.bytes_B = (uint32_t)(((2 * T + 3 * n + N2) * Pb + (T + N2) * Kb) * 8);
  a.bytes_F = (uint32_t)(((2 * T + 2 * n + N2) * Pb + (T + N2) * Kb + (2 * T + n) * LPb) * 8);
  (void)SE;
  const unsigned grid = (unsigned)((q.nplans + P - 1) / P);
#define GVP_V3_KS(NN, LL, CC, KK)                                                               \
  {                                                                                             \
    using LOH = v3::Lay<NN, LL, KK, CC>;                                                            \
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
    switch (L) {                               \
      case 1: GVP_V3(NN, 1, true) break;       \
      case 4: GVP_V3(NN, 4, true) break;       \
      default: GVP_V3(NN, 16, true) break;     \
    }                                          \
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

// bisection (L candidate lanes per plan): the accepted beta of each plan -> q.beta
int launch_select_bisect(const V2Launch& q, cudaStream_t s) {
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
  // GVP_TWO_PASS=1 selects the two-pass bisection kernel (A/B comparisons)
  static const bool two_pass = [] {
    const char* e = std::getenv("GVP_TWO_PASS");
    return e && e[0] == '1';
  }();
  return two_pass ? launch_v3(q, L, false, s) : launch_probe(q, L, s);
}

// the commit of the accepted beta: next iterate, marginals, KL, log det, costs
int launch_select_commit(const V2Launch& q, cudaStream_t s) {
  if (q.nplans == 0 || q.K == 0) return GVP_OK;
  // One write-mode probe per plan. The commit is bound by each warp's serial
  // per-knot latency (and TMA latency), not by lanes: few plans per CTA keep
  // the stage small (deep prefetch ring) and spread plans over more SMs.
  // GVP_COMMIT_LANES overrides (A/B measurements).
  static const int forced = [] {
    const char* e = std::getenv("GVP_COMMIT_LANES");
    return e ? std::atoi(e) : 0;
  }();
  // default: the 4-warp commit (commit.cu); GVP_COMMIT_LANES selects this file's kernel
  if (forced == 0) return launch_commit_split(q, s);
  const int L = forced == 1 || forced == 4 || forced == 16 ? forced : (q.nplans <= 2 ? 16 : 1);
  return launch_v3(q, L, true, s);
}

int launch_select_step_v2(const V2Launch& q, cudaStream_t s) {
  int r = launch_select_bisect(q, s);
  if (r) return r;
  return launch_select_commit(q, s);
}

}  // namespace gvp
