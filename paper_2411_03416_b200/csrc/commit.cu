// Kernel (b)+(c), commit half: the accepted beta of every plan re-probed once
// in write mode (optimizer.py:129-177 for the chosen beta): next mean mu',
// precision Lambda', GBP marginals Sigma_ii / Sigma_i,i+1 (gbp.py:43-80), KL,
// log det, prior cost (optimizer.py:238-256) and Lambda' mu' for the next rhs.
//
// Exact two-pass scheme (the reference's quantities, not the probe's tangents):
//   pass B (K-1 .. 0)  warp 0: backward GBP Schur of Lambda' -> Phi^-1 (scratch),
//                      log det;  warp 1: backward elimination of the mean system
//                      S mu' = rhs -> Li, y (scratch)
//   pass F (0 .. K-1)  warp 0: covariance recursion Sigma_{i+1} = Phi^-1 +
//                      (U' Phi^-1)' Sigma_ii (U' Phi^-1);  warp 1: forward
//                      substitution mu'_i and the Mahalanobis term;
//                      warps 2/3 (one knot behind, fed through a shared-memory
//                      ring): every output store, tr(Lambda Sigma'), the prior
//                      cost terms and Lambda' mu'.
// The commit is bound by each warp's serial per-knot instruction stream (one
// CTA of 32 plans per SM), so moving the side work off the two recursion warps
// shortens the critical path (C5: 2.55 -> 1.83 ms against the 2-warp version).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "gvp_internal.cuh"
#include "step_common.cuh"

namespace gvp {
namespace v5 {

using v3::T_;
using v3::cx_gran;
using v3::cx_round;

template <int N, bool KS>
struct Lay {
  static constexpr int T = T_<N>, N2 = N * N, SE = 2 * T + N;
  // scratch entries per knot per plan: PHIINV | LIPSI | Y
  static constexpr int S_PHI = 0, S_LIPSI = T, S_Y = 2 * T;
  static constexpr int P = 32, Pb = 32, Kb = KS ? 2 : 32;
  static constexpr int gP = cx_gran(Pb), gK = cx_gran(Kb);
  // pass B plan rows: LD T | GD T | E N | (unused N | unused N) | LO N2
  static constexpr int B0 = 0, B1 = cx_round(T, gP), B2 = cx_round(B1 + T, gP), B3 = cx_round(B2 + N, gP),
                       B4 = cx_round(B3 + N, gP), B5 = cx_round(B4 + N, gP), BR = cx_round(B5 + N2, gP);
  // pass F plan rows: LD T | GD T | MU N | PM N | LO N2
  static constexpr int F0 = 0, F1 = cx_round(T, gP), F2 = cx_round(F1 + T, gP), F3 = cx_round(F2 + N, gP),
                       F4 = cx_round(F3 + N, gP), FR = cx_round(F4 + N2, gP);
  // prior rows: KD T | KO N2
  static constexpr int K0 = 0, K1 = cx_round(T, gK), KR = cx_round(K1 + N2, gK);
  static constexpr int OFF_PRIOR = cx_round((BR > FR ? BR : FR) * Pb, 16),
                       OFF_PHI = OFF_PRIOR + cx_round(KR * Kb, 16),
                       OFF_PSIY = OFF_PHI + cx_round(T * Pb, 16),
                       STAGE = OFF_PSIY + cx_round((T + N) * Pb, 16);
  // chain -> side ring (2 steps): Sigma_ii T | M N2 (A), mu' N (B), per plan
  static constexpr int ENT = T + N2 + N, E_SIG = 0, E_M = T, E_MU = T + N2;
  static constexpr int RING_D = 2 * ENT * 32;
  static constexpr int MISC = 8 * 32 + 16;  // exchange + barriers
  // as many stages as fit in ~200 KB (one CTA per SM), at most 8
  static constexpr int NS_FIT = (25600 - RING_D - MISC) / STAGE;
  static constexpr int NS = NS_FIT > 8 ? 8 : (NS_FIT < 4 ? 4 : NS_FIT);
  static constexpr int AH = NS - 3;  // pass F: side warps still read knots s-1 and s-2
  static constexpr int RING = NS * STAGE, XCH = RING + RING_D, BAR = XCH + 8 * 32;
  static constexpr size_t BYTES = (size_t)(BAR + 16) * 8;
  static constexpr uint32_t TX_B = ((2 * T + N + N2) * Pb + (T + N2) * Kb) * 8;
  static constexpr uint32_t TX_F = ((2 * T + 2 * N + N2) * Pb + (T + N2) * Kb + (2 * T + N) * Pb) * 8;
};

struct Args {
  CUtensorMap m_ld, m_lo, m_kd, m_ko, m_gd, m_e, m_mu, m_pm, m_phi, m_psiy;
  int B;
  int64_t K, Bp, BLp;
  double *o_mu, *o_ld, *o_lo, *o_cov, *o_cr, *o_v;
  const double* beta;
  double *kl, *ld_next, *shift, *prior_cost;
  const double *temp, *ld_cur;
  int *status, *where;
  double* scratch;
  const int* active;
  // search_kl: the search already wrote the accepted probe's KL and forward
  // log det (step.kl, optimizer.py:209-211); the commit writes its own only
  // where fixkl[b] != 0 (a step size that was not probed, gvp_engine_step_beta)
  int search_kl;
  const int* fixkl;
};

template <int N>
GVP_DEV double symv(const double (&A)[T_<N>], int r, int c) {
  return r >= c ? A[tri_idx(r, c)] : A[tri_idx(c, r)];
}

#ifdef GVP_COMMIT_PROFILE
__device__ unsigned long long g_commit_prof[3];  // diagnostic build (tools/commit_profile.py)
__device__ unsigned long long g_commit_role[2][4][2];  // [pass B / F][warp][work, wait] cycles
#endif

template <int N, bool KS>
__global__ void __launch_bounds__(128, 1) commit_kernel(const __grid_constant__ Args a) {
  using LO = Lay<N, KS>;
  constexpr int T = LO::T, N2 = LO::N2, SE = LO::SE;
  constexpr int Pb = LO::Pb, Kb = LO::Kb;
  extern __shared__ __align__(1024) double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LO::BAR);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int role = warp & 1;            // 0: Lambda' / covariance, 1: mean
  const bool side = warp >= 2;          // output warps, one knot behind
  const int p = tid & 31;               // plan column in the CTA
  const int64_t b0 = (int64_t)blockIdx.x * 32;
  const int64_t b = b0 + p;
  const int kcol = KS ? 0 : p;
  const int K = (int)a.K;  // 32-bit step arithmetic (every loop-control op one integer op)
  double* ring = smem + LO::RING;
  double* xch = smem + LO::XCH;

  if (tid == 0) {
    for (int s = 0; s < LO::NS; ++s) v3::mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const bool ok = b < a.B && (!a.active || a.active[b]) && a.status[b] == GVP_OK;
  const double beta = ok ? a.beta[b] : 1.0;
  const double temp = ok ? a.temp[b] : 1.0, ldc = ok ? a.ld_cur[b] : 0.0;
  const double inv_t = 1.0 / temp, two_t = 2.0 / temp;
  const double inv_b = ok ? 1.0 / beta : 0.0, c = ok ? beta / (beta + 1.0) : 0.0;
  double* scr = a.scratch + b;

  auto slot = [&](int s) { return smem + ((unsigned)s % LO::NS) * LO::STAGE; };
  auto issue = [&](int s, int i, bool passB) {
    double* st = slot(s);
    uint64_t* bar = &bars[(unsigned)s % LO::NS];
    v3::mbar_expect_tx(bar, passB ? LO::TX_B : LO::TX_F);
    const int ck = KS ? 0 : (int)b0;
    double* pr = st + LO::OFF_PRIOR;
    v3::tma3(pr + LO::K0 * Kb, &a.m_kd, ck, 0, (int)i, bar);
    v3::tma3(pr + LO::K1 * Kb, &a.m_ko, ck, 0, (int)i, bar);
    if (passB) {
      v3::tma3(st + LO::B0 * Pb, &a.m_ld, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::B1 * Pb, &a.m_gd, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::B2 * Pb, &a.m_e, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::B5 * Pb, &a.m_lo, (int)b0, 0, (int)i, bar);
    } else {
      v3::tma3(st + LO::F0 * Pb, &a.m_ld, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::F1 * Pb, &a.m_gd, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::F2 * Pb, &a.m_mu, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::F3 * Pb, &a.m_pm, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::F4 * Pb, &a.m_lo, (int)b0, 0, (int)i, bar);
      v3::tma3(st + LO::OFF_PHI, &a.m_phi, (int)b0, 0, (int)(i + 1), bar);        // PHIINV of knot i+1
      v3::tma3(st + LO::OFF_PSIY, &a.m_psiy, (int)b0, LO::S_LIPSI, (int)i, bar);  // LIPSI | Y of knot i
    }
  };
  auto wait = [&](int s) { v3::mbar_wait(&bars[(unsigned)s % LO::NS], ((unsigned)s / LO::NS) & 1u); };
  auto rg = [&](int st, int e) -> double* { return ring + ((int)(st & 1) * LO::ENT + e) * 32 + p; };

#ifdef GVP_COMMIT_PROFILE
  const long long pc0 = clock64();
#endif
  // =============================== pass B: knots K-1 .. 0 (warps 0, 1)
  int res = 0, fail_knot = -1;
  double pm = 1.0;
  int pe = 0;
  {
    double LiN[T], yN[N];
    if (tid == 0)
      for (int s = 0; s < LO::AH + 1 && s < K; ++s) issue(s, K - 1 - s, true);
#ifdef GVP_COMMIT_PROFILE
    long long rp_prev = clock64(), rp_work = 0, rp_wait = 0;
#endif
    for (int s = 0; s < K; ++s) {
#ifdef GVP_COMMIT_PROFILE
      const long long rp0 = clock64();
#endif
      wait(s);
      __syncthreads();
#ifdef GVP_COMMIT_PROFILE
      const long long rp1 = clock64();
      rp_work += rp0 - rp_prev;
      rp_wait += rp1 - rp0;
      rp_prev = rp1;
#endif
      if (tid == 0 && s + LO::AH + 1 < K) issue(s + LO::AH + 1, K - 1 - (s + LO::AH + 1), true);
      const int i = K - 1 - s;
      if (side || !ok || res != 0) continue;
      const double* st = slot(s);
      const double* pr = st + LO::OFF_PRIOR;
      auto pv = [&](int row) { return st[row * Pb + p]; };
      auto kv = [&](int row) { return pr[row * Kb + kcol]; };
      double A_[T], rhs[N];
      if (role == 0) {  // Lambda' diag block (optimizer.py:151-153)
#pragma unroll
        for (int q = 0; q < T; ++q)
          A_[q] = ((pv(LO::B1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::B0 + q) * inv_b) * c;
      } else {  // S diag block (optimizer.py:155-159); the system is solved for the
                // step delta = mu - mu' = S^-1 e, e = S mu - rhs = (K mu + g - eta) / T
                // (beta-free, the probes' residual): |delta| << |mu| keeps the
                // cond(S) ~ 1e10 rounding relative to the step, not the iterate
#pragma unroll
        for (int q = 0; q < T; ++q) A_[q] = kv(LO::K0 + q) * inv_t + pv(LO::B0 + q) * inv_b;
#pragma unroll
        for (int r = 0; r < N; ++r) rhs[r] = pv(LO::B2 + r) * inv_t;
      }
      if (i < K - 1) {
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
      if (!v3::chol_inv<N>(A_, Li, pp)) {
        res = role == 0 ? 1 : 2;
        fail_knot = (int)i;
        continue;
      }
      double* sc = scr + (i * SE) * a.BLp;
      if (role == 0) {
        int ex;
        pm = frexp_pos(pm * pp, &ex);
        pe += ex;
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k2 = r; k2 < N; ++k2) t += Li[tri_idx(k2, r)] * Li[tri_idx(k2, q)];
            sc[(LO::S_PHI + tri_idx(r, q)) * a.BLp] = t;
          }
      } else {
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int k2 = 0; k2 <= r; ++k2) t += Li[tri_idx(r, k2)] * rhs[k2];
          yN[r] = t;
          sc[(LO::S_Y + r) * a.BLp] = t;
        }
#pragma unroll
        for (int q = 0; q < T; ++q) sc[(LO::S_LIPSI + q) * a.BLp] = Li[q];
      }
#pragma unroll
      for (int q = 0; q < T; ++q) LiN[q] = Li[q];
    }
#ifdef GVP_COMMIT_PROFILE
    if ((tid & 31) == 0) {  // per warp: pass B work / wait cycles
      atomicAdd(&g_commit_role[0][warp][0], (unsigned long long)rp_work);
      atomicAdd(&g_commit_role[0][warp][1], (unsigned long long)rp_wait);
    }
#endif
  }
  v3::fence_proxy_async();  // scratch stores (generic proxy) -> TMA reads (async proxy)
  int* xi = reinterpret_cast<int*>(xch);
  if (!side) {
    xi[role * 32 + p] = res;
    xi[64 + role * 32 + p] = fail_knot;
  }
  __syncthreads();
  {
    const int rA = xi[p], rB = xi[32 + p];
    res = rB ? 2 : (rA ? 1 : 0);
    fail_knot = rB ? xi[96 + p] : xi[64 + p];
  }
  __syncthreads();
  const bool passF = ok && res == 0;

#ifdef GVP_COMMIT_PROFILE
  const long long pc1 = clock64();
#endif
  // =============================== pass F: knots 0 .. K-1 (+1 step for the side warps)
  double acc0 = 0.0, acc1 = 0.0;  // chain A: -; chain B: mahal, |delta|^2; side A: trace, tr(K Sigma); side B: pq
  {
    double Sig[T], mprev[N], dprev[N], part[N], dpprev[N];
    if (passF && !side && role == 0) {
#pragma unroll
      for (int q = 0; q < T; ++q) Sig[q] = scr[(LO::S_PHI + q) * a.BLp];  // Sigma_00 = Phi_0^-1
    }
    const int sbase = K;
    if (tid == 0)
      for (int s = 0; s < LO::AH && s < K; ++s) issue(sbase + s, s, false);
#ifdef GVP_COMMIT_PROFILE
    long long rf_prev = clock64(), rf_work = 0, rf_wait = 0;
#endif
    for (int st_ = 0; st_ <= K; ++st_) {
      const int s = sbase + st_;
#ifdef GVP_COMMIT_PROFILE
      const long long rf0 = clock64();
#endif
      if (st_ < K) wait(s);
      __syncthreads();
#ifdef GVP_COMMIT_PROFILE
      const long long rf1 = clock64();
      rf_work += rf0 - rf_prev;
      rf_wait += rf1 - rf0;
      rf_prev = rf1;
      if (st_ == K && (tid & 31) == 0) {  // per warp: pass F work / wait cycles
        atomicAdd(&g_commit_role[1][warp][0], (unsigned long long)rf_work);
        atomicAdd(&g_commit_role[1][warp][1], (unsigned long long)rf_wait);
      }
#endif
      if (tid == 0 && st_ + LO::AH < K) issue(s + LO::AH, st_ + LO::AH, false);
      if (!passF) continue;
      if (!side) {
        const int i = st_;
        if (i >= K) continue;
        const double* sg = slot(s);
        const double* pr = sg + LO::OFF_PRIOR;
        auto pv = [&](int row) { return sg[row * Pb + p]; };
        auto kv = [&](int row) { return pr[row * Kb + kcol]; };
        if (role == 1) {
          // ---- step: delta_i = Li^T (y_i - Li S_{i-1,i}^T delta_{i-1}); mu'_i = mu_i - delta_i
          const double* sp = slot(s - 1);
          const double* prp = sp + LO::OFF_PRIOR;
          auto pvp = [&](int row) { return sp[row * Pb + p]; };
          auto kvp = [&](int row) { return prp[row * Kb + kcol]; };
          auto psi = [&](int q) { return sg[LO::OFF_PSIY + q * Pb + p]; };  // LIPSI rows then Y rows
          double dl[N];
          {
            double z[N], w[N];
#pragma unroll
            for (int r = 0; r < N; ++r) {
              double t = 0.0;
              if (i > 0) {
#pragma unroll
                for (int q = 0; q < N; ++q)
                  t += (kvp(LO::K1 + q * N + r) * inv_t + pvp(LO::F4 + q * N + r) * inv_b) * dprev[q];
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
              dl[r] = t;  // delta = cur.mean - nxt.mean
            }
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            *rg(st_, LO::E_MU + r) = pv(LO::F2 + r) - dl[r];
            acc1 += dl[r] * dl[r];
          }
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q)
              acc0 += ((q == r) ? 1.0 : 2.0) * pv(LO::F0 + tri_idx(r, q)) * dl[r] * dl[q];
          if (i > 0) {
            double t = 0.0;
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q < N; ++q) t += dprev[r] * pvp(LO::F4 + r * N + q) * dl[q];
            acc0 += 2.0 * t;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) dprev[r] = dl[r];
        } else {
          // ---- covariance recursion (gbp.py:72-78)
#pragma unroll
          for (int q = 0; q < T; ++q) *rg(st_, LO::E_SIG + q) = Sig[q];
          if (i + 1 < K) {
            auto phi = [&](int q) { return sg[LO::OFF_PHI + q * Pb + p]; };
            double bm[N2], M[N2];
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q < N; ++q) {
                double t = 0.0;
#pragma unroll
                for (int k2 = 0; k2 < N; ++k2)
                  t += ((kv(LO::K1 + r * N + k2) * inv_t + pv(LO::F4 + r * N + k2) * inv_b) * c) *
                       phi(k2 >= q ? tri_idx(k2, q) : tri_idx(q, k2));
                bm[r * N + q] = t;  // U' Phi_{i+1}^-1
              }
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q < N; ++q) {
                double t = 0.0;
#pragma unroll
                for (int k2 = 0; k2 < N; ++k2) t += symv<N>(Sig, r, k2) * bm[k2 * N + q];
                M[r * N + q] = t;  // = -Sigma_{i,i+1}
              }
#pragma unroll
            for (int q = 0; q < N2; ++q) *rg(st_, LO::E_M + q) = M[q];
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
      } else {
        // ---------------------------- side warps, knot i = st_ - 1
        const int i = st_ - 1;
        if (i < 0) continue;
        const double* sg = slot(s - 1);
        const double* pr = sg + LO::OFF_PRIOR;
        auto pv = [&](int row) { return sg[row * Pb + p]; };
        auto kv = [&](int row) { return pr[row * Kb + kcol]; };
        if (role == 0) {
          double Sg[T];
#pragma unroll
          for (int q = 0; q < T; ++q) Sg[q] = *rg(st_ - 1, LO::E_SIG + q);
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q) {
              const double f = (q == r) ? 1.0 : 2.0;
              acc0 += f * pv(LO::F0 + tri_idx(r, q)) * Sg[tri_idx(r, q)];  // tr(Lambda_ii Sigma_ii)
              acc1 += f * kv(LO::K0 + tri_idx(r, q)) * Sg[tri_idx(r, q)];  // tr(K_ii Sigma_ii)
            }
#pragma unroll
          for (int q = 0; q < T; ++q) {
            a.o_ld[(i * T + q) * a.Bp + b] =
                ((pv(LO::F1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::F0 + q) * inv_b) * c;
            a.o_cov[(i * T + q) * a.Bp + b] = Sg[q];
          }
          if (i + 1 < K) {
            double tc = 0.0, tk = 0.0;
#pragma unroll
            for (int q = 0; q < N2; ++q) {
              const double Mq = *rg(st_ - 1, LO::E_M + q);
              tc += pv(LO::F4 + q) * Mq;
              tk += kv(LO::K1 + q) * Mq;
              a.o_cr[(i * N2 + q) * a.Bp + b] = -Mq;
              a.o_lo[(i * N2 + q) * a.Bp + b] = (kv(LO::K1 + q) * inv_t + pv(LO::F4 + q) * inv_b) * c;
            }
            acc0 -= 2.0 * tc;  // 2 <Lambda_{i,i+1}, Sigma_{i,i+1}>
            acc1 -= 2.0 * tk;
          }
        } else {
          const double* spp = slot(s - 2);  // knot i-1
          const double* prp = spp + LO::OFF_PRIOR;
          auto pvp = [&](int row) { return spp[row * Pb + p]; };
          auto kvp = [&](int row) { return prp[row * Kb + kcol]; };
          double m[N], dp[N], Pn[T], pt[N];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            m[r] = *rg(st_ - 1, LO::E_MU + r);
            a.o_mu[(i * N + r) * a.Bp + b] = m[r];
            dp[r] = m[r] - pv(LO::F3 + r);
          }
#pragma unroll
          for (int q = 0; q < T; ++q)
            Pn[q] = ((pv(LO::F1 + q) * two_t + kv(LO::K0 + q) * inv_t) + pv(LO::F0 + q) * inv_b) * c;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int q = 0; q <= r; ++q)
              acc0 += ((q == r) ? 1.0 : 2.0) * kv(LO::K0 + tri_idx(r, q)) * dp[r] * dp[q];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < N; ++q) t += symv<N>(Pn, r, q) * m[q];
            if (i > 0) {
#pragma unroll
              for (int q = 0; q < N; ++q)
                t += ((kvp(LO::K1 + q * N + r) * inv_t + pvp(LO::F4 + q * N + r) * inv_b) * c) * mprev[q];
            }
            pt[r] = t;
          }
          if (i > 0) {  // prior cross term and (Lambda' mu')_{i-1}
            double t2 = 0.0;
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q < N; ++q) t2 += dpprev[r] * kvp(LO::K1 + r * N + q) * dp[q];
            acc0 += 2.0 * t2;
#pragma unroll
            for (int r = 0; r < N; ++r) {
              double t = part[r];
#pragma unroll
              for (int q = 0; q < N; ++q)
                t += ((kvp(LO::K1 + r * N + q) * inv_t + pvp(LO::F4 + r * N + q) * inv_b) * c) * m[q];
              a.o_v[((i - 1) * N + r) * a.Bp + b] = t;
            }
          }
          if (i == K - 1) {
#pragma unroll
            for (int r = 0; r < N; ++r) a.o_v[(i * N + r) * a.Bp + b] = pt[r];
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            part[r] = pt[r];
            dpprev[r] = dp[r];
            mprev[r] = m[r];
          }
        }
      }
    }
  }
  // ---------------- KL and the records (optimizer.py:164-177, 238-256)
#ifdef GVP_COMMIT_PROFILE
  if (tid == 0) {  // diagnostic build: cycles of pass B / pass F, summed over CTAs
    const long long pc2 = clock64();
    atomicAdd(&g_commit_prof[0], (unsigned long long)(pc1 - pc0));
    atomicAdd(&g_commit_prof[1], (unsigned long long)(pc2 - pc1));
    atomicAdd(&g_commit_prof[2], 1ull);
  }
#endif
  xch[(2 * warp) * 32 + p] = acc0;
  xch[(2 * warp + 1) * 32 + p] = acc1;
  __syncthreads();
  if (tid < 32 && b < a.B && ok) {
    if (res != 0) {  // the probe said feasible; a failing exact pass is reported, not committed
      a.status[b] = GVP_ERR_NOT_SPD;
      a.where[b] = res == 2 ? (fail_knot | GVP_WHERE_MEAN_SOLVE_BIAS) : fail_knot;
    } else {
      const double ld = 2.0 * (log(pm) + (double)pe * 0.6931471805599453);
      const double mh = xch[2 * 32 + p], sh2 = xch[3 * 32 + p];
      const double tr = xch[4 * 32 + p], ptr = xch[5 * 32 + p], pq = xch[6 * 32 + p];
      const double x = 0.5 * ((((tr + mh) - (double)(K * N)) + ld) - ldc);
      if (!a.search_kl || (a.fixkl && a.fixkl[b])) {
        a.kl[b] = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
        a.ld_next[b] = ld;
      }
      a.shift[b] = sqrt(sh2);
      if (a.prior_cost) a.prior_cost[b] = 0.5 * pq + 0.5 * ptr;
    }
  }
}

}  // namespace v5

int launch_commit_split(const V2Launch& q, cudaStream_t s) {
  const int n = q.n;
  const int T = n * (n + 1) / 2, N2 = n * n, SE = 2 * T + n;
  const int64_t K = q.K, K1 = std::max<int64_t>(K - 1, 1);
  const int64_t KW = q.kshared ? 2 : q.Bp;
  const int Kb = q.kshared ? 2 : 32;
  const int64_t BLp = q.Bp + 64;  // one scratch column per plan
  v5::Args a;
  std::memset(&a, 0, sizeof(a));
  a.B = q.nplans;
  a.K = K;
  a.Bp = q.Bp;
  a.BLp = BLp;
  int r;
  if ((r = v3::make_map(&a.m_ld, q.ld, q.Bp, T, K, 32, T)) || (r = v3::make_map(&a.m_lo, q.lo, q.Bp, N2, K1, 32, N2)) ||
      (r = v3::make_map(&a.m_kd, q.kd, KW, T, K, Kb, T)) || (r = v3::make_map(&a.m_ko, q.ko, KW, N2, K1, Kb, N2)) ||
      (r = v3::make_map(&a.m_gd, q.gd, q.Bp, T, K, 32, T)) ||
      (r = v3::make_map(&a.m_e, q.scratch + probe_residual_offset(q.nplans, K, n), q.Bp, n, K, 32, n)) ||
      (r = v3::make_map(&a.m_mu, q.mu, q.Bp, n, K, 32, n)) || (r = v3::make_map(&a.m_pm, q.pmean, q.Bp, n, K, 32, n)) ||
      (r = v3::make_map(&a.m_phi, q.scratch, BLp, SE, K, 32, T)) ||
      (r = v3::make_map(&a.m_psiy, q.scratch, BLp, SE, K, 32, T + n)))
    return r;
  a.o_mu = q.o_mu; a.o_ld = q.o_ld; a.o_lo = q.o_lo; a.o_cov = q.o_cov; a.o_cr = q.o_cr; a.o_v = q.o_v;
  a.beta = q.beta; a.kl = q.kl; a.ld_next = q.ld_next; a.shift = q.shift; a.prior_cost = q.prior_cost;
  a.temp = q.temp; a.ld_cur = q.ld_cur;
  a.status = q.status; a.where = q.where;
  a.scratch = q.scratch;
  a.active = q.active;
  a.search_kl = q.search_kl ? 1 : 0;
  a.fixkl = q.fixkl;
  const unsigned grid = (unsigned)((q.nplans + 31) / 32);
#define GVP_V5_KS(NN, KK)                                                                              \
  {                                                                                                    \
    using LOH = v5::Lay<NN, KK>;                                                                       \
    GVP_CUDA(cudaFuncSetAttribute(v5::commit_kernel<NN, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  (int)LOH::BYTES));                                                   \
    v5::commit_kernel<NN, KK><<<grid, 128, LOH::BYTES, s>>>(a);                                        \
  }
#define GVP_V5(NN) \
  if (q.kshared) GVP_V5_KS(NN, true) else GVP_V5_KS(NN, false)
  switch (n) {
    case 2: GVP_V5(2) break;
    case 4: GVP_V5(4) break;
    case 6: GVP_V5(6) break;
    default:
      set_error("step kernel supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_V5
#undef GVP_V5_KS
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp

#ifdef GVP_COMMIT_PROFILE
// (diagnostic build) out = {pass B cycles, pass F cycles, CTAs, then [pass][warp][work, wait]
// (16)} since the last call
extern "C" int gvp_commit_profile(double* out) {
  unsigned long long h[3], r[16];
  GVP_CUDA(cudaMemcpyFromSymbol(h, gvp::v5::g_commit_prof, sizeof(h)));
  GVP_CUDA(cudaMemcpyFromSymbol(r, gvp::v5::g_commit_role, sizeof(r)));
  const unsigned long long z[16] = {};
  GVP_CUDA(cudaMemcpyToSymbol(gvp::v5::g_commit_prof, z, sizeof(h)));
  GVP_CUDA(cudaMemcpyToSymbol(gvp::v5::g_commit_role, z, sizeof(r)));
  for (int i = 0; i < 3; ++i) out[i] = (double)h[i];
  for (int i = 0; i < 16; ++i) out[3 + i] = (double)r[i];
  return GVP_OK;
}
#endif
