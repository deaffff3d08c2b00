// Kernel (b)+(c), bisection half: every probe of select_step_size
// (optimizer.py:188-231) as ONE forward sweep over the knots.
//
// The reference evaluates a candidate beta by forming the proximal update
// (optimizer.py:129-161: mean solve with S = K/T + Lambda/beta, new precision
// Lambda' = c (S + 2 G/T)), running GBP for the new marginals (gbp.py:43-80)
// and then kl_joint (optimizer.py:164-177):
//   KL = 1/2 [ tr(Lambda Sigma') + d' Lambda d - Kn + logdet Lambda' - logdet Lambda ],
//   d = mu - mu' = S^{-1} e,  e = S mu - rhs = (K mu + g - eta) / T   (beta-free).
// Both data-dependent terms are directional derivatives of quantities a
// single forward Schur sweep produces:
//   tr(Lambda Lambda'^{-1}) =  d/dt logdet(Lambda' + t Lambda)       |t=0
//   d' Lambda d            = -d/dt e' (S + t Lambda)^{-1} e          |t=0
// so each lane carries, next to the block-Cholesky pivots Phi_i of its
// matrix, their tangents Phi'_i (forward-mode differentiation of the
// recursion Phi_i = M_i - M_{i-1,i}' Phi_{i-1}^{-1} M_{i-1,i}):
//   W = Li_{i-1} M_{i-1,i},  G = Li_{i-1} Lambda_{i-1,i},  Psi = Li Phi' Li'
//   Phi'_i = Lambda_ii + W'(Psi_{i-1} W - G) - G'W,   tr += trace(Psi_i)
// and (mean chain) the eliminated rhs v_i = Li_i w_i with its tangent
// u_i = Li_i w'_i:  w_i = e_i - W'v_{i-1},  w'_i = W'(Psi_{i-1} v_{i-1} - u_{i-1}) - G'v_{i-1},
//   d' Lambda d = sum_i v_i' Psi_i v_i - 2 u_i . v_i.
// No backward sweep, no per-lane scratch in HBM: a probe reads each plan's
// per-knot data once (LD, GD, E, LO: 40 doubles at n = 4) from shared memory
// staged by TMA, shared by all lanes of the plan. The KL agrees with the
// reference's to ~1e-11 relative (tests/test_gpu_parity.py); the accepted
// beta's update itself (mean, marginals, KL record) is produced by the exact
// two-pass commit kernel (commit.cu).
//
// Failure semantics follow the reference: the mean chain is the forward
// elimination of gbp_mean_solve (gbp.py:83-106), so a non-SPD pivot there is
// an error at the same knot; a non-SPD pivot of Lambda' makes the probe
// infeasible (gbp_marginals raising, optimizer.py:203-207).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <cstdlib>

#include "gvp_internal.cuh"
#include "step_common.cuh"

namespace gvp {
namespace v4 {

#ifdef GVP_PROBE_PROFILE
// diagnostic build only (-DGVP_PROBE_PROFILE): per-role cycles spent working vs
// waiting (TMA + CTA barrier) in probe_split_kernel, summed over lane-0 threads
__device__ unsigned long long g_probe_prof[8];
#endif

using v3::PlanSt;
using v3::Pick;
using v3::T_;
// resident split-probe CTAs per SM the register budget targets. 3 at n = 4
// (168 registers, spilling) made every step ~12% slower and lost overall
// (C5: 13.7 ms vs 11.6 ms per bisection), so 2.
template <int N>
constexpr int probe_minb() {
#ifdef GVP_PROBE_MINB
  return GVP_PROBE_MINB;
#else
  return 2;
#endif
}

// Compile-time shared-memory layout (32 lane slots = P plans x L lanes, four
// warps over the same 32 slots, see the kernel).
constexpr int kMaxStagesTail = 8;  // mbarriers
template <int N, int L, bool KS, bool SPLIT>
struct Lay {
  static constexpr int T = T_<N>, N2 = N * N;
  static constexpr int P = 32 / L, Pb = P, Kb = KS ? 2 : P;
  static constexpr int gP = v3::cx_gran(Pb), gK = v3::cx_gran(Kb);
  // plan rows: LD T | GD T | E N | LO N2 (block (i-1, i))
  static constexpr int R_LD = 0, R_GD = v3::cx_round(T, gP), R_E = v3::cx_round(R_GD + T, gP),
                       R_LO = v3::cx_round(R_E + N, gP), PR = v3::cx_round(R_LO + N2, gP);
  // prior rows: KD T | KO N2 (block (i-1, i))
  static constexpr int R_KD = 0, R_KO = v3::cx_round(T, gK), KR = v3::cx_round(R_KO + N2, gK);
  static constexpr int OFF_PRIOR = v3::cx_round(PR * Pb, 16),
                       STAGE = OFF_PRIOR + v3::cx_round(KR * Kb, 16);
  // producer -> consumer ring (2 steps x 2 chains): Li T | W N2 | v N, per slot
  static constexpr int ENT = T + N2 + N, E_LI = 0, E_W = T, E_V = T + N2;
  // split: as many stages (4..8) as fit probe_minb CTAs per SM (228 KB, 1 KB
  // reserved per CTA) next to the producer ring and the fixed tail
  static constexpr int FIXED = (SPLIT ? 2 * 2 * ENT * 32 : 0) + (5 + 10 + 5) * 32 + kMaxStagesTail;
  static constexpr int FIT = ((233472 / probe_minb<N>() - 1024) / 8 - FIXED) / STAGE;
  // prefetch distance: at step s the consumers still read knot s-1's slot
  static constexpr int NS = SPLIT ? (FIT < 4 ? 4 : FIT > 8 ? 8 : FIT) : v3::ring_stages(STAGE),
                       AH = SPLIT ? NS - 2 : NS - 1;
  static constexpr int RING = NS * STAGE;
  static constexpr int XCH = RING + (SPLIT ? 2 * 2 * ENT * 32 : 0);  // 4 roles x 32 doubles + 2 x 32 ints
  static constexpr int PST = XCH + 5 * 32;
  static constexpr int RES = PST + 10 * 32;
  static constexpr int BAR = RES + 5 * 32;
  static constexpr size_t BYTES = (size_t)(BAR + NS) * 8;
  static constexpr uint32_t TX = ((2 * T + N + N2) * Pb + (T + N2) * Kb) * 8;
};

struct Args {
  CUtensorMap m_ld, m_gd, m_e, m_lo, m_kd, m_ko;
  int B;
  int64_t K, Bp;
  const double *temp, *ld_cur;
  double kl_bound, beta_min, beta_max;
  double* beta;
  double *kl, *ld_next;  // the accepted probe's KL and forward-Schur log det (search end)
  int *status, *where, *nprobes;
  double* probe_log;
  int max_probes;
  const int* active;
  int ppc;  // plans per CTA (<= the layout's P = 32 / L)
  int rotate;  // split kernel: rotate the warp roles by the CTA's SM residency slot
};


template <int N>
GVP_DEV double symv(const double (&A)[T_<N>], int r, int c) {
  return r >= c ? A[tri_idx(r, c)] : A[tri_idx(c, r)];
}

// Four warps per 32 lane slots, one chain stage each:
//   warp 0  Lambda' Schur:   W = Li_{i-1} Lambda'_{i-1,i}, Phi_i, chol -> Li_i, log det
//   warp 1  Lambda' tangent: Phi'_i, Psi_i, trace                 (one knot behind warp 0)
//   warp 2  S Schur:         W, Phi_i, chol -> Li_i, v_i = Li_i (e_i - W'v_{i-1})
//   warp 3  S tangent:       Phi'_i, Psi_i, u_i, Mahalanobis      (one knot behind warp 2)
// The Schur warps hand Li_i, W_i (and v_i) to their tangent warp through a
// two-step shared-memory ring; one CTA barrier per step orders everything.
// Splitting the chains (instead of more speculative lanes) doubles the warps
// that hide the fp64 dependency latency without adding probes.
template <int N, int L, bool KS>
__global__ void __launch_bounds__(128, probe_minb<N>()) probe_split_kernel(const __grid_constant__ Args a) {
  using LO = Lay<N, L, KS, true>;
  constexpr int T = LO::T, N2 = LO::N2;
  extern __shared__ __align__(1024) double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LO::BAR);
  const int tid = threadIdx.x;
  // The four roles carry unequal fp64 work (tangent of the S chain the most)
  // and warp w of every resident CTA lands on sub-partition w % 4, so with
  // identical role maps one scheduler's fp64 pipe sets the step time while the
  // others idle at the barrier. Rotating the role map by the CTA's residency
  // slot (its first warp's hardware slot / 4) mixes the roles on each
  // sub-partition. Any rotation is correct; it only changes the balance.
  // (kept in the result area's spare ints: no static shared memory, whose
  // extra bytes would cost the second resident CTA)
  int* s_rot = reinterpret_cast<int*>(smem + LO::RES + 64) + 96;
  if (tid == 0) {
    unsigned wid = 0;
    if (a.rotate) asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    *s_rot = (int)(((wid >> 2) & 1u) * 2u + ((wid >> 3) & 1u));
  }
  __syncthreads();
  const int role = ((tid >> 5) + *s_rot) & 3;  // warp-uniform
  const int chain = role >> 1;          // 0: Lambda', 1: S
  const bool tangent = (role & 1) != 0;
  const int lcol = tid & 31;            // lane slot
  constexpr int P = LO::P, Pb = LO::Pb, Kb = LO::Kb, LP = P * L;
  const int64_t b0 = (int64_t)blockIdx.x * a.ppc;
  const int K = (int)a.K;  // 32-bit step arithmetic: every loop-control op is a single integer op
  double* ring = smem + LO::RING;
  double* xch = smem + LO::XCH;
  int* ffail = reinterpret_cast<int*>(xch + 4 * 32);  // [chain][slot] first failing knot
  PlanSt* pst = reinterpret_cast<PlanSt*>(smem + LO::PST);
  double* r_beta = smem + LO::RES;
  double* r_kl = r_beta + 32;
  int* r_res = reinterpret_cast<int*>(r_kl + 32);
  int* r_fail = r_res + 32;
  int* r_on = r_fail + 32;

  if (tid == 0) {
    for (int s = 0; s < LO::NS; ++s) v3::mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  v3::search_init(a, pst, a.ppc, b0, false, tid);
  __syncthreads();

  auto slot = [&](int s) { return smem + ((unsigned)s % LO::NS) * LO::STAGE; };
  auto issue = [&](int s, int i) {
    double* st = slot(s);
    uint64_t* bar = &bars[(unsigned)s % LO::NS];
    v3::mbar_expect_tx(bar, LO::TX);
    const int ck = KS ? 0 : (int)b0;
    const int io = i > 0 ? i - 1 : 0;  // off-diagonal block (i-1, i)
    double* pr = st + LO::OFF_PRIOR;
    v3::tma3(pr + LO::R_KD * Kb, &a.m_kd, ck, 0, i, bar);
    v3::tma3(pr + LO::R_KO * Kb, &a.m_ko, ck, 0, io, bar);
    v3::tma3(st + LO::R_LD * Pb, &a.m_ld, (int)b0, 0, i, bar);
    v3::tma3(st + LO::R_GD * Pb, &a.m_gd, (int)b0, 0, i, bar);
    v3::tma3(st + LO::R_E * Pb, &a.m_e, (int)b0, 0, i, bar);
    v3::tma3(st + LO::R_LO * Pb, &a.m_lo, (int)b0, 0, io, bar);
  };
  auto wait_slot = [&](int s) {
    v3::mbar_wait(&bars[(unsigned)s % LO::NS], ((unsigned)s / LO::NS) & 1u);
  };
  auto rg = [&](int s, int ch, int e) -> double* {
    return ring + (((s & 1) * 2 + ch) * LO::ENT + e) * 32 + lcol;
  };

  int sbase = 0;
  for (;;) {
    const Pick pk = v3::search_pick(a, pst, a.ppc, LP, lcol, tid, false);
    if (pk.kl == 0) break;  // uniform: every thread read the same shared state
    const int p = pk.p, my_rank = pk.my_rank;
    const int kcol = KS ? 0 : p;
    const double temp = pst[p].temp, ldc = pst[p].ldc;
    const bool lane_on = pk.on;
    const double beta = pk.beta;
    if (!tangent) ffail[chain * 32 + lcol] = -1;
    __syncthreads();  // plan state read, fail flags reset

    const double inv_t = 1.0 / temp, two_t = 2.0 / temp;
    const double inv_b = lane_on ? 1.0 / beta : 0.0, c = lane_on ? beta / (beta + 1.0) : 0.0;
    const double so = chain == 0 ? c : 1.0;  // Lambda' off blocks carry the factor c
    bool alive = lane_on;
    double acc = 0.0;       // Schur A: log det mantissa part; tangents: trace / Mahalanobis
    int acc_e = 0;          // Schur A: binary exponent of the pivot product
    double pm = 1.0;        // Schur A: pivot product mantissa
    double Li[T], Ps[T], v[N], u[N];

    if (tid == 0)
      for (int s = 0; s < LO::AH && s < K; ++s) issue(sbase + s, s);
#ifdef GVP_PROBE_PROFILE
    long long prof_work = 0, prof_wait = 0, tprev = 0;
#endif
    for (int st_ = 0; st_ <= K; ++st_) {
      const int s = sbase + st_;
#ifdef GVP_PROBE_PROFILE
      const long long tp0 = clock64();
#endif
      if (st_ < K) wait_slot(s);
      __syncthreads();  // step st_-1 complete: ring / stage slots may be reused
#ifdef GVP_PROBE_PROFILE
      const long long tp1 = clock64();
      if (st_ > 0) prof_work += tp0 - tprev;
      prof_wait += tp1 - tp0;
      tprev = tp1;
#endif
      if (tid == 0 && st_ + LO::AH < K) issue(s + LO::AH, st_ + LO::AH);
      if (!tangent) {
        // ---------------------------- Schur producer, knot i = st_
        // W is formed one row at a time; each row is a rank-1 update of the
        // pivot (and of the eliminated rhs) and goes straight to the ring.
        const int i = st_;
        if (i >= K) continue;  // (a failed or idle lane keeps computing on garbage the
                               // combine discards: no lane-divergent branch in the step)
        const double* sg = slot(s);
        const double* pr = sg + LO::OFF_PRIOR;
        auto pv = [&](int row) { return sg[row * Pb + p]; };
        auto kv = [&](int row) { return pr[row * Kb + kcol]; };
        double M[T], w[N];
        if (chain == 0) {
          // the reference's assembly order (optimizer.py:151-153): the probes' KL is
          // judged against the exact KL of exactly these matrices (cond ~1e10 turns
          // a re-associated ulp into 1e-4 of KL)
#pragma unroll
          for (int q = 0; q < T; ++q)
            M[q] = ((pv(LO::R_GD + q) * two_t + kv(LO::R_KD + q) * inv_t) + pv(LO::R_LD + q) * inv_b) * c;
        } else {
#pragma unroll
          for (int q = 0; q < T; ++q) M[q] = kv(LO::R_KD + q) * inv_t + pv(LO::R_LD + q) * inv_b;
#pragma unroll
          for (int r = 0; r < N; ++r) w[r] = pv(LO::R_E + r) * inv_t;
        }
        if (i > 0) {
          double Mo[N2];
#pragma unroll
          for (int q = 0; q < N2; ++q) Mo[q] = (kv(LO::R_KO + q) * inv_t + pv(LO::R_LO + q) * inv_b) * so;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double wk[N];
#pragma unroll
            for (int q = 0; q < N; ++q) {
              double t = 0.0;
#pragma unroll
              for (int j = 0; j <= k; ++j) t += Li[tri_idx(k, j)] * Mo[j * N + q];
              wk[q] = t;
              *rg(s, chain, LO::E_W + k * N + q) = t;
            }
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q <= r; ++q) M[tri_idx(r, q)] -= wk[r] * wk[q];
            if (chain == 1) {
#pragma unroll
              for (int r = 0; r < N; ++r) w[r] -= wk[r] * v[k];
            }
          }
        }
        double pp;
        if (!v3::chol_inv<N>(M, Li, pp) && alive) {
          ffail[chain * 32 + lcol] = (int)i;
          alive = false;
        }
        if (chain == 0) {  // log det = 2 log prod(pivots), product kept normalised
          int ex;
          pm = frexp_pos(pm * pp, &ex);
          acc_e += ex;
        } else {
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k <= r; ++k) t += Li[tri_idx(r, k)] * w[k];
            v[r] = t;
            *rg(s, 1, LO::E_V + r) = t;
          }
        }
#pragma unroll
        for (int q = 0; q < T; ++q) *rg(s, chain, LO::E_LI + q) = Li[q];
      } else {
        // ---------------------------- tangent consumer, knot i = st_ - 1
        // Phi'_i = Lambda_ii - (G'W + W'G) + W'(Psi_{i-1} W), accumulated over
        // the rows of W (ring) and G = Li_{i-1} Lambda_{i-1,i} (formed here).
        const int i = st_ - 1;
        if (i < 0) continue;
        const double* sg = slot(s - 1);
        auto pv = [&](int row) { return sg[row * Pb + p]; };
        double Pd[T], wp[N];
#pragma unroll
        for (int q = 0; q < T; ++q) Pd[q] = pv(LO::R_LD + q);
#pragma unroll
        for (int r = 0; r < N; ++r) wp[r] = 0.0;
        if (i > 0) {
          double tv[N], Y[N2];  // tv = Psi_{i-1} v_{i-1} - u_{i-1};  Y = Psi_{i-1} W
          if (chain == 1) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
              double t = -u[k];
#pragma unroll
              for (int j = 0; j < N; ++j) t += symv<N>(Ps, k, j) * v[j];
              tv[k] = t;
            }
          }
#pragma unroll
          for (int q = 0; q < N2; ++q) Y[q] = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double wk[N], gk[N];
#pragma unroll
            for (int q = 0; q < N; ++q) {
              wk[q] = *rg(s - 1, chain, LO::E_W + k * N + q);
              double t = 0.0;
#pragma unroll
              for (int j = 0; j <= k; ++j) t += Li[tri_idx(k, j)] * pv(LO::R_LO + j * N + q);
              gk[q] = t;
            }
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q <= r; ++q) {
                Pd[tri_idx(r, q)] -= gk[r] * wk[q];  // two fused steps (no separate multiply / add)
                Pd[tri_idx(r, q)] -= wk[r] * gk[q];
              }
#pragma unroll
            for (int j = 0; j < N; ++j) {
              const double pj = symv<N>(Ps, j, k);
#pragma unroll
              for (int q = 0; q < N; ++q) Y[j * N + q] += pj * wk[q];
            }
            if (chain == 1) {
#pragma unroll
              for (int r = 0; r < N; ++r) wp[r] += wk[r] * tv[k] - gk[r] * v[k];
            }
          }
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double wk[N];
#pragma unroll
            for (int q = 0; q < N; ++q) wk[q] = *rg(s - 1, chain, LO::E_W + k * N + q);
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int q = 0; q <= r; ++q) Pd[tri_idx(r, q)] += wk[r] * Y[k * N + q];
          }
        }
        // Psi_i = Li_i Phi'_i Li_i', one row at a time
#pragma unroll
        for (int q = 0; q < T; ++q) Li[q] = *rg(s - 1, chain, LO::E_LI + q);
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double xr[N];
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k <= r; ++k) t += Li[tri_idx(r, k)] * symv<N>(Pd, k, q);
            xr[q] = t;
          }
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k <= q; ++k) t += xr[k] * Li[tri_idx(q, k)];
            Ps[tri_idx(r, q)] = t;
          }
        }
        if (chain == 0) {
#pragma unroll
          for (int r = 0; r < N; ++r) acc += Ps[tri_idx(r, r)];
        } else {
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k <= r; ++k) t += Li[tri_idx(r, k)] * wp[k];
            u[r] = t;
            v[r] = *rg(s - 1, 1, LO::E_V + r);
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) t += symv<N>(Ps, r, k) * v[k];
            acc += v[r] * t - 2.0 * u[r] * v[r];
          }
        }
      }
    }
    sbase += K;
#ifdef GVP_PROBE_PROFILE
    if (lcol == 0) {
      atomicAdd(&g_probe_prof[role * 2], (unsigned long long)prof_work);
      atomicAdd(&g_probe_prof[role * 2 + 1], (unsigned long long)prof_wait);
    }
#endif

    // ---------------- combine the chains: the mean chain fails first
    // (proximal_update raises before gbp_marginals, optimizer.py:203-207)
    if (role == 0) acc = 2.0 * (log(pm) + (double)acc_e * 0.6931471805599453);
    xch[role * 32 + lcol] = acc;
    __syncthreads();
    if (role == 0) {
      const int fA = ffail[lcol], fB = ffail[32 + lcol];
      const int rr = fB >= 0 ? 2 : (fA >= 0 ? 1 : 0);
      double klv = 0.0;
      if (lane_on && rr == 0) {
        const double ld = xch[lcol], tr = xch[32 + lcol], mh = xch[96 + lcol];
        const double x = 0.5 * ((((tr + mh) - (double)(K * N)) + ld) - ldc);
        klv = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
      }
      r_beta[lcol] = beta;
      r_kl[lcol] = klv;
      r_res[lcol] = rr;
      r_fail[lcol] = fB >= 0 ? fB : fA;
      r_on[lcol] = lane_on ? 1 : 0;
    }
    __syncthreads();
    if (my_rank >= 0)
      v3::search_decide(a, pst, tid, pk.dbase, pk.dkl, b0, false, r_beta, r_kl, r_res, r_fail, r_on, xch);
    __syncthreads();
  }
}

// Two warps per 32 lane slots: warp 0 runs the whole Lambda' chain (Schur +
// tangent), warp 1 the whole S chain. Fewer barriers and no ring traffic;
// preferred when the grid already fills the GPU (large batches).
template <int N, int L, bool KS>
__global__ void __launch_bounds__(64) probe_fused_kernel(const __grid_constant__ Args a) {
  using LO = Lay<N, L, KS, false>;
  constexpr int T = LO::T, N2 = LO::N2;
  constexpr int AH = LO::AH;  // only the current knot's slot is read
  extern __shared__ __align__(1024) double smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LO::BAR);
  const int tid = threadIdx.x;
  const int role = tid >> 5;  // 0: Lambda' chain (log det, trace), 1: S chain (Mahalanobis)
  const int lcol = tid & 31;
  constexpr int P = LO::P, Pb = LO::Pb, Kb = LO::Kb, LP = P * L;
  const int64_t b0 = (int64_t)blockIdx.x * a.ppc;
  const int64_t K = a.K;
  double* xch = smem + LO::XCH;
  PlanSt* pst = reinterpret_cast<PlanSt*>(smem + LO::PST);
  double* r_beta = smem + LO::RES;
  double* r_kl = r_beta + 32;
  int* r_res = reinterpret_cast<int*>(r_kl + 32);
  int* r_fail = r_res + 32;
  int* r_on = r_fail + 32;

  if (tid == 0) {
    for (int s = 0; s < LO::NS; ++s) v3::mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  v3::search_init(a, pst, a.ppc, b0, false, tid);
  __syncthreads();

  auto slot = [&](int64_t s) { return smem + (s % LO::NS) * LO::STAGE; };
  auto issue = [&](int64_t s, int64_t i) {
    double* st = slot(s);
    uint64_t* bar = &bars[s % LO::NS];
    v3::mbar_expect_tx(bar, LO::TX);
    const int ck = KS ? 0 : (int)b0;
    const int io = (int)(i > 0 ? i - 1 : 0);
    double* pr = st + LO::OFF_PRIOR;
    v3::tma3(pr + LO::R_KD * Kb, &a.m_kd, ck, 0, (int)i, bar);
    v3::tma3(pr + LO::R_KO * Kb, &a.m_ko, ck, 0, io, bar);
    v3::tma3(st + LO::R_LD * Pb, &a.m_ld, (int)b0, 0, (int)i, bar);
    v3::tma3(st + LO::R_GD * Pb, &a.m_gd, (int)b0, 0, (int)i, bar);
    v3::tma3(st + LO::R_E * Pb, &a.m_e, (int)b0, 0, (int)i, bar);
    v3::tma3(st + LO::R_LO * Pb, &a.m_lo, (int)b0, 0, io, bar);
  };

  int64_t sbase = 0;
  for (;;) {
    const Pick pk = v3::search_pick(a, pst, a.ppc, LP, lcol, tid, false);
    if (pk.kl == 0) break;
    const int p = pk.p, my_rank = pk.my_rank;
    const int kcol = KS ? 0 : p;
    const double temp = pst[p].temp, ldc = pst[p].ldc;
    const bool lane_on = pk.on;
    const double beta = pk.beta;
    __syncthreads();

    const double inv_t = 1.0 / temp, two_t = 2.0 / temp;
    const double inv_b = lane_on ? 1.0 / beta : 0.0, c = lane_on ? beta / (beta + 1.0) : 0.0;
    const double so = role == 0 ? c : 1.0;
    int fail_knot = -1;
    double acc = 0.0, pm = 1.0;
    int acc_e = 0;
    double Li[T], Ps[T], v[N], u[N];

    if (tid == 0)
      for (int s = 0; s < AH && s < K; ++s) issue(sbase + s, s);
    for (int64_t i = 0; i < K; ++i) {
      const int64_t s = sbase + i;
      v3::mbar_wait(&bars[s % LO::NS], (uint32_t)((s / LO::NS) & 1));
      __syncthreads();
      if (tid == 0 && i + AH < K) issue(s + AH, i + AH);
      if (!(lane_on && fail_knot < 0)) continue;
      const double* sg = slot(s);
      const double* pr = sg + LO::OFF_PRIOR;
      auto pv = [&](int row) { return sg[row * Pb + p]; };
      auto kv = [&](int row) { return pr[row * Kb + kcol]; };
      double M[T], Pd[T], w[N], wp[N];
      if (role == 0) {
#pragma unroll
        for (int q = 0; q < T; ++q)
          M[q] = ((pv(LO::R_GD + q) * two_t + kv(LO::R_KD + q) * inv_t) + pv(LO::R_LD + q) * inv_b) * c;
      } else {
#pragma unroll
        for (int q = 0; q < T; ++q) M[q] = kv(LO::R_KD + q) * inv_t + pv(LO::R_LD + q) * inv_b;
#pragma unroll
        for (int r = 0; r < N; ++r) {
          w[r] = pv(LO::R_E + r) * inv_t;
          wp[r] = 0.0;
        }
      }
#pragma unroll
      for (int q = 0; q < T; ++q) Pd[q] = pv(LO::R_LD + q);
      if (i > 0) {
        double W[N2], G[N2];
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double tw = 0.0, tg = 0.0;
#pragma unroll
            for (int k = 0; k <= r; ++k) {
              const double lo_ = pv(LO::R_LO + k * N + q);
              tw += Li[tri_idx(r, k)] * ((kv(LO::R_KO + k * N + q) * inv_t + lo_ * inv_b) * so);
              tg += Li[tri_idx(r, k)] * lo_;
            }
            W[r * N + q] = tw;
            G[r * N + q] = tg;
          }
        if (role == 1) {
          double tv[N];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double t = -u[k];
#pragma unroll
            for (int j = 0; j < N; ++j) t += symv<N>(Ps, k, j) * v[j];
            tv[k] = t;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double t1 = 0.0, t2 = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
              t1 += W[k * N + r] * v[k];
              t2 += W[k * N + r] * tv[k] - G[k * N + r] * v[k];
            }
            w[r] -= t1;
            wp[r] = t2;
          }
        }
        double Z[N2];
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q < N; ++q) {
            double t = -G[r * N + q];
#pragma unroll
            for (int k = 0; k < N; ++k) t += symv<N>(Ps, r, k) * W[k * N + q];
            Z[r * N + q] = t;
          }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) {
            double tm = 0.0, td = 0.0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
              tm += W[k * N + r] * W[k * N + q];
              td += W[k * N + r] * Z[k * N + q] - G[k * N + r] * W[k * N + q];
            }
            M[tri_idx(r, q)] -= tm;
            Pd[tri_idx(r, q)] += td;
          }
      }
      double pp;
      if (!v3::chol_inv<N>(M, Li, pp)) {
        fail_knot = (int)i;
        continue;
      }
      if (role == 0) {
        int ex;
        pm = frexp_pos(pm * pp, &ex);
        acc_e += ex;
      }
      double X[N2];
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k <= r; ++k) t += Li[tri_idx(r, k)] * symv<N>(Pd, k, q);
          X[r * N + q] = t;
        }
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int q = 0; q <= r; ++q) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k <= q; ++k) t += X[r * N + k] * Li[tri_idx(q, k)];
          Ps[tri_idx(r, q)] = t;
        }
      if (role == 0) {
#pragma unroll
        for (int r = 0; r < N; ++r) acc += Ps[tri_idx(r, r)];
      } else {
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double tv = 0.0, tu = 0.0;
#pragma unroll
          for (int k = 0; k <= r; ++k) {
            tv += Li[tri_idx(r, k)] * w[k];
            tu += Li[tri_idx(r, k)] * wp[k];
          }
          v[r] = tv;
          u[r] = tu;
        }
#pragma unroll
        for (int r = 0; r < N; ++r) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) t += symv<N>(Ps, r, k) * v[k];
          acc += v[r] * t - 2.0 * u[r] * v[r];
        }
      }
    }
    sbase += K;

    // combine: the mean chain fails first (optimizer.py:203-207)
    int* xi = reinterpret_cast<int*>(xch + 4 * 32);
    xi[role * 32 + lcol] = fail_knot;
    xch[role * 32 + lcol] = acc;
    xch[(2 + role) * 32 + lcol] = role == 0 ? 2.0 * (log(pm) + (double)acc_e * 0.6931471805599453) : 0.0;
    __syncthreads();
    if (role == 0) {
      const int fA = fail_knot, fB = xi[32 + lcol];
      const int rr = fB >= 0 ? 2 : (fA >= 0 ? 1 : 0);
      double klv = 0.0;
      if (lane_on && rr == 0) {
        const double tr = acc, mh = xch[32 + lcol], ld = xch[64 + lcol];
        const double x = 0.5 * ((((tr + mh) - (double)(K * N)) + ld) - ldc);
        klv = (0.0 > x) ? 0.0 : x;
      }
      r_beta[lcol] = beta;
      r_kl[lcol] = klv;
      r_res[lcol] = rr;
      r_fail[lcol] = fB >= 0 ? fB : fA;
      r_on[lcol] = lane_on ? 1 : 0;
    }
    __syncthreads();
    if (my_rank >= 0)
      v3::search_decide(a, pst, tid, pk.dbase, pk.dkl, b0, false, r_beta, r_kl, r_res, r_fail, r_on,
                        xch + 64);
    __syncthreads();
  }
}

// e = K mu + g - eta per knot (plan-minor, the probe's beta-free residual).
// One thread per (plan, run of kRun knots): the mean window slides through
// registers, so every mean block is read about once and all loads are
// coalesced across plans.
constexpr int kRun = 8;
template <int N>
__global__ void __launch_bounds__(128, 4) residual_kernel(int B, int64_t K, int64_t Bp, const double* kd, const double* ko, int64_t KW,
                                bool kshared, const double* mu, const double* g, const double* eta, double* e) {
  constexpr int T = N * (N + 1) / 2, N2 = N * N;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t runs = (K + kRun - 1) / kRun;
  if (t >= runs * Bp) return;
  const int64_t b = t % Bp, i0 = (t / Bp) * kRun;
  if (b >= B) return;
  const int64_t kc = kshared ? 0 : b;
  auto ld_mu = [&](int64_t i, double (&m)[N]) {
#pragma unroll
    for (int r = 0; r < N; ++r) m[r] = (i >= 0 && i < K) ? mu[(i * N + r) * Bp + b] : 0.0;
  };
  double mp[N], mc[N], mn[N];
  ld_mu(i0 - 1, mp);
  ld_mu(i0, mc);
  const int64_t i1 = i0 + kRun < K ? i0 + kRun : K;
#pragma unroll 1
  for (int64_t i = i0; i < i1; ++i) {
    ld_mu(i + 1, mn);
#pragma unroll 1
    for (int r = 0; r < N; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const int tq = r >= q ? r * (r + 1) / 2 + q : q * (q + 1) / 2 + r;
        acc += kd[(i * T + tq) * KW + kc] * mc[q];
        if (i > 0) acc += ko[((i - 1) * N2 + q * N + r) * KW + kc] * mp[q];
        if (i + 1 < K) acc += ko[(i * N2 + r * N + q) * KW + kc] * mn[q];
      }
      e[(i * N + r) * Bp + b] = (acc + g[(i * N + r) * Bp + b]) - eta[(i * N + r) * Bp + b];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      mp[r] = mc[r];
      mc[r] = mn[r];
    }
  }
}

// Forward-Schur log det of packed precisions, the probes' chain-0 recursion
// op for op (W rows as rank-1 updates, chol_inv, normalised pivot product),
// so ld_cur and the probes' log dets of nearby Lambda' carry correlated
// rounding (the KL is their difference). Thread per plan; NaN on a non-SPD pivot.
template <int N>
__global__ void logdet_fwd_packed_kernel(int B, int64_t K, int64_t Bp, const double* __restrict__ ld,
                                         const double* __restrict__ lo, double* __restrict__ out,
                                         const int* __restrict__ mask, int* status, int* where) {
  constexpr int T = T_<N>, N2 = N * N;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || (mask && !mask[b])) return;
  double Li[T], pm = 1.0;
  int acc_e = 0;
  for (int64_t i = 0; i < K; ++i) {
    double M[T];
#pragma unroll
    for (int q = 0; q < T; ++q) M[q] = ld[(i * T + q) * Bp + b];
    if (i > 0) {
      double Mo[N2];
#pragma unroll
      for (int q = 0; q < N2; ++q) Mo[q] = lo[((i - 1) * N2 + q) * Bp + b];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double wk[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j <= k; ++j) t += Li[tri_idx(k, j)] * Mo[j * N + q];
          wk[q] = t;
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int q = 0; q <= r; ++q) M[tri_idx(r, q)] -= wk[r] * wk[q];
      }
    }
    double pp;
    if (!v3::chol_inv<N>(M, Li, pp)) {
      out[b] = NAN;
      if (status) {
        status[b] = GVP_ERR_NOT_SPD;
        where[b] = (int)i;
      }
      return;
    }
    int ex;
    pm = frexp_pos(pm * pp, &ex);
    acc_e += ex;
  }
  out[b] = 2.0 * (log(pm) + (double)acc_e * 0.6931471805599453);
}

}  // namespace v4

int launch_logdet_fwd_packed(int nplans, int64_t K, int n, int64_t Bp, const double* ld, const double* lo,
                             double* logdet, const int* mask, int* status, int* where, cudaStream_t s) {
  const unsigned nb = (unsigned)((nplans + 63) / 64);
  switch (n) {
    case 2: v4::logdet_fwd_packed_kernel<2><<<nb, 64, 0, s>>>(nplans, K, Bp, ld, lo, logdet, mask, status, where); break;
    case 4: v4::logdet_fwd_packed_kernel<4><<<nb, 64, 0, s>>>(nplans, K, Bp, ld, lo, logdet, mask, status, where); break;
    case 6: v4::logdet_fwd_packed_kernel<6><<<nb, 64, 0, s>>>(nplans, K, Bp, ld, lo, logdet, mask, status, where); break;
    default:
      set_error("packed log det supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int64_t probe_residual_offset(int nplans, int64_t K, int n) {
  const int64_t T = (int64_t)n * (n + 1) / 2;
  return K * (2 * T + n) * (step_plan_stride(nplans) + 64);  // after the commit kernel's scratch
}

int launch_probe(const V2Launch& q, const int L, cudaStream_t s) {
  const int n = q.n;
  const int T = n * (n + 1) / 2, N2 = n * n;
  const int P = 32 / L;
  const int Kb = q.kshared ? 2 : P;
  const int64_t K = q.K, K1 = std::max<int64_t>(K - 1, 1);
  const int64_t KW = q.kshared ? 2 : q.Bp;
  double* e = q.scratch + probe_residual_offset(q.nplans, K, n);
  {
    const int64_t total = (K + v4::kRun - 1) / v4::kRun * q.Bp;
    const int tb = 128;
    const unsigned nb = (unsigned)((total + tb - 1) / tb);
    switch (n) {
      case 2: v4::residual_kernel<2><<<nb, tb, 0, s>>>(q.nplans, K, q.Bp, q.kd, q.ko, KW, q.kshared, q.mu, q.g, q.eta, e); break;
      case 4: v4::residual_kernel<4><<<nb, tb, 0, s>>>(q.nplans, K, q.Bp, q.kd, q.ko, KW, q.kshared, q.mu, q.g, q.eta, e); break;
      case 6: v4::residual_kernel<6><<<nb, tb, 0, s>>>(q.nplans, K, q.Bp, q.kd, q.ko, KW, q.kshared, q.mu, q.g, q.eta, e); break;
      default:
        set_error("step kernel supports n in {2, 4, 6}");
        return GVP_ERR_UNSUPPORTED;
    }
  }
  if (q.ev_residual_done) GVP_CUDA(cudaEventRecord(q.ev_residual_done, s));
  v4::Args a;
  std::memset(&a, 0, sizeof(a));
  a.B = q.nplans;
  a.K = K;
  a.Bp = q.Bp;
  int r;
  if ((r = v3::make_map(&a.m_ld, q.ld, q.Bp, T, K, P, T)) || (r = v3::make_map(&a.m_gd, q.gd, q.Bp, T, K, P, T)) ||
      (r = v3::make_map(&a.m_e, e, q.Bp, n, K, P, n)) || (r = v3::make_map(&a.m_lo, q.lo, q.Bp, N2, K1, P, N2)) ||
      (r = v3::make_map(&a.m_kd, q.kd, KW, T, K, Kb, T)) || (r = v3::make_map(&a.m_ko, q.ko, KW, N2, K1, Kb, N2)))
    return r;
  a.temp = q.temp;
  a.ld_cur = q.ld_cur;
  a.kl_bound = q.kl_bound;
  a.beta_min = q.beta_min;
  a.beta_max = q.beta_max;
  a.beta = q.beta;
  a.kl = q.kl;
  a.ld_next = q.ld_next;
  a.status = q.status;
  a.where = q.where;
  a.nprobes = q.nprobes;
  a.probe_log = q.probe_log;
  a.max_probes = q.max_probes;
  a.active = q.active;
  a.ppc = P;
  static const int rot_env = [] {
    const char* e = std::getenv("GVP_PROBE_ROT");
    return e ? std::atoi(e) : 1;
  }();
  a.rotate = rot_env;
  const unsigned grid = (unsigned)((q.nplans + P - 1) / P);
  // split chains (4 warps) while the grid is far from filling the GPU, fused
  // chains (2 warps, fewer barriers) once every SM has several CTAs;
  // GVP_PROBE=split|fused overrides (A/B measurements)
  static const int forced = [] {
    const char* e = std::getenv("GVP_PROBE");
    return !e ? 0 : (std::strcmp(e, "split") == 0 ? 1 : std::strcmp(e, "fused") == 0 ? 2 : 0);
  }();
  const bool split = forced ? forced == 1 : grid < 2u * 148u;
  // q.fill (auto lanes): the split CTA's time is its step latency times its
  // rounds, nearly independent of how many CTAs share the SM, so spread the
  // plans over every resident CTA slot; each plan then gets 32 / ppc lanes
  auto fill_ppc = [&](const void* fn, size_t bytes, int threads) {
    if (!q.fill) return;
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, bytes) != cudaSuccess || occ < 1) occ = 1;
    const int64_t slots = (int64_t)occ * std::max(nsm, 1);
    // even: a TMA box must start on a 16-byte boundary of the plan-minor rows
    const int64_t want = (q.nplans + slots - 1) / slots;
    a.ppc = (int)std::min<int64_t>(P, std::max<int64_t>(2, (want + 1) / 2 * 2));
  };
#define GVP_V4_KS(NN, LL, KK)                                                                          \
  {                                                                                                    \
    if (split) {                                                                                \
      using LOH = v4::Lay<NN, LL, KK, true>;                                                           \
      GVP_CUDA(cudaFuncSetAttribute(v4::probe_split_kernel<NN, LL, KK>,                                \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LOH::BYTES));    \
      fill_ppc((const void*)v4::probe_split_kernel<NN, LL, KK>, LOH::BYTES, 128);                      \
      v4::probe_split_kernel<NN, LL, KK><<<(unsigned)((q.nplans + a.ppc - 1) / a.ppc), 128, LOH::BYTES, s>>>(a); \
    } else {                                                                                           \
      using LOH = v4::Lay<NN, LL, KK, false>;                                                          \
      GVP_CUDA(cudaFuncSetAttribute(v4::probe_fused_kernel<NN, LL, KK>,                                \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LOH::BYTES));    \
      v4::probe_fused_kernel<NN, LL, KK><<<grid, 64, LOH::BYTES, s>>>(a);                              \
    }                                                                                                  \
  }
#define GVP_V4(NN, LL) \
  if (q.kshared) GVP_V4_KS(NN, LL, true) else GVP_V4_KS(NN, LL, false)
#define GVP_V4_L(NN)                     \
  switch (L) {                           \
    case 1: GVP_V4(NN, 1) break;         \
    case 2: GVP_V4(NN, 2) break;         \
    case 4: GVP_V4(NN, 4) break;         \
    case 8: GVP_V4(NN, 8) break;         \
    default: GVP_V4(NN, 16) break;       \
  }
  switch (n) {
    case 2: GVP_V4_L(2) break;
    case 4: GVP_V4_L(4) break;
    case 6: GVP_V4_L(6) break;
    default:
      set_error("step kernel supports n in {2, 4, 6}");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_V4_L
#undef GVP_V4
#undef GVP_V4_KS
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp

#ifdef GVP_PROBE_PROFILE
// (diagnostic build) out[2 role + {0,1}] = cycles working / waiting since the last call
extern "C" int gvp_probe_profile(double* out) {
  unsigned long long h[8];
  GVP_CUDA(cudaMemcpyFromSymbol(h, gvp::v4::g_probe_prof, sizeof(h)));
  const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  GVP_CUDA(cudaMemcpyToSymbol(gvp::v4::g_probe_prof, z, sizeof(z)));
  for (int i = 0; i < 8; ++i) out[i] = (double)h[i];
  return GVP_OK;
}
#endif
