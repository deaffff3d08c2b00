// Kernels (b) and (c): block-tridiagonal chain algebra on B200.
//
// One thread owns one plan's chain (the recursions are sequential in the
// knot index), plans are interleaved in memory (plan-minor) so a warp's
// block loads are fully coalesced, and all n x n block arithmetic stays in
// registers. Sweep intermediates spill to a plan-minor scratch array.
//
//  * marginals_kernel      gbp_marginals  (gbp.py:43-80) + log det from the
//                          backward Schur pivots
//  * mean_solve_kernel     gbp_mean_solve (gbp.py:83-106), reference order
//  * logdet_fwd_kernel     logdet_block_tridiag (blocktri.py:151-174)
//  * prox_update_kernel    proximal_update (optimizer.py:129-161), reference order
//  * select_step_kernel    select_step_size (optimizer.py:188-231): the whole
//                          bisection per plan on device. Each probe is TWO
//                          passes over the chain instead of the reference's
//                          five (mean solve fwd+bwd, GBP bwd+fwd, log det):
//                            pass B (knot K-1 -> 0): GBP backward Schur of the
//                              candidate precision (SPD test + log det) fused
//                              with a backward block elimination of the mean
//                              system;
//                            pass F (knot 0 -> K-1): forward substitution of
//                              the mean fused with the covariance sweep, the
//                              trace tr(Lambda_k Sigma'), and the Mahalanobis
//                              term of kl_joint (optimizer.py:164-177).
//                          Candidates are evaluated without writing results;
//                          the accepted beta is re-run once in write mode.
#include <cuda_runtime.h>

#include <cmath>

#include "gvp_internal.cuh"

namespace gvp {

template <int N> constexpr int kT = N * (N + 1) / 2;

// plan-minor scratch: entry e of knot i of plan b at s[(i*E + e)*B + b]
struct Scratch {
  double* p;
  int64_t E, B;
  GVP_DEV double& at(int64_t b, int64_t i, int64_t e) const { return p[(i * E + e) * B + b]; }
};

template <int N>
GVP_DEV void store_tri(const Scratch& s, int64_t b, int64_t i, int off, const double (&A)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) s.at(b, i, off + tri_idx(r, c)) = A[r][c];
}
// lower-triangular (chol factor) load; upper zero
template <int N>
GVP_DEV void load_tri_lower(const Scratch& s, int64_t b, int64_t i, int off, double (&A)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) A[r][c] = (c <= r) ? s.at(b, i, off + tri_idx(r, c)) : 0.0;
}
// symmetric load (mirror)
template <int N>
GVP_DEV void load_tri_sym(const Scratch& s, int64_t b, int64_t i, int off, double (&A)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      const double v = s.at(b, i, off + tri_idx(r, c));
      A[r][c] = v;
      A[c][r] = v;
    }
}

// W <- L^{-1} U^T
template <int N>
GVP_DEV void solve_lower_transposed(const double (&L)[N][N], const double (&U)[N][N],
                                    double (&W)[N][N]) {
  transpose<N>(U, W);
  trsm_lower<N, N>(L, W);
}

// ============================================================ marginals (c)
template <int N>
__global__ void __launch_bounds__(64)
marginals_kernel(int nplans, int64_t K, View D, View U, MutView covs, MutView crosses,
                 double* __restrict__ logdet, int* __restrict__ status, int* __restrict__ where,
                 Scratch scr, const int* __restrict__ active) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  if (active && !active[b]) return;
  // ---- backward Schur sweep: Phi_i = D_i - U_i Phi_{i+1}^{-1} U_i^T (gbp.py:61-69)
  double Lnext[N][N], ld = 0.0;
  for (int64_t i = K - 1; i >= 0; --i) {
    double Phi[N][N];
    load_blk<N>(D, b, i, Phi);
    if (i < K - 1) {
      double Ui[N][N], W[N][N], G[N][N];
      load_blk<N>(U, b, i, Ui);
      solve_lower_transposed<N>(Lnext, Ui, W);
      gram_tn<N>(W, G);
      symmetrize<N>(Phi);  // symmetrize(D - U Phi^{-1} U^T), gbp.py:69
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) Phi[r][c] -= G[r][c];
    }
    double L[N][N];
    if (!chol<N>(Phi, L)) {
      status[b] = GVP_ERR_NOT_SPD;
      where[b] = (int)i;
      return;
    }
    ld += logdet_from_chol<N>(L);
    double Pinv[N][N];
    spd_inv_from_chol<N>(L, Pinv);
    store_tri<N>(scr, b, i, 0, Pinv);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) Lnext[r][c] = L[r][c];
  }
  // ---- forward covariance sweep (gbp.py:71-78)
  double S[N][N];
  load_tri_sym<N>(scr, b, 0, 0, S);  // Sigma_00 = Phi_0^{-1}
  store_blk<N>(covs, b, 0, S);
  for (int64_t i = 0; i + 1 < K; ++i) {
    double Ui[N][N], Pinv[N][N], A[N][N], M[N][N], Bm[N][N];
    load_blk<N>(U, b, i, Ui);
    load_tri_sym<N>(scr, b, i + 1, 0, Pinv);
    matmul<N>(S, Ui, A);     // Sigma_ii U_i
    matmul<N>(A, Pinv, M);   // Sigma_ii U_i Phi^{-1} = -Sigma_{i,i+1}
    matmul<N>(Ui, Pinv, Bm); // U_i Phi^{-1}
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) A[r][c] = -M[r][c];
    store_blk<N>(crosses, b, i, A);
    // Sigma_{i+1} = sym(Phi^{-1} + (U Phi^{-1})^T Sigma_ii U Phi^{-1})
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double t = Pinv[r][c];
#pragma unroll
        for (int k = 0; k < N; ++k) t += Bm[k][r] * M[k][c];
        S[r][c] = t;
      }
    symmetrize<N>(S);
    store_blk<N>(covs, b, i + 1, S);
  }
  if (logdet) logdet[b] = ld;
  status[b] = GVP_OK;
}

// ============================================================ mean solve
template <int N>
__global__ void __launch_bounds__(64)
mean_solve_kernel(int nplans, int64_t K, View D, View U, View eta, MutView out,
                  int* __restrict__ status, int* __restrict__ where, Scratch scr) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  // forward elimination (gbp.py:89-101); scratch: pivot chol (T) + rhs (N)
  double Lprev[N][N], rprev[N];
  for (int64_t i = 0; i < K; ++i) {
    double d[N][N], r[N];
    load_blk<N>(D, b, i, d);
    load_vec<N>(eta, b, i, r);
    if (i > 0) {
      double u[N][N], W[N][N], G[N][N];
      load_blk<N>(U, b, i - 1, u);
#pragma unroll
      for (int rr = 0; rr < N; ++rr)
#pragma unroll
        for (int c = 0; c < N; ++c) W[rr][c] = u[rr][c];
      trsm_lower<N, N>(Lprev, W);  // W = L^{-1} u
      gram_tn<N>(W, G);            // u^T P^{-1} u
      double y[N];
#pragma unroll
      for (int rr = 0; rr < N; ++rr) y[rr] = rprev[rr];
      trsv_lower<N>(Lprev, y);     // L^{-1} r_{i-1}
#pragma unroll
      for (int rr = 0; rr < N; ++rr) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) t += W[k][rr] * y[k];
        r[rr] -= t;
#pragma unroll
        for (int c = 0; c < N; ++c) d[rr][c] -= G[rr][c];
      }
    }
    symmetrize<N>(d);
    double L[N][N];
    if (!chol<N>(d, L)) {
      status[b] = GVP_ERR_NOT_SPD;
      where[b] = (int)i;
      return;
    }
    store_tri<N>(scr, b, i, 0, L);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) {
      scr.at(b, i, kT<N> + rr) = r[rr];
      rprev[rr] = r[rr];
#pragma unroll
      for (int c = 0; c < N; ++c) Lprev[rr][c] = L[rr][c];
    }
  }
  // back substitution (gbp.py:103-106)
  double xnext[N];
  for (int64_t i = K - 1; i >= 0; --i) {
    double L[N][N], r[N];
    load_tri_lower<N>(scr, b, i, 0, L);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) r[rr] = scr.at(b, i, kT<N> + rr);
    if (i < K - 1) {
      double u[N][N], t[N];
      load_blk<N>(U, b, i, u);
      matvec<N>(u, xnext, t);
#pragma unroll
      for (int rr = 0; rr < N; ++rr) r[rr] -= t[rr];
    }
    trsv_lower<N>(L, r);
    trsv_lower_t<N>(L, r);
    store_vec<N>(out, b, i, r);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) xnext[rr] = r[rr];
  }
  status[b] = GVP_OK;
}

// ============================================================ log det
template <int N>
__global__ void __launch_bounds__(64)
logdet_fwd_kernel(int nplans, int64_t K, View D, View U, double* __restrict__ out,
                  int* __restrict__ status, int* __restrict__ where, double* __restrict__ chols) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  double Lprev[N][N], ld = 0.0;
  for (int64_t i = 0; i < K; ++i) {
    double s[N][N];
    load_blk<N>(D, b, i, s);
    if (i > 0) {  // S_i = D_i - W^T W, W = L_{i-1}^{-1} U_{i-1} (blocktri.py:160-163)
      double W[N][N], G[N][N];
      load_blk<N>(U, b, i - 1, W);
      trsm_lower<N, N>(Lprev, W);
      gram_tn<N>(W, G);
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) s[r][c] -= G[r][c];
    }
    double L[N][N];
    if (!chol<N>(s, L)) {
      status[b] = GVP_ERR_NOT_SPD;
      where[b] = (int)i;
      return;
    }
    ld += logdet_from_chol<N>(L);
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Lprev[r][c] = L[r][c];
        if (chols) chols[((b * K + i) * N + r) * N + c] = c <= r ? L[r][c] : 0.0;  // forward_schur_chols
      }
  }
  out[b] = ld;
  status[b] = GVP_OK;
}

// ============================================================ step machinery
struct Coef {
  double inv_t, two_t, inv_b, c;  // 1/T, 2/T, 1/beta, beta/(beta+1)
};
GVP_DEV Coef make_coef(double temp, double beta) {
  Coef k;
  k.inv_t = 1.0 / temp;
  k.two_t = 2.0 / temp;
  k.inv_b = 1.0 / beta;
  k.c = beta / (beta + 1.0);
  return k;
}

// Lambda' block = c * ((G*(2/T) + K*(1/T)) + Lambda*(1/beta))  (optimizer.py:151-153)
template <int N>
GVP_DEV void next_prec_blk(const Coef& k, const double (&G)[N][N], const double (&Kb)[N][N],
                           const double (&Lb)[N][N], double (&out)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c)
      out[r][c] = (__dadd_rn(__dmul_rn(G[r][c], k.two_t), __dmul_rn(Kb[r][c], k.inv_t)) +
                   Lb[r][c] * k.inv_b) * k.c;
}
// system block S = K*(1/T) + Lambda*(1/beta)  (optimizer.py:155)
template <int N>
GVP_DEV void sys_blk(const Coef& k, const double (&Kb)[N][N], const double (&Lb)[N][N],
                     double (&out)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) out[r][c] = __dadd_rn(__dmul_rn(Kb[r][c], k.inv_t), __dmul_rn(Lb[r][c], k.inv_b));
}

template <int N>
GVP_DEV void load_blk_or_zero(const View& v, bool has, int64_t b, int64_t i, double (&a)[N][N]) {
  if (has) {
    load_blk<N>(v, b, i, a);
  } else {
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) a[r][c] = 0.0;
  }
}

// rhs_i = ((-g_i)/T + eta_i/T) + [Lob_ii mu_i + Lob_{i-1,i}^T mu_{i-1} + Lob_{i,i+1} mu_{i+1}]
// (optimizer.py:157-158 with BlockTridiagonalMatrix.matvec order, blocktri.py:117-127)
template <int N>
GVP_DEV void rhs_at(const Coef& k, const double (&g)[N], const double (&e)[N],
                    const double (&Ldiag)[N][N], const double (&mu)[N], bool has_prev,
                    const double (&Lprev)[N][N], const double (&mprev)[N], bool has_next,
                    const double (&Lnext)[N][N], const double (&mnext)[N], double temp,
                    double (&out)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double mv = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) mv += (Ldiag[r][c] * k.inv_b) * mu[c];
    if (has_prev) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) t += (Lprev[c][r] * k.inv_b) * mprev[c];
      mv += t;
    }
    if (has_next) {
      double t = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) t += (Lnext[r][c] * k.inv_b) * mnext[c];
      mv += t;
    }
    out[r] = (__ddiv_rn(-g[r], temp) + __ddiv_rn(e[r], temp)) + mv;
  }
}

// scratch layout of one probe: [PhiInv (T) | Lpsi (T) | y (N)]
template <int N> constexpr int kProbeE = 2 * kT<N> + N;

enum ProbeResult { kProbeOk = 0, kProbeNotSpd = 1, kProbeMeanFail = 2 };

struct ProbeIO {
  const StepProblem* pb;
  const StepOut* out;
  Scratch scr;
  int64_t K;
  double temp, logdet_cur;
};

// One candidate beta: returns ProbeResult; on kProbeOk sets kl (clipped like
// optimizer.py:177, NaN kept), ld_next, shift2 (= ||mu'-mu||^2).
template <int N, bool WRITE>
GVP_DEV int probe(const ProbeIO& io, int64_t b, double beta, double& kl, double& ld_next,
                  double& shift2, int& fail_knot) {
  const StepProblem& P = *io.pb;
  const int64_t K = io.K;
  const Coef k = make_coef(io.temp, beta);
  const Scratch& s = io.scr;
  constexpr int T = kT<N>;

  // ------------------------------------------------ pass B (backward)
  double LphiN[N][N], LpsiN[N][N], yN[N];
  double mu_i[N], mu_n[N], Loff_i[N][N];  // carried: mu_i, mu_{i+1}, Lambda_{i,i+1}
  double ld = 0.0;
  load_vec<N>(P.mean, b, K - 1, mu_i);
  for (int64_t i = K - 1; i >= 0; --i) {
    double Ld[N][N], Kd[N][N], Gd[N][N];
    load_blk<N>(P.diag, b, i, Ld);
    load_blk<N>(P.kdiag, b, i, Kd);
    load_blk<N>(P.gdiag, b, i, Gd);
    double mu_p[N], Loff_p[N][N];
    if (i > 0) {
      load_vec<N>(P.mean, b, i - 1, mu_p);
      load_blk<N>(P.off, b, i - 1, Loff_p);
    }
    // rhs of the mean system at knot i
    double g[N], e[N], rhs[N];
    load_vec<N>(P.gmu, b, i, g);
    load_vec<N>(P.info, b, i, e);
    rhs_at<N>(k, g, e, Ld, mu_i, i > 0, Loff_p, mu_p, i < K - 1, Loff_i, mu_n, io.temp, rhs);

    // candidate precision diag block and the GBP backward Schur step
    double Phi[N][N], Sd[N][N];
    next_prec_blk<N>(k, Gd, Kd, Ld, Phi);
    symmetrize<N>(Phi);  // .symmetrized() (blocktri.py:112-115)
    sys_blk<N>(k, Kd, Ld, Sd);
    symmetrize<N>(Sd);   // pivots are symmetrised in gbp_mean_solve (gbp.py:100)
    if (i < K - 1) {
      double Ko[N][N], Go[N][N], Up[N][N], So[N][N], W[N][N], G2[N][N];
      load_blk<N>(P.koff, b, i, Ko);
      load_blk_or_zero<N>(P.goff, P.has_goff, b, i, Go);
      next_prec_blk<N>(k, Go, Ko, Loff_i, Up);
      sys_blk<N>(k, Ko, Loff_i, So);
      solve_lower_transposed<N>(LphiN, Up, W);
      gram_tn<N>(W, G2);
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) Phi[r][c] -= G2[r][c];
      // mean: Psi_i = S_ii - S_{i,i+1} Psi_{i+1}^{-1} S_{i,i+1}^T ; r~_i = rhs_i - V^T y_{i+1}
      solve_lower_transposed<N>(LpsiN, So, W);
      gram_tn<N>(W, G2);
#pragma unroll
      for (int r = 0; r < N; ++r) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) t += W[q][r] * yN[q];
        rhs[r] -= t;
#pragma unroll
        for (int c = 0; c < N; ++c) Sd[r][c] -= G2[r][c];
      }
    }
    double Lphi[N][N];
    if (!chol<N>(Phi, Lphi)) {
      fail_knot = (int)i;
      return kProbeNotSpd;
    }
    ld += logdet_from_chol<N>(Lphi);
    double Lpsi[N][N];
    if (!chol<N>(Sd, Lpsi)) {
      fail_knot = (int)i;
      return kProbeMeanFail;
    }
    trsv_lower<N>(Lpsi, rhs);  // y_i = Lpsi^{-1} r~_i
    {
      double Pinv[N][N];
      spd_inv_from_chol<N>(Lphi, Pinv);
      store_tri<N>(s, b, i, 0, Pinv);
    }
    store_tri<N>(s, b, i, T, Lpsi);
#pragma unroll
    for (int r = 0; r < N; ++r) {
      s.at(b, i, 2 * T + r) = rhs[r];
      yN[r] = rhs[r];
      mu_n[r] = mu_i[r];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        LphiN[r][c] = Lphi[r][c];
        LpsiN[r][c] = Lpsi[r][c];
      }
    }
    if (i > 0) {
#pragma unroll
      for (int r = 0; r < N; ++r) {
        mu_i[r] = mu_p[r];
#pragma unroll
        for (int c = 0; c < N; ++c) Loff_i[r][c] = Loff_p[r][c];
      }
    }
  }

  // ------------------------------------------------ pass F (forward)
  double Sig[N][N], Sprev[N][N], Lo_prev[N][N], mprev[N], dprev[N];
  load_tri_sym<N>(s, b, 0, 0, Sig);  // Sigma_00 = Phi_0^{-1}
  double trace = 0.0, mahal = 0.0, sh2 = 0.0;
  double pq = 0.0, ptr = 0.0, dpprev[N], Ko_prev[N][N];  // prior-cost pieces (WRITE only)
  for (int64_t i = 0; i < K; ++i) {
    // mean: mu'_i = Lpsi^{-T} (y_i - Lpsi^{-1} S_{i-1,i}^T mu'_{i-1})
    double Lpsi[N][N], m[N];
    load_tri_lower<N>(s, b, i, T, Lpsi);
#pragma unroll
    for (int r = 0; r < N; ++r) m[r] = s.at(b, i, 2 * T + r);
    if (i > 0) {
      double z[N];
      matvec_t<N>(Sprev, mprev, z);
      trsv_lower<N>(Lpsi, z);
#pragma unroll
      for (int r = 0; r < N; ++r) m[r] -= z[r];
    }
    trsv_lower_t<N>(Lpsi, m);
    double Ld[N][N], mu[N], dl[N];
    load_blk<N>(P.diag, b, i, Ld);
    load_vec<N>(P.mean, b, i, mu);
#pragma unroll
    for (int r = 0; r < N; ++r) {
      dl[r] = mu[r] - m[r];  // delta = cur.mean - nxt.mean (optimizer.py:173)
      sh2 += dl[r] * dl[r];
    }
    // KL pieces at knot i: tr(Lambda_ii Sigma_ii), delta' Lambda delta
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        trace += Ld[r][c] * Sig[c][r];
        mahal += dl[r] * Ld[r][c] * dl[c];
      }
    if (i > 0) {
      double t = 0.0;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) t += dprev[r] * Lo_prev[r][c] * dl[c];
      mahal += 2.0 * t;
    }
    double dp[N];  // m - prior mean (cost_breakdown, optimizer.py:260-263)
    if (WRITE) {
      double Kd[N][N], Gd[N][N], Pn[N][N];
      load_blk<N>(P.kdiag, b, i, Kd);
      load_blk<N>(P.gdiag, b, i, Gd);
      next_prec_blk<N>(k, Gd, Kd, Ld, Pn);
      symmetrize<N>(Pn);
      store_vec<N>(io.out->mean, b, i, m);
      store_blk<N>(io.out->diag, b, i, Pn);
      store_blk<N>(io.out->covs, b, i, Sig);
      if (P.has_pmean) {
        double pm[N];
        load_vec<N>(P.pmean, b, i, pm);
#pragma unroll
        for (int r = 0; r < N; ++r) dp[r] = m[r] - pm[r];
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c) {
            pq += dp[r] * Kd[r][c] * dp[c];
            ptr += Kd[r][c] * Sig[c][r];
          }
        if (i > 0) {
          double t = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int c = 0; c < N; ++c) t += dpprev[r] * Ko_prev[r][c] * dp[c];
          pq += 2.0 * t;
        }
      }
    }
    if (i + 1 < K) {
      double Lo[N][N], Ko[N][N], Go[N][N], Up[N][N], Pinv[N][N], A[N][N], M[N][N], Bm[N][N];
      load_blk<N>(P.off, b, i, Lo);
      load_blk<N>(P.koff, b, i, Ko);
      load_blk_or_zero<N>(P.goff, P.has_goff, b, i, Go);
      next_prec_blk<N>(k, Go, Ko, Lo, Up);
      sys_blk<N>(k, Ko, Lo, Sprev);
      load_tri_sym<N>(s, b, i + 1, 0, Pinv);
      matmul<N>(Sig, Up, A);
      matmul<N>(A, Pinv, M);   // -Sigma_{i,i+1}
      matmul<N>(Up, Pinv, Bm);
      double tc = 0.0;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          tc += Lo[r][c] * M[r][c];
          A[r][c] = -M[r][c];
        }
      trace -= 2.0 * tc;  // 2 <Lambda_{i,i+1}, Sigma_{i,i+1}> (gbp.py:118-119)
      if (WRITE) {
        store_blk<N>(io.out->crosses, b, i, A);
        store_blk<N>(io.out->off, b, i, Up);
        if (P.has_pmean) {
          double t = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int c = 0; c < N; ++c) {
              t += Ko[r][c] * A[r][c];
              Ko_prev[r][c] = Ko[r][c];
            }
          ptr += 2.0 * t;
        }
      }
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double t = Pinv[r][c];
#pragma unroll
          for (int q = 0; q < N; ++q) t += Bm[q][r] * M[q][c];
          Sig[r][c] = t;
        }
      symmetrize<N>(Sig);
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) Lo_prev[r][c] = Lo[r][c];
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      mprev[r] = m[r];
      dprev[r] = dl[r];
      if (WRITE) dpprev[r] = dp[r];
    }
  }
  if (WRITE && P.has_pmean && io.out->prior_cost)
    io.out->prior_cost[b] = 0.5 * pq + 0.5 * ptr;
  const double dim = (double)(K * N);
  const double x = 0.5 * ((((trace + mahal) - dim) + ld) - io.logdet_cur);
  kl = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
  ld_next = ld;
  shift2 = sh2;
  return kProbeOk;
}

template <int N>
__global__ void __launch_bounds__(64)
select_step_kernel(int nplans, int64_t K, StepProblem pb, StepParams pr, StepOut out,
                   Scratch scr, const int* __restrict__ active) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  if (active && !active[b]) return;
  ProbeIO io{&pb, &out, scr, K, pr.temp[b], pr.logdet_cur ? pr.logdet_cur[b] : 0.0};
  int nprobe = 0;
  double kl = 0.0, ld = 0.0, sh = 0.0;
  int fk = -1;
  auto log_probe = [&](double beta, int res, double klv) {
    if (out.probe_log && nprobe < out.max_probes) {
      double* row = out.probe_log + (b * out.max_probes + nprobe) * 3;
      row[0] = beta;
      row[1] = res == kProbeOk ? 1.0 : 0.0;
      row[2] = res == kProbeOk ? klv : INFINITY;
    }
    ++nprobe;
  };
  auto feasible = [&](int res, double klv) { return res == kProbeOk && !(klv > pr.kl_bound); };
  auto fail = [&](int code, int w) {
    out.status[b] = code;
    out.where[b] = w;
    if (out.nprobes) out.nprobes[b] = nprobe;
  };

  // select_step_size as one loop (one inlined probe): phase 0 probes beta_max,
  // phase 1 beta_min, phase 2 bisects while (hi - lo) > 1e-3 hi
  // (_BISECTION_RTOL, optimizer.py:39,213-230).
  double best = pr.beta_max, lo = pr.beta_min, hi = pr.beta_max, beta = pr.beta_max;
  int phase = 0, res;
  for (;;) {
    res = probe<N, false>(io, b, beta, kl, ld, sh, fk);
    log_probe(beta, res, kl);
    if (res == kProbeMeanFail) return fail(GVP_ERR_NOT_SPD, fk | GVP_WHERE_MEAN_SOLVE_BIAS);
    const bool ok = feasible(res, kl);
    if (phase == 0) {
      if (ok) break;  // best = beta_max
      phase = 1;
      beta = pr.beta_min;
      continue;
    }
    if (phase == 1) {
      if (!ok) return fail(GVP_ERR_NO_FEASIBLE_STEP, -1);
      best = pr.beta_min;
      phase = 2;
    } else if (ok) {
      lo = beta;
      best = beta;
    } else {
      hi = beta;
    }
    if (!((hi - lo) > 1e-3 * hi)) break;
    beta = 0.5 * (lo + hi);
  }
  // commit: re-run the accepted candidate writing state + marginals
  res = probe<N, true>(io, b, best, kl, ld, sh, fk);
  out.beta[b] = best;
  out.kl[b] = kl;
  if (out.logdet_next) out.logdet_next[b] = ld;
  if (out.mean_shift) out.mean_shift[b] = sqrt(sh);
  if (out.nprobes) out.nprobes[b] = nprobe;
  out.status[b] = GVP_OK;
  out.where[b] = -1;
}

// proximal_update alone (optimizer.py:129-161), mean solve in the reference's
// forward-elimination order (gbp.py:83-106) on the system K/T + Lambda/beta.
template <int N>
__global__ void __launch_bounds__(64)
prox_update_kernel(int nplans, int64_t K, StepProblem pb, StepParams pr, StepOut out,
                   Scratch scr) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nplans) return;
  const double temp = pr.temp[b];
  const Coef k = make_coef(temp, pr.beta_fixed[b]);
  constexpr int T = kT<N>;
  double Lprev[N][N], rprev[N];
  double mu_p[N], mu_i[N], mu_n[N], Lo_p[N][N], Lo_i[N][N];
  load_vec<N>(pb.mean, b, 0, mu_i);
  for (int64_t i = 0; i < K; ++i) {
    double Ld[N][N], Kd[N][N], Gd[N][N], d[N][N], g[N], e[N], r[N];
    load_blk<N>(pb.diag, b, i, Ld);
    load_blk<N>(pb.kdiag, b, i, Kd);
    load_blk<N>(pb.gdiag, b, i, Gd);
    if (i + 1 < K) {
      load_vec<N>(pb.mean, b, i + 1, mu_n);
      load_blk<N>(pb.off, b, i, Lo_i);
    }
    load_vec<N>(pb.gmu, b, i, g);
    load_vec<N>(pb.info, b, i, e);
    rhs_at<N>(k, g, e, Ld, mu_i, i > 0, Lo_p, mu_p, i + 1 < K, Lo_i, mu_n, temp, r);
    // next precision blocks
    {
      double Pn[N][N];
      next_prec_blk<N>(k, Gd, Kd, Ld, Pn);
      symmetrize<N>(Pn);
      store_blk<N>(out.diag, b, i, Pn);
      if (i + 1 < K) {
        double Ko[N][N], Go[N][N], Up[N][N];
        load_blk<N>(pb.koff, b, i, Ko);
        load_blk_or_zero<N>(pb.goff, pb.has_goff, b, i, Go);
        next_prec_blk<N>(k, Go, Ko, Lo_i, Up);
        store_blk<N>(out.off, b, i, Up);
      }
    }
    sys_blk<N>(k, Kd, Ld, d);
    if (i > 0) {
      double Ko[N][N], u[N][N], W[N][N], G[N][N], y[N];
      load_blk<N>(pb.koff, b, i - 1, Ko);
      sys_blk<N>(k, Ko, Lo_p, u);
#pragma unroll
      for (int rr = 0; rr < N; ++rr)
#pragma unroll
        for (int c = 0; c < N; ++c) W[rr][c] = u[rr][c];
      trsm_lower<N, N>(Lprev, W);
      gram_tn<N>(W, G);
#pragma unroll
      for (int rr = 0; rr < N; ++rr) y[rr] = rprev[rr];
      trsv_lower<N>(Lprev, y);
#pragma unroll
      for (int rr = 0; rr < N; ++rr) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) t += W[q][rr] * y[q];
        r[rr] -= t;
#pragma unroll
        for (int c = 0; c < N; ++c) d[rr][c] -= G[rr][c];
      }
    }
    symmetrize<N>(d);
    double L[N][N];
    if (!chol<N>(d, L)) {
      out.status[b] = GVP_ERR_NOT_SPD;
      out.where[b] = (int)i;
      return;
    }
    store_tri<N>(scr, b, i, 0, L);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) {
      scr.at(b, i, T + rr) = r[rr];
      rprev[rr] = r[rr];
      mu_p[rr] = mu_i[rr];
      mu_i[rr] = mu_n[rr];
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Lprev[rr][c] = L[rr][c];
        Lo_p[rr][c] = Lo_i[rr][c];
      }
    }
  }
  double xnext[N];
  for (int64_t i = K - 1; i >= 0; --i) {
    double L[N][N], r[N];
    load_tri_lower<N>(scr, b, i, 0, L);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) r[rr] = scr.at(b, i, T + rr);
    if (i < K - 1) {
      double Ko[N][N], Lo[N][N], u[N][N], t[N];
      load_blk<N>(pb.koff, b, i, Ko);
      load_blk<N>(pb.off, b, i, Lo);
      sys_blk<N>(k, Ko, Lo, u);
      matvec<N>(u, xnext, t);
#pragma unroll
      for (int rr = 0; rr < N; ++rr) r[rr] -= t[rr];
    }
    trsv_lower<N>(L, r);
    trsv_lower_t<N>(L, r);
    store_vec<N>(out.mean, b, i, r);
#pragma unroll
    for (int rr = 0; rr < N; ++rr) xnext[rr] = r[rr];
  }
  out.status[b] = GVP_OK;
  out.where[b] = -1;
}

// ============================================================ launchers
static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
constexpr int kChainTpb = 32;

int64_t chain_scratch_doubles(int nplans, int64_t K, int n, int lanes) {
  const int64_t T = (int64_t)n * (n + 1) / 2;
  const int64_t E = 2 * T + n;
  return std::max<int64_t>(1, K * E * (int64_t)nplans * std::max(1, lanes));
}

#define GVP_DISPATCH_N(n, ...)                          \
  switch (n) {                                           \
    case 1: { constexpr int NN = 1; __VA_ARGS__; } break;       \
    case 2: { constexpr int NN = 2; __VA_ARGS__; } break;       \
    case 3: { constexpr int NN = 3; __VA_ARGS__; } break;       \
    case 4: { constexpr int NN = 4; __VA_ARGS__; } break;       \
    case 5: { constexpr int NN = 5; __VA_ARGS__; } break;       \
    case 6: { constexpr int NN = 6; __VA_ARGS__; } break;       \
    case 7: { constexpr int NN = 7; __VA_ARGS__; } break;       \
    case 8: { constexpr int NN = 8; __VA_ARGS__; } break;       \
    default:                                             \
      set_error("block size n must be in 1..8");         \
      return GVP_ERR_UNSUPPORTED;                        \
  }

int launch_marginals(int nplans, int64_t K, int n, const View& D, const View& U,
                     const MutView& covs, const MutView& crosses, double* logdet, int* status,
                     int* where, double* scratch, const int* active, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  GVP_DISPATCH_N(n, {
    Scratch scr{scratch, (int64_t)kProbeE<NN>, nplans};
    marginals_kernel<NN><<<nblk(nplans, kChainTpb), kChainTpb, 0, s>>>(
        nplans, K, D, U, covs, crosses, logdet, status, where, scr, active);
  });
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int launch_mean_solve(int nplans, int64_t K, int n, const View& D, const View& U,
                      const View& eta, const MutView& out, int* status, int* where,
                      double* scratch, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  GVP_DISPATCH_N(n, {
    Scratch scr{scratch, (int64_t)kProbeE<NN>, nplans};
    mean_solve_kernel<NN><<<nblk(nplans, kChainTpb), kChainTpb, 0, s>>>(
        nplans, K, D, U, eta, out, status, where, scr);
  });
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int launch_logdet_fwd(int nplans, int64_t K, int n, const View& D, const View& U, double* out,
                      int* status, int* where, double* chols, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  GVP_DISPATCH_N(n, {
    logdet_fwd_kernel<NN><<<nblk(nplans, kChainTpb), kChainTpb, 0, s>>>(nplans, K, D, U, out,
                                                                         status, where, chols);
  });
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int launch_select_step(int nplans, int64_t K, int n, const StepProblem& pb, const StepParams& pr,
                       const StepOut& out, double* scratch, const int* active, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  GVP_DISPATCH_N(n, {
    Scratch scr{scratch, (int64_t)kProbeE<NN>, nplans};
    if (pr.fixed_beta) {
      prox_update_kernel<NN><<<nblk(nplans, kChainTpb), kChainTpb, 0, s>>>(nplans, K, pb, pr,
                                                                             out, scr);
    } else {
      select_step_kernel<NN><<<nblk(nplans, kChainTpb), kChainTpb, 0, s>>>(nplans, K, pb, pr,
                                                                             out, scr, active);
    }
  });
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp
