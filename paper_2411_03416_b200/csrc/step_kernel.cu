// Packed-layout chain helpers shared by the engine and the drop-in step:
// GBP marginals (gbp.py:43-80) with the log det from the backward Schur
// pivots, and v = Lambda mu (the rhs piece of the proximal mean system,
// optimizer.py:157-158). Diagonal blocks packed lower-symmetric, plan-minor.
#include <cuda_runtime.h>

#include <cmath>

#include "gvp_internal.cuh"

namespace gvp {
namespace v2 {

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

}  // namespace gvp
