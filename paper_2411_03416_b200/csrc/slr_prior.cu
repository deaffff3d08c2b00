// iP-GVIMP on the device: the statistical linearisation of
// the planar quadrotor (slr.py:49-92) and the LTV prior assembly
// (prior.py:56-170) for every knot / step in parallel.
//
//   slr_kernel          one thread per (plan, knot): gaussian_sqrt root of the
//                       nominal covariance, sigma points through one Euler step
//                       of the drift (dynamics.py:99-124), weighted affine fit
//                       A_d = P_yx P_xx^-1 (relative 1e-9 jitter on a singular
//                       P_xx), A = (A_d - I)/dt, a = a_d/dt.
//   prior_node_kernel   one thread per (plan, step, node): node < Q: the
//                       Gauss-Legendre term w expm(A (dt-s)) q_c BB' expm(.)'
//                       of the Grammian; node Q: expm([[A, a], [0, 0]] dt).
//   prior_step_kernel   one thread per (plan, step): Grammian sum in node order,
//                       symmetrise, Cholesky (+1e-10 I retry), Q^-1.
//   prior_knot_kernel   one thread per (plan, knot): the anchored precision
//                       blocks and information vector in the reference's
//                       accumulation order, diagonal symmetrised.
// expm is scaling-and-squaring with diagonal Pade approximants of degree
// 3/5/7/9/13 (Higham 2005). scipy's expm (Al-Mohy & Higham 2009) may pick a
// different degree/scaling; both are accurate to ~1e-15 relative, and the
// tests bound the difference in the assembled prior accordingly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "gvp_internal.cuh"

namespace gvp {
namespace slrp {

constexpr int NS = 6;   // quadrotor state
constexpr int MI = 2;   // noise inputs

template <int M>
GVP_DEV void matmul(const double (&A)[M * M], const double (&B)[M * M], double (&C)[M * M]) {
#pragma unroll
  for (int r = 0; r < M; ++r)
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < M; ++k) t += A[r * M + k] * B[k * M + c];
      C[r * M + c] = t;
    }
}

// X = (V - U)^-1 (V + U) by Gaussian elimination with partial pivoting
template <int M>
GVP_DEV bool pade_solve(double (&P)[M * M], double (&Q)[M * M]) {
#pragma unroll 1
  for (int c = 0; c < M; ++c) {
    int piv = c;
    double best = fabs(P[c * M + c]);
    for (int r = c + 1; r < M; ++r)
      if (fabs(P[r * M + c]) > best) {
        best = fabs(P[r * M + c]);
        piv = r;
      }
    if (!(best > 0.0)) return false;
    if (piv != c)
      for (int k = 0; k < M; ++k) {
        double t = P[c * M + k];
        P[c * M + k] = P[piv * M + k];
        P[piv * M + k] = t;
        t = Q[c * M + k];
        Q[c * M + k] = Q[piv * M + k];
        Q[piv * M + k] = t;
      }
    const double inv = 1.0 / P[c * M + c];
    for (int r = c + 1; r < M; ++r) {
      const double f = P[r * M + c] * inv;
      if (f == 0.0) continue;
      for (int k = c; k < M; ++k) P[r * M + k] -= f * P[c * M + k];
      for (int k = 0; k < M; ++k) Q[r * M + k] -= f * Q[c * M + k];
    }
  }
  for (int c = M - 1; c >= 0; --c) {
    const double inv = 1.0 / P[c * M + c];
    for (int k = 0; k < M; ++k) {
      double t = Q[c * M + k];
      for (int j = c + 1; j < M; ++j) t -= P[c * M + j] * Q[j * M + k];
      Q[c * M + k] = t * inv;
    }
  }
  return true;
}

// exp(A) in place (Higham 2005 scaling and squaring, Pade 3..13)
template <int M>
GVP_DEV bool expm(double (&A)[M * M]) {
  constexpr double theta[5] = {1.495585217958292e-2, 2.539398330063230e-1, 9.504178996162932e-1,
                               2.097847961257068e0, 5.371920351148152e0};
  constexpr double c3[4] = {120., 60., 12., 1.};
  constexpr double c5[6] = {30240., 15120., 3360., 420., 30., 1.};
  constexpr double c7[8] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.};
  constexpr double c9[10] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                             2162160., 110880., 3960., 90., 1.};
  constexpr double c13[14] = {64764752532480000., 32382376266240000., 7771770303897600.,
                              1187353796428800., 129060195264000., 10559470521600., 670442572800.,
                              33522128640., 1323241920., 40840800., 960960., 16380., 182., 1.};
  double nrm = 0.0;  // 1-norm
  for (int c = 0; c < M; ++c) {
    double t = 0.0;
    for (int r = 0; r < M; ++r) t += fabs(A[r * M + c]);
    nrm = fmax(nrm, t);
  }
  if (!isfinite(nrm)) return false;
  int s = 0;
  int deg = 13;
  if (nrm <= theta[0]) deg = 3;
  else if (nrm <= theta[1]) deg = 5;
  else if (nrm <= theta[2]) deg = 7;
  else if (nrm <= theta[3]) deg = 9;
  else {
    s = (int)ceil(log2(nrm / theta[4]));
    if (s < 0) s = 0;
    const double sc = ldexp(1.0, -s);
    for (int k = 0; k < M * M; ++k) A[k] *= sc;
  }
  double A2[M * M], A4[M * M], A6[M * M], U[M * M], V[M * M], T[M * M];
  matmul<M>(A, A, A2);
  if (deg == 13) {
    matmul<M>(A2, A2, A4);
    matmul<M>(A4, A2, A6);
    for (int k = 0; k < M * M; ++k) T[k] = c13[13] * A6[k] + c13[11] * A4[k] + c13[9] * A2[k];
    matmul<M>(A6, T, U);  // A6 (b13 A6 + b11 A4 + b9 A2)
    for (int k = 0; k < M * M; ++k) U[k] += c13[7] * A6[k] + c13[5] * A4[k] + c13[3] * A2[k];
    for (int r = 0; r < M; ++r) U[r * M + r] += c13[1];
    matmul<M>(A, U, T);
    for (int k = 0; k < M * M; ++k) U[k] = T[k];
    for (int k = 0; k < M * M; ++k) T[k] = c13[12] * A6[k] + c13[10] * A4[k] + c13[8] * A2[k];
    matmul<M>(A6, T, V);
    for (int k = 0; k < M * M; ++k) V[k] += c13[6] * A6[k] + c13[4] * A4[k] + c13[2] * A2[k];
    for (int r = 0; r < M; ++r) V[r * M + r] += c13[0];
  } else {
    const double* c = deg == 3 ? c3 : deg == 5 ? c5 : deg == 7 ? c7 : c9;
    // U = A sum_k c[2k+1] A^{2k},  V = sum_k c[2k] A^{2k}
    double P[M * M];
    for (int k = 0; k < M * M; ++k) {
      T[k] = c[1] * ((k / M) == (k % M) ? 1.0 : 0.0);
      V[k] = c[0] * ((k / M) == (k % M) ? 1.0 : 0.0);
      P[k] = (k / M) == (k % M) ? 1.0 : 0.0;
    }
    for (int j = 1; 2 * j <= deg; ++j) {
      matmul<M>(P, A2, A4);  // P <- A^{2j}
      for (int k = 0; k < M * M; ++k) {
        P[k] = A4[k];
        T[k] += c[2 * j + 1] * P[k];
        V[k] += c[2 * j] * P[k];
      }
    }
    matmul<M>(A, T, U);
  }
  double L[M * M];
  for (int k = 0; k < M * M; ++k) {
    L[k] = V[k] - U[k];
    A[k] = V[k] + U[k];
  }
  if (!pade_solve<M>(L, A)) return false;
  for (int k = 0; k < s; ++k) {
    matmul<M>(A, A, T);
    for (int q = 0; q < M * M; ++q) A[q] = T[q];
  }
  return true;
}

// lower Cholesky of a full symmetric M x M (numpy's cholesky reads the lower triangle)
template <int M>
GVP_DEV bool chol_full(const double (&S)[M * M], double (&L)[M * M], double jitter) {
  for (int k = 0; k < M * M; ++k) L[k] = 0.0;
  for (int j = 0; j < M; ++j) {
    double s = S[j * M + j] + jitter;
    for (int k = 0; k < j; ++k) s -= L[j * M + k] * L[j * M + k];
    if (!(s > 0.0)) return false;
    const double d = sqrt(s);
    L[j * M + j] = d;
    for (int i = j + 1; i < M; ++i) {
      double t = S[i * M + j];
      for (int k = 0; k < j; ++k) t -= L[i * M + k] * L[j * M + k];
      L[i * M + j] = t / d;
    }
  }
  return true;
}

struct Quad {
  double inv_mass, len_over_inertia, gravity;
};

GVP_DEV void quad_drift(const double* x, const Quad& q, double* f) {
  double sp, cp;
  sincos(x[2], &sp, &cp);
  f[0] = x[3] * cp - x[4] * sp;
  f[1] = x[3] * sp + x[4] * cp;
  f[2] = x[5];
  f[3] = x[4] * x[5] - q.gravity * sp;
  f[4] = -x[3] * x[5] - q.gravity * cp;
  f[5] = 0.0;
}

__global__ void slr_kernel(int nplans, int K, const double* __restrict__ means, const double* __restrict__ covs,
                           const double* __restrict__ pts, const double* __restrict__ wts, int Q, double dt,
                           Quad qp, double* __restrict__ Aout, double* __restrict__ aout, int* status,
                           int* where) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nplans * K) return;
  const int b = t / K, i = t % K;
  constexpr int M = NS;
  double S[M * M], L[M * M], xb[M];
  for (int k = 0; k < M * M; ++k) S[k] = covs[(size_t)t * M * M + k];
  for (int k = 0; k < M; ++k) xb[k] = means[(size_t)t * M + k];
  // gaussian_sqrt (quadrature.py:164-181): Cholesky, then +1e-10 I; the eigh root is host-only
  if (!chol_full<M>(S, L, 0.0) && !chol_full<M>(S, L, 1e-10)) {
    atomicCAS(&status[b], GVP_OK, GVP_ERR_SQRT);
    atomicCAS(&where[b], -1, i);
    return;
  }
  auto point = [&](int l, double (&x)[M], double (&y)[M]) {
    for (int r = 0; r < M; ++r) {
      double v = 0.0;
      for (int k = 0; k <= r; ++k) v += L[r * M + k] * pts[l * M + k];
      x[r] = xb[r] + v;
    }
    double f[M];
    quad_drift(x, qp, f);
    for (int r = 0; r < M; ++r) y[r] = x[r] + f[r] * dt;
  };
  double xm[M] = {0}, ym[M] = {0};
  bool finite = true;
  for (int l = 0; l < Q; ++l) {
    double x[M], y[M];
    point(l, x, y);
    const double w = wts[l];
    for (int r = 0; r < M; ++r) {
      xm[r] += w * x[r];
      ym[r] += w * y[r];
      finite = finite && isfinite(y[r]);
    }
  }
  if (!finite) {  // euler_step raises FloatingPointError (dynamics.py:118-121)
    atomicCAS(&status[b], GVP_OK, GVP_ERR_NONFINITE);
    atomicCAS(&where[b], -1, i);
    return;
  }
  double Pxx[M * M] = {0}, Pyx[M * M] = {0};
  for (int l = 0; l < Q; ++l) {
    double x[M], y[M];
    point(l, x, y);
    const double w = wts[l];
    double dx[M];
    for (int r = 0; r < M; ++r) dx[r] = (x[r] - xm[r]) * w;
    for (int r = 0; r < M; ++r) {
      const double ex = x[r] - xm[r], ey = y[r] - ym[r];
      for (int c = 0; c < M; ++c) {
        Pxx[r * M + c] += ex * dx[c];
        Pyx[r * M + c] += ey * dx[c];
      }
    }
  }
  // _fit_affine (slr.py:49-66): Cholesky of P_xx, relative jitter on failure
  double Lx[M * M];
  if (!chol_full<M>(Pxx, Lx, 0.0)) {
    double tr = 0.0;
    for (int r = 0; r < M; ++r) tr += Pxx[r * M + r];
    const double scale = fmax(tr / M, 2.2250738585072014e-308);
    if (!chol_full<M>(Pxx, Lx, 1e-9 * scale)) {
      atomicCAS(&status[b], GVP_OK, GVP_ERR_NOT_SPD);
      atomicCAS(&where[b], -1, i);
      return;
    }
  }
  // A_d = (Lx^-T Lx^-1 Pyx^T)^T, row by row of A_d (= column of the solve)
  double* Ao = Aout + (size_t)t * M * M;
  double ad[M * M];
  for (int r = 0; r < M; ++r) {
    double z[M];
    for (int j = 0; j < M; ++j) {  // forward: Lx z = Pyx[r, :]^T
      double v = Pyx[r * M + j];
      for (int k = 0; k < j; ++k) v -= Lx[j * M + k] * z[k];
      z[j] = v / Lx[j * M + j];
    }
    for (int j = M - 1; j >= 0; --j) {  // backward: Lx^T x = z
      double v = z[j];
      for (int k = j + 1; k < M; ++k) v -= Lx[k * M + j] * ad[r * M + k];
      ad[r * M + j] = v / Lx[j * M + j];
    }
  }
  for (int r = 0; r < M; ++r) {
    double v = 0.0;
    for (int c = 0; c < M; ++c) {
      v += ad[r * M + c] * xm[c];
      Ao[r * M + c] = (ad[r * M + c] - (r == c ? 1.0 : 0.0)) / dt;
    }
    aout[(size_t)t * M + r] = (ym[r] - v) / dt;
  }
}

// one (plan, step, node): node < nodes: Grammian term; node == nodes: augmented expm
__global__ void prior_node_kernel(int nplans, int S, int n, int m, const double* __restrict__ A,
                                  const double* __restrict__ av, const double* __restrict__ Bm, double dt,
                                  double q_c, const double* __restrict__ gl_s, const double* __restrict__ gl_w,
                                  int nodes, double* __restrict__ terms, double* __restrict__ phis,
                                  double* __restrict__ offs, int* status, int* where) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int per = nodes + 1;
  if (t >= nplans * S * per) return;
  const int node = t % per, bs = t / per, b = bs / S, i = bs % S;
  const double* Ai = A + (size_t)bs * n * n;
  if (n != NS) return;  // host checks n == 6
  constexpr int M = NS;
  if (node == nodes) {
    constexpr int M1 = M + 1;
    double E[M1 * M1];
    for (int r = 0; r < M1; ++r)
      for (int c = 0; c < M1; ++c)
        E[r * M1 + c] = (r < M ? (c < M ? Ai[r * M + c] : av[(size_t)bs * M + r]) : 0.0) * dt;
    if (!expm<M1>(E)) {
      atomicCAS(&status[b], GVP_OK, GVP_ERR_NONFINITE);
      atomicCAS(&where[b], -1, i);
      return;
    }
    for (int r = 0; r < M; ++r) {
      for (int c = 0; c < M; ++c) phis[((size_t)bs * M + r) * M + c] = E[r * M1 + c];
      offs[(size_t)bs * M + r] = E[r * M1 + M];
    }
    return;
  }
  // w expm(A (dt - s)) (q_c B B') expm(.)'   (prior.py:86-94)
  const double sv = 0.5 * dt * (gl_s[node] + 1.0), wv = 0.5 * dt * gl_w[node];
  double E[M * M];
  for (int k = 0; k < M * M; ++k) E[k] = Ai[k] * (dt - sv);
  if (!expm<M>(E)) {
    atomicCAS(&status[b], GVP_OK, GVP_ERR_NONFINITE);
    atomicCAS(&where[b], -1, i);
    return;
  }
  const double* Bi = Bm + (size_t)bs * M * m;
  double bqb[M * M], EB[M * M];
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) {
      double v = 0.0;
      for (int k = 0; k < m; ++k) v += Bi[r * m + k] * Bi[c * m + k];
      bqb[r * M + c] = q_c * v;
    }
  matmul<M>(E, bqb, EB);
  double* out = terms + ((size_t)bs * nodes + node) * M * M;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) {
      double v = 0.0;
      for (int k = 0; k < M; ++k) v += EB[r * M + k] * E[c * M + k];
      out[r * M + c] = wv * v;
    }
}

// Grammian (node order), symmetrise, SPD check with 1e-10 retry, inverse
__global__ void prior_step_kernel(int nplans, int S, int nodes, const double* __restrict__ terms,
                                  double* __restrict__ grams, double* __restrict__ qinv, int* status, int* where,
                                  double reg) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nplans * S) return;
  constexpr int M = NS;
  const int b = t / S, i = t % S;
  double G[M * M] = {0};
  for (int k = 0; k < nodes; ++k)
    for (int q = 0; q < M * M; ++q) G[q] += terms[((size_t)t * nodes + k) * M * M + q];
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < r; ++c) {
      const double v = 0.5 * (G[r * M + c] + G[c * M + r]);
      G[r * M + c] = v;
      G[c * M + r] = v;
    }
  if (reg > 0.0) {  // robust-conditioning mode: Q + reg tr(Q)/n I (deviates from the reference)
    double tr = 0.0;
    for (int r = 0; r < M; ++r) tr += G[r * M + r];
    for (int r = 0; r < M; ++r) G[r * M + r] += reg * tr / M;
  }
  double L[M * M];
  if (!chol_full<M>(G, L, 0.0)) {
    for (int r = 0; r < M; ++r) G[r * M + r] += 1e-10;  // _GRAMMIAN_JITTER (prior.py:96-98)
    if (!chol_full<M>(G, L, 0.0)) {
      atomicCAS(&status[b], GVP_OK, GVP_ERR_NOT_SPD);
      atomicCAS(&where[b], -1, i);
      return;
    }
  }
  for (int q = 0; q < M * M; ++q) grams[(size_t)t * M * M + q] = G[q];
  // Q^-1 = L^-T L^-1, symmetrised (prior.py:152-153)
  double X[M * M];
  for (int c = 0; c < M; ++c) {
    double z[M];
    for (int j = 0; j < M; ++j) {
      double v = (j == c) ? 1.0 : 0.0;
      for (int k = 0; k < j; ++k) v -= L[j * M + k] * z[k];
      z[j] = v / L[j * M + j];
    }
    for (int j = M - 1; j >= 0; --j) {
      double v = z[j];
      for (int k = j + 1; k < M; ++k) v -= L[k * M + j] * X[k * M + c];
      X[j * M + c] = v / L[j * M + j];
    }
  }
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) qinv[(size_t)t * M * M + r * M + c] = 0.5 * (X[r * M + c] + X[c * M + r]);
}

// anchored precision blocks + information (prior.py:140-160 accumulation order)
__global__ void prior_knot_kernel(int nplans, int S, const double* __restrict__ phis, const double* __restrict__ offs,
                                  const double* __restrict__ qinv, const double* __restrict__ x0,
                                  const double* __restrict__ goal, double anchor, double* __restrict__ diag,
                                  double* __restrict__ off, double* __restrict__ info) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = S + 1;
  if (t >= nplans * K) return;
  constexpr int M = NS;
  const int b = t / K, i = t % K;
  double D[M * M] = {0}, e[M] = {0};
  if (i == 0 || i == S) {
    const double* xa = (i == 0 ? x0 : goal) + (size_t)b * M;
    for (int r = 0; r < M; ++r) {
      D[r * M + r] = anchor;
      e[r] = anchor * xa[r];
    }
    if (S == 0 && i == 0) {  // single knot: both anchors
      for (int r = 0; r < M; ++r) {
        D[r * M + r] += anchor;
        e[r] += anchor * goal[(size_t)b * M + r];
      }
    }
  }
  if (i >= 1) {  // step i-1: += Q^-1, info += Q^-1 phi
    const size_t s = (size_t)b * S + (i - 1);
    const double* Qi = qinv + s * M * M;
    const double* ph = offs + s * M;
    for (int q = 0; q < M * M; ++q) D[q] += Qi[q];
    for (int r = 0; r < M; ++r) {
      double v = 0.0;
      for (int k = 0; k < M; ++k) v += Qi[r * M + k] * ph[k];
      e[r] += v;
    }
  }
  if (i < S) {  // step i: += Phi' Q^-1 Phi, off = -Phi' Q^-1, info -= Phi' (Q^-1 phi)
    const size_t s = (size_t)b * S + i;
    const double* Qi = qinv + s * M * M;
    const double* Ph = phis + s * M * M;
    const double* ph = offs + s * M;
    double PtQ[M * M], qf[M];
    for (int r = 0; r < M; ++r)
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
        for (int k = 0; k < M; ++k) v += Ph[k * M + r] * Qi[k * M + c];
        PtQ[r * M + c] = v;
      }
    for (int r = 0; r < M; ++r) {
      double v = 0.0;
      for (int k = 0; k < M; ++k) v += Qi[r * M + k] * ph[k];
      qf[r] = v;
    }
    for (int r = 0; r < M; ++r) {
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
        for (int k = 0; k < M; ++k) v += PtQ[r * M + k] * Ph[k * M + c];
        D[r * M + c] += v;
        off[(s * M + r) * M + c] = -PtQ[r * M + c];
      }
      double v = 0.0;
      for (int k = 0; k < M; ++k) v += Ph[k * M + r] * qf[k];
      e[r] += -v;
    }
  }
  double* Do = diag + (size_t)t * M * M;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < M; ++c) Do[r * M + c] = 0.5 * (D[r * M + c] + D[c * M + r]);
  for (int r = 0; r < M; ++r) info[(size_t)t * M + r] = e[r];
}

}  // namespace slrp
}  // namespace gvp

using namespace gvp;

namespace {
struct DevBuf {
  std::vector<void*> p;
  ~DevBuf() {
    for (void* x : p) cudaFree(x);
  }
  template <class T>
  int get(T** out, size_t count) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) {
      set_error("cudaMalloc failed");
      return GVP_ERR_CUDA;
    }
    p.push_back(q);
    *out = static_cast<T*>(q);
    return GVP_OK;
  }
};
int nblk(int64_t n, int tb) { return (int)((n + tb - 1) / tb); }
int gvp_require_device() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device visible");
    return GVP_ERR_NO_DEVICE;
  }
  return GVP_OK;
}
}  // namespace

// Batched SLR of the planar quadrotor (slr.py:69-92). Host arrays:
// means (B, K, 6), covs (B, K, 6, 6), points (Q, 6), weights (Q), params =
// {1/mass, length/inertia, gravity}; out A (B, K, 6, 6), a (B, K, 6).
extern "C" int gvp_slr_quadrotor(int32_t nplans, int32_t K, const double* means, const double* covs,
                                 const double* points, const double* weights, int32_t Q, double dt,
                                 const double* params, double* A, double* a, int32_t* status, int32_t* where) {
  if (nplans < 1 || K < 1 || Q < 1 || !(dt > 0) || !means || !covs || !points || !weights || !params || !A || !a)
    return GVP_ERR_ARG;
  int r = gvp_require_device();
  if (r) return r;
  constexpr int M = slrp::NS;
  DevBuf d;
  double *dm, *dc, *dp, *dw, *dA, *da;
  int *ds, *dwh;
  const size_t BK = (size_t)nplans * K;
  if ((r = d.get(&dm, BK * M)) || (r = d.get(&dc, BK * M * M)) || (r = d.get(&dp, (size_t)Q * M)) ||
      (r = d.get(&dw, Q)) || (r = d.get(&dA, BK * M * M)) || (r = d.get(&da, BK * M)) || (r = d.get(&ds, nplans)) ||
      (r = d.get(&dwh, nplans)))
    return r;
  GVP_CUDA(cudaMemcpy(dm, means, BK * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dc, covs, BK * M * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dp, points, (size_t)Q * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dw, weights, (size_t)Q * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemset(ds, 0, nplans * sizeof(int)));
  GVP_CUDA(cudaMemset(dwh, 0xff, nplans * sizeof(int)));
  slrp::Quad qp{params[0], params[1], params[2]};
  slrp::slr_kernel<<<nblk(BK, 64), 64>>>(nplans, K, dm, dc, dp, dw, Q, dt, qp, dA, da, ds, dwh);
  GVP_CUDA(cudaGetLastError());
  GVP_CUDA(cudaMemcpy(A, dA, BK * M * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(a, da, BK * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(status, ds, nplans * sizeof(int), cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(where, dwh, nplans * sizeof(int), cudaMemcpyDeviceToHost));
  return GVP_OK;
}

// Batched LTV prior assembly (prior.py:56-170) for n = 6: per plan S steps
// A (S, 6, 6), a (S, 6), B (S, 6, m); Gauss-Legendre nodes/weights on [-1, 1].
// Out: phis (S,6,6), offsets (S,6), grammians (S,6,6), diag (S+1,6,6),
// off (S,6,6), info (S+1,6). The anchored mean is a separate mean solve.
extern "C" int gvp_prior_assemble_reg(int32_t nplans, int32_t S, int32_t n, int32_t m, const double* A,
                                      const double* a, const double* B, double dt, double q_c, double sigma_b,
                                      const double* x0, const double* goal, const double* gl_nodes,
                                      const double* gl_weights, int32_t nodes, double grammian_reg, double* phis,
                                      double* offs, double* grams, double* diag, double* off, double* info,
                                      int32_t* status, int32_t* where) {
  if (!(grammian_reg >= 0.0)) return GVP_ERR_ARG;
  if (nplans < 1 || S < 1 || nodes < 1 || !(dt > 0) || !(q_c > 0) || !(sigma_b > 0)) return GVP_ERR_ARG;
  if (n != slrp::NS || m < 1 || m > 6) {
    set_error("device prior assembly supports n = 6 (planar quadrotor)");
    return GVP_ERR_UNSUPPORTED;
  }
  int r = gvp_require_device();
  if (r) return r;
  constexpr int M = slrp::NS;
  const size_t BS = (size_t)nplans * S, BK = (size_t)nplans * (S + 1);
  DevBuf d;
  double *dA, *da, *dB, *dgs, *dgw, *dterms, *dphi, *doff, *dgram, *dqi, *dx0, *dgoal, *ddiag, *dof, *dinfo;
  int *ds, *dwh;
  if ((r = d.get(&dA, BS * M * M)) || (r = d.get(&da, BS * M)) || (r = d.get(&dB, BS * M * m)) ||
      (r = d.get(&dgs, nodes)) || (r = d.get(&dgw, nodes)) || (r = d.get(&dterms, BS * nodes * M * M)) ||
      (r = d.get(&dphi, BS * M * M)) || (r = d.get(&doff, BS * M)) || (r = d.get(&dgram, BS * M * M)) ||
      (r = d.get(&dqi, BS * M * M)) || (r = d.get(&dx0, (size_t)nplans * M)) ||
      (r = d.get(&dgoal, (size_t)nplans * M)) || (r = d.get(&ddiag, BK * M * M)) || (r = d.get(&dof, BS * M * M)) ||
      (r = d.get(&dinfo, BK * M)) || (r = d.get(&ds, nplans)) || (r = d.get(&dwh, nplans)))
    return r;
  GVP_CUDA(cudaMemcpy(dA, A, BS * M * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(da, a, BS * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dB, B, BS * M * m * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dgs, gl_nodes, nodes * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dgw, gl_weights, nodes * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dx0, x0, (size_t)nplans * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemcpy(dgoal, goal, (size_t)nplans * M * 8, cudaMemcpyHostToDevice));
  GVP_CUDA(cudaMemset(ds, 0, nplans * sizeof(int)));
  GVP_CUDA(cudaMemset(dwh, 0xff, nplans * sizeof(int)));
  slrp::prior_node_kernel<<<nblk(BS * (nodes + 1), 64), 64>>>(nplans, S, n, m, dA, da, dB, dt, q_c, dgs, dgw, nodes,
                                                              dterms, dphi, doff, ds, dwh);
  GVP_CUDA(cudaGetLastError());
  slrp::prior_step_kernel<<<nblk(BS, 64), 64>>>(nplans, S, nodes, dterms, dgram, dqi, ds, dwh, grammian_reg);
  GVP_CUDA(cudaGetLastError());
  const double anchor = 1.0 / (sigma_b * sigma_b);
  slrp::prior_knot_kernel<<<nblk(BK, 64), 64>>>(nplans, S, dphi, doff, dqi, dx0, dgoal, anchor, ddiag, dof, dinfo);
  GVP_CUDA(cudaGetLastError());
  GVP_CUDA(cudaMemcpy(phis, dphi, BS * M * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(offs, doff, BS * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(grams, dgram, BS * M * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(diag, ddiag, BK * M * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(off, dof, BS * M * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(info, dinfo, BK * M * 8, cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(status, ds, nplans * sizeof(int), cudaMemcpyDeviceToHost));
  GVP_CUDA(cudaMemcpy(where, dwh, nplans * sizeof(int), cudaMemcpyDeviceToHost));
  return GVP_OK;
}

extern "C" int gvp_prior_assemble(int32_t nplans, int32_t S, int32_t n, int32_t m, const double* A, const double* a,
                                  const double* B, double dt, double q_c, double sigma_b, const double* x0,
                                  const double* goal, const double* gl_nodes, const double* gl_weights,
                                  int32_t nodes, double* phis, double* offs, double* grams, double* diag,
                                  double* off, double* info, int32_t* status, int32_t* where) {
  return gvp_prior_assemble_reg(nplans, S, n, m, A, a, B, dt, q_c, sigma_b, x0, goal, gl_nodes, gl_weights, nodes,
                                0.0, phis, offs, grams, diag, off, info, status, where);
}
