// Small dense fp64 block algebra for the chain kernels (register-resident,
// fully unrolled for a compile-time block size N <= 8).
//
// Conventions follow the reference's numerics:
//  * SPD predicate of blocktri.py:24-32 — a Cholesky pivot that is not > 0
//    (LAPACK dpotrf failure, incl. NaN) or whose square root is <= 1e-300
//    means "not positive definite".
//  * Only the lower triangle of the input is read by chol(), like LAPACK
//    uplo='L' as used by numpy.linalg.cholesky.
#pragma once
#include <cstdint>

#define GVP_DEV __device__ __forceinline__

namespace gvp {

constexpr double kPivotFloor = 1e-300;  // blocktri.py:17

// Branch-free pieces of the per-knot Cholesky: the library's double rsqrt and
// frexp carry special-value slow paths (a CALL under a convergence barrier in
// the hot loop); pivots here are positive normal numbers (anything else already
// fails the SPD test, whose value is then irrelevant), so: the hardware
// approximation + two Newton steps (~1 ulp), and exponent extraction from the bits.
GVP_DEV double rsqrt_nb(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
GVP_DEV double frexp_pos(double x, int* e) {  // x > 0 normal: x = m 2^e, m in [0.5, 1)
  const long long bits = __double_as_longlong(x);
  *e = (int)((bits >> 52) & 0x7ff) - 1022;
  return __longlong_as_double((bits & ~(0x7ffLL << 52)) | (1022LL << 52));
}

// ---------------------------------------------------------------- strided views
// element (plan b, knot i, entry e) lives at p[i*sk + e*se + b*sp].
// Plan-minor ("interleaved") batches use sp=1, se=B, sk=E*B; a view shared by
// every plan (e.g. one prior precision for a whole batch) uses sp=0.
// Plain (coherent) loads: engine state is updated in place by the same kernel
// that reads it, so views must not use the non-coherent __ldg path.
struct View {
  const double* p;
  int64_t sk, se, sp;
  GVP_DEV double operator()(int64_t b, int64_t i, int64_t e) const {
    return p[i * sk + e * se + b * sp];
  }
};
struct MutView {
  double* p;
  int64_t sk, se, sp;
  GVP_DEV double& operator()(int64_t b, int64_t i, int64_t e) const {
    return p[i * sk + e * se + b * sp];
  }
};

template <int N>
GVP_DEV void load_blk(const View& v, int64_t b, int64_t i, double (&a)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) a[r][c] = v(b, i, r * N + c);
}
template <int N>
GVP_DEV void store_blk(const MutView& v, int64_t b, int64_t i, const double (&a)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) v(b, i, r * N + c) = a[r][c];
}
template <int N>
GVP_DEV void load_vec(const View& v, int64_t b, int64_t i, double (&x)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) x[r] = v(b, i, r);
}
template <int N>
GVP_DEV void store_vec(const MutView& v, int64_t b, int64_t i, const double (&x)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) v(b, i, r) = x[r];
}

// packed lower triangle: entry (r, c), c <= r, at r*(r+1)/2 + c
template <int N> struct Tri { static constexpr int kLen = N * (N + 1) / 2; };
GVP_DEV constexpr int tri_idx(int r, int c) { return r * (r + 1) / 2 + c; }

// ---------------------------------------------------------------- factorisations
// Lower Cholesky of the lower triangle of a; returns false on a non-SPD pivot
// (blocktri.py:24-32). L's strict upper triangle is zeroed.
template <int N, bool FLOOR = true>
GVP_DEV bool chol(const double (&a)[N][N], double (&L)[N][N]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int c = j + 1; c < N; ++c) L[j][c] = 0.0;
    double s = a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
    ok = ok && (s > 0.0);
    const double d = sqrt(s);
    if (FLOOR) ok = ok && (d > kPivotFloor);
    L[j][j] = d;
    const double inv = 1.0 / d;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double t = a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
      L[i][j] = t * inv;
    }
  }
  return ok;
}

// Multiplication-only variant for the fused kernels: one rsqrt per pivot,
// inv[j] = 1 / L[j][j]; same SPD predicate.
template <int N, bool FLOOR = true>
GVP_DEV bool chol_fast(const double (&a)[N][N], double (&L)[N][N], double (&inv)[N]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < N; ++j) {
#pragma unroll
    for (int c = j + 1; c < N; ++c) L[j][c] = 0.0;
    double s = a[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
    ok = ok && (s > 0.0);
    const double r = rsqrt(s);
    const double d = s * r;
    if (FLOOR) ok = ok && (d > kPivotFloor);
    L[j][j] = d;
    inv[j] = r;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double t = a[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
      L[i][j] = t * r;
    }
  }
  return ok;
}
template <int N>
GVP_DEV void tri_inv_fast(const double (&L)[N][N], const double (&inv)[N], double (&Li)[N][N]) {
#pragma unroll
  for (int c = 0; c < N; ++c) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (r < c) {
        Li[r][c] = 0.0;
      } else if (r == c) {
        Li[r][c] = inv[r];
      } else {
        double t = 0.0;
#pragma unroll
        for (int k = c; k < r; ++k) t += L[r][k] * Li[k][c];
        Li[r][c] = -t * inv[r];
      }
    }
  }
}

// X <- L^{-1} X  (L lower), X has M columns
template <int N, int M>
GVP_DEV void trsm_lower(const double (&L)[N][N], double (&X)[N][M]) {
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double t = X[r][c];
#pragma unroll
      for (int k = 0; k < r; ++k) t -= L[r][k] * X[k][c];
      X[r][c] = t / L[r][r];
    }
  }
}
// X <- L^{-T} X
template <int N, int M>
GVP_DEV void trsm_lower_t(const double (&L)[N][N], double (&X)[N][M]) {
#pragma unroll
  for (int c = 0; c < M; ++c) {
#pragma unroll
    for (int r = N - 1; r >= 0; --r) {
      double t = X[r][c];
#pragma unroll
      for (int k = r + 1; k < N; ++k) t -= L[k][r] * X[k][c];
      X[r][c] = t / L[r][r];
    }
  }
}
template <int N>
GVP_DEV void trsv_lower(const double (&L)[N][N], double (&x)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double t = x[r];
#pragma unroll
    for (int k = 0; k < r; ++k) t -= L[r][k] * x[k];
    x[r] = t / L[r][r];
  }
}
template <int N>
GVP_DEV void trsv_lower_t(const double (&L)[N][N], double (&x)[N]) {
#pragma unroll
  for (int r = N - 1; r >= 0; --r) {
    double t = x[r];
#pragma unroll
    for (int k = r + 1; k < N; ++k) t -= L[k][r] * x[k];
    x[r] = t / L[r][r];
  }
}

// inverse of a lower-triangular L (result lower-triangular)
template <int N>
GVP_DEV void tri_inv(const double (&L)[N][N], double (&Li)[N][N]) {
#pragma unroll
  for (int c = 0; c < N; ++c) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      if (r < c) {
        Li[r][c] = 0.0;
      } else {
        double t = (r == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = c; k < r; ++k) t -= L[r][k] * Li[k][c];
        Li[r][c] = t / L[r][r];
      }
    }
  }
}

// (L L^T)^{-1} = L^{-T} L^{-1} from the triangular inverse, exactly symmetric
template <int N>
GVP_DEV void spd_inv_from_chol(const double (&L)[N][N], double (&P)[N][N]) {
  double Li[N][N];
  tri_inv<N>(L, Li);
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = r; k < N; ++k) t += Li[k][r] * Li[k][c];
      P[r][c] = t;
      P[c][r] = t;
    }
}

template <int N>
GVP_DEV double logdet_from_chol(const double (&L)[N][N]) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) s += log(L[j][j]);
  return 2.0 * s;
}

// ---------------------------------------------------------------- products
template <int N>
GVP_DEV void matmul(const double (&A)[N][N], const double (&B)[N][N], double (&C)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) t += A[r][k] * B[k][c];
      C[r][c] = t;
    }
}
// C = A^T B
template <int N>
GVP_DEV void matmul_tn(const double (&A)[N][N], const double (&B)[N][N], double (&C)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) t += A[k][r] * B[k][c];
      C[r][c] = t;
    }
}
// C = W^T W (symmetric, lower computed and mirrored)
template <int N>
GVP_DEV void gram_tn(const double (&W)[N][N], double (&C)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) t += W[k][r] * W[k][c];
      C[r][c] = t;
      C[c][r] = t;
    }
}
template <int N>
GVP_DEV void transpose(const double (&A)[N][N], double (&T)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) T[r][c] = A[c][r];
}
template <int N>
GVP_DEV void symmetrize(double (&A)[N][N]) {  // 0.5 (A + A^T), blocktri.py:43-45
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < r; ++c) {
      const double s = 0.5 * (A[r][c] + A[c][r]);
      A[r][c] = s;
      A[c][r] = s;
    }
}
// y = A x
template <int N>
GVP_DEV void matvec(const double (&A)[N][N], const double (&x)[N], double (&y)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) t += A[r][k] * x[k];
    y[r] = t;
  }
}
// y = A^T x
template <int N>
GVP_DEV void matvec_t(const double (&A)[N][N], const double (&x)[N], double (&y)[N]) {
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) t += A[k][r] * x[k];
    y[r] = t;
  }
}

}  // namespace gvp
