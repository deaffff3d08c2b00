// Warp-level dense fp64 block algebra for wide blocks (9 <= n <= 32): one
// warp per block chain, lane r owns row r (registers), blocks other lanes
// need live in the warp's shared-memory tiles (odd row stride). Used by the
// wide chain kernels (wide_kernels.cu) and the 7-DOF arm factor stage
// (arm_factor.cu). Pivot conventions of gvp_block.cuh.
#pragma once
#include <cuda_runtime.h>

#include "gvp_block.cuh"

namespace gvp {
namespace wide {

constexpr unsigned FULL = 0xffffffffu;
GVP_DEV int lane() { return threadIdx.x & 31; }

template <int NM>
struct Tile {
  static constexpr int LD = NM + 1;   // odd stride
  static constexpr int MAT = NM * LD;  // doubles per tile
};

// per-warp shared workspace: 5 tiles + 4 vectors
template <int NM>
struct WarpWs {
  static constexpr int LD = Tile<NM>::LD, MAT = Tile<NM>::MAT;
  static constexpr int DOUBLES = 5 * MAT + 4 * 32;
  double *T, *L, *Li, *U, *X, *v0, *v1, *v2, *v3;
  GVP_DEV explicit WarpWs(double* base) {
    T = base;
    L = base + MAT;
    Li = base + 2 * MAT;
    U = base + 3 * MAT;
    X = base + 4 * MAT;
    v0 = base + 5 * MAT;
    v1 = v0 + 32;
    v2 = v1 + 32;
    v3 = v2 + 32;
  }
};

// dst[r][c] = f(r, c) for the n x n block, lanes over the flattened entries
template <int NM, class F>
GVP_DEV void stage(double* dst, int n, F f) {
  // all of a lane's loads are issued before its first shared store, so one
  // block costs one global-memory latency, not NM*NM/32 of them
  constexpr int LD = Tile<NM>::LD, IT = (NM * NM + 31) / 32;
  double v[IT];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int idx = lane() + 32 * it;
    const int r = idx / n, c = idx - r * n;
    v[it] = idx < n * n ? f(r, c) : 0.0;
  }
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int idx = lane() + 32 * it;
    const int r = idx / n, c = idx - r * n;
    if (idx < n * n) dst[r * LD + c] = v[it];
  }
  __syncwarp();
}

// Cholesky of the n x n block in tile A (lower triangle of A, or of
// 0.5 (A + A') when SYM — the reference's chol_spd(symmetrize(.))) into tile
// L (row r by lane r). Pivots multiply into (pm, pe) (mantissa, exponent).
template <int NM, bool SYM, bool FLOOR = true>
GVP_DEV bool chol(const double* A, double* L, int n, double& pm, int& pe) {
  constexpr int LD = Tile<NM>::LD;
  const int r = lane();
  double a[NM], l[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) {
    a[j] = 0.0;
    l[j] = 0.0;
    if (j < n && r < n && j <= r) a[j] = SYM ? 0.5 * (A[r * LD + j] + A[j * LD + r]) : A[r * LD + j];
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < NM; ++j) {
    if (j < n) {
      double s = a[j];
#pragma unroll
      for (int k = 0; k < j; ++k) s -= l[k] * L[j * LD + k];
      const double d = __shfl_sync(FULL, s, j);
      // sqrt and the column scale through one reciprocal square root (no IEEE
      // sqrt / division subroutines on the chain); d is warp-uniform, so is the
      // exact fallback for pivots near the subnormal range
      double piv, rp;
      if (d > 1e-280) {
        rp = rsqrt_nb(d);
        piv = d * rp;
      } else {
        piv = sqrt(d);
        rp = 1.0 / piv;
      }
      ok = ok && (d > 0.0) && (!FLOOR || piv > kPivotFloor);
      l[j] = (r == j) ? piv : (r > j ? s * rp : 0.0);
      if (r < n && r >= j) L[r * LD + j] = l[j];
      int e;
      if (d > 1e-280) {
        pm = frexp_pos(pm * piv, &e);  // pm in [0.5, 1), piv > 1e-140: a positive normal product
      } else {
        pm = frexp(pm * piv, &e);
      }
      pe += e;
      __syncwarp();
    }
  }
  return ok;
}

// Li = L^-1 (lower), lane c computes column c by forward substitution; the
// n diagonal reciprocals are formed once, one per lane, and broadcast by
// shuffle (no division on the substitution chain)
template <int NM>
GVP_DEV void trinv(const double* L, double* Li, int n) {
  constexpr int LD = Tile<NM>::LD;
  const int c = lane();
  const double dinv = c < n ? 1.0 / L[c * LD + c] : 0.0;
  double x[NM];
#pragma unroll
  for (int r = 0; r < NM; ++r) {
    x[r] = 0.0;
    if (r < n) {
      double t = (r == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < r; ++k) t -= L[r * LD + k] * x[k];
      const double dr = __shfl_sync(FULL, dinv, r);  // every lane (not under the select)
      x[r] = (r >= c) ? t * dr : 0.0;
      if (c < n) Li[r * LD + c] = x[r];
    }
  }
  __syncwarp();
}

// P = Li' Li (symmetric, exactly: entry (r, c) and (c, r) sum the same
// products in the same order); row r by lane r into tile P
template <int NM>
GVP_DEV void ltl(const double* Li, double* P, int n) {
  constexpr int LD = Tile<NM>::LD;
  const int r = lane();
  double p[NM];
#pragma unroll
  for (int c = 0; c < NM; ++c) {
    double t = 0.0;
    if (c < n && r < n) {
#pragma unroll
      for (int k = 0; k < NM; ++k)
        if (k < n && k >= r && k >= c) t += Li[k * LD + r] * Li[k * LD + c];
    }
    p[c] = t;
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NM; ++c)
    if (c < n && r < n) P[r * LD + c] = p[c];
  __syncwarp();
}

// ltl with two lanes per row (lane r + 16 h: columns [h H, h H + H)), NM <= 16
template <int NM>
GVP_DEV void ltl2(const double* Li, double* P, int n) {
  constexpr int LD = Tile<NM>::LD, H = (NM + 1) / 2;
  const int r = lane() & 15, c0 = (lane() >> 4) * H;
  double p[H];
#pragma unroll
  for (int cc = 0; cc < H; ++cc) {
    const int c = c0 + cc;
    double t = 0.0;
    if (c < n && r < n) {
#pragma unroll
      for (int k = 0; k < NM; ++k)
        if (k < n && k >= r && k >= c) t += Li[k * LD + r] * Li[k * LD + c];
    }
    p[cc] = t;
  }
  __syncwarp();
#pragma unroll
  for (int cc = 0; cc < H; ++cc)
    if (c0 + cc < n && r < n) P[r * LD + c0 + cc] = p[cc];
  __syncwarp();
}

// tile -> global rows (n x n, row-major, stride n)
template <int NM>
GVP_DEV void store_g(double* g, const double* S, int n) {
  constexpr int LD = Tile<NM>::LD;
  for (int idx = lane(); idx < n * n; idx += 32) {
    const int r = idx / n, c = idx - r * n;
    g[idx] = S[r * LD + c];
  }
}
template <int NM>
GVP_DEV void load_g(double* S, const double* g, int n) {
  constexpr int LD = Tile<NM>::LD;
  for (int idx = lane(); idx < n * n; idx += 32) {
    const int r = idx / n, c = idx - r * n;
    S[r * LD + c] = g[idx];
  }
  __syncwarp();
}

GVP_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

}  // namespace wide
}  // namespace gvp
