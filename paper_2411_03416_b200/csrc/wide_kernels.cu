// Block-chain kernels for wide blocks, 9 <= n <= 32 (the 7-DOF arm of
// configuration C3 has n = 14). The n <= 8 kernels keep a whole block per
// thread in registers; at n = 14 a block is 196 doubles, so here one warp
// owns one chain and its 32 lanes own the ROWS of the current blocks
// (registers), with the blocks the other lanes need staged in the warp's
// own shared-memory tiles (odd row stride: row-parallel reads are
// bank-conflict free, column reads are broadcasts). No CTA barriers inside
// a chain: each warp synchronises with __syncwarp only.
//
// The algorithms are the reference's, step for step:
//   gbp_marginals   (gbp.py:43-80)   backward Schur with Cholesky of the
//                                    symmetrised trailing block, forward
//                                    covariance recursion;
//   gbp_mean_solve  (gbp.py:83-106)  block forward elimination, back
//                                    substitution;
//   forward_schur_chols / logdet_block_tridiag (blocktri.py:151-174);
//   select_step_size (optimizer.py:188-231) with proximal_update
//                                    (optimizer.py:129-161) and kl_joint
//                                    (optimizer.py:164-177): every probe is
//                                    the mean solve on one warp and the
//                                    marginals + trace on another; W probe
//                                    slots per CTA evaluate the bisection's
//                                    candidate betas speculatively (the
//                                    shared search logic of step_common.cuh
//                                    replays the reference's sequence).
// Cholesky pivots follow chol_spd (blocktri.py:24-32): not > 0 (or NaN) or a
// square root <= 1e-300 is "not positive definite".
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "gvp_internal.cuh"
#include "step_common.cuh"
#include "wide_block.cuh"

#include <cooperative_groups.h>

namespace gvp {
namespace wide {

// One plan's knot-major dense array (every wide caller passes one plan with
// contiguous n x n blocks / n-vectors): entry e of knot i at p[i * E + e].
// 32-bit index arithmetic and no per-entry stride multiplies; the plan index
// of the strided views is dropped (launchers check the layout).
template <class Ptr>
struct DenseT {
  Ptr p;
  int E;
  GVP_DEV auto& operator()(int64_t, int64_t i, int64_t e) const { return p[(int)i * E + (int)e]; }
};
using DView = DenseT<const double*>;
using DMut = DenseT<double*>;

// Two lanes per block row for the n x n products of the chain steps (NM <= 16:
// lane r + 16 h owns row r, columns [h H, h H + H)): every product takes half
// the issue slots of the lane-per-row form on the warp's otherwise idle lanes.
template <int NM>
struct Half {
  static constexpr bool ON = NM <= 16;
  static constexpr int H = (NM + 1) / 2;
};
// the full row (NM entries) of a value held as halves by lanes r and r + 16
template <int H>
GVP_DEV void halves(const double (&mine)[H], double (&lo)[H], double (&hi)[H]) {
  const bool up = (lane() >> 4) != 0;
#pragma unroll
  for (int cc = 0; cc < H; ++cc) {
    const double o = __shfl_xor_sync(FULL, mine[cc], 16);
    lo[cc] = up ? o : mine[cc];
    hi[cc] = up ? mine[cc] : o;
  }
}

// ------------------------------------------------------------------ chain A
// Forward covariance recursion of gbp_marginals (gbp.py:72-78) from the
// backward sweep's Phi_i^-1 in the global scratch pg: Sigma_ii / Sigma_i,i+1
// out, and tr(Lambda Sigma) against a second chain (trc) when asked.
template <int NM, class Src, class Out, class Tr>
GVP_DEV void chain_cov_forward(const Src& src, int64_t K, int n, const double* pg, WarpWs<NM>& w, const Out& out,
                               const Tr& trc, double& trace) {
  constexpr int LD = Tile<NM>::LD;
  const int r = lane();
  // T holds Sigma_ii
  __syncwarp();
  load_g<NM>(w.T, pg, n);  // Sigma_00 = Phi_0^-1 (exactly symmetric)
  double tr = 0.0;
  for (int64_t i = 0; i < K; ++i) {
    if (r < n) {
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n) {
          const double s = w.T[r * LD + c];
          out.cov(i, r, c, s);
          tr += trc.diag(i, r, c) * w.T[c * LD + r];
        }
    }
    if (i + 1 >= K) break;
    load_g<NM>(w.X, pg + (i + 1) * (int64_t)n * n, n);  // Pn = Phi_{i+1}^-1
    stage<NM>(w.U, n, [&](int a, int b) { return src.off(i, a, b); });
    // G = U Pn -> L tile
    {
      double g[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        double t = 0.0;
        if (c < n && r < n) {
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t += w.U[r * LD + k] * w.X[k * LD + c];
        }
        g[c] = t;
      }
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) w.L[r * LD + c] = g[c];
      __syncwarp();
    }
    // C = Sigma_ii G = -Sigma_{i,i+1} -> Li tile
    {
      double cg[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        double t = 0.0;
        if (c < n && r < n) {
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t += w.T[r * LD + k] * w.L[k * LD + c];
        }
        cg[c] = t;
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) {
          w.Li[r * LD + c] = cg[c];
          out.cross(i, r, c, -cg[c]);
          tr += 2.0 * trc.off(i, r, c) * (-cg[c]);
        }
      __syncwarp();
    }
    // Sigma_{i+1} = Pn + G' C, symmetrised
    {
      double s[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        double t = 0.0;
        if (c < n && r < n) {
          t = w.X[r * LD + c];
          double u = 0.0;
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) u += w.L[k * LD + r] * w.Li[k * LD + c];
          t += u;
        }
        s[c] = t;
      }
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) w.U[r * LD + c] = s[c];
      __syncwarp();
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) w.T[r * LD + c] = 0.5 * (w.U[r * LD + c] + w.U[c * LD + r]);
      __syncwarp();
    }
  }
  trace = warp_sum(tr);
}

// gbp_marginals of the chain whose blocks the source gives (diag(i, r, c),
// off(i, r, c) = block (i, i+1)): backward Schur pivots Phi_i -> Phi_i^-1 in
// the global scratch pg (K x n x n), then the forward covariance recursion.
// Optional: covs/crosses out, tr(Lambda Sigma) against a second chain (tr),
// log det from the backward pivots. Returns the failing knot or -1.
template <int NM, class Src, class Out, class Tr>
GVP_DEV int chain_marginals(const Src& src, int64_t K, int n, double* pg, WarpWs<NM>& w, const Out& out,
                            const Tr& trc, double& trace, double& logdet) {
  constexpr int LD = Tile<NM>::LD;
  const int r = lane();
  double pm = 1.0;
  int pe = 0;
  // ---- backward sweep: X holds Phi_{i+1}^-1
  for (int64_t i = K - 1; i >= 0; --i) {
    stage<NM>(w.T, n, [&](int a, int b) { return src.diag(i, a, b); });
    if (i < K - 1) {
      stage<NM>(w.U, n, [&](int a, int b) { return src.off(i, a, b); });
      // trailing = D - U Phi^-1 U'
      double y[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        double t = 0.0;
        if (c < n && r < n) {
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t += w.U[r * LD + k] * w.X[k * LD + c];
        }
        y[c] = t;
      }
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        if (c < n && r < n) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t += y[k] * w.U[c * LD + k];
          w.T[r * LD + c] -= t;
        }
      }
      __syncwarp();
    }
    if (!chol<NM, true>(w.T, w.L, n, pm, pe)) return (int)i;
    trinv<NM>(w.L, w.Li, n);
    ltl<NM>(w.Li, w.X, n);
    store_g<NM>(pg + i * (int64_t)n * n, w.X, n);
  }
  logdet = 2.0 * (log(pm) + (double)pe * 0.6931471805599453);
  chain_cov_forward<NM>(src, K, n, pg, w, out, trc, trace);
  return -1;
}

// pair barrier of the two chain-A warps of one probe slot (named barrier id)
GVP_DEV void pair_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

// Chain A of a probe in one backward pass on two warps. The Schur warp runs
// the backward GBP Schur of Lambda' (gbp.py:58-70: y = U_i Phi_{i+1}^-1,
// Phi_i = sym(D_i - y U_i'), its Cholesky -> log det, Phi_i^-1 = Li' Li); the
// tangent warp, one knot behind, carries the same recursion's derivative along
// the current precision Lambda (D -> D + t Lambda_ii, U -> U + t Lambda_i,i+1):
//   Phi'_i = Lambda_ii - (Lo_i y' + y Lo_i') + y Phi'_{i+1} y'   (symmetrised)
// and sums tr(Phi_i^-1 Phi'_i) = d/dt log det(Lambda' + t Lambda) = tr(Lambda
// Sigma'), kl_joint's trace term (optimizer.py:164-177), with no forward
// covariance sweep. y_i and Phi_i^-1 pass through a two-slot ring (4 tiles);
// one pair barrier per step. pg (optional): Phi_i^-1 to the global scratch for
// a following chain_cov_forward (write mode). fail: the failing knot or -1.
template <int NM, class Src, class Tr>
GVP_DEV void chain_trace_split(const Src& src, const Tr& trc, int64_t K, int n, bool tangent, WarpWs<NM>& w,
                               double* ring, int bar_id, volatile int* s_fail, double* pg, double& trace,
                               double& logdet, int& fail) {
  constexpr int LD = Tile<NM>::LD, MAT = Tile<NM>::MAT;
  const int r = lane();
  auto ringY = [&](int64_t s) { return ring + ((s & 1) * 2) * MAT; };
  auto ringX = [&](int64_t s) { return ring + ((s & 1) * 2 + 1) * MAT; };
  double pm = 1.0, tr = 0.0;
  int pe = 0;
  if (!tangent && r == 0) *s_fail = -1;
  for (int64_t s = 0; s <= K; ++s) {
    pair_sync(bar_id);  // step s-1 of both warps complete: ring slot s & 1 is free, s_fail current
    if (*s_fail >= 0) break;
    if (!tangent) {
      if (s == K) break;
      const int64_t i = K - 1 - s;
      stage<NM>(w.T, n, [&](int a, int b) { return src.diag(i, a, b); });
      if (i < K - 1) {
        stage<NM>(w.U, n, [&](int a, int b) { return src.off(i, a, b); });
        const double* Xn = ringX(s - 1);  // Phi_{i+1}^-1
        double* Y = ringY(s);
        if constexpr (Half<NM>::ON) {
          constexpr int H = Half<NM>::H;
          const int r2 = lane() & 15, c0 = (lane() >> 4) * H;
          double yh[H], ylo[H], yhi[H];
#pragma unroll
          for (int cc = 0; cc < H; ++cc) {
            const int c = c0 + cc;
            double t = 0.0;
            if (c < n && r2 < n) {
#pragma unroll
              for (int k = 0; k < NM; ++k)
                if (k < n) t += w.U[r2 * LD + k] * Xn[k * LD + c];
              Y[r2 * LD + c] = t;
            }
            yh[cc] = t;
          }
          halves<H>(yh, ylo, yhi);
#pragma unroll
          for (int cc = 0; cc < H; ++cc) {
            const int c = c0 + cc;
            if (c < n && r2 < n) {
              double t = 0.0;
#pragma unroll
              for (int k = 0; k < NM; ++k)
                if (k < n) t += (k < H ? ylo[k] : yhi[k - H]) * w.U[c * LD + k];
              w.T[r2 * LD + c] -= t;
            }
          }
          __syncwarp();
        } else {
        double y[NM];
#pragma unroll
        for (int c = 0; c < NM; ++c) {
          double t = 0.0;
          if (c < n && r < n) {
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) t += w.U[r * LD + k] * Xn[k * LD + c];
          }
          y[c] = t;
        }
#pragma unroll
        for (int c = 0; c < NM; ++c) {
          if (c < n && r < n) {
            Y[r * LD + c] = y[c];
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) t += y[k] * w.U[c * LD + k];
            w.T[r * LD + c] -= t;
          }
        }
        __syncwarp();
        }
      }
      if (!chol<NM, true>(w.T, w.L, n, pm, pe)) {
        if (r == 0) *s_fail = (int)i;
        __syncwarp();
        continue;  // the next pair barrier publishes the failure
      }
      trinv<NM>(w.L, w.Li, n);
      if constexpr (Half<NM>::ON) ltl2<NM>(w.Li, ringX(s), n); else ltl<NM>(w.Li, ringX(s), n);
      if (pg) store_g<NM>(pg + i * (int64_t)n * n, ringX(s), n);
    } else {
      if (s == 0) continue;
      const int64_t j = K - s;  // the knot the Schur warp finished in step s - 1
      const double* Xj = ringX(s - 1);
      const double* Yj = ringY(s - 1);
      stage<NM>(w.T, n, [&](int a, int b) { return trc.diag(j, a, b); });  // Lambda_jj
      if constexpr (Half<NM>::ON) {
        constexpr int H = Half<NM>::H;
        const int r2 = lane() & 15, c0 = (lane() >> 4) * H;
        double ph[H];
        if (j < K - 1) {
          stage<NM>(w.U, n, [&](int a, int b) { return trc.off(j, a, b); });  // Lambda_j,j+1
          double zh[H], zlo[H], zhi[H];
#pragma unroll
          for (int cc = 0; cc < H; ++cc) {
            const int c = c0 + cc;
            double t = 0.0, u = 0.0;
            if (c < n && r2 < n) {
#pragma unroll
              for (int k = 0; k < NM; ++k)
                if (k < n) {
                  t += w.U[r2 * LD + k] * Yj[c * LD + k];
                  u += Yj[r2 * LD + k] * w.X[k * LD + c];
                }
              w.L[r2 * LD + c] = t;
            }
            zh[cc] = u;
          }
          halves<H>(zh, zlo, zhi);
          __syncwarp();
#pragma unroll
          for (int cc = 0; cc < H; ++cc) {
            const int c = c0 + cc;
            double t = 0.0;
            if (c < n && r2 < n) {
#pragma unroll
              for (int k = 0; k < NM; ++k)
                if (k < n) t += (k < H ? zlo[k] : zhi[k - H]) * Yj[c * LD + k];
              t = (w.T[r2 * LD + c] - (w.L[r2 * LD + c] + w.L[c * LD + r2])) + t;
            }
            ph[cc] = t;
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < H; ++cc) ph[cc] = (c0 + cc < n && r2 < n) ? w.T[r2 * LD + c0 + cc] : 0.0;
        }
#pragma unroll
        for (int cc = 0; cc < H; ++cc)
          if (c0 + cc < n && r2 < n) w.Li[r2 * LD + c0 + cc] = ph[cc];
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < H; ++cc) {
          const int c = c0 + cc;
          if (c < n && r2 < n) {
            const double v = 0.5 * (w.Li[r2 * LD + c] + w.Li[c * LD + r2]);
            w.X[r2 * LD + c] = v;
            tr += Xj[r2 * LD + c] * v;
          }
        }
        __syncwarp();
        continue;
      }
      double ph[NM];
      if (j < K - 1) {
        stage<NM>(w.U, n, [&](int a, int b) { return trc.off(j, a, b); });  // Lambda_j,j+1
        // M = Lo Y' -> L tile;  Z = Y Phi'_{j+1} (X tile) -> registers
        double z[NM];
#pragma unroll
        for (int c = 0; c < NM; ++c) {
          double t = 0.0, u = 0.0;
          if (c < n && r < n) {
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) {
                t += w.U[r * LD + k] * Yj[c * LD + k];
                u += Yj[r * LD + k] * w.X[k * LD + c];
              }
          }
          if (c < n && r < n) w.L[r * LD + c] = t;
          z[c] = u;
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < NM; ++c) {
          double t = 0.0;
          if (c < n && r < n) {
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) t += z[k] * Yj[c * LD + k];
            t = (w.T[r * LD + c] - (w.L[r * LD + c] + w.L[c * LD + r])) + t;
          }
          ph[c] = t;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NM; ++c) ph[c] = (c < n && r < n) ? w.T[r * LD + c] : 0.0;
      }
      // Phi'_j symmetrised into the X tile (read above as Phi'_{j+1}: Li tile first)
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) w.Li[r * LD + c] = ph[c];
      __syncwarp();
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) {
          const double v = 0.5 * (w.Li[r * LD + c] + w.Li[c * LD + r]);
          w.X[r * LD + c] = v;
          tr += Xj[r * LD + c] * v;
        }
      __syncwarp();
    }
  }
  fail = *s_fail;
  trace = warp_sum(tr);
  logdet = 2.0 * (log(pm) + (double)pe * 0.6931471805599453);
}

// ------------------------------------------------------------------ chain B
// gbp_mean_solve: forward elimination (pivots Cholesky-checked, the
// reference's "pivot block i"), back substitution. Li_i and z_i = Li_i r_i
// go to the global scratch (lg: K x n x n, zg: K x n). Optional: the result
// (out.mean) and the Mahalanobis term d' Lambda d of d = mu - x against a
// second chain (mh.diag / mh.off / mh.mean). Returns the failing knot or -1.
template <int NM, class Src, class Out, class Mh>
GVP_DEV int chain_mean(const Src& src, int64_t K, int n, double* lg, double* zg, WarpWs<NM>& w, const Out& out,
                       const Mh& mh, double& mahal) {
  constexpr int LD = Tile<NM>::LD;
  const int r = lane();
  double pm = 1.0;
  int pe = 0;
  for (int64_t i = 0; i < K; ++i) {
    stage<NM>(w.T, n, [&](int a, int b) { return src.diag(i, a, b); });
    double rv = r < n ? src.rhs(i, r) : 0.0;
    if (i > 0) {
      stage<NM>(w.U, n, [&](int a, int b) { return src.off(i - 1, a, b); });
      // Z = Li_{i-1} U_{i-1} -> X tile;  trailing -= Z'Z;  r -= Z' z_{i-1}
      if constexpr (Half<NM>::ON) {  // two lanes per row, half the columns each
        constexpr int H = Half<NM>::H;
        const int r2 = lane() & 15, c0 = (lane() >> 4) * H;
#pragma unroll
        for (int cc = 0; cc < H; ++cc) {
          const int c = c0 + cc;
          double t = 0.0;
          if (c < n && r2 < n) {
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n && k <= r2) t += w.Li[r2 * LD + k] * w.U[k * LD + c];
            w.X[r2 * LD + c] = t;
          }
        }
        __syncwarp();
#pragma unroll
        for (int cc = 0; cc < H; ++cc) {
          const int c = c0 + cc;
          if (c < n && r2 < n) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) t += w.X[k * LD + r2] * w.X[k * LD + c];
            w.T[r2 * LD + c] -= t;
          }
        }
        if (r < n) {
          double t2 = 0.0;
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t2 += w.X[k * LD + r] * w.v0[k];
          rv -= t2;
        }
      } else {
        double z[NM];
#pragma unroll
        for (int c = 0; c < NM; ++c) {
          double t = 0.0;
          if (c < n && r < n) {
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n && k <= r) t += w.Li[r * LD + k] * w.U[k * LD + c];
          }
          z[c] = t;
        }
#pragma unroll
        for (int c = 0; c < NM; ++c)
          if (c < n && r < n) w.X[r * LD + c] = z[c];
        __syncwarp();
        if (r < n) {
          double t2 = 0.0;
#pragma unroll
          for (int c = 0; c < NM; ++c)
            if (c < n) {
              double t = 0.0;
#pragma unroll
              for (int k = 0; k < NM; ++k)
                if (k < n) t += w.X[k * LD + r] * w.X[k * LD + c];
              w.T[r * LD + c] -= t;
            }
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n) t2 += w.X[k * LD + r] * w.v0[k];
          rv -= t2;
        }
      }
      __syncwarp();
    }
    if (!chol<NM, true>(w.T, w.L, n, pm, pe)) return (int)i;
    trinv<NM>(w.L, w.Li, n);
    if (r < 32) w.v1[r] = rv;
    __syncwarp();
    double zr = 0.0;
    if (r < n) {
#pragma unroll
      for (int k = 0; k < NM; ++k)
        if (k < n && k <= r) zr += w.Li[r * LD + k] * w.v1[k];
    }
    __syncwarp();
    w.v0[r] = zr;
    if (r < n) zg[i * n + r] = zr;
    store_g<NM>(lg + i * (int64_t)n * n, w.Li, n);
    __syncwarp();
  }
  // ---- back substitution: v2 holds x_{i+1}, v3 holds d_{i+1}
  double mhl = 0.0;
  for (int64_t i = K - 1; i >= 0; --i) {
    load_g<NM>(w.Li, lg + i * (int64_t)n * n, n);
    double wr = r < n ? zg[i * n + r] : 0.0;
    if (i < K - 1) {
      stage<NM>(w.U, n, [&](int a, int b) { return src.off(i, a, b); });
      double q = 0.0;
      if (r < n) {
#pragma unroll
        for (int k = 0; k < NM; ++k)
          if (k < n) q += w.U[r * LD + k] * w.v2[k];
      }
      w.v1[r] = q;
      __syncwarp();
      double t = 0.0;
      if (r < n) {
#pragma unroll
        for (int k = 0; k < NM; ++k)
          if (k < n && k <= r) t += w.Li[r * LD + k] * w.v1[k];
      }
      wr -= t;
      __syncwarp();
    }
    w.v1[r] = wr;
    __syncwarp();
    double x = 0.0;
    if (r < n) {
#pragma unroll
      for (int k = 0; k < NM; ++k)
        if (k < n && k >= r) x += w.Li[k * LD + r] * w.v1[k];
      out.mean(i, r, x);
    }
    const double d = r < n ? mh.mean(i, r) - x : 0.0;
    w.v0[r] = d;
    __syncwarp();
    if (r < n) {
      double t = 0.0, t2 = 0.0;
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n) {
          t += mh.diag(i, r, c) * w.v0[c];
          if (i < K - 1) t2 += mh.off(i, r, c) * w.v3[c];
        }
      mhl += d * t + 2.0 * d * t2;
    }
    __syncwarp();
    w.v2[r] = x;
    w.v3[r] = d;
    __syncwarp();
  }
  mahal = warp_sum(mhl);
  return -1;
}

// NM = 16 / 32: any n up to NM (runtime guards); other NM are exact-size
// instantiations (n = NM at compile time: no guards, constant strides)
template <int NM>
GVP_DEV constexpr int exact_n(int n) {
  return (NM == 16 || NM == 32) ? n : NM;
}

// ------------------------------------------------------------------ sources
struct BtSrc {  // a stored block-tridiagonal matrix (+ rhs)
  DView D, U, E;
  int64_t b;
  int n;
  GVP_DEV double diag(int64_t i, int r, int c) const { return D(b, i, r * n + c); }
  GVP_DEV double off(int64_t i, int r, int c) const { return U(b, i, r * n + c); }
  GVP_DEV double rhs(int64_t i, int r) const { return E(b, i, r); }
};
struct NoOut {
  GVP_DEV void cov(int64_t, int, int, double) const {}
  GVP_DEV void cross(int64_t, int, int, double) const {}
  GVP_DEV void mean(int64_t, int, double) const {}
};
struct BtOut {
  DMut C, X, M;
  int64_t b;
  int n;
  GVP_DEV void cov(int64_t i, int r, int c, double v) const {
    if (C.p) C(b, i, r * n + c) = v;
  }
  GVP_DEV void cross(int64_t i, int r, int c, double v) const {
    if (X.p) X(b, i, r * n + c) = v;
  }
  GVP_DEV void mean(int64_t i, int r, double v) const {
    if (M.p) M(b, i, r) = v;
  }
};
struct NoTr {
  GVP_DEV double diag(int64_t, int, int) const { return 0.0; }
  GVP_DEV double off(int64_t, int, int) const { return 0.0; }
  GVP_DEV double mean(int64_t, int) const { return 0.0; }
};

// ------------------------------------------------------------------ drop-in kernels (one warp per plan)
template <int NM>
__global__ void __launch_bounds__(32) marginals_kernel(int64_t K, int n_in, DView D, DView U, DMut cov, DMut cross,
                                                       double* logdet, double* scratch, int* status, int* where) {
  extern __shared__ __align__(16) double sm[];
  const int n = exact_n<NM>(n_in);
  WarpWs<NM> w(sm);
  const int64_t b = blockIdx.x;
  BtSrc src{D, U, DView{nullptr, 0}, b, n};
  BtOut out{cov, cross, DMut{nullptr, 0}, b, n};
  double tr, ld;
  const int f = chain_marginals<NM>(src, K, n, scratch + b * K * n * n, w, out, NoTr{}, tr, ld);
  if (lane() == 0) {
    status[b] = f < 0 ? GVP_OK : GVP_ERR_NOT_SPD;
    where[b] = f;
    if (logdet && f < 0) logdet[b] = ld;
  }
}

template <int NM>
__global__ void __launch_bounds__(32) mean_solve_kernel(int64_t K, int n_in, DView D, DView U, DView E, DMut x,
                                                        double* scratch, int* status, int* where) {
  extern __shared__ __align__(16) double sm[];
  const int n = exact_n<NM>(n_in);
  WarpWs<NM> w(sm);
  const int64_t b = blockIdx.x;
  BtSrc src{D, U, E, b, n};
  BtOut out{DMut{nullptr, 0}, DMut{nullptr, 0}, x, b, n};
  double mh;
  double* lg = scratch + b * K * (n * n + n);
  const int f = chain_mean<NM>(src, K, n, lg, lg + K * n * n, w, out, NoTr{}, mh);
  if (lane() == 0) {
    status[b] = f < 0 ? GVP_OK : GVP_ERR_NOT_SPD;
    where[b] = f;
  }
}

// forward_schur_chols (blocktri.py:151-165): S_0 = D_0, S_i = D_i - W'W with
// W = L_{i-1}^-1 U_{i-1}; chol_spd without symmetrising (LAPACK reads the
// lower triangle); log det = 2 sum log diag L
template <int NM>
__global__ void __launch_bounds__(32) logdet_kernel(int64_t K, int n_in, DView D, DView U, double* logdet, double* chols,
                                                    int* status, int* where) {
  constexpr int LD = Tile<NM>::LD;
  extern __shared__ __align__(16) double sm[];
  const int n = exact_n<NM>(n_in);
  WarpWs<NM> w(sm);
  const int64_t b = blockIdx.x;
  const int r = lane();
  double pm = 1.0;
  int pe = 0;
  int f = -1;
  for (int64_t i = 0; i < K; ++i) {
    stage<NM>(w.T, n, [&](int a, int c) { return D(b, i, a * n + c); });
    if (i > 0) {
      stage<NM>(w.U, n, [&](int a, int c) { return U(b, i - 1, a * n + c); });
      double z[NM];
#pragma unroll
      for (int c = 0; c < NM; ++c) {
        double t = 0.0;
        if (c < n && r < n) {
#pragma unroll
          for (int k = 0; k < NM; ++k)
            if (k < n && k <= r) t += w.Li[r * LD + k] * w.U[k * LD + c];
        }
        z[c] = t;
      }
#pragma unroll
      for (int c = 0; c < NM; ++c)
        if (c < n && r < n) w.X[r * LD + c] = z[c];
      __syncwarp();
      if (r < n) {
#pragma unroll
        for (int c = 0; c < NM; ++c)
          if (c < n) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < NM; ++k)
              if (k < n) t += w.X[k * LD + r] * w.X[k * LD + c];
            w.T[r * LD + c] -= t;
          }
      }
      __syncwarp();
    }
    if (!chol<NM, false>(w.T, w.L, n, pm, pe)) {
      f = (int)i;
      break;
    }
    if (chols) {
      double* g = chols + (b * K + i) * n * n;
      for (int idx = lane(); idx < n * n; idx += 32) {
        const int a = idx / n, c = idx - a * n;
        g[idx] = c <= a ? w.L[a * LD + c] : 0.0;
      }
    }
    trinv<NM>(w.L, w.Li, n);
  }
  if (lane() == 0) {
    status[b] = f < 0 ? GVP_OK : GVP_ERR_NOT_SPD;
    where[b] = f;
    if (f < 0) logdet[b] = 2.0 * (log(pm) + (double)pe * 0.6931471805599453);
  }
}

// ------------------------------------------------------------------ step (bisection) kernel
struct StepArgs {
  // problem (one plan per CTA; plan-minor views)
  DView mean, diag, off, kdiag, koff, info, gmu, gdiag, goff;
  bool has_goff;
  int n;
  int64_t K;
  // outputs (write mode)
  DMut o_mean, o_diag, o_off, o_cov, o_cross;
  // search state / records (the field names step_common's search expects)
  int B;
  const int* active;
  int* status;
  int* where;
  int* nprobes;
  double* beta;
  double* kl;
  double* ld_next;
  const double* temp;
  const double* ld_cur;
  double kl_bound, beta_min, beta_max;
  double* probe_log;
  int max_probes;
  double* scratch;  // per plan: W slots x (A: K n^2 | B: K n^2 + K n)
  int fixed;        // 1: proximal_update only (beta = beta[b], mean solve + Lambda')
};

// Lambda' and the mean system S of one probe (optimizer.py:151-159)
struct ProbeSrcA {  // Lambda' = ((2 G / T + K / T) + Lambda / beta) * c, diag blocks symmetrised
  const StepArgs* a;
  int64_t b;
  double two_t, inv_t, inv_b, c;
  GVP_DEV double raw(int64_t i, int r, int q) const {
    const int n = a->n;
    return ((a->gdiag(b, i, r * n + q) * two_t + a->kdiag(b, i, r * n + q) * inv_t) + a->diag(b, i, r * n + q) * inv_b) * c;
  }
  GVP_DEV double diag(int64_t i, int r, int q) const { return 0.5 * (raw(i, r, q) + raw(i, q, r)); }
  GVP_DEV double off(int64_t i, int r, int q) const {
    const int n = a->n;
    const double g = a->has_goff ? a->goff(b, i, r * n + q) : 0.0;
    return ((g * two_t + a->koff(b, i, r * n + q) * inv_t) + a->off(b, i, r * n + q) * inv_b) * c;
  }
};
struct ProbeSrcB {  // S = K / T + Lambda / beta; rhs = (-g / T + eta / T) + (Lambda / beta) mu
  const StepArgs* a;
  int64_t b;
  double temp, inv_t, inv_b;
  GVP_DEV double diag(int64_t i, int r, int q) const {
    const int n = a->n;
    return a->kdiag(b, i, r * n + q) * inv_t + a->diag(b, i, r * n + q) * inv_b;
  }
  GVP_DEV double off(int64_t i, int r, int q) const {
    const int n = a->n;
    return a->koff(b, i, r * n + q) * inv_t + a->off(b, i, r * n + q) * inv_b;
  }
  GVP_DEV double rhs(int64_t i, int r) const {
    const int n = a->n;
    double mv = 0.0;  // blocktri matvec of Lambda * (1/beta): D_i mu_i + U_i mu_{i+1} + U_{i-1}' mu_{i-1}
#pragma unroll 8
    for (int q = 0; q < n; ++q) mv += (a->diag(b, i, r * n + q) * inv_b) * a->mean(b, i, q);
    if (i + 1 < a->K) {
#pragma unroll 8
      for (int q = 0; q < n; ++q) mv += (a->off(b, i, r * n + q) * inv_b) * a->mean(b, i + 1, q);
    }
    if (i > 0) {
#pragma unroll 8
      for (int q = 0; q < n; ++q) mv += (a->off(b, i - 1, q * n + r) * inv_b) * a->mean(b, i - 1, q);
    }
    return ((-a->gmu(b, i, r)) / temp + a->info(b, i, r) / temp) + mv;
  }
};
struct CurTr {  // the current precision Lambda and mean (trace / Mahalanobis terms)
  const StepArgs* a;
  int64_t b;
  GVP_DEV double diag(int64_t i, int r, int c) const { return a->diag(b, i, r * a->n + c); }
  GVP_DEV double off(int64_t i, int r, int c) const { return a->off(b, i, r * a->n + c); }
  GVP_DEV double mean(int64_t i, int r) const { return a->mean(b, i, r); }
};

// G > 1: one plan's search spread over a thread-block cluster of G CTAs (G x W
// probe slots on G SMs); each CTA runs the same search state machine on the
// whole round's results, which every CTA scatters into all the others' shared
// memory (DSMEM) before a cluster barrier. A single wide plan (C3) otherwise
// runs on one SM with W slots per round.
template <int NM, int W, int G>
__global__ void __launch_bounds__(96 * W) step_kernel(const __grid_constant__ StepArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double sm[];
  constexpr int WG = W * G, MAT = Tile<NM>::MAT;
  // three warps per probe slot: 0 chain A Schur, 1 chain B (mean system), 2 chain A tangent
  const int tid = threadIdx.x, warp = tid >> 5, slot = warp / 3, role = warp - 3 * slot;
  const int g = G > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t b = blockIdx.x / G;
  const int n = exact_n<NM>(a.n);
  const int64_t K = a.K;
  WarpWs<NM> w(sm + warp * WarpWs<NM>::DOUBLES);
  double* ring = sm + 3 * W * WarpWs<NM>::DOUBLES + slot * 4 * MAT;  // chain A Schur -> tangent
  double* tail = sm + 3 * W * WarpWs<NM>::DOUBLES + W * 4 * MAT;
  v3::PlanSt* pst = reinterpret_cast<v3::PlanSt*>(tail);  // 10 doubles
  double* r_beta = tail + 16;
  double* r_kl = r_beta + WG;
  int* r_res = reinterpret_cast<int*>(r_kl + WG);
  int* r_fail = r_res + WG;
  int* r_on = r_fail + WG;
  double* xv = reinterpret_cast<double*>(r_on + WG + (WG & 1));  // per local slot: trace, logdet, mahal
  int* xf = reinterpret_cast<int*>(xv + 3 * W);                   // per local slot: fail A, fail B
  int* s_fail = xf + 2 * W;                                       // per local slot: chain A failure (pair)
  const int64_t per_slot = K * n * n * 2 + K * n;
  double* scr = a.scratch + ((b * G + g) * W + slot) * per_slot;
  auto cluster_sync = [&]() {
    if constexpr (G > 1) cg::this_cluster().sync(); else __syncthreads();
  };

  auto run = [&](double beta, bool write) {
    const double temp = a.temp[b];
    const double inv_t = 1.0 / temp, two_t = 2.0 / temp, inv_b = 1.0 / beta, c = beta / (beta + 1.0);
    double tr = 0.0, ld = 0.0, mh = 0.0;
    int f = -1;
    if (role != 1) {
      if (!a.fixed) {
        ProbeSrcA src{&a, b, two_t, inv_t, inv_b, c};
        // one backward pass: log det (Schur warp) and tr(Lambda Sigma') (tangent warp);
        // write mode keeps Phi^-1 for the forward covariance sweep (Schur warp)
        chain_trace_split<NM>(src, CurTr{&a, b}, K, n, role == 2, w, ring, 1 + slot, s_fail + slot,
                              write ? scr : nullptr, tr, ld, f);
        if (write && role == 0 && f < 0) {
          __syncwarp();
          BtOut out{a.o_cov, a.o_cross, DMut{nullptr, 0}, b, n};
          double unused;
          chain_cov_forward<NM>(src, K, n, scr, w, out, NoTr{}, unused);
        }
      }
      if (write && role == 0) {  // Lambda' blocks (symmetrised diagonal, optimizer.py:151-153)
        ProbeSrcA src{&a, b, two_t, inv_t, inv_b, c};
        for (int64_t idx = lane(); idx < K * n * n; idx += 32) {
          const int64_t i = idx / (n * n);
          const int e = (int)(idx - i * n * n), r = e / n, q = e - r * n;
          a.o_diag(b, i, e) = src.diag(i, r, q);
          if (i + 1 < K) a.o_off(b, i, e) = src.off(i, r, q);
        }
      }
    } else {
      ProbeSrcB src{&a, b, temp, inv_t, inv_b};
      BtOut out{DMut{nullptr, 0}, DMut{nullptr, 0}, write ? a.o_mean : DMut{nullptr, 0},
                b, n};
      f = chain_mean<NM>(src, K, n, scr + K * n * n, scr + 2 * K * n * n, w, out, CurTr{&a, b}, mh);
    }
    if (lane() == 0) {
      if (role == 0) {
        xv[slot * 3 + 1] = ld;
        xf[slot * 2 + 0] = f;
      } else if (role == 2) {
        xv[slot * 3 + 0] = tr;
      } else {
        xv[slot * 3 + 2] = mh;
        xf[slot * 2 + 1] = f;
      }
    }
  };

  if (a.fixed) {  // proximal_update: slot 0 of the cluster's first CTA only
    if (slot == 0 && g == 0) run(a.beta[b], true);
    __syncthreads();
    if (tid == 0 && g == 0) {
      const int fB = xf[1];
      a.status[b] = fB < 0 ? GVP_OK : GVP_ERR_NOT_SPD;
      a.where[b] = fB;
    }
    return;
  }

  v3::search_init(a, pst, 1, b, false, tid);
  __syncthreads();
  for (;;) {
    const v3::Pick pk = v3::search_pick(a, pst, 1, WG, g * W + slot, tid, false);
    if (pk.kl == 0) break;
    __syncthreads();
    if (pk.on) run(pk.beta, false);
    __syncthreads();
    if (tid < W) {
      const int s = tid, gs = g * W + s;
      const v3::Pick ps = v3::search_pick(a, pst, 1, WG, gs, -1, false);
      const int fA = xf[s * 2], fB = xf[s * 2 + 1];
      const int rr = fB >= 0 ? 2 : (fA >= 0 ? 1 : 0);
      double klv = 0.0;
      if (ps.on && rr == 0) {
        const double x = 0.5 * ((((xv[s * 3] + xv[s * 3 + 2]) - (double)(K * n)) + xv[s * 3 + 1]) - a.ld_cur[b]);
        klv = (0.0 > x) ? 0.0 : x;  // python max(x, 0.0): NaN stays NaN
      }
      for (int dst = 0; dst < G; ++dst) {  // every CTA of the cluster gets the whole round
        double *rb = r_beta, *rk = r_kl;
        int *rs = r_res, *rf = r_fail, *ro = r_on;
        if constexpr (G > 1) {
          cg::cluster_group cl = cg::this_cluster();
          rb = cl.map_shared_rank(r_beta, dst);
          rk = cl.map_shared_rank(r_kl, dst);
          rs = cl.map_shared_rank(r_res, dst);
          rf = cl.map_shared_rank(r_fail, dst);
          ro = cl.map_shared_rank(r_on, dst);
        }
        rb[gs] = ps.beta;
        rk[gs] = klv;
        rs[gs] = rr;
        rf[gs] = fB >= 0 ? fB : fA;
        ro[gs] = ps.on ? 1 : 0;
      }
    }
    cluster_sync();
    if (tid == 0) v3::search_decide(a, pst, 0, pk.dbase, pk.dkl, b, false, r_beta, r_kl, r_res, r_fail, r_on);
    cluster_sync();  // nobody scatters the next round into a CTA still deciding this one
  }
  // commit (the cluster's first CTA): the accepted beta re-probed in write mode
  // (deterministic: the same numbers as its probe), KL and log det of the accepted state
  const bool ok = (b < a.B) && (!a.active || a.active[b]) && a.status[b] == GVP_OK && g == 0;
  if (ok && slot == 0) run(a.beta[b], true);
  __syncthreads();
  if (ok && tid == 0) {
    const int fA = xf[0], fB = xf[1];
    if (fA >= 0 || fB >= 0) {
      a.status[b] = GVP_ERR_NOT_SPD;
      a.where[b] = fB >= 0 ? (fB | GVP_WHERE_MEAN_SOLVE_BIAS) : fA;
    } else {
      const double x = 0.5 * ((((xv[0] + xv[2]) - (double)(K * n)) + xv[1]) - a.ld_cur[b]);
      a.kl[b] = (0.0 > x) ? 0.0 : x;
      if (a.ld_next) a.ld_next[b] = xv[1];
    }
  }
}

// probe slots per CTA (3 warps each), bounded by the shared workspace
template <int NM>
constexpr int slots() {
  return NM <= 16 ? 4 : 1;
}

}  // namespace wide

// ---------------------------------------------------------------------- host
// probe slots of one plan spread over a cluster of kWideCluster CTAs while the
// batch is small (n <= 16); a large batch fills the GPU with one CTA per plan
constexpr int kWideCluster = 4;
static int wide_cluster(int nplans, int n) { return (n <= 16 && nplans <= 148 / kWideCluster) ? kWideCluster : 1; }

int64_t wide_scratch_doubles(int nplans, int64_t K, int n) {
  const int W = n <= 16 ? wide::slots<16>() : wide::slots<32>();
  return (int64_t)nplans * W * wide_cluster(nplans, n) * (K * n * n * 2 + K * n);
}

template <class F>
static int wide_dispatch(int n, F f) {
  if (n == 14) return f(std::integral_constant<int, 14>{});  // the 7-DOF arm (q, q_dot)
  if (n >= 9 && n <= 16) return f(std::integral_constant<int, 16>{});
  if (n >= 17 && n <= 32) return f(std::integral_constant<int, 32>{});
  set_error("wide block kernels support 9 <= n <= 32");
  return GVP_ERR_UNSUPPORTED;
}

// the wide kernels read one plan's dense blocks (wide::DenseT): strided views
// must be that layout (one plan, entry stride 1, knot stride = entries)
static bool dense_ok(int nplans, const double* p, int64_t sk, int64_t se, int64_t E) {
  return nplans == 1 && (p == nullptr || (se == 1 && sk == E));
}
static wide::DView dv(const View& v, int64_t E) { return wide::DView{v.p, (int)E}; }
static wide::DMut dm(const MutView& v, int64_t E) { return wide::DMut{v.p, (int)E}; }
#define GVP_WIDE_DENSE(nplans, v, E)                                                  \
  if (!dense_ok(nplans, (v).p, (v).sk, (v).se, (E))) {                                \
    set_error("wide block kernels take one plan's contiguous blocks (" #v ")");      \
    return GVP_ERR_ARG;                                                               \
  }

int launch_wide_marginals(int nplans, int64_t K, int n, const View& D, const View& U, const MutView& cov,
                          const MutView& cross, double* logdet, double* scratch, int* status, int* where,
                          cudaStream_t s) {
  return wide_dispatch(n, [&](auto tag) -> int {
    constexpr int NM = decltype(tag)::value;
    const size_t bytes = wide::WarpWs<NM>::DOUBLES * 8;
    GVP_CUDA(cudaFuncSetAttribute(wide::marginals_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    const int64_t N2 = (int64_t)n * n;
    GVP_WIDE_DENSE(nplans, D, N2) GVP_WIDE_DENSE(nplans, U, N2) GVP_WIDE_DENSE(nplans, cov, N2)
    GVP_WIDE_DENSE(nplans, cross, N2)
    wide::marginals_kernel<NM><<<nplans, 32, bytes, s>>>(K, n, dv(D, N2), dv(U, N2), dm(cov, N2), dm(cross, N2),
                                                         logdet, scratch, status, where);
    GVP_CUDA(cudaGetLastError());
    return GVP_OK;
  });
}

int launch_wide_mean_solve(int nplans, int64_t K, int n, const View& D, const View& U, const View& E,
                           const MutView& x, double* scratch, int* status, int* where, cudaStream_t s) {
  return wide_dispatch(n, [&](auto tag) -> int {
    constexpr int NM = decltype(tag)::value;
    const size_t bytes = wide::WarpWs<NM>::DOUBLES * 8;
    GVP_CUDA(cudaFuncSetAttribute(wide::mean_solve_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    const int64_t N2 = (int64_t)n * n;
    GVP_WIDE_DENSE(nplans, D, N2) GVP_WIDE_DENSE(nplans, U, N2) GVP_WIDE_DENSE(nplans, E, n)
    GVP_WIDE_DENSE(nplans, x, n)
    wide::mean_solve_kernel<NM><<<nplans, 32, bytes, s>>>(K, n, dv(D, N2), dv(U, N2), dv(E, n), dm(x, n), scratch,
                                                          status, where);
    GVP_CUDA(cudaGetLastError());
    return GVP_OK;
  });
}

int launch_wide_logdet(int nplans, int64_t K, int n, const View& D, const View& U, double* logdet, double* chols,
                       int* status, int* where, cudaStream_t s) {
  return wide_dispatch(n, [&](auto tag) -> int {
    constexpr int NM = decltype(tag)::value;
    const size_t bytes = wide::WarpWs<NM>::DOUBLES * 8;
    GVP_CUDA(cudaFuncSetAttribute(wide::logdet_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    const int64_t N2 = (int64_t)n * n;
    GVP_WIDE_DENSE(nplans, D, N2) GVP_WIDE_DENSE(nplans, U, N2)
    wide::logdet_kernel<NM><<<nplans, 32, bytes, s>>>(K, n, dv(D, N2), dv(U, N2), logdet, chols, status, where);
    GVP_CUDA(cudaGetLastError());
    return GVP_OK;
  });
}

int launch_wide_step(const WideStep& q, cudaStream_t s) {
  wide::StepArgs a;
  std::memset(&a, 0, sizeof(a));
  const int64_t N2 = (int64_t)q.n * q.n, nv = q.n;
  GVP_WIDE_DENSE(q.nplans, q.mean, nv) GVP_WIDE_DENSE(q.nplans, q.diag, N2) GVP_WIDE_DENSE(q.nplans, q.off, N2)
  GVP_WIDE_DENSE(q.nplans, q.kdiag, N2) GVP_WIDE_DENSE(q.nplans, q.koff, N2) GVP_WIDE_DENSE(q.nplans, q.info, nv)
  GVP_WIDE_DENSE(q.nplans, q.gmu, nv) GVP_WIDE_DENSE(q.nplans, q.gdiag, N2)
  if (q.has_goff) { GVP_WIDE_DENSE(q.nplans, q.goff, N2) }
  GVP_WIDE_DENSE(q.nplans, q.o_mean, nv) GVP_WIDE_DENSE(q.nplans, q.o_diag, N2) GVP_WIDE_DENSE(q.nplans, q.o_off, N2)
  GVP_WIDE_DENSE(q.nplans, q.o_cov, N2) GVP_WIDE_DENSE(q.nplans, q.o_cross, N2)
  a.mean = dv(q.mean, nv); a.diag = dv(q.diag, N2); a.off = dv(q.off, N2); a.kdiag = dv(q.kdiag, N2);
  a.koff = dv(q.koff, N2); a.info = dv(q.info, nv);
  a.gmu = dv(q.gmu, nv); a.gdiag = dv(q.gdiag, N2); a.goff = dv(q.goff, N2); a.has_goff = q.has_goff;
  a.n = q.n; a.K = q.K;
  a.o_mean = dm(q.o_mean, nv); a.o_diag = dm(q.o_diag, N2); a.o_off = dm(q.o_off, N2); a.o_cov = dm(q.o_cov, N2);
  a.o_cross = dm(q.o_cross, N2);
  a.B = q.nplans; a.active = q.active; a.status = q.status; a.where = q.where; a.nprobes = q.nprobes;
  a.beta = q.beta; a.kl = q.kl; a.ld_next = q.ld_next; a.temp = q.temp; a.ld_cur = q.ld_cur;
  a.kl_bound = q.kl_bound; a.beta_min = q.beta_min; a.beta_max = q.beta_max;
  a.probe_log = q.probe_log; a.max_probes = q.max_probes; a.scratch = q.scratch; a.fixed = q.fixed ? 1 : 0;
  const int G = wide_cluster(q.nplans, q.n);
  return wide_dispatch(q.n, [&](auto tag) -> int {
    constexpr int NM = decltype(tag)::value;
    constexpr int W = wide::slots<NM>();
    auto go = [&](auto gtag) -> int {
      constexpr int GG = decltype(gtag)::value;
      const size_t bytes =
          (3 * W * wide::WarpWs<NM>::DOUBLES + 4 * W * wide::Tile<NM>::MAT + 16 + 4 * W * GG + 6 * W + 8) * 8;
      GVP_CUDA(cudaFuncSetAttribute(wide::step_kernel<NM, W, GG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)bytes));
      if constexpr (GG == 1) {
        wide::step_kernel<NM, W, 1><<<q.nplans, 96 * W, bytes, s>>>(a);
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(q.nplans * GG));
        cfg.blockDim = dim3(96 * W);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = GG;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        GVP_CUDA(cudaLaunchKernelEx(&cfg, wide::step_kernel<NM, W, GG>, a));
      }
      GVP_CUDA(cudaGetLastError());
      return GVP_OK;
    };
    if constexpr (NM <= 16) {
      if (G == kWideCluster) return go(std::integral_constant<int, kWideCluster>{});
    }
    return go(std::integral_constant<int, 1>{});
  });
}

}  // namespace gvp
