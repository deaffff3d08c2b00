// GBP marginals by cyclic reduction (SURVEY.md §8a row a10 / north star (c):
// "the GBP marginal-covariance sweep, parallelised as a cyclic-reduction
// message pass"). The reference's sweep (gbp.py:43-80) is a chain of K
// dependent block steps per plan; for one or a few plans that chain is pure
// latency. Odd-even cyclic reduction computes the same marginal covariances
// Sigma_ii and crosses Sigma_i,i+1 in 2 ceil(log2 K) dependent levels, the
// knots of a level in parallel (one CTA per plan, threads over knots):
//
//   reduction, h = 1, 2, 4, ...: every knot j = h (mod 2h) is eliminated into
//     its neighbours l = j - h, r = j + h of the level:  with P = M_j,
//     V_l = P^-1 A_jl, V_r = P^-1 A_jr:   M_l -= A_lj V_l,  M_r -= A_rj V_r,
//     new coupling A_lr = -A_lj V_r;  knot 0 is left and Sigma_00 = M_0^-1.
//   selected inversion, h = ..., 2, 1 (reverse): for each eliminated j
//     Sigma_jl = -(V_l S_ll + V_r S_rl),  Sigma_jr = -(V_l S_lr + V_r S_rr),
//     Sigma_jj = P^-1 - Sigma_jl V_l' - Sigma_jr V_r'
//   from the already known blocks of its level neighbours (S_lr is the cross
//   of the coarser level, stored at l), leaving Sigma_i,i+1 at the finest level.
// Pivots are Cholesky-factored (SPD check); a failure is re-run through the
// sequential kernel so the error names the reference's knot.
#include <cuda_runtime.h>

#include <algorithm>

#include "gvp_internal.cuh"

namespace gvp {
namespace cr {

// per-plan workspace per knot: M | A (coupling to the next knot of the level) | PINV | VL | VR
template <int N> struct WS {
  static constexpr int N2 = N * N, M = 0, A = N2, PINV = 2 * N2, VL = 3 * N2, VR = 4 * N2, E = 5 * N2;
};

template <int N>
GVP_DEV void ldw(const double* w, double (&a)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) a[r][c] = w[r * N + c];
}
template <int N>
GVP_DEV void stw(double* w, const double (&a)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) w[r * N + c] = a[r][c];
}
// C = A B (TA/TB: use the transpose of A/B)
template <int N, bool TA, bool TB>
GVP_DEV void mm(const double (&A)[N][N], const double (&B)[N][N], double (&C)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) t += (TA ? A[k][r] : A[r][k]) * (TB ? B[c][k] : B[k][c]);
      C[r][c] = t;
    }
}

template <int N>
__global__ void __launch_bounds__(256) cr_marginals_kernel(int64_t K, View D, View U, MutView cov, MutView cross,
                                                           double* __restrict__ ws_all, int* status, int* where) {
  using W = WS<N>;
  const int64_t b = blockIdx.x;
  double* ws = ws_all + b * K * W::E;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = -1;
  for (int64_t i = threadIdx.x; i < K; i += blockDim.x) {
    double a[N][N];
    load_blk<N>(D, b, i, a);
    stw<N>(ws + i * W::E + W::M, a);
    if (i + 1 < K) {
      load_blk<N>(U, b, i, a);
      stw<N>(ws + i * W::E + W::A, a);
    }
  }
  __syncthreads();
  int64_t h = 1;
  for (; h < K; h *= 2) {
    // ---- eliminate j = h (mod 2h)
    for (int64_t j = h + 2 * h * threadIdx.x; j < K; j += 2 * h * blockDim.x) {
      double P[N][N], L[N][N], Li[N][N], Pi[N][N], Ajl[N][N], X[N][N];
      ldw<N>(ws + j * W::E + W::M, P);
      if (!chol<N>(P, L)) {
        atomicCAS(&fail, -1, (int)j);
        continue;
      }
      tri_inv<N>(L, Li);
      mm<N, true, false>(Li, Li, Pi);  // P^-1 = Li' Li
      stw<N>(ws + j * W::E + W::PINV, Pi);
      ldw<N>(ws + (j - h) * W::E + W::A, X);  // A_lj (block (l, j))
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) Ajl[r][c] = X[c][r];
      mm<N, false, false>(Pi, Ajl, X);  // V_l = P^-1 A_jl
      stw<N>(ws + j * W::E + W::VL, X);
      if (j + h < K) {
        ldw<N>(ws + j * W::E + W::A, Ajl);  // A_jr
        mm<N, false, false>(Pi, Ajl, X);    // V_r = P^-1 A_jr
      } else {
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c) X[r][c] = 0.0;
      }
      stw<N>(ws + j * W::E + W::VR, X);
    }
    __syncthreads();
    if (fail >= 0) break;
    // ---- update the surviving knots i = 0 (mod 2h)
    for (int64_t i = 2 * h * threadIdx.x; i < K; i += 2 * h * blockDim.x) {
      double M[N][N], T1[N][N], T2[N][N];
      ldw<N>(ws + i * W::E + W::M, M);
      if (i + h < K) {  // right neighbour j2 = i + h
        const double* w2 = ws + (i + h) * W::E;
        double A[N][N], V[N][N];
        ldw<N>(ws + i * W::E + W::A, A);  // A_i,j2
        ldw<N>(w2 + W::VL, V);
        mm<N, false, false>(A, V, T1);  // A_ij2 V_l(j2)
        ldw<N>(w2 + W::VR, V);
        mm<N, false, false>(A, V, T2);  // A_ij2 V_r(j2): new coupling to i + 2h is -T2
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c) {
            M[r][c] -= T1[r][c];
            T2[r][c] = (i + 2 * h < K) ? -T2[r][c] : 0.0;
          }
        stw<N>(ws + i * W::E + W::A, T2);
      }
      if (i >= h) {  // left neighbour j1 = i - h: M_i -= A_i,j1 V_r(j1) = A_j1,i' V_r(j1)
        const double* w1 = ws + (i - h) * W::E;
        double A[N][N], V[N][N];
        ldw<N>(w1 + W::A, A);
        ldw<N>(w1 + W::VR, V);
        mm<N, true, false>(A, V, T1);
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int c = 0; c < N; ++c) M[r][c] -= T1[r][c];
      }
      stw<N>(ws + i * W::E + W::M, M);
    }
    __syncthreads();
  }
  if (fail < 0 && threadIdx.x == 0) {  // the last surviving knot: Sigma_00 = M_0^-1
    double M[N][N], L[N][N], Li[N][N], S[N][N];
    ldw<N>(ws + W::M, M);
    if (!chol<N>(M, L)) {
      fail = 0;
    } else {
      tri_inv<N>(L, Li);
      mm<N, true, false>(Li, Li, S);
      store_blk<N>(cov, b, 0, S);
    }
  }
  __syncthreads();
  if (fail >= 0) {
    if (threadIdx.x == 0) {
      status[b] = GVP_ERR_NOT_SPD;
      where[b] = fail;
    }
    return;
  }
  // ---- selected inversion, coarse to fine
  for (h /= 2; h >= 1; h /= 2) {
    for (int64_t j = h + 2 * h * threadIdx.x; j < K; j += 2 * h * blockDim.x) {
      const int64_t l = j - h, r = j + h;
      const bool hr = r < K;
      double VL[N][N], VR[N][N], Sll[N][N], Slr[N][N], Srr[N][N], A[N][N], Bm[N][N], T[N][N];
      ldw<N>(ws + j * W::E + W::VL, VL);
      ldw<N>(ws + j * W::E + W::VR, VR);
      load_blk<N>(View{cov.p, cov.sk, cov.se, cov.sp}, b, l, Sll);
      if (hr) {
        load_blk<N>(View{cross.p, cross.sk, cross.se, cross.sp}, b, l, Slr);  // Sigma_l,r (coarser level)
        load_blk<N>(View{cov.p, cov.sk, cov.se, cov.sp}, b, r, Srr);
      }
      mm<N, false, false>(VL, Sll, A);
      if (hr) {
        mm<N, false, true>(VR, Slr, T);  // V_r S_rl = V_r S_lr'
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int c = 0; c < N; ++c) A[a][c] += T[a][c];
        mm<N, false, false>(VL, Slr, Bm);
        mm<N, false, false>(VR, Srr, T);
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int c = 0; c < N; ++c) Bm[a][c] += T[a][c];
      }
      // Sigma_jj = P^-1 + A V_l' + B V_r'   (Sigma_jl = -A, Sigma_jr = -B)
      double S[N][N];
      ldw<N>(ws + j * W::E + W::PINV, S);
      mm<N, false, true>(A, VL, T);
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int c = 0; c < N; ++c) S[a][c] += T[a][c];
      if (hr) {
        mm<N, false, true>(Bm, VR, T);
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int c = 0; c < N; ++c) S[a][c] += T[a][c];
      }
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int c = 0; c < a; ++c) {
          const double v = 0.5 * (S[a][c] + S[c][a]);
          S[a][c] = v;
          S[c][a] = v;
        }
      store_blk<N>(cov, b, j, S);
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int c = 0; c < N; ++c) T[a][c] = -A[c][a];  // Sigma_l,j = Sigma_j,l'
      store_blk<N>(cross, b, l, T);
      if (hr) {
#pragma unroll
        for (int a = 0; a < N; ++a)
#pragma unroll
          for (int c = 0; c < N; ++c) T[a][c] = -Bm[a][c];
        store_blk<N>(cross, b, j, T);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    status[b] = GVP_OK;
    where[b] = -1;
  }
}

}  // namespace cr

int64_t cr_workspace_doubles(int nplans, int64_t K, int n) { return (int64_t)nplans * K * 5 * n * n; }

int launch_cr_marginals(int nplans, int64_t K, int n, const View& D, const View& U, const MutView& cov,
                        const MutView& cross, double* ws, int* status, int* where, cudaStream_t s) {
  if (nplans == 0 || K == 0) return GVP_OK;
  const int tb = (int)std::min<int64_t>(256, std::max<int64_t>(32, ((K / 2 + 31) / 32) * 32));
#define GVP_CR(NN) \
  case NN: cr::cr_marginals_kernel<NN><<<nplans, tb, 0, s>>>(K, D, U, cov, cross, ws, status, where); break;
  switch (n) {
    GVP_CR(1) GVP_CR(2) GVP_CR(3) GVP_CR(4) GVP_CR(5) GVP_CR(6) GVP_CR(7) GVP_CR(8)
    default:
      set_error("cyclic-reduction marginals support n <= 8");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_CR
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp
