// Kernel (a) for the 7-DOF sphere arm (configuration C3):
// the reference's factor moments (_kernels.pyx:93-129) with the hinge cost
// summed over spheres attached to the links of a 7-joint arm,
//   psi(q) = sigma * sum_s max(r_s + eps - d(FK_s(q)), 0)^2,   q = x[:7],
// d the trilinear SDF (sdf.py:80-122). The state is (q, q_dot), n = 14.
//
// One warp per factor. psi depends on x[:7] = mu[:7] + L[:7,:7] xi[:7] only, so
// the 421 Smolyak points (k_q = 3, d = 14) collapse to 113 distinct joint-space
// projections: lane j evaluates the forward kinematics (standard DH) and the
// sphere hinge costs of projections j, j+32, ..., the warp then contracts
// psi with the per-projection weight moments (m0, m1 (14), m2 (105)) and maps
// the xi-basis moments back with L: e1 = L E1, e2 = L E2 L^T.
#include <cuda_runtime.h>

#include <vector>

#include "gvp_internal.cuh"
#include "wide_block.cuh"

namespace gvp {
namespace arm {

constexpr int NQ = 7, NX = 14, TX = NX * (NX + 1) / 2, NM = 1 + NX + TX;  // moments per projection
constexpr int kMaxSpheres = 64, kMaxProj = 256;

struct ArmConst {
  double dh[NQ][4];  // a, d, alpha, theta offset
  double base[3];
  int nsph;
  int link[kMaxSpheres];
  double geom[kMaxSpheres][4];  // local x, y, z, radius
};

// trilinear SDF with the reference's border clamp and OOB flag (x-pair packed rows)
GVP_DEV double sdf3(const FieldDev& F, double px, double py, double pz, bool& out) {
  double u = (px - F.ox) * F.inv_cell, v = (py - F.oy) * F.inv_cell, w = (pz - F.oz) * F.inv_cell;
  const double tx = (double)(F.nx - 1), ty = (double)(F.ny - 1), tz = (double)(F.nz - 1);
  out = (u < 0.0) | (u > tx) | (v < 0.0) | (v > ty) | (w < 0.0) | (w > tz);
  u = fmin(fmax(u, 0.0), tx);
  v = fmin(fmax(v, 0.0), ty);
  w = fmin(fmax(w, 0.0), tz);
  const int64_t ix = (int64_t)fmin(floor(u), tx - 1.0), iy = (int64_t)fmin(floor(v), ty - 1.0),
                iz = (int64_t)fmin(floor(w), tz - 1.0);
  const double fx = u - (double)ix, fy = v - (double)iy, fz = w - (double)iz;
  const int64_t cx = F.nx - 1;
  auto row = [&](int64_t z, int64_t y) {
    const double2 c = *reinterpret_cast<const double2*>(F.corners + ((z * F.ny + y) * cx + ix) * 2);
    return c.x * (1.0 - fx) + c.y * fx;
  };
  const double p0 = row(iz, iy) * (1.0 - fy) + row(iz, iy + 1) * fy;
  const double p1 = row(iz + 1, iy) * (1.0 - fy) + row(iz + 1, iy + 1) * fy;
  return p0 * (1.0 - fz) + p1 * fz;
}

// psi(q) and the count of out-of-bounds sphere centres
GVP_DEV double arm_psi(const ArmConst& A, const FieldDev& F, const double (&q)[NQ], double re, double so,
                       int& oob) {
  // frames 0..7 as 3x4 [R | t]
  double fr[NQ + 1][12];
#pragma unroll
  for (int k = 0; k < 12; ++k) fr[0][k] = 0.0;
  fr[0][0] = fr[0][5] = fr[0][10] = 1.0;
  fr[0][3] = A.base[0];
  fr[0][7] = A.base[1];
  fr[0][11] = A.base[2];
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    double st, ct, sa, ca;
    sincos(q[j] + A.dh[j][3], &st, &ct);
    sincos(A.dh[j][2], &sa, &ca);
    const double a = A.dh[j][0], d = A.dh[j][1];
    // standard DH: [[ct, -st ca, st sa, a ct], [st, ct ca, -ct sa, a st], [0, sa, ca, d]]
    const double M[12] = {ct, -st * ca, st * sa, a * ct, st, ct * ca, -ct * sa, a * st, 0.0, sa, ca, d};
    const double* P = fr[j];
    double* O = fr[j + 1];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        O[r * 4 + c] = P[r * 4 + 0] * M[0 * 4 + c] + P[r * 4 + 1] * M[1 * 4 + c] + P[r * 4 + 2] * M[2 * 4 + c];
      O[r * 4 + 3] = P[r * 4 + 0] * M[3] + P[r * 4 + 1] * M[7] + P[r * 4 + 2] * M[11] + P[r * 4 + 3];
    }
  }
  double psi = 0.0;
  for (int s = 0; s < A.nsph; ++s) {
    const double* T = fr[A.link[s]];
    const double* g = A.geom[s];
    double c3[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) c3[r] = T[r * 4 + 0] * g[0] + T[r * 4 + 1] * g[1] + T[r * 4 + 2] * g[2] + T[r * 4 + 3];
    bool o;
    const double dist = sdf3(F, c3[0], c3[1], c3[2], o);
    oob += o ? 1 : 0;
    const double gap = g[3] + re - dist;
    psi += gap > 0.0 ? gap * gap : 0.0;
  }
  return so * psi;
}

__global__ void __launch_bounds__(128) arm_factor_kernel(int64_t nfac, const double* __restrict__ means,
                                                         const double* __restrict__ chols, int nproj,
                                                         const double* __restrict__ proj,
                                                         const double* __restrict__ mom,
                                                         const int* __restrict__ cnt, FieldDev F,
                                                         const __grid_constant__ ArmConst A, double re,
                                                         double so, double* __restrict__ e0,
                                                         double* __restrict__ e1, double* __restrict__ e2,
                                                         unsigned long long* oob_total) {
  __shared__ double s_psi[4][kMaxProj];
  __shared__ double s_L[4][NX * NX];
  __shared__ double s_E[4][NM];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * 4 + wid;
  if (f >= nfac) return;  // whole warps leave together
  const double* mu = means + f * NX;
  const double* Lg = chols + f * NX * NX;
  for (int k = lane; k < NX * NX; k += 32) s_L[wid][k] = Lg[k];
  __syncwarp();
  // ---- psi at every joint-space projection
  unsigned long long nout = 0;
  for (int j = lane; j < nproj; j += 32) {
    double q[NQ];
#pragma unroll
    for (int r = 0; r < NQ; ++r) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k <= r; ++k) t += s_L[wid][r * NX + k] * proj[j * NQ + k];
      q[r] = mu[r] + t;
    }
    int o = 0;
    s_psi[wid][j] = arm_psi(A, F, q, re, so, o);
    nout += (unsigned long long)o * (unsigned long long)cnt[j];
  }
  __syncwarp();
  // ---- xi-basis moments: E_k = sum_j psi_j mom_j[k]  (k: m0 | m1 (14) | m2 packed (105))
  for (int k = lane; k < NM; k += 32) {
    double t = 0.0;
    for (int j = 0; j < nproj; ++j) t += s_psi[wid][j] * mom[j * NM + k];
    s_E[wid][k] = t;
  }
  for (int off = 16; off > 0; off >>= 1) nout += __shfl_down_sync(0xffffffffu, nout, off);
  if (lane == 0 && nout) atomicAdd(oob_total, nout);
  __syncwarp();
  // ---- back to the x basis: e1 = L E1, e2 = L E2 L^T (lane r < 14 owns row r)
  if (lane == 0) e0[f] = s_E[wid][0];
  if (lane < NX) {
    const int r = lane;
    const double* E1 = s_E[wid] + 1;
    const double* E2 = s_E[wid] + 1 + NX;
    auto e2at = [&](int a, int b) { return a >= b ? E2[a * (a + 1) / 2 + b] : E2[b * (b + 1) / 2 + a]; };
    double t = 0.0, v[NX];
    for (int k = 0; k <= r; ++k) t += s_L[wid][r * NX + k] * E1[k];
    e1[f * NX + r] = t;
    for (int c = 0; c < NX; ++c) {  // v = row r of L E2
      double a = 0.0;
      for (int k = 0; k <= r; ++k) a += s_L[wid][r * NX + k] * e2at(k, c);
      v[c] = a;
    }
    for (int c = 0; c < NX; ++c) {
      double a = 0.0;
      for (int k = 0; k <= c; ++k) a += v[k] * s_L[wid][c * NX + k];
      e2[(f * NX + r) * NX + c] = a;
    }
  }
}

// gaussian_sqrt (quadrature.py:164-181) of each factor's covariance, one warp
// per factor: np.linalg.cholesky (lower triangle, no pivot floor), one
// +1e-10 I retry; a failure of both is the eigh branch, reported (GVP_ERR_SQRT)
__global__ void __launch_bounds__(128) arm_chol_kernel(int64_t nfac, const double* __restrict__ covs,
                                                       double* __restrict__ chols, int* status, int* where) {
  using WS = wide::WarpWs<16>;
  constexpr int LD = WS::LD;
  extern __shared__ __align__(16) double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * 4 + wid;
  if (f >= nfac) return;
  WS w(sm + wid * WS::DOUBLES);
  const double* C = covs + f * NX * NX;
  double pm = 1.0;
  int pe = 0;
  wide::stage<16>(w.T, NX, [&](int a, int b) { return C[a * NX + b]; });
  bool ok = wide::chol<16, false, false>(w.T, w.L, NX, pm, pe);
  if (!ok) {
    wide::stage<16>(w.T, NX, [&](int a, int b) { return C[a * NX + b] + (a == b ? 1e-10 : 0.0); });
    ok = wide::chol<16, false, false>(w.T, w.L, NX, pm, pe);
  }
  if (!ok) {
    if (lane == 0) {
      atomicMax(status, GVP_ERR_SQRT);
      atomicMin(where, (int)f);
    }
    return;
  }
  for (int idx = lane; idx < NX * NX; idx += 32) {
    const int a = idx / NX, b = idx - a * NX;
    chols[f * NX * NX + idx] = b <= a ? w.L[a * LD + b] : 0.0;
  }
}

// _moment_gradients (factors.py:95-104) from the factor's Cholesky root:
// P = L^-T L^-1, g_mu = P e1, g_Sigma = sym(-1/2 P e0 + 1/2 P e2 P);
// e_psi = max(e0, 0) (factors.py:218-224); non-finite moments -> GVP_ERR_NONFINITE
__global__ void __launch_bounds__(128) arm_grads_kernel(int64_t nfac, const double* __restrict__ chols,
                                                        const double* __restrict__ e0, const double* __restrict__ e1,
                                                        const double* __restrict__ e2, double* __restrict__ epsi,
                                                        double* __restrict__ gmu, double* __restrict__ gsig,
                                                        int* status, int* where) {
  using WS = wide::WarpWs<16>;
  constexpr int LD = WS::LD;
  extern __shared__ __align__(16) double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * 4 + wid;
  if (f >= nfac) return;
  WS w(sm + wid * WS::DOUBLES);
  bool fin = isfinite(e0[f]);
  for (int idx = lane; idx < NX * NX; idx += 32) fin = fin && isfinite(e2[f * NX * NX + idx]);
  if (lane < NX) fin = fin && isfinite(e1[f * NX + lane]);
  fin = __all_sync(0xffffffffu, fin);
  if (!fin) {
    if (lane == 0) {
      atomicMax(status, GVP_ERR_NONFINITE);
      atomicMin(where, (int)f);
    }
    return;
  }
  wide::stage<16>(w.L, NX, [&](int a, int b) { return chols[f * NX * NX + a * NX + b]; });
  wide::trinv<16>(w.L, w.Li, NX);
  wide::ltl<16>(w.Li, w.X, NX);                                                   // X = P
  wide::stage<16>(w.U, NX, [&](int a, int b) { return e2[f * NX * NX + a * NX + b]; });  // U = e2
  const int r = lane;
  const double ee0 = e0[f];
  // row r of (1/2 P) e2 -> T
  double t[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    double a = 0.0;
    if (r < NX && c < NX) {
#pragma unroll
      for (int k = 0; k < NX; ++k) a += (0.5 * w.X[r * LD + k]) * w.U[k * LD + c];
    }
    t[c] = a;
  }
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (r < NX && c < NX) w.T[r * LD + c] = t[c];
  __syncwarp();
  // G = -1/2 P e0 + ((1/2 P) e2) P -> U (e2 no longer needed)
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    double a = 0.0;
    if (r < NX && c < NX) {
#pragma unroll
      for (int k = 0; k < NX; ++k) a += w.T[r * LD + k] * w.X[k * LD + c];
      a = (-0.5 * w.X[r * LD + c]) * ee0 + a;
    }
    t[c] = a;
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 16; ++c)
    if (r < NX && c < NX) w.U[r * LD + c] = t[c];
  __syncwarp();
  if (r < NX) {
    double g = 0.0;
#pragma unroll
    for (int k = 0; k < NX; ++k) g += w.X[r * LD + k] * e1[f * NX + k];
    gmu[f * NX + r] = g;
#pragma unroll
    for (int c = 0; c < NX; ++c) gsig[(f * NX + r) * NX + c] = 0.5 * (w.U[r * LD + c] + w.U[c * LD + r]);
  }
  if (lane == 0) epsi[f] = ee0 > 0.0 ? ee0 : 0.0;
}

// device-resident arm collision model: grid (corner-packed), arm constants,
// the rule's projection tables and per-call buffers (gvp_arm_create)
struct ArmCtx {
  Field field;
  ArmConst A{};
  double re = 0.0, so = 0.0;
  int nproj = 0;
  double *proj = nullptr, *mom = nullptr;
  int* cnt = nullptr;
  int64_t cap = 0;
  double *means = nullptr, *covs = nullptr, *chols = nullptr, *e0 = nullptr, *e1 = nullptr, *e2 = nullptr,
         *epsi = nullptr, *gmu = nullptr, *gsig = nullptr;
  int* st = nullptr;
  unsigned long long* oob = nullptr;
  cudaStream_t s = nullptr;
  ~ArmCtx() {
    for (void* p : {(void*)proj, (void*)mom, (void*)cnt, (void*)means, (void*)covs, (void*)chols, (void*)e0,
                    (void*)e1, (void*)e2, (void*)epsi, (void*)gmu, (void*)gsig, (void*)st, (void*)oob})
      if (p) cudaFree(p);
    if (s) cudaStreamDestroy(s);
  }
  int reserve(int64_t F) {
    if (F <= cap) return GVP_OK;
    for (double** p : {&means, &covs, &chols, &e0, &e1, &e2, &epsi, &gmu, &gsig}) {
      if (*p) cudaFree(*p);
      *p = nullptr;
    }
    const size_t v = F * NX * 8, m = F * NX * NX * 8, sc = F * 8;
    GVP_CUDA(cudaMalloc(&means, v));
    GVP_CUDA(cudaMalloc(&covs, m));
    GVP_CUDA(cudaMalloc(&chols, m));
    GVP_CUDA(cudaMalloc(&e0, sc));
    GVP_CUDA(cudaMalloc(&e1, v));
    GVP_CUDA(cudaMalloc(&e2, m));
    GVP_CUDA(cudaMalloc(&epsi, sc));
    GVP_CUDA(cudaMalloc(&gmu, v));
    GVP_CUDA(cudaMalloc(&gsig, m));
    cap = F;
    return GVP_OK;
  }
};

}  // namespace arm
}  // namespace gvp

using namespace gvp;

// Batched sphere-arm factor moments (the reference's factor_expectations
// contract, _kernels.pyx:132-177, for the 7-DOF arm of SURVEY C3). Host arrays:
// means (F,14), chols (F,14,14) lower; the rule's joint-space projection
// tables proj (NP,7), mom (NP,120) = [m0 | m1 (14) | m2 packed (105)], cnt (NP);
// grid (nz,ny,nx) with origin (x,y,z) and cell; dh (7,4) = (a, d, alpha,
// theta offset) per joint, base (3); spheres: link (S) in 0..7 and geom (S,4)
// = (local x, y, z, radius). Out: e0 (F), e1 (F,14), e2 (F,14,14), oob.
extern "C" int gvp_arm_factor_expectations(int64_t nfac, const double* means, const double* chols, int32_t nproj,
                                           const double* proj, const double* mom, const int32_t* cnt,
                                           const double* grid, const int64_t* shape, const double* origin,
                                           double cell, const double* dh, const double* base, int32_t nspheres,
                                           const int32_t* sphere_link, const double* sphere_geom,
                                           double radius_eps, double sigma_obs, double* e0, double* e1,
                                           double* e2, int64_t* oob) {
  using namespace gvp::arm;
  if (nfac < 0 || nproj < 1 || nproj > kMaxProj || nspheres < 0 || nspheres > kMaxSpheres || !grid || !shape ||
      !origin || !(cell > 0) || !dh || !base)
    return GVP_ERR_ARG;
  for (int s = 0; s < nspheres; ++s)
    if (sphere_link[s] < 0 || sphere_link[s] > NQ) return GVP_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device visible");
    return GVP_ERR_NO_DEVICE;
  }
  if (oob) *oob = 0;
  if (nfac == 0) return GVP_OK;
  ArmConst A{};
  for (int j = 0; j < NQ; ++j)
    for (int k = 0; k < 4; ++k) A.dh[j][k] = dh[j * 4 + k];
  for (int k = 0; k < 3; ++k) A.base[k] = base[k];
  A.nsph = nspheres;
  for (int s = 0; s < nspheres; ++s) {
    A.link[s] = sphere_link[s];
    for (int k = 0; k < 4; ++k) A.geom[s][k] = sphere_geom[s * 4 + k];
  }
  Field field;
  int r = field.build(grid, 3, shape, origin, cell, 0);
  if (r) return r;
  std::vector<void*> bufs;
  auto get = [&](size_t bytes, void** p) {
    if (cudaMalloc(p, std::max<size_t>(bytes, 8)) != cudaSuccess) return false;
    bufs.push_back(*p);
    return true;
  };
  double *dm, *dc, *dp, *dmo, *d0, *d1, *d2;
  int* dcnt;
  unsigned long long* doob;
  bool ok = get(nfac * NX * 8, (void**)&dm) && get(nfac * NX * NX * 8, (void**)&dc) &&
            get((size_t)nproj * NQ * 8, (void**)&dp) && get((size_t)nproj * NM * 8, (void**)&dmo) &&
            get((size_t)nproj * 4, (void**)&dcnt) && get(nfac * 8, (void**)&d0) && get(nfac * NX * 8, (void**)&d1) &&
            get(nfac * NX * NX * 8, (void**)&d2) && get(8, (void**)&doob);
  if (ok) {
    cudaMemcpy(dm, means, nfac * NX * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, chols, nfac * NX * NX * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, proj, (size_t)nproj * NQ * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dmo, mom, (size_t)nproj * NM * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dcnt, cnt, (size_t)nproj * 4, cudaMemcpyHostToDevice);
    cudaMemset(doob, 0, 8);
    arm_factor_kernel<<<(unsigned)((nfac + 3) / 4), 128>>>(nfac, dm, dc, nproj, dp, dmo, dcnt, field.dev, A,
                                                            radius_eps, sigma_obs, d0, d1, d2, doob);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      set_error(cudaGetErrorString(e));
      r = GVP_ERR_CUDA;
    } else {
      unsigned long long h = 0;
      cudaMemcpy(e0, d0, nfac * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(e1, d1, nfac * NX * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(e2, d2, nfac * NX * NX * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&h, doob, 8, cudaMemcpyDeviceToHost);
      if (oob) *oob = (int64_t)h;
    }
  } else {
    set_error("cudaMalloc failed");
    r = GVP_ERR_CUDA;
  }
  for (void* p : bufs) cudaFree(p);
  return r;
}

// ---------------------------------------------------------------- arm model handle
extern "C" int gvp_arm_create(gvp_arm** out, const double* grid, const int64_t* shape, const double* origin,
                              double cell, const double* dh, const double* base, int32_t nspheres,
                              const int32_t* sphere_link, const double* sphere_geom, double radius_eps,
                              double sigma_obs, int32_t nproj, const double* proj, const double* mom,
                              const int32_t* cnt) {
  using namespace gvp::arm;
  if (!out || nproj < 1 || nproj > kMaxProj || nspheres < 0 || nspheres > kMaxSpheres || !grid || !shape ||
      !origin || !(cell > 0) || !dh || !base || !proj || !mom || !cnt) {
    set_error("gvp_arm_create: bad argument");
    return GVP_ERR_ARG;
  }
  for (int s = 0; s < nspheres; ++s)
    if (sphere_link[s] < 0 || sphere_link[s] > NQ) return set_error("sphere_link must be in 0..7"), GVP_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device visible");
    return GVP_ERR_NO_DEVICE;
  }
  auto* c = new ArmCtx();
  for (int j = 0; j < NQ; ++j)
    for (int k = 0; k < 4; ++k) c->A.dh[j][k] = dh[j * 4 + k];
  for (int k = 0; k < 3; ++k) c->A.base[k] = base[k];
  c->A.nsph = nspheres;
  for (int s = 0; s < nspheres; ++s) {
    c->A.link[s] = sphere_link[s];
    for (int k = 0; k < 4; ++k) c->A.geom[s][k] = sphere_geom[s * 4 + k];
  }
  c->re = radius_eps;
  c->so = sigma_obs;
  c->nproj = nproj;
  int r = GVP_OK;
  auto fail = [&](int code) {
    delete c;
    return code;
  };
  if (cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking) != cudaSuccess) return fail(GVP_ERR_CUDA);
  if ((r = c->field.build(grid, 3, shape, origin, cell, c->s))) return fail(r);
  if (cudaMalloc(&c->proj, (size_t)nproj * NQ * 8) != cudaSuccess ||
      cudaMalloc(&c->mom, (size_t)nproj * NM * 8) != cudaSuccess || cudaMalloc(&c->cnt, (size_t)nproj * 4) != cudaSuccess ||
      cudaMalloc(&c->st, 8) != cudaSuccess || cudaMalloc(&c->oob, 8) != cudaSuccess) {
    set_error("cudaMalloc failed");
    return fail(GVP_ERR_CUDA);
  }
  cudaMemcpy(c->proj, proj, (size_t)nproj * NQ * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->mom, mom, (size_t)nproj * NM * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->cnt, cnt, (size_t)nproj * 4, cudaMemcpyHostToDevice);
  *out = reinterpret_cast<gvp_arm*>(c);
  return GVP_OK;
}

extern "C" void gvp_arm_destroy(gvp_arm* h) { delete reinterpret_cast<gvp::arm::ArmCtx*>(h); }

// The factor stage of evaluate_all_factors (factors.py:167-225) for the arm:
// per factor covariance -> gaussian_sqrt -> moments -> gradients, all on the
// device. means (F,14), covs (F,14,14) of the factors' knots; out e_psi (F),
// g_mu (F,14), g_sigma (F,14,14), oob. GVP_ERR_SQRT / GVP_ERR_NONFINITE with
// *where = the factor's position in the batch.
extern "C" int gvp_arm_factor_grads(gvp_arm* h, int64_t nfac, const double* means, const double* covs,
                                    double* e_psi, double* g_mu, double* g_sigma, int64_t* oob, int64_t* where) {
  using namespace gvp::arm;
  auto* c = reinterpret_cast<ArmCtx*>(h);
  if (!c || nfac < 0) return set_error("gvp_arm_factor_grads: bad argument"), GVP_ERR_ARG;
  if (oob) *oob = 0;
  if (where) *where = -1;
  if (nfac == 0) return GVP_OK;
  int r = c->reserve(nfac);
  if (r) return r;
  cudaStream_t s = c->s;
  const size_t v = nfac * NX * 8, m = nfac * NX * NX * 8;
  const int init[2] = {GVP_OK, 0x7fffffff};
  GVP_CUDA(cudaMemcpyAsync(c->means, means, v, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(c->covs, covs, m, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(c->st, init, 8, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemsetAsync(c->oob, 0, 8, s));
  const unsigned nb = (unsigned)((nfac + 3) / 4);
  const size_t wbytes = 4 * gvp::wide::WarpWs<16>::DOUBLES * 8;
  arm_chol_kernel<<<nb, 128, wbytes, s>>>(nfac, c->covs, c->chols, c->st, c->st + 1);
  int hst[2];
  GVP_CUDA(cudaMemcpyAsync(hst, c->st, 8, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  if (hst[0] != GVP_OK) {
    if (where) *where = hst[1];
    set_error("covariance needs the eigendecomposition root");
    return hst[0];
  }
  arm_factor_kernel<<<nb, 128, 0, s>>>(nfac, c->means, c->chols, c->nproj, c->proj, c->mom, c->cnt, c->field.dev,
                                       c->A, c->re, c->so, c->e0, c->e1, c->e2, c->oob);
  arm_grads_kernel<<<nb, 128, wbytes, s>>>(nfac, c->chols, c->e0, c->e1, c->e2, c->epsi, c->gmu, c->gsig, c->st,
                                           c->st + 1);
  GVP_CUDA(cudaGetLastError());
  unsigned long long ho = 0;
  GVP_CUDA(cudaMemcpyAsync(hst, c->st, 8, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaMemcpyAsync(&ho, c->oob, 8, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaMemcpyAsync(e_psi, c->epsi, nfac * 8, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaMemcpyAsync(g_mu, c->gmu, v, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaMemcpyAsync(g_sigma, c->gsig, m, cudaMemcpyDeviceToHost, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  if (oob) *oob = (int64_t)ho;
  if (hst[0] != GVP_OK) {
    if (where) *where = hst[1];
    set_error("non-finite expectation");
    return hst[0];
  }
  return GVP_OK;
}
