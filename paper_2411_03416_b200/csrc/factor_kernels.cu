// Kernel (a): collision-factor quadrature on B200.
//
// Two kernels, both one thread per (plan, factor), plan index fastest so a
// warp's loads of a knot's mean/covariance are 256 B contiguous:
//
//  * factor_moments_kernel — the reference's exact contract
//    (_kernels.pyx:93-177): given (means, chols) produce e0/e1/e2 and the OOB
//    count. It loops over every sigma point in ascending order and uses
//    explicitly rounded fp64 ops (__dmul_rn/__dadd_rn, no FMA contraction) in
//    the reference's evaluation order, so it reproduces the compiled
//    reference (gcc -O3 on x86-64, no FMA) bit for bit.
//
//  * factor_grads_kernel — the fused engine kernel (factors.py:167-225 after
//    marginal extraction): Cholesky of the knot covariance in registers, hinge
//    potential evaluated once per distinct position projection of the rule
//    (13 of 41 points at k_q=3, 57 of 385 at k_q=5), moments
//    contracted with per-projection weight tensors, moment-form gradients via
//    the triangular inverse (g_mu = L^{-T} E1, g_S = sym(-e0/2 P^{-1} +
//    L^{-T} E2 L^{-1}/2)). Writes straight into the joint-gradient layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "gvp_internal.cuh"

namespace gvp {

// Inside a cell the x-derivative of the multilinear interpolant interpolates
// the cell's x-edge differences, so |grad| <= sqrt(sum over axes of (max |edge
// difference| on that axis)^2) / cell, exact in 2D where each component is
// affine in the other coordinate; the maximum over cells is the Lipschitz
// constant. An SDF gives ~1 (a global per-axis bound gives sqrt(2) in 2D).
double field_lipschitz(const double* grids, int64_t nmaps, int ndim, int64_t nx, int64_t ny, int64_t nz,
                       double cell) {
  const int64_t sx = 1, sy = nx, sz = nx * ny, cells = nx * ny * nz;
  for (int64_t i = 0; i < cells * nmaps; ++i)
    if (!std::isfinite(grids[i])) return INFINITY;
  const int64_t cz = ndim == 3 ? nz - 1 : 1;
  const int nc = ndim == 3 ? 2 : 1;
  double l2 = 0.0;
  for (int64_t m = 0; m < nmaps; ++m)
    for (int64_t iz = 0; iz < cz; ++iz)
      for (int64_t iy = 0; iy + 1 < ny; ++iy)
        for (int64_t ix = 0; ix + 1 < nx; ++ix) {
          const double* g = grids + m * cells + iz * sz + iy * sy + ix;
          double mx = 0.0, my = 0.0, mz = 0.0;
          for (int c = 0; c < nc; ++c)
            for (int r = 0; r < 2; ++r) {
              mx = std::max(mx, std::fabs(g[c * sz + r * sy + sx] - g[c * sz + r * sy]));  // x-edges
              my = std::max(my, std::fabs(g[c * sz + r * sx + sy] - g[c * sz + r * sx]));  // y-edges
              if (ndim == 3) mz = std::max(mz, std::fabs(g[r * sx + c * sy + sz] - g[r * sx + c * sy]));
            }
          l2 = std::max(l2, mx * mx + my * my + mz * mz);
        }
  return std::sqrt(l2) / cell * (1.0 + 1e-12);
}

// ======================================================================= Field
Field::~Field() {
  if (d_corners) cudaFree(d_corners);
}

int Field::build(const double* grid, int ndim, const int64_t* shape, const double* origin,
                 double cell, cudaStream_t s) {
  if (ndim != 2 && ndim != 3) {
    set_error("grid must be 2D or 3D");
    return GVP_ERR_UNSUPPORTED;
  }
  FieldDev f{};
  f.ndim = ndim;
  f.nz = ndim == 3 ? shape[0] : 1;
  f.ny = shape[ndim - 2];
  f.nx = shape[ndim - 1];
  if (f.nx < 2 || f.ny < 2 || (ndim == 3 && f.nz < 2)) {
    set_error("grid needs at least 2 nodes per axis");
    return GVP_ERR_ARG;
  }
  f.ox = origin[0];
  f.oy = origin[1];
  f.oz = ndim == 3 ? origin[2] : 0.0;
  f.cell = cell;
  f.inv_cell = 1.0 / cell;
  f.lip = field_lipschitz(grid, 1, ndim, f.nx, f.ny, f.nz, cell);
  std::vector<double> packed;
  if (ndim == 2) {
    // corner-packed cells: (iy, ix) -> {g[iy][ix], g[iy][ix+1], g[iy+1][ix], g[iy+1][ix+1]}
    const int64_t cy = f.ny - 1, cx = f.nx - 1;
    packed.resize((size_t)(cy * cx * 4));
    for (int64_t iy = 0; iy < cy; ++iy)
      for (int64_t ix = 0; ix < cx; ++ix) {
        double* c = &packed[(size_t)((iy * cx + ix) * 4)];
        const double* r0 = grid + iy * f.nx + ix;
        const double* r1 = r0 + f.nx;
        c[0] = r0[0];
        c[1] = r0[1];
        c[2] = r1[0];
        c[3] = r1[1];
      }
  } else {
    // x-pair packed rows: (iz, iy, ix) -> {g[iz][iy][ix], g[iz][iy][ix+1]}
    const int64_t cx = f.nx - 1;
    packed.resize((size_t)(f.nz * f.ny * cx * 2));
    for (int64_t iz = 0; iz < f.nz; ++iz)
      for (int64_t iy = 0; iy < f.ny; ++iy)
        for (int64_t ix = 0; ix < cx; ++ix) {
          double* c = &packed[(size_t)(((iz * f.ny + iy) * cx + ix) * 2)];
          const double* g = grid + (iz * f.ny + iy) * f.nx + ix;
          c[0] = g[0];
          c[1] = g[1];
        }
  }
  const int64_t nbytes = (int64_t)(packed.size() * sizeof(double));
  if (nbytes > bytes) {
    if (d_corners) cudaFree(d_corners);
    d_corners = nullptr;
    GVP_CUDA(cudaMalloc(&d_corners, nbytes));
    bytes = nbytes;
  }
  GVP_CUDA(cudaMemcpyAsync(d_corners, packed.data(), nbytes, cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  f.corners = d_corners;
  dev = f;
  return GVP_OK;
}

// ======================================================================= Rule
Rule::~Rule() {
  if (d_buf) cudaFree(d_buf);
  if (d_cnt) cudaFree(d_cnt);
}

int Rule::build(const double* points, const double* weights, int64_t npts, int n, int P,
                cudaStream_t s) {
  if (P > n) P = n;
  // group points by the exact bit pattern of their first P coordinates
  std::map<std::vector<uint64_t>, int64_t> key_to_proj;
  std::vector<int64_t> order;  // first point of each projection, in order of appearance
  std::vector<int64_t> proj_of(npts);
  for (int64_t l = 0; l < npts; ++l) {
    std::vector<uint64_t> key(P);
    for (int k = 0; k < P; ++k) std::memcpy(&key[k], &points[l * n + k], sizeof(double));
    auto it = key_to_proj.find(key);
    if (it == key_to_proj.end()) {
      const int64_t j = (int64_t)order.size();
      key_to_proj.emplace(key, j);
      order.push_back(l);
      proj_of[l] = j;
    } else {
      proj_of[l] = it->second;
    }
  }
  const int64_t nproj = (int64_t)order.size();
  const int T = n * (n + 1) / 2;
  const int M = 1 + n + T;
  std::vector<double> proj((size_t)(nproj * P)), mom((size_t)(nproj * M), 0.0);
  std::vector<int> cnt((size_t)nproj, 0);
  double prad = 0.0;
  for (int64_t j = 0; j < nproj; ++j) {
    double r2 = 0.0;
    for (int k = 0; k < P; ++k) {
      proj[j * P + k] = points[order[j] * n + k];
      r2 += proj[j * P + k] * proj[j * P + k];
    }
    prad = std::max(prad, std::sqrt(r2));
  }
  for (int64_t l = 0; l < npts; ++l) {  // ascending point order within each group
    const int64_t j = proj_of[l];
    const double w = weights[l];
    const double* x = points + l * n;
    double* m = &mom[(size_t)(j * M)];
    m[0] += w;
    for (int r = 0; r < n; ++r) m[1 + r] += w * x[r];
    for (int r = 0; r < n; ++r)
      for (int c = 0; c <= r; ++c) m[1 + n + r * (r + 1) / 2 + c] += w * x[r] * x[c];
    cnt[j] += 1;
  }
  const int64_t nd = npts * n + npts + nproj * P + nproj * M;
  if (d_buf) cudaFree(d_buf);
  if (d_cnt) cudaFree(d_cnt);
  d_buf = nullptr;
  d_cnt = nullptr;
  GVP_CUDA(cudaMalloc(&d_buf, std::max<int64_t>(nd, 1) * sizeof(double)));
  GVP_CUDA(cudaMalloc(&d_cnt, std::max<int64_t>(nproj, 1) * sizeof(int)));
  double* p = d_buf;
  GVP_CUDA(cudaMemcpyAsync(p, points, npts * n * sizeof(double), cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(p + npts * n, weights, npts * sizeof(double), cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(p + npts * n + npts, proj.data(), nproj * P * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(p + npts * n + npts + nproj * P, mom.data(), nproj * M * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaMemcpyAsync(d_cnt, cnt.data(), nproj * sizeof(int), cudaMemcpyHostToDevice, s));
  GVP_CUDA(cudaStreamSynchronize(s));
  h_proj = proj;
  h_mom = mom;
  h_cnt = cnt;
  dev.host = this;
  dev.n = n;
  dev.P = P;
  dev.npts = npts;
  dev.nproj = nproj;
  dev.proj_radius = prad * (1.0 + 1e-12);
  dev.points = p;
  dev.weights = p + npts * n;
  dev.proj = p + npts * n + npts;
  dev.mom = p + npts * n + npts + nproj * P;
  dev.cnt = d_cnt;
  return GVP_OK;
}

// ============================================================ interpolation
// Border-clamped bilinear interpolation with the reference's operation order
// (_kernels.pyx:18-45). EXACT=true uses explicitly rounded ops (no FMA) so
// the result equals gcc's x86-64 evaluation of the Cython kernel.
template <bool EXACT>
GVP_DEV double fmul(double a, double b) { return EXACT ? __dmul_rn(a, b) : a * b; }
template <bool EXACT>
GVP_DEV double fadd(double a, double b) { return EXACT ? __dadd_rn(a, b) : a + b; }
template <bool EXACT>
GVP_DEV double fsub(double a, double b) { return EXACT ? __dsub_rn(a, b) : a - b; }

// branch-free border clamp; same values as the reference's if/elif for finite u
GVP_DEV double clamp_axis(double u, double top, bool& out) {
  out = out || (u < 0.0) || (u > top);
  return fmin(fmax(u, 0.0), top);
}

template <bool EXACT>
GVP_DEV double interp2(const FieldDev& F, double px, double py, bool& out) {
  // exact path divides like the reference; the fused path multiplies by 1/cell
  double u = EXACT ? __ddiv_rn(__dsub_rn(px, F.ox), F.cell) : (px - F.ox) * F.inv_cell;
  double v = EXACT ? __ddiv_rn(__dsub_rn(py, F.oy), F.cell) : (py - F.oy) * F.inv_cell;
  out = false;
  u = clamp_axis(u, (double)(F.nx - 1), out);
  v = clamp_axis(v, (double)(F.ny - 1), out);
  int64_t ix = (int64_t)floor(u);
  int64_t iy = (int64_t)floor(v);
  if (ix > F.nx - 2) ix = F.nx - 2;
  if (iy > F.ny - 2) iy = F.ny - 2;
  const double fx = fsub<EXACT>(u, (double)ix);
  const double fy = fsub<EXACT>(v, (double)iy);
  // one 32 B sector: {g00, g01, g10, g11}
  const double2* c = reinterpret_cast<const double2*>(F.corners + (iy * (F.nx - 1) + ix) * 4);
  const double2 a = __ldg(c);
  const double2 b = __ldg(c + 1);
  const double gx = fsub<EXACT>(1.0, fx), gy = fsub<EXACT>(1.0, fy);
  double r = fmul<EXACT>(fmul<EXACT>(a.x, gx), gy);
  r = fadd<EXACT>(r, fmul<EXACT>(fmul<EXACT>(a.y, fx), gy));
  r = fadd<EXACT>(r, fmul<EXACT>(fmul<EXACT>(b.x, gx), fy));
  r = fadd<EXACT>(r, fmul<EXACT>(fmul<EXACT>(b.y, fx), fy));
  return r;
}

// interp2 for a point the caller has proven strictly inside the grid (the
// factor kernel's cloud test): no clamping or OOB flag, the cell index is a
// truncation, and the bilinear form is three lerps
GVP_DEV double interp2_in(const FieldDev& F, double px, double py) {
  const double u = (px - F.ox) * F.inv_cell, v = (py - F.oy) * F.inv_cell;
  const int ix = __double2int_rz(u), iy = __double2int_rz(v);
  const double fx = u - (double)ix, fy = v - (double)iy;
  const double2* c = reinterpret_cast<const double2*>(F.corners) + 2 * (size_t)(unsigned)(iy * (int)(F.nx - 1) + ix);
  const double2 a = __ldg(c), b = __ldg(c + 1);
  const double top = fma(fx, a.y - a.x, a.x), bot = fma(fx, b.y - b.x, b.x);
  return fma(fy, bot - top, top);
}

// interp2<false> with 32-bit cell indices and the bilinear form as three lerps
// (the engine's quadrature; ~30 fewer instructions per lookup). Same clamping
// and out-of-bounds flag; the grid has < 2^31 cells.
GVP_DEV double interp2_clamped(const FieldDev& F, double px, double py, bool& out) {
  double u = (px - F.ox) * F.inv_cell, v = (py - F.oy) * F.inv_cell;
  const double tx = (double)(F.nx - 1), ty = (double)(F.ny - 1);
  out = (u < 0.0) || (u > tx) || (v < 0.0) || (v > ty);
  u = fmin(fmax(u, 0.0), tx);
  v = fmin(fmax(v, 0.0), ty);
  const int ix = min(__double2int_rz(u), (int)F.nx - 2), iy = min(__double2int_rz(v), (int)F.ny - 2);
  const double fx = u - (double)ix, fy = v - (double)iy;
  const double2* c = reinterpret_cast<const double2*>(F.corners) + 2 * (size_t)(unsigned)(iy * (int)(F.nx - 1) + ix);
  const double2 a = __ldg(c), b = __ldg(c + 1);
  const double top = fma(fx, a.y - a.x, a.x), bot = fma(fx, b.y - b.x, b.x);
  return fma(fy, bot - top, top);
}

// the out-of-bounds flag interp2_clamped / interp3<false> would raise at (px, py[, pz])
template <int P>
GVP_DEV bool outside_grid(const FieldDev& F, const double (&pos)[P]) {
  const double u = (pos[0] - F.ox) * F.inv_cell, v = (pos[1] - F.oy) * F.inv_cell;
  bool o = (u < 0.0) || (u > (double)(F.nx - 1)) || (v < 0.0) || (v > (double)(F.ny - 1));
  if (P == 3) {
    const double w = (pos[P - 1] - F.oz) * F.inv_cell;
    o = o || (w < 0.0) || (w > (double)(F.nz - 1));
  }
  return o;
}

// trilinear (_kernels.pyx:48-90): two bilinear planes combined in z
template <bool EXACT>
GVP_DEV double interp3(const FieldDev& F, double px, double py, double pz, bool& out) {
  double u = EXACT ? __ddiv_rn(__dsub_rn(px, F.ox), F.cell) : (px - F.ox) * F.inv_cell;
  double v = EXACT ? __ddiv_rn(__dsub_rn(py, F.oy), F.cell) : (py - F.oy) * F.inv_cell;
  double w = EXACT ? __ddiv_rn(__dsub_rn(pz, F.oz), F.cell) : (pz - F.oz) * F.inv_cell;
  out = false;
  u = clamp_axis(u, (double)(F.nx - 1), out);
  v = clamp_axis(v, (double)(F.ny - 1), out);
  w = clamp_axis(w, (double)(F.nz - 1), out);
  int64_t ix = (int64_t)floor(u), iy = (int64_t)floor(v), iz = (int64_t)floor(w);
  if (ix > F.nx - 2) ix = F.nx - 2;
  if (iy > F.ny - 2) iy = F.ny - 2;
  if (iz > F.nz - 2) iz = F.nz - 2;
  const double fx = fsub<EXACT>(u, (double)ix);
  const double fy = fsub<EXACT>(v, (double)iy);
  const double fz = fsub<EXACT>(w, (double)iz);
  const int64_t cx = F.nx - 1;
  const double2* base = reinterpret_cast<const double2*>(F.corners);
  const double2 c00 = __ldg(base + (iz * F.ny + iy) * cx + ix);
  const double2 c01 = __ldg(base + (iz * F.ny + iy + 1) * cx + ix);
  const double2 c10 = __ldg(base + ((iz + 1) * F.ny + iy) * cx + ix);
  const double2 c11 = __ldg(base + ((iz + 1) * F.ny + iy + 1) * cx + ix);
  const double gx = fsub<EXACT>(1.0, fx), gy = fsub<EXACT>(1.0, fy), gz = fsub<EXACT>(1.0, fz);
  double v0 = fmul<EXACT>(fmul<EXACT>(c00.x, gx), gy);
  v0 = fadd<EXACT>(v0, fmul<EXACT>(fmul<EXACT>(c00.y, fx), gy));
  v0 = fadd<EXACT>(v0, fmul<EXACT>(fmul<EXACT>(c01.x, gx), fy));
  v0 = fadd<EXACT>(v0, fmul<EXACT>(fmul<EXACT>(c01.y, fx), fy));
  double v1 = fmul<EXACT>(fmul<EXACT>(c10.x, gx), gy);
  v1 = fadd<EXACT>(v1, fmul<EXACT>(fmul<EXACT>(c10.y, fx), gy));
  v1 = fadd<EXACT>(v1, fmul<EXACT>(fmul<EXACT>(c11.x, gx), fy));
  v1 = fadd<EXACT>(v1, fmul<EXACT>(fmul<EXACT>(c11.y, fx), fy));
  return fadd<EXACT>(fmul<EXACT>(v0, gz), fmul<EXACT>(v1, fz));
}

// ============================================= exact-contract moments kernel
template <int N>
__global__ void __launch_bounds__(128)
factor_moments_kernel(int64_t nfac, const double* __restrict__ means,
                      const double* __restrict__ chols, RuleDev R, FieldDev F, double radius_eps,
                      double sigma_obs, double* __restrict__ e0, double* __restrict__ e1,
                      double* __restrict__ e2, unsigned long long* __restrict__ oob) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nfac) return;
  double L[N][N], mu[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    mu[r] = __ldg(means + f * N + r);
#pragma unroll
    for (int c = 0; c < N; ++c) L[r][c] = __ldg(chols + (f * N + r) * N + c);
  }
  double s0 = 0.0, s1[N], s2[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    s1[r] = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) s2[r][c] = 0.0;
  }
  unsigned long long nout = 0;
  for (int64_t l = 0; l < R.npts; ++l) {
    double dx[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc = __dadd_rn(acc, __dmul_rn(L[r][k], __ldg(R.points + l * N + k)));
      dx[r] = acc;
    }
    bool out;
    double dist;
    if (F.ndim == 2) {
      dist = interp2<true>(F, __dadd_rn(mu[0], dx[0]), __dadd_rn(mu[1], dx[1]), out);
    } else {
      dist = interp3<true>(F, __dadd_rn(mu[0], dx[0]), __dadd_rn(mu[1], dx[1]),
                           __dadd_rn(mu[N > 2 ? 2 : 0], dx[N > 2 ? 2 : 0]), out);
    }
    nout += out ? 1ull : 0ull;
    const double gap = __dsub_rn(radius_eps, dist);
    if (gap > 0.0) {
      const double wc = __dmul_rn(__dmul_rn(__dmul_rn(__ldg(R.weights + l), sigma_obs), gap), gap);
      s0 = __dadd_rn(s0, wc);
#pragma unroll
      for (int r = 0; r < N; ++r) s1[r] = __dadd_rn(s1[r], __dmul_rn(wc, dx[r]));
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int c = 0; c < N; ++c) s2[r][c] = __dadd_rn(s2[r][c], __dmul_rn(__dmul_rn(wc, dx[r]), dx[c]));
    }
  }
  e0[f] = s0;
#pragma unroll
  for (int r = 0; r < N; ++r) {
    e1[f * N + r] = s1[r];
#pragma unroll
    for (int c = 0; c < N; ++c) e2[(f * N + r) * N + c] = s2[r][c];
  }
  if (nout) atomicAdd(oob, nout);
}

template <int N>
static int moments_impl(int64_t nfac, const double* means, const double* chols, const RuleDev& R,
                        const FieldDev& F, double re, double so, double* e0, double* e1, double* e2,
                        unsigned long long* oob, cudaStream_t s) {
  if (nfac == 0) return GVP_OK;
  const int tpb = 128;
  factor_moments_kernel<N><<<(unsigned)((nfac + tpb - 1) / tpb), tpb, 0, s>>>(
      nfac, means, chols, R, F, re, so, e0, e1, e2, oob);
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int launch_factor_moments(int64_t nfac, int n, const double* means, const double* chols,
                          const RuleDev& R, const FieldDev& F, double re, double so, double* e0,
                          double* e1, double* e2, unsigned long long* oob, cudaStream_t s) {
  if (F.ndim == 3 && n < 3) {
    set_error("3D field needs a state of at least 3 dims");
    return GVP_ERR_ARG;
  }
  switch (n) {
#define GVP_CASE(K) \
  case K:           \
    return moments_impl<K>(nfac, means, chols, R, F, re, so, e0, e1, e2, oob, s);
    GVP_CASE(1) GVP_CASE(2) GVP_CASE(3) GVP_CASE(4) GVP_CASE(5) GVP_CASE(6) GVP_CASE(7) GVP_CASE(8)
#undef GVP_CASE
    default:
      set_error("block size n must be in 1..8");
      return GVP_ERR_UNSUPPORTED;
  }
}

// ===================================================== fused gradients kernel
#ifndef GVP_FACTOR_MINBLOCKS
#define GVP_FACTOR_MINBLOCKS 4
#endif
// projection tables of a rule with NP distinct projections, passed by value
template <int NP, int P, int M>
struct RuleConst {
  double proj[NP * P];
  double mom[NP * M];
  int cnt[NP];
};

// Moment entries that vanish for a rule symmetric under xi_k -> -xi_k in every non-position
// coordinate k >= P (Smolyak/Gauss-Hermite rules are): within a group of points sharing one
// position projection, sum w xi_k = 0 and sum w xi_r xi_c = 0 for r != c with max(r, c) >= P.
// Packed lower index t = r(r+1)/2 + c. The grouped tables hold these as rounding residues
// (<= 1.4e-16 at k_q = 3/5, n = 4/6); grads_impl checks them before SYM is chosen.
__host__ __device__ constexpr bool sym_zero2(int r, int c, int P) { return r != c && (r >= P || c >= P); }
__host__ __device__ constexpr bool sym_zero_tri(int t, int P) {
  int r = 0;
  while ((r + 1) * (r + 2) / 2 <= t) ++r;
  return sym_zero2(r, t - r * (r + 1) / 2, P);
}

// gaussian_sqrt's last resort (quadrature.py:178-181): the symmetric
// eigendecomposition root R = V diag(sqrt(max(lambda, 0))) of the covariance,
// here by cyclic Jacobi rotations (eigenvalues to ~eps |lambda|_max). A
// non-triangular root mixes every coordinate into the positions, so the
// projection grouping does not apply: every sigma point of the rule is
// evaluated. _moment_gradients (factors.py:95-104) then inverts R
// (np.linalg.solve): a clipped (zero) eigenvalue makes R singular and the
// reference raises numpy.linalg.LinAlgError -> GVP_ERR_SQRT here.
template <int N>
GVP_DEV void jacobi_eigh(double (&A)[N][N], double (&V)[N][N]) {
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) V[r][c] = r == c ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, dia = 0.0;
#pragma unroll
    for (int p = 0; p < N; ++p) {
      dia += A[p][p] * A[p][p];
#pragma unroll
      for (int q = p + 1; q < N; ++q) off += A[p][q] * A[p][q];
    }
    if (!(off > 1e-36 * dia)) break;
#pragma unroll
    for (int p = 0; p < N; ++p)
#pragma unroll
      for (int q = p + 1; q < N; ++q) {
        const double apq = A[p][q];
        if (apq == 0.0) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * apq);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - sn * akq;
          A[k][q] = sn * akp + c * akq;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - sn * aqk;
          A[q][k] = sn * apk + c * aqk;
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - sn * vkq;
          V[k][q] = sn * vkp + c * vkq;
        }
      }
  }
}

// The whole factor through the eigh root (see jacobi_eigh): moments over every
// rule point, then the moment-form gradients with P^-1 = V diag(1/lambda) V'.
// S: the covariance (lower triangle read, symmetrised like 0.5 (cov + cov')).
template <int N, int P>
GVP_DEV void factor_eigh_path(const double (&S)[N][N], const double (&mu)[N], const RuleDev& R, const FieldDev& F,
                              double radius_eps, double sigma_obs, const FactorOut& out, int64_t b, int64_t f,
                              int64_t knot) {
  constexpr int T = N * (N + 1) / 2;
  double A[N][N], V[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) A[r][c] = A[c][r] = S[r][c];
  jacobi_eigh<N>(A, V);
  double root[N][N], lam[N];
  bool singular = false;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    lam[k] = A[k][k] > 0.0 ? A[k][k] : 0.0;  // np.clip(eigvals, 0.0, None)
    singular = singular || !(lam[k] > 0.0);
    const double sq = sqrt(lam[k]);
#pragma unroll
    for (int r = 0; r < N; ++r) root[r][k] = V[r][k] * sq;
  }
  double e0 = 0.0, E1[N], E2[T];
#pragma unroll
  for (int r = 0; r < N; ++r) E1[r] = 0.0;
#pragma unroll
  for (int k = 0; k < T; ++k) E2[k] = 0.0;
  unsigned long long nout = 0;
  for (int64_t l = 0; l < R.npts; ++l) {
    double dx[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc += root[r][k] * __ldg(R.points + l * N + k);
      dx[r] = acc;
    }
    bool o;
    const double d = (P == 2) ? interp2_clamped(F, mu[0] + dx[0], mu[1] + dx[1], o)
                              : interp3<false>(F, mu[0] + dx[0], mu[1] + dx[1], mu[P - 1] + dx[P - 1], o);
    nout += o ? 1ull : 0ull;
    const double gap = radius_eps - d;
    if (gap > 0.0) {
      const double wc = __ldg(R.weights + l) * sigma_obs * gap * gap;
      e0 += wc;
#pragma unroll
      for (int r = 0; r < N; ++r) {
        E1[r] += wc * dx[r];
#pragma unroll
        for (int c = 0; c <= r; ++c) E2[tri_idx(r, c)] += wc * dx[r] * dx[c];
      }
    }
  }
  if (nout) atomicAdd(out.oob + b, nout);
  bool finite = isfinite(e0);
#pragma unroll
  for (int r = 0; r < N; ++r) finite = finite && isfinite(E1[r]);
#pragma unroll
  for (int k = 0; k < T; ++k) finite = finite && isfinite(E2[k]);
  if (singular || !finite) {
    atomicMax(out.status + b, singular ? GVP_ERR_SQRT : GVP_ERR_NONFINITE);
    atomicMin(out.where + b, (int)knot);
    return;
  }
  double Pi[N][N];  // P^-1 = V diag(1/lambda) V'
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc += V[r][k] * (V[c][k] / lam[k]);
      Pi[r][c] = acc;
    }
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) acc += Pi[r][k] * E1[k];
    out.g_mu.p[knot * out.g_mu.sk + b * out.g_mu.sp + r * out.g_mu.se] = acc;
  }
  double W[N][N];  // E2 P^-1
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc += E2[r >= k ? tri_idx(r, k) : tri_idx(k, r)] * Pi[k][c];
      W[r][c] = acc;
    }
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double hrc = 0.0, hcr = 0.0;  // (P^-1 E2 P^-1)[r][c] and [c][r]
#pragma unroll
      for (int k = 0; k < N; ++k) {
        hrc += Pi[r][k] * W[k][c];
        hcr += Pi[c][k] * W[k][r];
      }
      // symmetrize(-0.5 P^-1 e0 + 0.5 P^-1 E2 P^-1)
      const double grc = -0.5 * Pi[r][c] * e0 + 0.5 * hrc, gcr = -0.5 * Pi[c][r] * e0 + 0.5 * hcr;
      out.g_diag.p[knot * out.g_diag.sk + b * out.g_diag.sp + tri_idx(r, c) * out.g_diag.se] = 0.5 * (grc + gcr);
    }
  out.e_psi(b, f, 0) = e0 > 0.0 ? e0 : 0.0;
}

template <int N, int P, bool GRID2D, int NP, bool SYM>
__global__ void __launch_bounds__(128, GVP_FACTOR_MINBLOCKS)
factor_grads_kernel(int nplans, int64_t nfac, View mean, View covs, RuleDev R, FieldDev F,
                    double radius_eps, double sigma_obs, FactorOut out,
                    const int* __restrict__ active,
                    const __grid_constant__ RuleConst<(NP > 0 ? NP : 1), P, 1 + N + N * (N + 1) / 2> RC) {
  constexpr int T = N * (N + 1) / 2;
  constexpr int M = 1 + N + T;
  int64_t b, f;
  if (GRID2D) {  // plans along x, factors along y: no integer division
    b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    f = blockIdx.y;
    if (b >= nplans) return;
  } else {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nfac * nplans) return;
    b = t % nplans;
    f = t / nplans;
  }
  const int64_t knot = f + 1;  // interior factors 1..N-1 (factors.py:159-164)
  if (active && !active[b]) return;
  if (F.plan_map) F.corners += (int64_t)F.plan_map[b] * F.map_stride;  // this plan's map of the bank

  double mu[N], S[N][N], L[N][N];
  {
    const double* mp = mean.p + knot * mean.sk + b * mean.sp;
    const double* cp = covs.p + knot * covs.sk + b * covs.sp;
#pragma unroll
    for (int r = 0; r < N; ++r) mu[r] = mp[r * mean.se];
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) S[r][c] = cp[tri_idx(r, c) * covs.se];  // packed lower
  }
  // gaussian_sqrt (quadrature.py:164-177): Cholesky, then one 1e-10 jitter retry
  // np.linalg.cholesky has no 1e-300 pivot floor: FLOOR=false
  double dinv[N];
  // false: the factor went through the eigh root (factor_eigh_path) and is done
  auto gsqrt = [&]() -> bool {
    bool ok = chol_fast<N, false>(S, L, dinv);
    if (!ok) {  // (in place: the clear-cloud bound below then covers the jittered cloud)
#pragma unroll
      for (int r = 0; r < N; ++r) S[r][r] += 1e-10;
      ok = chol_fast<N, false>(S, L, dinv);
    }
    if (!ok) {  // the eigh root (a separate fix-up kernel keeps its registers off this one)
      if (out.eigh_list) {
        out.eigh_list[1 + atomicAdd(out.eigh_list, 1)] = (int)(b * nfac + f);
      } else {
        atomicMax(out.status + b, GVP_ERR_SQRT);
        atomicMin(out.where + b, (int)knot);
      }
    }
    return ok;
  };
  if (!gsqrt()) return;

  // ---- quadrature over distinct position projections
  double e0 = 0.0, E1[N], E2[T];
#pragma unroll
  for (int r = 0; r < N; ++r) E1[r] = 0.0;
#pragma unroll
  for (int k = 0; k < T; ++k) E2[k] = 0.0;
  unsigned long long nout = 0;
  if constexpr (NP > 0) {
    // rule tables live in the kernel's parameter space: every projection
    // coordinate and moment is a constant-bank operand of its DFMA (no loads),
    // the loop is fully unrolled and the accumulation is branch-free
    // Provably clear: every sigma position lies within Rad = |L[:P,:P]| * max_j |xi_j[:P]| of
    // mu[:P] and the interpolated field is F.lip-Lipschitz, so if d(mu) - lip * Rad exceeds
    // radius_eps (margin 1e-9 >> rounding) no point can hit; with the cloud inside the grid no
    // point is out of bounds either. One gather instead of NP — the same zeros as below.
    double fr = 0.0;
    if (P == 2) {
      // spectral norm of L[:2,:2]: |L_pp xi| <= sqrt(lambda_max(L_pp L_pp')) |xi|, and
      // L_pp L_pp' = S[:2,:2] (the Cholesky's leading block), closed form; up to sqrt(2)
      // tighter than the Frobenius bound for a round cloud. (1 + 1e-12) covers rounding.
      const double a = S[0][0], c = S[1][1], h = 0.5 * (a - c);
      fr = (0.5 * (a + c) + sqrt(h * h + S[1][0] * S[1][0])) * (1.0 + 1e-12);
    } else {
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k <= r; ++k) fr += L[r][k] * L[r][k];
    }
    const double Rad = sqrt(fr) * R.proj_radius;
    const double slack = 1e-9 * F.cell;
    bool inside = (mu[0] - Rad > F.ox + slack) && (mu[0] + Rad < F.ox + (double)(F.nx - 1) * F.cell - slack) &&
                  (mu[1] - Rad > F.oy + slack) && (mu[1] + Rad < F.oy + (double)(F.ny - 1) * F.cell - slack);
    if (P == 3)
      inside = inside && (mu[P - 1] - Rad > F.oz + slack) &&
               (mu[P - 1] + Rad < F.oz + (double)(F.nz - 1) * F.cell - slack);
    // The test also holds for clouds that leave the grid: every lookup clamps its point to the
    // grid box (a 1-Lipschitz projection), so clamp(p_j) stays within Rad of clamp(mu) and
    // the interpolant is lip-Lipschitz on the box. Only the OOB count then needs the points.
    if (F.lip < INFINITY) {
      bool oc;
      const double dc = (P == 2) ? interp2_clamped(F, mu[0], mu[1], oc)
                                 : interp3<false>(F, mu[0], mu[1], mu[P - 1], oc);
      if (dc - F.lip * Rad - radius_eps > 1e-9) {
        if (!inside) {  // bounds test of every projection, as the quadrature below does it
#pragma unroll
          for (int j = 0; j < NP; ++j) {
            double pos[P];
#pragma unroll
            for (int r = 0; r < P; ++r) {
              double acc = 0.0;
#pragma unroll
              for (int k = 0; k <= r; ++k) acc += L[r][k] * RC.proj[j * P + k];
              pos[r] = mu[r] + acc;
            }
            nout += outside_grid<P>(F, pos) ? (unsigned long long)RC.cnt[j] : 0ull;
          }
          if (nout) atomicAdd(out.oob + b, nout);
        }
#pragma unroll
        for (int r = 0; r < N; ++r) out.g_mu.p[knot * out.g_mu.sk + b * out.g_mu.sp + r * out.g_mu.se] = 0.0;
#pragma unroll
        for (int k = 0; k < T; ++k)
          out.g_diag.p[knot * out.g_diag.sk + b * out.g_diag.sp + k * out.g_diag.se] = 0.0;
        out.e_psi(b, f, 0) = 0.0;
        return;
      }
    }
    double psi[NP];
    bool any_hit = false;
    if (P == 2 && __all_sync(__activemask(), inside)) {
      // the whole cloud is strictly inside the grid: no clamping, no OOB count (warp-uniform,
      // so a warp never runs both loops)
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const double px = mu[0] + L[0][0] * RC.proj[j * P];
        const double py = mu[1] + (L[1][0] * RC.proj[j * P] + L[1][1] * RC.proj[j * P + 1]);
        const double gap = radius_eps - interp2_in(F, px, py);
        psi[j] = gap > 0.0 ? sigma_obs * gap * gap : 0.0;
        any_hit = any_hit || (gap > 0.0);
      }
    } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double pos[P];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k <= r; ++k) acc += L[r][k] * RC.proj[j * P + k];
        pos[r] = mu[r] + acc;
      }
      bool o;
      const double d = (P == 2) ? interp2_clamped(F, pos[0], pos[1], o)
                                : interp3<false>(F, pos[0], pos[1], pos[P - 1], o);
      nout += o ? (unsigned long long)RC.cnt[j] : 0ull;
      const double gap = radius_eps - d;
      psi[j] = gap > 0.0 ? sigma_obs * gap * gap : 0.0;
      any_hit = any_hit || (gap > 0.0);
    }
    }
    if (!any_hit) {  // clear of every obstacle: all moments, gradients and e_psi are zero
      if (nout) atomicAdd(out.oob + b, nout);
#pragma unroll
      for (int r = 0; r < N; ++r) out.g_mu.p[knot * out.g_mu.sk + b * out.g_mu.sp + r * out.g_mu.se] = 0.0;
#pragma unroll
      for (int k = 0; k < T; ++k)
        out.g_diag.p[knot * out.g_diag.sk + b * out.g_diag.sp + k * out.g_diag.se] = 0.0;
      out.e_psi(b, f, 0) = 0.0;
      return;
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      e0 += psi[j] * RC.mom[j * M];
#pragma unroll
      for (int r = 0; r < N; ++r)
        if (!SYM || r < P) E1[r] += psi[j] * RC.mom[j * M + 1 + r];
#pragma unroll
      for (int k = 0; k < T; ++k)
        if (!SYM || !sym_zero_tri(k, P)) E2[k] += psi[j] * RC.mom[j * M + 1 + N + k];
    }
  } else {
  // projections in chunks of CH: all CH cell gathers are issued before any
  // hinge is evaluated, so their L1/L2 latencies overlap
  constexpr int CH = 4;
  for (int64_t j0 = 0; j0 < R.nproj; j0 += CH) {
    double dist[CH];
    bool o[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int64_t j = (j0 + u < R.nproj) ? j0 + u : R.nproj - 1;
      double pos[P];
#pragma unroll
      for (int r = 0; r < P; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k <= r; ++k) acc += L[r][k] * __ldg(R.proj + j * P + k);
        pos[r] = mu[r] + acc;
      }
      dist[u] = (P == 2) ? interp2_clamped(F, pos[0], pos[1], o[u])
                         : interp3<false>(F, pos[0], pos[1], pos[P - 1], o[u]);
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int64_t j = j0 + u;
      if (j >= R.nproj) break;
      if (o[u]) nout += (unsigned long long)__ldg(R.cnt + j);
      const double gap = radius_eps - dist[u];
      if (gap > 0.0) {
        const double psi = sigma_obs * gap * gap;
        const double* m = R.mom + j * M;
        e0 += psi * __ldg(m);
#pragma unroll
        for (int r = 0; r < N; ++r) E1[r] += psi * __ldg(m + 1 + r);
#pragma unroll
        for (int k = 0; k < T; ++k) E2[k] += psi * __ldg(m + 1 + N + k);
      }
    }
  }
  }
  if (nout) atomicAdd(out.oob + b, nout);

  // ---- moment-form gradients (factors.py:95-104) in the L^{-1} basis
  double Li[N][N];
  tri_inv_fast<N>(L, dinv, Li);
  bool finite = isfinite(e0);
#pragma unroll
  for (int r = 0; r < N; ++r) finite = finite && isfinite(E1[r]);
#pragma unroll
  for (int k = 0; k < T; ++k) finite = finite && isfinite(E2[k]);
  if (!finite) {
    atomicMax(out.status + b, GVP_ERR_NONFINITE);
    atomicMin(out.where + b, (int)knot);
    return;
  }
  // g_mu = L^{-T} E1
#pragma unroll
  for (int r = 0; r < N; ++r) {
    double acc = 0.0;
#pragma unroll
    for (int k = r; k < N; ++k)
      if (!SYM || k < P) acc += Li[k][r] * E1[k];
    out.g_mu.p[knot * out.g_mu.sk + b * out.g_mu.sp + r * out.g_mu.se] = acc;
  }
  // W = E2 L^{-1}  (E2 symmetric, packed)
  double W[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = c; k < N; ++k)
        if (!SYM || !sym_zero2(r, k, P)) acc += E2[r >= k ? tri_idx(r, k) : tri_idx(k, r)] * Li[k][c];
      W[r][c] = acc;
    }
  const double h0 = -0.5 * e0;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      double hp = 0.0, pp = 0.0;  // (L^{-T} W)[r][c] and P^{-1}[r][c]
#pragma unroll
      for (int k = r; k < N; ++k) {
        hp += Li[k][r] * W[k][c];
        pp += Li[k][r] * Li[k][c];
      }
      out.g_diag.p[knot * out.g_diag.sk + b * out.g_diag.sp + tri_idx(r, c) * out.g_diag.se] =
          h0 * pp + 0.5 * hp;  // packed lower
    }
  out.e_psi(b, f, 0) = e0 > 0.0 ? e0 : 0.0;  // e_psi = max(e0, 0) (factors.py:218-224)
}

// Factors whose covariance needed gaussian_sqrt's eigh root (listed by
// factor_grads_kernel): the whole factor through factor_eigh_path.
template <int N, int P>
__global__ void factor_eigh_kernel(int64_t nfac, View mean, View covs, RuleDev R, FieldDev F, double radius_eps,
                                   double sigma_obs, FactorOut out) {
  const int cnt = out.eigh_list[0];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const int64_t code = out.eigh_list[1 + t], b = code / nfac, f = code % nfac, knot = f + 1;
    FieldDev Fb = F;
    if (Fb.plan_map) Fb.corners += (int64_t)Fb.plan_map[b] * Fb.map_stride;
    double mu[N], S[N][N];
    const double* mp = mean.p + knot * mean.sk + b * mean.sp;
    const double* cp = covs.p + knot * covs.sk + b * covs.sp;
#pragma unroll
    for (int r = 0; r < N; ++r) mu[r] = mp[r * mean.se];
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) S[r][c] = cp[tri_idx(r, c) * covs.se];
    factor_eigh_path<N, P>(S, mu, R, Fb, radius_eps, sigma_obs, out, b, f, knot);
  }
}

template <int N, int P>
static int grads_impl(int nplans, int64_t K, const View& mean, const View& covs, const RuleDev& R,
                      const FieldDev& F, double re, double so, const FactorOut& out,
                      const int* active, cudaStream_t s) {
  const int64_t nfac = K - 2;
  if (nfac <= 0 || nplans == 0) return GVP_OK;
  const int tpb = 128;
  constexpr int M = 1 + N + N * (N + 1) / 2;
  const Rule* host = static_cast<const Rule*>(R.host);
  // SYM: the rule's grouped moments carry the sign symmetry of sym_zero_tri (residues at
  // the rounding level only), so the kernel skips those products
  bool sym = false;
  if (host && (int64_t)host->h_mom.size() == R.nproj * M) {
    double big = 0.0, odd = 0.0;
    for (int64_t j = 0; j < R.nproj; ++j) {
      const double* m = &host->h_mom[(size_t)(j * M)];
      for (int t = 0; t < M; ++t) big = std::max(big, std::fabs(m[t]));
      for (int r = P; r < N; ++r) odd = std::max(odd, std::fabs(m[1 + r]));
      for (int t = 0; t < N * (N + 1) / 2; ++t)
        if (sym_zero_tri(t, P)) odd = std::max(odd, std::fabs(m[1 + N + t]));
    }
    sym = odd <= 1e-15 * big;
  }
  auto go = [&](auto np_tag) {
    constexpr int NPc = decltype(np_tag)::value;
    RuleConst<(NPc > 0 ? NPc : 1), P, M> rc{};
    if (NPc > 0 && host) {
      std::memcpy(rc.proj, host->h_proj.data(), sizeof(rc.proj));
      std::memcpy(rc.mom, host->h_mom.data(), sizeof(rc.mom));
      std::memcpy(rc.cnt, host->h_cnt.data(), sizeof(rc.cnt));
    }
    auto launch = [&](auto sym_tag) {
      constexpr bool S = decltype(sym_tag)::value;
    if (nplans >= 64 && nfac <= 65535) {
      const dim3 grid((unsigned)((nplans + tpb - 1) / tpb), (unsigned)nfac);
      factor_grads_kernel<N, P, true, NPc, S><<<grid, tpb, 0, s>>>(nplans, nfac, mean, covs, R, F, re,
                                                                   so, out, active, rc);
    } else {
      const int64_t total = nfac * nplans;
      factor_grads_kernel<N, P, false, NPc, S><<<(unsigned)((total + tpb - 1) / tpb), tpb, 0, s>>>(
          nplans, nfac, mean, covs, R, F, re, so, out, active, rc);
    }
    };
    if constexpr (NPc > 0) {
      if (sym) {
        launch(std::true_type{});
        return;
      }
    }
    launch(std::false_type{});
  };
  if (out.eigh_list && out.reset_eigh && (out.phases & 1))
    GVP_CUDA(cudaMemsetAsync(out.eigh_list, 0, sizeof(int), s));
  // specialisations for the configurations of SURVEY §8d: 13 projections
  // (k_q = 3, P = 2) and 57 (k_q = 5, P = 2); anything else takes the loop
  if (out.phases & 1) {
    if (host && R.nproj == 13 && (int64_t)host->h_proj.size() == 13 * P)
      go(std::integral_constant<int, 13>{});
    else if (host && R.nproj == 57 && (int64_t)host->h_proj.size() == 57 * P)
      go(std::integral_constant<int, 57>{});
    else
      go(std::integral_constant<int, 0>{});
    GVP_CUDA(cudaGetLastError());
  }
  if (out.eigh_list && (out.phases & 2)) {  // one small grid; exits at once when no factor needed the eigh root
    factor_eigh_kernel<N, P><<<148, 64, 0, s>>>(nfac, mean, covs, R, F, re, so, out);
    GVP_CUDA(cudaGetLastError());
  }
  return GVP_OK;
}

int launch_factor_grads(int nplans, int64_t K, int n, const View& mean, const View& covs,
                        const RuleDev& R, const FieldDev& F, double re, double so,
                        const FactorOut& out, const int* active, cudaStream_t s) {
  if (F.ndim > n) {
    set_error("field dimension exceeds state dimension");
    return GVP_ERR_ARG;
  }
  if (R.P != F.ndim) {
    set_error("rule projection dim must equal the field dim");
    return GVP_ERR_ARG;
  }
#define GVP_CASE2(K_) \
  case K_:            \
    return F.ndim == 2 ? grads_impl<K_, 2>(nplans, K, mean, covs, R, F, re, so, out, active, s) \
                       : grads_impl<K_, 3>(nplans, K, mean, covs, R, F, re, so, out, active, s);
  switch (n) {
    case 2:
      return grads_impl<2, 2>(nplans, K, mean, covs, R, F, re, so, out, active, s);
    GVP_CASE2(3) GVP_CASE2(4) GVP_CASE2(5) GVP_CASE2(6) GVP_CASE2(7) GVP_CASE2(8)
    default:
      set_error("fused factor kernel supports n in 2..8");
      return GVP_ERR_UNSUPPORTED;
  }
#undef GVP_CASE2
}

}  // namespace gvp
