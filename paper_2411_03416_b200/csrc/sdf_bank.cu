// Signed-distance maps on the device: rasterisation of
// primitive unions (sdf.py:134-185) and the corner-packed map bank the factor
// kernel reads through a per-plan map index.
//
// rasterize_kernel reproduces the reference's numpy evaluation bit for bit:
// grid coordinates origin + cell * k, Disc = |p - c| - r with the norm as
// sqrt of the in-order sum of squares, Box = |max(q, 0)| + min(max_k q_k, 0)
// with q = |p - c| - h, the union as the minimum over primitives in order —
// every product/sum explicitly rounded (no FMA contraction), sqrt correctly
// rounded on both sides.
#include <cuda_runtime.h>

#include <vector>

#include "gvp_internal.cuh"

namespace gvp {

namespace {
constexpr double kEmptyField = 1e6;  // sdf.py _EMPTY_FIELD_VALUE

__global__ void rasterize_kernel(int dim, int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                                 double cell, int nmaps, const int* __restrict__ prim_off,
                                 const int* __restrict__ kinds, const double* __restrict__ params,
                                 double* __restrict__ out) {
  const int64_t cells = nx * ny * nz;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cells * nmaps) return;
  const int m = (int)(t / cells);
  const int64_t c = t % cells, ix = c % nx, iy = (c / nx) % ny, iz = c / (nx * ny);
  double p[3];
  p[0] = __dadd_rn(ox, __dmul_rn(cell, (double)ix));
  p[1] = __dadd_rn(oy, __dmul_rn(cell, (double)iy));
  p[2] = __dadd_rn(oz, __dmul_rn(cell, (double)iz));
  const int a0 = prim_off[m], a1 = prim_off[m + 1];
  double best = kEmptyField;
  for (int k = a0; k < a1; ++k) {
    const double* pr = params + (int64_t)k * 2 * dim;
    double d;
    if (kinds[k] == 0) {  // Disc / sphere: norm(p - c) - r
      double ss = 0.0;
      for (int j = 0; j < dim; ++j) {
        const double q = __dsub_rn(p[j], pr[j]);
        ss = __dadd_rn(ss, __dmul_rn(q, q));
      }
      d = __dsub_rn(__dsqrt_rn(ss), pr[dim]);
    } else {  // Box: norm(max(q, 0)) + min(max(q), 0), q = |p - c| - h
      double ss = 0.0, qmax = -INFINITY;
      for (int j = 0; j < dim; ++j) {
        const double q = __dsub_rn(fabs(__dsub_rn(p[j], pr[j])), pr[dim + j]);
        const double qp = fmax(q, 0.0);
        ss = __dadd_rn(ss, __dmul_rn(qp, qp));
        qmax = fmax(qmax, q);
      }
      d = __dadd_rn(__dsqrt_rn(ss), fmin(qmax, 0.0));
    }
    best = (k == a0) ? d : fmin(best, d);
  }
  out[t] = best;
}

__global__ void pack2_kernel(int64_t nx, int64_t ny, int nmaps, int64_t stride, const double* __restrict__ raw,
                             double* __restrict__ dst) {
  const int64_t cx = nx - 1, cy = ny - 1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cx * cy * nmaps) return;
  const int m = (int)(t / (cx * cy));
  const int64_t c = t % (cx * cy), ix = c % cx, iy = c / cx;
  const double* g = raw + (int64_t)m * nx * ny + iy * nx + ix;
  double* o = dst + (int64_t)m * stride + c * 4;
  o[0] = g[0];
  o[1] = g[1];
  o[2] = g[nx];
  o[3] = g[nx + 1];
}

__global__ void pack3_kernel(int64_t nx, int64_t ny, int64_t nz, int nmaps, int64_t stride,
                             const double* __restrict__ raw, double* __restrict__ dst) {
  const int64_t cx = nx - 1;
  const int64_t rows = ny * nz;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cx * rows * nmaps) return;
  const int m = (int)(t / (cx * rows));
  const int64_t c = t % (cx * rows), ix = c % cx, row = c / cx;
  const double* g = raw + (int64_t)m * nx * rows + row * nx + ix;
  double* o = dst + (int64_t)m * stride + c * 2;
  o[0] = g[0];
  o[1] = g[1];
}
}  // namespace

int64_t packed_field_doubles(const FieldDev& f) {
  return f.ndim == 2 ? (f.ny - 1) * (f.nx - 1) * 4 : f.nz * f.ny * (f.nx - 1) * 2;
}

int pack_field_maps(const FieldDev& f, int nmaps, const double* raw, double* dst, cudaStream_t s) {
  const int64_t stride = packed_field_doubles(f);
  const int tb = 256;
  if (f.ndim == 2) {
    const int64_t n = (f.nx - 1) * (f.ny - 1) * nmaps;
    pack2_kernel<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(f.nx, f.ny, nmaps, stride, raw, dst);
  } else {
    const int64_t n = (f.nx - 1) * f.ny * f.nz * nmaps;
    pack3_kernel<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(f.nx, f.ny, f.nz, nmaps, stride, raw, dst);
  }
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

int rasterize_maps(int dim, const int64_t* counts, const double* origin, double cell, int nmaps,
                   const int* prim_off, const int* kinds, const double* params, double* raw, cudaStream_t s) {
  if (dim != 2 && dim != 3) {
    set_error("rasterize: 2 or 3 axes");
    return GVP_ERR_ARG;
  }
  const int64_t nx = counts[0], ny = counts[1], nz = dim == 3 ? counts[2] : 1;
  const int64_t n = nx * ny * nz * nmaps;
  const int tb = 256;
  rasterize_kernel<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(dim, nx, ny, nz, origin[0], origin[1],
                                                                dim == 3 ? origin[2] : 0.0, cell, nmaps,
                                                                prim_off, kinds, params, raw);
  GVP_CUDA(cudaGetLastError());
  return GVP_OK;
}

}  // namespace gvp

using namespace gvp;

// Drop-in for rasterize (sdf.py:156-185): counts per axis (x, y[, z]) as the
// reference derives them from bounds; primitives as (kind, center, radius |
// halfextents). out: row-major values (ny, nx) or (nz, ny, nx), host memory.
extern "C" int gvp_rasterize(int32_t dim, const int64_t* counts, const double* origin, double cell_size,
                             int32_t nprim, const int32_t* kinds, const double* params, double* out) {
  if ((dim != 2 && dim != 3) || !counts || !origin || !(cell_size > 0) || nprim < 0 || !out ||
      (nprim > 0 && (!kinds || !params)))
    return GVP_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    set_error("no CUDA device visible");
    return GVP_ERR_NO_DEVICE;
  }
  const int64_t cells = counts[0] * counts[1] * (dim == 3 ? counts[2] : 1);
  int *d_off = nullptr, *d_kind = nullptr;
  double *d_par = nullptr, *d_out = nullptr;
  const int off[2] = {0, nprim};
  auto cleanup = [&]() {
    cudaFree(d_off);
    cudaFree(d_kind);
    cudaFree(d_par);
    cudaFree(d_out);
  };
  if (cudaMalloc(&d_off, sizeof(off)) != cudaSuccess || cudaMalloc(&d_kind, sizeof(int) * (nprim + 1)) != cudaSuccess ||
      cudaMalloc(&d_par, sizeof(double) * (2 * dim * nprim + 1)) != cudaSuccess ||
      cudaMalloc(&d_out, sizeof(double) * cells) != cudaSuccess) {
    cleanup();
    set_error("cudaMalloc failed");
    return GVP_ERR_CUDA;
  }
  cudaMemcpy(d_off, off, sizeof(off), cudaMemcpyHostToDevice);
  if (nprim) {
    cudaMemcpy(d_kind, kinds, sizeof(int) * nprim, cudaMemcpyHostToDevice);
    cudaMemcpy(d_par, params, sizeof(double) * 2 * dim * nprim, cudaMemcpyHostToDevice);
  }
  int r = rasterize_maps(dim, counts, origin, cell_size, 1, d_off, d_kind, d_par, d_out, 0);
  if (!r && cudaMemcpy(out, d_out, sizeof(double) * cells, cudaMemcpyDeviceToHost) != cudaSuccess) {
    set_error("copy back failed");
    r = GVP_ERR_CUDA;
  }
  cleanup();
  return r;
}
