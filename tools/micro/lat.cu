// Dependent-chain latency microbenchmark (cycles per op) for fp64 on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = out[0];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_rsqrt(double* out, int n, long long* cyc) {
  double x = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = rsqrt(x) + 1.5; }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_log(double* out, int n, long long* cyc) {
  double x = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = log(x) + 2.5; }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_div(double* out, int n, long long* cyc) {
  double x = out[0] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = 1.0 / x + 1.5; }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void k_sync(double* out, int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread, many warps
__global__ void k_tput(double* out, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 24); cudaMalloc(&c, 64);
  cudaMemset(d, 0, 1 << 24);
  long long h; int n = 100000;
  k_dfma<<<1, 1>>>(d, 0.999, 0.001, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (4.0 * n));
  k_rsqrt<<<1, 1>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt(double)+add dependent latency: %.2f cycles\n", (double)h / n);
  k_log<<<1, 1>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("log(double)+add dependent latency: %.2f cycles\n", (double)h / n);
  k_div<<<1, 1>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("1/x (double)+add dependent latency: %.2f cycles\n", (double)h / n);
  k_sync<<<1, 64>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (64 thr): %.2f cycles\n", (double)h / n);
  k_sync<<<1, 128>>>(d, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (128 thr): %.2f cycles\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int m = 20000;
  k_tput<<<148 * 8, 256>>>(d, 0.999, 0.001, m);
  cudaEventRecord(e0); k_tput<<<148 * 8, 256>>>(d, 0.999, 0.001, m); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * m * 148.0 * 8 * 256;
  printf("DFMA throughput: %.2f TFLOP/s\n", fl / ms / 1e9);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock rate attr %d kHz\n", clk);
  return 0;
}
