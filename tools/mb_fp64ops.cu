// Latency / throughput of fp64 division, sqrt, DFMA and 64-bit shuffles on one SM (clock64 cycles).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, double a, double b, int iters) {
  double x = a + threadIdx.x * 1e-3, y = b;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x / y + 1.0;
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = sqrt(x) + 1.0;
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = __fma_rn(x, y, 1.0);
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x * __drcp_rn(y) + 1.0;
  t1 = clock64(); cyc[4] = t1 - t0;
  out[threadIdx.x] = x;
}
// throughput: W warps, 8 independent chains per thread
__global__ void thr(double *out, long long *cyc, double b, int iters, int op) {
  double x[8];
  for (int q = 0; q < 8; q++) x[q] = 1.0 + q + threadIdx.x * 1e-3;
  __syncthreads();
  long long t0 = clock64();
  if (op == 0) for (int i = 0; i < iters; i++) for (int q = 0; q < 8; q++) x[q] = x[q] / b;
  else if (op == 1) for (int i = 0; i < iters; i++) for (int q = 0; q < 8; q++) x[q] = sqrt(x[q]) + b;
  else for (int i = 0; i < iters; i++) for (int q = 0; q < 8; q++) x[q] = __fma_rn(x[q], b, 1.0);
  __syncthreads();
  long long t1 = clock64();
  double s = 0; for (int q = 0; q < 8; q++) s += x[q];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double *out; long long *cyc, h[8];
  cudaMalloc(&out, 1 << 16); cudaMalloc(&cyc, 64);
  int it = 2000;
  lat<<<1, 32>>>(out, cyc, 1.5, 1.0000001, it); cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
  lat<<<1, 32>>>(out, cyc, 1.5, 1.0000001, it); cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
  printf("latency cycles: div %.1f sqrt %.1f dfma %.1f shfl64 %.1f mul*rcp %.1f\n", h[0] / (double)it,
         h[1] / (double)it, h[2] / (double)it, h[3] / (double)it, h[4] / (double)it);
  const char *nm[3] = {"div", "sqrt", "dfma"};
  for (int op = 0; op < 3; op++)
    for (int w : {1, 4, 16, 32}) {
      thr<<<1, 32 * w>>>(out, cyc, 1.0000001, 200, op);
      thr<<<1, 32 * w>>>(out, cyc, 1.0000001, 200, op);
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("throughput %s warps %2d: %.2f cycles per warp-op\n", nm[op], w, h[0] / (200.0 * 8 * w));
    }
  return 0;
}
