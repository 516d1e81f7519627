// Latency microbenchmarks (one warp): dependent chains of DFMA, DMUL, SHFL(double), and the TRSV step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int iters) {
  int lane = threadIdx.x;
  double x = a + lane, y = b;
  long long t0, t1;
  // 1: DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = __fma_rn(x, y, 1e-300);
  t1 = clock64(); cyc[0] = t1 - t0;
  // 2: DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x * y;
  t1 = clock64(); cyc[1] = t1 - t0;
  // 3: SHFL chain (double)
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = __shfl_sync(0xffffffffu, x, (i + 1) & 31);
  t1 = clock64(); cyc[2] = t1 - t0;
  // 4: step = DMUL -> SHFL -> DFMA
  double acc = x;
  t0 = clock64();
  for (int i = 0; i < iters; i++) {
    double t = __shfl_sync(0xffffffffu, acc * y, i & 31);
    acc = __fma_rn(-a, t, acc);
  }
  t1 = clock64(); cyc[3] = t1 - t0;
  // 5: SHFL chain (int)
  int xi = lane;
  t0 = clock64();
  for (int i = 0; i < iters; i++) xi = __shfl_sync(0xffffffffu, xi, (xi + 1) & 31);
  t1 = clock64(); cyc[4] = t1 - t0;
  // 6: DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = x + y;
  t1 = clock64(); cyc[5] = t1 - t0;
  // 7: FFMA chain (fp32)
  float f = a;
  t0 = clock64();
  for (int i = 0; i < iters; i++) f = __fmaf_rn(f, (float)b, 1e-30f);
  t1 = clock64(); cyc[6] = t1 - t0;
  // 8: DFMA throughput: 8 independent chains
  double c0 = x, c1 = x + 1, c2 = x + 2, c3 = x + 3, c4 = x + 4, c5 = x + 5, c6 = x + 6, c7 = x + 7;
  t0 = clock64();
  for (int i = 0; i < iters; i++) {
    c0 = __fma_rn(c0, y, 1e-300); c1 = __fma_rn(c1, y, 1e-300); c2 = __fma_rn(c2, y, 1e-300); c3 = __fma_rn(c3, y, 1e-300);
    c4 = __fma_rn(c4, y, 1e-300); c5 = __fma_rn(c5, y, 1e-300); c6 = __fma_rn(c6, y, 1e-300); c7 = __fma_rn(c7, y, 1e-300);
  }
  t1 = clock64(); cyc[7] = t1 - t0;
  out[lane] = x + acc + xi + f + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}
int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 32 * 8); cudaMallocManaged(&cyc, 8 * 8);
  int iters = 4096;
  for (int rep = 0; rep < 2; rep++) {
    k<<<1, 32>>>(out, cyc, 1.0000001, 0.9999999, iters);
    cudaDeviceSynchronize();
  }
  const char *names[] = {"DFMA chain", "DMUL chain", "SHFL f64 chain", "DMUL->SHFL->DFMA step", "SHFL i32 chain",
                         "DADD chain", "FFMA chain", "DFMA x8 indep (per iter)"};
  for (int i = 0; i < 8; i++) printf("%-28s %7.2f cycles/iter\n", names[i], (double)cyc[i] / iters);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
