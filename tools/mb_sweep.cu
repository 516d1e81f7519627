// Microbenchmark of the filter block sweep (band_sweep.cuh) on a synthetic band: 8 blocks of 940 rows,
// bw 133 (cfg 3's leaves).  Prints microseconds per launch, L2-warm and after an L2 flush, and cycles per
// pivot.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 tools/mb_sweep.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2505_18576_b200/csrc/band_sweep.cuh"
using namespace amgf;

#define CKK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int R, int NB, bool FWD, bool BLK, bool LA = false>
float run(int nb, const int *p0, const int *len, int bw, const double *Lc, const double *Lr, const double *dv,
          const double *in, double *out, bool flush, double *junk, size_t junk_n) {
  const size_t smem = (size_t)NB * 32 * (32 * R) * sizeof(double);
  cudaFuncSetAttribute(k_band_sweep<R, NB, FWD, BLK, LA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  for (int it = 0; it < 12; it++) {
    if (flush) cudaMemsetAsync(junk, it, junk_n * 8);
    cudaEventRecord(a);
    k_band_sweep<R, NB, FWD, BLK, LA><<<nb, 32, smem>>>(p0, len, bw, Lc, Lr, dv, in, nullptr, out, nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 2) tot += ms;
  }
  return tot / 10 * 1e3f;
}

__global__ void k_pivchain(const double *v, double *out, int n) {
  double acc = v[threadIdx.x], d = v[32 + threadIdx.x], l = v[64 + threadIdx.x];
  for (int k = 0; k < n; k += 32) {
#pragma unroll
    for (int j = 0; j < 32; j++) {
      const double y = __shfl_sync(0xffffffffu, acc * d, j);
      acc = __fma_rn(-l, y, acc);
    }
  }
  out[threadIdx.x] = acc;
}
__global__ void k_pivchain_smem(const double *v, double *out, int n) {
  __shared__ double sy[32];
  double acc = v[threadIdx.x], d = v[32 + threadIdx.x], l = v[64 + threadIdx.x];
  for (int k = 0; k < n; k += 32) {
#pragma unroll
    for (int j = 0; j < 32; j++) {
      if (threadIdx.x == j) sy[j] = acc * d;
      __syncwarp();
      const double y = sy[j];
      acc = __fma_rn(-l, y, acc);
    }
  }
  out[threadIdx.x] = acc;
}
__global__ void k_chain2(const double *v, double *out, int n) {
  double acc = v[threadIdx.x], d = v[32 + threadIdx.x], l = v[64 + threadIdx.x];
  for (int k = 0; k < n; k++) {
    const double y = acc * d;
    acc = __fma_rn(-l, y, acc);
  }
  out[threadIdx.x] = acc;
}

template <int NF, int NL>
__global__ void k_pivmix(const double *v, double *out, int n) {
  __shared__ double sm[32 * 192];
  for (int i = threadIdx.x; i < 32 * 192; i += 32) sm[i] = v[i & 127];
  __syncwarp();
  double acc = v[threadIdx.x], d = v[32 + threadIdx.x];
  double a2[8], lc[8];
#pragma unroll
  for (int u = 0; u < 8; u++) { a2[u] = v[u]; lc[u] = v[8 + u]; }
  for (int k = 0; k < n; k += 32) {
#pragma unroll
    for (int j = 0; j < 32; j++) {
      double ln[8];
#pragma unroll
      for (int u = 0; u < NL; u++) ln[u] = sm[((j + 1) & 31) * 191 + 32 * u + threadIdx.x];
      const double y = __shfl_sync(0xffffffffu, acc * d, j);
      acc = __fma_rn(-lc[0], y, acc);
#pragma unroll
      for (int u = 0; u < NF; u++) a2[u] = __fma_rn(-lc[u + 1], y, a2[u]);
#pragma unroll
      for (int u = 0; u < NL; u++) lc[u] = ln[u];
    }
  }
  double t = acc;
#pragma unroll
  for (int u = 0; u < 8; u++) t += a2[u];
  out[threadIdx.x] = t;
}
template <int NF, int NL>
void mix(const double *v, double *o, int clk) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int N = 32 * 4096;
  float ms;
  k_pivmix<NF, NL><<<1, 32>>>(v, o, 32);
  cudaEventRecord(a); k_pivmix<NF, NL><<<1, 32>>>(v, o, N); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("chain + %d DFMA + %d LDS: %.1f cycles/step\n", NF, NL, ms * 1e-3 * clk * 1e3 / N);
}

int main() {
  const int nb = 8, L = 940, bw = 133, R = 6, W = 32 * R, n = nb * L, PAD = 64;
  std::vector<double> h((size_t)(n + 2 * PAD) * W, 0.0);
  for (int j = 0; j < n; j++)
    for (int t = 0; t <= bw && j + t < n; t++) h[(size_t)(j + PAD) * W + t] = (t == 0) ? 1.0 : 1e-3 / (1 + t);
  double *Lc, *Lr, *dv, *in, *out, *junk;
  const size_t junk_n = 64ull << 20;
  CKK(cudaMalloc(&Lc, h.size() * 8));
  CKK(cudaMalloc(&Lr, h.size() * 8));
  CKK(cudaMalloc(&dv, n * 8));
  CKK(cudaMalloc(&in, n * 8));
  CKK(cudaMalloc(&out, n * 8));
  CKK(cudaMalloc(&junk, junk_n * 8));
  CKK(cudaMemcpy(Lc, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  CKK(cudaMemcpy(Lr, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
  std::vector<double> one(n, 1.0);
  CKK(cudaMemcpy(dv, one.data(), n * 8, cudaMemcpyHostToDevice));
  CKK(cudaMemcpy(in, one.data(), n * 8, cudaMemcpyHostToDevice));
  std::vector<int> hp(nb), hl(nb, L);
  for (int i = 0; i < nb; i++) hp[i] = i * L;
  int *p0, *len;
  CKK(cudaMalloc(&p0, nb * 4));
  CKK(cudaMalloc(&len, nb * 4));
  CKK(cudaMemcpy(p0, hp.data(), nb * 4, cudaMemcpyHostToDevice));
  CKK(cudaMemcpy(len, hl.data(), nb * 4, cudaMemcpyHostToDevice));
  const double *Lcp = Lc + (size_t)PAD * W, *Lrp = Lr + (size_t)PAD * W;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto rep = [&](const char *name, float us) {
    printf("%-28s %8.1f us  %6.1f cycles/pivot (at %d MHz)\n", name, us, us * 1e-6 * clk * 1e3 / L, clk / 1000);
  };
  {
    double *v, *o;
    cudaMalloc(&v, 128 * 8);
    cudaMalloc(&o, 128 * 8);
    cudaMemset(v, 0, 128 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int N = 32 * 4096;
    float ms;
    k_pivchain<<<1, 32>>>(v, o, 32);
    cudaEventRecord(a); k_pivchain<<<1, 32>>>(v, o, N); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DMUL->SHFL64->DFMA chain: %.1f cycles/step\n", ms * 1e-3 * clk * 1e3 / N);
    k_pivchain_smem<<<1, 32>>>(v, o, 32);
    cudaEventRecord(a); k_pivchain_smem<<<1, 32>>>(v, o, N); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DMUL->STS/syncwarp/LDS->DFMA chain: %.1f cycles/step\n", ms * 1e-3 * clk * 1e3 / N);
    k_chain2<<<1, 32>>>(v, o, 32);
    cudaEventRecord(a); k_chain2<<<1, 32>>>(v, o, N); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("DMUL->DFMA chain: %.1f cycles/step\n", ms * 1e-3 * clk * 1e3 / N);
  }
  {
    double *v, *o;
    cudaMalloc(&v, 128 * 8);
    cudaMalloc(&o, 128 * 8);
    cudaMemset(v, 0, 128 * 8);
    mix<0, 0>(v, o, clk);
    mix<5, 0>(v, o, clk);
    mix<0, 6>(v, o, clk);
    mix<5, 6>(v, o, clk);
    mix<5, 3>(v, o, clk);
  }
  rep("fwd pivotwise warm", run<R, 4, true, false>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  rep("fwd pivotwise flushed", run<R, 4, true, false>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, true, junk, junk_n));
  rep("fwd lookahead warm", run<R, 4, true, false, true>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  rep("bwd lookahead warm", run<R, 4, false, false, true>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  rep("fwd blocked warm", run<R, 4, true, true>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  rep("fwd blocked flushed", run<R, 4, true, true>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, true, junk, junk_n));
  rep("bwd pivotwise warm", run<R, 4, false, false>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  rep("bwd blocked warm", run<R, 4, false, true>(nb, p0, len, bw, Lcp, Lrp, dv, in, out, false, junk, junk_n));
  CKK(cudaDeviceSynchronize());
  return 0;
}
