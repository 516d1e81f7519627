// Microbenchmark of the separator forward-dot kernel (nd_kernels.cuh) on a synthetic top separator of cfg 3:
// 133 rows, subtree of 8,317 columns.  Prints microseconds per launch (L2 flushed before each) and cycles per
// chain term.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 tools/mb_sepfwd.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2505_18576_b200/csrc/devutil.cuh"
#include "../paper_2505_18576_b200/csrc/nd_kernels.cuh"
using namespace amgf;

template <int G, int NS>
float run(const NdBlk *blk, int len, const double *Loff, const double *r1, const double *w, const double *w2,
          double *acc, double *junk, size_t junk_n) {
  std::vector<int> gr;
  for (int r0 = 0; r0 < len; r0 += G) { gr.push_back(0); gr.push_back(r0); }
  int *dg;
  cudaMalloc(&dg, gr.size() * 4);
  cudaMemcpy(dg, gr.data(), gr.size() * 4, cudaMemcpyHostToDevice);
  const int ng = (int)gr.size() / 2;
  const size_t smem = sf_smem(G, NS, SF_KC);
  cudaFuncSetAttribute(k_nd_sep_fwd<G, NS, SF_KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  for (int it = 0; it < 12; it++) {
    cudaMemsetAsync(junk, it, junk_n * 8);
    cudaEventRecord(a);
    k_nd_sep_fwd<G, NS, SF_KC><<<ng, 32, smem>>>((const int2 *)dg, blk, Loff, r1, nullptr, w, w2, acc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 2) tot += ms;
  }
  cudaFree(dg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return tot / 10 * 1e3f;
}


// experimental variant: KC-column chunks, explicit 8-term register pipeline inside a chunk
template <int G, int NS, int KC>
__global__ void __launch_bounds__(32) k_sf2(const int2 *groups, const NdBlk *blk, const double *Loff,
                                           const double *r1, const double *w, const double *w2, double *accbuf) {
  constexpr int LD = KC + 2;
  extern __shared__ __align__(16) double sfm[];
  const NdBlk S = blk[groups[blockIdx.x].x];
  const int row0 = groups[blockIdx.x].y;
  const int lane = threadIdx.x;
  const int nrow = min(G, S.len - row0);
  const int ncol = S.p0 - S.t0;
  const int nch = (ncol + KC - 1) / KC;
  double *sW = sfm + NS * G * LD;
  const double *wsrc = (S.t0 & 1) ? w2 + S.t0 + 1 : w + S.t0;
  const double *Lq = Loff + S.off + (long)row0 * S.rs;
  auto issue = [&](int c) {
    if (c < nch) {
      const int k0 = c * KC, st = c % NS;
      for (int p = lane; p < KC / 2; p += 32) {
        if (2 * p < ncol - k0) {
          double *dst = sfm + st * G * LD + 2 * p;
          for (int r = 0; r < nrow; r++) cp_async16(dst + r * LD, Lq + (long)r * S.rs + k0 + 2 * p);
        }
        cp_async16(sW + st * KC + 2 * p, wsrc + k0 + 2 * p);
      }
    }
    asm volatile("cp.async.commit_group;");
  };
#pragma unroll
  for (int c = 0; c < NS - 1; c++) issue(c);
  double acc = (lane < nrow) ? r1[S.p0 + row0 + lane] : 0.0;
  const int me = min(lane, G - 1);
  for (int c = 0; c < nch; c++) {
    issue(c + NS - 1);
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 1));
    __syncwarp();
    const int st = c % NS;
    const double2 *buf = (const double2 *)(sfm + st * G * LD + me * LD);
    const double2 *wb = (const double2 *)(sW + st * KC);
    const int kn = min(KC, ncol - c * KC);
    if (kn == KC) {
      double2 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; u++) { a[u] = buf[u]; b[u] = wb[u]; }
#pragma unroll
      for (int t = 0; t < KC / 2; t += 4) {
        double2 an[4], bn[4];
        if (t + 4 < KC / 2) {
#pragma unroll
          for (int u = 0; u < 4; u++) { an[u] = buf[t + 4 + u]; bn[u] = wb[t + 4 + u]; }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          acc = __fma_rn(-a[u].x, b[u].x, acc);
          acc = __fma_rn(-a[u].y, b[u].y, acc);
        }
#pragma unroll
        for (int u = 0; u < 4; u++) { a[u] = an[u]; b[u] = bn[u]; }
      }
    } else {
      const double *bs = (const double *)buf, *ws = (const double *)wb;
      for (int kk = 0; kk < kn; kk++) acc = __fma_rn(-bs[kk], ws[kk], acc);
    }
    __syncwarp();
  }
  asm volatile("cp.async.wait_group 0;");
  if (lane < nrow) accbuf[S.p0 + row0 + lane] = acc;
}

template <int G, int NS, int KC>
float run2(const NdBlk *blk, int len, const double *Loff, const double *r1, const double *w, const double *w2,
           double *acc, double *junk, size_t junk_n) {
  std::vector<int> gr;
  for (int r0 = 0; r0 < len; r0 += G) { gr.push_back(0); gr.push_back(r0); }
  int *dg;
  cudaMalloc(&dg, gr.size() * 4);
  cudaMemcpy(dg, gr.data(), gr.size() * 4, cudaMemcpyHostToDevice);
  const int ng = (int)gr.size() / 2;
  const size_t smem = (size_t)NS * (G * (KC + 2) + KC) * 8;
  cudaFuncSetAttribute(k_sf2<G, NS, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float tot = 0;
  for (int it = 0; it < 12; it++) {
    cudaMemsetAsync(junk, it, junk_n * 8);
    cudaEventRecord(a);
    k_sf2<G, NS, KC><<<ng, 32, smem>>>((const int2 *)dg, blk, Loff, r1, w, w2, acc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (it >= 2) tot += ms;
  }
  cudaFree(dg);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return tot / 10 * 1e3f;
}

__global__ void k_chain(const double *v, double *out, int n) {
  double a[8], b[8];
#pragma unroll
  for (int u = 0; u < 8; u++) { a[u] = v[u]; b[u] = v[8 + u]; }
  double acc = v[16];
  for (int k = 0; k < n; k += 8)
#pragma unroll
    for (int u = 0; u < 8; u++) acc = __fma_rn(-a[u], b[u], acc);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
  const int len = 133, ncol = 8317, rs = (ncol + 1) & ~1;
  NdBlk h{};
  h.p0 = ncol; h.len = len; h.kind = 1; h.t0 = 0; h.off = 0; h.level = 0; h.rs = rs;
  NdBlk *blk;
  cudaMalloc(&blk, sizeof(NdBlk));
  cudaMemcpy(blk, &h, sizeof(NdBlk), cudaMemcpyHostToDevice);
  std::vector<double> L((size_t)len * rs, 1e-3), wv(ncol + 80, 0.5);
  double *Loff, *w, *w2, *r1, *acc, *junk;
  const size_t junk_n = 64ull << 20;
  cudaMalloc(&Loff, L.size() * 8);
  cudaMalloc(&w, wv.size() * 8);
  cudaMalloc(&w2, wv.size() * 8);
  cudaMalloc(&r1, (ncol + len) * 8);
  cudaMalloc(&acc, (ncol + len) * 8);
  cudaMalloc(&junk, junk_n * 8);
  cudaMemcpy(Loff, L.data(), L.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(w, wv.data(), wv.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(w2, wv.data(), wv.size() * 8, cudaMemcpyHostToDevice);
  cudaMemset(r1, 0, (ncol + len) * 8);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto rep = [&](const char *name, float us) {
    printf("%-22s %8.1f us  %6.2f cycles/term\n", name, us, us * 1e-6 * clk * 1e3 / ncol);
  };
  {
    double *v, *o;
    cudaMalloc(&v, 64 * 8);
    cudaMalloc(&o, 64 * 8);
    cudaMemset(v, 0, 64 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_chain<<<1, 32>>>(v, o, 8320);
    cudaEventRecord(a);
    for (int i = 0; i < 10; i++) k_chain<<<1, 32>>>(v, o, 8320 * 8);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("pure register DFMA chain: %.2f cycles/term\n", ms / 10 * 1e-3 * clk * 1e3 / (8320 * 8));
  }
  rep("library G=1 NS=6", run<1, 6>(blk, len, Loff, r1, w, w2, acc, junk, junk_n));
  rep("library G=4 NS=4", run<4, 4>(blk, len, Loff, r1, w, w2, acc, junk, junk_n));
  rep("v2 G=1 NS=6 KC=512", run2<1, 6, 512>(blk, len, Loff, r1, w, w2, acc, junk, junk_n));
  cudaDeviceSynchronize();
  return 0;
}
