// Band Cholesky microbenchmark: k_band_chol_t (and the round-1 k_band_chol) on a synthetic SPD band
// (n, bw), one block per CTA; per-panel phase clocks; bitwise check against a host left-looking C9 chain.
#define AMGF_CHOL_TRACE
#include "../paper_2505_18576_b200/csrc/setup.cu"
#include <cmath>
#include <cstring>
using namespace amgf;
int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 940, bw = argc > 2 ? atoi(argv[2]) : 133, nblk = argc > 3 ? atoi(argv[3]) : 8;
  const int W = band_stride(bw);
  std::vector<double> A((size_t)n * W, 0.0);
  unsigned long long s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return ((s >> 11) * 0x1.0p-53) - 0.5; };
  for (int i = 0; i < n; i++)
    for (int k = std::max(0, i - bw); k <= i; k++) A[(size_t)i * W + bw - (i - k)] = (k == i) ? 2.0 * bw : rnd();
  // host reference: dense-definition left-looking chains (C9), band-limited
  std::vector<double> L = A;
  auto at = [&](int i, int k) -> double & { return L[(size_t)i * W + bw - (i - k)]; };
  for (int j = 0; j < n; j++) {
    for (int i = j; i < std::min(n, j + bw + 1); i++) {
      double acc = at(i, j);
      for (int k = std::max(0, i - bw); k < j; k++) acc = std::fma(-at(i, k), at(j, k), acc);
      if (i == j) at(j, j) = std::sqrt(acc);
      else at(i, j) = acc / at(j, j);
    }
  }
  const size_t tot = (size_t)(n * nblk + 2 * BAND_PAD_ROWS) * W;
  double *d; int *err, *p0, *len; long long *tr;
  cudaMalloc(&d, tot * 8); cudaMalloc(&err, 8); cudaMalloc(&p0, 4 * nblk); cudaMalloc(&len, 4 * nblk);
  cudaMalloc(&tr, 8 * 4 * 128 * nblk);
  std::vector<int> hp(nblk), hl(nblk, n);
  for (int b = 0; b < nblk; b++) hp[b] = b * n;
  cudaMemcpy(p0, hp.data(), 4 * nblk, cudaMemcpyHostToDevice); cudaMemcpy(len, hl.data(), 4 * nblk, cudaMemcpyHostToDevice);
  double *Lr = d + (size_t)BAND_PAD_ROWS * W;
  cudaMemcpyToSymbol(g_chol_trace, &tr, sizeof(tr));
  const int rows = 32 + bw, r4 = (rows + 3) & ~3, ldk = r4 + (r4 % 8 == 0 ? 4 : 0);
  const size_t smem_t = (64 * (size_t)ldk + (size_t)rows * PLD) * sizeof(double);
  cudaFuncSetAttribute(k_band_chol_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
  const size_t smem_o = (2 * (size_t)(32 + bw) * PLD + 32 * (size_t)(33 + bw)) * sizeof(double);
  cudaFuncSetAttribute(k_band_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_o);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int which = 0; which < 2; which++) {
    for (int rep = 0; rep < 3; rep++) {
      cudaMemset(d, 0, tot * 8); cudaMemset(err, 0, 8);
      for (int b = 0; b < nblk; b++) cudaMemcpy(Lr + (size_t)b * n * W, A.data(), (size_t)n * W * 8, cudaMemcpyHostToDevice);
      cudaEventRecord(e0);
      if (which == 0) k_band_chol_t<<<nblk, CHT_THREADS, smem_t>>>(n, p0, len, bw, W, Lr, err, 1);
      else k_band_chol<<<nblk, CHOL_THREADS, smem_o>>>(n, p0, len, bw, W, Lr, err, 1);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t ce = cudaGetLastError();
      std::vector<double> h((size_t)n * W);
      cudaMemcpy(h.data(), Lr, (size_t)n * W * 8, cudaMemcpyDeviceToHost);
      long bad = 0;
      for (int i = 0; i < n; i++)
        for (int k = std::max(0, i - bw); k <= i; k++) {
          const size_t q = (size_t)i * W + bw - (i - k);
          if (h[q] != L[q]) bad++;
        }
      printf("%s n=%d bw=%d blocks=%d: %.1f us, mismatches %ld, %s\n", which ? "k_band_chol  " : "k_band_chol_t", n, bw,
             nblk, ms * 1e3, bad, cudaGetErrorString(ce));
      if (which == 0 && rep == 2) {
        std::vector<long long> t(4 * 128);
        cudaMemcpy(t.data(), tr, 8 * 4 * 128, cudaMemcpyDeviceToHost);
        double ph[3] = {0, 0, 0};
        const int np = (n + 31) / 32;
        for (int p = 0; p < np; p++)
          for (int k = 0; k < 3; k++) ph[k] += t[p * 4 + k + 1] - t[p * 4 + k];
        printf("  per panel cycles: phase A %.0f, B1 %.0f, B2 %.0f (panels %d)\n", ph[0] / np, ph[1] / np, ph[2] / np, np);
      }
    }
  }
  return 0;
}
