// band_sweep.cuh -- the block sweep kernel of the nested-dissection filter (included by solve.cu and by the
// microbenchmark tools/mb_sweep.cu).
#pragma once
#include "devutil.cuh"

namespace amgf {

// volatile shuffle / shared load: keeps the pivot broadcast ahead of the next pivot's shared-memory loads in
// the issue order (both go through the MIO pipe; a broadcast queued behind six loads waits for them)
__device__ __forceinline__ double shfl64_v(double v, int src) {
  int lo = __double2loint(v), hi = __double2hiint(v);
  asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(lo) : "r"(src));
  asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(hi) : "r"(src));
  return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double lds64_v(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// Block sweep (nested-dissection filter, filter.cu): one warp per diagonal block [p0, p0+len) of a band,
// forward (w = L_B^{-1} in, column sweep over Lcol) or backward (out = L_B^{-T} in, row sweep over Lrev),
// starting from the accumulators in[] (gathered through gather[] if given).  Same round structure, TMA ring
// and chain order as k_band_trsv; entries outside the block are zero in the band storage.
template <int R, int NB, bool FWD, bool BLOCKED, bool LOOKAHEAD = false>
__global__ void __launch_bounds__(32) k_band_sweep(const int *__restrict__ blk_p0, const int *__restrict__ blk_len,
                                                   int bw, const double *__restrict__ Lcol,
                                                   const double *__restrict__ Lrev, const double *__restrict__ dinv,
                                                   const double *__restrict__ in, const int *__restrict__ gather,
                                                   double *__restrict__ out, double *__restrict__ out_shift) {
  constexpr int Ws = 32 * R;
  constexpr unsigned CHUNK = 32u * Ws * 8u;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[NB];
  const int lane = threadIdx.x;
  pdl_launch_dependents();
  const int p0 = blk_p0[blockIdx.x], n = blk_len[blockIdx.x];
  const int F = (n + 31) / 32;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; b++) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int g) {
    if (g >= F || lane != 0) return;
    const double *src = FWD ? Lcol + (long)(p0 + 32 * g) * Ws : Lrev + (long)(p0 + n - 1 - 32 * g - 31) * Ws;
    uint64_t *br = &bar[g % NB];
    mbar_arrive_expect(br, CHUNK);
    bulk_g2s(sm + (g % NB) * 32 * Ws, src, CHUNK, br);
  };
#pragma unroll
  for (int g = 0; g < NB - 1; g++) issue(g);
  // local row index t in [0, n): forward row p0 + t, backward row p0 + n - 1 - t
  auto row = [&](int t) { return FWD ? p0 + t : p0 + n - 1 - t; };
  auto ld_in = [&](int t) -> double {
    if (t >= n) return 0.0;
    const int r = row(t);
    return gather ? in[gather[r]] : in[r];
  };
  // the factor (TMA rounds above) and 1/L_ii do not depend on the previous kernel: fetched before the wait
  double dv = (lane < n) ? dinv[row(lane)] : 0.0;
  double dq1 = (32 + lane < n) ? dinv[row(32 + lane)] : 0.0;
  pdl_wait();
  double acc[R];
#pragma unroll
  for (int s = 0; s < R; s++) acc[s] = ld_in(lane + 32 * s);
  double vq1 = ld_in(32 + lane + 32 * (R - 1));
  for (int q = 0; q < F; q++) {
    const int t0 = 32 * q;
    __syncwarp();
    fence_proxy_async();
    issue(q + NB - 1);
    const double vq2 = ld_in(t0 + 64 + lane + 32 * (R - 1));
    const double dq2 = (t0 + 64 + lane < n) ? dinv[row(t0 + 64 + lane)] : 0.0;
    mbar_wait(&bar[q % NB], (q / NB) & 1);
    // forward: column jj of the round at jj*Ws, row offset lane + 32s - jj
    // backward: row k = k1 - jj at (31 - jj)*Ws, distance lane + 32s - jj
    const double *cur = sm + (q % NB) * 32 * Ws + lane;
    double mine = 0.0;
    // element of pivot jj for accumulator slot s (forward: column jj of the round; backward: row k1 - jj)
    auto Lat = [&](int jj, int s) { return FWD ? cur[jj * (Ws - 1) + 32 * s] : cur[(31 - jj) * Ws - jj + 32 * s]; };
    if (BLOCKED) {
      // (1) the round's own 32 rows (slot 0): the pivot chain DFMA -> DMUL -> SHFL carries one FMA per
      //     pivot; (2) the rows below (slots 1..R-1) then take the round's 32 pivots in ascending order.
      //     Every row sees the same FMAs in the same order as the per-pivot form (C10).
      const int m = min(32, n - t0);
      double l0 = Lat(0, 0);
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        if (jj >= m) break;
        const double l0n = Lat((jj + 1) & 31, 0);
        const double yj = __shfl_sync(0xffffffffu, acc[0] * dv, jj);
        mine = (lane == jj) ? yj : mine;
        acc[0] = __fma_rn(-l0, yj, acc[0]);
        l0 = l0n;
      }
#ifndef AMGF_MB_TONLY  // microbenchmark switch: time the pivot triangle alone
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        if (jj >= m) break;
        const double yj = __shfl_sync(0xffffffffu, mine, jj);
#pragma unroll
        for (int s = 1; s < R; s++) acc[s] = __fma_rn(-Lat(jj, s), yj, acc[s]);
      }
#endif
    } else if (LOOKAHEAD) {
      // the next pivot's value (lane jj+1's accumulator is final once it took pivot jj) is formed and
      // broadcast right after that one FMA, so its DMUL -> SHFL latency overlaps this pivot's other R-1
      // FMAs and the next loads; across the round boundary the next pivot sits in slot 1, so the last
      // pivot of a round falls back to the plain order.  Same FMAs, same values (C10).
      double lc[R];
#pragma unroll
      for (int s = 0; s < R; s++) lc[s] = Lat(0, s);
      const int m = min(32, n - t0);
      double ycur = shfl64_v(acc[0] * dv, 0);
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        if (jj >= m) break;
        double ln[R];
        const int jn = (jj + 1) & 31;
        mine = (lane == jj) ? ycur : mine;
        acc[0] = __fma_rn(-lc[0], ycur, acc[0]);
        const double ynext = shfl64_v(acc[0] * dv, jn);
#pragma unroll
        for (int s = 0; s < R; s++)
          ln[s] = lds64_v(FWD ? cur + jn * (Ws - 1) + 32 * s : cur + (31 - jn) * Ws - jn + 32 * s);
#pragma unroll
        for (int s = 1; s < R; s++) acc[s] = __fma_rn(-lc[s], ycur, acc[s]);
#pragma unroll
        for (int s = 0; s < R; s++) lc[s] = ln[s];
        ycur = ynext;
      }
    } else {
      double lc[R];
#pragma unroll
      for (int s = 0; s < R; s++) lc[s] = Lat(0, s);
#pragma unroll
      for (int jj = 0; jj < 32; jj++) {
        if (t0 + jj >= n) break;
        double ln[R];
        const int jn = (jj + 1) & 31;
#pragma unroll
        for (int s = 0; s < R; s++) ln[s] = Lat(jn, s);
        const double yj = __shfl_sync(0xffffffffu, acc[0] * dv, jj);
        mine = (lane == jj) ? yj : mine;
#pragma unroll
        for (int s = 0; s < R; s++) acc[s] = __fma_rn(-lc[s], yj, acc[s]);
#pragma unroll
        for (int s = 0; s < R; s++) lc[s] = ln[s];
      }
    }
    if (t0 + lane < n) {
      out[row(t0 + lane)] = mine;
      if (out_shift) out_shift[row(t0 + lane) + 1] = mine;  // copy shifted by one (TMA alignment, filter.cu)
    }
#pragma unroll
    for (int s = 0; s < R - 1; s++) acc[s] = acc[s + 1];
    acc[R - 1] = vq1;
    dv = dq1;
    vq1 = vq2;
    dq1 = dq2;
  }
}


}  // namespace amgf
