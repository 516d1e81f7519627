// tail.cu -- the coarse end of the V-cycle (level t = nlev-2 and the coarsest level) as ONE kernel on one
// thread-block cluster (<= 16 CTAs, distributed over SMs of a GPC), cluster barriers between the steps.
//
// At cfg 3 the levels below level 1 are 948 + 12 dofs: the separate launches (jacobi, residual SpMV,
// restriction, coarsest TRSV, prolongation, smoothing) are each 3-17 us of latency for ~2 MB of data.
// Here each CTA first stages its SELL slices of A_t into shared memory (one TMA bulk copy), so every
// row chain then runs from shared memory; vectors go through L2 (ld.cg / st.cg) between barriers.
//
// Arithmetic: every step is the same chain, in the same order, as the separate kernels it replaces
// (DESIGN.md section 3): jacobi0 x = b/d; SELL row chain acc = fma(a, x, acc) over slots then the 6
// block components (C2); smoothing x + (b - acc)/d; restriction lane-strided chains over blocks and
// the xor butterfly (C5); coarsest forward/backward substitution y_j = acc_j * dinv_j, acc_i =
// fma(-L_ij, y_j, acc_i) ascending j / descending k (C10); prolongation x + acc.  The result is
// bitwise identical to vcycle(c, t, ...) (tests/test_gpu_parity.py runs both).
#include <cooperative_groups.h>

#include <stdio.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "devutil.cuh"

namespace amgf {
namespace cg = cooperative_groups;

constexpr int TAIL_THREADS = 256;
constexpr int TAIL_MAX_CTA = 16;
constexpr int TAIL_MAX_NCO = 64;

struct TailArgs {
  int n, pre, post;
  const int *cta_s;                                   // [ncta+1] SELL slice range of each CTA
  const int *a_sp, *a_len, *a_col;                    // A_t (SELL-32, 1 x 6 rows)
  const double *a_val;
  const int *p_sp, *p_len, *p_col;                    // P_t (SELL-32, 1 x 6 rows)
  const double *p_val;
  int r_nbr;                                          // R_t (BSR 6 x 6)
  const int *r_ptr, *r_col;
  const double *r_val;
  int nco, Wc;                                        // coarsest factor (band storage, bw = nco-1)
  const double *Lc, *dinv_c;
  const double *d, *b;                                // l1 diagonal and right-hand side of level t
  double *x, *x2, *r, *bc, *xc;                       // level t solution / second buffer / residual, coarse b, x
  int xs, maxv, maxc, maxpv, maxpc;                   // shared-memory layout (doubles / ints per array)
  unsigned long long *tm;                             // optional per-phase timestamps [ncta][16]
  int cheb, kdeg;                                     // smoother: 0 = l1-Jacobi, 1 = Chebyshev of degree kdeg
  double *dir;                                        // Chebyshev direction of level t
  double c0, ca[33], cb[33];                          // Chebyshev coefficients (C23)
};

__device__ __forceinline__ void tail_mark(const TailArgs &a, int ph) {
  if (a.tm && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tm[blockIdx.x * 16 + ph] = t;
  }
}

__device__ __forceinline__ void tail_sync(cg::cluster_group &cl) {
  __threadfence();
  cl.sync();
}

// out[i] (rows of this CTA) from the SELL chain over A_t with x staged in shared memory (C2)
// One SELL row chain (C2) from shared memory: slot q's 6 values and x entries are loaded while slot
// q-1's FMAs run, the column index two slots ahead.
__device__ __forceinline__ double tail_row(const double *sv, const int *sc, const double *xv, int base, int len,
                                           int lane) {
  double acc = 0.0;
  if (len <= 0) return acc;
  double v[6], xx[6];
  int cn = sc[base * 32 + lane];
#pragma unroll
  for (int e = 0; e < 6; e++) { v[e] = sv[(base * 6 + e) * 32 + lane]; xx[e] = xv[cn * 6 + e]; }
  cn = sc[(base + min(1, len - 1)) * 32 + lane];
  for (int q = 0; q < len; q++) {
    const int qn = base + min(q + 1, len - 1);
    double vn[6], xn[6];
#pragma unroll
    for (int e = 0; e < 6; e++) { vn[e] = sv[(qn * 6 + e) * 32 + lane]; xn[e] = xv[cn * 6 + e]; }
    cn = sc[(base + min(q + 2, len - 1)) * 32 + lane];
#pragma unroll
    for (int e = 0; e < 6; e++) acc = __fma_rn(v[e], xx[e], acc);
#pragma unroll
    for (int e = 0; e < 6; e++) { v[e] = vn[e]; xx[e] = xn[e]; }
  }
  return acc;
}

// out[i] (rows of this CTA) from the SELL chain over A_t with x staged in shared memory (C2)
template <int MODE>
__device__ __forceinline__ void tail_spmv(const TailArgs &a, int row0, int row1, int q0, const double *sx,
                                          const double *sv, const int *sc, double *out, int step = 0) {
  for (int i = row0 + threadIdx.x; i < row1; i += blockDim.x) {
    // the epilogue's vector operands are loaded before the row chain (their latency hides behind it)
    const double bi = a.b[i];
    const double di = (MODE == SPMV_RESID) ? 0.0 : a.d[i];
    const double diri = (MODE == SPMV_CHEB) ? __ldcg(a.dir + i) : 0.0;
    const double acc = tail_row(sv, sc, sx, a.a_sp[i >> 5] - q0, a.a_len[i], i & 31);
    if (MODE == SPMV_RESID) {
      __stcg(out + i, bi - acc);
    } else if (MODE == SPMV_SMOOTH) {
      const double res = bi - acc;
      const double t = res / di;
      __stcg(out + i, sx[i] + t);
    } else {  // SPMV_CHEB1 / SPMV_CHEB (C23), step s in a.ca / a.cb
      const double t = (bi - acc) / di;
      const double dv = (MODE == SPMV_CHEB1) ? a.c0 * t : __fma_rn(a.ca[step], diri, a.cb[step] * t);
      __stcg(a.dir + i, dv);
      __stcg(out + i, sx[i] + dv);
    }
  }
}

__global__ void __launch_bounds__(TAIL_THREADS) k_vcycle_tail(TailArgs a) {
  extern __shared__ __align__(128) double tsm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double ys[TAIL_MAX_NCO];
  cg::cluster_group cl = cg::this_cluster();
  const int cta = blockIdx.x, tid = threadIdx.x;
  double *sx = tsm;
  double *sv = tsm + a.xs;
  double *spv = sv + a.maxv;
  int *sc = (int *)(spv + a.maxpv);
  int *spc = sc + a.maxc;
  double *sL = (double *)(spc + a.maxpc);  // CTA 0: dense coarsest factor, row-major nco x nco
  const int s0 = a.cta_s[cta], s1 = a.cta_s[cta + 1];
  const int q0 = a.a_sp[s0], q1 = a.a_sp[s1];
  const int p0 = a.p_sp[s0], p1 = a.p_sp[s1];
  const int row0 = s0 * 32, row1 = min(s1 * 32, a.n);
  tail_mark(a, 12);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool staged = (q1 > q0) || (p1 > p0);
  if (tid == 0 && staged) {
    const unsigned vb = (unsigned)(q1 - q0) * 32u * 6u * 8u, cb = (unsigned)(q1 - q0) * 32u * 4u;
    const unsigned pvb = (unsigned)(p1 - p0) * 32u * 6u * 8u, pcb = (unsigned)(p1 - p0) * 32u * 4u;
    mbar_arrive_expect(&bar, vb + cb + pvb + pcb);
    if (vb) {
      bulk_g2s(sv, a.a_val + (long)q0 * 32 * 6, vb, &bar);
      bulk_g2s(sc, a.a_col + (long)q0 * 32, cb, &bar);
    }
    if (pvb) {
      bulk_g2s(spv, a.p_val + (long)p0 * 32 * 6, pvb, &bar);
      bulk_g2s(spc, a.p_col + (long)p0 * 32, pcb, &bar);
    }
  }
  if (tid == 32 && a.r_nbr > 0) {  // R_t (read after two barriers) into L2 while A_t streams in
    const long nb = a.r_ptr[a.r_nbr];
    const long lo = nb * cta / gridDim.x, hi = nb * (cta + 1) / gridDim.x;
    const char *v0 = (const char *)(a.r_val + lo * 36), *v1 = (const char *)(a.r_val + hi * 36);
    for (const char *p = (const char *)((uintptr_t)v0 & ~(uintptr_t)127); p < v1; p += 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
    const char *c0 = (const char *)(a.r_col + lo), *c1 = (const char *)(a.r_col + hi);
    for (const char *p = (const char *)((uintptr_t)c0 & ~(uintptr_t)127); p < c1; p += 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
  const int nco = a.nco;
  if (cta == 0)
    for (int idx = tid; idx < nco * nco; idx += blockDim.x) {
      const int i = idx / nco, j = idx % nco;
      sL[idx] = (i >= j) ? a.Lc[(long)j * a.Wc + (i - j)] : 0.0;
    }
  double *xb[2] = {a.x, a.x2};
  int ci = a.cheb ? (((a.kdeg - 1) + (a.pre - 1) * a.kdeg + a.post * a.kdeg) & 1) : (((a.pre - 1) + a.post) & 1);
  if (a.cheb) {  // Chebyshev from zero (C23): t = b/d, dir = c0 t, x = dir
    for (int i = row0 + tid; i < row1; i += blockDim.x) {
      const double v = a.c0 * (a.b[i] / a.d[i]);
      __stcg(a.dir + i, v);
      __stcg(xb[ci] + i, v);
    }
  } else {
    for (int i = row0 + tid; i < row1; i += blockDim.x) __stcg(xb[ci] + i, a.b[i] / a.d[i]);  // jacobi0
  }
  if (staged) mbar_wait(&bar, 0);
  tail_mark(a, 0);
  tail_sync(cl);
  tail_mark(a, 1);
  auto stage_x = [&](const double *xin) {
    for (int i = tid; i < a.n; i += blockDim.x) sx[i] = __ldcg(xin + i);
    __syncthreads();
  };
  // one smoothing step = stage x, SpMV epilogue into the other buffer, barrier
  auto cheb_step = [&](bool first, int st) {
    stage_x(xb[ci]);
    if (first) tail_spmv<SPMV_CHEB1>(a, row0, row1, q0, sx, sv, sc, xb[1 - ci]);
    else tail_spmv<SPMV_CHEB>(a, row0, row1, q0, sx, sv, sc, xb[1 - ci], st);
    ci = 1 - ci;
  };
  if (a.cheb) {
    for (int st = 1; st < a.kdeg; st++) {
      cheb_step(false, st);
      tail_sync(cl);
    }
    for (int sw = 1; sw < a.pre; sw++)
      for (int st = 0; st < a.kdeg; st++) {
        cheb_step(st == 0, st);
        tail_sync(cl);
      }
  } else {
    for (int s = 1; s < a.pre; s++) {
      stage_x(xb[ci]);
      tail_spmv<SPMV_SMOOTH>(a, row0, row1, q0, sx, sv, sc, xb[1 - ci]);
      ci = 1 - ci;
      tail_sync(cl);
    }
  }
  stage_x(xb[ci]);
  tail_mark(a, 2);
  tail_spmv<SPMV_RESID>(a, row0, row1, q0, sx, sv, sc, a.r);
  tail_mark(a, 3);
  tail_sync(cl);
  tail_mark(a, 4);
  // restriction: one warp per scalar row of R (k_restrict_row<6> chain and butterfly, C5)
  {
    const int lane = tid & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    // warps round-robin over the CTAs, so that the few rows of R spread over all SMs of the cluster
    for (int w = (tid >> 5) * gridDim.x + cta; w < a.r_nbr * 6; w += nw) {
      const int blk = w / 6, rr = w % 6;
      const int beg = a.r_ptr[blk], end = a.r_ptr[blk + 1];
      double acc = 0.0;
      // 4 lane-strided blocks per batch: their columns, values and r entries are all in flight at once
      for (int k0 = beg + lane; k0 < end; k0 += 4 * 32) {
        int cc[4];
        double vv[4][6], rv[4][6];
        int kk[4];  // clamped: unconditional loads, all issued before the chain
#pragma unroll
        for (int u = 0; u < 4; u++) kk[u] = min(k0 + 32 * u, end - 1);
#pragma unroll
        for (int u = 0; u < 4; u++) cc[u] = a.r_col[kk[u]];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int e = 0; e < 6; e++) {
            vv[u][e] = a.r_val[(long)kk[u] * 36 + rr * 6 + e];
            rv[u][e] = __ldcg(a.r + (long)cc[u] * 6 + e);
          }
#pragma unroll
        for (int u = 0; u < 4; u++)
          if (k0 + 32 * u < end)
#pragma unroll
            for (int e = 0; e < 6; e++) acc = __fma_rn(vv[u][e], rv[u][e], acc);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc = acc + __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) __stcg(a.bc + w, acc);
    }
  }
  tail_mark(a, 5);
  tail_sync(cl);
  tail_mark(a, 6);
  // coarsest: forward and backward substitution by one warp (C10), rows lane and lane + 32
  if (cta == 0 && tid < 32) {
    const int lane = tid;
    const int i0 = lane, i1 = lane + 32;
    double acc0 = (i0 < nco) ? __ldcg(a.bc + i0) : 0.0, acc1 = (i1 < nco) ? __ldcg(a.bc + i1) : 0.0;
    const double d0 = (i0 < nco) ? a.dinv_c[i0] : 0.0, d1 = (i1 < nco) ? a.dinv_c[i1] : 0.0;
    for (int j = 0; j < nco; j++) {
      const double yj = __shfl_sync(0xffffffffu, (j < 32) ? acc0 * d0 : acc1 * d1, j & 31);
      if (lane == 0) ys[j] = yj;
      if (i0 > j && i0 < nco) acc0 = __fma_rn(-sL[i0 * nco + j], yj, acc0);
      if (i1 > j && i1 < nco) acc1 = __fma_rn(-sL[i1 * nco + j], yj, acc1);
    }
    __syncwarp();
    acc0 = (i0 < nco) ? ys[i0] : 0.0;
    acc1 = (i1 < nco) ? ys[i1] : 0.0;
    for (int k = nco - 1; k >= 0; k--) {
      const double xk = __shfl_sync(0xffffffffu, (k < 32) ? acc0 * d0 : acc1 * d1, k & 31);
      if (lane == 0) __stcg(a.xc + k, xk);
      if (i0 < k) acc0 = __fma_rn(-sL[k * nco + i0], xk, acc0);
      if (i1 < k) acc1 = __fma_rn(-sL[k * nco + i1], xk, acc1);
    }
  }
  tail_mark(a, 7);
  tail_sync(cl);
  tail_mark(a, 8);
  // prolongation x += P_t x_c (SELL chain, C2) from the staged P_t slices, rows of this CTA
  // (sx still holds x of level t as staged for the residual; the coarse x goes to ys)
  for (int i = tid; i < nco; i += blockDim.x) ys[i] = __ldcg(a.xc + i);
  __syncthreads();
  for (int i = row0 + tid; i < row1; i += blockDim.x) {
    const double acc = tail_row(spv, spc, ys, a.p_sp[i >> 5] - p0, a.p_len[i], i & 31);
    __stcg(xb[ci] + i, sx[i] + acc);
  }
  tail_mark(a, 9);
  tail_sync(cl);
  tail_mark(a, 10);
  if (a.cheb) {
    const int nsteps = a.post * a.kdeg;
    for (int q = 0; q < nsteps; q++) {
      cheb_step(q % a.kdeg == 0, q % a.kdeg);
      if (q + 1 < nsteps) tail_sync(cl);
    }
  } else {
    for (int s = 0; s < a.post; s++) {
      stage_x(xb[ci]);
      tail_spmv<SPMV_SMOOTH>(a, row0, row1, q0, sx, sv, sc, xb[1 - ci]);
      ci = 1 - ci;
      if (s + 1 < a.post) tail_sync(cl);
    }
  }
  tail_mark(a, 11);
}

static bool tail_disabled() {
  const char *e = getenv("AMGF_NO_TAIL");  // A/B experiments and the parity test of the unfused path
  return e && atoi(e) != 0;
}

void tail_plan(Ctx &c) {
  c.tail_level = -1;
  if (tail_disabled() || c.nlev < 3 || c.cfg.smoother == 2) return;  // the tail smooths with C23 / C4 only
  const int t = c.nlev - 2;
  Level &L = c.lev[t];
  if (L.b != 6 || L.As.br != 1 || L.As.bc != 6 || L.Ps.br != 1 || L.Ps.bc != 6 || L.R.bc != 6) return;
  if (c.nco > TAIL_MAX_NCO || c.nco != 6 * L.R.nbr || L.Ps.perm || L.As.perm) return;
  const int ns = L.As.nslices;
  std::vector<int> sp(ns + 1);
  CK(cudaMemcpy(sp.data(), L.As.slice_ptr, (ns + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  // contiguous slice ranges, at most TAIL_MAX_CTA, minimising the largest slot count (binary search on
  // the capacity, greedy fill)
  auto chunks = [&](long cap, std::vector<int> *out) {
    int k = 0;
    long cur = 0;
    if (out) out->assign(1, 0);
    for (int q = 0; q < ns; q++) {
      const long w = sp[q + 1] - sp[q];
      if (w > cap) return 1 << 30;
      if (cur + w > cap) {
        k++;
        cur = 0;
        if (out) out->push_back(q);
      }
      cur += w;
    }
    if (out) out->push_back(ns);
    return k + 1;
  };
  long lo = 1, hi = std::max<long>(1, sp[ns]);
  while (lo < hi) {
    const long mid = (lo + hi) / 2;
    if (chunks(mid, nullptr) <= TAIL_MAX_CTA) hi = mid;
    else lo = mid + 1;
  }
  std::vector<int> cs;
  const int ncta = chunks(lo, &cs);
  std::vector<int> pp(ns + 1);
  REQUIRE(L.Ps.nslices == ns, AMGF_ERR_ARG, "tail: P and A slice counts differ");
  CK(cudaMemcpy(pp.data(), L.Ps.slice_ptr, (ns + 1) * sizeof(int), cudaMemcpyDeviceToHost));
  long maxslots = 0, maxp = 0;
  for (int k = 0; k < ncta; k++) {
    maxslots = std::max<long>(maxslots, sp[cs[k + 1]] - sp[cs[k]]);
    maxp = std::max<long>(maxp, pp[cs[k + 1]] - pp[cs[k]]);
  }
  const int xs = (int)((L.n + 1) & ~1L);
  const long maxv = maxslots * 32 * 6, maxc = maxslots * 32;
  const long maxpv = maxp * 32 * 6, maxpc = maxp * 32;
  const size_t smem = (size_t)xs * 8 + (maxv + maxpv) * 8 + (maxc + maxpc) * 4 + (size_t)c.nco * c.nco * 8;
  const bool dbg = getenv("AMGF_DEBUG_TAIL") != nullptr;
  if (dbg) fprintf(stderr, "tail plan: level %d n %ld slices %d ncta %d maxslots %ld smem %zu\n", t, L.n, ns, ncta,
                   maxslots, smem);
  if (smem > 225 * 1024) return;  // 227 KB per CTA minus the static part
  CK(cudaFuncSetAttribute(k_vcycle_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (ncta > 8) CK(cudaFuncSetAttribute(k_vcycle_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(TAIL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  const cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, k_vcycle_tail, &cfg);
  if (dbg) fprintf(stderr, "tail plan: max active clusters %d (%s)\n", nclusters, cudaGetErrorString(oe));
  if (oe != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return;
  }
  c.tail_cta_s = c.alloc<int>(ncta + 1);
  CK(cudaMemcpy(c.tail_cta_s, cs.data(), (ncta + 1) * sizeof(int), cudaMemcpyHostToDevice));
  c.tail_level = t;
  c.tail_ncta = ncta;
  c.tail_xs = xs;
  c.tail_maxv = (int)maxv;
  c.tail_maxc = (int)maxc;
  c.tail_maxpv = (int)maxpv;
  c.tail_maxpc = (int)maxpc;
  c.tail_smem = smem;
}

void tail_vcycle(Ctx &c, const double *b, double *x) {
  const int t = c.tail_level;
  Level &L = c.lev[t], &Lc = c.lev[t + 1];
  TailArgs a;
  a.n = (int)L.n;
  a.pre = c.cfg.pre_sweeps;
  a.post = c.cfg.post_sweeps;
  a.cta_s = c.tail_cta_s;
  a.a_sp = L.As.slice_ptr; a.a_len = L.As.rowlen; a.a_col = L.As.col; a.a_val = L.As.val;
  a.p_sp = L.Ps.slice_ptr; a.p_len = L.Ps.rowlen; a.p_col = L.Ps.col; a.p_val = L.Ps.val;
  a.r_nbr = L.R.nbr; a.r_ptr = L.R.ptr; a.r_col = L.R.col; a.r_val = L.R.val;
  a.nco = c.nco;
  a.Wc = band_stride(c.nco - 1);
  a.Lc = c.Lc_col;
  a.dinv_c = c.Lc_dinv;
  a.d = L.dl1;
  a.b = b;
  a.x = x; a.x2 = L.x2; a.r = L.r; a.bc = Lc.bv; a.xc = Lc.x;
  a.xs = c.tail_xs; a.maxv = c.tail_maxv; a.maxc = c.tail_maxc; a.maxpv = c.tail_maxpv; a.maxpc = c.tail_maxpc;
  a.cheb = c.cfg.smoother == 1;
  a.kdeg = c.cfg.cheb_degree;
  a.dir = L.dir;
  a.c0 = c.cheb_c0;
  for (int k = 0; k < 33; k++) { a.ca[k] = c.cheb_a[k]; a.cb[k] = c.cheb_b[k]; }
  static const bool timing = getenv("AMGF_TAIL_TIMING") != nullptr;  // phase timestamps (tools only)
  a.tm = nullptr;
  if (timing && !c.capturing) a.tm = c.alloc<unsigned long long>(c.tail_ncta * 16);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = c.tail_ncta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(c.tail_ncta);
  cfg.blockDim = dim3(TAIL_THREADS);
  cfg.dynamicSmemBytes = c.tail_smem;
  cfg.stream = c.stream;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_vcycle_tail, a));
  after_launch(c, "k_vcycle_tail");
  if (a.tm) {
    std::vector<unsigned long long> h(c.tail_ncta * 16);
    CK(cudaMemcpy(h.data(), a.tm, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (int k = 0; k < c.tail_ncta; k++) t0 = std::min(t0, h[k * 16 + 12]);
    fprintf(stderr, "tail phases (ns after the first CTA started, max over CTAs):");
    for (int ph = 0; ph < 12; ph++) {
      unsigned long long m = 0;
      for (int k = 0; k < c.tail_ncta; k++) m = std::max(m, h[k * 16 + ph] - t0);
      fprintf(stderr, " %d:%llu", ph, m);
    }
    fprintf(stderr, "\n");
  }
}

}  // namespace amgf
