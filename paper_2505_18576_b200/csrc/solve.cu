// solve.cu -- solve-phase kernels of libamgf.so.
//
//   k_sell      SELL-32 block SpMV, one thread per block row, fused epilogues:
//               y = Ax | r = b - Ax | l1-Jacobi sweep | y = Ax + CTA partial of x.y | sweep + add
//               (contracts C2, C4, C6, C14 level 1).  Used for S, every A_l, and P (prolongation).
//   k_restrict  b_c = R r, one warp per coarse block row, strided lanes + xor butterfly (C5).
//   k_dot_*     two-level fixed-tree dot products (C14) with the PCG scalar updates (C15).
//   k_band_trsv A_w^{-1} v by the banded Cholesky factor, one warp, shuffle broadcast, cp.async
//               double-buffered band columns (C10); gather r1[Z] and scatter x2[Z] += y fused.
//   k_thin      r2 = r1 - S[:,Z] y over the rows that touch Z (C11).
#include <cstdlib>

#include "common.cuh"
#include "devutil.cuh"
#include "nd_kernels.cuh"

namespace amgf {

__device__ __forceinline__ double ldg_stream(const double *p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldg_stream_i(const int *p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Fixed tree of C14 over 256 values in shared memory; returns s[0] to all threads.
__device__ __forceinline__ double cta_tree(double v, double *s) {
  int t = threadIdx.x;
  s[t] = v;
  __syncthreads();
#pragma unroll
  for (int w = CTA / 2; w >= 1; w >>= 1) {
    if (t < w) s[t] = s[t] + s[t + w];
    __syncthreads();
  }
  double r = s[0];
  __syncthreads();
  return r;
}

enum { MODE_Y = SPMV_Y, MODE_RESID = SPMV_RESID, MODE_SMOOTH = SPMV_SMOOTH, MODE_DOT = SPMV_DOT,
       MODE_SMOOTH_ADD = SPMV_SMOOTH_ADD, MODE_ADDTO = 5, MODE_CHEB1 = SPMV_CHEB1, MODE_CHEB = SPMV_CHEB,
       MODE_CHEB_DOT = 8, MODE_YDIV = SPMV_YDIV, MODE_POW = SPMV_POW };

// Chebyshev step epilogue (contract C23): t = (b - acc)/d; first step dir = ca t, later dir = fma(ca, dir,
// cb t); x_new = x + dir (then add + x_new when add is given, as SMOOTH_ADD).
__device__ __forceinline__ double cheb_epilogue(int mode, double res, double di, double xi, double *dir, long i,
                                                double ca, double cb, const double *add) {
  const double t = res / di;
  const double dv = (mode == MODE_CHEB1) ? ca * t : __fma_rn(ca, dir[i], cb * t);  // MODE_CHEB(_DOT)
  dir[i] = dv;
  double xn = xi + dv;
  if (add) xn = add[i] + xn;
  return xn;
}

// x block of column c (BC consecutive doubles): 16-byte vector loads when BC is even (x is 16-byte aligned,
// checked by the dispatcher), i.e. half the load instructions and L1 requests of the scalar gathers.
template <int BC>
__device__ __forceinline__ void gather_x(const double *__restrict__ x, int c, double (&v)[BC]) {
  if constexpr (BC % 2 == 0) {
    const double2 *p = reinterpret_cast<const double2 *>(x + (long)c * BC);
#pragma unroll
    for (int h = 0; h < BC / 2; h++) {
      const double2 t = p[h];
      v[2 * h] = t.x;
      v[2 * h + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int e = 0; e < BC; e++) v[e] = x[(long)c * BC + e];
  }
}

// The SELL row chain of one block row (C2): acc[r] = sum over slots s (ascending) and block columns e
// (ascending) of val * x, software-pipelined (slot s+1's column, values and x gather in flight while slot s
// is consumed).
template <int BR, int BC>
__device__ __forceinline__ void sell_row(int row, const int *__restrict__ slice_ptr, const int *__restrict__ rowlen,
                                         const int *__restrict__ col, const double *__restrict__ val,
                                         const double *__restrict__ x, double (&acc)[BR]) {
  const int lane = row & 31;
#pragma unroll
  for (int r = 0; r < BR; r++) acc[r] = 0.0;
  {
    const int len = rowlen[row];
    const long base = slice_ptr[row >> 5];
    const int *cp = col + base * 32 + lane;
    const double *vp = val + base * (BR * BC * 32) + lane;
    // software pipeline: slot s+1's column, values and x gather are in flight while slot s is consumed
    double vcur[BR * BC], xcur[BC];
    int cnext = 0, c0 = 0;
    if (len > 0) {
      c0 = ldg_stream_i(cp);
#pragma unroll
      for (int q = 0; q < BR * BC; q++) vcur[q] = ldg_stream(vp + q * 32);
      cnext = ldg_stream_i(cp + (len > 1 ? 32 : 0));
    }
    // PDL: the operator's first slot is in flight before the wait for the previous kernel (x, b, d are its
    // results); a no-op without a programmatic launch
    pdl_wait();
    if (len > 0) gather_x<BC>(x, c0, xcur);
    for (int s = 0; s < len; s++) {
      // branch-free prefetch (the last slot is re-read once at the end)
      const int s1 = min(s + 1, len - 1), s2 = min(s + 2, len - 1);
      const double *v = vp + (long)s1 * (BR * BC * 32);
      double vnx[BR * BC], xnx[BC];
#pragma unroll
      for (int q = 0; q < BR * BC; q++) vnx[q] = ldg_stream(v + q * 32);
      gather_x<BC>(x, cnext, xnx);
      const int cnn = ldg_stream_i(cp + (long)s2 * 32);
#pragma unroll
      for (int r = 0; r < BR; r++)
#pragma unroll
        for (int e = 0; e < BC; e++) acc[r] = __fma_rn(vcur[r * BC + e], xcur[e], acc[r]);
#pragma unroll
      for (int q = 0; q < BR * BC; q++) vcur[q] = vnx[q];
#pragma unroll
      for (int e = 0; e < BC; e++) xcur[e] = xnx[e];
      cnext = cnn;
    }
  }
}

template <int BR, int BC, int MODE>
__global__ void __launch_bounds__(CTA) k_sell(int nrows, const int *__restrict__ slice_ptr,
                                              const int *__restrict__ rowlen, const int *__restrict__ col,
                                              const double *__restrict__ val, const double *__restrict__ x,
                                              const double *__restrict__ b, const double *__restrict__ d,
                                              const double *__restrict__ add, double *__restrict__ y,
                                              double *__restrict__ dot_part, const int *__restrict__ perm,
                                              ChebArgs ch) {
  const int row = blockIdx.x * CTA + threadIdx.x;
  double acc[BR];
#pragma unroll
  for (int r = 0; r < BR; r++) acc[r] = 0.0;
  if (row < nrows) sell_row<BR, BC>(row, slice_ptr, rowlen, col, val, x, acc);
  pdl_launch_dependents();  // the next kernel's CTAs may start their operator prologue in our tail
  if (MODE == MODE_DOT) {
    __shared__ double red[CTA];
    double s = 0.0;
    if (row < nrows) {
#pragma unroll
      for (int r = 0; r < BR; r++) {
        y[(long)row * BR + r] = acc[r];
        s = __fma_rn(x[(long)row * BR + r], acc[r], s);
      }
    }
    double tot = cta_tree(s, red);
    if (threadIdx.x == 0) dot_part[blockIdx.x] = tot;
    return;
  }
  if (MODE == MODE_CHEB_DOT) {  // last Chebyshev step (+ add) fused with the C14 partials of dot(r, y)
    __shared__ double red2[CTA];
    double s = 0.0;
    if (row < nrows) {
#pragma unroll
      for (int r = 0; r < BR; r++) {
        const long i = (long)row * BR + r;
        const double yi = cheb_epilogue(MODE_CHEB, b[i] - acc[r], d[i], x[i], ch.dir, i, ch.ca, ch.cb, add);
        y[i] = yi;
        s = __fma_rn(ch.dot_r[i], yi, s);
      }
    }
    double tot = cta_tree(s, red2);
    if (threadIdx.x == 0) ch.dot_part[blockIdx.x] = tot;
    return;
  }
  if (MODE == MODE_POW) {  // power step (C18): w = acc / d, C14 partials of w.w (dot_part) and v.v (ch.dot_part)
    __shared__ double red3[CTA];
    double sw = 0.0, sv = 0.0;
    if (row < nrows) {
#pragma unroll
      for (int r = 0; r < BR; r++) {
        const long i = (long)row * BR + r;
        const double wi = acc[r] / d[i];
        y[i] = wi;
        sw = __fma_rn(wi, wi, sw);
      }
#pragma unroll
      for (int r = 0; r < BR; r++) {
        const double vi = x[(long)row * BR + r];
        sv = __fma_rn(vi, vi, sv);
      }
    }
    const double tw = cta_tree(sw, red3);
    const double tv = cta_tree(sv, red3);
    if (threadIdx.x == 0) {
      dot_part[blockIdx.x] = tw;
      ch.dot_part[blockIdx.x] = tv;
    }
    return;
  }
  if (row >= nrows) return;
  const int orow = (MODE == MODE_ADDTO && perm) ? perm[row] : row;
#pragma unroll
  for (int r = 0; r < BR; r++) {
    const long i = (long)orow * BR + r;
    if (MODE == MODE_Y) {
      y[i] = acc[r];
    } else if (MODE == MODE_RESID) {
      y[i] = b[i] - acc[r];
    } else if (MODE == MODE_SMOOTH || MODE == MODE_SMOOTH_ADD) {
      double res = b[i] - acc[r];
      double t = res / d[i];
      double xn = x[i] + t;
      if (MODE == MODE_SMOOTH_ADD) xn = add[i] + xn;
      y[i] = xn;
    } else if (MODE == MODE_ADDTO) {
      y[i] = y[i] + acc[r];
    } else if (MODE == MODE_CHEB1 || MODE == MODE_CHEB) {
      y[i] = cheb_epilogue(MODE, b[i] - acc[r], d[i], x[i], ch.dir, i, ch.ca, ch.cb, add);
    } else if (MODE == MODE_YDIV) {
      y[i] = acc[r] / d[i];
    }
  }
}

// Latency-oriented variant for scalar-row (1 x BC) SELL of the small coarse levels: D slots of values and
// x in flight (register ring, fully unrolled), column indices 2D slots ahead.  Same chain as k_sell (C2).
#ifdef AMGF_R1_TRACE
__device__ unsigned long long g_r1_trace[8192 * 4];
int r1_trace_read(unsigned long long *h, int n) {
  return cudaMemcpyFromSymbol(h, g_r1_trace, sizeof(unsigned long long) * std::min(n, 8192 * 4)) == cudaSuccess ? 0 : -1;
}
#endif
__constant__ int c_r1_prefetch = 2;  // L2 prefetch distance of k_sell_r1 in slots beyond the register ring (0: off).
                                 // Measured at cfg 3 with the PDL-chained kernels (apply us): off 2239, 1-2 2209-2211,
                                 // 4 2215, 8 2224, 16 2242; 8 was the best before PDL (round 1)
__device__ __forceinline__ int r1_prefetch_slots() { return c_r1_prefetch; }

template <int BC, int MODE, int D>
__global__ void __launch_bounds__(CTA) k_sell_r1(int nrows, const int *__restrict__ slice_ptr,
                                                 const int *__restrict__ rowlen, const int *__restrict__ col,
                                                 const double *__restrict__ val, const double *__restrict__ x,
                                                 const double *__restrict__ b, const double *__restrict__ d,
                                                 const double *__restrict__ add, double *__restrict__ y,
                                                 const int *__restrict__ perm, ChebArgs ch) {
  const int row = blockIdx.x * CTA + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
#ifdef AMGF_R1_TRACE
  unsigned long long t_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
  const int len = rowlen[row];
  const long base = slice_ptr[row >> 5];
  const int *cp = col + base * 32 + lane;
  const double *vp = val + base * (BC * 32) + lane;
  double acc = 0.0;
  double rv[D][BC], rx[D][BC];
  int rc[D];
  const int last = len - 1;
  int rc2[D];
  if (len > 0) {
#pragma unroll
    for (int q = 0; q < D; q++) {
      rc[q] = ldg_stream_i(cp + (long)min(q, last) * 32);
      rc2[q] = ldg_stream_i(cp + (long)min(q + D, last) * 32);
    }
#pragma unroll
    for (int q = 0; q < D; q++) {
      const int sq = min(q, last);
#pragma unroll
      for (int e = 0; e < BC; e++) rv[q][e] = ldg_stream(vp + ((long)sq * BC + e) * 32);
    }
  }
  pdl_wait();  // PDL: columns and values of the first D slots are in flight; x is the previous kernel's result
  if (len > 0) {
  // prologue: columns of slots D..2D-1, values + x of slots 0..D-1
#pragma unroll
  for (int q = 0; q < D; q++) {
#pragma unroll
    gather_x<BC>(x, rc[q], rx[q]);
    rc[q] = rc2[q];
  }
  // L2 prefetch window (pf slots ahead of the register ring): the slice's values of slots
  // [s0 + pf, s0 + pf + D) by one TMA bulk prefetch from the lowest active lane, so the ring's loads
  // find their lines in L2 (long rows of the large coarse levels are latency chains)
  const int pf = r1_prefetch_slots();
  const int sw = slice_ptr[(row >> 5) + 1] - (int)base;
  const char *vslice = (const char *)(val + base * (BC * 32));
  if (pf > 0 && lane == __ffs(__activemask()) - 1) {
    const int p1 = min(D + pf, sw);
    if (p1 > D)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vslice + (long)D * BC * 32 * 8),
                   "r"((p1 - D) * BC * 32 * 8)
                   : "memory");
  }
  for (int s0 = 0; s0 < len; s0 += D) {
    if (pf > 0 && lane == __ffs(__activemask()) - 1) {
      const int p0 = s0 + D + pf, p1 = min(p0 + D, sw);
      if (p1 > p0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vslice + (long)p0 * BC * 32 * 8),
                     "r"((p1 - p0) * BC * 32 * 8)
                     : "memory");
    }
#pragma unroll
    for (int q = 0; q < D; q++) {
      const int sl = s0 + q;
      if (sl < len) {
#pragma unroll
        for (int e = 0; e < BC; e++) acc = __fma_rn(rv[q][e], rx[q][e], acc);
      }
      // refill stage q with slot sl + D (column already loaded), and fetch the column of slot sl + 2D
      const int sn = min(sl + D, last), sc = min(sl + 2 * D, last);
#pragma unroll
      for (int e = 0; e < BC; e++) rv[q][e] = ldg_stream(vp + ((long)sn * BC + e) * 32);
#pragma unroll
      gather_x<BC>(x, rc[q], rx[q]);
      rc[q] = ldg_stream_i(cp + (long)sc * 32);
    }
  }
  }
  pdl_launch_dependents();
  const long i = perm ? perm[row] : row;  // rows sorted by length (SELL packing), any mode
  if (MODE == MODE_Y) {
    y[i] = acc;
  } else if (MODE == MODE_RESID) {
    y[i] = b[i] - acc;
  } else if (MODE == MODE_SMOOTH || MODE == MODE_SMOOTH_ADD) {
    double res = b[i] - acc;
    double t = res / d[i];
    double xn = x[i] + t;
    if (MODE == MODE_SMOOTH_ADD) xn = add[i] + xn;
    y[i] = xn;
  } else if (MODE == MODE_ADDTO) {
    y[i] = y[i] + acc;
  } else if (MODE == MODE_CHEB1 || MODE == MODE_CHEB) {
    y[i] = cheb_epilogue(MODE, b[i] - acc, d[i], x[i], ch.dir, i, ch.ca, ch.cb, add);
  } else if (MODE == MODE_YDIV) {
    y[i] = acc / d[i];
  }
#ifdef AMGF_R1_TRACE  // per-warp start / end / SM / longest row of the last launch (A/B builds only)
  {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    int mlen = len;
    for (int o = 16; o; o >>= 1) mlen = max(mlen, __shfl_xor_sync(__activemask(), mlen, o));
    const int wg = row >> 5;
    if (lane == 0 && wg < 8192) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_r1_trace[wg * 4 + 0] = t_start;
      g_r1_trace[wg * 4 + 1] = t_end;
      g_r1_trace[wg * 4 + 2] = smid;
      g_r1_trace[wg * 4 + 3] = (unsigned long long)mlen | ((unsigned long long)nrows << 32);
    }
  }
#endif
}

// launch with programmatic dependent launch (the SELL kernels wait for their predecessor only before the
// first x gather, so their operator prologue overlaps its tail); AMGF_NO_PDL=1 launches plainly (A/B)
template <typename... KA, typename... A>
static void go(Ctx &c, bool pdl, void (*k)(KA...), dim3 g, dim3 t, A... a) {
  if (pdl) launch_pdl(c.stream, k, g, t, 0, a...);
  else k<<<g, t, 0, c.stream>>>(((KA)a)...);
}
static bool sell_pdl() {
  static const bool on = getenv("AMGF_NO_PDL") == nullptr;
  return on;
}

template <int BR, int BC>
static void sell_dispatch(Ctx &c, const Sell &A, int mode, const double *x, const double *b, const double *d,
                          const double *add, double *y, double *dp, ChebArgs ch = ChebArgs{}) {
  dim3 g(nblk(A.nrows)), t(CTA);
  if (A.nrows == 0) return;
  // the x gathers of even block widths are 16-byte vector loads (gather_x)
  if (BC % 2 == 0) REQUIRE(((uintptr_t)x & 15) == 0, AMGF_ERR_ARG, "SELL SpMV: x must be 16-byte aligned");
  {
    size_t &pf_set = device_slot((const void *)&c_r1_prefetch);
    if (!pf_set) {
      pf_set = 1;
      const int pf = getenv("AMGF_R1_PF") ? atoi(getenv("AMGF_R1_PF")) : 2;  // measured: 1-2 slots best
      CK(cudaMemcpyToSymbol(c_r1_prefetch, &pf, sizeof(int)));
    }
  }
  {
    // An explicit carveout preference for the residual SpMV lets the A_w solve, which runs concurrently on
    // the filter stream (apply_M), get SMs while the SpMV is resident: the driver default cost ~50 us per
    // AMGF apply at cfg 3; any value in 0..60 % gave the same time, above that the SpMV loses L1.
    size_t &once = device_slot((const void *)k_sell<BR, BC, MODE_RESID>);
    if (!once) {
      once = 1;
      CK(cudaFuncSetAttribute(k_sell<BR, BC, MODE_RESID>, cudaFuncAttributePreferredSharedMemoryCarveout, 50));
      // the setup's power iteration (MODE_Y) runs beside the A_w factorization: same reason
      CK(cudaFuncSetAttribute(k_sell<BR, BC, MODE_Y>, cudaFuncAttributePreferredSharedMemoryCarveout, 50));
      CK(cudaFuncSetAttribute(k_sell<BR, BC, MODE_POW>, cudaFuncAttributePreferredSharedMemoryCarveout, 50));
    }
  }
  const bool pdl = sell_pdl();
  if (BR == 1 && mode != MODE_DOT) {
    switch (mode) {
      case MODE_Y: go(c, pdl, k_sell_r1<BC, MODE_Y, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_RESID: go(c, pdl, k_sell_r1<BC, MODE_RESID, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_SMOOTH: go(c, pdl, k_sell_r1<BC, MODE_SMOOTH, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_SMOOTH_ADD: go(c, pdl, k_sell_r1<BC, MODE_SMOOTH_ADD, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_ADDTO: go(c, pdl, k_sell_r1<BC, MODE_ADDTO, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_CHEB1: go(c, pdl, k_sell_r1<BC, MODE_CHEB1, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_CHEB: go(c, pdl, k_sell_r1<BC, MODE_CHEB, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      case MODE_YDIV: go(c, pdl, k_sell_r1<BC, MODE_YDIV, 4>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, A.perm, ch); break;
      default: throw Error{AMGF_ERR_ARG, "sell spmv: mode not available for scalar-row SELL"};
    }
    after_launch(c, "k_sell_r1");
    return;
  }
  switch (mode) {
    case MODE_Y: go(c, pdl, k_sell<BR, BC, MODE_Y>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_RESID: go(c, pdl, k_sell<BR, BC, MODE_RESID>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_SMOOTH: go(c, pdl, k_sell<BR, BC, MODE_SMOOTH>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_DOT: go(c, pdl, k_sell<BR, BC, MODE_DOT>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_SMOOTH_ADD: go(c, pdl, k_sell<BR, BC, MODE_SMOOTH_ADD>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_ADDTO: go(c, pdl, k_sell<BR, BC, MODE_ADDTO>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_CHEB1: go(c, pdl, k_sell<BR, BC, MODE_CHEB1>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_CHEB: go(c, pdl, k_sell<BR, BC, MODE_CHEB>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_CHEB_DOT: go(c, pdl, k_sell<BR, BC, MODE_CHEB_DOT>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_YDIV: go(c, pdl, k_sell<BR, BC, MODE_YDIV>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    case MODE_POW: go(c, pdl, k_sell<BR, BC, MODE_POW>, g, t, A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, d, add, y, dp, A.perm, ch); break;
    default: throw Error{AMGF_ERR_ARG, "sell spmv: unknown mode"};
  }
  after_launch(c, __func__);
}

void launch_sell_spmv(Ctx &c, const Sell &A, int mode, const double *x, const double *b, const double *d,
                      const double *add, double *y, double *dp) {
  if (A.br == 3 && A.bc == 3) sell_dispatch<3, 3>(c, A, mode, x, b, d, add, y, dp);
  else if (A.br == 1 && A.bc == 6) sell_dispatch<1, 6>(c, A, mode, x, b, d, add, y, dp);
  else if (A.br == 6 && A.bc == 6) sell_dispatch<6, 6>(c, A, mode, x, b, d, add, y, dp);
  else throw Error{AMGF_ERR_ARG, "sell spmv: unsupported block shape"};
}

void launch_sell_pow(Ctx &c, const Sell &A, const double *v, const double *d, double *w, double *part_w,
                     double *part_v) {
  REQUIRE(A.br == 3 && A.bc == 3 && !A.perm, AMGF_ERR_ARG, "fused power step: fine level only");
  ChebArgs ch;
  ch.dot_part = part_v;
  sell_dispatch<3, 3>(c, A, MODE_POW, v, nullptr, d, nullptr, w, part_w, ch);
}

void launch_sell_cheb(Ctx &c, const Sell &A, bool first, const double *x, const double *b, const double *dl1,
                      double *dir, double ca, double cb, const double *add, double *y, const double *dot_r) {
  const ChebArgs ch{ca, cb, dir, dot_r, c.dot_part};
  REQUIRE(!dot_r || (!first && A.br == 3 && A.bc == 3 && !A.perm), AMGF_ERR_ARG, "fused dot: fine level, later step");
  const int mode = dot_r ? MODE_CHEB_DOT : (first ? MODE_CHEB1 : MODE_CHEB);
  if (A.br == 3 && A.bc == 3) sell_dispatch<3, 3>(c, A, mode, x, b, dl1, add, y, nullptr, ch);
  else if (A.br == 1 && A.bc == 6) sell_dispatch<1, 6>(c, A, mode, x, b, dl1, add, y, nullptr, ch);
  else throw Error{AMGF_ERR_ARG, "sell cheb: unsupported block shape"};
}

// PCG update (C15) fused with the from-zero Chebyshev start of the next V-cycle #1 at level 0 (C23):
// x = fma(alpha, p, x); r = fma(-alpha, q, r); t = r/d; dir = c0 t; xs = dir.
__global__ void k_axpy2_cheb0(long n, const Scalars *__restrict__ sc, const double *__restrict__ p,
                              const double *__restrict__ q, double *__restrict__ x, double *__restrict__ r,
                              const double *__restrict__ d, double c0, double *__restrict__ dir,
                              double *__restrict__ xs) {
  pdl_wait();  // alpha is the previous kernel's result
  const double a = sc->alpha;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    x[i] = __fma_rn(a, p[i], x[i]);
    const double rn = __fma_rn(-a, q[i], r[i]);
    r[i] = rn;
    const double v = c0 * (rn / d[i]);
    dir[i] = v;
    xs[i] = v;
  }
  pdl_launch_dependents();
}
// the same per-element arithmetic on pairs (16-byte loads and stores)
__global__ void k_axpy2_cheb0_v2(long n2, const Scalars *__restrict__ sc, const double2 *__restrict__ p,
                                 const double2 *__restrict__ q, double2 *__restrict__ x, double2 *__restrict__ r,
                                 const double2 *__restrict__ d, double c0, double2 *__restrict__ dir,
                                 double2 *__restrict__ xs) {
  pdl_wait();
  const double a = sc->alpha;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 pp = p[i], qq = q[i], dd = d[i];
    double2 xx = x[i], rr = r[i], v;
    xx.x = __fma_rn(a, pp.x, xx.x);
    xx.y = __fma_rn(a, pp.y, xx.y);
    x[i] = xx;
    rr.x = __fma_rn(-a, qq.x, rr.x);
    rr.y = __fma_rn(-a, qq.y, rr.y);
    r[i] = rr;
    v.x = c0 * (rr.x / dd.x);
    v.y = c0 * (rr.y / dd.y);
    dir[i] = v;
    xs[i] = v;
  }
  pdl_launch_dependents();
}
static bool pairs_ok(long n, std::initializer_list<const void *> ps) {
  if (n % 2) return false;
  for (const void *p : ps)
    if ((uintptr_t)p & 15) return false;
  return true;
}
void launch_axpy2_cheb0(Ctx &c, long n, const double *p, const double *q, double *x, double *r, const double *d,
                        double c0, double *dir, double *xs) {
  if (pairs_ok(n, {p, q, x, r, d, dir, xs}))
    go(c, sell_pdl(), k_axpy2_cheb0_v2, nblk(n / 2), CTA, n / 2, c.sc, (const double2 *)p, (const double2 *)q,
       (double2 *)x, (double2 *)r, (const double2 *)d, c0, (double2 *)dir, (double2 *)xs);
  else
    go(c, sell_pdl(), k_axpy2_cheb0, nblk(n), CTA, n, c.sc, p, q, x, r, d, c0, dir, xs);
  after_launch(c, "k_axpy2_cheb0");
}

// Chebyshev application from x = 0 (C23): t = b/d, dir = c0 t, x = dir.
__global__ void k_cheb0(long n, const double *__restrict__ b, const double *__restrict__ d, double c0,
                        double *__restrict__ dir, double *__restrict__ x) {
  pdl_wait();  // b is the previous kernel's result
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const double t = b[i] / d[i];
    const double v = c0 * t;
    dir[i] = v;
    x[i] = v;
  }
  pdl_launch_dependents();
}
// the same per-element arithmetic on pairs (16-byte loads and stores)
__global__ void k_cheb0_v2(long n2, const double2 *__restrict__ b, const double2 *__restrict__ d, double c0,
                           double2 *__restrict__ dir, double2 *__restrict__ x) {
  const long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const double2 d0 = i0 < n2 ? d[i0] : make_double2(1.0, 1.0);  // the diagonal is not the predecessor's output
  pdl_wait();
  for (long i = i0; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 bb = b[i], dd = (i == i0) ? d0 : d[i];
    double2 v;
    v.x = c0 * (bb.x / dd.x);
    v.y = c0 * (bb.y / dd.y);
    dir[i] = v;
    x[i] = v;
  }
  pdl_launch_dependents();
}
void launch_cheb0(Ctx &c, long n, const double *b, const double *d, double c0, double *dir, double *x) {
  const bool v2 = (n % 2 == 0) && !(((uintptr_t)b | (uintptr_t)d | (uintptr_t)dir | (uintptr_t)x) & 15);
  if (v2)
    go(c, sell_pdl(), k_cheb0_v2, nblk(n / 2), CTA, n / 2, (const double2 *)b, (const double2 *)d, c0,
       (double2 *)dir, (double2 *)x);
  else
    go(c, sell_pdl(), k_cheb0, nblk(n), CTA, n, b, d, c0, dir, x);
  after_launch(c, "k_cheb0");
}

// Nodal-block l1 smoothing step (C25), one thread per node: t = B_i^{-1} v_i by the C10 chains on the node's
// stored factor; out_i = t (from zero), x_i + t, or add_i + (x_i + t).
template <int B>
__global__ void k_block_smooth(int nodes, const double *__restrict__ bfac, const double *__restrict__ v,
                               const double *__restrict__ xin, const double *__restrict__ add, double *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  constexpr int NL = B * (B + 1) / 2;
  const double *f = bfac + (long)i * (NL + B), *rinv = f + NL;
  double y[B], t[B];
#pragma unroll
  for (int r = 0; r < B; r++) {
    double acc = v[(long)i * B + r];
#pragma unroll
    for (int k = 0; k < r; k++) acc = __fma_rn(-f[r * (r + 1) / 2 + k], y[k], acc);
    y[r] = acc * rinv[r];
  }
#pragma unroll
  for (int r = B - 1; r >= 0; r--) {
    double acc = y[r];
#pragma unroll
    for (int k = B - 1; k > r; k--) acc = __fma_rn(-f[k * (k + 1) / 2 + r], t[k], acc);
    t[r] = acc * rinv[r];
  }
#pragma unroll
  for (int r = 0; r < B; r++) {
    const long e = (long)i * B + r;
    double o = xin ? xin[e] + t[r] : t[r];
    if (add) o = add[e] + o;
    out[e] = o;
  }
}
void launch_block_smooth(Ctx &c, const Level &L, const double *v, const double *x_in, const double *add, double *out) {
  REQUIRE(L.bfac, AMGF_ERR_ARG, "block smoother data missing");
  if (L.b == 3) k_block_smooth<3><<<nblk(L.nodes), CTA, 0, c.stream>>>(L.nodes, L.bfac, v, x_in, add, out);
  else k_block_smooth<6><<<nblk(L.nodes), CTA, 0, c.stream>>>(L.nodes, L.bfac, v, x_in, add, out);
  after_launch(c, "k_block_smooth");
}

void launch_prolong(Ctx &c, const Sell &P, const double *xc, double *x) {
  if (P.br == 3) sell_dispatch<3, 6>(c, P, MODE_ADDTO, xc, nullptr, nullptr, nullptr, x, nullptr);
  else if (P.br == 1) sell_dispatch<1, 6>(c, P, MODE_ADDTO, xc, nullptr, nullptr, nullptr, x, nullptr);
  else if (P.br == 6) sell_dispatch<6, 6>(c, P, MODE_ADDTO, xc, nullptr, nullptr, nullptr, x, nullptr);
  else throw Error{AMGF_ERR_ARG, "prolong: unsupported block shape"};
}

// Residual y = b - S x on a partition of the SMs: a grid-stride loop over block rows in CTAs of 1024
// threads that each reserve most of an SM's shared memory, so the grid (one CTA per SM, fewer CTAs than
// SMs) leaves whole SMs free for the A_w solve running concurrently on the filter stream (apply_M).  Same
// row chain as k_sell (C2).
template <int BR, int BC>
__global__ void __launch_bounds__(1024) k_sell_resid_part(int nrows, const int *__restrict__ slice_ptr,
                                                          const int *__restrict__ rowlen, const int *__restrict__ col,
                                                          const double *__restrict__ val,
                                                          const double *__restrict__ x,
                                                          const double *__restrict__ b, double *__restrict__ y) {
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < nrows; row += gridDim.x * blockDim.x) {
    double acc[BR];
    sell_row<BR, BC>(row, slice_ptr, rowlen, col, val, x, acc);
#pragma unroll
    for (int r = 0; r < BR; r++) {
      const long i = (long)row * BR + r;
      y[i] = b[i] - acc[r];
    }
  }
}

void launch_resid_partition(Ctx &c, const Sell &A, const double *x, const double *b, double *y, int nsm,
                            size_t reserve) {
  REQUIRE(A.br == 3 && A.bc == 3 && !A.perm, AMGF_ERR_ARG, "resid_partition: fine-level 3x3 SELL expected");
  size_t &attr = device_slot((const void *)k_sell_resid_part<3, 3>);
  if (reserve > attr) {
    CK(cudaFuncSetAttribute(k_sell_resid_part<3, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reserve));
    attr = reserve;
  }
  k_sell_resid_part<3, 3><<<nsm, 1024, reserve, c.stream>>>(A.nrows, A.slice_ptr, A.rowlen, A.col, A.val, x, b, y);
  after_launch(c, "k_sell_resid_part");
}

// Residual b - S x at the dofs dof[p] only (p < n), into out[p]: the same chain as k_sell<3,3> for that
// scalar row (C2: the row's blocks in order, components ascending), so the values equal the full residual's
// at those rows bitwise.  The rows come from the compact copy Ctx::zr_* (contiguous per row, refreshed by
// every numeric re-setup) instead of the SELL slices, where each of them is a strided 8-byte-per-sector
// gather.  One warp per dof: lane s loads block s (column, 3 values, 3 x entries), all in flight at once,
// then every lane runs the row's chain over shuffled operands and lane 0 writes.  Used to start the A_w
// solve before the full residual SpMV (apply_M).
__global__ void __launch_bounds__(CTA) k_resid_dofs(int n, const int *__restrict__ dof, const int *__restrict__ zr_ptr,
                                                    const int *__restrict__ zr_col, const double *__restrict__ zr_val,
                                                    const double *__restrict__ x, const double *__restrict__ b,
                                                    double *__restrict__ out) {
  const int p = (blockIdx.x * CTA + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= n) return;  // warp-uniform
  const int beg = zr_ptr[p], len = zr_ptr[p + 1] - beg;
  double acc = 0.0;
  for (int s0 = 0; s0 < len; s0 += 32) {
    const int s = s0 + lane;
    double v[3] = {0.0, 0.0, 0.0}, xv[3] = {0.0, 0.0, 0.0};
    if (s < len) {
      const long k = beg + s;
      const int c = zr_col[k];
#pragma unroll
      for (int e = 0; e < 3; e++) {
        v[e] = zr_val[k * 3 + e];
        xv[e] = x[(long)c * 3 + e];
      }
    }
    const int m = min(32, len - s0);
    for (int q = 0; q < m; q++)
#pragma unroll
      for (int e = 0; e < 3; e++)
        acc = __fma_rn(__shfl_sync(0xffffffffu, v[e], q), __shfl_sync(0xffffffffu, xv[e], q), acc);
  }
  if (lane == 0) out[p] = b[dof[p]] - acc;
}

void launch_resid_dofs(Ctx &c, int n, const int *dof, const double *x, const double *b, double *out) {
  if (n == 0) return;
  REQUIRE(c.zr_ptr && c.zr_val, AMGF_ERR_ARG, "resid_dofs: compact Z rows missing");
  k_resid_dofs<<<nblk((long)n * 32), CTA, 0, c.stream>>>(n, dof, c.zr_ptr, c.zr_col, c.zr_val, x, b, out);
  after_launch(c, "k_resid_dofs");
}

// ------------------------------------------------------------------ restriction (C5)
template <int B>
__global__ void __launch_bounds__(CTA, 2) k_restrict(int nrows, const int *__restrict__ ptr, const int *__restrict__ col,
                                                  const double *__restrict__ val, const double *__restrict__ r,
                                                  double *__restrict__ out) {
  const int w = (blockIdx.x * CTA + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;  // warp-uniform
  pdl_wait();  // r is the previous kernel's result
  double acc[6];
#pragma unroll
  for (int q = 0; q < 6; q++) acc[q] = 0.0;
  const int beg = ptr[w], end = ptr[w + 1];
  // lane-strided blocks k = beg + lane + 32 t (C5 order).  No software pipeline: at 126 registers two
  // CTAs per SM stay resident and their loads carry enough bytes in flight (measured 71 -> ~60 us at cfg 3
  // against the register-heavy prefetching version)
  for (int k = beg + lane; k < end; k += 32) {
    const int c = col[k];
    double2 v[3 * B];
    double rv[B];
#pragma unroll
    for (int h = 0; h < 3 * B; h++) {
      // group-interleaved layout (Bsr::ival): block k = gb + lane of the group starting at gb = k - lane
      const int gb = k - lane, gs = min(32, end - gb);
      const double *q = val + (long)gb * 6 * B + lane;
      v[h].x = __ldg(q + (2 * h) * gs);
      v[h].y = __ldg(q + (2 * h + 1) * gs);
    }
#pragma unroll
    for (int e = 0; e < B; e++) rv[e] = r[(long)c * B + e];
#pragma unroll
    for (int h = 0; h < 3 * B; h++) {
      const int e0 = 2 * h, e1 = 2 * h + 1;
      acc[e0 / B] = __fma_rn(v[h].x, rv[e0 % B], acc[e0 / B]);
      acc[e1 / B] = __fma_rn(v[h].y, rv[e1 % B], acc[e1 / B]);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
    for (int q = 0; q < 6; q++) acc[q] = acc[q] + __shfl_xor_sync(0xffffffffu, acc[q], o);
  if (lane < 6) {
    double vv = acc[0];
#pragma unroll
    for (int q = 1; q < 6; q++)
      if (lane == q) vv = acc[q];
    out[(long)w * 6 + lane] = vv;
  }
}

// CTA size of k_restrict_row: two warps, so that the ~1k warps of level 1 spread over all 148 SMs
constexpr int RCTA = 64;

// One warp per SCALAR row of R (6 per coarse block row): the same lane-strided chain and butterfly per
// scalar row as k_restrict (C5), with 6x more warps for the latency-bound coarse levels.
template <int B>
__global__ void __launch_bounds__(RCTA) k_restrict_row(int nrows6, const int *__restrict__ ptr,
                                                      const int *__restrict__ col, const double *__restrict__ val,
                                                      const double *__restrict__ r, double *__restrict__ out) {
  const int w = (blockIdx.x * RCTA + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows6) return;  // warp-uniform
  pdl_wait();
  const int a = w / 6, rr = w % 6;
  const int beg = ptr[a], end = ptr[a + 1];
  double acc = 0.0;
  // software pipeline over batches of U lane-strided blocks (k, k+32, ...; U = 4: 18 -> 15 us at cfg 3, with
  // 64-thread CTAs 13 us): the next batch's values and
  // r entries are in flight while this batch's FMAs run, its columns one batch further ahead; the chain
  // still runs over the lane's blocks in ascending order (C5).  Indices are clamped so that every load
  // is unconditional.
  constexpr int U = 4;
  if (beg + lane < end) {
    const int last = end - 1;
    double v[U][B], rv[U][B];
    int cn[U];
    int k0 = beg + lane;
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int kk = min(k0 + 32 * u, last);
      const int cc = col[kk];
#pragma unroll
      for (int e = 0; e < B; e++) { v[u][e] = __ldg(val + (long)kk * 6 * B + rr * B + e); rv[u][e] = r[(long)cc * B + e]; }
    }
#pragma unroll
    for (int u = 0; u < U; u++) cn[u] = col[min(k0 + 32 * (U + u), last)];
    for (; k0 < end; k0 += U * 32) {
      double vn[U][B], rn[U][B];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int kk = min(k0 + 32 * (U + u), last);
#pragma unroll
        for (int e = 0; e < B; e++) { vn[u][e] = __ldg(val + (long)kk * 6 * B + rr * B + e); rn[u][e] = r[(long)cn[u] * B + e]; }
      }
#pragma unroll
      for (int u = 0; u < U; u++) cn[u] = col[min(k0 + 32 * (2 * U + u), last)];
#pragma unroll
      for (int u = 0; u < U; u++)
        if (k0 + 32 * u < end)
#pragma unroll
          for (int e = 0; e < B; e++) acc = __fma_rn(v[u][e], rv[u][e], acc);
#pragma unroll
      for (int u = 0; u < U; u++)
#pragma unroll
        for (int e = 0; e < B; e++) { v[u][e] = vn[u][e]; rv[u][e] = rn[u][e]; }
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc = acc + __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[w] = acc;
}

void launch_restrict(Ctx &c, const Bsr &R, const double *r, double *bc) {
  if (R.nbr == 0) return;
  long threads = (long)R.nbr * 32;
  // level 0 (3 x 3 -> 6 x 3 blocks): one warp per coarse block row moves full blocks (measured 69 us at cfg 3
  // vs 112 us split by scalar row); coarse levels are latency-bound: one warp per scalar row (23 vs 31 us)
  // (level 0 reads the group-interleaved copy of R's values: 68 -> 59 us at cfg 3)
  if (R.bc == 3) {
    REQUIRE(R.ival, AMGF_ERR_ARG, "restriction: interleaved R values missing");
    go(c, sell_pdl(), k_restrict<3>, nblk(threads), CTA, R.nbr, R.ptr, R.col, (const double *)R.ival, r, bc);
  }
  else go(c, sell_pdl(), k_restrict_row<6>, nblk(threads * 6, RCTA), RCTA, R.nbr * 6, R.ptr, R.col, (const double *)R.val, r, bc);
  after_launch(c, __func__);
}

// ------------------------------------------------------------------ vector kernels
__global__ void k_jacobi0(long n, const double *__restrict__ b, const double *__restrict__ d, double *__restrict__ x) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) x[i] = b[i] / d[i];
}
__global__ void k_copy(long n, const double *__restrict__ s, double *__restrict__ d) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) d[i] = s[i];
}
__global__ void k_zero(long n, double *__restrict__ d) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) d[i] = 0.0;
}
__global__ void k_add(long n, const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ o) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) o[i] = a[i] + b[i];
}
// x = fma(alpha, p, x); r = fma(-alpha, q, r)   (C15)
__global__ void k_axpy2(long n, const Scalars *__restrict__ sc, const double *__restrict__ p,
                        const double *__restrict__ q, double *__restrict__ x, double *__restrict__ r) {
  const double a = sc->alpha;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    x[i] = __fma_rn(a, p[i], x[i]);
    r[i] = __fma_rn(-a, q[i], r[i]);
  }
}
// p = fma(beta, p, z)   (C15)
__global__ void k_xpby(long n, const Scalars *__restrict__ sc, const double *__restrict__ z, double *__restrict__ p) {
  pdl_wait();
  const double be = sc->beta;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    p[i] = __fma_rn(be, p[i], z[i]);
}
__global__ void k_xpby_v2(long n2, const Scalars *__restrict__ sc, const double2 *__restrict__ z,
                          double2 *__restrict__ p) {
  pdl_wait();  // beta is the previous kernel's result
  const double be = sc->beta;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) {
    const double2 zz = z[i];
    double2 pp = p[i];
    pp.x = __fma_rn(be, pp.x, zz.x);
    pp.y = __fma_rn(be, pp.y, zz.y);
    p[i] = pp;
  }
}

static int vgrid(long n) {
  long g = (n + CTA - 1) / CTA;
  return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

void launch_jacobi0(Ctx &c, long n, const double *b, const double *d, double *x) {
  k_jacobi0<<<vgrid(n), CTA, 0, c.stream>>>(n, b, d, x); after_launch(c, __func__);
}
void launch_copy(Ctx &c, long n, const double *s, double *d) {
  k_copy<<<vgrid(n), CTA, 0, c.stream>>>(n, s, d); after_launch(c, __func__);
}
void launch_zero(Ctx &c, long n, double *d) {
  k_zero<<<vgrid(n), CTA, 0, c.stream>>>(n, d); after_launch(c, __func__);
}
void launch_add(Ctx &c, long n, const double *a, const double *b, double *o) {
  k_add<<<vgrid(n), CTA, 0, c.stream>>>(n, a, b, o); after_launch(c, __func__);
}
void launch_axpy2(Ctx &c, long n, const double *p, const double *q, double *x, double *r) {
  k_axpy2<<<vgrid(n), CTA, 0, c.stream>>>(n, c.sc, p, q, x, r); after_launch(c, __func__);
}
void launch_xpby(Ctx &c, long n, const double *z, double *p) {
  if (pairs_ok(n, {z, p}))
    go(c, sell_pdl(), k_xpby_v2, vgrid(n / 2), CTA, n / 2, (const Scalars *)c.sc, (const double2 *)z, (double2 *)p);
  else
    go(c, sell_pdl(), k_xpby, vgrid(n), CTA, n, (const Scalars *)c.sc, z, p);
  after_launch(c, __func__);
}

// ------------------------------------------------------------------ dots (C14, C15)
__global__ void __launch_bounds__(CTA) k_dot1(long nb, int b, const double *__restrict__ u,
                                              const double *__restrict__ v, double *__restrict__ part) {
  __shared__ double red[CTA];
  const long i = blockIdx.x * (long)CTA + threadIdx.x;
  double s = 0.0;
  if (i < nb)
    for (int e = 0; e < b; e++) s = __fma_rn(u[i * b + e], v[i * b + e], s);
  double tot = cta_tree(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(CTA) k_dot2(long C, const double *__restrict__ part, Scalars *sc, int kind, int *err) {
  __shared__ double red[CTA];
  pdl_wait();  // the partials are the previous kernel's result
  double acc = 0.0;
  // the same sequential sum per thread (c = tid, tid + CTA, ...), its loads issued 8 at a time
  long c = threadIdx.x;
  for (; c + 7 * CTA < C; c += 8 * CTA) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = part[c + u * CTA];
#pragma unroll
    for (int u = 0; u < 8; u++) acc = acc + v[u];
  }
  for (; c < C; c += CTA) acc = acc + part[c];
  double s = cta_tree(acc, red);
  if (threadIdx.x == 0) {
    switch (kind) {
      case DOT_PLAIN: sc->dot = s; break;
      case DOT_PI:
        sc->pi = s;
        if (!(s > 0.0)) raise_err(err, DERR_BREAKDOWN, 1);
        sc->alpha = sc->rho / s;
        break;
      case DOT_RHO0: sc->rho0 = s; sc->rho = s; sc->rho1 = s; break;
      case DOT_RHO1:
        sc->rho1 = s;
        if (s < 0.0) raise_err(err, DERR_BREAKDOWN, 2);
        sc->beta = s / sc->rho;
        sc->rho = s;
        break;
    }
  }
}

// power step (C18) dot partials: C14 level 1 of w.w and v.v in one pass (block rows of b entries)
__global__ void __launch_bounds__(CTA) k_pow_dots(long nb, int b, const double *__restrict__ w,
                                                  const double *__restrict__ v, double *__restrict__ pw_,
                                                  double *__restrict__ pv_) {
  __shared__ double red[CTA];
  const long i = blockIdx.x * (long)CTA + threadIdx.x;
  double sw = 0.0, sv = 0.0;
  if (i < nb) {
    for (int e = 0; e < b; e++) sw = __fma_rn(w[i * b + e], w[i * b + e], sw);
    for (int e = 0; e < b; e++) sv = __fma_rn(v[i * b + e], v[i * b + e], sv);
  }
  const double tw = cta_tree(sw, red);
  const double tv = cta_tree(sv, red);
  if (threadIdx.x == 0) {
    pw_[blockIdx.x] = tw;
    pv_[blockIdx.x] = tv;
  }
}
// C14 level 2 of both partial arrays (the k_dot2 order): pw[0] = w.w, pw[1] = v.v
__device__ __forceinline__ double dot_level2(long C, const double *__restrict__ part, double *red) {
  double acc = 0.0;
  long c = threadIdx.x;
  for (; c + 7 * CTA < C; c += 8 * CTA) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = part[c + u * CTA];
#pragma unroll
    for (int u = 0; u < 8; u++) acc = acc + v[u];
  }
  for (; c < C; c += CTA) acc = acc + part[c];
  return cta_tree(acc, red);
}
__global__ void __launch_bounds__(CTA) k_pow_fin(long C, const double *__restrict__ pw_, const double *__restrict__ pv_,
                                                 double *__restrict__ pw) {
  __shared__ double red[CTA];
  const double sw = dot_level2(C, pw_, red);
  const double sv = dot_level2(C, pv_, red);
  if (threadIdx.x == 0) {
    pw[0] = sw;
    pw[1] = sv;
  }
}
// k_pow_fin and k_pow_scale in one launch for levels with few partials: every CTA forms both level-2 sums
// itself (the k_pow_fin arithmetic), then scales its elements: v = w / ||w||; block 0 stores the scalars
__global__ void __launch_bounds__(CTA) k_pow_fin_scale(long C, const double *__restrict__ pw_,
                                                       const double *__restrict__ pv_, double *__restrict__ pw,
                                                       long n, const double *__restrict__ w, double *__restrict__ v) {
  __shared__ double red[CTA];
  const double sw = dot_level2(C, pw_, red);
  const double sv = dot_level2(C, pv_, red);
  const double nw = sqrt(sw);
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i == 0) {
    pw[0] = sw;
    pw[1] = sv;
    const double lam = nw / sqrt(sv);
    pw[2] = lam;
    pw[3] = 4.0 / (3.0 * lam);  // R6 (k_pow_scale's formula)
  }
  if (i < n) v[i] = w[i] / nw;
}
void launch_pow_fin_scale(Ctx &c, long C, const double *part_w, const double *part_v, double *pw, long n,
                          const double *w, double *v) {
  k_pow_fin_scale<<<nblk(n), CTA, 0, c.stream>>>(C, part_w, part_v, pw, n, w, v);
  after_launch(c, __func__);
}
void launch_pow_dots(Ctx &c, long nb, int b, const double *w, const double *v, double *part_w, double *part_v) {
  const long C = (nb + CTA - 1) / CTA;
  if (C > 0) k_pow_dots<<<(int)C, CTA, 0, c.stream>>>(nb, b, w, v, part_w, part_v);
  after_launch(c, __func__);
}
void launch_pow_fin(Ctx &c, long C, const double *part_w, const double *part_v, double *pw) {
  k_pow_fin<<<1, CTA, 0, c.stream>>>(C, part_w, part_v, pw);
  after_launch(c, __func__);
}

void launch_dot_finish(Ctx &c, long C, int finish) {
  go(c, sell_pdl(), k_dot2, 1, CTA, C, (const double *)c.dot_part, c.sc, finish, c.err);
  after_launch(c, __func__);
}

void launch_dot(Ctx &c, long n, int b, const double *u, const double *v, int finish) {
  long nb = n / b;
  long C = (nb + CTA - 1) / CTA;
  if (C > 0) {
    k_dot1<<<(int)C, CTA, 0, c.stream>>>(nb, b, u, v, c.dot_part);
    after_launch(c, "k_dot1");
  }
  k_dot2<<<1, CTA, 0, c.stream>>>(C, c.dot_part, c.sc, finish, c.err);
  after_launch(c, __func__);
}

// ------------------------------------------------------------------ banded triangular solves (C10)


// One warp solves L L^T y = v[gather] (C10).  Forward: column sweep j ascending over Lcol
// (Lcol[j*W + t] = L_{j+t,j}); backward: row sweep k descending over Lrev (Lrev[k*W + d] = L_{k,k-d}).
// Lane l keeps the accumulators of rows j0 + l + 32 s (s < R, 32(R-1) >= bw) in registers.  Each round of
// 32 pivots stages its 32 band columns (rows) in shared memory with row stride Ws = 32 R, zero beyond the
// band, so that every update is an unconditional FMA: out-of-band terms are exact zeros (fma(-0, y, a) = a)
// and updates of already finished rows are dead.  Lane jj issues the TMA bulk copy of the round's jj-th
// column; the next round's copies are in flight while the current round computes (double buffer).
// x[idx[a]] += y[a] for a < n by one warp, 8 independent elements per lane in flight
__device__ __forceinline__ void scatter_add_warp(int n, const int *__restrict__ idx, const double *__restrict__ y,
                                                 double *__restrict__ x, int lane) {
  for (int a0 = 0; a0 < n; a0 += 32 * 8) {
    int id[8];
    double yv[8], xv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int a = a0 + 32 * u + lane;
      id[u] = a < n ? idx[a] : -1;
      yv[u] = a < n ? y[a] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) xv[u] = id[u] >= 0 ? x[id[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (id[u] >= 0) x[id[u]] = xv[u] + yv[u];
  }
}
// y[a] = v[idx[a]] (or v[a]) by one warp, batched
__device__ __forceinline__ void gather_warp(int n, const int *__restrict__ idx, const double *__restrict__ v,
                                            double *__restrict__ y, int lane) {
  for (int a0 = 0; a0 < n; a0 += 32 * 8) {
    int id[8];
    double vv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int a = a0 + 32 * u + lane;
      id[u] = a < n ? (idx ? idx[a] : a) : -1;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) vv[u] = id[u] >= 0 ? v[id[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (a0 + 32 * u + lane < n) y[a0 + 32 * u + lane] = vv[u];
  }
}

template <int R, int NB>
__global__ void __launch_bounds__(32) k_band_trsv(int n, int bw, const double *__restrict__ Lcol,
                                                  const double *__restrict__ Lrev, const double *__restrict__ dinv,
                                                  const double *__restrict__ v, const int *__restrict__ gather,
                                                  double *__restrict__ y, const int *__restrict__ scatter,
                                                  double *__restrict__ xout, double *__restrict__ w) {
  constexpr int Ws = 32 * R;               // = band storage stride (band_stride)
  constexpr unsigned CHUNK = 32u * Ws * 8u; // one round = 32 consecutive band columns / rows
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[NB];
  const int lane = threadIdx.x;
  const int F = (n + 31) / 32;  // rounds per sweep
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; b++) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  // stage global round g (forward g < F: columns 32g..32g+31; backward: rows k1-31..k1) into buffer g % NB
  auto issue = [&](int g) {
    if (g >= 2 * F || lane != 0) return;
    const double *src = (g < F) ? Lcol + (long)(32 * g) * Ws : Lrev + (long)(n - 1 - 32 * (g - F) - 31) * Ws;
    uint64_t *br = &bar[g % NB];
    mbar_arrive_expect(br, CHUNK);
    bulk_g2s(sm + (g % NB) * 32 * Ws, src, CHUNK, br);
  };
#pragma unroll
  for (int g = 0; g < NB - 1; g++) issue(g);
  gather_warp(n, gather, v, y, lane);
  __syncwarp();
  double acc[R];
  // ---------------- forward: w = L^{-1} y (column sweep)
#pragma unroll
  for (int s = 0; s < R; s++) acc[s] = (lane + 32 * s < n) ? y[lane + 32 * s] : 0.0;
  double dv = (lane < n) ? dinv[lane] : 0.0;
  double vq1, dq1;  // operands of the next round, loaded one round ahead
  {
    const int i1 = 32 + lane + 32 * (R - 1);
    vq1 = (i1 < n) ? y[i1] : 0.0;
    dq1 = (32 + lane < n) ? dinv[32 + lane] : 0.0;
  }
  for (int q = 0; q < F; q++) {
    const int j0 = 32 * q;
    __syncwarp();
    fence_proxy_async();
    issue(q + NB - 1);
    const int i2 = j0 + 64 + lane + 32 * (R - 1);
    const double vq2 = (i2 < n) ? y[i2] : 0.0;
    const double dq2 = (j0 + 64 + lane < n) ? dinv[j0 + 64 + lane] : 0.0;
    mbar_wait(&bar[q % NB], (q / NB) & 1);
    // column jj of the round at cur + jj*Ws; row i = j0+lane+32s is at offset t = lane + 32s - jj
    const double *cur = sm + (q % NB) * 32 * Ws + lane;
    double lc[R], mine = 0.0;
#pragma unroll
    for (int s = 0; s < R; s++) lc[s] = cur[32 * s];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      if (j0 + jj >= n) break;
      double ln[R];  // band values of the next pivot, loaded before this pivot's broadcast
#pragma unroll
      for (int s = 0; s < R; s++) ln[s] = cur[((jj + 1) & 31) * (Ws - 1) + 32 * s];
      const double yj = __shfl_sync(0xffffffffu, acc[0] * dv, jj);
      mine = (lane == jj) ? yj : mine;
#pragma unroll
      for (int s = 0; s < R; s++) acc[s] = __fma_rn(-lc[s], yj, acc[s]);
#pragma unroll
      for (int s = 0; s < R; s++) lc[s] = ln[s];
    }
    if (j0 + lane < n) w[j0 + lane] = mine;
#pragma unroll
    for (int s = 0; s < R - 1; s++) acc[s] = acc[s + 1];
    acc[R - 1] = vq1;
    dv = dq1;
    vq1 = vq2;
    dq1 = dq2;
  }
  __syncwarp();
  // ---------------- backward: y = L^{-T} w (row sweep), pivots k = k1 - jj, k1 = n-1-32q
#pragma unroll
  for (int s = 0; s < R; s++) {
    const int i = n - 1 - lane - 32 * s;
    acc[s] = (i >= 0) ? w[i] : 0.0;
  }
  dv = (n - 1 - lane >= 0) ? dinv[n - 1 - lane] : 0.0;
  {
    const int i1 = n - 1 - 32 - lane - 32 * (R - 1);
    vq1 = (i1 >= 0) ? w[i1] : 0.0;
    dq1 = (n - 1 - 32 - lane >= 0) ? dinv[n - 1 - 32 - lane] : 0.0;
  }
  for (int q = 0; q < F; q++) {
    const int g = F + q;
    const int k1 = n - 1 - 32 * q;
    __syncwarp();
    fence_proxy_async();
    issue(g + NB - 1);
    const int i2 = k1 - 64 - lane - 32 * (R - 1);
    const double wnew = (i2 >= 0) ? w[i2] : 0.0;
    const double dq2 = (k1 - 64 - lane >= 0) ? dinv[k1 - 64 - lane] : 0.0;
    mbar_wait(&bar[g % NB], (g / NB) & 1);
    // row k = k1 - jj of the round at cur + (31 - jj)*Ws; row i = k1-lane-32s at offset d = lane + 32s - jj
    const double *cur = sm + (g % NB) * 32 * Ws + lane;
    double lc[R], mine = 0.0;
#pragma unroll
    for (int s = 0; s < R; s++) lc[s] = cur[31 * Ws + 32 * s];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      if (k1 - jj < 0) break;
      double ln[R];
#pragma unroll
      for (int s = 0; s < R; s++) ln[s] = cur[(31 - ((jj + 1) & 31)) * Ws - ((jj + 1) & 31) + 32 * s];
      const double xk = __shfl_sync(0xffffffffu, acc[0] * dv, jj);
      mine = (lane == jj) ? xk : mine;
#pragma unroll
      for (int s = 0; s < R; s++) acc[s] = __fma_rn(-lc[s], xk, acc[s]);
#pragma unroll
      for (int s = 0; s < R; s++) lc[s] = ln[s];
    }
    if (k1 - lane >= 0) y[k1 - lane] = mine;
#pragma unroll
    for (int s = 0; s < R - 1; s++) acc[s] = acc[s + 1];
    acc[R - 1] = vq1;
    dv = dq1;
    vq1 = wnew;
    dq1 = dq2;
  }
  __syncwarp();
  if (scatter) scatter_add_warp(n, scatter, y, xout, lane);
}

}  // namespace amgf
#include "band_sweep.cuh"
namespace amgf {

template <int R, int NB, bool BLOCKED>
static void sweep_RN(Ctx &c, int nblocks, const int *p0, const int *len, int bw, bool fwd, const double *Lcol,
                     const double *Lrev, const double *dinv, const double *in, const int *gather, double *out,
                     double *out_shift) {
  const size_t smem = (size_t)NB * 32 * (32 * R) * sizeof(double);
  size_t &attr_f = device_slot((const void *)k_band_sweep<R, NB, true, BLOCKED>);
  size_t &attr_b = device_slot((const void *)k_band_sweep<R, NB, false, BLOCKED>);
  if (fwd) {
    if (!attr_f) {
      CK(cudaFuncSetAttribute(k_band_sweep<R, NB, true, BLOCKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
      attr_f = 1;
    }
    launch_pdl(c.stream, k_band_sweep<R, NB, true, BLOCKED>, dim3(nblocks), dim3(32), smem, p0, len, bw, Lcol, Lrev,
               dinv, in, gather, out, out_shift);
  } else {
    if (!attr_b) {
      CK(cudaFuncSetAttribute(k_band_sweep<R, NB, false, BLOCKED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
      attr_b = 1;
    }
    launch_pdl(c.stream, k_band_sweep<R, NB, false, BLOCKED>, dim3(nblocks), dim3(32), smem, p0, len, bw, Lcol,
               Lrev, dinv, in, gather, out, out_shift);
  }
}

template <int R>
static void sweep_R(Ctx &c, int nblocks, const int *p0, const int *len, int bw, bool fwd, const double *Lcol,
                    const double *Lrev, const double *dinv, const double *in, const int *gather, double *out,
                    double *out_shift) {
  // as many rounds in flight as 220 KB of shared memory allow (2 stages measured slower at cfg 3)
  constexpr int NB = (220 * 1024) / (32 * 32 * R * 8) >= 4 ? 4 : 3;
  // per-pivot form: the blocked form (triangle, then the rows below) measured 150 vs 99 cycles per pivot
  // (tools/mb_sweep.cu), so it is kept only as a microbenchmark variant
  sweep_RN<R, NB, false>(c, nblocks, p0, len, bw, fwd, Lcol, Lrev, dinv, in, gather, out, out_shift);
}

// Generic fallback sweep for wide bands: one CTA per block, barrier per pivot.
__global__ void __launch_bounds__(1024) k_band_sweep_wide(const int *blk_p0, const int *blk_len, int bw, int W, bool fwd,
                                                          const double *__restrict__ Lcol,
                                                          const double *__restrict__ Lrev,
                                                          const double *__restrict__ dinv,
                                                          const double *__restrict__ in, const int *__restrict__ gather,
                                                          double *__restrict__ out, double *__restrict__ out_shift) {
  __shared__ double piv;
  const int p0 = blk_p0[blockIdx.x], n = blk_len[blockIdx.x];
  for (int t = threadIdx.x; t < n; t += blockDim.x) out[p0 + t] = gather ? in[gather[p0 + t]] : in[p0 + t];
  __syncthreads();
  for (int u = 0; u < n; u++) {
    const int j = fwd ? p0 + u : p0 + n - 1 - u;
    if (threadIdx.x == 0) { piv = out[j] * dinv[j]; out[j] = piv; }
    __syncthreads();
    const double yj = piv;
    for (int d = 1 + threadIdx.x; d <= bw; d += blockDim.x) {
      const int i = fwd ? j + d : j - d;
      if (i < p0 || i >= p0 + n) continue;
      const double l = fwd ? Lcol[(long)j * W + d] : Lrev[(long)j * W + d];
      out[i] = __fma_rn(-l, yj, out[i]);
    }
    __syncthreads();
  }
  if (out_shift)
    for (int t = threadIdx.x; t < n; t += blockDim.x) out_shift[p0 + t + 1] = out[p0 + t];
}

// Separator rows against a factored diagonal block B (the A_w factorization's off-block part, C9):
// L_sj = (a_sj - sum_{k in B, k < j} L_sk L_jk) / L_jj for j in B ascending -- a forward substitution with B's
// band factor whose right-hand side is the separator row, so it runs as the solve's warp sweep (column TMA ring,
// shuffle broadcast of the pivot, one FMA per window entry per pivot; acc = fma(-L_jk, L_sk, acc) is the C9
// term fma(-L_sk, L_jk, acc) with the operands swapped, the same correctly rounded result) instead of one
// (bw)-term chain per entry.  The pivot is divided by L_jj (C9), not multiplied by 1/L_jj.  A CTA of G warps
// takes G consecutive rows of the separator and shares B's band rounds (stage refill after a CTA barrier).
// grid: (pairs, ceil(max separator length / G)); rows are read and written in place in Loff.
template <int R, int NB, int G>
__global__ void __launch_bounds__(32 * G) k_sep_rows_sweep(const int2 *__restrict__ pairs, const NdBlk *__restrict__ blk,
                                                          const double *__restrict__ Lcol, double *__restrict__ Loff) {
  constexpr int Ws = 32 * R;
  constexpr unsigned CHUNK = 32u * Ws * 8u;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar[NB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const NdBlk S = blk[pairs[blockIdx.x].x], B = blk[pairs[blockIdx.x].y];
  const int s = blockIdx.y * G + warp;
  if ((int)(blockIdx.y * G) >= S.len) return;  // whole CTA beyond the separator
  const bool act = s < S.len;
  double *row = Loff + S.off + (long)(act ? s : 0) * S.rs - S.t0;  // row[k] = entry (p0(S) + s, k), k in B
  const int p0 = B.p0, n = B.len;
  const int F = (n + 31) / 32;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int b = 0; b < NB; b++) mbar_init(&bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int g) {
    if (g >= F || threadIdx.x != 0) return;
    uint64_t *br = &bar[g % NB];
    mbar_arrive_expect(br, CHUNK);
    bulk_g2s(sm + (g % NB) * 32 * Ws, Lcol + (long)(p0 + 32 * g) * Ws, CHUNK, br);
  };
#pragma unroll
  for (int g = 0; g < NB - 1; g++) issue(g);
  auto ld_in = [&](int t) -> double { return (act && t < n) ? row[p0 + t] : 0.0; };
  auto ld_d = [&](int t) -> double { return t < n ? Lcol[(long)(p0 + t) * Ws] : 1.0; };  // L_jj
  double acc[R];
#pragma unroll
  for (int q = 0; q < R; q++) acc[q] = ld_in(lane + 32 * q);
  double vq1 = ld_in(32 + lane + 32 * (R - 1));
  double dv = ld_d(lane), dq1 = ld_d(32 + lane);
  for (int q = 0; q < F; q++) {
    const int t0 = 32 * q;
    __syncthreads();  // every warp is done with the stage refilled next
    fence_proxy_async();
    issue(q + NB - 1);
    const double vq2 = ld_in(t0 + 64 + lane + 32 * (R - 1));
    const double dq2 = ld_d(t0 + 64 + lane);
    mbar_wait(&bar[q % NB], (q / NB) & 1);
    const double *cur = sm + (q % NB) * 32 * Ws + lane;
    double mine = 0.0, lc[R];
#pragma unroll
    for (int u = 0; u < R; u++) lc[u] = cur[32 * u];
#pragma unroll
    for (int jj = 0; jj < 32; jj++) {
      if (t0 + jj >= n) break;
      double ln[R];
      const int jn = (jj + 1) & 31;
#pragma unroll
      for (int u = 0; u < R; u++) ln[u] = cur[jn * (Ws - 1) + 32 * u];
      const double yj = __shfl_sync(0xffffffffu, acc[0] / dv, jj);
      mine = (lane == jj) ? yj : mine;
#pragma unroll
      for (int u = 0; u < R; u++) acc[u] = __fma_rn(-lc[u], yj, acc[u]);
#pragma unroll
      for (int u = 0; u < R; u++) lc[u] = ln[u];
    }
    if (act && t0 + lane < n) row[p0 + t0 + lane] = mine;
#pragma unroll
    for (int u = 0; u < R - 1; u++) acc[u] = acc[u + 1];
    acc[R - 1] = vq1;
    dv = dq1;
    vq1 = vq2;
    dq1 = dq2;
  }
}

template <int R>
static void sep_rows_R(Ctx &c, int np, const int *pairs, const NdBlk *blk, int maxsep, const double *Lcol,
                       double *Loff) {
  constexpr int NB = 2, G = 4;
  const size_t smem = (size_t)NB * 32 * (32 * R) * sizeof(double);
  size_t &attr = device_slot((const void *)k_sep_rows_sweep<R, NB, G>);
  if (smem > attr) {
    CK(cudaFuncSetAttribute(k_sep_rows_sweep<R, NB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const dim3 grid(np, (maxsep + G - 1) / G);
  k_sep_rows_sweep<R, NB, G><<<grid, 32 * G, smem, c.stream>>>((const int2 *)pairs, blk, Lcol, Loff);
  after_launch(c, "k_sep_rows_sweep");
}

bool launch_sep_rows_sweep(Ctx &c, int np, const int *pairs, const void *blk, int maxsep, int bw, const double *Lcol,
                           double *Loff) {
  if (!np) return true;
  const NdBlk *b = (const NdBlk *)blk;
  switch ((bw + 31) / 32 + 1) {
    case 1: case 2: sep_rows_R<2>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    case 3: sep_rows_R<3>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    case 4: sep_rows_R<4>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    case 5: sep_rows_R<5>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    case 6: sep_rows_R<6>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    case 7: sep_rows_R<7>(c, np, pairs, b, maxsep, Lcol, Loff); return true;
    default: return false;  // R = 8 needs 128 KB per stage pair: the shared-memory ring kernel instead
  }
}

void launch_band_sweep(Ctx &c, int nblocks, const int *d_p0, const int *d_len, int max_len, int bw, bool forward,
                       const double *Lcol, const double *Lrev, const double *dinv, const double *in, const int *gather,
                       double *out, double *out_shift) {
  if (nblocks == 0 || max_len == 0) return;
  const int R = (bw + 31) / 32 + 1;
  switch (R) {
    case 1: case 2: sweep_R<2>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 3: sweep_R<3>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 4: sweep_R<4>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 5: sweep_R<5>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 6: sweep_R<6>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 7: sweep_R<7>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    case 8: sweep_R<8>(c, nblocks, d_p0, d_len, bw, forward, Lcol, Lrev, dinv, in, gather, out, out_shift); break;
    default:
      k_band_sweep_wide<<<nblocks, 1024, 0, c.stream>>>(d_p0, d_len, bw, band_stride(bw), forward, Lcol, Lrev, dinv,
                                                        in, gather, out, out_shift);
  }
  after_launch(c, "k_band_sweep");
}

// Generic fallback for wide bands: one CTA, thread per row of the window, barrier per pivot.
__global__ void __launch_bounds__(1024) k_band_trsv_wide(int n, int bw, const double *__restrict__ Lcol,
                                                         const double *__restrict__ Lrev,
                                                         const double *__restrict__ dinv, const double *__restrict__ v,
                                                         const int *__restrict__ gather, double *__restrict__ y,
                                                         const int *__restrict__ scatter, double *__restrict__ xout,
                                                         double *__restrict__ w) {
  __shared__ double piv;
  const int W = band_stride(bw);
  for (int i = threadIdx.x; i < n; i += blockDim.x) w[i] = gather ? v[gather[i]] : v[i];
  __syncthreads();
  for (int j = 0; j < n; j++) {
    if (threadIdx.x == 0) { piv = w[j] * dinv[j]; w[j] = piv; }
    __syncthreads();
    const double yj = piv;
    for (int i = j + 1 + threadIdx.x; i <= j + bw && i < n; i += blockDim.x)
      w[i] = __fma_rn(-Lcol[(long)j * W + (i - j)], yj, w[i]);
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = w[i];
  __syncthreads();
  for (int k = n - 1; k >= 0; k--) {
    if (threadIdx.x == 0) { piv = y[k] * dinv[k]; y[k] = piv; }
    __syncthreads();
    const double xk = piv;
    for (int i = k - 1 - threadIdx.x; i >= k - bw && i >= 0; i -= blockDim.x)
      y[i] = __fma_rn(-Lrev[(long)k * W + (k - i)], xk, y[i]);
    __syncthreads();
  }
  if (scatter)
    for (int a = threadIdx.x; a < n; a += blockDim.x) xout[scatter[a]] = xout[scatter[a]] + y[a];
}

template <int R>
static void trsv_R(Ctx &c, int n, int bw, const double *Lcol, const double *Lrev, const double *dinv,
                   const double *v, const int *gather, double *y, const int *scatter, double *xout, double *w) {
  // as many rounds in flight as 220 KB of shared memory allow (TMA latency > one round of 32 pivots)
  constexpr int NB = (220 * 1024) / (32 * 32 * R * 8) >= 4 ? 4 : 3;
  const size_t smem = (size_t)NB * 32 * (32 * R) * sizeof(double);
  size_t &attr_set = device_slot((const void *)k_band_trsv<R, NB>);
  if (!attr_set) {
    CK(cudaFuncSetAttribute(k_band_trsv<R, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = 1;
  }
  k_band_trsv<R, NB><<<1, 32, smem, c.stream>>>(n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, w);
}

void launch_band_trsv(Ctx &c, int n, int bw, const double *Lcol, const double *Lrev, const double *dinv,
                      const double *v, const int *gather, double *y, const int *scatter, double *xout,
                      double *work) {
  if (n == 0) return;
  const int R = (bw + 31) / 32 + 1;
  switch (R) {
    case 1: case 2: trsv_R<2>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 3: trsv_R<3>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 4: trsv_R<4>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 5: trsv_R<5>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 6: trsv_R<6>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 7: trsv_R<7>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    case 8: trsv_R<8>(c, n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work); break;
    default:
      k_band_trsv_wide<<<1, 1024, 0, c.stream>>>(n, bw, Lcol, Lrev, dinv, v, gather, y, scatter, xout, work);
  }
  after_launch(c, "k_band_trsv");
}

// ------------------------------------------------------------------ thin second residual (C11)
// threads [nthin, nthin + nsc) also do the filter scatter x2[sdof[p]] += y[p] (one launch for both)
__global__ void k_thin(int nthin, const int *__restrict__ rows, const int *__restrict__ ptr,
                       const int *__restrict__ pos, const double *__restrict__ val, const double *__restrict__ y,
                       double *__restrict__ r, int nsc, const int *__restrict__ sdof, double *__restrict__ x2) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nthin) {
    const int q = t - nthin;
    if (q < nsc) x2[sdof[q]] = x2[sdof[q]] + y[q];
    return;
  }
  double acc = 0.0;
  const int e0 = ptr[t], e1 = ptr[t + 1];
  const int p = rows[t];
  const double rp = r[p];
  // batches of 4 entries: positions, values and y gathers of a batch in flight together; chain order kept
  int e = e0;
  for (; e + 4 <= e1; e += 4) {
    int q[4];
    double v[4], yv[4];
#pragma unroll
    for (int u = 0; u < 4; u++) { q[u] = pos[e + u]; v[u] = val[e + u]; }
#pragma unroll
    for (int u = 0; u < 4; u++) yv[u] = y[q[u]];
#pragma unroll
    for (int u = 0; u < 4; u++) acc = __fma_rn(v[u], yv[u], acc);
  }
  for (; e < e1; e++) acc = __fma_rn(val[e], y[pos[e]], acc);
  r[p] = rp - acc;
}

void launch_thin_resid(Ctx &c, int nthin, const int *rows, const int *ptr, const int *pos, const double *val,
                       const double *y, double *r, int nsc, const int *sdof, double *x2) {
  if (nthin + nsc == 0) return;
  k_thin<<<nblk(nthin + nsc, 64), 64, 0, c.stream>>>(nthin, rows, ptr, pos, val, y, r, nsc, sdof,
                                                      x2);  // 64: spread over all SMs
  after_launch(c, __func__);
}

// ------------------------------------------------------------------ setup-side BSR SpMV (C2)
__global__ void k_bsr_spmv(int nbr, int br, int bc, const int *__restrict__ ptr, const int *__restrict__ col,
                           const double *__restrict__ val, const double *__restrict__ x, double *__restrict__ y) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)nbr * br) return;
  const int i = (int)(t / br), r = (int)(t % br);
  double acc = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; k++) {
    const double *v = val + (long)k * br * bc + (long)r * bc;
    const double *xs = x + (long)col[k] * bc;
    for (int e = 0; e < bc; e++) acc = __fma_rn(v[e], xs[e], acc);
  }
  y[t] = acc;
}

void launch_bsr_spmv(Ctx &c, const Bsr &A, const double *x, double *y) {
  long rows = (long)A.nbr * A.br;
  if (rows == 0) return;
  k_bsr_spmv<<<nblk(rows), CTA, 0, c.stream>>>(A.nbr, A.br, A.bc, A.ptr, A.col, A.val, x, y);
  after_launch(c, __func__);
}

}  // namespace amgf
