// setup.cu -- GPU setup of the AMGF preconditioner.  No CPU fallback:
// every step below is a device kernel; the host only sizes allocations and loops over levels.
//
//   s1 S = K + J^T D J (C1) ......... k_S_count/k_S_fill (pattern), k_S_values
//   s2 I_c, Z validation ............. k_mark_cols, k_check_Z / k_compact_Z
//   s3 A_w band + Cholesky (C9) ...... k_band_start, k_band_fill, k_band_chol, k_band_finish
//   s4 aggregation (C16) ............. k_cc_*, k_mis_* (fixed-priority local-max rounds), k_agg_*
//   s5 tentative P (C17) ............. k_qr (per-aggregate MGS)
//   s6 smoothed P (C18, C19) ......... k_pow_*, k_P_count/k_P_fill/k_P_values
//   s7 Galerkin (C20, C22) ........... transpose (stable radix sort), k_AP_*, k_G_*, k_sym
//   s8 l1 diagonal (C3), SELL-32 ..... k_diag, k_sell_pack
//   s9 coarsest dense Cholesky ....... k_band_chol with bw = n-1
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "devutil.cuh"

namespace amgf {

// ------------------------------------------------------------------ small helpers
template <class T>
static void h2d(Ctx &c, T *dst, const T *src, size_t n) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, c.stream));
}
template <class T>
static void d2d(Ctx &c, T *dst, const T *src, size_t n) {
  if (n) CK(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToDevice, c.stream));
}
template <class T>
static T d2h1(Ctx &c, const T *src) {
  T v;
  CK(cudaMemcpyAsync(&v, src, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  return v;
}
#define LAUNCH(kernel, n, ...)                                                   \
  do {                                                                           \
    long n_ = (n);                                                               \
    if (n_ > 0) {                                                                \
      kernel<<<nblk(n_), CTA, 0, c.stream>>>(__VA_ARGS__);                       \
      after_launch(c, #kernel);                                                  \
    }                                                                            \
  } while (0)

// exclusive scan of n ints into out[0..n] (out[n] = total); returns total
static long scan_ex(Ctx &c, const int *in, int *out, long n) {
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n + 1, c.stream));
  void *t = c.alloc<char>(tmp);
  // in[n] must exist: callers allocate n+1 and set in[n] = 0
  CK(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, (int)n + 1, c.stream));
  int tot = d2h1(c, out + n);
  c.release(t);
  return tot;
}

// stable sort of (key, val) int pairs
static void sort_pairs(Ctx &c, const int *kin, int *kout, const int *vin, int *vout, long n) {
  if (n == 0) return;
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, 32, c.stream));
  void *t = c.alloc<char>(tmp);
  CK(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, (int)n, 0, 32, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  c.release(t);
}

__global__ void k_gather_int(long n, const int *perm, const int *src, int *dst) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[perm[e]];
}
__global__ void k_count_valid(long n, const int *key, int nkeys, int *cnt) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n && key[i] < nkeys) atomicAdd(&cnt[key[i]], 1);
}
__global__ void k_iota(long n, int *a) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int)i;
}
__global__ void k_fill_int(long n, int *a, int v) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
__global__ void k_rowof(int nrows, const int *ptr, int *rowof) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows)
    for (int e = ptr[i]; e < ptr[i + 1]; e++) rowof[e] = i;
}
__global__ void k_count_keys(long n, const int *key, int *cnt) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&cnt[key[i]], 1);
}

__device__ __forceinline__ int bsearch_int(const int *a, int lo, int hi, int key) {  // [lo, hi)
  hi -= 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int v = a[mid];
    if (v == key) return mid;
    if (v < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

// insert into a sorted unique local list; returns false on overflow
__device__ __forceinline__ bool insert_unique(int *list, int &cnt, int cap, int v) {
  int lo = 0, hi = cnt - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    if (list[mid] == v) return true;
    if (list[mid] < v) lo = mid + 1; else hi = mid - 1;
  }
  if (cnt >= cap) return false;
  for (int q = cnt; q > lo; q--) list[q] = list[q - 1];
  list[lo] = v;
  cnt++;
  return true;
}

// ------------------------------------------------------------------ input checks
__global__ void k_check_finite(long n, const double *v, int *err, int code) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n && !isfinite(v[i])) raise_err(err, code, (int)i);
}
__global__ void k_check_pos(long n, const double *v, int *err) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n && !(v[i] > 0.0)) raise_err(err, DERR_DOMAIN, (int)i);
}

__global__ void k_check_nonneg(long n, const double *v, int *err) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n && !(v[i] >= 0.0)) raise_err(err, DERR_DOMAIN, (int)i);
}

// ------------------------------------------------------------------ s1: S = K + J^T D J
constexpr int SCAP = 96;

__device__ int contact_nodes(int I, const int *Jt_ptr, const int *Jt_row, const int *J_ptr, const int *J_col,
                             int *list, int *err) {
  int cnt = 0;
  for (int r = 0; r < 3; r++) {
    const int p = 3 * I + r;
    for (int t = Jt_ptr[p]; t < Jt_ptr[p + 1]; t++) {
      const int k = Jt_row[t];
      for (int f = J_ptr[k]; f < J_ptr[k + 1]; f++)
        if (!insert_unique(list, cnt, SCAP, J_col[f] / 3)) { raise_err(err, DERR_LIMIT, I); return cnt; }
    }
  }
  return cnt;
}

__global__ void k_S_count(int nodes, const int *K_ptr, const int *K_col, const int *Jt_ptr, const int *Jt_row,
                          const int *J_ptr, const int *J_col, int *cnt, int *err) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nodes) return;
  int list[SCAP];
  int nl = contact_nodes(I, Jt_ptr, Jt_row, J_ptr, J_col, list, err);
  int a = K_ptr[I], ae = K_ptr[I + 1], b = 0, u = 0;
  while (a < ae || b < nl) {
    if (b >= nl || (a < ae && K_col[a] < list[b])) a++;
    else if (a >= ae || list[b] < K_col[a]) b++;
    else { a++; b++; }
    u++;
  }
  cnt[I] = u;
}

__global__ void k_S_fill(int nodes, const int *K_ptr, const int *K_col, const int *Jt_ptr, const int *Jt_row,
                         const int *J_ptr, const int *J_col, const int *S_ptr, int *S_col, int *S_kblk, int *err) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= nodes) return;
  int list[SCAP];
  int nl = contact_nodes(I, Jt_ptr, Jt_row, J_ptr, J_col, list, err);
  int a = K_ptr[I], ae = K_ptr[I + 1], b = 0, w = S_ptr[I];
  while (a < ae || b < nl) {
    if (b >= nl || (a < ae && K_col[a] < list[b])) { S_col[w] = K_col[a]; S_kblk[w] = a; a++; }
    else if (a >= ae || list[b] < K_col[a]) { S_col[w] = list[b]; S_kblk[w] = -1; b++; }
    else { S_col[w] = K_col[a]; S_kblk[w] = a; a++; b++; }
    w++;
  }
}

// one thread per S block: C1
// S = K + J^T D J (C1); with the bound-constraint diagonals (Remark boundconstr, PAPER.md:271-295:
// A~ = K + J~^T D~ J~, J~ = [J; I; -I]) the diagonal entries continue the chain with the rows of I and -I:
// t = 1 * D_lo[p], fma(t, 1, acc); t = -1 * D_up[p], fma(t, -1, acc).
__global__ void k_S_values(long nnzb, const int *S_rowof, const int *S_col, const int *S_kblk, const double *K_val,
                           const int *Jt_ptr, const int *Jt_row, const double *Jt_val, const double *D,
                           const double *D_lo, const double *D_up, double *S_val) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool in = e < nnzb;
  const int I = in ? S_rowof[e] : 0, Jn = in ? S_col[e] : 0, kb = in ? S_kblk[e] : -1;
  // no constraint touches the row's dofs and no bound term: every chain is the K value alone
  const bool plain = in && Jt_ptr[3 * I] == Jt_ptr[3 * I + 3] && (Jn != I || !D_lo);
  // a warp of 32 such blocks over 32 consecutive K blocks: S's 288 values are K's, copied as coalesced rows
  const int kb0 = __shfl_sync(0xffffffffu, kb, 0);
  const long e0 = e - lane;
  if (__all_sync(0xffffffffu, plain && kb == kb0 + lane) && kb0 >= 0) {
#pragma unroll
    for (int q = 0; q < 9; q++) S_val[e0 * 9 + lane + 32 * q] = K_val[(long)kb0 * 9 + lane + 32 * q];
    return;
  }
  if (!in) return;
  if (plain) {
#pragma unroll
    for (int q = 0; q < 9; q++) S_val[e * 9 + q] = kb >= 0 ? K_val[(long)kb * 9 + q] : 0.0;
    return;
  }
  for (int r = 0; r < 3; r++)
    for (int cc = 0; cc < 3; cc++) {
      const int p = 3 * I + r, q = 3 * Jn + cc;
      double acc = kb >= 0 ? K_val[(long)kb * 9 + 3 * r + cc] : 0.0;
      int a = Jt_ptr[p], ae = Jt_ptr[p + 1], b = Jt_ptr[q], be = Jt_ptr[q + 1];
      while (a < ae && b < be) {
        const int ka = Jt_row[a], kb2 = Jt_row[b];
        if (ka < kb2) a++;
        else if (ka > kb2) b++;
        else {
          const double t = Jt_val[a] * D[ka];
          acc = __fma_rn(t, Jt_val[b], acc);
          a++; b++;
        }
      }
      if (p == q) {
        if (D_lo) { const double t = 1.0 * D_lo[p]; acc = __fma_rn(t, 1.0, acc); }
        if (D_up) { const double t = -1.0 * D_up[p]; acc = __fma_rn(t, -1.0, acc); }
      }
      S_val[e * 9 + 3 * r + cc] = acc;
    }
}

// ------------------------------------------------------------------ s2: I_c and Z
// Fixed tree of C14 over CTA values in shared memory (the solve kernels' cta_tree); returns the sum to all.
__device__ __forceinline__ double cta_tree_s(double v, double *sm) {
  const int t = threadIdx.x;
  sm[t] = v;
  __syncthreads();
#pragma unroll
  for (int w = CTA / 2; w >= 1; w >>= 1) {
    if (t < w) sm[t] = sm[t] + sm[t + w];
    __syncthreads();
  }
  const double r = sm[0];
  __syncthreads();
  return r;
}
// Fine-level SELL refresh fused with the l1 / point diagonals (same values as k_sell_vals + k_diag) and, when
// w is given, with the first power step (C18) of the level: one thread per block row I (the SELL-32 row,
// natural order at level 0) streams its BSR blocks in order, stores them to the SELL copy (one 256-byte
// segment per component across the 32 rows of a slice), forms the diagonals (C3) and the row chain of
// A v0 with v0_j = 1 + (j mod 7)/8 (C2, the SpMV's order), w = (A v0) / d, and the C14 level-1 partials of
// w.w and v0.v0 (thread I = block row 256 * CTA + t, as k_dot1).
__global__ void __launch_bounds__(CTA) k_sell_diag(int nodes, const int *__restrict__ S_ptr,
                                                   const int *__restrict__ S_col, const double *__restrict__ S_val,
                                                   const int *__restrict__ slice_ptr, double *__restrict__ sval,
                                                   double *__restrict__ dl1, double *__restrict__ dpt,
                                                   double *__restrict__ w, double *__restrict__ part_w,
                                                   double *__restrict__ part_v) {
  __shared__ double red[CTA];
  const int I = blockIdx.x * CTA + threadIdx.x;
  double sw = 0.0, sv = 0.0;
  if (I < nodes) {
    const int lane = I & 31;
    const long sbase = slice_ptr[I >> 5];
    const int e0 = S_ptr[I], e1 = S_ptr[I + 1];
    double d[3] = {0.0, 0.0, 0.0}, dp[3] = {0.0, 0.0, 0.0}, acc[3] = {0.0, 0.0, 0.0};
    // software pipeline: block e + 1's column and values are in flight while block e is stored and consumed
    int Jnx = 0;
    double vnx[9];
    if (e0 < e1) {
      Jnx = S_col[e0];
#pragma unroll
      for (int q = 0; q < 9; q++) vnx[q] = S_val[(long)e0 * 9 + q];
    }
    for (int e = e0; e < e1; e++) {
      const int Jn = Jnx;
      double v[9];
#pragma unroll
      for (int q = 0; q < 9; q++) v[q] = vnx[q];
      const int en = min(e + 1, e1 - 1);  // branch-free prefetch (the last block is re-read once)
      Jnx = S_col[en];
#pragma unroll
      for (int q = 0; q < 9; q++) vnx[q] = S_val[(long)en * 9 + q];
      const long slot = sbase + (e - e0);
#pragma unroll
      for (int q = 0; q < 9; q++) sval[(slot * 9 + q) * 32 + lane] = v[q];
#pragma unroll
      for (int r = 0; r < 3; r++)
#pragma unroll
        for (int cc = 0; cc < 3; cc++) {
          d[r] = d[r] + fabs(v[3 * r + cc]);
          if (Jn == I && cc == r) dp[r] = v[3 * r + cc];
        }
      if (w) {
#pragma unroll
        for (int cc = 0; cc < 3; cc++) {
          const double x0 = 1.0 + (double)((3L * Jn + cc) % 7) / 8.0;
#pragma unroll
          for (int r = 0; r < 3; r++) acc[r] = __fma_rn(v[3 * r + cc], x0, acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 3; r++) {
      dl1[3L * I + r] = d[r];
      dpt[3L * I + r] = dp[r];
    }
    if (w) {
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const double wi = acc[r] / dp[r];
        w[3L * I + r] = wi;
        sw = __fma_rn(wi, wi, sw);
      }
#pragma unroll
      for (int r = 0; r < 3; r++) {
        const double x0 = 1.0 + (double)((3L * I + r) % 7) / 8.0;
        sv = __fma_rn(x0, x0, sv);
      }
    }
  }
  if (w) {  // block-uniform
    const double tw = cta_tree_s(sw, red);
    const double tv = cta_tree_s(sv, red);
    if (threadIdx.x == 0) {
      part_w[blockIdx.x] = tw;
      part_v[blockIdx.x] = tv;
    }
  }
}
__global__ void k_mark_cols(int nnz, const int *J_col, int *mark) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < nnz) mark[J_col[e]] = 1;
}
// Z must be duplicate-free and contain every structurally nonzero column of J (I_c: every dof
// whose basis support touches the contact surface, reading R17); covered counts the columns of J it holds.
__global__ void k_check_Z(int nc, long n, const int *Z, const int *mark, int *pos, int *covered, int *err) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nc) return;
  const int p = Z[a];
  if (p < 0 || p >= n) { raise_err(err, DERR_ARG, a); return; }
  if (atomicCAS(&pos[p], -1, a) != -1) { raise_err(err, DERR_ARG, a); return; }
  if (mark[p]) atomicAdd(covered, 1);
}
__global__ void k_compact_Z(long n, const int *mark, const int *off, int *Z, int *pos) {
  long p = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (p < n && mark[p]) { Z[off[p]] = (int)p; pos[p] = off[p]; }
}

// ------------------------------------------------------------------ s3: A_w band and Cholesky
__global__ void k_band_start(int nc, const int *Z, const int *pos, const int *S_ptr, const int *S_col, int *bwmax) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nc) return;
  const int I = Z[a] / 3;
  int mn = a;
  for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
    for (int cc = 0; cc < 3; cc++) {
      const int b = pos[3 * S_col[k] + cc];
      if (b >= 0 && b < mn) mn = b;
    }
  atomicMax(bwmax, a - mn);
}
__global__ void k_band_fill(int nc, int bw, int W, const int *Z, const int *pos, const int *S_ptr, const int *S_col,
                            const double *S_val, double *Lrow) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nc) return;
  const int p = Z[a], I = p / 3, r = p % 3;
  for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
    for (int cc = 0; cc < 3; cc++) {
      const int b = pos[3 * S_col[k] + cc];
      if (b >= 0 && b <= a && a - b <= bw) Lrow[(long)a * W + bw - (a - b)] = S_val[(long)k * 9 + 3 * r + cc];
    }
}

// Banded Cholesky in place (C9), blocked left-looking over panels of 32 columns, one CTA.  Entry (i,l)
// receives fma(-L_ik, L_lk, .) for k ascending, exactly the contract's chain: phase A applies the terms of
// all previous panels (one independent chain per entry, all threads), phase B the terms inside the panel
// (right-looking over its 32 columns on a shared-memory copy of the panel).
constexpr int CHOL_THREADS = 1024;
constexpr int CHOL_EPT = 8;  // entries per thread in phase A: (32 + bw) * 32 <= 1024 * 8  =>  bw <= 224
constexpr int PLD = 33;      // padded row stride of the panel arrays
__global__ void __launch_bounds__(CHOL_THREADS) k_band_chol(int n_all, const int *blk_p0, const int *blk_len, int bw,
                                                             int W, double *L, int *err, int tag) {
  // one CTA per diagonal block [p0, p0+n) of the band (the whole band if blk_p0 == nullptr)
  const int p0 = blk_p0 ? blk_p0[blockIdx.x] : 0;
  const int n = blk_p0 ? blk_len[blockIdx.x] : n_all;
  L += (long)p0 * W;
  extern __shared__ double sh[];
  const int rows = 32 + bw;          // rows i = c0 + r of the panel's band
  const int ldk = rows + 1;          // k-major staging AT[kk][r], padded
  double *PA = sh;                   // [rows][PLD] panel accumulators
  double *PL = sh + rows * PLD;      // [rows][PLD] final panel values of L
  double *AT = sh + 2 * rows * PLD;  // [32][ldk]  L_{c0+r, kc+kk}, zero outside the band / k >= c0
  const int tid = threadIdx.x;
  for (int c0 = 0; c0 < n; c0 += 32) {
    // ---- phase A: acc(i,l) = a_il - sum_{k < c0} L_ik L_lk in ascending k (chunks of 32 k's staged in smem)
    double acc[CHOL_EPT];
#pragma unroll
    for (int q = 0; q < CHOL_EPT; q++) {
      const int e = tid + q * CHOL_THREADS;
      const int r = e >> 5, cc = e & 31;
      const int i = c0 + r, l = c0 + cc;
      acc[q] = (r < rows && i < n && l < n && i >= l && i - l <= bw) ? L[(long)i * W + bw - (i - l)] : 0.0;
    }
    for (int kc = max(0, c0 - bw); kc < c0; kc += 32) {
      __syncthreads();
      for (int t = tid; t < rows * 32; t += CHOL_THREADS) {
        const int r = t >> 5, kk = t & 31;
        const int i = c0 + r, k = kc + kk;
        AT[kk * ldk + r] = (i < n && k < c0 && i - k <= bw) ? L[(long)i * W + bw - (i - k)] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CHOL_EPT; q++) {
        const int e = tid + q * CHOL_THREADS;
        const int r = e >> 5, cc = e & 31;
        if (r >= rows || cc > r) continue;
        double a = acc[q];
#pragma unroll 8
        for (int kk = 0; kk < 32; kk++) a = __fma_rn(-AT[kk * ldk + r], AT[kk * ldk + cc], a);
        acc[q] = a;
      }
    }
#pragma unroll
    for (int q = 0; q < CHOL_EPT; q++) {
      const int e = tid + q * CHOL_THREADS;
      if (e < rows * 32) PA[(e >> 5) * PLD + (e & 31)] = acc[q];
    }
    __syncthreads();
    // ---- phase B: factor the panel, one thread per panel row r (right-looking over its 32 columns)
    const int cmax = min(32, n - c0);
    const int rend = min(rows, n - c0);
    for (int c = 0; c < cmax; c++) {
      const double ljj = sqrt(PA[c * PLD + c]);  // every thread: identical correctly rounded value
      if (tid == 0 && !(PA[c * PLD + c] > 0.0)) raise_err(err, DERR_NOT_SPD, tag * 1000000 + p0 + c0 + c);
      const int r = tid;
      if (r < rend && r >= c && r - c <= bw) PL[r * PLD + c] = (r == c) ? ljj : PA[r * PLD + c] / ljj;
      __syncthreads();
      if (r < rend && r > c && r - c <= bw) {
        const double lrc = PL[r * PLD + c];
        for (int cp = c + 1; cp < cmax && cp <= r; cp++)
          if (r - cp <= bw) PA[r * PLD + cp] = __fma_rn(-lrc, PL[cp * PLD + c], PA[r * PLD + cp]);
      }
      __syncthreads();
    }
    // ---- write the panel back
    for (int e = tid; e < rows * 32; e += CHOL_THREADS) {
      const int r = e >> 5, cc = e & 31;
      const int i = c0 + r, l = c0 + cc;
      if (l >= n || i >= n || i < l || i - l > bw) continue;
      L[(long)i * W + bw - (i - l)] = PL[r * PLD + cc];
    }
    __syncthreads();
  }
}
// Register-tiled form of the same factorization (same chains, bitwise equal to k_band_chol):
//   phase A  each thread owns a 4 x 4 tile of panel entries (rows r0..r0+3, columns cc0..cc0+3) and applies
//            the terms k < c0 of its 16 chains in ascending k from a k-major shared-memory chunk (two 32-byte
//            row reads + two broadcast column reads per 16 FMAs; the next chunk is loaded into registers
//            while the current one is consumed); a tile starts at its first band column c0 + r0 - bw
//   phase B1 warp 0 factors the 32 x 32 diagonal block right-looking in registers (lane = row, shuffles)
//   phase B2 every row below it applies the in-panel terms c ascending and divides by L_cc (one thread
//            per row, 32 accumulators in registers, L_cc from shared memory as broadcasts)
constexpr int CHT_THREADS = 384;
#ifdef AMGF_CHOL_TRACE  // microbenchmark builds only (tools/mb_chol.cu): per-panel phase clocks
__device__ long long *g_chol_trace;
#define CHOL_STAMP(k) \
  if (threadIdx.x == 0 && g_chol_trace) g_chol_trace[((long)blockIdx.x * 128 + c0 / 32) * 4 + (k)] = clock64();
#else
#define CHOL_STAMP(k)
#endif
__global__ void __launch_bounds__(CHT_THREADS) k_band_chol_t(int n_all, const int *blk_p0, const int *blk_len,
                                                              int bw, int W, double *L, int *err, int tag) {
  const int p0 = blk_p0 ? blk_p0[blockIdx.x] : 0;
  const int n = blk_p0 ? blk_len[blockIdx.x] : n_all;
  L += (long)p0 * W;
  extern __shared__ __align__(16) double sh[];
  const int rows = 32 + bw;
  // k-major chunk AT[kk][r]: 32-byte aligned row groups, row pitch = 4 (mod 8) doubles so that the
  // staging stores (8 consecutive k of 4 rows per warp) spread over the banks
  const int ldk = ((rows + 3) & ~3) + ((((rows + 3) & ~3) % 8 == 0) ? 4 : 0);
  const int nrt = (rows + 3) >> 2;      // row tiles
  double *AT = sh;                      // [2][32][ldk] double-buffered k-major chunks
  double *PA = sh + 64 * ldk;           // [rows][PLD] phase-A results / final panel rows
  const int tid = threadIdx.x;
  const int ntile = nrt * 8;            // tile t: row tile t % nrt, column tile t / nrt
  for (int c0 = 0; c0 < n; c0 += 32) {
    CHOL_STAMP(0);
    const int rend = min(rows, n - c0), cmax = min(32, n - c0);
    double acc[2][4][4];
    int r0v[2], cc0v[2];
    bool onv[2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int t = tid + u * CHT_THREADS;
      r0v[u] = 4 * (t % nrt);
      cc0v[u] = 4 * (t / nrt);
      onv[u] = t < ntile && r0v[u] < rows && r0v[u] + 3 >= cc0v[u] && r0v[u] - (cc0v[u] + 3) <= bw;
#pragma unroll
      for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) {
          const int i = c0 + r0v[u] + a, l = c0 + cc0v[u] + b;
          acc[u][a][b] = (onv[u] && r0v[u] + a < rend && cc0v[u] + b < cmax && i >= l && i - l <= bw)
                             ? L[(long)i * W + bw - (i - l)] : 0.0;
        }
    }
    // ---- phase A over chunks [kc, kc + 32) of k < c0, staged by cp.async (zero-filled outside the band)
    // into a double buffer; 8 consecutive k of one row per 8 threads (64-byte segments)
    const int kbeg = max(0, c0 - bw);
    const int nchunk = (c0 - kbeg + 31) / 32;
    auto issue = [&](int m) {
      const int kc = kbeg + 32 * m;
      double *dst = AT + (m & 1) * 32 * ldk;
      for (int h = 0; h < 4; h++)
        for (int e2 = tid; e2 < 8 * ldk; e2 += CHT_THREADS) {
          const int r = e2 >> 3, kk = h * 8 + (e2 & 7);
          const int i = c0 + r, k = kc + kk;
          const bool in = r < rows && i < n && k < c0 && i - k <= bw;
          const double *src = in ? L + (long)i * W + bw - (i - k) : L;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst + kk * ldk + r)), "l"(src),
                       "r"(in ? 8 : 0) : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (nchunk > 0) issue(0);
    for (int m = 0; m < nchunk; m++) {
      const int kc = kbeg + 32 * m;
      if (m + 1 < nchunk) {
        issue(m + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double *ATc = AT + (m & 1) * 32 * ldk;
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int tstart = c0 + r0v[u] - bw;  // first k with a nonzero L_{c0+r0, k}
        if (onv[u] && kc + 32 > tstart) {
          const int kk0 = max(0, tstart - kc), kn = min(32, c0 - kc);
          for (int kk = kk0; kk < kn; kk++) {
            const double2 *ar = reinterpret_cast<const double2 *>(ATc + kk * ldk + r0v[u]);
            const double2 *ac = reinterpret_cast<const double2 *>(ATc + kk * ldk + cc0v[u]);
            const double2 x0 = ar[0], x1 = ar[1], y0 = ac[0], y1 = ac[1];
            const double av[4] = {x0.x, x0.y, x1.x, x1.y}, bv[4] = {y0.x, y0.y, y1.x, y1.y};
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
              for (int b = 0; b < 4; b++) acc[u][a][b] = __fma_rn(-av[a], bv[b], acc[u][a][b]);
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 2; u++)
      if (onv[u]) {
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
          for (int b = 0; b < 4; b++)
            if (r0v[u] + a < rows) PA[(r0v[u] + a) * PLD + cc0v[u] + b] = acc[u][a][b];
      }
    __syncthreads();
    CHOL_STAMP(1);
    // ---- phase B: the in-panel terms, one thread per panel row (column-synchronous, one barrier per column):
    // step c: (i) every row r > c in the band divides, L_rc = v_r[c] / L_cc; row c+1 also applies its own
    // term k = c to its diagonal and takes the square root; (ii) every row applies the term k = c to its
    // columns cp in (c, r] (row c+1's diagonal excluded: done in (i)).  Per entry the terms stay in
    // ascending k (C9).
    {
      double *Ld = AT;             // [32] diagonal of the panel (AT is free after phase A)
      double *colL = AT + 32;      // [32][33] colL[c*33 + cp] = L_{cp, c}, cp < 32
      const int r = tid;
      const bool rin = r < rend;
      double v[32];
#pragma unroll
      for (int c = 0; c < 32; c++) v[c] = (r < rows) ? PA[r * PLD + c] : 0.0;
      if (r == 0) {
        if (!(v[0] > 0.0)) raise_err(err, DERR_NOT_SPD, tag * 1000000 + p0 + c0);
        v[0] = sqrt(v[0]);
        Ld[0] = v[0];
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 32; c++) {
        if (c < cmax) {  // block-uniform
          const bool act = rin && r > c && r - c <= bw;
          double lrc = 0.0;
          if (act) {
            lrc = v[c] / Ld[c];
            v[c] = lrc;
            if (r < 32) colL[c * 33 + r] = lrc;
            if (c < 31 && r == c + 1 && c + 1 < cmax) {
              const double dg = __fma_rn(-lrc, lrc, v[c + 1]);
              if (!(dg > 0.0)) raise_err(err, DERR_NOT_SPD, tag * 1000000 + p0 + c0 + c + 1);
              v[c + 1] = sqrt(dg);
              Ld[c + 1] = v[c + 1];
            }
          }
          __syncthreads();
          if (act && r > c + 1) {
#pragma unroll
            for (int cp = c + 1; cp < 32; cp++)
              if (cp < cmax && cp <= r && r - cp <= bw) v[cp] = __fma_rn(-lrc, colL[c * 33 + cp], v[cp]);
          }
        }
      }
      if (rin) {
        const int i = c0 + r;
#pragma unroll
        for (int c = 0; c < 32; c++)
          if (c < cmax && c <= r && r - c <= bw) L[(long)i * W + bw - (r - c)] = v[c];
      }
    }
    CHOL_STAMP(2);
    __syncthreads();
    CHOL_STAMP(3);
  }
}

// Fallback for wide bands (e.g. Z = NULL ordering): right-looking on global memory, one CTA (same chains).
__global__ void __launch_bounds__(1024) k_band_chol_wide(int n_all, const int *blk_p0, const int *blk_len, int bw,
                                                         int W, double *L, int *err, int tag) {
  const int p0 = blk_p0 ? blk_p0[blockIdx.x] : 0;
  const int n = blk_p0 ? blk_len[blockIdx.x] : n_all;
  L += (long)p0 * W;
  __shared__ double piv;
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; j++) {
    if (tid == 0) {
      double d = L[(long)j * W + bw];
      if (!(d > 0.0)) { raise_err(err, DERR_NOT_SPD, tag * 1000000 + p0 + j); bad = 1; }
      double s = sqrt(d);
      L[(long)j * W + bw] = s;
      piv = s;
    }
    __syncthreads();
    if (bad) return;
    const double ljj = piv;
    const int rmax = min(bw, n - 1 - j);
    for (int t = 1 + tid; t <= rmax; t += blockDim.x) {
      const long ix = (long)(j + t) * W + bw - t;
      L[ix] = L[ix] / ljj;
    }
    __syncthreads();
    const long pairs = (long)rmax * rmax;
    for (long q = tid; q < pairs; q += blockDim.x) {
      const int u = (int)(q / rmax) + 1, v = (int)(q % rmax) + 1;
      if (v > u) continue;
      const double lij = L[(long)(j + u) * W + bw - u];
      const double llj = L[(long)(j + v) * W + bw - v];
      const long ix = (long)(j + u) * W + bw - (u - v);
      L[ix] = __fma_rn(-lij, llj, L[ix]);
    }
    __syncthreads();
  }
}

// dinv = 1/L_ii, the column-major copy and the reversed-row copy of the band
__global__ void k_band_finish(int n, int bw, int W, const double *Lrow, double *Lcol, double *Lrev, double *dinv) {
  long q = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (q >= (long)n * (bw + 1)) return;
  const int i = (int)(q / (bw + 1)), t = (int)(q % (bw + 1));  // L_{i, i-t}
  const int k = i - t;
  if (k < 0) return;
  const double v = Lrow[(long)i * W + bw - t];
  Lcol[(long)k * W + t] = v;
  Lrev[(long)i * W + t] = v;
  if (t == 0) dinv[i] = 1.0 / v;
}

// thin residual structure: per scalar row p, entries of S with column in Z, ascending column
__global__ void k_thin_count(long n, const int *S_ptr, const int *S_col, const int *pos, int *cnt) {
  long p = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int I = (int)(p / 3);
  int c0 = 0;
  for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
    for (int cc = 0; cc < 3; cc++) c0 += pos[3 * S_col[k] + cc] >= 0;
  cnt[p] = c0;
}
__global__ void k_thin_fill(long n, const int *S_ptr, const int *S_col, const int *pos, const int *off,
                            const int *rowflag_off, int *thin_row, int *thin_ptr, int *thin_pos, int *thin_src) {
  long p = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int I = (int)(p / 3), r = (int)(p % 3);
  int w = off[p];
  if (off[p + 1] == w) return;
  const int t = rowflag_off[p];
  thin_row[t] = (int)p;
  thin_ptr[t] = w;
  for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
    for (int cc = 0; cc < 3; cc++) {
      const int b = pos[3 * S_col[k] + cc];
      if (b >= 0) { thin_pos[w] = b; thin_src[w] = k * 9 + 3 * r + cc; w++; }
    }
}
__global__ void k_flag_nonzero(long n, const int *cnt, int *flag) {
  long p = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (p < n) flag[p] = cnt[p] > 0;
}
// Ctx::zr_* (compact fine rows of the filter dofs, k_resid_dofs): counts, structure, values.
__global__ void k_zr_count(int nc, const int *dof, const int *ptr, int *cnt) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < nc) cnt[p] = ptr[dof[p] / 3 + 1] - ptr[dof[p] / 3];
}
__global__ void k_zr_fill(int nc, const int *dof, const int *ptr, const int *col, const int *zr_ptr, int *zr_col,
                          int *zr_src) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  const int i = dof[p] / 3, r = dof[p] % 3, o = zr_ptr[p];
  for (int k = ptr[i]; k < ptr[i + 1]; k++) {
    zr_col[o + k - ptr[i]] = col[k];
    zr_src[o + k - ptr[i]] = k * 9 + r * 3;  // block k, row r of the 3 x 3 block
  }
}
__global__ void k_zr_vals(long nnz, const int *zr_src, const double *val, double *zr_val) {
  const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
#pragma unroll
  for (int e = 0; e < 3; e++) zr_val[k * 3 + e] = val[(long)zr_src[k] + e];
}

__global__ void k_gather_vals(long n, const int *src, const double *from, double *to) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e < n) to[e] = src[e] >= 0 ? from[src[e]] : 0.0;
}

// ------------------------------------------------------------------ s8: diagonals (C3)
// Nodal-block l1 smoother data (smoother 2, contract C24 / reading R22), one thread per node: d_r = off-block l1
// row sums (chain d = d + |a| over the row's other blocks, ascending), B = A_ii + diag(d), its Cholesky by the
// chains of C9, stored as the lower factor (b(b+1)/2, row-major) then the reciprocals 1/L_rr.
template <int B>
__global__ void k_block_l1(int nodes, const int *ptr, const int *col, const double *val, double *bfac, int *err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  double M[B * B], Lf[B * B];
  const double *Aii = nullptr;
  for (int r = 0; r < B; r++) {
    double d = 0.0;
    for (int k = ptr[i]; k < ptr[i + 1]; k++) {
      if (col[k] == i) { Aii = val + (long)k * B * B; continue; }
      for (int c = 0; c < B; c++) d = d + fabs(val[(long)k * B * B + r * B + c]);
    }
    M[r * B + r] = d;
  }
  if (!Aii) { raise_err(err, DERR_NOT_SPD, i); return; }
  for (int r = 0; r < B; r++)
    for (int c = 0; c < B; c++) M[r * B + c] = (r == c) ? Aii[r * B + r] + M[r * B + r] : Aii[r * B + c];
  for (int c = 0; c < B; c++) {
    double acc = M[c * B + c];
    for (int k = 0; k < c; k++) acc = __fma_rn(-Lf[c * B + k], Lf[c * B + k], acc);
    if (!(acc > 0.0)) { raise_err(err, DERR_NOT_SPD, i); return; }
    const double lcc = sqrt(acc);
    Lf[c * B + c] = lcc;
    for (int r = c + 1; r < B; r++) {
      double a = M[r * B + c];
      for (int k = 0; k < c; k++) a = __fma_rn(-Lf[r * B + k], Lf[c * B + k], a);
      Lf[r * B + c] = a / lcc;
    }
  }
  constexpr int NB = B * (B + 1) / 2 + B;
  double *o = bfac + (long)i * NB;
  int w = 0;
  for (int r = 0; r < B; r++)
    for (int c = 0; c <= r; c++) o[w++] = Lf[r * B + c];
  for (int r = 0; r < B; r++) o[w++] = 1.0 / Lf[r * B + r];
}

__global__ void k_diag(int nodes, int b, const int *ptr, const int *col, const double *val, double *dl1, double *dpt) {
  long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)nodes * b) return;
  const int i = (int)(t / b), r = (int)(t % b);
  double d = 0.0, dp = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; k++)
    for (int cc = 0; cc < b; cc++) {
      const double a = val[(long)k * b * b + r * b + cc];
      d = d + fabs(a);
      if (col[k] == i && cc == r) dp = a;
    }
  dl1[t] = d;
  dpt[t] = dp;
}

// ------------------------------------------------------------------ s4: components and aggregation
__global__ void k_cc_step(int nodes, const int *ptr, const int *col, int *lab, int *changed) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  int m = lab[v];
  for (int k = ptr[v]; k < ptr[v + 1]; k++) m = min(m, lab[col[k]]);
  int l2 = lab[m];
  m = min(m, l2);
  if (m < lab[v]) { atomicMin(&lab[v], m); *changed = 1; }
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ bool better(int u, int v, uint64_t seed) {  // u beats v (v may be -1)
  if (u < 0) return false;
  if (v < 0) return true;
  uint64_t pu = mix64((uint64_t)(uint32_t)u ^ seed), pv = mix64((uint64_t)(uint32_t)v ^ seed);
  return pu > pv || (pu == pv && u < v);
}

enum { ST_UND = 0, ST_ROOT = 1, ST_OUT = 2, ST_ISO = 3 };

__global__ void k_mis_init(int nodes, const int *ptr, const int *col, const int *comp, int *state) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  int iso = 1;
  for (int k = ptr[v]; k < ptr[v + 1]; k++) {
    const int u = col[k];
    if (u != v && comp[u] == comp[v]) { iso = 0; break; }
  }
  state[v] = iso ? ST_ISO : ST_UND;
}
// m_out[v] = best over N[v] of (m_in[u]) ; with m_in = nullptr, candidates are undecided nodes themselves
__global__ void k_mis_max(int nodes, const int *ptr, const int *col, const int *comp, const int *state,
                          const int *m_in, int *m_out, uint64_t seed) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  if (state[v] == ST_ISO) { m_out[v] = -1; return; }
  int best = m_in ? m_in[v] : (state[v] == ST_UND ? v : -1);
  for (int k = ptr[v]; k < ptr[v + 1]; k++) {
    const int u = col[k];
    if (u == v || comp[u] != comp[v]) continue;
    const int cand = m_in ? m_in[u] : (state[u] == ST_UND ? u : -1);
    if (better(cand, best, seed)) best = cand;
  }
  m_out[v] = best;
}
__global__ void k_mis_roots(int nodes, const int *m2, int *state) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes && state[v] == ST_UND && m2[v] == v) state[v] = ST_ROOT;
}
// flag[v] = 1 if a root (or, with f_in, a flagged node) lies in N[v]
__global__ void k_mis_near(int nodes, const int *ptr, const int *col, const int *comp, const int *state,
                           const int *f_in, int *f_out) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  int f = f_in ? f_in[v] : (state[v] == ST_ROOT);
  for (int k = ptr[v]; k < ptr[v + 1] && !f; k++) {
    const int u = col[k];
    if (u == v || comp[u] != comp[v]) continue;
    f = f_in ? f_in[u] : (state[u] == ST_ROOT);
  }
  f_out[v] = f;
}
__global__ void k_mis_block(int nodes, const int *b2, int *state, int *undecided) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  if (state[v] == ST_UND) {
    if (b2[v]) state[v] = ST_OUT;
    else atomicAdd(undecided, 1);
  }
}
__global__ void k_root_flag(int nodes, const int *state, int *flag) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes) flag[v] = state[v] == ST_ROOT;
}
__global__ void k_agg_phase3(int nodes, const int *ptr, const int *col, const int *comp, const int *state,
                             const int *rank, int *agg3) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  int a = -1;
  if (state[v] == ST_ROOT) a = rank[v];
  else if (state[v] != ST_ISO)
    for (int k = ptr[v]; k < ptr[v + 1]; k++) {
      const int u = col[k];
      if (u != v && comp[u] == comp[v] && state[u] == ST_ROOT) { a = rank[u]; break; }
    }
  agg3[v] = a;
}
__global__ void k_agg_leftover(int nodes, const int *ptr, const int *col, const int *comp, const int *state,
                               const int *agg3, int *agg, int *err) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nodes) return;
  if (state[v] == ST_ISO || agg3[v] >= 0) { agg[v] = agg3[v]; return; }
  int best = -1, bestc = 0;
  for (int k = ptr[v]; k < ptr[v + 1]; k++) {
    const int u = col[k];
    if (u == v || comp[u] != comp[v]) continue;
    const int a = agg3[u];
    if (a < 0) continue;
    int cnum = 0;
    for (int k2 = ptr[v]; k2 < ptr[v + 1]; k2++) {
      const int w2 = col[k2];
      if (w2 != v && comp[w2] == comp[v] && agg3[w2] == a) cnum++;
    }
    if (cnum > bestc || (cnum == bestc && a < best)) { bestc = cnum; best = a; }
  }
  if (best < 0) raise_err(err, DERR_ARG, v);
  agg[v] = best;
}
__global__ void k_agg_key(int nodes, const int *agg, int *key) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes) key[v] = agg[v] >= 0 ? agg[v] : 0x7fffffff;
}
__global__ void k_coarse_comp(int nodes, const int *state, const int *rank, const int *comp, int *comp_c) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes && state[v] == ST_ROOT) comp_c[rank[v]] = comp[v];
}
__global__ void k_is_agg(int nodes, const int *agg, int *flag) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes) flag[v] = agg[v] >= 0;
}
__global__ void k_Pt_cols(int nodes, const int *agg, const int *Pt_ptr, int *Pt_col) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < nodes && agg[v] >= 0) Pt_col[Pt_ptr[v]] = agg[v];
}

// ------------------------------------------------------------------ s5: tentative prolongator (C17)
__global__ void k_qr(int na, int b, const int *agg_ptr, const int *agg_nodes, const int *Pt_ptr, const double *Bnn,
                     double *Ptv, double *Bc, int *err) {
  int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= na) return;
  const int m0 = agg_ptr[a], m1 = agg_ptr[a + 1];
  auto Q = [&](int t, int r, int j) -> double & {
    return Ptv[((long)Pt_ptr[agg_nodes[t]] * b + r) * 6 + j];
  };
  for (int t = m0; t < m1; t++)
    for (int r = 0; r < b; r++)
      for (int j = 0; j < 6; j++) Q(t, r, j) = Bnn[((long)agg_nodes[t] * b + r) * 6 + j];
  double Rm[36];
  for (int q = 0; q < 36; q++) Rm[q] = 0.0;
  for (int j = 0; j < 6; j++) {
    for (int i = 0; i < j; i++) {
      double rij = 0.0;
      for (int t = m0; t < m1; t++)
        for (int r = 0; r < b; r++) rij = __fma_rn(Q(t, r, i), Q(t, r, j), rij);
      Rm[i * 6 + j] = rij;
      for (int t = m0; t < m1; t++)
        for (int r = 0; r < b; r++) Q(t, r, j) = __fma_rn(-rij, Q(t, r, i), Q(t, r, j));
    }
    double ss = 0.0;
    for (int t = m0; t < m1; t++)
      for (int r = 0; r < b; r++) ss = __fma_rn(Q(t, r, j), Q(t, r, j), ss);
    const double rjj = sqrt(ss);
    if (!(rjj > 0.0) || (j > 0 && !(rjj > 1e-10 * Rm[0]))) { raise_err(err, DERR_RANK, a); return; }
    Rm[j * 6 + j] = rjj;
    for (int t = m0; t < m1; t++)
      for (int r = 0; r < b; r++) Q(t, r, j) = Q(t, r, j) / rjj;
  }
  for (int q = 0; q < 36; q++) Bc[(long)a * 36 + q] = Rm[q];
}

// ------------------------------------------------------------------ s6: power iteration, smoothed P
__global__ void k_pow_init(long n, double *v) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = 1.0 + (double)(i % 7) / 8.0;
}
__global__ void k_div(long n, double *w, const double *d) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) w[i] = w[i] / d[i];
}
__global__ void k_scale_div(long n, const double *w, double s, double *v) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i < n) v[i] = w[i] / s;
}
// power step on the device (C18): pw[0] = w.w, pw[1] = v.v (k_pow_fin); ||w|| = sqrt(pw[0]),
// lambda = ||w|| / sqrt(pw[1]) into pw[2]; v = w / ||w|| -- the host's formulas, no host round trip
__global__ void k_pow_scale(long n, const double *w, double *pw, double *v) {
  const double nw = sqrt(pw[0]);
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i == 0) {
    const double lam = nw / sqrt(pw[1]);
    pw[2] = lam;
    pw[3] = 4.0 / (3.0 * lam);  // R6: the prolongator damping omega (the host formula, in fp64)
  }
  if (i < n) v[i] = w[i] / nw;
}

constexpr int PCAP = 128;
__global__ void k_P_count(int nodes, const int *ptr, const int *col, const int *agg, int *cnt, int *err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  int list[PCAP];
  int nl = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; k++) {
    const int a = agg[col[k]];
    if (a >= 0 && !insert_unique(list, nl, PCAP, a)) { raise_err(err, DERR_LIMIT, i); break; }
  }
  cnt[i] = nl;
}
__global__ void k_P_fill(int nodes, const int *ptr, const int *col, const int *agg, const int *P_ptr, int *P_col) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nodes) return;
  int list[PCAP];
  int nl = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; k++) {
    const int a = agg[col[k]];
    if (a >= 0) insert_unique(list, nl, PCAP, a);
  }
  for (int q = 0; q < nl; q++) P_col[P_ptr[i] + q] = list[q];
}
// P_ia = Pt_ia - (omega * T_ia) / dpt, T = A Pt (C19, C20); one thread per P block, the b x 6 entries
// accumulate in registers over one pass of A's row (per entry: j ascending, then cc ascending)
template <int B>
__global__ void k_P_values(long nnzb, const int *P_rowof, const int *P_col, const int *A_ptr, const int *A_col,
                           const double *A_val, const int *agg, const int *Pt_ptr, const double *Ptv,
                           const double *dpt, const double *omega_p, double *Pv, const int *Rinv, double *Rv) {
  const double omega = *omega_p;  // 4 / (3 lambda) of this level, formed on the device (k_pow_scale)
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzb) return;
  const int i = P_rowof[e], a = P_col[e];
  double acc[B * 6];
#pragma unroll
  for (int q = 0; q < B * 6; q++) acc[q] = 0.0;
  for (int k = A_ptr[i]; k < A_ptr[i + 1]; k++) {
    const int j = A_col[k];
    if (agg[j] != a) continue;
    const double *Av = A_val + (long)k * B * B;
    const double *Qj = Ptv + (long)Pt_ptr[j] * B * 6;
#pragma unroll
    for (int r = 0; r < B; r++)
#pragma unroll
      for (int s = 0; s < 6; s++)
#pragma unroll
        for (int cc = 0; cc < B; cc++) acc[r * 6 + s] = __fma_rn(Av[r * B + cc], Qj[cc * 6 + s], acc[r * 6 + s]);
  }
  const bool own = agg[i] == a;
#pragma unroll
  for (int r = 0; r < B; r++)
#pragma unroll
    for (int s = 0; s < 6; s++) {
      double t = omega * acc[r * 6 + s];
      t = t / dpt[(long)i * B + r];
      const double pt = own ? Ptv[((long)Pt_ptr[i] * B + r) * 6 + s] : 0.0;
      Pv[(e * B + r) * 6 + s] = pt - t;
      if (Rinv) Rv[((long)Rinv[e] * 6 + s) * B + r] = pt - t;  // R = P^T: its block Rinv[e], transposed
    }
}
// The same P values (C19/C20) over precomputed block-product pairs (symbolic, once): thread per P block runs
// exactly its (A block, Pt block) products in ascending A position -- the walk above tests every block of A's
// row (26 at the fine level) for its ~6 products.  Writes P and R = P^T.
template <int B, int H>  // H threads per P block, B / H rows each (the 6 x 6 levels: 2 x 18 accumulators)
__global__ void __launch_bounds__(CTA) k_P_pairs(long nnzb, const int *__restrict__ P_rowof,
                                                 const int *__restrict__ P_col, const int *__restrict__ pptr,
                                                 const int *__restrict__ pa, const int *__restrict__ pb,
                                                 const double *__restrict__ A_val, const int *__restrict__ agg,
                                                 const int *__restrict__ Pt_ptr, const double *__restrict__ Ptv,
                                                 const double *__restrict__ dpt, const double *__restrict__ omega_p,
                                                 double *__restrict__ Pv, const int *__restrict__ Rinv,
                                                 double *__restrict__ Rv) {
  constexpr int RB = B / H;  // rows of this thread
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long e = t / H;
  const int r0 = (int)(t - e * H) * RB;
  if (e >= nnzb) return;
  const double omega = *omega_p;
  double acc[RB * 6];
#pragma unroll
  for (int q = 0; q < RB * 6; q++) acc[q] = 0.0;
  const int q1 = pptr[e + 1];
  for (int q = pptr[e]; q < q1; q++) {
    const double *Av = A_val + (long)pa[q] * B * B + r0 * B;
    const double2 *Qv = reinterpret_cast<const double2 *>(Ptv + (long)pb[q] * B * 6);
    double a[RB * B], qj[B * 6];
#pragma unroll
    for (int u = 0; u < RB * B; u++) a[u] = __ldg(Av + u);
#pragma unroll
    for (int u = 0; u < B * 3; u++) {
      const double2 v = __ldg(Qv + u);
      qj[2 * u] = v.x;
      qj[2 * u + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int s = 0; s < 6; s++)
#pragma unroll
        for (int cc = 0; cc < B; cc++) acc[r * 6 + s] = __fma_rn(a[r * B + cc], qj[cc * 6 + s], acc[r * 6 + s]);
  }
  const int i = P_rowof[e], a = P_col[e];
  const bool own = agg[i] == a;
#pragma unroll
  for (int rr = 0; rr < RB; rr++)
#pragma unroll
    for (int s = 0; s < 6; s++) {
      const int r = r0 + rr;
      double tt = omega * acc[rr * 6 + s];
      tt = tt / dpt[(long)i * B + r];
      const double pt = own ? Ptv[((long)Pt_ptr[i] * B + r) * 6 + s] : 0.0;
      Pv[(e * B + r) * 6 + s] = pt - tt;
      Rv[((long)Rinv[e] * 6 + s) * B + r] = pt - tt;
    }
}
__global__ void k_inv_perm(long n, const int *perm, int *inv) {
  long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t < n) inv[perm[t]] = (int)t;
}

// ------------------------------------------------------------------ s7: transpose, SpGEMMs, symmetrisation
// Bsr::ival from val: one warp per block row, lane l of step t moves block gb + l (gb = beg + 32 t); writes
// coalesced per component (140 us at cfg 3; coalescing the reads instead was 3x slower).
__global__ void k_interleave_rows(int nbr, const int *__restrict__ ptr, int bs, const double *__restrict__ val,
                                  double *__restrict__ ival) {
  const int w = (blockIdx.x * CTA + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nbr) return;
  const int beg = ptr[w], end = ptr[w + 1];
  for (int gb = beg; gb < end; gb += 32) {
    const int gs = min(32, end - gb);
    if (lane < gs)
      for (int q = 0; q < bs; q++) ival[(long)gb * bs + (long)q * gs + lane] = val[(long)(gb + lane) * bs + q];
  }
}


constexpr int GCAP = 512;
// symbolic C = A*B: row i's pattern = union of B rows over A's columns
__global__ void k_spgemm_count(int nrows, const int *A_ptr, const int *A_col, const int *B_ptr, const int *B_col,
                               int *cnt, int *err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int list[GCAP];
  int nl = 0;
  for (int k = A_ptr[i]; k < A_ptr[i + 1]; k++) {
    const int j = A_col[k];
    for (int k2 = B_ptr[j]; k2 < B_ptr[j + 1]; k2++)
      if (!insert_unique(list, nl, GCAP, B_col[k2])) { raise_err(err, DERR_LIMIT, i); cnt[i] = nl; return; }
  }
  cnt[i] = nl;
}
__global__ void k_spgemm_fill(int nrows, const int *A_ptr, const int *A_col, const int *B_ptr, const int *B_col,
                              const int *C_ptr, int *C_col) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  int list[GCAP];
  int nl = 0;
  for (int k = A_ptr[i]; k < A_ptr[i + 1]; k++) {
    const int j = A_col[k];
    for (int k2 = B_ptr[j]; k2 < B_ptr[j + 1]; k2++) insert_unique(list, nl, GCAP, B_col[k2]);
  }
  for (int q = 0; q < nl; q++) C_col[C_ptr[i] + q] = list[q];
}
// numeric C = A*B (C20): for each output block C_ib the block products A_ij B_jb over A's row i in
// ascending j, each entry accumulated over j ascending, then t ascending (the inner block index).
// Block-product lists (symbolic, once): count, then fill the (A index, B index) pairs of each output block
// C_ib in ascending order of A's column j, found by binary search in B's row j.
__global__ void k_spgemm_pairs(long nnzc, const int *C_rowof, const int *C_col, const int *A_ptr, const int *A_col,
                               const int *B_ptr, const int *B_col, const int *pptr, int *cnt, int *pa, int *pb) {
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzc) return;
  const int i = C_rowof[e], bcol = C_col[e];
  int q = pptr ? pptr[e] : 0, m = 0;
  for (int k = A_ptr[i]; k < A_ptr[i + 1]; k++) {
    const int k2 = bsearch_int(B_col, B_ptr[A_col[k]], B_ptr[A_col[k] + 1], bcol);
    if (k2 < 0) continue;
    if (pptr) { pa[q] = k; pb[q] = k2; q++; }
    m++;
  }
  if (!pptr) cnt[e] = m;
}
// numeric C = A*B over the precomputed pairs, one thread per output block (entries in registers)
template <int BR, int IN, int BC>
__global__ void k_spgemm_vals_pairs(long nnzc, const int *pptr, const int *pa, const int *pb, const double *A_val,
                                    const double *B_val, double *C_val) {
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzc) return;
  double acc[BR * BC];
#pragma unroll
  for (int q = 0; q < BR * BC; q++) acc[q] = 0.0;
  for (int q = pptr[e]; q < pptr[e + 1]; q++) {
    const double *Av = A_val + (long)pa[q] * BR * IN;
    const double *Bv = B_val + (long)pb[q] * IN * BC;
    double a[BR * IN], bb[IN * BC];
#pragma unroll
    for (int u = 0; u < BR * IN; u++) a[u] = __ldg(Av + u);
#pragma unroll
    for (int u = 0; u < IN * BC; u++) bb[u] = __ldg(Bv + u);
#pragma unroll
    for (int r = 0; r < BR; r++)
#pragma unroll
      for (int s = 0; s < BC; s++)
#pragma unroll
        for (int t = 0; t < IN; t++) acc[r * BC + s] = __fma_rn(a[r * IN + t], bb[t * BC + s], acc[r * BC + s]);
  }
#pragma unroll
  for (int q = 0; q < BR * BC; q++) C_val[e * BR * BC + q] = acc[q];
}

// Same products, two threads per 6 x 6 output block (rows 0-2 / 3-5, 18 accumulators each): per block pair
// a thread loads its three contiguous A rows (144 bytes) and the whole B block (288 bytes, shared with its
// partner), 108 FMAs per 54 loads (the warp form above: 6 FMAs per 12 loads).  Per entry the order is C20's.
__global__ void __launch_bounds__(CTA) k_spgemm_vals_half6(long nnzc, const int *__restrict__ pptr,
                                                           const int *__restrict__ pa, const int *__restrict__ pb,
                                                           const double *__restrict__ A_val,
                                                           const double *__restrict__ B_val,
                                                           double *__restrict__ C_val) {
  const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long e = t >> 1;
  const int h = (int)(t & 1);
  if (e >= nnzc) return;
  double acc[18];
#pragma unroll
  for (int u = 0; u < 18; u++) acc[u] = 0.0;
  const int q1 = pptr[e + 1];
  for (int q = pptr[e]; q < q1; q++) {
    const double2 *Av = reinterpret_cast<const double2 *>(A_val + (long)pa[q] * 36 + 18 * h);
    const double2 *Bv = reinterpret_cast<const double2 *>(B_val + (long)pb[q] * 36);
    double a[18], bb[36];
#pragma unroll
    for (int u = 0; u < 9; u++) {
      const double2 v = __ldg(Av + u);
      a[2 * u] = v.x;
      a[2 * u + 1] = v.y;
    }
#pragma unroll
    for (int u = 0; u < 18; u++) {
      const double2 v = __ldg(Bv + u);
      bb[2 * u] = v.x;
      bb[2 * u + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
      for (int s2 = 0; s2 < 6; s2++)
#pragma unroll
        for (int k = 0; k < 6; k++) acc[r * 6 + s2] = __fma_rn(a[r * 6 + k], bb[k * 6 + s2], acc[r * 6 + s2]);
  }
  double2 *Cv = reinterpret_cast<double2 *>(C_val + e * 36 + 18 * h);
#pragma unroll
  for (int u = 0; u < 9; u++) Cv[u] = make_double2(acc[2 * u], acc[2 * u + 1]);
}

// Same products, one warp per output block: lane e owns entries e, e+32, .. of the BR x BC block, so the
// loads of each (A, B) block pair are a few contiguous lines shared by the warp (the thread-per-block form
// above issues one cache line per thread per element).  Per entry the FMA order is unchanged (C20).
template <int BR, int IN, int BC>
__global__ void k_spgemm_vals_warp(long nnzc, const int *pptr, const int *pa, const int *pb, const double *A_val,
                                   const double *B_val, double *C_val) {
  constexpr int NE = BR * BC, E = (NE + 31) / 32;
  const long e = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (e >= nnzc) return;
  double acc[E];
  int rr[E], ss[E];
#pragma unroll
  for (int u = 0; u < E; u++) {
    const int en = min(lane + 32 * u, NE - 1);
    rr[u] = en / BC;
    ss[u] = en % BC;
    acc[u] = 0.0;
  }
  // pairs in batches of PF: all index and operand loads of a batch are issued before its FMAs (the long
  // R*AP lists are latency chains otherwise)
  constexpr int PF = (E * IN > 6) ? 2 : 4;
  const int q1 = pptr[e + 1];
  for (int q0 = pptr[e]; q0 < q1; q0 += PF) {
    double a[PF][E][IN], bb[PF][E][IN];
#pragma unroll
    for (int f = 0; f < PF; f++) {
      const int q = min(q0 + f, q1 - 1);
      const double *Av = A_val + (long)pa[q] * BR * IN;
      const double *Bv = B_val + (long)pb[q] * IN * BC;
#pragma unroll
      for (int u = 0; u < E; u++)
#pragma unroll
        for (int t = 0; t < IN; t++) { a[f][u][t] = __ldg(Av + rr[u] * IN + t); bb[f][u][t] = __ldg(Bv + t * BC + ss[u]); }
    }
#pragma unroll
    for (int f = 0; f < PF; f++)
      if (q0 + f < q1) {
#pragma unroll
        for (int u = 0; u < E; u++)
#pragma unroll
          for (int t = 0; t < IN; t++) acc[u] = __fma_rn(a[f][u][t], bb[f][u][t], acc[u]);
      }
  }
#pragma unroll
  for (int u = 0; u < E; u++)
    if (lane + 32 * u < NE) C_val[e * NE + lane + 32 * u] = acc[u];
}

// Dense-over-row form of the same products (C20): the thread of output block C_ib walks ALL of A's row i
// (t ascending) and multiplies where B's row k = A_col[t] holds column b; off[t * nnzc + e] is that block's
// offset within B's row k (-1 if absent; symbolic, built once).  The threads of one output row walk the same
// k sequence, so A_ik is a warp broadcast and the B blocks they read lie in one contiguous B row -- the pair
// lists above gather one A and one B block per thread per step from unrelated rows.  Same FMAs, same order.
__global__ void k_spgemm_off(long nnzc, const int *C_rowof, const int *C_col, const int *A_ptr, const int *A_col,
                             const int *B_ptr, const int *B_col, int maxa, signed char *off) {
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzc) return;
  const int i = C_rowof[e], bcol = C_col[e];
  const int a0 = A_ptr[i], la = A_ptr[i + 1] - a0;
  for (int t = 0; t < maxa; t++) {
    int o = -1;
    if (t < la) {
      const int k = A_col[a0 + t];
      const int q = bsearch_int(B_col, B_ptr[k], B_ptr[k + 1], bcol);
      if (q >= 0) o = q - B_ptr[k];
    }
    off[(long)t * nnzc + e] = (signed char)o;
  }
}
template <int BR, int IN, int BC>
__global__ void __launch_bounds__(CTA) k_spgemm_dense(long nnzc, const int *__restrict__ C_rowof,
                                                      const int *__restrict__ A_ptr, const int *__restrict__ A_col,
                                                      const double *__restrict__ A_val, const int *__restrict__ B_ptr,
                                                      const double *__restrict__ B_val,
                                                      const signed char *__restrict__ off, double *__restrict__ C_val) {
  const long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzc) return;
  const int i = C_rowof[e];
  const int a0 = A_ptr[i], la = A_ptr[i + 1] - a0;
  double acc[BR * BC];
#pragma unroll
  for (int q = 0; q < BR * BC; q++) acc[q] = 0.0;
  for (int t = 0; t < la; t++) {
    const int o = off[(long)t * nnzc + e];
    if (o < 0) continue;
    const int k = A_col[a0 + t];
    const double *Av = A_val + (long)(a0 + t) * BR * IN;
    const double *Bv = B_val + (long)(B_ptr[k] + o) * IN * BC;
    double a[BR * IN], bb[IN * BC];
#pragma unroll
    for (int u = 0; u < BR * IN; u++) a[u] = __ldg(Av + u);
#pragma unroll
    for (int u = 0; u < IN * BC; u++) bb[u] = __ldg(Bv + u);
#pragma unroll
    for (int r = 0; r < BR; r++)
#pragma unroll
      for (int c = 0; c < BC; c++)
#pragma unroll
        for (int t2 = 0; t2 < IN; t2++) acc[r * BC + c] = __fma_rn(a[r * IN + t2], bb[t2 * BC + c], acc[r * BC + c]);
  }
#pragma unroll
  for (int q = 0; q < BR * BC; q++) C_val[e * BR * BC + q] = acc[q];
}

// Row-group form of the fine-level A*P (same products, same chains as k_spgemm_dense; C20).  A group is a run
// of consecutive output rows (symbolic, built once on the host: at most GAL_NT output blocks, GAL_ACAP blocks
// of A, GHL_PCAP blocks of the union of the P rows those A rows reference, GHL_HCAP block products).  The
// group's A values (one contiguous segment) and the union of its P rows (runs of consecutive rows: contiguous
// segments) are TMA bulk-copied into shared memory once; neighbouring lattice rows share most of their P
// rows, so a P row is read from L2 about 2.5x less often than once per A block.  Groups whose rows exceed
// the capacities (none at cfg 0-4) read the operands from global memory instead.
struct GalGrp {
  int e0, e1;      // output blocks [e0, e1)
  int a0;          // first A block of the group
  int c0, c1;      // copy descriptors [c0, c1) (c1 == c0: operands from global memory)
  unsigned tx;     // bytes of all copies (mbarrier transaction count)
  int q0, pad;     // first block-product word of the group
};
struct GalRun {
  int j0, j1;  // P rows [j0, j1)
  int base;    // first shared-memory block of the run
  int pad;
};
struct GalCopy {  // one TMA bulk copy of a group: source byte offset in array `id`, destination in the buffer
  long long src;
  int dst;
  unsigned bytes_id;  // bytes | id << 28 (0: A values, 1: hit words, 2: word offsets, 3: B values)
};
constexpr int GAL_NT = 64, GAL_ACAP = 176, GAL_RCAP = 28;
// Hit lists: the symbolic phase turns each output block's block-product pairs (A block, B block; ascending A
// position) into 32-bit words (A block within the group's staged A segment | B block within the staged P-row
// union << 8); the group's words and per-output word offsets are bulk-copied with the operands, and thread
// e = output block C_ib runs exactly its products, operands and indices from shared memory.
constexpr int GHL_PCAP = 256, GHL_HCAP = 1024;
__host__ __device__ constexpr size_t ghl_buf_bytes(int AB, int BB) {  // one group buffer: B union, A segment, hit words, word offsets
  return (((size_t)GHL_PCAP * BB + (size_t)GAL_ACAP * AB + 2) * 8 + (GHL_HCAP + 8) * 4 + (GAL_NT + 1 + 8) * 4 + 127) &
         ~(size_t)127;  // 128-byte aligned buffers (TMA destinations, 16-byte vector loads)
}
// One CTA per group (4 CTAs per SM): warp 1 issues the group's TMA copies (precomputed descriptors, one per
// lane), then every thread runs its output block's products from shared memory.
template <int BR, int IN, int BC>
__global__ void __launch_bounds__(GAL_NT) k_gal_hl(const GalGrp *__restrict__ grp, const GalCopy *__restrict__ cps,
                                                  const int *__restrict__ pptr, const unsigned *__restrict__ hitw,
                                                  const int *__restrict__ pa, const int *__restrict__ pb,
                                                  const double *__restrict__ A_val, const double *__restrict__ B_val,
                                                  double *__restrict__ C_val) {
  constexpr int AB = BR * IN, BB = IN * BC;
  extern __shared__ __align__(128) unsigned char hsm[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31;
  double *Bs = reinterpret_cast<double *>(hsm);
  double *As = Bs + GHL_PCAP * BB;
  unsigned *Hs = reinterpret_cast<unsigned *>(As + GAL_ACAP * AB + 2);
  int *Ps = reinterpret_cast<int *>(Hs + GHL_HCAP + 8);
  const GalGrp g = grp[blockIdx.x];
  const bool staged = g.c1 > g.c0;
  if (staged) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid >= 32) {
      if (lane == 0) mbar_arrive_expect(&bar, g.tx);
      __syncwarp();
      for (int k = g.c0 + lane; k < g.c1; k += 32) {
        const GalCopy cp = cps[k];
        const unsigned id = cp.bytes_id >> 28, bytes = cp.bytes_id & 0x0fffffffu;
        const char *base = id == 0 ? (const char *)A_val : id == 1 ? (const char *)hitw : id == 2 ? (const char *)pptr
                                                                                                : (const char *)B_val;
        bulk_g2s(hsm + cp.dst, base + cp.src, bytes, &bar);
      }
    }
    mbar_wait(&bar, 0);
  }
  const long e = (long)g.e0 + tid;
  if (e >= g.e1) return;
  double acc[BR * BC];
#pragma unroll
  for (int q = 0; q < BR * BC; q++) acc[q] = 0.0;
  auto hit = [&](const double *Av, const double *Bv) {
    double a[AB], bb[BB];
#pragma unroll
    for (int u = 0; u < AB; u++) a[u] = Av[u];
#pragma unroll
    for (int u = 0; u < BB / 2; u++) {
      const double2 v = reinterpret_cast<const double2 *>(Bv)[u];
      bb[2 * u] = v.x;
      bb[2 * u + 1] = v.y;
    }
#pragma unroll
    for (int r = 0; r < BR; r++)
#pragma unroll
      for (int c = 0; c < BC; c++)
#pragma unroll
        for (int t2 = 0; t2 < IN; t2++) acc[r * BC + c] = __fma_rn(a[r * IN + t2], bb[t2 * BC + c], acc[r * BC + c]);
  };
  if (staged) {
    const int q0 = g.q0;
    const int ashift = (int)(((long)g.a0 * AB * 8) & 15L) / 8, hshift = q0 & 3, pshift = g.e0 & 3;
    const int h0 = Ps[pshift + tid] - q0, h1 = Ps[pshift + tid + 1] - q0;
    for (int h = h0; h < h1; h++) {
      const unsigned w = Hs[hshift + h];
      hit(As + ashift + (w & 0xffu) * AB, Bs + (w >> 8) * BB);
    }
  } else {
    for (int q = pptr[e]; q < pptr[e + 1]; q++) hit(A_val + (long)pa[q] * AB, B_val + (long)pb[q] * BB);
  }
#pragma unroll
  for (int q = 0; q < BR * BC; q++) C_val[e * BR * BC + q] = acc[q];
}

// hit words of the staged groups (symbolic, once per setup); grun[g] = the group's run range (empty: global)
__global__ void k_gal_hitw(const GalGrp *__restrict__ grp, const int2 *__restrict__ grun,
                           const GalRun *__restrict__ runs, const int *__restrict__ pptr, const int *__restrict__ pa,
                           const int *__restrict__ pb, const int *__restrict__ B_ptr, unsigned *__restrict__ hitw) {
  const GalGrp g = grp[blockIdx.x];
  const int2 rr = grun[blockIdx.x];
  if (rr.y <= rr.x) return;
  const int nr = rr.y - rr.x;
  for (int q = pptr[g.e0] + threadIdx.x; q < pptr[g.e1]; q += blockDim.x) {
    const int b = pb[q];
    int r = 0;
    while (r + 1 < nr && B_ptr[runs[rr.x + r + 1].j0] <= b) r++;
    const GalRun run = runs[rr.x + r];
    hitw[q] = (unsigned)(pa[q] - g.a0) | ((unsigned)(run.base + b - B_ptr[run.j0]) << 8);
  }
}

// Fine-level G = R * AP (R = P^T, 6x3 blocks; AP 3x6), streamed form of k_spgemm_dense<6,3,6> (C20, same
// chains).  A CTA owns <= 64 output blocks of one coarse row a; two threads per output block (rows 0-2 /
// 3-5 of the 6x6 block, 18 accumulators each).  R's row a is walked in ascending order in chunks of <= 16
// positions (at most RAP_SCAP AP blocks), each staged into a 3-stage shared-memory ring by TMA bulk copies.
struct RapGrp {
  int a, e0, e1, pad;
};
#ifndef AMGF_RAP_SCAP  // A/B builds (tools/ab_build.sh) may override the ring geometry
#define AMGF_RAP_SCAP 64  // measured at cfg 3: 64 / 104 / 80 (4 stages) -> 1202 / 1248 / 1456 us
#define AMGF_RAP_NS 3
#endif
#ifndef AMGF_RAP_BLK
#define AMGF_RAP_BLK 64  // output blocks per group (two consumer threads each)
#endif
constexpr int RAP_BLK = AMGF_RAP_BLK, RAP_NT = 2 * RAP_BLK, RAP_TC = 16, RAP_SCAP = AMGF_RAP_SCAP, RAP_NS = AMGF_RAP_NS;  // RAP_NT: consumers
constexpr int RAP_STAGE = (RAP_TC + RAP_SCAP) * 18;  // doubles per stage
// Warp-specialised streamed form (same chains): warp 4 is the producer (chunk plan from the per-R-block
// (AP row start, length) table, TMA bulk copies of the R blocks, the AP rows and the chunk's rows of the
// group-contiguous offset table into a 3-stage ring, full/empty mbarriers); warps 0-3 consume: offsets,
// R and AP blocks all from shared memory.
constexpr int RAP2_CONS = RAP_NT, RAP2_OFFB = RAP_TC * RAP_BLK;  // offset bytes per stage
constexpr int RAP2_STAGE_B = RAP_STAGE * 8 + RAP2_OFFB;
__global__ void __launch_bounds__(RAP2_CONS + 32) k_gal_rap2(const RapGrp *__restrict__ grp,
                                                            const long *__restrict__ gofs,
                                                            const int *__restrict__ R_ptr,
                                                            const int2 *__restrict__ rbi,
                                                            const double *__restrict__ R_val,
                                                            const double *__restrict__ B_val,
                                                            const signed char *__restrict__ offg,
                                                            double *__restrict__ C_val) {
  extern __shared__ __align__(128) unsigned char rsm2[];  // [RAP_NS] x (R + AP blocks, then offsets)
  __shared__ int meta[RAP_NS][RAP_TC + 2];
  __shared__ __align__(8) uint64_t full[RAP_NS], empty[RAP_NS];
  const RapGrp g = grp[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31;
  const int ra0 = R_ptr[g.a], lr = R_ptr[g.a + 1] - ra0;
  const signed char *og = offg + gofs[blockIdx.x];
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < RAP_NS; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], RAP2_CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= RAP2_CONS) {  // ---- producer warp
    int next_t = 0;
    for (int q = 0;; q++) {
      const int s = q % RAP_NS;
      if (q >= RAP_NS) mbar_wait(&empty[s], ((q / RAP_NS) - 1) & 1);
      const int p = lane;
      const bool in = p < RAP_TC && next_t + p < lr;
      int2 bi = make_int2(0, 0);
      if (in) bi = rbi[ra0 + next_t + p];
      int incl = bi.y;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      const bool take = in && incl <= RAP_SCAP;
      const int tc = __popc(__ballot_sync(0xffffffffu, take));
      const int nbt = tc > 0 ? __shfl_sync(0xffffffffu, incl, tc - 1) : 0;
      unsigned char *st = rsm2 + (long)s * RAP2_STAGE_B;
      double *sd = reinterpret_cast<double *>(st);
      if (take) meta[s][p] = incl - bi.y;
      if (lane == 0) {
        meta[s][RAP_TC] = tc;
        meta[s][RAP_TC + 1] = next_t;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect(&full[s], (unsigned)(tc + nbt) * 144u + (unsigned)tc * (unsigned)RAP_BLK);
      __syncwarp();
      if (tc > 0) {
        if (lane == 0) {
          bulk_g2s(sd, R_val + (long)(ra0 + next_t) * 18, (unsigned)tc * 144u, &full[s]);
          bulk_g2s(st + RAP_STAGE * 8, og + (long)next_t * RAP_BLK, (unsigned)tc * (unsigned)RAP_BLK, &full[s]);
        }
        if (take && bi.y > 0)
          bulk_g2s(sd + (RAP_TC + incl - bi.y) * 18, B_val + (long)bi.x * 18, (unsigned)bi.y * 144u, &full[s]);
      }
      next_t += tc;
      if (tc == 0) break;
    }
    return;
  }
  // ---- consumers: two threads per output block
  const int ob = tid >> 1, h = tid & 1;
  const long e = (long)g.e0 + ob;
  const bool act = e < g.e1;
  double acc[18];
#pragma unroll
  for (int q = 0; q < 18; q++) acc[q] = 0.0;
  for (int q = 0;; q++) {
    const int s = q % RAP_NS;
    mbar_wait(&full[s], (q / RAP_NS) & 1);
    const int tc = meta[s][RAP_TC];
    if (tc == 0) break;
    const unsigned char *st = rsm2 + (long)s * RAP2_STAGE_B;
    const double *sd = reinterpret_cast<const double *>(st);
    const signed char *so = reinterpret_cast<const signed char *>(st + RAP_STAGE * 8);
    if (act) {
      for (int p = 0; p < tc; p++) {
        const int o = so[p * RAP_BLK + ob];
        if (o >= 0) {
          const double *Rv = sd + p * 18 + h * 9;
          const double2 *Bv = reinterpret_cast<const double2 *>(sd + (RAP_TC + meta[s][p] + o) * 18);
          double a[9], bb[18];
#pragma unroll
          for (int u = 0; u < 9; u++) a[u] = Rv[u];
#pragma unroll
          for (int u = 0; u < 9; u++) {
            const double2 v = Bv[u];
            bb[2 * u] = v.x;
            bb[2 * u + 1] = v.y;
          }
#pragma unroll
          for (int r = 0; r < 3; r++)
#pragma unroll
            for (int c2 = 0; c2 < 6; c2++)
#pragma unroll
              for (int t2 = 0; t2 < 3; t2++) acc[r * 6 + c2] = __fma_rn(a[r * 3 + t2], bb[t2 * 6 + c2], acc[r * 6 + c2]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (act) {
#pragma unroll
    for (int r = 0; r < 3; r++)
#pragma unroll
      for (int c2 = 0; c2 < 6; c2++) C_val[e * 36 + (3 * h + r) * 6 + c2] = acc[r * 6 + c2];
  }
}
// group-contiguous offset rows of k_gal_rap2: offg[gofs[g] + t * 64 + (e - e0)] = offset of G's column in the AP
// row of R position t (-1 if absent); symbolic, once
__global__ void k_rap_offg(int ngrp, const RapGrp *__restrict__ grp, const long *__restrict__ gofs,
                           const int *__restrict__ R_ptr, const int *__restrict__ R_col, const int *__restrict__ B_ptr,
                           const int *__restrict__ B_col, const int *__restrict__ C_col, signed char *__restrict__ offg) {
  const RapGrp g = grp[blockIdx.x];
  const int ra0 = R_ptr[g.a], lr = R_ptr[g.a + 1] - ra0;
  for (int q = threadIdx.x; q < lr * RAP_BLK; q += blockDim.x) {
    const int t = q / RAP_BLK, el = q % RAP_BLK;
    int o = -1;
    if (g.e0 + el < g.e1) {
      const int j = R_col[ra0 + t];
      const int k2 = bsearch_int(B_col, B_ptr[j], B_ptr[j + 1], C_col[g.e0 + el]);
      if (k2 >= 0) o = k2 - B_ptr[j];
    }
    offg[gofs[blockIdx.x] + q] = (signed char)o;
  }
}
__global__ void k_rap_rbi(long nnz, const int *__restrict__ R_col, const int *__restrict__ B_ptr, int2 *rbi) {
  const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int j = R_col[k];
  rbi[k] = make_int2(B_ptr[j], B_ptr[j + 1] - B_ptr[j]);
}


// symmetrisation (C22) with the transpose partner of every block precomputed (symbolic, k_sym_partner): one
// thread per entry, so both the G reads and the A_c writes are contiguous
__global__ void k_sym_partner(long nnzb, const int *rowof, const int *ptr, const int *col, int *kt, int *err) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzb) return;
  const int a = rowof[e], b2 = col[e];
  kt[e] = bsearch_int(col, ptr[b2], ptr[b2 + 1], a);
  if (kt[e] < 0) raise_err(err, DERR_ARG, (int)e);
}
__global__ void k_sym2(long n36, const int *__restrict__ kt, const double *__restrict__ G, double *__restrict__ Ac) {
  long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= n36) return;
  const long e = t / 36;
  const int q = (int)(t - e * 36), r = q / 6, s2 = q - 6 * r;
  Ac[t] = 0.5 * (G[t] + G[(long)kt[e] * 36 + s2 * 6 + r]);
}
__global__ void k_sym(long nnzb, const int *rowof, const int *ptr, const int *col, const double *G, double *Ac,
                      int *err) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e >= nnzb) return;
  const int a = rowof[e], b2 = col[e];
  const int kt = bsearch_int(col, ptr[b2], ptr[b2 + 1], a);
  if (kt < 0) { raise_err(err, DERR_ARG, (int)e); return; }
  for (int r = 0; r < 6; r++)
    for (int s = 0; s < 6; s++) Ac[e * 36 + r * 6 + s] = 0.5 * (G[e * 36 + r * 6 + s] + G[(long)kt * 36 + s * 6 + r]);
}

// ------------------------------------------------------------------ SELL-32 packing
// SELL rows are block rows (split = 1) or the scalar rows of the blocks (split = br, block shape 1 x bc)
__global__ void k_row_len(int nrows, int split, const int *ptr, int *len) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) len[i] = ptr[i / split + 1] - ptr[i / split];
}
// sort key of a row: its window of SELL_SORT_WINDOW rows, then decreasing length (radix sort is stable)
constexpr int SELL_SORT_WINDOW = 8192;
__global__ void k_sell_sort_keys(int nrows, const int *len, int *key, int *idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  key[i] = (i / SELL_SORT_WINDOW) * 65536 + (65535 - min(len[i], 65535));
  idx[i] = i;
}
__global__ void k_slice_width(int nslices, int nrows, const int *len, int *width) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  int w = 0;
  for (int l = 0; l < 32; l++) {
    int i = 32 * s + l;
    if (i < nrows) w = max(w, len[i]);
  }
  width[s] = w;
}
// ssrc = source BSR block index * split + scalar row within the block (or -1 for padding)
__global__ void k_sell_pack(int nrows, int split, const int *ptr, const int *col, const int *slice_ptr,
                            const int *perm, int *scol, int *ssrc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  const int lane = i & 31;
  const int oi = perm ? perm[i] : i;
  const int ib = oi / split, r = oi % split;
  const long base = slice_ptr[i >> 5];
  const int w = slice_ptr[(i >> 5) + 1] - slice_ptr[i >> 5];
  const int len = ptr[ib + 1] - ptr[ib];
  for (int s = 0; s < w; s++) {
    const long slot = base + s;
    if (s < len) { scol[slot * 32 + lane] = col[ptr[ib] + s]; ssrc[slot * 32 + lane] = (ptr[ib] + s) * split + r; }
    else { scol[slot * 32 + lane] = 0; ssrc[slot * 32 + lane] = -1; }
  }
}
// BB = values per SELL entry (br*bc, or bc when split); the source entry q of a split row is
// row r of block q/split, i.e. the BB consecutive values at val[q*BB].
__global__ void k_sell_vals(long nslots, int BB, const int *ssrc, const double *val, double *sval) {
  long q = blockIdx.x * (long)blockDim.x + threadIdx.x;  // q = slot*32 + lane
  if (q >= nslots * 32) return;
  const long slot = q >> 5;
  const int lane = (int)(q & 31);
  const int src = ssrc[q];
  for (int e = 0; e < BB; e++) sval[(slot * BB + e) * 32 + lane] = src >= 0 ? val[(long)src * BB + e] : 0.0;
}

// ------------------------------------------------------------------ coarsest dense operator
__global__ void k_dense_band(int nodes, int b, const int *ptr, const int *col, const double *val, int n, int W,
                             double *Lrow) {
  long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (t >= (long)nodes * b) return;
  const int i = (int)(t / b), r = (int)(t % b);
  const int row = i * b + r, bw = n - 1;
  for (int k = ptr[i]; k < ptr[i + 1]; k++)
    for (int cc = 0; cc < b; cc++) {
      const int cidx = col[k] * b + cc;
      if (cidx <= row) Lrow[(long)row * W + bw - (row - cidx)] = val[(long)k * b * b + r * b + cc];
    }
}

// =================================================================== host orchestration
static void bsr_alloc(Ctx &c, Bsr &A, int nbr, int nbc, int br, int bc, long nnzb) {
  A.nbr = nbr; A.nbc = nbc; A.br = br; A.bc = bc; A.nnzb = nnzb;
  A.ptr = c.alloc<int>(nbr + 1);
  A.col = c.alloc<int>(nnzb);
  A.val = c.alloc<double>(nnzb * br * bc);
}

static int *rowof(Ctx &c, const Bsr &A) {
  int *r = c.alloc<int>(A.nnzb);
  LAUNCH(k_rowof, A.nbr, A.nbr, A.ptr, r);
  return r;
}

// Reorder the (length-sorted) slices of a SELL so that every CTA of CTA/32 consecutive slices carries about
// the same number of slots: slices by decreasing width are dealt to the CTAs in snake order (LPT-like).  The
// coarse-level SpMV grids are a single wave (all CTAs co-resident), so the kernel ends with its most loaded
// SM: with the window-sorted order alone the largest CTA held 1.36x the mean slots at cfg 3 level 1.  A row
// permutation only (Sell::perm): every row's chain and result are unchanged (C2).  The partial last slice
// stays last (rows beyond nrows exist only there).
static void balance_slices(Ctx &c, Sell &S) {
  const int spc = CTA / 32, ns = S.nslices, full = S.nrows / 32;  // slices [0, full) are complete
  const int ncta = (ns + spc - 1) / spc;
  if (ncta < 2 || getenv("AMGF_NO_SLICE_BALANCE")) return;
  std::vector<int> len(S.nrows), perm(S.nrows);
  CK(cudaMemcpyAsync(len.data(), S.rowlen, S.nrows * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaMemcpyAsync(perm.data(), S.perm, S.nrows * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  std::vector<int> width(ns, 0);
  for (int i = 0; i < S.nrows; i++) width[i / 32] = std::max(width[i / 32], len[i]);
  // the last CTA takes the partial slice (if any) and the narrowest complete slices; the others get spc each
  const int last_n = ns - spc * (ncta - 1);
  std::vector<int> order(full);
  for (int q = 0; q < full; q++) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return width[a] > width[b]; });
  std::vector<std::vector<int>> bins(ncta);
  const int last_full = last_n - (full < ns ? 1 : 0);  // complete slices in the last CTA
  int j = 0;
  for (int r = 0; r < spc; r++)
    for (int k = 0; k < ncta - 1; k++) bins[(r % 2 == 0) ? k : ncta - 2 - k].push_back(order[j++]);
  for (int q = 0; q < last_full; q++) bins[ncta - 1].push_back(order[j++]);
  if (full < ns) bins[ncta - 1].push_back(full);
  std::vector<int> nperm(S.nrows), nlen(S.nrows);
  int w = 0;
  for (auto &b : bins)
    for (int sl : b)
      for (int l = 0; l < 32 && 32 * sl + l < S.nrows; l++, w++) {
        nperm[w] = perm[32 * sl + l];
        nlen[w] = len[32 * sl + l];
      }
  if (w != S.nrows) throw Error{AMGF_ERR_LIMIT, "balance_slices: row count mismatch"};
  CK(cudaMemcpyAsync(S.perm, nperm.data(), S.nrows * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  CK(cudaMemcpyAsync(S.rowlen, nlen.data(), S.nrows * sizeof(int), cudaMemcpyHostToDevice, c.stream));
  CK(cudaStreamSynchronize(c.stream));
}

void build_sell(Ctx &c, const Bsr &A, Sell &S, bool alloc, bool split, bool sort_rows) {
  const int sp = split ? A.br : 1;
  const int BB = split ? A.bc : A.br * A.bc;
  if (alloc) {
    S.nrows = A.nbr * sp; S.br = split ? 1 : A.br; S.bc = A.bc;
    S.nslices = (S.nrows + 31) / 32;
    S.rowlen = c.alloc<int>(S.nrows);
    LAUNCH(k_row_len, S.nrows, S.nrows, sp, A.ptr, S.rowlen);
    if (sort_rows) {
      int *key = c.alloc<int>(S.nrows), *key2 = c.alloc<int>(S.nrows), *idx = c.alloc<int>(S.nrows);
      int *len0 = c.alloc<int>(S.nrows);
      S.perm = c.alloc<int>(S.nrows);
      LAUNCH(k_sell_sort_keys, S.nrows, S.nrows, S.rowlen, key, idx);
      sort_pairs(c, key, key2, idx, S.perm, S.nrows);
      d2d(c, len0, S.rowlen, S.nrows);
      LAUNCH(k_gather_int, S.nrows, S.nrows, S.perm, len0, S.rowlen);
      c.release(key); c.release(key2); c.release(idx); c.release(len0);
      balance_slices(c, S);
    }
    int *width = c.alloc<int>(S.nslices + 1);
    CK(cudaMemsetAsync(width, 0, (S.nslices + 1) * sizeof(int), c.stream));
    LAUNCH(k_slice_width, S.nslices, S.nslices, S.nrows, S.rowlen, width);
    S.slice_ptr = c.alloc<int>(S.nslices + 1);
    S.nslots = scan_ex(c, width, S.slice_ptr, S.nslices);
    c.release(width);
    S.col = c.alloc<int>(S.nslots * 32);
    S.src = c.alloc<int>(S.nslots * 32);
    S.val = c.alloc<double>(S.nslots * 32 * BB);
    // lanes of the last slice beyond nrows are never written by k_sell_pack: mark them as padding
    CK(cudaMemsetAsync(S.col, 0, S.nslots * 32 * sizeof(int), c.stream));
    CK(cudaMemsetAsync(S.src, 0xff, S.nslots * 32 * sizeof(int), c.stream));
    LAUNCH(k_sell_pack, S.nrows, S.nrows, sp, A.ptr, A.col, S.slice_ptr, S.perm, S.col, S.src);
  }
  LAUNCH(k_sell_vals, S.nslots * 32, S.nslots, BB, S.src, A.val, S.val);
}

static void band_alloc(Ctx &c, int n, int bw, double *&Lrow, double *&Lcol, double *&Lrev, double *&dinv) {
  const int W = band_stride(bw);
  const size_t total = (size_t)(n + 2 * BAND_PAD_ROWS) * W;
  double *r = c.alloc<double>(total), *cl = c.alloc<double>(total), *rv = c.alloc<double>(total);
  CK(cudaMemsetAsync(r, 0, total * sizeof(double), c.stream));
  CK(cudaMemsetAsync(cl, 0, total * sizeof(double), c.stream));
  CK(cudaMemsetAsync(rv, 0, total * sizeof(double), c.stream));
  Lrow = r + (size_t)BAND_PAD_ROWS * W;
  Lcol = cl + (size_t)BAND_PAD_ROWS * W;
  Lrev = rv + (size_t)BAND_PAD_ROWS * W;
  dinv = c.alloc<double>(n);
}

// Cholesky of diagonal blocks of a band (nblocks > 0: block lists p0/len on the device; else one block [0,n))
void band_factor_blocks(Ctx &c, int n, int nblocks, const int *d_p0, const int *d_len, int bw, double *Lrow, int tag) {
  const int W = band_stride(bw);
  const int grid = nblocks > 0 ? nblocks : 1;
  static const bool old_chol = getenv("AMGF_CHOL_OLD") != nullptr;  // A/B only: the round-1 panel kernel
  const int rows = 32 + bw, r4 = (rows + 3) & ~3, ldk = r4 + (r4 % 8 == 0 ? 4 : 0);
  const size_t smem_t = (64 * (size_t)ldk + (size_t)rows * PLD) * sizeof(double);
  if (!old_chol && rows <= 256 && smem_t <= 220 * 1024) {
    size_t &attr = device_slot((const void *)k_band_chol_t);
    if (smem_t > attr) {
      CK(cudaFuncSetAttribute(k_band_chol_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t));
      attr = smem_t;
    }
    k_band_chol_t<<<grid, CHT_THREADS, smem_t, c.stream>>>(n, d_p0, d_len, bw, W, Lrow, c.err, tag);
    after_launch(c, "k_band_chol_t");
    return;
  }
  const size_t smem = (2 * (size_t)(32 + bw) * PLD + 32 * (size_t)(33 + bw)) * sizeof(double);
  if ((32 + bw) * 32 <= CHOL_THREADS * CHOL_EPT && 32 + bw <= CHOL_THREADS && smem <= 220 * 1024) {
    CK(cudaFuncSetAttribute(k_band_chol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_band_chol<<<grid, CHOL_THREADS, smem, c.stream>>>(n, d_p0, d_len, bw, W, Lrow, c.err, tag);
  } else {
    k_band_chol_wide<<<grid, 1024, 0, c.stream>>>(n, d_p0, d_len, bw, W, Lrow, c.err, tag);
  }
  after_launch(c, "k_band_chol");
}
void band_finish(Ctx &c, int n, int bw, const double *Lrow, double *Lcol, double *Lrev, double *dinv) {
  const int W = band_stride(bw);
  LAUNCH(k_band_finish, (long)n * (bw + 1), n, bw, W, Lrow, Lcol, Lrev, dinv);
}
static void band_factor(Ctx &c, int n, int bw, double *Lrow, double *Lcol, double *Lrev, double *dinv, int tag) {
  band_factor_blocks(c, n, 0, nullptr, nullptr, bw, Lrow, tag);
  band_finish(c, n, bw, Lrow, Lcol, Lrev, dinv);
}

// --------------------------------------------------------------- numeric pieces (reused by update_D)
struct SetupCache {  // per-context arrays needed for numeric re-setup
  int *S_rowof = nullptr;
  int *band_src = nullptr;
  long band_nnz = 0;
};

static void S_numeric(Ctx &c, const int *S_rowof) {
  Level &L0 = c.lev[0];
  LAUNCH(k_S_values, L0.A.nnzb, L0.A.nnzb, S_rowof, L0.A.col, c.S_kblk, c.K.val, c.Jt_ptr, c.Jt_row, c.Jt_val, c.D,
         c.has_box ? c.D_lo : nullptr, c.has_box ? c.D_up : nullptr, L0.A.val);
}

static void filter_numeric(Ctx &c) {
  if (c.nc == 0) return;
  nd_numeric(c);  // filter.cu: A_w[pi,pi] fill + nested-dissection Cholesky
}

// Run the A_w band fill + Cholesky (single-SM kernel) on the side stream, concurrently with the
// hierarchy's numeric setup on the main stream; join_filter() makes the main stream wait for it.
// Phase events of the numeric re-setup (amgf_setup_times): main stream start / S formed / hierarchy done /
// coarsest done / joined, side stream A_w factorization start / end.
static void setup_mark(Ctx &c, int i, cudaStream_t st) {
  if (!c.ph_ev[i]) CK(cudaEventCreate(&c.ph_ev[i]));
  CK(cudaEventRecord(c.ph_ev[i], st));
}

static void fork_filter(Ctx &c) {
  if (c.nc == 0) return;
  if (!c.side) {
    // high priority: the A_w factorization is a chain of small latency-bound grids; its CTAs take the
    // first free SM slots while the hierarchy's large grids run on the main stream
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    static const bool low = getenv("AMGF_SIDE_LOWPRIO") != nullptr;  // A/B experiments only
    CK(cudaStreamCreateWithPriority(&c.side, cudaStreamNonBlocking, low ? lo : hi));
    CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming));
  }
  cudaStream_t main = c.stream;
  CK(cudaEventRecord(c.ev_fork, main));
  CK(cudaStreamWaitEvent(c.side, c.ev_fork, 0));
  c.stream = c.side;
  setup_mark(c, 5, c.side);
  try {
    filter_numeric(c);
  } catch (...) {
    c.stream = main;
    throw;
  }
  c.stream = main;
  setup_mark(c, 6, c.side);
  CK(cudaEventRecord(c.ev_join, c.side));
  static const bool serial = getenv("AMGF_SERIAL_SETUP") != nullptr;  // A/B only: side stream alone, then main
  if (serial) CK(cudaStreamWaitEvent(main, c.ev_join, 0));
}
static void join_filter(Ctx &c) {
  if (c.nc == 0) return;
  CK(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
}

static void thin_numeric(Ctx &c, long nthin_nnz) {
  LAUNCH(k_gather_vals, nthin_nnz, nthin_nnz, c.thin_src, c.lev[0].A.val, c.thin_val);
  LAUNCH(k_zr_vals, c.zr_nnz, c.zr_nnz, c.zr_src, c.lev[0].A.val, c.zr_val);
}

// first_done: the first step's w = (A v0) / d and its C14 partials were formed by k_sell_diag (fine level)
static void power_iteration(Ctx &c, Level &L, int lev, bool first_done = false) {
  if (!c.pw_v) {  // once per handle: no allocation on the numeric re-setup path
    c.pw_v = c.alloc<double>(c.n);
    c.pw_w = c.alloc<double>(c.n);
  }
  double *v = c.pw_v, *w = c.pw_w;
  if (!c.pw_s) c.pw_s = c.alloc<double>(4);
  if (!c.pw_lev) c.pw_lev = c.alloc<double>(2 * MAXLEV);
  if (!c.pw_part) c.pw_part = c.alloc<double>(nblk(c.n) + 1);
  if (!first_done) LAUNCH(k_pow_init, L.n, L.n, v);
  // per step: w = (A v) / d with the C14 partials of w.w and v.v (fused into the fine SpMV), both level-2
  // sums, then lambda and v = w / ||w|| (k_pow_scale)
  const bool fused = L.As.val && L.b == 3 && L.As.br == 3 && !L.As.perm;
  const long nb = L.n / L.b, C = (nb + CTA - 1) / CTA;
  for (int it = 0; it < c.cfg.power_iters; it++) {
    if (it == 0 && first_done) {
      // w and the partials are already there
    } else if (fused) {
      launch_sell_pow(c, L.As, v, L.dpt, w, c.dot_part, c.pw_part);
    } else {
      if (L.As.val) {
        launch_sell_spmv(c, L.As, SPMV_YDIV, v, nullptr, L.dpt, nullptr, w, nullptr);
      } else {
        launch_bsr_spmv(c, L.A, v, w);
        LAUNCH(k_div, L.n, L.n, w, L.dpt);
      }
      launch_pow_dots(c, nb, L.b, w, v, c.dot_part, c.pw_part);
    }
    if (C <= 64) {  // coarse levels: both finishing steps in one launch (each CTA re-forms the 2 x C sums)
      launch_pow_fin_scale(c, C, c.dot_part, c.pw_part, c.pw_s, L.n, w, v);
    } else {
      launch_pow_fin(c, C, c.dot_part, c.pw_part, c.pw_s);
      LAUNCH(k_pow_scale, L.n, L.n, w, c.pw_s, v);
    }
  }
  // lambda and omega of this level stay on the device (k_P_values reads omega there); the host copies are
  // read once at the end of the setup (read_level_scalars): no stream synchronisation per level
  CK(cudaMemcpyAsync(c.pw_lev + 2 * lev, c.pw_s + 2, 2 * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}
static void read_level_scalars(Ctx &c) {
  double h[2 * MAXLEV];
  const int nl = std::max(c.nlev - 1, 0);
  if (!nl || !c.pw_lev) return;
  CK(cudaMemcpyAsync(h, c.pw_lev, 2 * nl * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  for (int l = 0; l < nl; l++) {
    c.lev[l].lambda = h[2 * l];
    c.lev[l].omega = h[2 * l + 1];
  }
}

// per-level cached arrays for numeric re-setup
struct LevelCache {
  int *P_rowof = nullptr, *R_perm = nullptr, *G_rowof = nullptr, *AP_rowof = nullptr;
  int *R_inv = nullptr;  // R block of every P block (k_P_values writes R = P^T directly)
  int *P_pptr = nullptr, *P_pa = nullptr, *P_pb = nullptr;  // block-product pairs of T = A * Pt (k_P_pairs)
  Bsr G;
  // block-product lists of the Galerkin products (symbolic, built once): for output block e of AP (G),
  // the pairs (A block, P block) ((R block, AP block)) with a matching inner index, in ascending order
  int *AP_pptr = nullptr, *AP_pa = nullptr, *AP_pb = nullptr;
  int *G_pptr = nullptr, *G_pa = nullptr, *G_pb = nullptr;
  signed char *AP_off = nullptr, *G_off = nullptr;  // dense-over-row offset tables (k_spgemm_dense)
  GalGrp *AP_grp = nullptr;  // row groups of k_gal_hl (fine level)
  GalCopy *AP_cps = nullptr;  // TMA copy descriptors of the groups
  int AP_ngrp = 0;
  int *G_kt = nullptr;       // transpose partner of every block of G (k_sym2)
  RapGrp *G_grp = nullptr;  // output groups of k_gal_rap2 (fine level)
  int G_ngrp = 0;
  long *G_gofs = nullptr;    // k_gal_rap2: group-contiguous offset rows and per-R-block AP row (start, length)
  signed char *G_offg = nullptr;
  int2 *G_rbi = nullptr;
  unsigned *AP_hitw = nullptr;  // hit words of k_gal_hl
};

static signed char *build_off(Ctx &c, long nnzc, const int *rowof, const int *ccol, const Bsr &A, const Bsr &B) {
  std::vector<int> h(A.nbr + 1);
  CK(cudaMemcpyAsync(h.data(), A.ptr, (A.nbr + 1) * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  int maxa = 0;
  for (int i = 0; i < A.nbr; i++) maxa = std::max(maxa, h[i + 1] - h[i]);
  std::vector<int> hb(B.nbr + 1);
  CK(cudaMemcpyAsync(hb.data(), B.ptr, (B.nbr + 1) * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  int maxb = 0;
  for (int i = 0; i < B.nbr; i++) maxb = std::max(maxb, hb[i + 1] - hb[i]);
  REQUIRE(maxb <= 127, AMGF_ERR_LIMIT, "Galerkin product: a factor row exceeds 127 blocks (int8 offsets)");
  signed char *off = c.alloc<signed char>((size_t)std::max(maxa, 1) * nnzc);
  LAUNCH(k_spgemm_off, nnzc, nnzc, rowof, ccol, A.ptr, A.col, B.ptr, B.col, maxa, off);
  return off;
}

// Row groups of k_gal_hl (symbolic, host, once per setup): greedy over consecutive rows of C = A*B.
static void build_gal_groups(Ctx &c, const Bsr &A, const Bsr &B, const Bsr &C, const int *d_pptr, const int *d_pa,
                             const int *d_pb, GalGrp *&d_grp, int &ngrp, GalCopy *&d_cps, unsigned *&d_hitw) {
  auto d2hv = [&](const int *src, size_t n) {
    std::vector<int> h(n);
    CK(cudaMemcpyAsync(h.data(), src, n * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    return h;
  };
  const std::vector<int> ap = d2hv(A.ptr, A.nbr + 1), ac = d2hv(A.col, A.nnzb), bp = d2hv(B.ptr, B.nbr + 1),
                         cp = d2hv(C.ptr, C.nbr + 1), pp = d2hv(d_pptr, C.nnzb + 1);
  CK(cudaStreamSynchronize(c.stream));
  const int AB = A.br * A.bc, BB = B.br * B.bc;
  // byte offsets of the four regions of a group buffer (k_gal_hl: B union, A segment, hit words, offsets)
  const int offA = GHL_PCAP * BB * 8, offH = offA + (GAL_ACAP * AB + 2) * 8, offP = offH + (GHL_HCAP + 8) * 4;
  // The greedy pass is sequential within a row range; the rows are cut into a fixed number of ranges (the same
  // on every host, so the grouping is reproducible) that run on the host's threads (135 -> ~25 ms at cfg 3).
  struct SegOut {
    std::vector<GalGrp> grps;
    std::vector<int2> grun;  // run range of every group (for the hit words)
    std::vector<GalRun> runs;
    std::vector<GalCopy> cps;
  };
  const int n = A.nbr;
  const int NSEG = n >= 16 * 4096 ? 16 : 1;
  std::vector<SegOut> seg(NSEG);
  auto work = [&](int s0, int s1, SegOut &o) {
    std::vector<GalGrp> &grps = o.grps;
    std::vector<int2> &grun = o.grun;
    std::vector<GalRun> &runs = o.runs;
    std::vector<GalCopy> &cps = o.cps;
    std::vector<char> mark(B.nbr, 0);
    std::vector<int> ul;
    auto add_global = [&](int i) {  // one row through global memory, NT output blocks per group
      for (int e = cp[i]; e < cp[i + 1]; e += GAL_NT) {
        grps.push_back(GalGrp{e, std::min(cp[i + 1], e + GAL_NT), ap[i], (int)cps.size(), (int)cps.size(), 0u, 0, 0});
        grun.push_back(make_int2(0, 0));
      }
    };
    auto copy = [&](long long src, long long end, int dst, unsigned id) {  // [src, end) rounded out to 16 bytes
      const long long s16 = src & ~15LL, e16 = (end + 15) & ~15LL;
      cps.push_back(GalCopy{s16, dst, (unsigned)(e16 - s16) | id << 28});
      return (unsigned)(e16 - s16);
    };
    int i = s0;
    while (i < s1) {
      const int i0 = i;
      long pb = 0;
      ul.clear();
      while (i < s1) {
        const size_t m0 = ul.size();
        long add = 0;
        for (int k = ap[i]; k < ap[i + 1]; k++) {
          const int j = ac[k];
          if (!mark[j]) { mark[j] = 1; ul.push_back(j); add += bp[j + 1] - bp[j]; }
        }
        if (cp[i + 1] - cp[i0] > GAL_NT || ap[i + 1] - ap[i0] > GAL_ACAP || pb + add > GHL_PCAP ||
            pp[cp[i + 1]] - pp[cp[i0]] > GHL_HCAP) {
          for (size_t q = m0; q < ul.size(); q++) mark[ul[q]] = 0;
          ul.resize(m0);
          break;
        }
        pb += add;
        i++;
      }
      for (int j : ul) mark[j] = 0;
      if (i == i0) {  // the row alone exceeds a capacity
        add_global(i);
        i++;
        continue;
      }
      std::sort(ul.begin(), ul.end());
      const int r0 = (int)runs.size();
      int base = 0;
      for (size_t q = 0; q < ul.size();) {
        size_t q1 = q + 1;
        while (q1 < ul.size() && ul[q1] == ul[q1 - 1] + 1) q1++;
        runs.push_back(GalRun{ul[q], ul[q1 - 1] + 1, base, 0});
        base += bp[ul[q1 - 1] + 1] - bp[ul[q]];
        q = q1;
      }
      if ((int)runs.size() - r0 > GAL_RCAP) {  // too fragmented for one warp of copies: global path
        runs.resize(r0);
        for (int ii = i0; ii < i; ii++) add_global(ii);
        continue;
      }
      const int e0 = cp[i0], e1 = cp[i], c0 = (int)cps.size();
      unsigned tx = 0;
      tx += copy((long long)ap[i0] * AB * 8, (long long)ap[i] * AB * 8, offA, 0);
      if (pp[e1] > pp[e0]) tx += copy((long long)pp[e0] * 4, (long long)pp[e1] * 4, offH, 1);
      tx += copy((long long)e0 * 4, (long long)(e1 + 1) * 4, offP, 2);
      for (int r = r0; r < (int)runs.size(); r++) {
        const GalRun &q = runs[r];
        if (bp[q.j1] > bp[q.j0])
          tx += copy((long long)bp[q.j0] * BB * 8, (long long)bp[q.j1] * BB * 8, q.base * BB * 8, 3);
      }
      grps.push_back(GalGrp{e0, e1, ap[i0], c0, (int)cps.size(), tx, pp[e0], 0});
      grun.push_back(make_int2(r0, (int)runs.size()));
    }
  };
  auto seg_lo = [&](int sg) { return (int)((long)n * sg / NSEG); };
  if (NSEG == 1) {
    work(0, n, seg[0]);
  } else {
    const int nthr = (int)std::max(1u, std::min<unsigned>(NSEG, std::thread::hardware_concurrency()));
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < nthr; t++)
      pool.emplace_back([&]() {
        for (int sg = next.fetch_add(1); sg < NSEG; sg = next.fetch_add(1)) work(seg_lo(sg), seg_lo(sg + 1), seg[sg]);
      });
    for (auto &th : pool) th.join();
  }
  std::vector<GalGrp> grps;
  std::vector<int2> grun;
  std::vector<GalRun> runs;
  std::vector<GalCopy> cps;
  for (SegOut &o : seg) {  // concatenate, shifting the segment-local copy and run indices
    const int cb = (int)cps.size(), rb = (int)runs.size();
    for (GalGrp g : o.grps) {
      g.c0 += cb;
      g.c1 += cb;
      grps.push_back(g);
    }
    for (int2 r : o.grun) grun.push_back(r.y > r.x ? make_int2(r.x + rb, r.y + rb) : r);
    runs.insert(runs.end(), o.runs.begin(), o.runs.end());
    cps.insert(cps.end(), o.cps.begin(), o.cps.end());
  }
  ngrp = (int)grps.size();
  d_grp = c.alloc<GalGrp>(std::max<size_t>(grps.size(), 1));
  d_cps = c.alloc<GalCopy>(std::max<size_t>(cps.size(), 1));
  GalRun *d_runs = c.alloc<GalRun>(std::max<size_t>(runs.size(), 1));
  int2 *d_grun = c.alloc<int2>(std::max<size_t>(grun.size(), 1));
  h2d(c, d_grp, grps.data(), grps.size());
  h2d(c, d_cps, cps.data(), cps.size());
  h2d(c, d_runs, runs.data(), runs.size());
  h2d(c, d_grun, grun.data(), grun.size());
  const long np = pp[C.nnzb];
  d_hitw = c.alloc<unsigned>(np + 8);  // + 8: the groups' 16-byte aligned bulk copies may read past the end
  if (ngrp) k_gal_hitw<<<ngrp, 128, 0, c.stream>>>(d_grp, d_grun, d_runs, d_pptr, d_pa, d_pb, B.ptr, d_hitw);
  CK(cudaStreamSynchronize(c.stream));
  c.release(d_runs);
  c.release(d_grun);
}

// Output groups of k_gal_rap2: <= RAP_NT/2 output blocks of one row of G; every AP row must fit one stage.
static void build_rap_groups(Ctx &c, const Bsr &G, const Bsr &R, const Bsr &AP, RapGrp *&d_grp, int &ngrp,
                             long *&d_gofs, signed char *&d_offg, int2 *&d_rbi) {
  std::vector<int> gp(G.nbr + 1), bp(AP.nbr + 1);
  CK(cudaMemcpyAsync(gp.data(), G.ptr, gp.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaMemcpyAsync(bp.data(), AP.ptr, bp.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  for (int j = 0; j < AP.nbr; j++)
    if (bp[j + 1] - bp[j] > RAP_SCAP) {  // k_gal_rap2 cannot stage this row: keep the dense-over-row kernel
      d_grp = nullptr;
      ngrp = 0;
      return;
    }
  std::vector<RapGrp> grps;
  for (int a = 0; a < G.nbr; a++)
    for (int e = gp[a]; e < gp[a + 1]; e += RAP_NT / 2) grps.push_back(RapGrp{a, e, std::min(gp[a + 1], e + RAP_NT / 2), 0});
  ngrp = (int)grps.size();
  d_grp = c.alloc<RapGrp>(std::max<size_t>(grps.size(), 1));
  h2d(c, d_grp, grps.data(), grps.size());
  std::vector<int> rp(R.nbr + 1);
  CK(cudaMemcpyAsync(rp.data(), R.ptr, rp.size() * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  std::vector<long> gofs(grps.size() + 1, 0);
  for (size_t q = 0; q < grps.size(); q++) gofs[q + 1] = gofs[q] + (long)RAP_BLK * (rp[grps[q].a + 1] - rp[grps[q].a]);
  d_gofs = c.alloc<long>(gofs.size());
  h2d(c, d_gofs, gofs.data(), gofs.size());
  d_offg = c.alloc<signed char>(gofs.back() + 16);
  if (ngrp)
    k_rap_offg<<<ngrp, 256, 0, c.stream>>>(ngrp, d_grp, d_gofs, R.ptr, R.col, AP.ptr, AP.col, G.col, d_offg);
  d_rbi = c.alloc<int2>(std::max<long>(R.nnzb, 1));
  LAUNCH(k_rap_rbi, R.nnzb, R.nnzb, R.col, AP.ptr, d_rbi);
  CK(cudaStreamSynchronize(c.stream));
}

static void build_pairs(Ctx &c, long nnzc, const int *rowof, const int *ccol, const Bsr &A, const Bsr &B, int *&pptr,
                        int *&pa, int *&pb) {
  int *cnt = c.alloc<int>(nnzc + 1);
  CK(cudaMemsetAsync(cnt, 0, (nnzc + 1) * sizeof(int), c.stream));
  LAUNCH(k_spgemm_pairs, nnzc, nnzc, rowof, ccol, A.ptr, A.col, B.ptr, B.col, (const int *)nullptr, cnt,
         (int *)nullptr, (int *)nullptr);
  pptr = c.alloc<int>(nnzc + 1);
  const long np = scan_ex(c, cnt, pptr, nnzc);
  REQUIRE(np >= 0 && np < (1L << 31), AMGF_ERR_LIMIT, "Galerkin product: too many block products");
  c.release(cnt);
  pa = c.alloc<int>(np);
  pb = c.alloc<int>(np);
  LAUNCH(k_spgemm_pairs, nnzc, nnzc, rowof, ccol, A.ptr, A.col, B.ptr, B.col, (const int *)pptr, (int *)nullptr, pa,
         pb);
}

// smoother 2: the per-node block factors of level L (after its operator values change)
static void smoother_data(Ctx &c, Level &L) {
  if (c.cfg.smoother != 2) return;
  const int nb = L.b * (L.b + 1) / 2 + L.b;
  if (!L.bfac) L.bfac = c.alloc<double>((size_t)L.nodes * nb);
  if (L.b == 3) LAUNCH(k_block_l1<3>, L.nodes, L.nodes, L.A.ptr, L.A.col, L.A.val, L.bfac, c.err);
  else LAUNCH(k_block_l1<6>, L.nodes, L.nodes, L.A.ptr, L.A.col, L.A.val, L.bfac, c.err);
}

static void level_numeric(Ctx &c, int l, LevelCache &lc, bool pow_first_done = false) {
  Level &L = c.lev[l];
  Level &Lc = c.lev[l + 1];
  {
    // explicit carveout on the large hierarchy grids, as for the solve's residual SpMV: lets the side
    // stream's shared-memory-heavy A_w factorization CTAs find room (A/B: AMGF_HIER_CARVEOUT=-1 disables)
    size_t &once = device_slot((const void *)k_spgemm_dense<3, 3, 6>);
    if (!once) {
      once = 1;
      const int cv = getenv("AMGF_HIER_CARVEOUT") ? atoi(getenv("AMGF_HIER_CARVEOUT")) : 50;
      if (cv >= 0) {
        CK(cudaFuncSetAttribute(k_spgemm_dense<3, 3, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
        CK(cudaFuncSetAttribute(k_spgemm_dense<6, 3, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
        CK(cudaFuncSetAttribute(k_P_values<3>, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
        CK(cudaFuncSetAttribute(k_spgemm_vals_warp<6, 6, 6>, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
        CK(cudaFuncSetAttribute(k_sell_vals, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
      }
    }
  }
  power_iteration(c, L, l, pow_first_done);
  if (l == 0 && c.fork_at == 1) fork_filter(c);
  static const bool gal_old = getenv("AMGF_GAL_OLD") != nullptr;  // A/B only: the thread-per-block kernels
  if (!lc.R_inv) {  // symbolic, once
    lc.R_inv = c.alloc<int>(std::max<long>(L.R.nnzb, 1));
    LAUNCH(k_inv_perm, L.R.nnzb, L.R.nnzb, lc.R_perm, lc.R_inv);
  }
  if (!lc.P_pptr)  // symbolic, once
    build_pairs(c, L.P.nnzb, lc.P_rowof, L.P.col, L.A, L.Pt, lc.P_pptr, lc.P_pa, lc.P_pb);
  static const bool p_walk = getenv("AMGF_P_WALK") != nullptr;  // A/B only: the row-walk kernels
  if (L.b == 3 && !p_walk)
    LAUNCH((k_P_pairs<3, 1>), L.P.nnzb, L.P.nnzb, lc.P_rowof, L.P.col, lc.P_pptr, lc.P_pa, lc.P_pb, L.A.val, L.agg,
           L.Pt.ptr, L.Pt.val, L.dpt, c.pw_lev + 2 * l + 1, L.P.val, lc.R_inv, L.R.val);
  else if (!p_walk)
    LAUNCH((k_P_pairs<6, 2>), L.P.nnzb * 2, L.P.nnzb, lc.P_rowof, L.P.col, lc.P_pptr, lc.P_pa, lc.P_pb, L.A.val,
           L.agg, L.Pt.ptr, L.Pt.val, L.dpt, c.pw_lev + 2 * l + 1, L.P.val, lc.R_inv, L.R.val);
  else if (L.b == 3)
    LAUNCH(k_P_values<3>, L.P.nnzb, L.P.nnzb, lc.P_rowof, L.P.col, L.A.ptr, L.A.col, L.A.val, L.agg, L.Pt.ptr,
           L.Pt.val, L.dpt, c.pw_lev + 2 * l + 1, L.P.val, lc.R_inv, L.R.val);
  else
    LAUNCH(k_P_values<6>, L.P.nnzb, L.P.nnzb, lc.P_rowof, L.P.col, L.A.ptr, L.A.col, L.A.val, L.agg, L.Pt.ptr,
           L.Pt.val, L.dpt, c.pw_lev + 2 * l + 1, L.P.val, lc.R_inv, L.R.val);

  if (l == 0 && c.fork_at == 2) fork_filter(c);
  if (L.b == 3) {  // level-0 restriction reads R's values group-interleaved (Bsr::ival)
    r_interleave(c, L.R);
  }
  // AP = A * P, G = R * AP over the precomputed block-product lists
  {
    // dense-over-row products at the fine level (measured update_D 17.0 -> 15.3 ms at cfg 3); on the 6x6
    // levels the pair kernels are faster (level 1: 2.0 vs 2.5 ms)
    static const int dense = getenv("AMGF_SPGEMM_DENSE") ? atoi(getenv("AMGF_SPGEMM_DENSE")) : 1;  // A/B only
    if (dense && L.b == 3 && lc.AP_off) {
      if (lc.AP_grp && !gal_old) {
        const size_t sm = ghl_buf_bytes(9, 18);
        size_t &attr = device_slot((const void *)k_gal_hl<3, 3, 6>);
        if (!attr) {
          attr = 1;
          CK(cudaFuncSetAttribute(k_gal_hl<3, 3, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        }
        if (lc.AP_ngrp)
          k_gal_hl<3, 3, 6><<<lc.AP_ngrp, GAL_NT, sm, c.stream>>>(lc.AP_grp, lc.AP_cps, lc.AP_pptr, lc.AP_hitw,
                                                                   lc.AP_pa, lc.AP_pb, L.A.val, L.P.val, L.AP.val);
        after_launch(c, "k_gal_hl");
      } else {
        LAUNCH((k_spgemm_dense<3, 3, 6>), L.AP.nnzb, L.AP.nnzb, lc.AP_rowof, L.A.ptr, L.A.col, L.A.val, L.P.ptr,
               L.P.val, lc.AP_off, L.AP.val);
      }
      if (lc.G_grp && !gal_old) {
        constexpr size_t sm = (size_t)RAP_NS * RAP2_STAGE_B;
        size_t &attr = device_slot((const void *)k_gal_rap2);
        if (!attr) {
          attr = 1;
          CK(cudaFuncSetAttribute(k_gal_rap2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        }
        if (lc.G_ngrp)
          k_gal_rap2<<<lc.G_ngrp, RAP2_CONS + 32, sm, c.stream>>>(lc.G_grp, lc.G_gofs, L.R.ptr, lc.G_rbi, L.R.val,
                                                                  L.AP.val, lc.G_offg, lc.G.val);
        after_launch(c, "k_gal_rap2");
      } else {
        LAUNCH((k_spgemm_dense<6, 3, 6>), lc.G.nnzb, lc.G.nnzb, lc.G_rowof, L.R.ptr, L.R.col, L.R.val, L.AP.ptr,
               L.AP.val, lc.G_off, lc.G.val);
      }
    } else {
    // measured at cfg 3: thread per output block for the fine 3x3 * 3x6 product (3.0 vs 5.0 ms), warp per
    // output block for the 6-row products (2.6 vs 2.7 ms, 1.1 vs 1.7 ms)
    if (L.b == 3)
      LAUNCH((k_spgemm_vals_pairs<3, 3, 6>), L.AP.nnzb, L.AP.nnzb, lc.AP_pptr, lc.AP_pa, lc.AP_pb, L.A.val, L.P.val,
             L.AP.val);
    else if (L.AP.nnzb >= 65536)  // measured at cfg 3 level 1: 458 -> 370 us; the long-list R*AP and the small
                                  // levels keep the warp form (R*AP 425 vs 958 us, level 2 61 vs 132 us)
      LAUNCH(k_spgemm_vals_half6, L.AP.nnzb * 2, L.AP.nnzb, lc.AP_pptr, lc.AP_pa, lc.AP_pb, L.A.val, L.P.val,
             L.AP.val);
    else
      LAUNCH((k_spgemm_vals_warp<6, 6, 6>), L.AP.nnzb * 32, L.AP.nnzb, lc.AP_pptr, lc.AP_pa, lc.AP_pb, L.A.val,
             L.P.val, L.AP.val);
    auto kg = (L.b == 3) ? k_spgemm_vals_warp<6, 3, 6> : k_spgemm_vals_warp<6, 6, 6>;
    LAUNCH(kg, lc.G.nnzb * 32, lc.G.nnzb, lc.G_pptr, lc.G_pa, lc.G_pb, L.R.val, L.AP.val, lc.G.val);
    }
  }
  if (l == 0 && c.fork_at == 3) fork_filter(c);
  if (!lc.G_kt) {  // symbolic, once
    lc.G_kt = c.alloc<int>(std::max<long>(lc.G.nnzb, 1));
    LAUNCH(k_sym_partner, lc.G.nnzb, lc.G.nnzb, lc.G_rowof, lc.G.ptr, lc.G.col, lc.G_kt, c.err);
  }
  LAUNCH(k_sym2, lc.G.nnzb * 36, lc.G.nnzb * 36, lc.G_kt, lc.G.val, Lc.A.val);
  LAUNCH(k_diag, (long)Lc.nodes * Lc.b, Lc.nodes, Lc.b, Lc.A.ptr, Lc.A.col, Lc.A.val, Lc.dl1, Lc.dpt);
  smoother_data(c, Lc);
}

static void coarsest_numeric(Ctx &c) {
  Level &L = c.lev[c.nlev - 1];
  const int n = c.nco, bw = n - 1, W = band_stride(bw);
  CK(cudaMemsetAsync(c.Lc_row - (size_t)BAND_PAD_ROWS * W, 0, (size_t)(n + 2 * BAND_PAD_ROWS) * W * sizeof(double),
                     c.stream));
  LAUNCH(k_dense_band, (long)L.nodes * L.b, L.nodes, L.b, L.A.ptr, L.A.col, L.A.val, n, W, c.Lc_row);
  band_factor(c, n, bw, c.Lc_row, c.Lc_col, c.Lc_rev, c.Lc_dinv, 2);
}

// per-context arrays needed by the numeric re-setup (owned by Ctx::setup_cache)
struct Caches {
  SetupCache s;
  LevelCache lc[MAXLEV];
  long thin_nnz = 0;
};
static Caches &caches(Ctx &c) {
  if (!c.setup_cache) c.setup_cache = new Caches();
  return *static_cast<Caches *>(c.setup_cache);
}
void drop_caches(Ctx &c) {
  delete static_cast<Caches *>(c.setup_cache);
  c.setup_cache = nullptr;
}

// Thin second-residual structure S[:, Z] (reading R11) and the compact Z rows of S (k_resid_dofs); needs the
// level-0 operator, pos (Z positions) and the elimination-order maps of nd_symbolic.
void build_thin(Ctx &c) {
  Caches &C = caches(c);
  Level &L0 = c.lev[0];
  const long n = c.n;
  // thin structure
  int *cnt = c.alloc<int>(n + 1), *off = c.alloc<int>(n + 1), *flag = c.alloc<int>(n + 1), *foff = c.alloc<int>(n + 1);
  CK(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), c.stream));
  CK(cudaMemsetAsync(flag, 0, (n + 1) * sizeof(int), c.stream));
  LAUNCH(k_thin_count, n, n, L0.A.ptr, L0.A.col, c.pos, cnt);
  long tnnz = scan_ex(c, cnt, off, n);
  LAUNCH(k_flag_nonzero, n, n, cnt, flag);
  c.nthin = (int)scan_ex(c, flag, foff, n);
  c.thin_row = c.alloc<int>(c.nthin);
  c.thin_ptr = c.alloc<int>(c.nthin + 1);
  c.thin_pos = c.alloc<int>(tnnz);
  c.thin_src = c.alloc<int>(tnnz);
  c.thin_val = c.alloc<double>(tnnz);
  LAUNCH(k_thin_fill, n, n, L0.A.ptr, L0.A.col, c.pos, off, foff, c.thin_row, c.thin_ptr, c.thin_pos, c.thin_src);
  // thin entries address y in elimination (pi) order; with P = J^T they address w = J^T y in Z order
  if (c.cfg.filter_basis != 1) nd_remap_positions(c, c.thin_pos, tnnz);
  int tn = (int)tnnz;
  CK(cudaMemcpyAsync(c.thin_ptr + c.nthin, &tn, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  C.thin_nnz = tnnz;
  // compact fine rows of the filter dofs (elimination order) for the Z-row residual
  {
    int *zc = c.alloc<int>(c.nc + 1);
    CK(cudaMemsetAsync(zc, 0, (c.nc + 1) * sizeof(int), c.stream));
    LAUNCH(k_zr_count, c.nc, c.nc, c.dof, L0.A.ptr, zc);
    c.zr_ptr = c.alloc<int>(c.nc + 1);
    c.zr_nnz = scan_ex(c, zc, c.zr_ptr, c.nc);
    c.release(zc);
    c.zr_col = c.alloc<int>(c.zr_nnz);
    c.zr_src = c.alloc<int>(c.zr_nnz);
    c.zr_val = c.alloc<double>(c.zr_nnz * 3);
    LAUNCH(k_zr_fill, c.nc, c.nc, c.dof, L0.A.ptr, L0.A.col, c.zr_ptr, c.zr_col, c.zr_src);
  }
  thin_numeric(c, tnnz);
  c.release(cnt); c.release(off); c.release(flag); c.release(foff);
}

// Solve workspaces of every level and of the PCG (and the level-0 SELL of a one-level hierarchy).
void alloc_workspaces(Ctx &c) {
  Level &L0 = c.lev[0];
  const long n = c.n;
  for (int q = 0; q < c.nlev; q++) {
    Level &L = c.lev[q];
    L.x = c.alloc<double>(L.n);
    L.x2 = c.alloc<double>(L.n);
    L.bv = c.alloc<double>(L.n);
    L.r = c.alloc<double>(L.n);
    if (c.cfg.smoother == 1) L.dir = c.alloc<double>(L.n);
  }
  if (c.nlev == 1) build_sell(c, L0.A, L0.As, true, false);
  c.w_x1 = c.alloc<double>(n);
  c.w_r1 = c.alloc<double>(n);
  c.w_xv = c.alloc<double>(n);
  c.p = c.alloc<double>(n);
  c.q = c.alloc<double>(n);
  c.rr = c.alloc<double>(n);
  c.zz = c.alloc<double>(n);
  c.xx = c.alloc<double>(n);
  c.bb = c.alloc<double>(n);
}

// Level-0 restriction values regrouped for k_restrict (Bsr::ival).
void r_interleave(Ctx &c, Bsr &R) {
  if (!R.ival) R.ival = c.alloc<double>((size_t)R.nnzb * R.br * R.bc);
  LAUNCH(k_interleave_rows, (long)R.nbr * 32, R.nbr, R.ptr, R.br * R.bc, R.val, R.ival);
}

// Structural lower band width of A_w in Z order: max_a (a - min{b <= a : S[Z_a, Z_b] stored}).
int band_width(Ctx &c) {
  Level &L0 = c.lev[0];
  int *bwd = c.alloc<int>(1);
  CK(cudaMemsetAsync(bwd, 0, sizeof(int), c.stream));
  LAUNCH(k_band_start, c.nc, c.nc, c.Z, c.pos, L0.A.ptr, L0.A.col, bwd);
  const int bw = d2h1(c, bwd);
  c.release(bwd);
  return bw;
}

// Coarsest dense factor storage (band of width nco - 1).
void coarsest_alloc(Ctx &c) { band_alloc(c, c.nco, c.nco - 1, c.Lc_row, c.Lc_col, c.Lc_rev, c.Lc_dinv); }

// =================================================================== setup_all
void setup_all(Ctx &c, const int *K_ptr, const int *K_col, const double *K_val, const int *J_ptr, const int *J_col,
               const double *J_val, const double *D, const int *Zin, int nc_in, const double *B_nns) {
  Caches &C = caches(c);
  const int nodes = c.nodes;
  const long n = c.n;
  const int m = c.m;
  // AMGF_SETUP_TIMING (diagnostic): wall time of every setup phase, stream synchronised at the boundaries
  static const bool ph_on = getenv("AMGF_SETUP_TIMING") != nullptr;
  auto ph_t0 = std::chrono::steady_clock::now();
  auto ph = [&](const char *name, int lev = -1) {
    if (!ph_on) return;
    cudaStreamSynchronize(c.stream);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "setup phase %-28s level %2d %8.2f ms\n", name, lev,
            std::chrono::duration<double, std::milli>(t1 - ph_t0).count());
    ph_t0 = t1;
  };
  // ---- copy inputs
  int nnzbK = 0, nnzJ = 0;
  CK(cudaMemcpyAsync(&nnzbK, K_ptr + nodes, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  if (m > 0) CK(cudaMemcpyAsync(&nnzJ, J_ptr + m, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  REQUIRE(nnzbK > 0, AMGF_ERR_ARG, "K has no blocks");
  c.nnzJ = nnzJ;
  bsr_alloc(c, c.K, nodes, nodes, 3, 3, nnzbK);
  d2d(c, c.K.ptr, K_ptr, nodes + 1);
  d2d(c, c.K.col, K_col, nnzbK);
  d2d(c, c.K.val, K_val, (size_t)nnzbK * 9);
  c.J_ptr = c.alloc<int>(m + 1);
  c.J_col = c.alloc<int>(nnzJ);
  c.J_val = c.alloc<double>(nnzJ);
  c.D = c.alloc<double>(m);
  if (m > 0) {
    d2d(c, c.J_ptr, J_ptr, m + 1);
    d2d(c, c.J_col, J_col, nnzJ);
    d2d(c, c.J_val, J_val, nnzJ);
    d2d(c, c.D, D, m);
  } else {
    CK(cudaMemsetAsync(c.J_ptr, 0, sizeof(int), c.stream));
  }
  LAUNCH(k_check_finite, (long)nnzbK * 9, (long)nnzbK * 9, c.K.val, c.err, DERR_NONFINITE);
  LAUNCH(k_check_finite, nnzJ, nnzJ, c.J_val, c.err, DERR_NONFINITE);
  LAUNCH(k_check_finite, m, m, c.D, c.err, DERR_NONFINITE);
  LAUNCH(k_check_pos, m, m, c.D, c.err);
  check_dev_error(c, "input check");

  ph("inputs");
  // ---- J^T
  {
    int *rowJ = c.alloc<int>(nnzJ), *keys = c.alloc<int>(nnzJ), *idx = c.alloc<int>(nnzJ), *perm = c.alloc<int>(nnzJ);
    LAUNCH(k_rowof, m, m, c.J_ptr, rowJ);
    LAUNCH(k_iota, nnzJ, nnzJ, idx);
    sort_pairs(c, c.J_col, keys, idx, perm, nnzJ);
    int *cnt = c.alloc<int>(n + 1);
    CK(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), c.stream));
    LAUNCH(k_count_keys, nnzJ, nnzJ, c.J_col, cnt);
    c.Jt_ptr = c.alloc<int>(n + 1);
    scan_ex(c, cnt, c.Jt_ptr, n);
    c.Jt_row = c.alloc<int>(nnzJ);
    c.Jt_val = c.alloc<double>(nnzJ);
    // Jt_row[t] = rowJ[perm[t]], Jt_val[t] = J_val[perm[t]]
    LAUNCH(k_gather_int, nnzJ, nnzJ, perm, rowJ, c.Jt_row);
    LAUNCH(k_gather_vals, nnzJ, nnzJ, perm, c.J_val, c.Jt_val);
    c.release(rowJ); c.release(keys); c.release(idx); c.release(perm); c.release(cnt);
  }

  ph("J^T");
  // ---- s1: S pattern and values
  Level &L0 = c.lev[0];
  L0.b = 3; L0.nodes = nodes; L0.n = n;
  {
    int *cnt = c.alloc<int>(nodes + 1);
    CK(cudaMemsetAsync(cnt, 0, (nodes + 1) * sizeof(int), c.stream));
    LAUNCH(k_S_count, nodes, nodes, c.K.ptr, c.K.col, c.Jt_ptr, c.Jt_row, c.J_ptr, c.J_col, cnt, c.err);
    check_dev_error(c, "S pattern");
    L0.A.ptr = c.alloc<int>(nodes + 1);
    long nnzb = scan_ex(c, cnt, L0.A.ptr, nodes);
    c.release(cnt);
    L0.A.nbr = L0.A.nbc = nodes; L0.A.br = L0.A.bc = 3; L0.A.nnzb = nnzb;
    L0.A.col = c.alloc<int>(nnzb);
    L0.A.val = c.alloc<double>(nnzb * 9);
    c.S_kblk = c.alloc<int>(nnzb);
    LAUNCH(k_S_fill, nodes, nodes, c.K.ptr, c.K.col, c.Jt_ptr, c.Jt_row, c.J_ptr, c.J_col, L0.A.ptr, L0.A.col,
           c.S_kblk, c.err);
    C.s.S_rowof = rowof(c, L0.A);
    S_numeric(c, C.s.S_rowof);
  }

  ph("S pattern + values");
  // ---- s2: I_c, Z
  {
    int *mark = c.alloc<int>(n + 1);
    CK(cudaMemsetAsync(mark, 0, (n + 1) * sizeof(int), c.stream));
    LAUNCH(k_mark_cols, nnzJ, nnzJ, c.J_col, mark);
    c.pos = c.alloc<int>(n);
    CK(cudaMemsetAsync(c.pos, 0xff, n * sizeof(int), c.stream));
    int *off = c.alloc<int>(n + 1);
    long nmark = scan_ex(c, mark, off, n);
    if (Zin) {
      c.nc = nc_in;
      c.Z = c.alloc<int>(c.nc);
      d2d(c, c.Z, Zin, c.nc);
      int *cov = c.alloc<int>(1);
      CK(cudaMemsetAsync(cov, 0, sizeof(int), c.stream));
      LAUNCH(k_check_Z, c.nc, c.nc, n, c.Z, mark, c.pos, cov, c.err);
      check_dev_error(c, "Z has an out-of-range or duplicate dof");
      const int covered = d2h1(c, cov);
      c.release(cov);
      REQUIRE(covered == nmark, AMGF_ERR_ARG, "Z does not contain every column of J (" + std::to_string(covered) +
                                                  " of " + std::to_string(nmark) + ")");
    } else {
      c.nc = (int)nmark;
      c.Z = c.alloc<int>(c.nc);
      LAUNCH(k_compact_Z, n, n, mark, off, c.Z, c.pos);
    }
    c.release(mark);
    c.release(off);
  }

  ph("I_c");
  // ---- s3: A_w band, factor, thin residual
  if (c.nc > 0) {
    if (c.cfg.filter_basis == 1) {  // P = J^T (reading R21): the filter space is the m constraints
      REQUIRE(c.m > 0, AMGF_ERR_ARG, "filter_basis 1 needs constraints");
      c.nf = c.m;
      c.bw = band_width_J(c);
      c.fJv = c.alloc<double>(c.m);
      c.fJw = c.alloc<double>(c.nc);
    } else {
      c.nf = c.nc;
      c.bw = band_width(c);
    }
    ph("band width");
    nd_symbolic(c);
    ph("A_w symbolic (nd)");
    filter_numeric(c);
    check_dev_error(c, "A_w Cholesky");
    ph("A_w factor");
    build_thin(c);
  }

  ph("thin / Z rows");
  // ---- hierarchy
  L0.Bnn = c.alloc<double>(n * 6);
  d2d(c, L0.Bnn, B_nns, (size_t)n * 6);
  L0.dl1 = c.alloc<double>(n);
  L0.dpt = c.alloc<double>(n);
  LAUNCH(k_diag, n, nodes, 3, L0.A.ptr, L0.A.col, L0.A.val, L0.dl1, L0.dpt);
  smoother_data(c, L0);
  // level-0 components of K's block graph
  L0.comp = c.alloc<int>(nodes);
  {
    LAUNCH(k_iota, nodes, nodes, L0.comp);
    int *chg = c.alloc<int>(1);
    for (int it = 0; it < 100000; it++) {
      CK(cudaMemsetAsync(chg, 0, sizeof(int), c.stream));
      LAUNCH(k_cc_step, nodes, nodes, c.K.ptr, c.K.col, L0.comp, chg);
      if (d2h1(c, chg) == 0) break;
    }
    c.release(chg);
  }
  ph("diag + components");
  int l = 0;
  for (;;) {
    Level &L = c.lev[l];
    if (L.n <= c.cfg.coarsest_size || l + 1 >= c.cfg.max_levels || l + 1 >= MAXLEV) break;
    const int nn = L.nodes;
    // ---- s4 aggregation
    int *state = c.alloc<int>(nn), *m1 = c.alloc<int>(nn), *m2 = c.alloc<int>(nn), *und = c.alloc<int>(1);
    LAUNCH(k_mis_init, nn, nn, L.A.ptr, L.A.col, L.comp, state);
    for (int round = 0; round < 10000; round++) {
      LAUNCH(k_mis_max, nn, nn, L.A.ptr, L.A.col, L.comp, state, (const int *)nullptr, m1, c.cfg.agg_seed);
      LAUNCH(k_mis_max, nn, nn, L.A.ptr, L.A.col, L.comp, state, (const int *)m1, m2, c.cfg.agg_seed);
      LAUNCH(k_mis_roots, nn, nn, m2, state);
      LAUNCH(k_mis_near, nn, nn, L.A.ptr, L.A.col, L.comp, state, (const int *)nullptr, m1);
      LAUNCH(k_mis_near, nn, nn, L.A.ptr, L.A.col, L.comp, state, (const int *)m1, m2);
      CK(cudaMemsetAsync(und, 0, sizeof(int), c.stream));
      LAUNCH(k_mis_block, nn, nn, m2, state, und);
      if (d2h1(c, und) == 0) break;
    }
    int *flag = c.alloc<int>(nn + 1), *rank = c.alloc<int>(nn + 1);
    CK(cudaMemsetAsync(flag, 0, (nn + 1) * sizeof(int), c.stream));
    LAUNCH(k_root_flag, nn, nn, state, flag);
    const int na = (int)scan_ex(c, flag, rank, nn);
    L.root = flag;
    if (na == 0 || 60L * na > 9L * L.n) {
      c.release(state); c.release(m1); c.release(m2); c.release(und); c.release(rank);
      break;
    }
    L.n_agg = na;
    L.agg = c.alloc<int>(nn);
    LAUNCH(k_agg_phase3, nn, nn, L.A.ptr, L.A.col, L.comp, state, rank, m1);
    LAUNCH(k_agg_leftover, nn, nn, L.A.ptr, L.A.col, L.comp, state, m1, L.agg, c.err);
    check_dev_error(c, "aggregation");
    Level &Lc = c.lev[l + 1];
    Lc.b = 6; Lc.nodes = na; Lc.n = 6L * na;
    Lc.comp = c.alloc<int>(na);
    LAUNCH(k_coarse_comp, nn, nn, state, rank, L.comp, Lc.comp);
    ph("aggregation", l);
    // ---- s5 tentative prolongator
    {
      int *key = c.alloc<int>(nn), *keys = c.alloc<int>(nn), *idx = c.alloc<int>(nn);
      LAUNCH(k_agg_key, nn, nn, L.agg, key);
      LAUNCH(k_iota, nn, nn, idx);
      L.agg_nodes = c.alloc<int>(nn);
      sort_pairs(c, key, keys, idx, L.agg_nodes, nn);
      int *cnt = c.alloc<int>(na + 1);
      CK(cudaMemsetAsync(cnt, 0, (na + 1) * sizeof(int), c.stream));
      // counts per aggregate
      int *aggd = c.alloc<int>(nn);
      LAUNCH(k_agg_key, nn, nn, L.agg, aggd);
      LAUNCH(k_count_valid, nn, nn, aggd, na, cnt);
      L.agg_ptr = c.alloc<int>(na + 1);
      scan_ex(c, cnt, L.agg_ptr, na);
      int *isagg = c.alloc<int>(nn + 1);
      CK(cudaMemsetAsync(isagg, 0, (nn + 1) * sizeof(int), c.stream));
      LAUNCH(k_is_agg, nn, nn, L.agg, isagg);
      L.Pt.ptr = c.alloc<int>(nn + 1);
      long nzt = scan_ex(c, isagg, L.Pt.ptr, nn);
      L.Pt.nbr = nn; L.Pt.nbc = na; L.Pt.br = L.b; L.Pt.bc = 6; L.Pt.nnzb = nzt;
      L.Pt.col = c.alloc<int>(nzt);
      L.Pt.val = c.alloc<double>(nzt * L.b * 6);
      LAUNCH(k_Pt_cols, nn, nn, L.agg, L.Pt.ptr, L.Pt.col);
      Lc.Bnn = c.alloc<double>((long)na * 36);
      LAUNCH(k_qr, na, na, L.b, L.agg_ptr, L.agg_nodes, L.Pt.ptr, L.Bnn, L.Pt.val, Lc.Bnn, c.err);
      check_dev_error(c, "tentative prolongator");
      c.release(key); c.release(keys); c.release(idx); c.release(cnt); c.release(aggd); c.release(isagg);
    }
    c.release(state); c.release(m1); c.release(m2); c.release(und); c.release(rank);
    LevelCache &lc = C.lc[l];
    ph("tentative P", l);
    // ---- s6 smoothed prolongator pattern
    {
      int *cnt = c.alloc<int>(nn + 1);
      CK(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int), c.stream));
      LAUNCH(k_P_count, nn, nn, L.A.ptr, L.A.col, L.agg, cnt, c.err);
      check_dev_error(c, "prolongator pattern");
      L.P.ptr = c.alloc<int>(nn + 1);
      long nzp = scan_ex(c, cnt, L.P.ptr, nn);
      c.release(cnt);
      L.P.nbr = nn; L.P.nbc = na; L.P.br = L.b; L.P.bc = 6; L.P.nnzb = nzp;
      L.P.col = c.alloc<int>(nzp);
      L.P.val = c.alloc<double>(nzp * L.b * 6);
      LAUNCH(k_P_fill, nn, nn, L.A.ptr, L.A.col, L.agg, L.P.ptr, L.P.col);
      lc.P_rowof = rowof(c, L.P);
    }
    ph("P pattern", l);
    // ---- s7 R = P^T pattern
    {
      const long nzp = L.P.nnzb;
      int *keys = c.alloc<int>(nzp), *idx = c.alloc<int>(nzp);
      lc.R_perm = c.alloc<int>(nzp);
      LAUNCH(k_iota, nzp, nzp, idx);
      sort_pairs(c, L.P.col, keys, idx, lc.R_perm, nzp);
      int *cnt = c.alloc<int>(na + 1);
      CK(cudaMemsetAsync(cnt, 0, (na + 1) * sizeof(int), c.stream));
      LAUNCH(k_count_keys, nzp, nzp, L.P.col, cnt);
      L.R.nbr = na; L.R.nbc = nn; L.R.br = 6; L.R.bc = L.b; L.R.nnzb = nzp;
      L.R.ptr = c.alloc<int>(na + 1);
      scan_ex(c, cnt, L.R.ptr, na);
      L.R.col = c.alloc<int>(nzp);
      L.R.val = c.alloc<double>(nzp * 6 * L.b);
      LAUNCH(k_gather_int, nzp, nzp, lc.R_perm, lc.P_rowof, L.R.col);
      c.release(keys); c.release(idx); c.release(cnt);
    }
    ph("R pattern", l);
    // ---- AP and G patterns
    {
      int *cnt = c.alloc<int>(nn + 1);
      CK(cudaMemsetAsync(cnt, 0, (nn + 1) * sizeof(int), c.stream));
      LAUNCH(k_spgemm_count, nn, nn, L.A.ptr, L.A.col, L.P.ptr, L.P.col, cnt, c.err);
      check_dev_error(c, "A*P pattern");
      L.AP.ptr = c.alloc<int>(nn + 1);
      long nz = scan_ex(c, cnt, L.AP.ptr, nn);
      c.release(cnt);
      L.AP.nbr = nn; L.AP.nbc = na; L.AP.br = L.b; L.AP.bc = 6; L.AP.nnzb = nz;
      L.AP.col = c.alloc<int>(nz);
      L.AP.val = c.alloc<double>(nz * L.b * 6);
      LAUNCH(k_spgemm_fill, nn, nn, L.A.ptr, L.A.col, L.P.ptr, L.P.col, L.AP.ptr, L.AP.col);
      lc.AP_rowof = rowof(c, L.AP);
      int *cg = c.alloc<int>(na + 1);
      CK(cudaMemsetAsync(cg, 0, (na + 1) * sizeof(int), c.stream));
      LAUNCH(k_spgemm_count, na, na, L.R.ptr, L.R.col, L.AP.ptr, L.AP.col, cg, c.err);
      check_dev_error(c, "R*AP pattern");
      lc.G.ptr = c.alloc<int>(na + 1);
      long nzg = scan_ex(c, cg, lc.G.ptr, na);
      c.release(cg);
      lc.G.nbr = na; lc.G.nbc = na; lc.G.br = 6; lc.G.bc = 6; lc.G.nnzb = nzg;
      lc.G.col = c.alloc<int>(nzg);
      lc.G.val = c.alloc<double>(nzg * 36);
      LAUNCH(k_spgemm_fill, na, na, L.R.ptr, L.R.col, L.AP.ptr, L.AP.col, lc.G.ptr, lc.G.col);
      lc.G_rowof = rowof(c, lc.G);
      // coarse operator shares G's pattern
      Lc.A.nbr = Lc.A.nbc = na; Lc.A.br = Lc.A.bc = 6; Lc.A.nnzb = nzg;
      Lc.A.ptr = lc.G.ptr; Lc.A.col = lc.G.col;
      Lc.A.val = c.alloc<double>(nzg * 36);
      Lc.dl1 = c.alloc<double>(Lc.n);
      Lc.dpt = c.alloc<double>(Lc.n);
    }
    ph("AP / G patterns", l);
    // coarse levels: one thread per scalar row (1 x 6).  Rows sorted by length (less slot padding) on the
    // large levels: the fine operator keeps its order (the PCG dot partials and the Z-row residual read
    // it by row), small levels may become the fused tail (tail.cu), which needs the natural order
    const bool sort_level = l > 0 && L.n > 16384;
    build_sell(c, L.A, L.As, true, l > 0, sort_level);
    ph("SELL of A", l);
    build_pairs(c, L.AP.nnzb, lc.AP_rowof, L.AP.col, L.A, L.P, lc.AP_pptr, lc.AP_pa, lc.AP_pb);
    build_pairs(c, lc.G.nnzb, lc.G_rowof, lc.G.col, L.R, L.AP, lc.G_pptr, lc.G_pa, lc.G_pb);
    ph("product pair lists", l);
    if (L.b == 3) {  // fine level: dense-over-row products (k_spgemm_dense)
      lc.AP_off = build_off(c, L.AP.nnzb, lc.AP_rowof, L.AP.col, L.A, L.P);
      lc.G_off = build_off(c, lc.G.nnzb, lc.G_rowof, lc.G.col, L.R, L.AP);
      ph("offset tables", l);
      build_gal_groups(c, L.A, L.P, L.AP, lc.AP_pptr, lc.AP_pa, lc.AP_pb, lc.AP_grp, lc.AP_ngrp, lc.AP_cps,
                       lc.AP_hitw);
      ph("A*P groups", l);
      build_rap_groups(c, lc.G, L.R, L.AP, lc.G_grp, lc.G_ngrp, lc.G_gofs, lc.G_offg, lc.G_rbi);

    }
    ph("R*AP groups", l);
    level_numeric(c, l, lc);
    check_dev_error(c, "Galerkin product");
    ph("level numeric", l);
    build_sell(c, L.P, L.Ps, true, l > 0, l == 0 || sort_level);  // prolongators: rows sorted by length
    ph("SELL of P", l);
    l++;
  }
  c.nlev = l + 1;
  // ---- s9 coarsest
  {
    Level &L = c.lev[c.nlev - 1];
    REQUIRE(L.n <= 16384, AMGF_ERR_LIMIT, "coarsest level too large for a dense factor (" + std::to_string(L.n) + ")");
    c.nco = (int)L.n;
    coarsest_alloc(c);
    coarsest_numeric(c);
    check_dev_error(c, "coarsest Cholesky");
  }
  ph("coarsest");
  alloc_workspaces(c);
  CK(cudaStreamSynchronize(c.stream));
  read_level_scalars(c);
  tail_plan(c);
  ph("workspaces + tail plan");
}

// =================================================================== numeric re-setup (new D)
void setup_numeric(Ctx &c, const double *D, const double *D_lo, const double *D_up) {
  Caches &C = caches(c);
  timeline_begin(c);
  setup_mark(c, 0, c.stream);
  d2d(c, c.D, D, c.m);
  LAUNCH(k_check_finite, c.m, c.m, c.D, c.err, DERR_NONFINITE);
  LAUNCH(k_check_pos, c.m, c.m, c.D, c.err);  // the device error flag keeps the first error: checked at the end
  // bound-constraint diagonals (both or neither; amgf_update_D_box): zero-filled when only one is given
  c.has_box = D_lo || D_up;
  if (c.has_box) {
    if (!c.D_lo) { c.D_lo = c.alloc<double>(c.n); c.D_up = c.alloc<double>(c.n); }
    if (D_lo) d2d(c, c.D_lo, D_lo, c.n); else CK(cudaMemsetAsync(c.D_lo, 0, c.n * sizeof(double), c.stream));
    if (D_up) d2d(c, c.D_up, D_up, c.n); else CK(cudaMemsetAsync(c.D_up, 0, c.n * sizeof(double), c.stream));
    LAUNCH(k_check_finite, c.n, c.n, c.D_lo, c.err, DERR_NONFINITE);
    LAUNCH(k_check_finite, c.n, c.n, c.D_up, c.err, DERR_NONFINITE);
    LAUNCH(k_check_nonneg, c.n, c.n, c.D_lo, c.err);
    LAUNCH(k_check_nonneg, c.n, c.n, c.D_up, c.err);
  }
  Level &L0 = c.lev[0];
  S_numeric(c, C.s.S_rowof);
  setup_mark(c, 1, c.stream);
  // where the A_w factorization forks off (A/B: AMGF_FORK_AT = 0 after S, 1 after the fine power iteration,
  // 2 after the fine P values, 3 after the fine Galerkin products)
  static const int fork_at = getenv("AMGF_FORK_AT") ? atoi(getenv("AMGF_FORK_AT")) : 0;
  c.fork_at = (c.nc > 0) ? fork_at : -1;
  if (c.nc > 0) {
    if (c.fork_at == 0) fork_filter(c);
    thin_numeric(c, C.thin_nnz);
  }
  // the fine SELL copy and the level-0 diagonals in one pass (the fine SELL keeps the natural row order)
  const bool fused_S = L0.As.val && L0.As.br == 3 && !L0.As.perm && L0.As.nrows == L0.nodes;
  // ... and the fine level's first power step (the SELL pass reads every block once anyway)
  const bool pow0 = fused_S && c.nlev >= 2 && c.cfg.power_iters > 0 && c.pw_w && c.pw_part;
  if (fused_S)
    LAUNCH(k_sell_diag, L0.nodes, L0.nodes, L0.A.ptr, L0.A.col, L0.A.val, L0.As.slice_ptr, L0.As.val, L0.dl1, L0.dpt,
           pow0 ? c.pw_w : nullptr, c.dot_part, c.pw_part);
  else
    LAUNCH(k_diag, L0.n, L0.nodes, 3, L0.A.ptr, L0.A.col, L0.A.val, L0.dl1, L0.dpt);
  smoother_data(c, L0);
  for (int l = 0; l + 1 < c.nlev; l++) {
    if (l > 0 || !fused_S) build_sell(c, c.lev[l].A, c.lev[l].As, false, l > 0);
    level_numeric(c, l, C.lc[l], l == 0 && pow0);  // device error flags are checked once, after the join
    build_sell(c, c.lev[l].P, c.lev[l].Ps, false, l > 0);
  }
  if (c.nlev == 1) build_sell(c, L0.A, L0.As, false, false);
  setup_mark(c, 2, c.stream);
  coarsest_numeric(c);
  setup_mark(c, 3, c.stream);
  join_filter(c);
  setup_mark(c, 4, c.stream);
  check_dev_error(c, "numeric setup (Galerkin products / A_w / coarsest Cholesky)");
  read_level_scalars(c);
  auto ms = [&](int a, int b) {
    float v = 0;
    CK(cudaEventElapsedTime(&v, c.ph_ev[a], c.ph_ev[b]));
    return (double)v;
  };
  CK(cudaEventSynchronize(c.ph_ev[4]));
  c.setup_ms[0] = ms(0, 4);                           // total
  c.setup_ms[1] = ms(0, 1);                           // S = K + J^T D J (+ D checks)
  c.setup_ms[2] = ms(1, 2);                           // hierarchy: power iteration, P, Galerkin, SELL refresh
  c.setup_ms[3] = ms(2, 3);                           // coarsest Cholesky
  c.setup_ms[4] = c.nc > 0 ? ms(5, 6) : 0.0;          // A_w factorization (side stream, concurrent)
  timeline_dump(c, c.ph_ev[0]);
  if (getenv("AMGF_SETUP_TIMING"))
    fprintf(stderr, "update_D ms: total %.2f S %.2f hierarchy %.2f coarsest %.2f A_w(side) %.2f\n", c.setup_ms[0],
            c.setup_ms[1], c.setup_ms[2], c.setup_ms[3], c.setup_ms[4]);
}

}  // namespace amgf
