// nd_kernels.cuh -- nested-dissection block table and the separator forward-dot kernel (included by
// filter.cu and by the microbenchmark tools/mb_sepfwd.cu).
#pragma once
#include <stdint.h>

#include "devutil.cuh"

namespace amgf {

struct NdBlk {
  int p0, len, kind;  // kind 0 = leaf, 1 = separator
  int t0;             // separator: first pi position of its subtree
  long off;           // separator: offset of its rows in Loff (row-major: s * rs + (k - t0))
  int level;          // separator depth (root 0)
  int rs;             // separator: row stride of its rows in Loff (p0 - t0 rounded up to even)
};

// Forward, separator rows: acc_s = v_s - sum_{k in [t0, p0)} L_sk w_k (ascending k), into accbuf.
// One warp per group of G rows of a separator (G = 1 in use: a separator's rows stream through as many SMs
// as it has rows); lane l < G owns row row0 + l.  Chunks of KC columns of the G rows (row-major) and the
// matching w values go through an NS-deep cp.async ring; inside a chunk the operands of the next 8 terms
// are loaded (16-byte shared-memory loads) while the current 8 FMAs run.  Measured on the top separator of
// cfg 3 (133 rows x 8,317 columns, tools/mb_sepfwd.cu): 10.7 cycles per term against 8.2 for a bare
// register DFMA chain (the previous 64-column, 4-row form: 16.0).
constexpr int SF_KC = 512;
constexpr size_t sf_smem(int G, int NS, int KC) { return (size_t)NS * (G * (KC + 2) + KC) * sizeof(double); }
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}

template <int G, int NS, int KC>
__global__ void __launch_bounds__(32) k_nd_sep_fwd(const int2 *groups, const NdBlk *blk, const double *Loff,
                                                   const double *r1, const int *dof, const double *w,
                                                   const double *w2, double *accbuf) {
  constexpr int LD = KC + 2;
  extern __shared__ __align__(16) double sfm[];  // [NS][G * LD] rows, then [NS][KC] w
  pdl_launch_dependents();
  const NdBlk S = blk[groups[blockIdx.x].x];
  const int row0 = groups[blockIdx.x].y;
  const int lane = threadIdx.x;
  const int nrow = min(G, S.len - row0);
  const int ncol = S.p0 - S.t0;
  const int nch = (ncol + KC - 1) / KC;
  double *sW = sfm + NS * G * LD;
  const double *wsrc = (S.t0 & 1) ? w2 + S.t0 + 1 : w + S.t0;  // 16-byte aligned view of w[t0 + k]
  const double *Lq = Loff + S.off + (long)row0 * S.rs;
  auto issue_L = [&](int c) {
    if (c < nch) {
      const int k0 = c * KC, st = c % NS;
      for (int p = lane; p < KC / 2; p += 32)
        if (2 * p < ncol - k0) {  // the even row stride covers an odd tail element
          double *dst = sfm + st * G * LD + 2 * p;
          for (int r = 0; r < nrow; r++) cp_async16(dst + r * LD, Lq + (long)r * S.rs + k0 + 2 * p);
        }
    }
  };
  auto issue_w = [&](int c) {
    if (c < nch) {
      const int k0 = c * KC, st = c % NS;
      for (int p = lane; p < KC / 2; p += 32) cp_async16(sW + st * KC + 2 * p, wsrc + k0 + 2 * p);
    }
  };
  auto issue = [&](int c) {
    issue_L(c);
    issue_w(c);
    asm volatile("cp.async.commit_group;");
  };
  // The factor rows of the first NS-1 chunks do not depend on the previous kernel (PDL): they are issued
  // before the wait and land in group 0 with w of chunk 0; groups 1..NS-2 hold w of chunks 1..NS-2.
#pragma unroll
  for (int c = 0; c < NS - 1; c++) issue_L(c);
  pdl_wait();
#pragma unroll
  for (int c = 0; c < NS - 1; c++) {
    issue_w(c);
    asm volatile("cp.async.commit_group;");
  }
  const int prow = S.p0 + row0 + lane;
  double acc = (lane < nrow) ? r1[dof ? dof[prow] : prow] : 0.0;
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
    __syncwarp();  // stage st is refilled by the issue of iteration c + 1
  }
  asm volatile("cp.async.wait_group 0;");
  if (lane < nrow) accbuf[S.p0 + row0 + lane] = acc;
}

}  // namespace amgf
