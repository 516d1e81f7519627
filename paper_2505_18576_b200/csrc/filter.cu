// filter.cu -- the AMGF filter y = A_w^{-1} r1[Z] (Def. AMGF; A_w = P^T S P)
// with A_w factored in a nested-dissection elimination order (R16, contracts C9/C10).
//
// pi = ND(n_c, bw, levels) is a one-dimensional nested dissection of A_w's band (Z order): an interval is a
// leaf or is split by a separator of bw consecutive positions, which decouples its two halves; blocks are
// emitted in postorder.  The oracle factors the dense A_w[pi,pi]; here the factor is stored by structure:
//   - in-block entries (leaf rows within the band, separator rows inside their separator): band arrays
//     over pi positions (Lrow / Lcol / Lrev, stride band_stride(bw)), zero across blocks;
//   - separator rows against their subtree (dense by fill): Loff, row-major per separator
//     (Loff[off + s * rs + (k - t0)] = L_{p0+s, k}, rs = p0 - t0 rounded up to even).
// Every entry keeps the contract's chain (ascending k for the factor and the forward solve, descending k for
// the backward solve); terms skipped here are exact zeros of the dense factor.  Parallelism: leaves are
// independent (one CTA / warp each); separators of one level are independent.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "devutil.cuh"
#include "nd_kernels.cuh"

namespace amgf {


namespace {

struct Node {
  int z0, z1;  // Z interval
  bool leaf;
  int left = -1, right = -1;
  int depth;
};

// Same recursion as orc_nd_order (oracle/amgf_oracle.c): leaf if depth == 0 or b - a < 4 bw + 64.
int build(std::vector<Node> &nodes, int a, int b, int depth, int bw, int d) {
  Node nd;
  nd.z0 = a; nd.z1 = b; nd.depth = d;
  if (depth == 0 || b - a < 4 * bw + 64) {
    nd.leaf = true;
    nodes.push_back(nd);
    return (int)nodes.size() - 1;
  }
  nd.leaf = false;
  const int m = a + (b - a - bw) / 2;
  nodes.push_back(nd);
  const int id = (int)nodes.size() - 1;
  const int l = build(nodes, a, m, depth - 1, bw, d + 1);
  const int r = build(nodes, m + bw, b, depth - 1, bw, d + 1);
  nodes[id].left = l;
  nodes[id].right = r;
  nodes[id].z0 = m;  // separator interval [m, m + bw)
  nodes[id].z1 = m + bw;
  return id;
}

struct Emit {
  std::vector<NdBlk> blk;
  std::vector<int> pi;  // pi position -> Z position
  std::vector<std::vector<int>> sub_leaves, sub_seps;  // per block (separators): blocks in its subtree
};

// postorder emission; returns (first block id, subtree start pi)
int emit(const std::vector<Node> &nodes, int id, Emit &E, std::vector<int> &leaves, std::vector<int> &seps) {
  const Node &nd = nodes[id];
  if (nd.leaf) {
    NdBlk b{(int)E.pi.size(), nd.z1 - nd.z0, 0, (int)E.pi.size(), 0, nd.depth, 0};
    for (int z = nd.z0; z < nd.z1; z++) E.pi.push_back(z);
    E.blk.push_back(b);
    E.sub_leaves.emplace_back();
    E.sub_seps.emplace_back();
    leaves.push_back((int)E.blk.size() - 1);
    return b.t0;
  }
  std::vector<int> ll, ls, rl, rs;
  const int t0 = emit(nodes, nd.left, E, ll, ls);
  emit(nodes, nd.right, E, rl, rs);
  NdBlk b{(int)E.pi.size(), nd.z1 - nd.z0, 1, t0, 0, nd.depth, 0};
  for (int z = nd.z0; z < nd.z1; z++) E.pi.push_back(z);
  E.blk.push_back(b);
  std::vector<int> sl = ll, ss = ls;  // subtree blocks in pi order: left subtree, then right subtree
  sl.insert(sl.end(), rl.begin(), rl.end());
  ss.insert(ss.end(), rs.begin(), rs.end());
  E.sub_leaves.push_back(sl);
  E.sub_seps.push_back(ss);
  leaves.insert(leaves.end(), sl.begin(), sl.end());
  seps.insert(seps.end(), ss.begin(), ss.end());
  seps.push_back((int)E.blk.size() - 1);
  return t0;
}

template <class T>
T *upload(Ctx &c, const std::vector<T> &v) {
  T *d = c.alloc<T>(v.size());
  if (!v.empty()) CK(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c.stream));
  return d;
}

}  // namespace

// ------------------------------------------------------------------ kernels
// acc - sum_{t < n} a[t*sa] * b[t*sb] as one fma chain in ascending t (contract order), with the loads of
// the next 8 terms in flight while the current 8 are consumed (register double buffer).
__device__ __forceinline__ double chain_sub(double acc, const double *__restrict__ a, long sa,
                                            const double *__restrict__ b, long sb, int n) {
  int t = 0;
  double ra[8], rb[8];
  if (n >= 8) {
#pragma unroll
    for (int u = 0; u < 8; u++) { ra[u] = a[u * sa]; rb[u] = b[u * sb]; }
    for (; t + 16 <= n; t += 8) {
      double na[8], nb[8];
#pragma unroll
      for (int u = 0; u < 8; u++) { na[u] = a[(t + 8 + u) * sa]; nb[u] = b[(t + 8 + u) * sb]; }
#pragma unroll
      for (int u = 0; u < 8; u++) acc = __fma_rn(-ra[u], rb[u], acc);
#pragma unroll
      for (int u = 0; u < 8; u++) { ra[u] = na[u]; rb[u] = nb[u]; }
    }
#pragma unroll
    for (int u = 0; u < 8; u++) acc = __fma_rn(-ra[u], rb[u], acc);
    t += 8;
  }
  for (; t < n; t++) acc = __fma_rn(-a[t * sa], b[t * sb], acc);
  return acc;
}

__global__ void k_nd_maps(int nc, const int *pi_z, const int *Z, int *zpi, int *dof) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  zpi[pi_z[p]] = p;
  dof[p] = Z[pi_z[p]];
}
__global__ void k_nd_block_of(int nblk, const NdBlk *blk, int *block_of) {
  int b = blockIdx.x;
  if (b >= nblk) return;
  for (int t = threadIdx.x; t < blk[b].len; t += blockDim.x) block_of[blk[b].p0 + t] = b;
}
__global__ void k_remap(long n, const int *zpi, int *pos) {
  long e = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (e < n) pos[e] = zpi[pos[e]];
}

// A_w[pi,pi] entries of S: in-block lower entries into the band, separator-vs-subtree entries into Loff.
__global__ void k_nd_fill(int nc, int bw, int W, const NdBlk *blk, const int *block_of, const int *dof,
                          const int *pos, const int *zpi, const int *S_ptr, const int *S_col, const double *S_val,
                          double *Lrow, double *Loff) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nc) return;
  const NdBlk B = blk[block_of[p]];
  const int d = dof[p], I = d / 3, r = d % 3;
  for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
    for (int cc = 0; cc < 3; cc++) {
      const int zq = pos[3 * S_col[k] + cc];
      if (zq < 0) continue;
      const int q = zpi[zq];
      const double v = S_val[(long)k * 9 + 3 * r + cc];
      if (q >= B.p0 && q <= p) Lrow[(long)p * W + bw - (p - q)] = v;
      else if (B.kind == 1 && q >= B.t0 && q < B.p0) Loff[B.off + (long)(p - B.p0) * B.rs + (q - B.t0)] = v;
    }
}

// Filter basis P = J^T (variant f4, reading R21): A_w = J S J^T in constraint order, entry (a, b) as the oracle's
// chain: acc = +0; for e in J's row a: t = +0; t = fma(S_pq, J_bq, t) over f in J's row b with S_pq stored;
// acc = fma(J_ap, t, acc).  One thread per constraint a writes its lower entries of the nested-dissection layout
// (in-block band / separator rows), as k_nd_fill does for S[Z, Z].
__device__ __forceinline__ bool S_lookup(const int *S_ptr, const int *S_col, const double *S_val, int p, int q,
                                         double &v) {
  int lo = S_ptr[p / 3], hi = S_ptr[p / 3 + 1] - 1;
  const int cq = q / 3;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const int cm = S_col[mid];
    if (cm == cq) { v = S_val[(long)mid * 9 + 3 * (p % 3) + (q % 3)]; return true; }
    if (cm < cq) lo = mid + 1; else hi = mid - 1;
  }
  return false;
}
__global__ void k_nd_fill_J(int nf, int bw, int W, const NdBlk *blk, const int *block_of, const int *zpi,
                            const int *J_ptr, const int *J_col, const double *J_val, const int *S_ptr, const int *S_col,
                            const double *S_val, double *Lrow, double *Loff) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nf) return;
  const int p = zpi[a];
  const NdBlk B = blk[block_of[p]];
  const int b0 = max(0, a - bw), b1 = min(nf - 1, a + bw);
  for (int b = b0; b <= b1; b++) {
    const int q = zpi[b];
    const bool in_band = q >= B.p0 && q <= p;
    const bool in_off = B.kind == 1 && q >= B.t0 && q < B.p0;
    if (!in_band && !in_off) continue;
    double acc = 0.0;
    for (int e = J_ptr[a]; e < J_ptr[a + 1]; e++) {
      double t = 0.0;
      for (int g = J_ptr[b]; g < J_ptr[b + 1]; g++) {
        double spq;
        if (S_lookup(S_ptr, S_col, S_val, J_col[e], J_col[g], spq)) t = __fma_rn(spq, J_val[g], t);
      }
      acc = __fma_rn(J_val[e], t, acc);
    }
    if (in_band) Lrow[(long)p * W + bw - (p - q)] = acc;
    else Loff[B.off + (long)(p - B.p0) * B.rs + (q - B.t0)] = acc;
  }
}
// structural band width of J S J^T in constraint order (max over a of a - min{b : (J S J^T)_ab stored})
__global__ void k_bw_J(int m, const int *J_ptr, const int *J_col, const int *Jt_ptr, const int *Jt_row,
                       const int *S_ptr, const int *S_col, int *bw) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  int mn = a;
  for (int e = J_ptr[a]; e < J_ptr[a + 1]; e++) {
    const int I = J_col[e] / 3;
    for (int k = S_ptr[I]; k < S_ptr[I + 1]; k++)
      for (int cc = 0; cc < 3; cc++) {
        const int q = 3 * S_col[k] + cc;
        for (int t = Jt_ptr[q]; t < Jt_ptr[q + 1]; t++) mn = min(mn, Jt_row[t]);
      }
  }
  atomicMax(bw, a - mn);
}
// v = J r1 (P^T r1 for P = J^T): per constraint a the chain acc = fma(J_ap, r1_p, acc) over J's row, into the
// filter space's elimination order; r1 is given at the Z positions (rz, Z order)
__global__ void k_J_rz(int m, const int *J_ptr, const int *J_col, const double *J_val, const int *pos,
                       const double *rz, const int *zpi, double *v) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= m) return;
  double acc = 0.0;
  for (int e = J_ptr[a]; e < J_ptr[a + 1]; e++) acc = __fma_rn(J_val[e], rz[pos[J_col[e]]], acc);
  v[zpi[a]] = acc;
}
// w = J^T y (P y) at the Z positions: per dof the chain over its constraints ascending, y in elimination order
__global__ void k_Jt_y(int nc, const int *Z, const int *Jt_ptr, const int *Jt_row, const double *Jt_val,
                       const int *zpi, const double *y, double *w) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= nc) return;
  const int p = Z[a];
  double acc = 0.0;
  for (int t = Jt_ptr[p]; t < Jt_ptr[p + 1]; t++) acc = __fma_rn(Jt_val[t], y[zpi[Jt_row[t]]], acc);
  w[a] = acc;
}

// Separator rows against the columns of a diagonal block B (a leaf, or a lower separator S' after its
// subtree terms): for j in B ascending, L_sj = (acc_sj - sum_k L_sk L_jk) / L_jj with k ascending over
// [max(p0(B), j - bw), j) (C9; the only nonzero terms of the band row j).  One thread per separator row s;
// its last bw values L_sk live in a shared-memory ring (M = bw rounded up to odd: conflict-free), so each
// chain runs from shared memory (L_jk is the same band row for all threads: a broadcast load).
constexpr int OB_RC = 16, OB_NS = 3;  // band rows per staged chunk, chunks in flight
__global__ void __launch_bounds__(1024) k_nd_off_band(const int2 *pairs, const NdBlk *blk, int bw, int W, int M,
                                                      const double *Lrow, double *Loff) {
  extern __shared__ __align__(128) double ring[];  // [S.len][M] rings, then [OB_NS][OB_RC][W] band rows
  __shared__ __align__(8) uint64_t bar[OB_NS];
  const NdBlk S = blk[pairs[blockIdx.x].x], B = blk[pairs[blockIdx.x].y];
  const int s = blockIdx.y * blockDim.x + threadIdx.x;  // wide separators: rows split over grid.y
  if ((int)(blockIdx.y * blockDim.x) >= S.len) return;
  const bool act = s < S.len;
  double *Lbuf = ring + (((long)blockDim.x * M + 15) & ~15L);
  const int nch = (B.len + OB_RC - 1) / OB_RC;
  if (threadIdx.x == 0) {
    for (int q = 0; q < OB_NS; q++) mbar_init(&bar[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int ch) {  // band rows B.p0 + ch*RC .. (contiguous in Lrow) into stage ch % NS
    if (ch >= nch) return;
    const int r0 = B.p0 + ch * OB_RC, nr = min(OB_RC, B.p0 + B.len - r0);
    const unsigned bytes = (unsigned)nr * W * 8u;
    mbar_arrive_expect(&bar[ch % OB_NS], bytes);
    bulk_g2s(Lbuf + (long)(ch % OB_NS) * OB_RC * W, Lrow + (long)r0 * W, bytes, &bar[ch % OB_NS]);
  };
  if (threadIdx.x == 0)
    for (int ch = 0; ch < OB_NS - 1; ch++) issue(ch);
  double *rs = ring + (long)threadIdx.x * M;
  double *Ls = Loff + S.off + (long)min(s, S.len - 1) * S.rs - S.t0;  // Ls[k] = L_sk
  double init = act ? Ls[B.p0] : 0.0;
  for (int ch = 0; ch < nch; ch++) {
    if (threadIdx.x == 0) issue(ch + OB_NS - 1);
    mbar_wait(&bar[ch % OB_NS], (ch / OB_NS) & 1);
    const double *stage = Lbuf + (long)(ch % OB_NS) * OB_RC * W;
    const int jb = B.p0 + ch * OB_RC, je = min(jb + OB_RC, B.p0 + B.len);
    if (act)
      for (int j = jb; j < je; j++) {
        const double *Lj = stage + (long)(j - jb) * W + bw - j;  // Lj[k] = L_jk (shared memory)
        const int k0 = max(B.p0, j - bw), n = j - k0;
        const double nxt = (j + 1 < B.p0 + B.len) ? Ls[j + 1] : 0.0;
        const int st = (k0 - B.p0) % M, first = min(n, M - st);
        double acc = chain_sub(init, rs + st, 1, Lj + k0, 1, first);
        acc = chain_sub(acc, rs, 1, Lj + k0 + first, 1, n - first);
        const double v = acc / Lj[j];
        rs[(j - B.p0) % M] = v;
        Ls[j] = v;
        init = nxt;
      }
    __syncthreads();  // stage ch % NS is refilled by the issue of iteration ch + 1
    fence_proxy_async();
  }
}

// acc(s, j) = init(s, j) - sum_{k in [k0, k1)} A_sk B_jk (k ascending, C9 chains) for a 32 x 32 tile of
// (s, j), k in chunks of 32 staged through shared memory; each thread owns a 2 x 2 micro-tile, one chain
// per entry.  SCHUR: A = B = the separator's rows, lower tile entries j <= s, into the band; else A = rows
// of S, B = rows of the lower separator S', into Loff.
template <bool SCHUR>
__global__ void __launch_bounds__(256) k_nd_gemm(const int2 *pairs, const NdBlk *blk, int bw, int W, double *Lrow,
                                                 double *Loff) {
  // k-major chunks of 32 k for the 32 rows of each operand, double-buffered: the next chunk's cp.async copies
  // are in flight while the current one is consumed (the chunk loads were the critical path: 8,317-term
  // chains over 260 chunks at the top separator)
  __shared__ __align__(16) double As[2][32][34], Bs[2][32][34];
  const int2 pr = pairs[blockIdx.x];
  const NdBlk S = blk[pr.x], Sp = blk[SCHUR ? pr.x : pr.y];
  const int ti = blockIdx.y, tj = blockIdx.z;  // tile row / column
  const int s0 = ti * 32, j0 = tj * 32;
  if (s0 >= S.len || j0 >= Sp.len || (SCHUR && j0 > s0)) return;
  const int k0 = SCHUR ? S.t0 : Sp.t0, k1 = SCHUR ? S.p0 : Sp.p0;
  const double *Arow = Loff + S.off - S.t0;    // Arow[s * rs + k] = L_{p0+s, k}
  const double *Brow = Loff + Sp.off - Sp.t0;  // Brow[j * rs' + k]
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[2][2];
  auto out = [&](int a, int b) -> double * {  // destination of entry (s0 + 2ty + a, j0 + 2tx + b)
    const int s = s0 + 2 * ty + a, j = j0 + 2 * tx + b;
    if (s >= S.len || j >= Sp.len || (SCHUR && j > s)) return nullptr;
    if (SCHUR) return Lrow + (long)(S.p0 + s) * W + bw - (s - j);
    return Loff + S.off + (long)s * S.rs + (Sp.p0 + j - S.t0);
  };
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      double *o = out(a, b);
      acc[a][b] = o ? *o : 0.0;
    }
  auto issue = [&](int kc, int buf) {  // element (r, k) of both operands, zero-filled outside
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int r = e >> 5, k = e & 31;
      const bool kin = kc + k < k1;
      const bool ai = kin && s0 + r < S.len, bi = kin && j0 + r < Sp.len;
      const double *sa = ai ? Arow + (long)(s0 + r) * S.rs + kc + k : Arow;
      const double *sb = bi ? Brow + (long)(j0 + r) * Sp.rs + kc + k : Brow;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(&As[buf][k][r])), "l"(sa),
                   "r"(ai ? 8 : 0) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(&Bs[buf][k][r])), "l"(sb),
                   "r"(bi ? 8 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int nch = (k1 - k0 + 31) / 32;
  if (nch > 0) issue(k0, 0);
  for (int m = 0; m < nch; m++) {
    const int kc = k0 + 32 * m, buf = m & 1;
    if (m + 1 < nch) {
      issue(kc + 32, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int kn = min(32, k1 - kc);
    for (int kk = 0; kk < kn; kk++) {
      const double2 av = *reinterpret_cast<const double2 *>(&As[buf][kk][2 * ty]);
      const double2 bv = *reinterpret_cast<const double2 *>(&Bs[buf][kk][2 * tx]);
      acc[0][0] = __fma_rn(-av.x, bv.x, acc[0][0]);
      acc[0][1] = __fma_rn(-av.x, bv.y, acc[0][1]);
      acc[1][0] = __fma_rn(-av.y, bv.x, acc[1][0]);
      acc[1][1] = __fma_rn(-av.y, bv.y, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; a++)
#pragma unroll
    for (int b = 0; b < 2; b++) {
      double *o = out(a, b);
      if (o) *o = acc[a][b];
    }
}

typedef void (*SepFwdFn)(const int2 *, const NdBlk *, const double *, const double *, const int *, const double *,
                         const double *, double *);
struct SepFwdVariant {
  int G, NS;
  SepFwdFn fn;
};
// measured variants (tools/mb_sepfwd.cu); the first is used unless AMGF_SF_VARIANT selects another
static const SepFwdVariant kSepFwd[] = {{1, 6, k_nd_sep_fwd<1, 6, SF_KC>}, {2, 6, k_nd_sep_fwd<2, 6, SF_KC>},
                                        {4, 4, k_nd_sep_fwd<4, 4, SF_KC>}};
constexpr int kSepFwdDefault = 0;

static int sep_fwd_variant() {
  static int v = -1;
  if (v < 0) {
    v = kSepFwdDefault;
    if (const char *e = getenv("AMGF_SF_VARIANT")) {  // tuning experiments only
      int i = atoi(e);
      if (i >= 0 && i < (int)(sizeof(kSepFwd) / sizeof(kSepFwd[0]))) v = i;
    }
    const SepFwdVariant &V = kSepFwd[v];
    CK(cudaFuncSetAttribute((const void *)V.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)sf_smem(V.G, V.NS, SF_KC)));
  }
  return v;
}

// Backward, subtree rows of a separator: acc_k -= sum_{s descending} L_sk x_s (chain continues in w).
// One CTA per SB_TR consecutive subtree rows: the separator's len x SB_TR tile of L (row-major, 16-byte
// pieces) and x_S are staged with cp.async in one round trip, then thread k runs its chain from shared
// memory (the former thread-per-row form with an 8-deep register prefetch from HBM took 17 us per level).
constexpr int SB_TR = 64;
__global__ void __launch_bounds__(SB_TR) k_nd_sep_bwd(const int *ids, const NdBlk *blk, const double *Loff,
                                                      const double *x, double *w) {
  extern __shared__ __align__(16) double sbt[];  // [len][SB_TR] tile, then x_S [len]
  pdl_launch_dependents();
  const NdBlk S = blk[ids[blockIdx.y]];
  const int k0 = S.t0 + blockIdx.x * SB_TR;
  if (k0 >= S.p0) return;
  const int nk = min(SB_TR, S.p0 - k0), tid = threadIdx.x;
  double *sx = sbt + (long)S.len * SB_TR;
  const double *src = Loff + S.off + (k0 - S.t0);  // 16-byte aligned: off, rs and k0 - t0 are even
  for (int idx = tid; idx < S.len * (SB_TR / 2); idx += SB_TR) {
    const int sr = idx / (SB_TR / 2), p = idx % (SB_TR / 2);
    if (2 * p < nk) cp_async16(sbt + sr * SB_TR + 2 * p, src + (long)sr * S.rs + 2 * p);
  }
  asm volatile("cp.async.commit_group;");
  pdl_wait();  // the factor tile above does not depend on the previous kernel; x_S and w do
  for (int sr = tid; sr < S.len; sr += SB_TR) sx[sr] = x[S.p0 + sr];
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (tid < nk) {
    double acc = w[k0 + tid];
    for (int sr = S.len - 1; sr >= 0; sr--) acc = __fma_rn(-sbt[sr * SB_TR + tid], sx[sr], acc);
    w[k0 + tid] = acc;
  }
}

// ------------------------------------------------------------------ host
int band_width_J(Ctx &c) {
  Level &L0 = c.lev[0];
  int *d = c.alloc<int>(1);
  CK(cudaMemsetAsync(d, 0, sizeof(int), c.stream));
  k_bw_J<<<nblk(c.m), CTA, 0, c.stream>>>(c.m, c.J_ptr, c.J_col, c.Jt_ptr, c.Jt_row, L0.A.ptr, L0.A.col, d);
  after_launch(c, "k_bw_J");
  int bw = 0;
  CK(cudaMemcpyAsync(&bw, d, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  c.release(d);
  return bw;
}

void filter_J_apply(Ctx &c, const double *rz, double *v_pi, const double *y_pi, double *w_z) {
  if (v_pi) {
    k_J_rz<<<nblk(c.m), CTA, 0, c.stream>>>(c.m, c.J_ptr, c.J_col, c.J_val, c.pos, rz, c.zpi, v_pi);
    after_launch(c, "k_J_rz");
  } else {
    k_Jt_y<<<nblk(c.nc), CTA, 0, c.stream>>>(c.nc, c.Z, c.Jt_ptr, c.Jt_row, c.Jt_val, c.zpi, y_pi, w_z);
    after_launch(c, "k_Jt_y");
  }
}

void nd_remap_positions(Ctx &c, int *pos_z, long n) {
  if (n <= 0) return;
  k_remap<<<nblk(n), CTA, 0, c.stream>>>(n, c.zpi, pos_z);
  after_launch(c, "k_remap");
}

void nd_symbolic(Ctx &c) {
  const int nc = c.nf, bw = c.bw;  // the filter space: n_c Z positions (basis 0) or m constraints (basis 1)
  std::vector<Node> nodes;
  build(nodes, 0, nc, std::max(0, c.cfg.nd_levels), bw, 0);
  Emit E;
  std::vector<int> leaves, seps;
  emit(nodes, 0, E, leaves, seps);
  REQUIRE((int)E.pi.size() == nc, AMGF_ERR_ARG, "nd order size mismatch");
  // Loff offsets
  long off = 0;
  int depth = 0;
  std::vector<int> sep_blocks;
  for (int bi = 0; bi < (int)E.blk.size(); bi++) {
    NdBlk &b = E.blk[bi];
    if (b.kind == 1) {
      b.rs = (b.p0 - b.t0 + 1) & ~1;  // even row stride: 16-byte aligned rows
      b.off = off;
      off += (long)b.rs * b.len;
      depth = std::max(depth, b.level + 1);
      sep_blocks.push_back(bi);
    }
  }
  REQUIRE(depth <= 16, AMGF_ERR_LIMIT, "nested dissection deeper than 16 levels");
  c.nd_nblocks = (int)E.blk.size();
  c.nd_depth = depth;
  c.loff_size = off;
  c.nd_blk = upload(c, E.blk);
  c.pi_z = upload(c, E.pi);
  c.zpi = c.alloc<int>(nc);
  c.block_of = c.alloc<int>(nc);
  if (c.cfg.filter_basis == 1) {
    // P = J^T: the filter space is the constraint space; the fine rows the filter reads (r1 at I_c, the compact
    // Z rows, the x2 scatter) stay in Z order
    c.dof = c.alloc<int>(c.nc);
    CK(cudaMemcpyAsync(c.dof, c.Z, (size_t)c.nc * sizeof(int), cudaMemcpyDeviceToDevice, c.stream));
    int *scratch = c.alloc<int>(nc);
    k_nd_maps<<<nblk(nc), CTA, 0, c.stream>>>(nc, c.pi_z, c.pi_z, c.zpi, scratch);
    after_launch(c, "k_nd_maps");
    CK(cudaStreamSynchronize(c.stream));
    c.release(scratch);
  } else {
    c.dof = c.alloc<int>(nc);
    k_nd_maps<<<nblk(nc), CTA, 0, c.stream>>>(nc, c.pi_z, c.Z, c.zpi, c.dof);
    after_launch(c, "k_nd_maps");
  }
  k_nd_block_of<<<c.nd_nblocks, CTA, 0, c.stream>>>(c.nd_nblocks, (const NdBlk *)c.nd_blk, c.block_of);
  after_launch(c, "k_nd_block_of");
  // leaves
  std::vector<int> lp0, llen, pairs;
  for (int b = 0; b < (int)E.blk.size(); b++)
    if (E.blk[b].kind == 0) { lp0.push_back(E.blk[b].p0); llen.push_back(E.blk[b].len); }
  c.nd_nleaves = (int)lp0.size();
  c.nd_leaf_p0 = upload(c, lp0);
  c.nd_leaf_len = upload(c, llen);
  // separators by level, their lower separators, and (separator, leaf) pairs
  for (int l = 0; l < depth; l++) {
    std::vector<int> ids, p0, len, sptr{0}, slist;
    for (int b = 0; b < (int)E.blk.size(); b++)
      if (E.blk[b].kind == 1 && E.blk[b].level == l) {
        ids.push_back(b);
        p0.push_back(E.blk[b].p0);
        len.push_back(E.blk[b].len);
        for (int q : E.sub_seps[b]) slist.push_back(q);  // pi (post)order: deeper first
        sptr.push_back((int)slist.size());
      }
    Ctx::NdLevel &Lv = c.nd_lev[l];
    std::vector<int> groups;  // (separator block, first row) per warp of the forward dot kernel
    for (int b : ids)
      for (int r0 = 0; r0 < E.blk[b].len; r0 += kSepFwd[sep_fwd_variant()].G) {
        groups.push_back(b);
        groups.push_back(r0);
      }
    Lv.ngroups = (int)groups.size() / 2;
    Lv.groups = upload(c, groups);
    Lv.count = (int)ids.size();
    Lv.ids = upload(c, ids);
    std::vector<int> self;
    for (int b : ids) { self.push_back(b); self.push_back(b); c.nd_maxsep = std::max(c.nd_maxsep, E.blk[b].len); }
    Lv.selfpairs = upload(c, self);
    Lv.p0 = upload(c, p0);
    Lv.len = upload(c, len);
    Lv.sub_ptr = upload(c, sptr);
    Lv.sub_list = upload(c, slist);
  }
  for (int b = 0; b < (int)E.blk.size(); b++)
    if (E.blk[b].kind == 1)
      for (int lf : E.sub_leaves[b]) { pairs.push_back(b); pairs.push_back(lf); }
  c.nd_npairs = (int)pairs.size() / 2;
  c.nd_pairs = upload(c, pairs);
  // (S, S') pairs: S at level l, S' a separator in S's subtree at depth d > l; one list per (l, d)
  for (int l = 0; l < depth; l++)
    for (int d = l + 1; d < depth; d++) {
      std::vector<int> pr;
      for (int b = 0; b < (int)E.blk.size(); b++)
        if (E.blk[b].kind == 1 && E.blk[b].level == l)
          for (int q : E.sub_seps[b])
            if (E.blk[q].level == d) { pr.push_back(b); pr.push_back(q); }
      c.nd_sspairs_n[l][d] = (int)pr.size() / 2;
      c.nd_sspairs[l][d] = pr.empty() ? nullptr : upload(c, pr);
    }
  // storage
  const int W = band_stride(bw);
  const size_t total = (size_t)(nc + 2 * BAND_PAD_ROWS) * W;
  double *r = c.alloc<double>(total);
  CK(cudaMemsetAsync(r, 0, total * sizeof(double), c.stream));
  c.Lrow = r + (size_t)BAND_PAD_ROWS * W;
  // Everything the solve reads (the two band copies, the separator rows, 1/L_ii and the work vectors) in
  // one arena (one range for tools and for an L2 access-policy window; measured without benefit so far).
  auto al = [](size_t n) { return (n + 31) & ~(size_t)31; };  // 256-byte alignment
  const int nv = std::max(nc, c.nc);  // vectors of the filter space and of the Z rows
  const size_t n_band = al(total), n_off = al(off + 2), n_vec = al(nv), n_w = al(nv + SF_KC + 4);
  const size_t arena = 2 * n_band + n_off + 3 * n_vec + 2 * n_w;
  double *A = c.alloc<double>(arena);
  c.nd_arena = A;
  c.nd_arena_bytes = arena * sizeof(double);
  CK(cudaMemsetAsync(A, 0, 2 * n_band * sizeof(double), c.stream));
  c.Lcol = A + (size_t)BAND_PAD_ROWS * W;
  c.Lrev = A + n_band + (size_t)BAND_PAD_ROWS * W;
  c.Loff = A + 2 * n_band;  // +2: the 16-byte staging of an odd row tail may read one past the end
  c.Ldinv = c.Loff + n_off;
  c.fv = c.Ldinv + n_vec;
  c.rz = c.fv + n_vec;
  c.fw = c.rz + n_vec;
  c.fw2 = c.fw + n_w;
  c.nd_nsep = (int)sep_blocks.size();
  c.nd_sep_blocks = upload(c, sep_blocks);
}

static void launch_off_band(Ctx &c, int np, const int *pairs, const NdBlk *blk, int bw, int W) {
  if (!np) return;
  static const bool old_kernel = getenv("AMGF_OFFBAND_RING") != nullptr;  // A/B: the shared-memory ring kernel
  if (!old_kernel) {
    // B's column-major band copy must be current: refresh it from Lrow (the blocks factored so far)
    band_finish(c, c.nf, bw, c.Lrow, c.Lcol, c.Lrev, c.Ldinv);
    if (launch_sep_rows_sweep(c, np, pairs, blk, c.nd_maxsep, bw, c.Lcol, c.Loff)) return;
  }
  const int M = bw | 1;  // ring length >= bw, odd (bank-conflict-free rows)
  auto smem_of = [&](int t) {
    return ((((size_t)t * M + 15) & ~(size_t)15) + (size_t)OB_NS * OB_RC * W) * sizeof(double);
  };
  // as many separator rows per CTA as the rings fit in shared memory; the rest go to grid.y
  int threads = std::min(1024, (c.nd_maxsep + 31) / 32 * 32);
  while (threads > 32 && smem_of(threads) > 227 * 1024) threads -= 32;
  const size_t smem = smem_of(threads);
  REQUIRE(smem <= 227 * 1024, AMGF_ERR_LIMIT, "band too wide for the off-block factor kernel");
  const dim3 grid(np, (c.nd_maxsep + threads - 1) / threads);
  size_t &attr = device_slot((const void *)k_nd_off_band);
  if (smem > attr) {
    CK(cudaFuncSetAttribute(k_nd_off_band, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  k_nd_off_band<<<grid, threads, smem, c.stream>>>((const int2 *)pairs, blk, bw, W, M, c.Lrow, c.Loff);
  after_launch(c, "k_nd_off_band");
}

void nd_numeric(Ctx &c) {
  const int nc = c.nf, bw = c.bw, W = band_stride(bw);
  const NdBlk *blk = (const NdBlk *)c.nd_blk;
  Level &L0 = c.lev[0];
  CK(cudaMemsetAsync(c.Lrow - (size_t)BAND_PAD_ROWS * W, 0, (size_t)(nc + 2 * BAND_PAD_ROWS) * W * sizeof(double),
                     c.stream));
  if (c.loff_size) CK(cudaMemsetAsync(c.Loff, 0, c.loff_size * sizeof(double), c.stream));
  if (c.cfg.filter_basis == 1) {
    k_nd_fill_J<<<nblk(nc), CTA, 0, c.stream>>>(nc, bw, W, blk, c.block_of, c.zpi, c.J_ptr, c.J_col, c.J_val,
                                                L0.A.ptr, L0.A.col, L0.A.val, c.Lrow, c.Loff);
    after_launch(c, "k_nd_fill_J");
  } else {
    k_nd_fill<<<nblk(nc), CTA, 0, c.stream>>>(nc, bw, W, blk, c.block_of, c.dof, c.pos, c.zpi, L0.A.ptr, L0.A.col,
                                              L0.A.val, c.Lrow, c.Loff);
    after_launch(c, "k_nd_fill");
  }
  // leaves (independent), then separator-vs-leaf columns (independent given the leaves)
  band_factor_blocks(c, nc, c.nd_nleaves, c.nd_leaf_p0, c.nd_leaf_len, bw, c.Lrow, 1);
  if (c.nd_npairs) {
    launch_off_band(c, c.nd_npairs, c.nd_pairs, blk, bw, W);
  }
  // separators bottom-up; for a separator S at level l, its lower separators S' (depth d > l) in postorder
  // (deepest first), each in two parts (subtree terms in parallel, then the S'-internal chain)
  for (int l = c.nd_depth - 1; l >= 0; l--) {
    Ctx::NdLevel &Lv = c.nd_lev[l];
    if (!Lv.count) continue;
    for (int d = c.nd_depth - 1; d > l; d--) {
      const int np = c.nd_sspairs_n[l][d];
      if (!np) continue;
      const int nt = (c.nd_maxsep + 31) / 32;
      dim3 g1(np, nt, nt);
      k_nd_gemm<false><<<g1, 256, 0, c.stream>>>((const int2 *)c.nd_sspairs[l][d], blk, bw, W, c.Lrow, c.Loff);
      after_launch(c, "k_nd_gemm");
      launch_off_band(c, np, c.nd_sspairs[l][d], blk, bw, W);
    }
    const int nt = (c.nd_maxsep + 31) / 32;
    dim3 g2(Lv.count, nt, nt);
    k_nd_gemm<true><<<g2, 256, 0, c.stream>>>((const int2 *)Lv.selfpairs, blk, bw, W, c.Lrow, c.Loff);
    after_launch(c, "k_nd_gemm");
    band_factor_blocks(c, nc, Lv.count, Lv.p0, Lv.len, bw, c.Lrow, 1);
  }
  band_finish(c, nc, bw, c.Lrow, c.Lcol, c.Lrev, c.Ldinv);
}


void nd_solve(Ctx &c, const double *r1, const int *gather) {
  const int nc = c.nf, bw = c.bw;
  const NdBlk *blk = (const NdBlk *)c.nd_blk;
  double *w = c.fw, *y = c.fv;
  // forward: leaves (gathered r1), then separators bottom-up
  launch_band_sweep(c, c.nd_nleaves, c.nd_leaf_p0, c.nd_leaf_len, nc, bw, true, c.Lcol, c.Lrev, c.Ldinv, r1, gather,
                    w, c.fw2);
  for (int l = c.nd_depth - 1; l >= 0; l--) {
    Ctx::NdLevel &Lv = c.nd_lev[l];
    if (!Lv.count) continue;
    const SepFwdVariant &V = kSepFwd[sep_fwd_variant()];
    launch_pdl(c.stream, V.fn, dim3(Lv.ngroups), dim3(32), sf_smem(V.G, V.NS, SF_KC), (const int2 *)Lv.groups, blk,
               (const double *)c.Loff, r1, gather, (const double *)w, (const double *)c.fw2, y);
    after_launch(c, "k_nd_sep_fwd");
    launch_band_sweep(c, Lv.count, Lv.p0, Lv.len, nc, bw, true, c.Lcol, c.Lrev, c.Ldinv, y, nullptr, w, c.fw2);
  }
  // backward: separators top-down (then their subtree rows), then leaves
  const size_t sb_smem = (size_t)c.nd_maxsep * (SB_TR + 1) * sizeof(double);
  {
    size_t &attr = device_slot((const void *)k_nd_sep_bwd);
    if (sb_smem > attr && sb_smem > 48 * 1024) {
      CK(cudaFuncSetAttribute(k_nd_sep_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb_smem));
      attr = sb_smem;
    }
  }
  for (int l = 0; l < c.nd_depth; l++) {
    Ctx::NdLevel &Lv = c.nd_lev[l];
    if (!Lv.count) continue;
    launch_band_sweep(c, Lv.count, Lv.p0, Lv.len, nc, bw, false, c.Lcol, c.Lrev, c.Ldinv, w, nullptr, y);
    dim3 grid((nc + SB_TR - 1) / SB_TR, Lv.count);
    launch_pdl(c.stream, k_nd_sep_bwd, grid, dim3(SB_TR), sb_smem, (const int *)Lv.ids, blk, (const double *)c.Loff,
               (const double *)y, w);
    after_launch(c, "k_nd_sep_bwd");
  }
  launch_band_sweep(c, c.nd_nleaves, c.nd_leaf_p0, c.nd_leaf_len, nc, bw, false, c.Lcol, c.Lrev, c.Ldinv, w, nullptr,
                    y);
}

}  // namespace amgf
