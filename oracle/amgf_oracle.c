/*
 * amgf_oracle.c -- plain, slow, single-threaded CPU oracle for the AMGF-PCG
 * solve path (arxiv 2505.18576, "AMG with Filtering").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2505_18576_b200/csrc); its only common ground with that path is the
 * seeded input generator amgf_gen/ and the arithmetic contract written in
 * DESIGN.md section "Contract" (which FMA, which order, which reduction tree).
 *
 * Compiled with  gcc -O2 -ffp-contract=off -fno-fast-math  so that every
 * floating-point operation below is exactly one IEEE binary64 round-to-nearest
 * operation; fused multiply-adds happen only where fma() is written.
 *
 * Paper map (PAPER.md line numbers):
 *   S = K + J^T D J ........................ eq:linsystem1
 *   I_c, P (natural embedding), A_w=P^TAP .. Def. Discrete Operators
 *   M: I-MA = (I-BA)(I-P A_w^{-1} P^T A)(I-BA)  Def. AMGF eq:M_itmat
 *   B = AMG V-cycle with l1 smoother ........ Remark upper_bound_estimate
 *   PCG, relative preconditioned residual ... PAPER.md:368
 *   three-stage apply x1=Br; r1=r-Ax1; x2=x1+PA_w^{-1}P^Tr1; r2; x=x2+Br2 ... SPEC.md:245
 *   smoothed aggregation hierarchy ........... SPEC.md:165-173 (readings R4-R8 in DESIGN.md)
 *
 * Parity pins: every function below is pinned by a "-m 'not gpu'" test in
 * tests/test_oracle_pins.py (closed forms, dense numpy linear algebra, the
 * paper's lemmas, golden fixtures).  Functions without such a pin are listed
 * as "parity unpinned" in DESIGN.md; at present: none.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <time.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 1
#define ORC_ERR_ARG (-1)
#define ORC_ERR_NONFINITE (-2)
#define ORC_ERR_DOMAIN (-3)
#define ORC_ERR_NOT_SPD (-4)
#define ORC_ERR_RANK (-5)
#define ORC_ERR_BREAKDOWN (-6)
#define ORC_ERR_OOM (-8)

#define MAXLEV 32

static char g_err[512];
const char *orc_last_error(void) { return g_err; }
static int fail(int code, const char *msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------ */
/* Block sparse row matrix: nbr block rows of br x bc row-major blocks. */
typedef struct {
  int nbr, nbc, br, bc;
  int *ptr, *col;
  double *val;
} bsr_t;

static void bsr_free(bsr_t *a) {
  free(a->ptr); free(a->col); free(a->val);
  memset(a, 0, sizeof *a);
}
static int bsr_alloc(bsr_t *a, int nbr, int nbc, int br, int bc, long nnzb) {
  a->nbr = nbr; a->nbc = nbc; a->br = br; a->bc = bc;
  a->ptr = (int *)calloc((size_t)nbr + 1, sizeof(int));
  a->col = (int *)malloc((size_t)(nnzb > 0 ? nnzb : 1) * sizeof(int));
  a->val = (double *)calloc((size_t)(nnzb > 0 ? nnzb : 1) * br * bc, sizeof(double));
  return (a->ptr && a->col && a->val) ? ORC_OK : ORC_ERR_OOM;
}
static long bsr_nnzb(const bsr_t *a) { return a->ptr[a->nbr]; }

/* y = A x, per scalar row one accumulator from +0, fma over stored entries in
 * ascending scalar column (block column ascending, then column in block).
 * Contract C2.  mode 0: y = acc; mode 1: y = b - acc. */
static void bsr_spmv(const bsr_t *A, const double *x, const double *b, double *y, int mode) {
  int br = A->br, bc = A->bc;
  for (int i = 0; i < A->nbr; i++) {
    for (int r = 0; r < br; r++) {
      double acc = 0.0;
      for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
        const double *blk = A->val + (size_t)k * br * bc + (size_t)r * bc;
        const double *xs = x + (size_t)A->col[k] * bc;
        for (int c = 0; c < bc; c++) acc = fma(blk[c], xs[c], acc);
      }
      y[(size_t)i * br + r] = mode ? b[(size_t)i * br + r] - acc : acc;
    }
  }
}

/* Restriction y = R x with the warp-strided contract C5: per scalar row, lane l
 * (0..31) accumulates the row's blocks j = l, l+32, ... (row-relative index),
 * columns ascending inside a block, from +0 with fma; then the xor butterfly
 * s[l] = s[l] + s[l^o] for o = 16,8,4,2,1; result = s[0]. */
static void bsr_spmv_warp32(const bsr_t *A, const double *x, double *y) {
  int br = A->br, bc = A->bc;
  for (int i = 0; i < A->nbr; i++) {
    for (int r = 0; r < br; r++) {
      double s[32], t[32];
      for (int l = 0; l < 32; l++) {
        double acc = 0.0;
        for (int k = A->ptr[i] + l; k < A->ptr[i + 1]; k += 32) {
          const double *blk = A->val + (size_t)k * br * bc + (size_t)r * bc;
          const double *xs = x + (size_t)A->col[k] * bc;
          for (int c = 0; c < bc; c++) acc = fma(blk[c], xs[c], acc);
        }
        s[l] = acc;
      }
      for (int o = 16; o >= 1; o >>= 1) {
        for (int l = 0; l < 32; l++) t[l] = s[l] + s[l ^ o];
        memcpy(s, t, sizeof s);
      }
      y[(size_t)i * br + r] = s[0];
    }
  }
}

/* Contract C14: dot product over n = nb*b scalars grouped in block rows of b.
 * Level 1: CTA c of 256 "threads"; thread t owns block row 256c+t and sums its
 * b products with an fma chain from +0; then tree s[t] += s[t+w], w=128..1.
 * Level 2: lane l sums partials c = l, l+256, ... in ascending c with plain
 * adds from +0; then the same tree.  Returns s[0]. */
double orc_dot(long n, int b, const double *u, const double *v) {
  long nb = n / b;
  long C = (nb + 255) / 256;
  double *part = (double *)malloc((size_t)(C > 0 ? C : 1) * sizeof(double));
  double s[256];
  for (long c = 0; c < C; c++) {
    for (int t = 0; t < 256; t++) {
      long i = 256 * c + t;
      double acc = 0.0;
      if (i < nb)
        for (int e = 0; e < b; e++) acc = fma(u[i * b + e], v[i * b + e], acc);
      s[t] = acc;
    }
    for (int w = 128; w >= 1; w >>= 1)
      for (int t = 0; t < w; t++) s[t] = s[t] + s[t + w];
    part[c] = s[0];
  }
  for (int l = 0; l < 256; l++) {
    double acc = 0.0;
    for (long c = l; c < C; c += 256) acc = acc + part[c];
    s[l] = acc;
  }
  for (int w = 128; w >= 1; w >>= 1)
    for (int t = 0; t < w; t++) s[t] = s[t] + s[t + w];
  free(part);
  return s[0];
}

/* Dense Cholesky A = L L^T (lower, row-major n x n), left-looking, contract C9:
 * acc = a_ij; acc = fma(-L_ik, L_jk, acc) for k = 0..j-1 ascending;
 * L_jj = sqrt(acc) (NOT_SPD unless acc > 0); L_ij = acc / L_jj.
 * Entries above the diagonal are set to 0. */
int orc_cholesky_dense(int n, const double *A, double *L) {
  for (long q = 0; q < (long)n * n; q++) L[q] = 0.0;
  for (int j = 0; j < n; j++) {
    double acc = A[(size_t)j * n + j];
    for (int k = 0; k < j; k++) acc = fma(-L[(size_t)j * n + k], L[(size_t)j * n + k], acc);
    if (!(acc > 0.0)) {
      snprintf(g_err, sizeof g_err, "Cholesky: non-positive pivot %.3e at %d", acc, j);
      return ORC_ERR_NOT_SPD;
    }
    double ljj = sqrt(acc);
    L[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; i++) {
      double a = A[(size_t)i * n + j];
      for (int k = 0; k < j; k++) a = fma(-L[(size_t)i * n + k], L[(size_t)j * n + k], a);
      L[(size_t)i * n + j] = a / ljj;
    }
  }
  return ORC_OK;
}

/* Contract C10: forward  y_i = (v_i - sum_{k<i} L_ik y_k) * (1/L_ii), chain over k ascending;
 * backward x_i = (w_i - sum_{k>i} L_ki x_k) * (1/L_ii), chain over k descending.
 * The reciprocal 1/L_ii is one correctly rounded division (C10). */
void orc_trsv_dense(int n, const double *L, const double *v, double *x) {
  double *y = (double *)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  for (int i = 0; i < n; i++) {
    double acc = v[i];
    for (int k = 0; k < i; k++) acc = fma(-L[(size_t)i * n + k], y[k], acc);
    y[i] = acc * (1.0 / L[(size_t)i * n + i]);
  }
  for (int i = n - 1; i >= 0; i--) {
    double acc = y[i];
    for (int k = n - 1; k > i; k--) acc = fma(-L[(size_t)k * n + i], x[k], acc);
    x[i] = acc * (1.0 / L[(size_t)i * n + i]);
  }
  free(y);
}

/* SplitMix64 finalizer used for the aggregation priorities (contract C16). */
static uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
uint64_t orc_priority(int v, uint64_t seed) { return mix64((uint64_t)(uint32_t)v ^ seed); }

/* ------------------------------------------------------------------ */
typedef struct {
  int pre_sweeps, post_sweeps, coarsest_size, max_levels, power_iters, factor_filter;
  uint64_t agg_seed;
  int nd_levels;  /* nested-dissection depth of A_w's elimination order (contract C9/C10, reading R16) */
  int smoother;   /* 0 = l1-Jacobi, 1 = Chebyshev (default) in D_l1^{-1} A (variant f4, reading R18) */
  int cheb_degree;
  int filter_basis; /* 0: P = identity columns at I_c (Def. Discrete Operators); 1: P = J^T, the
                       generality remark's full-column-rank P (variant f4, reading R21) */
  double cheb_ratio;
} orc_config;

typedef struct {
  bsr_t A;          /* level operator, b x b blocks */
  int b, nodes;     /* block size and node (block-row) count */
  long n;           /* scalar size */
  double *dl1;      /* l1 row sums */
  double *dpt;      /* point diagonal */
  int *agg;         /* aggregate of each node, -1 isolated */
  int *comp;        /* component label of each node (aggregation graph) */
  int *root;        /* 1 if the node is an aggregate root */
  int n_agg;
  bsr_t Pt;         /* tentative prolongator (b x 6) */
  bsr_t P;          /* smoothed prolongator (b x 6) */
  bsr_t R;          /* restriction P^T (6 x b) */
  double *Bnn;      /* near-null space, n x 6 row-major */
  double *bfac;     /* smoother 2 (nodal-block l1): per node the lower Cholesky factor of B_i, row-major
                       b(b+1)/2 entries, then the b reciprocals 1/L_rr (contract C24) */
  double lambda, omega;
} level_t;

typedef struct {
  orc_config cfg;
  int nodes;
  long n;
  int m;
  bsr_t S;
  int nc;
  int *Z;        /* contact dofs, the column order of P */
  int *pos;      /* dof -> position in Z or -1 */
  int bw;        /* structural lower band width of A_w in Z order */
  int *pi;       /* elimination order: pi[i] = position in Z of the i-th eliminated dof */
  int nf;        /* filter-space dimension: n_c (basis 0) or m (basis 1) */
  int mJ;        /* basis 1: J (CSR, columns ascending) and J^T as per-dof constraint lists (rows ascending) */
  int *Jp, *Jc, *Jtp, *Jtr;
  double *Jv, *Jtv;
  double *Aw;    /* dense nf x nf: S[Z,Z] (basis 0, Z order) or J S J^T (basis 1, constraint order) */
  double *Lw;    /* Cholesky factor of Aw[pi, pi] */
  int nlev;
  level_t lev[MAXLEV];
  double *Ac, *Lc; /* coarsest dense operator and factor */
  int nco;
  double *work[MAXLEV][4];
  double t_phase[4]; /* wall seconds of orc_create's phases: S, A_w assembly, A_w Cholesky, hierarchy */
} orc_ctx;

/* Wall clock for the phase times (instrumentation only; no effect on any result). */
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int cmp_int(const void *a, const void *b) {
  int x = *(const int *)a, y = *(const int *)b;
  return (x > y) - (x < y);
}

/* ---------- S = K + J^T D J (eq:linsystem1), contract C1 ---------- */
static int form_S(orc_ctx *cx, const int *Kptr, const int *Kcol, const double *Kval,
                  int m, const int *Jptr, const int *Jcol, const double *Jval, const double *D,
                  const double *Dlo, const double *Dup) {
  int nodes = cx->nodes;
  long n = cx->n;
  /* J^T as lists per dof (constraint rows ascending) */
  int *cnt = (int *)calloc((size_t)n + 1, sizeof(int));
  for (int k = 0; k < m; k++)
    for (int e = Jptr[k]; e < Jptr[k + 1]; e++) cnt[Jcol[e] + 1]++;
  for (long p = 0; p < n; p++) cnt[p + 1] += cnt[p];
  int *tk = (int *)malloc((size_t)(cnt[n] > 0 ? cnt[n] : 1) * sizeof(int));
  double *tv = (double *)malloc((size_t)(cnt[n] > 0 ? cnt[n] : 1) * sizeof(double));
  int *fill = (int *)calloc((size_t)n, sizeof(int));
  for (int k = 0; k < m; k++)
    for (int e = Jptr[k]; e < Jptr[k + 1]; e++) {
      int p = Jcol[e];
      tk[cnt[p] + fill[p]] = k;
      tv[cnt[p] + fill[p]] = Jval[e];
      fill[p]++;
    }
  /* block pattern: K pattern union {(node(p), node(q)) : p, q in one J row} */
  int *tmp = (int *)malloc(4096 * sizeof(int));
  int *rowlen = (int *)calloc((size_t)nodes + 1, sizeof(int));
  int **rows = (int **)calloc((size_t)nodes, sizeof(int *));
  long total = 0;
  for (int I = 0; I < nodes; I++) {
    int t = 0;
    for (int e = Kptr[I]; e < Kptr[I + 1]; e++) tmp[t++] = Kcol[e];
    for (int r = 0; r < 3; r++) {
      long p = 3L * I + r;
      for (int e = cnt[p]; e < cnt[p + 1]; e++) {
        int k = tk[e];
        for (int f = Jptr[k]; f < Jptr[k + 1]; f++) {
          if (t >= 4096) { free(tmp); return fail(ORC_ERR_ARG, "S row too long"); }
          tmp[t++] = Jcol[f] / 3;
        }
      }
    }
    qsort(tmp, t, sizeof(int), cmp_int);
    int u = 0;
    for (int q = 0; q < t; q++)
      if (u == 0 || tmp[q] != tmp[u - 1]) tmp[u++] = tmp[q];
    rows[I] = (int *)malloc((size_t)u * sizeof(int));
    memcpy(rows[I], tmp, (size_t)u * sizeof(int));
    rowlen[I] = u;
    total += u;
  }
  if (bsr_alloc(&cx->S, nodes, nodes, 3, 3, total)) return fail(ORC_ERR_OOM, "oom S");
  long w = 0;
  for (int I = 0; I < nodes; I++) {
    cx->S.ptr[I] = (int)w;
    int ke = Kptr[I];
    for (int q = 0; q < rowlen[I]; q++) {
      int Jn = rows[I][q];
      cx->S.col[w] = Jn;
      double *blk = cx->S.val + 9 * w;
      while (ke < Kptr[I + 1] && Kcol[ke] < Jn) ke++;
      int hasK = (ke < Kptr[I + 1] && Kcol[ke] == Jn);
      for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) {
          long p = 3L * I + r, qd = 3L * Jn + c;
          double acc = hasK ? Kval[9L * ke + 3 * r + c] : 0.0;
          /* constraints touching both p and qd, ascending k */
          int a = cnt[p], ae = cnt[p + 1], bb = cnt[qd], be = cnt[qd + 1];
          while (a < ae && bb < be) {
            if (tk[a] < tk[bb]) a++;
            else if (tk[a] > tk[bb]) bb++;
            else {
              double t = tv[a] * D[tk[a]];
              acc = fma(t, tv[bb], acc);
              a++; bb++;
            }
          }
          if (p == qd) {
            /* bound-constrained A~ = K + J~^T D~ J~, J~ = [J; I; -I], D~ = diag(D, D_lo, D_up) (Remark
             * boundconstr): the rows of I and -I come after J's, so the diagonal entry
             * continues the same chain with t = 1 * D_lo[p], fma(t, 1, acc), then t = -1 * D_up[p],
             * fma(t, -1, acc) (contract C1); off-diagonal entries have no bound rows. */
            if (Dlo) { double t = 1.0 * Dlo[p]; acc = fma(t, 1.0, acc); }
            if (Dup) { double t = -1.0 * Dup[p]; acc = fma(t, -1.0, acc); }
          }
          blk[3 * r + c] = acc;
        }
      w++;
    }
    free(rows[I]);
  }
  cx->S.ptr[nodes] = (int)w;
  free(rows); free(rowlen); free(tmp); free(cnt); free(tk); free(tv); free(fill);
  return ORC_OK;
}

/* Elimination order of A_w (reading R16): one-dimensional nested dissection of the band.  The interval
 * [a, b) of Z positions is a leaf if depth == 0 or b - a < 4 bw + 64; otherwise it is split by the
 * separator [m, m + bw), m = a + (b - a - bw)/2, which decouples [a, m) from [m + bw, b) because A_w has
 * no entries farther than bw from the diagonal.  Postorder: left subtree, right subtree, separator. */
static void nd_rec(int a, int b, int depth, int bw, int *out, int *cnt) {
  if (depth == 0 || b - a < 4 * bw + 64) {
    for (int i = a; i < b; i++) out[(*cnt)++] = i;
    return;
  }
  int m = a + (b - a - bw) / 2;
  nd_rec(a, m, depth - 1, bw, out, cnt);
  nd_rec(m + bw, b, depth - 1, bw, out, cnt);
  for (int i = m; i < m + bw; i++) out[(*cnt)++] = i;
}
void orc_nd_order(int nc, int bw, int levels, int *out) {
  int cnt = 0;
  nd_rec(0, nc, levels, bw, out, &cnt);
}

/* ---------- I_c and A_w = P^T S P ---------- */
/* S_pq if stored (block row p/3, block column q/3), else *found = 0. */
static double S_entry(const orc_ctx *cx, long p, long q, int *found) {
  const int I = (int)(p / 3), Jn = (int)(q / 3);
  int lo = cx->S.ptr[I], hi = cx->S.ptr[I + 1] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (cx->S.col[mid] == Jn) { *found = 1; return cx->S.val[9L * mid + 3 * (p % 3) + (q % 3)]; }
    if (cx->S.col[mid] < Jn) lo = mid + 1; else hi = mid - 1;
  }
  *found = 0;
  return 0.0;
}

/* Filter basis P = J^T (variant f4; the generality remark: any full-column-rank P): the
 * filter space is the constraint space, A_w = P^T S P = J S J^T (m x m) in constraint order.  Entry (a, b)
 * follows the definition sum_p J_ap (sum_q S_pq J_bq) as one chain (reading R21): acc = +0; for p in J's row a
 * ascending: t = +0; t = fma(S_pq, J_bq, t) over q in J's row b ascending with S_pq stored; acc = fma(J_ap, t,
 * acc) -- pairs (a, b) whose rows touch no stored S entry are structural zeros.  Elimination order: the
 * nested dissection of R16 over the structural band width of J S J^T in constraint order. */
static int setup_filter_J(orc_ctx *cx, int m, const int *Jptr, const int *Jcol, const double *Jval) {
  const long n = cx->n;
  cx->mJ = m;
  cx->nf = m;
  cx->Jp = (int *)malloc((size_t)(m + 1) * sizeof(int));
  memcpy(cx->Jp, Jptr, (size_t)(m + 1) * sizeof(int));
  const int nnz = Jptr[m];
  cx->Jc = (int *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int));
  cx->Jv = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  memcpy(cx->Jc, Jcol, (size_t)nnz * sizeof(int));
  memcpy(cx->Jv, Jval, (size_t)nnz * sizeof(double));
  cx->Jtp = (int *)calloc((size_t)n + 1, sizeof(int));
  for (int e = 0; e < nnz; e++) cx->Jtp[Jcol[e] + 1]++;
  for (long p = 0; p < n; p++) cx->Jtp[p + 1] += cx->Jtp[p];
  cx->Jtr = (int *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int));
  cx->Jtv = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
  int *fill = (int *)calloc((size_t)n, sizeof(int));
  for (int a = 0; a < m; a++)
    for (int e = Jptr[a]; e < Jptr[a + 1]; e++) {
      const int p = Jcol[e];
      cx->Jtr[cx->Jtp[p] + fill[p]] = a;
      cx->Jtv[cx->Jtp[p] + fill[p]] = Jval[e];
      fill[p]++;
    }
  free(fill);
  /* structural band width of J S J^T in constraint order */
  char *cand = (char *)calloc((size_t)(m > 0 ? m : 1), 1);
  int bw = 0;
  for (int a = 0; a < m; a++) {
    int mn = a;
    for (int e = Jptr[a]; e < Jptr[a + 1]; e++) {
      const int I = Jcol[e] / 3;
      for (int k = cx->S.ptr[I]; k < cx->S.ptr[I + 1]; k++)
        for (int c = 0; c < 3; c++) {
          const long q = 3L * cx->S.col[k] + c;
          for (int t = cx->Jtp[q]; t < cx->Jtp[q + 1]; t++)
            if (cx->Jtr[t] < mn) mn = cx->Jtr[t];
        }
    }
    if (a - mn > bw) bw = a - mn;
  }
  free(cand);
  cx->bw = bw;
  cx->pi = (int *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int));
  orc_nd_order(m, bw, cx->cfg.nd_levels, cx->pi);
  if (!cx->cfg.factor_filter || m == 0) return ORC_OK;
  cx->Aw = (double *)calloc((size_t)m * m, sizeof(double));
  cx->Lw = (double *)malloc((size_t)m * m * sizeof(double));
  double *Ap = (double *)malloc((size_t)m * m * sizeof(double));
  if (!cx->Aw || !cx->Lw || !Ap) return fail(ORC_ERR_OOM, "oom A_w (J S J^T)");
  for (int a = 0; a < m; a++)
    for (int b = (a - bw > 0 ? a - bw : 0); b < m && b <= a + bw; b++) {
      double acc = 0.0;
      for (int e = Jptr[a]; e < Jptr[a + 1]; e++) {
        double t = 0.0;
        for (int f = Jptr[b]; f < Jptr[b + 1]; f++) {
          int found;
          const double spq = S_entry(cx, Jcol[e], Jcol[f], &found);
          if (found) t = fma(spq, Jval[f], t);
        }
        acc = fma(Jval[e], t, acc);
      }
      cx->Aw[(size_t)a * m + b] = acc;
    }
  for (int i = 0; i < m; i++)
    for (int j = 0; j < m; j++) Ap[(size_t)i * m + j] = cx->Aw[(size_t)cx->pi[i] * m + cx->pi[j]];
  double t0 = now_s();
  int st = orc_cholesky_dense(m, Ap, cx->Lw);
  cx->t_phase[2] = now_s() - t0;
  free(Ap);
  if (st) {
    char buf[512];
    snprintf(buf, sizeof buf, "A_w (J S J^T): %.470s", g_err);
    return fail(st, buf);
  }
  return ORC_OK;
}

static int setup_filter(orc_ctx *cx, int m, const int *Jptr, const int *Jcol, const double *Jval, const int *Z,
                        int nc) {
  long n = cx->n;
  char *mark = (char *)calloc((size_t)n, 1);
  for (int k = 0; k < m; k++)
    for (int e = Jptr[k]; e < Jptr[k + 1]; e++) mark[Jcol[e]] = 1;
  long nmark = 0;
  for (long p = 0; p < n; p++) nmark += mark[p];
  cx->pos = (int *)malloc((size_t)n * sizeof(int));
  for (long p = 0; p < n; p++) cx->pos[p] = -1;
  if (Z) {
    /* Z must be duplicate-free and contain every structurally nonzero column of J (reading R1/R17:
     * I_c = dofs whose basis support touches the contact surface, PAPER.md:384 - a superset of J's
     * column support, e.g. all components of the interface nodes). */
    cx->Z = (int *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(int));
    long covered = 0;
    for (int a = 0; a < nc; a++) {
      int p = Z[a];
      if (p < 0 || p >= n || cx->pos[p] >= 0) {
        free(mark);
        return fail(ORC_ERR_ARG, "Z has an out-of-range or duplicate dof");
      }
      cx->Z[a] = p;
      cx->pos[p] = a;
      covered += mark[p];
    }
    if (covered != nmark) { free(mark); return fail(ORC_ERR_ARG, "Z does not contain every column of J"); }
  } else {
    nc = (int)nmark;
    cx->Z = (int *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(int));
    int a = 0;
    for (long p = 0; p < n; p++)
      if (mark[p]) { cx->Z[a] = (int)p; cx->pos[p] = a; a++; }
  }
  free(mark);
  cx->nc = nc;
  /* structural band width in Z order: bw = max_a (a - min{b <= a : S[Z_a, Z_b] stored}) */
  int bw = 0;
  for (int a = 0; a < nc; a++) {
    int p = cx->Z[a], I = p / 3, mn = a;
    for (int k = cx->S.ptr[I]; k < cx->S.ptr[I + 1]; k++)
      for (int c = 0; c < 3; c++) {
        int b = cx->pos[3 * cx->S.col[k] + c];
        if (b >= 0 && b < mn) mn = b;
      }
    if (a - mn > bw) bw = a - mn;
  }
  cx->bw = bw;
  cx->nf = nc;
  if (cx->cfg.filter_basis == 1) return setup_filter_J(cx, m, Jptr, Jcol, Jval);
  cx->pi = (int *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(int));
  orc_nd_order(nc, bw, cx->cfg.nd_levels, cx->pi);
  if (!cx->cfg.factor_filter || nc == 0) return ORC_OK;
  cx->Aw = (double *)calloc((size_t)nc * nc, sizeof(double));
  cx->Lw = (double *)malloc((size_t)nc * nc * sizeof(double));
  double *Ap = (double *)malloc((size_t)nc * nc * sizeof(double));
  if (!cx->Aw || !cx->Lw || !Ap) return fail(ORC_ERR_OOM, "oom A_w");
  for (int a = 0; a < nc; a++) {
    int p = cx->Z[a], I = p / 3, r = p % 3;
    for (int k = cx->S.ptr[I]; k < cx->S.ptr[I + 1]; k++)
      for (int c = 0; c < 3; c++) {
        int q = 3 * cx->S.col[k] + c;
        if (cx->pos[q] >= 0) cx->Aw[(size_t)a * nc + cx->pos[q]] = cx->S.val[9L * k + 3 * r + c];
      }
  }
  for (int i = 0; i < nc; i++)
    for (int j = 0; j < nc; j++) Ap[(size_t)i * nc + j] = cx->Aw[(size_t)cx->pi[i] * nc + cx->pi[j]];
  double t0 = now_s();
  int st = orc_cholesky_dense(nc, Ap, cx->Lw);
  cx->t_phase[2] = now_s() - t0;
  free(Ap);
  if (st) {
    char buf[512];
    snprintf(buf, sizeof buf, "A_w: %.480s", g_err);
    return fail(st, buf);
  }
  return ORC_OK;
}

/* ---------- AMG setup helpers (R4-R8) ---------- */
/* Aggregation graph (reading R5): the off-diagonal block pattern of A_l
 * restricted to pairs of nodes with the same component label comp[] (level 0:
 * connected components of K's block graph, i.e. the bodies; coarse levels: the
 * label of the aggregate's nodes).  Contact couplings J^T D J between bodies are
 * left to the filter and do not merge aggregates. */
static int edge(const level_t *L, int v, int u) { return u != v && L->comp[u] == L->comp[v]; }

static int is_isolated(const level_t *L, int i) {
  const bsr_t *A = &L->A;
  for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++)
    if (edge(L, i, A->col[k])) return 0;
  return 1;
}

typedef struct { uint64_t pr; int id; } prio_t;
static int cmp_prio_desc(const void *a, const void *b) {
  const prio_t *x = (const prio_t *)a, *y = (const prio_t *)b;
  if (x->pr != y->pr) return x->pr < y->pr ? 1 : -1;
  return (x->id > y->id) - (x->id < y->id);
}

/* Aggregation, contract C16: sequential greedy distance-2 MIS over nodes in
 * descending (priority, -id); roots + their distance-1 neighbours; leftovers
 * join the neighbouring root-aggregate with most edges (ties: smallest id). */
static int aggregate(level_t *L, uint64_t seed) {
  const bsr_t *A = &L->A;
  int nn = L->nodes;
  L->agg = (int *)malloc((size_t)nn * sizeof(int));
  char *iso = (char *)malloc((size_t)nn);
  char *blocked = (char *)calloc((size_t)nn, 1);
  char *root = (char *)calloc((size_t)nn, 1);
  prio_t *ord = (prio_t *)malloc((size_t)nn * sizeof(prio_t));
  int no = 0;
  for (int v = 0; v < nn; v++) {
    iso[v] = (char)is_isolated(L, v);
    L->agg[v] = -1;
    if (!iso[v]) { ord[no].pr = orc_priority(v, seed); ord[no].id = v; no++; }
  }
  qsort(ord, no, sizeof(prio_t), cmp_prio_desc);
  for (int q = 0; q < no; q++) {
    int v = ord[q].id;
    if (blocked[v]) continue;
    root[v] = 1;
    blocked[v] = 1;
    for (int k = A->ptr[v]; k < A->ptr[v + 1]; k++) {
      int u = A->col[k];
      if (!edge(L, v, u)) continue;
      blocked[u] = 1;
      for (int k2 = A->ptr[u]; k2 < A->ptr[u + 1]; k2++)
        if (edge(L, u, A->col[k2])) blocked[A->col[k2]] = 1;
    }
  }
  int na = 0;
  L->root = (int *)malloc((size_t)nn * sizeof(int));
  for (int v = 0; v < nn; v++) {
    L->root[v] = root[v];
    if (root[v]) L->agg[v] = na++;
  }
  int *agg3 = (int *)malloc((size_t)nn * sizeof(int));
  for (int v = 0; v < nn; v++) agg3[v] = L->agg[v];
  for (int v = 0; v < nn; v++)
    if (root[v])
      for (int k = A->ptr[v]; k < A->ptr[v + 1]; k++)
        if (edge(L, v, A->col[k])) agg3[A->col[k]] = L->agg[v];
  for (int v = 0; v < nn; v++) L->agg[v] = agg3[v];
  for (int v = 0; v < nn; v++) {
    if (iso[v] || agg3[v] >= 0) continue;
    int best = -1, bestc = 0;
    for (int k = A->ptr[v]; k < A->ptr[v + 1]; k++) {
      if (!edge(L, v, A->col[k])) continue;
      int a = agg3[A->col[k]];
      if (a < 0) continue;
      int c = 0;
      for (int k2 = A->ptr[v]; k2 < A->ptr[v + 1]; k2++)
        if (edge(L, v, A->col[k2]) && agg3[A->col[k2]] == a) c++;
      if (c > bestc || (c == bestc && a < best)) { bestc = c; best = a; }
    }
    if (best < 0) {
      free(iso); free(blocked); free(root); free(ord); free(agg3);
      return fail(ORC_ERR_ARG, "aggregation: leftover node without aggregated neighbour");
    }
    L->agg[v] = best;
  }
  L->n_agg = na;
  free(iso); free(blocked); free(root); free(ord); free(agg3);
  return ORC_OK;
}

/* Tentative prolongator by per-aggregate modified Gram-Schmidt, contract C17. */
static int tentative(level_t *L, level_t *Lc) {
  int nn = L->nodes, b = L->b, na = L->n_agg;
  /* nodes per aggregate, ascending */
  int *cnt = (int *)calloc((size_t)na + 1, sizeof(int));
  for (int v = 0; v < nn; v++)
    if (L->agg[v] >= 0) cnt[L->agg[v] + 1]++;
  for (int a = 0; a < na; a++) cnt[a + 1] += cnt[a];
  int *mem = (int *)malloc((size_t)(cnt[na] > 0 ? cnt[na] : 1) * sizeof(int));
  int *fill = (int *)calloc((size_t)na, sizeof(int));
  for (int v = 0; v < nn; v++)
    if (L->agg[v] >= 0) { int a = L->agg[v]; mem[cnt[a] + fill[a]++] = v; }
  long nnz_pt = 0;
  for (int v = 0; v < nn; v++) nnz_pt += (L->agg[v] >= 0);
  if (bsr_alloc(&L->Pt, nn, na, b, 6, nnz_pt)) return fail(ORC_ERR_OOM, "oom Pt");
  long w = 0;
  for (int v = 0; v < nn; v++) {
    L->Pt.ptr[v] = (int)w;
    if (L->agg[v] >= 0) { L->Pt.col[w] = L->agg[v]; w++; }
  }
  L->Pt.ptr[nn] = (int)w;
  Lc->Bnn = (double *)calloc((size_t)na * 36, sizeof(double));
  for (int a = 0; a < na; a++) {
    int nr = (cnt[a + 1] - cnt[a]) * b;
    double *Q = (double *)malloc((size_t)nr * 6 * sizeof(double)); /* column-major nr x 6 */
    double Rm[36] = {0};
    for (int t = 0; t < cnt[a + 1] - cnt[a]; t++)
      for (int r = 0; r < b; r++)
        for (int j = 0; j < 6; j++)
          Q[(size_t)j * nr + t * b + r] = L->Bnn[((size_t)mem[cnt[a] + t] * b + r) * 6 + j];
    for (int j = 0; j < 6; j++) {
      double *vj = Q + (size_t)j * nr;
      for (int i = 0; i < j; i++) {
        double *qi = Q + (size_t)i * nr;
        double rij = 0.0;
        for (int t = 0; t < nr; t++) rij = fma(qi[t], vj[t], rij);
        Rm[i * 6 + j] = rij;
        for (int t = 0; t < nr; t++) vj[t] = fma(-rij, qi[t], vj[t]);
      }
      double ss = 0.0;
      for (int t = 0; t < nr; t++) ss = fma(vj[t], vj[t], ss);
      double rjj = sqrt(ss);
      if (!(rjj > 0.0) || (j > 0 && !(rjj > 1e-10 * Rm[0]))) {
        free(Q);
        snprintf(g_err, sizeof g_err, "rank-deficient tentative prolongator at aggregate %d (column %d)", a, j);
        return ORC_ERR_RANK;
      }
      Rm[j * 6 + j] = rjj;
      for (int t = 0; t < nr; t++) vj[t] = vj[t] / rjj;
    }
    for (int t = 0; t < cnt[a + 1] - cnt[a]; t++) {
      int v = mem[cnt[a] + t];
      double *blk = L->Pt.val + (size_t)L->Pt.ptr[v] * b * 6;
      for (int r = 0; r < b; r++)
        for (int j = 0; j < 6; j++) blk[r * 6 + j] = Q[(size_t)j * nr + t * b + r];
    }
    memcpy(Lc->Bnn + (size_t)a * 36, Rm, sizeof Rm);
    free(Q);
  }
  free(cnt); free(mem); free(fill);
  return ORC_OK;
}

/* lambda_max(D^{-1} A) by power iteration, contract C18. */
static void power_iter(level_t *L, int iters) {
  long n = L->n;
  double *v = (double *)malloc((size_t)n * sizeof(double));
  double *w = (double *)malloc((size_t)n * sizeof(double));
  for (long i = 0; i < n; i++) v[i] = 1.0 + (double)(i % 7) / 8.0;
  double lam = 0.0;
  for (int it = 0; it < iters; it++) {
    bsr_spmv(&L->A, v, NULL, w, 0);
    for (long i = 0; i < n; i++) w[i] = w[i] / L->dpt[i];
    double nw = sqrt(orc_dot(n, L->b, w, w));
    double nv = sqrt(orc_dot(n, L->b, v, v));
    lam = nw / nv;
    for (long i = 0; i < n; i++) v[i] = w[i] / nw;
  }
  L->lambda = lam;
  L->omega = 4.0 / (3.0 * lam);
  free(v); free(w);
}

static int find_col(const bsr_t *A, int i, int c) {
  int lo = A->ptr[i], hi = A->ptr[i + 1] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (A->col[mid] == c) return mid;
    if (A->col[mid] < c) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* Row-wise Gustavson product C = A * B with per-entry fma chains over
 * (block of A ascending, inner index ascending), contract C20/C21.  The output
 * pattern of row i is the sorted union of B's rows for A's columns in row i. */
static int spgemm(const bsr_t *A, const bsr_t *B, bsr_t *C) {
  int br = A->br, inner = A->bc, bc = B->bc;
  int *mark = (int *)malloc((size_t)(B->nbc > 0 ? B->nbc : 1) * sizeof(int));
  for (int q = 0; q < B->nbc; q++) mark[q] = -1;
  int *list = (int *)malloc((size_t)(B->nbc > 0 ? B->nbc : 1) * sizeof(int));
  int *rl = (int *)calloc((size_t)A->nbr + 1, sizeof(int));
  long total = 0;
  for (int i = 0; i < A->nbr; i++) {
    int u = 0;
    for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
      int j = A->col[k];
      for (int k2 = B->ptr[j]; k2 < B->ptr[j + 1]; k2++) {
        int c = B->col[k2];
        if (mark[c] != i) { mark[c] = i; u++; }
      }
    }
    rl[i] = u;
    total += u;
  }
  if (bsr_alloc(C, A->nbr, B->nbc, br, bc, total)) return fail(ORC_ERR_OOM, "oom spgemm");
  for (int q = 0; q < B->nbc; q++) mark[q] = -1;
  long w = 0;
  for (int i = 0; i < A->nbr; i++) {
    C->ptr[i] = (int)w;
    int u = 0;
    for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
      int j = A->col[k];
      for (int k2 = B->ptr[j]; k2 < B->ptr[j + 1]; k2++) {
        int c = B->col[k2];
        if (mark[c] != i) { mark[c] = i; list[u++] = c; }
      }
    }
    qsort(list, u, sizeof(int), cmp_int);
    for (int q = 0; q < u; q++) C->col[w + q] = list[q];
    /* numeric: entries start at +0 (calloc); walk A's row, then B's row */
    for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
      int j = A->col[k];
      const double *ab = A->val + (size_t)k * br * inner;
      for (int k2 = B->ptr[j]; k2 < B->ptr[j + 1]; k2++) {
        int c = B->col[k2];
        int lo = 0, hi = u - 1, at = -1;
        while (lo <= hi) {
          int mid = (lo + hi) / 2;
          if (list[mid] == c) { at = mid; break; }
          if (list[mid] < c) lo = mid + 1; else hi = mid - 1;
        }
        const double *bb = B->val + (size_t)k2 * inner * bc;
        double *cb = C->val + (size_t)(w + at) * br * bc;
        for (int r = 0; r < br; r++)
          for (int s = 0; s < bc; s++) {
            double acc = cb[r * bc + s];
            for (int t = 0; t < inner; t++) acc = fma(ab[r * inner + t], bb[t * bc + s], acc);
            cb[r * bc + s] = acc;
          }
      }
    }
    w += u;
  }
  C->ptr[A->nbr] = (int)w;
  free(mark); free(list); free(rl);
  return ORC_OK;
}

/* Explicit block transpose (exact). */
static int transpose(const bsr_t *A, bsr_t *T) {
  long nz = bsr_nnzb(A);
  if (bsr_alloc(T, A->nbc, A->nbr, A->bc, A->br, nz)) return fail(ORC_ERR_OOM, "oom transpose");
  int *cnt = T->ptr;
  for (long k = 0; k < nz; k++) cnt[A->col[k] + 1]++;
  for (int c = 0; c < A->nbc; c++) cnt[c + 1] += cnt[c];
  int *fill = (int *)calloc((size_t)A->nbc + 1, sizeof(int));
  for (int i = 0; i < A->nbr; i++)
    for (int k = A->ptr[i]; k < A->ptr[i + 1]; k++) {
      int c = A->col[k];
      long d = cnt[c] + fill[c]++;
      T->col[d] = i;
      for (int r = 0; r < A->br; r++)
        for (int s = 0; s < A->bc; s++)
          T->val[(size_t)d * A->br * A->bc + s * A->br + r] = A->val[(size_t)k * A->br * A->bc + r * A->bc + s];
    }
  free(fill);
  return ORC_OK;
}

/* Smoothed prolongator P = Pt - omega D^{-1} (A Pt), contract C19. */
static int smooth_P(level_t *L) {
  int st = spgemm(&L->A, &L->Pt, &L->P);
  if (st) return st;
  int b = L->b;
  for (int i = 0; i < L->nodes; i++) {
    for (int k = L->P.ptr[i]; k < L->P.ptr[i + 1]; k++) {
      double *blk = L->P.val + (size_t)k * b * 6;
      int a = L->P.col[k];
      const double *q = (L->agg[i] == a) ? L->Pt.val + (size_t)L->Pt.ptr[i] * b * 6 : NULL;
      for (int r = 0; r < b; r++)
        for (int s = 0; s < 6; s++) {
          double t = L->omega * blk[r * 6 + s];
          t = t / L->dpt[(size_t)i * b + r];
          double pt = q ? q[r * 6 + s] : 0.0;
          blk[r * 6 + s] = pt - t;
        }
    }
  }
  return ORC_OK;
}

/* Nodal-block l1 smoother data (variant f4, reading R22; the block form of the l1 smoothers of PAPER.md:589 /
 * Baker et al.): B_i = A_ii + diag(d_i), d_i,r = sum of |a_(i,r),(j,c)| over the off-diagonal blocks j != i of the
 * row (chain d = d + |a| from +0, blocks ascending, columns ascending); B_i = L L^T by the chains of C9 (acc = b_rc;
 * fma(-L_rk, L_ck, acc) for k ascending; L_cc = sqrt(acc); L_rc = acc / L_cc); reciprocals 1/L_rr for the solves
 * (C10).  B - A is block diagonally dominant, so lambda_max(B^{-1} A) <= 1: convergent with weight 1. */
static int block_l1_data(level_t *L) {
  const int b = L->b, nb = b * (b + 1) / 2 + b;
  L->bfac = (double *)malloc((size_t)L->nodes * nb * sizeof(double));
  for (int i = 0; i < L->nodes; i++) {
    double B[36], Lf[36];
    const double *Aii = NULL;
    for (int r = 0; r < b; r++) {
      double d = 0.0;
      for (int k = L->A.ptr[i]; k < L->A.ptr[i + 1]; k++) {
        if (L->A.col[k] == i) { Aii = L->A.val + (size_t)k * b * b; continue; }
        for (int c = 0; c < b; c++) d = d + fabs(L->A.val[(size_t)k * b * b + r * b + c]);
      }
      B[r * b + r] = d;  /* the diagonal sum is completed below, once A_ii is known */
    }
    if (!Aii) return fail(ORC_ERR_NOT_SPD, "block smoother: node without a diagonal block");
    for (int r = 0; r < b; r++)
      for (int c = 0; c < b; c++) B[r * b + c] = (r == c) ? Aii[r * b + r] + B[r * b + r] : Aii[r * b + c];
    for (int c = 0; c < b; c++) {
      double acc = B[c * b + c];
      for (int k = 0; k < c; k++) acc = fma(-Lf[c * b + k], Lf[c * b + k], acc);
      if (!(acc > 0.0)) return fail(ORC_ERR_NOT_SPD, "block smoother: non-positive pivot");
      const double lcc = sqrt(acc);
      Lf[c * b + c] = lcc;
      for (int r = c + 1; r < b; r++) {
        double a = B[r * b + c];
        for (int k = 0; k < c; k++) a = fma(-Lf[r * b + k], Lf[c * b + k], a);
        Lf[r * b + c] = a / lcc;
      }
    }
    double *o = L->bfac + (size_t)i * nb;
    int w = 0;
    for (int r = 0; r < b; r++)
      for (int c = 0; c <= r; c++) o[w++] = Lf[r * b + c];
    for (int r = 0; r < b; r++) o[w++] = 1.0 / Lf[r * b + r];
  }
  return ORC_OK;
}

/* t = B_i^{-1} v_i per node (C10 chains on the node's factor): forward acc = v_r; fma(-L_rk, y_k, acc) k ascending;
 * y_r = acc * (1/L_rr); backward acc = y_r; fma(-L_kr, t_k, acc) k descending; t_r = acc * (1/L_rr). */
static void block_solve(const level_t *L, const double *v, double *t) {
  const int b = L->b, nb = b * (b + 1) / 2 + b;
  for (int i = 0; i < L->nodes; i++) {
    const double *f = L->bfac + (size_t)i * nb, *rinv = f + b * (b + 1) / 2;
    const double *vi = v + (size_t)i * b;
    double y[6], x[6];
    for (int r = 0; r < b; r++) {
      double acc = vi[r];
      for (int k = 0; k < r; k++) acc = fma(-f[r * (r + 1) / 2 + k], y[k], acc);
      y[r] = acc * rinv[r];
    }
    for (int r = b - 1; r >= 0; r--) {
      double acc = y[r];
      for (int k = b - 1; k > r; k--) acc = fma(-f[k * (k + 1) / 2 + r], x[k], acc);
      x[r] = acc * rinv[r];
    }
    for (int r = 0; r < b; r++) t[(size_t)i * b + r] = x[r];
  }
}

static void level_diag(level_t *L) {
  int b = L->b;
  L->dl1 = (double *)malloc((size_t)L->n * sizeof(double));
  L->dpt = (double *)malloc((size_t)L->n * sizeof(double));
  for (int i = 0; i < L->nodes; i++)
    for (int r = 0; r < b; r++) {
      double d = 0.0, dp = 0.0;
      for (int k = L->A.ptr[i]; k < L->A.ptr[i + 1]; k++)
        for (int c = 0; c < b; c++) {
          double a = L->A.val[(size_t)k * b * b + r * b + c];
          d = d + fabs(a);
          if (L->A.col[k] == i && c == r) dp = a;
        }
      L->dl1[(size_t)i * b + r] = d;
      L->dpt[(size_t)i * b + r] = dp;
    }
}

/* Connected components of K's block graph; label = smallest node id. */
static int *k_components(int nodes, const int *Kptr, const int *Kcol) {
  int *comp = (int *)malloc((size_t)nodes * sizeof(int));
  int *stack = (int *)malloc((size_t)nodes * sizeof(int));
  for (int v = 0; v < nodes; v++) comp[v] = -1;
  for (int s0 = 0; s0 < nodes; s0++) {
    if (comp[s0] >= 0) continue;
    int top = 0;
    stack[top++] = s0;
    comp[s0] = s0;
    while (top) {
      int v = stack[--top];
      for (int k = Kptr[v]; k < Kptr[v + 1]; k++) {
        int u = Kcol[k];
        if (comp[u] < 0) { comp[u] = s0; stack[top++] = u; }
      }
    }
  }
  free(stack);
  return comp;
}

static int build_hierarchy(orc_ctx *cx, const double *Bnns, const int *Kptr, const int *Kcol) {
  level_t *L0 = &cx->lev[0];
  L0->comp = k_components(cx->nodes, Kptr, Kcol);
  L0->A = cx->S;               /* level 0 operator shares S's storage */
  L0->b = 3;
  L0->nodes = cx->nodes;
  L0->n = cx->n;
  L0->Bnn = (double *)malloc((size_t)cx->n * 6 * sizeof(double));
  memcpy(L0->Bnn, Bnns, (size_t)cx->n * 6 * sizeof(double));
  int l = 0;
  for (;;) {
    level_t *L = &cx->lev[l];
    level_diag(L);
    if (cx->cfg.smoother == 2) {
      int st2 = block_l1_data(L);
      if (st2) return st2;
    }
    if (L->n <= cx->cfg.coarsest_size || l + 1 >= cx->cfg.max_levels || l + 1 >= MAXLEV) break;
    int st = aggregate(L, cx->cfg.agg_seed);
    if (st) return st;
    if (L->n_agg == 0 || 60L * L->n_agg > 9L * L->n) { free(L->agg); L->agg = NULL; break; }
    level_t *Lc = &cx->lev[l + 1];
    Lc->comp = (int *)malloc((size_t)(L->n_agg > 0 ? L->n_agg : 1) * sizeof(int));
    for (int v = 0; v < L->nodes; v++)
      if (L->agg[v] >= 0) Lc->comp[L->agg[v]] = L->comp[v];
    st = tentative(L, Lc);
    if (st) return st;
    power_iter(L, cx->cfg.power_iters);
    if ((st = smooth_P(L))) return st;
    if ((st = transpose(&L->P, &L->R))) return st;
    bsr_t AP, G;
    memset(&AP, 0, sizeof AP); memset(&G, 0, sizeof G);
    if ((st = spgemm(&L->A, &L->P, &AP))) return st;
    if ((st = spgemm(&L->R, &AP, &G))) return st;
    bsr_free(&AP);
    /* exact symmetrisation A_c = (G + G^T)/2, contract C22 */
    if (bsr_alloc(&Lc->A, G.nbr, G.nbc, 6, 6, bsr_nnzb(&G))) return fail(ORC_ERR_OOM, "oom Ac");
    memcpy(Lc->A.ptr, G.ptr, ((size_t)G.nbr + 1) * sizeof(int));
    memcpy(Lc->A.col, G.col, (size_t)bsr_nnzb(&G) * sizeof(int));
    for (int a = 0; a < G.nbr; a++)
      for (int k = G.ptr[a]; k < G.ptr[a + 1]; k++) {
        int kt = find_col(&G, G.col[k], a);
        if (kt < 0) return fail(ORC_ERR_ARG, "Galerkin pattern not symmetric");
        for (int r = 0; r < 6; r++)
          for (int s = 0; s < 6; s++)
            Lc->A.val[(size_t)k * 36 + r * 6 + s] = 0.5 * (G.val[(size_t)k * 36 + r * 6 + s] + G.val[(size_t)kt * 36 + s * 6 + r]);
      }
    bsr_free(&G);
    Lc->b = 6;
    Lc->nodes = L->n_agg;
    Lc->n = 6L * L->n_agg;
    l++;
  }
  cx->nlev = l + 1;
  /* coarsest: dense Cholesky ("coarsest_factorization") */
  level_t *Lc = &cx->lev[l];
  int nco = (int)Lc->n;
  if (nco > 16384) return fail(ORC_ERR_ARG, "coarsest level too large for a dense factor");
  cx->nco = nco;
  cx->Ac = (double *)calloc((size_t)nco * nco, sizeof(double));
  cx->Lc = (double *)malloc((size_t)nco * nco * sizeof(double));
  int b = Lc->b;
  for (int i = 0; i < Lc->nodes; i++)
    for (int k = Lc->A.ptr[i]; k < Lc->A.ptr[i + 1]; k++)
      for (int r = 0; r < b; r++)
        for (int c = 0; c < b; c++)
          cx->Ac[(size_t)(i * b + r) * nco + Lc->A.col[k] * b + c] = Lc->A.val[(size_t)k * b * b + r * b + c];
  int st = orc_cholesky_dense(nco, cx->Ac, cx->Lc);
  if (st) {
    char buf[512];
    snprintf(buf, sizeof buf, "coarsest: %.480s", g_err);
    return fail(st, buf);
  }
  for (int q = 0; q < cx->nlev; q++)
    for (int t = 0; t < 4; t++) cx->work[q][t] = (double *)calloc((size_t)cx->lev[q].n, sizeof(double));
  return ORC_OK;
}

void orc_free(orc_ctx *cx) {
  if (!cx) return;
  for (int l = 0; l < MAXLEV; l++) {
    level_t *L = &cx->lev[l];
    if (l > 0) bsr_free(&L->A);
    bsr_free(&L->Pt); bsr_free(&L->P); bsr_free(&L->R);
    free(L->dl1); free(L->dpt); free(L->agg); free(L->comp); free(L->root); free(L->Bnn); free(L->bfac);
    for (int t = 0; t < 4; t++) free(cx->work[l][t]);
  }
  bsr_free(&cx->S);
  free(cx->Z); free(cx->pos); free(cx->pi); free(cx->Aw); free(cx->Lw); free(cx->Ac); free(cx->Lc);
  free(cx->Jp); free(cx->Jc); free(cx->Jv); free(cx->Jtp); free(cx->Jtr); free(cx->Jtv);
  free(cx);
}

static int all_finite(const double *x, long n) {
  for (long i = 0; i < n; i++)
    if (!isfinite(x[i])) return 0;
  return 1;
}

orc_ctx *orc_create_box(int nodes, const int *Kptr, const int *Kcol, const double *Kval,
                        int m, const int *Jptr, const int *Jcol, const double *Jval, const double *D,
                        const double *Dlo, const double *Dup,
                        const int *Z, int nc, const double *Bnns, const orc_config *cfg, int *status) {
  g_err[0] = 0;
  if (nodes <= 0 || m < 0 || !Kptr || !Kcol || !Kval || !Bnns || !cfg) {
    *status = fail(ORC_ERR_ARG, "bad arguments");
    return NULL;
  }
  if (!all_finite(Kval, 9L * Kptr[nodes]) || (m > 0 && (!all_finite(Jval, Jptr[m]) || !all_finite(D, m)))) {
    *status = fail(ORC_ERR_NONFINITE, "non-finite entry in K, J or D");
    return NULL;
  }
  for (int k = 0; k < m; k++)
    if (!(D[k] > 0.0)) { *status = fail(ORC_ERR_DOMAIN, "D must be strictly positive"); return NULL; }
  for (int w = 0; w < 2; w++) {
    const double *Db = w ? Dup : Dlo;
    if (!Db) continue;
    if (!all_finite(Db, 3L * nodes)) { *status = fail(ORC_ERR_NONFINITE, "non-finite bound diagonal"); return NULL; }
    for (long p = 0; p < 3L * nodes; p++)
      if (!(Db[p] >= 0.0)) { *status = fail(ORC_ERR_DOMAIN, "bound diagonals must be >= 0"); return NULL; }
  }
  if (cfg->smoother < 0 || cfg->smoother > 2 ||
      (cfg->smoother == 1 && (cfg->cheb_degree < 1 || cfg->cheb_degree > 32 || !(cfg->cheb_ratio > 1.0)))) {
    *status = fail(ORC_ERR_ARG, "bad smoother configuration");
    return NULL;
  }
  orc_ctx *cx = (orc_ctx *)calloc(1, sizeof(orc_ctx));
  cx->cfg = *cfg;
  cx->nodes = nodes;
  cx->n = 3L * nodes;
  cx->m = m;
  double t0 = now_s();
  int st = form_S(cx, Kptr, Kcol, Kval, m, Jptr, Jcol, Jval, D, Dlo, Dup);
  double t1 = now_s();
  cx->t_phase[0] = t1 - t0;
  if (!st) st = setup_filter(cx, m, Jptr, Jcol, Jval, Z, nc);
  double t2 = now_s();
  cx->t_phase[1] = (t2 - t1) - cx->t_phase[2];
  if (!st) st = build_hierarchy(cx, Bnns, Kptr, Kcol);
  cx->t_phase[3] = now_s() - t2;
  *status = st;
  if (st) { cx->lev[0].A.ptr = NULL; cx->lev[0].A.col = NULL; cx->lev[0].A.val = NULL; orc_free(cx); return NULL; }
  return cx;
}

orc_ctx *orc_create(int nodes, const int *Kptr, const int *Kcol, const double *Kval,
                    int m, const int *Jptr, const int *Jcol, const double *Jval, const double *D,
                    const int *Z, int nc, const double *Bnns, const orc_config *cfg, int *status) {
  return orc_create_box(nodes, Kptr, Kcol, Kval, m, Jptr, Jcol, Jval, D, NULL, NULL, Z, nc, Bnns, cfg, status);
}

/* ---------- solve phase ---------- */
/* Chebyshev smoother coefficients (reading R18): degree k polynomial in D_l1^{-1} A on the interval
 * [1/ratio, 1] (lambda_max(D_l1^{-1} A) <= 1 for the l1 diagonal), three-term recurrence
 *   theta = (1 + 1/ratio)/2, delta = (1 - 1/ratio)/2, sigma = theta/delta, rho_0 = 1/sigma,
 *   rho_s = 1/(2 sigma - rho_{s-1}),  a_s = rho_s rho_{s-1},  b_s = 2 rho_s / delta   (s = 1..k-1),
 *   c0 = 1/theta.  The error after one application is T_k((theta - lambda)/delta) / T_k(sigma). */
static void cheb_coefs(int k, double ratio, double *c0, double *a, double *bb) {
  const double theta = (1.0 + 1.0 / ratio) / 2.0, delta = (1.0 - 1.0 / ratio) / 2.0;
  const double sigma = theta / delta;
  double rho = 1.0 / sigma;
  *c0 = 1.0 / theta;
  for (int s = 1; s < k; s++) {
    const double rn = 1.0 / (2.0 * sigma - rho);
    a[s] = rn * rho;
    bb[s] = 2.0 * rn / delta;
    rho = rn;
  }
}
void orc_cheb_coefs(int k, double ratio, double *out) {  /* out = {c0, a_1, b_1, ..., a_{k-1}, b_{k-1}} */
  double a[64], bb[64];
  cheb_coefs(k, ratio, &out[0], a, bb);
  for (int s = 1; s < k; s++) { out[2 * s - 1] = a[s]; out[2 * s] = bb[s]; }
}

/* One Chebyshev application (contract C23): from zero: t = b/d, dir = c0 t, x = dir; else
 * r = b - A x, t = r/d, dir = c0 t, x = x + dir; then for s = 1..k-1: r = b - A x, t = r/d,
 * dir = fma(a_s, dir, b_s t), x = x + dir. */
static void cheb_smooth(orc_ctx *cx, level_t *L, const double *b, double *x, int from_zero, double *r,
                        double *dir) {
  const long n = L->n;
  const int k = cx->cfg.cheb_degree;
  double c0, a[64], bb[64];
  cheb_coefs(k, cx->cfg.cheb_ratio, &c0, a, bb);
  if (from_zero) {
    for (long i = 0; i < n; i++) {
      const double t = b[i] / L->dl1[i];
      dir[i] = c0 * t;
      x[i] = dir[i];
    }
  } else {
    bsr_spmv(&L->A, x, b, r, 1);
    for (long i = 0; i < n; i++) {
      const double t = r[i] / L->dl1[i];
      dir[i] = c0 * t;
      x[i] = x[i] + dir[i];
    }
  }
  for (int s = 1; s < k; s++) {
    bsr_spmv(&L->A, x, b, r, 1);
    for (long i = 0; i < n; i++) {
      const double t = r[i] / L->dl1[i];
      dir[i] = fma(a[s], dir[i], bb[s] * t);
      x[i] = x[i] + dir[i];
    }
  }
}

static void vcycle(orc_ctx *cx, int l, const double *b, double *x) {
  level_t *L = &cx->lev[l];
  long n = L->n;
  if (l == cx->nlev - 1) {
    orc_trsv_dense(cx->nco, cx->Lc, b, x);
    return;
  }
  double *r = cx->work[l][0];
  double *bc = cx->work[l + 1][1];
  double *xc = cx->work[l + 1][2];
  double *xn = cx->work[l][3];
  const int cheb = cx->cfg.smoother == 1;
  if (cx->cfg.smoother == 2) {
    /* nodal-block l1 smoother (C25): from zero x = B^{-1} b; a sweep x_i = x_i + (B^{-1} (b - A x))_i */
    block_solve(L, b, x);
    for (int s = 1; s < cx->cfg.pre_sweeps; s++) {
      bsr_spmv(&L->A, x, b, r, 1);
      block_solve(L, r, xn);
      for (long i = 0; i < n; i++) x[i] = x[i] + xn[i];
    }
    bsr_spmv(&L->A, x, b, r, 1);
    bsr_spmv_warp32(&L->R, r, bc);
    vcycle(cx, l + 1, bc, xc);
    bsr_spmv(&L->P, xc, NULL, xn, 0);
    for (long i = 0; i < n; i++) x[i] = x[i] + xn[i];
    for (int s = 0; s < cx->cfg.post_sweeps; s++) {
      bsr_spmv(&L->A, x, b, r, 1);
      block_solve(L, r, xn);
      for (long i = 0; i < n; i++) x[i] = x[i] + xn[i];
    }
    return;
  }
  if (cheb) {  /* pre-smoothing, Chebyshev (C23) */
    for (int s = 0; s < cx->cfg.pre_sweeps; s++) cheb_smooth(cx, L, b, x, s == 0, r, xn);
  } else {
    /* pre-smoothing, l1-Jacobi (contract C4) */
    for (long i = 0; i < n; i++) x[i] = b[i] / L->dl1[i];
    for (int s = 1; s < cx->cfg.pre_sweeps; s++) {
      bsr_spmv(&L->A, x, b, r, 1);
      for (long i = 0; i < n; i++) xn[i] = x[i] + r[i] / L->dl1[i];
      memcpy(x, xn, (size_t)n * sizeof(double));
    }
  }
  bsr_spmv(&L->A, x, b, r, 1);          /* r = b - A x            */
  bsr_spmv_warp32(&L->R, r, bc);        /* b_c = R r   (C5)       */
  vcycle(cx, l + 1, bc, xc);            /* x_c = B_{l+1} b_c      */
  bsr_spmv(&L->P, xc, NULL, xn, 0);     /* x += P x_c  (C6)       */
  for (long i = 0; i < n; i++) x[i] = x[i] + xn[i];
  if (cheb) {
    for (int s = 0; s < cx->cfg.post_sweeps; s++) cheb_smooth(cx, L, b, x, 0, r, xn);
    return;
  }
  for (int s = 0; s < cx->cfg.post_sweeps; s++) {
    bsr_spmv(&L->A, x, b, r, 1);
    for (long i = 0; i < n; i++) xn[i] = x[i] + r[i] / L->dl1[i];
    memcpy(x, xn, (size_t)n * sizeof(double));
  }
}

void orc_vcycle(orc_ctx *cx, const double *b, double *x) { vcycle(cx, 0, b, x); }

void orc_spmv(orc_ctx *cx, int level, const double *x, double *y) {
  bsr_spmv(&cx->lev[level].A, x, NULL, y, 0);
}

/* y = A_w^{-1} v (filter solve, contract C10): A_w[pi,pi] = L L^T, so y[pi] = L^{-T} L^{-1} v[pi]. */
static void filter_solve(orc_ctx *cx, const double *v, double *y) {
  int nc = cx->nf;
  double *vp = (double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
  double *yp = (double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
  for (int i = 0; i < nc; i++) vp[i] = v[cx->pi[i]];
  orc_trsv_dense(nc, cx->Lw, vp, yp);
  for (int i = 0; i < nc; i++) y[cx->pi[i]] = yp[i];
  free(vp); free(yp);
}
void orc_filter_solve(orc_ctx *cx, const double *v, double *y) { filter_solve(cx, v, y); }

/* AMGF apply (Def. AMGF eq:M_itmat PAPER.md:426; three stages SPEC.md:245,
 * thin second residual = reading R11):
 *   x1 = B r; r1 = r - S x1; y = A_w^{-1} r1[Z]; x2 = x1 + P y;
 *   r2 = r1 - S[:,Z] y; z = x2 + B r2. */
void orc_apply(orc_ctx *cx, const double *r, double *z) {
  long n = cx->n;
  int nc = cx->nc;
  double *x1 = (double *)malloc((size_t)n * sizeof(double));
  double *r1 = (double *)malloc((size_t)n * sizeof(double));
  double *xv = (double *)malloc((size_t)n * sizeof(double));
  double *v = (double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
  double *y = (double *)malloc((size_t)(nc > 0 ? nc : 1) * sizeof(double));
  vcycle(cx, 0, r, x1);
  bsr_spmv(&cx->S, x1, r, r1, 1);
  if (cx->cfg.filter_basis == 1) {
    /* P = J^T (reading R21): v = J r1 (row chains); y = (J S J^T)^{-1} v; w = J^T y per dof (chains over the
     * dof's constraints ascending), held at the Z positions for the x2 update and the thin residual */
    const int m = cx->mJ;
    double *vJ = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    double *yJ = (double *)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    for (int a = 0; a < m; a++) {
      double acc = 0.0;
      for (int e = cx->Jp[a]; e < cx->Jp[a + 1]; e++) acc = fma(cx->Jv[e], r1[cx->Jc[e]], acc);
      vJ[a] = acc;
    }
    if (m > 0) filter_solve(cx, vJ, yJ);
    for (int a = 0; a < nc; a++) {
      const int p = cx->Z[a];
      double acc = 0.0;
      for (int t = cx->Jtp[p]; t < cx->Jtp[p + 1]; t++) acc = fma(cx->Jtv[t], yJ[cx->Jtr[t]], acc);
      y[a] = acc;
    }
    free(vJ); free(yJ);
  } else {
    for (int a = 0; a < nc; a++) v[a] = r1[cx->Z[a]];
    if (nc > 0) filter_solve(cx, v, y);
  }
  /* x2 (stored in x1) and thin r2 (stored in r1) */
  const bsr_t *S = &cx->S;
  for (int I = 0; I < cx->nodes; I++)
    for (int r_ = 0; r_ < 3; r_++) {
      double acc = 0.0;
      int hit = 0;
      for (int k = S->ptr[I]; k < S->ptr[I + 1]; k++)
        for (int c = 0; c < 3; c++) {
          int q = 3 * S->col[k] + c;
          if (cx->pos[q] >= 0) {
            acc = fma(S->val[9L * k + 3 * r_ + c], y[cx->pos[q]], acc);
            hit = 1;
          }
        }
      if (hit) r1[3L * I + r_] = r1[3L * I + r_] - acc;
    }
  for (int a = 0; a < nc; a++) x1[cx->Z[a]] = x1[cx->Z[a]] + y[a];
  vcycle(cx, 0, r1, xv);
  for (long i = 0; i < n; i++) z[i] = x1[i] + xv[i];
  free(x1); free(r1); free(xv); free(v); free(y);
}

/* B-only apply (AMG-PCG baseline) */
static void apply_B(orc_ctx *cx, const double *r, double *z) { vcycle(cx, 0, r, z); }

/* PCG, contract C15.
 * precond: 0 = AMGF (M), 1 = AMG V-cycle only (B). hist (optional, >= maxit+1). */
int orc_pcg(orc_ctx *cx, const double *b, double *x, double rtol, int maxit, int precond,
            int *iters, double *relres, double *hist) {
  long n = cx->n;
  double *r = (double *)malloc((size_t)n * sizeof(double));
  double *z = (double *)malloc((size_t)n * sizeof(double));
  double *p = (double *)malloc((size_t)n * sizeof(double));
  double *q = (double *)malloc((size_t)n * sizeof(double));
  int st = ORC_NOT_CONVERGED;
  for (long i = 0; i < n; i++) { x[i] = 0.0; r[i] = b[i]; }
  *iters = 0;
  *relres = 0.0;
  if (precond) apply_B(cx, r, z); else orc_apply(cx, r, z);
  double rho0 = orc_dot(n, 3, r, z);
  if (hist) hist[0] = 1.0;
  if (rho0 == 0.0) { st = ORC_OK; goto done; }
  if (!(rho0 > 0.0)) { st = fail(ORC_ERR_BREAKDOWN, "PCG: r.Mr <= 0"); goto done; }
  double rho = rho0;
  memcpy(p, z, (size_t)n * sizeof(double));
  for (int it = 1; it <= maxit; it++) {
    bsr_spmv(&cx->S, p, NULL, q, 0);
    double pi = orc_dot(n, 3, p, q);
    if (!(pi > 0.0)) { st = fail(ORC_ERR_BREAKDOWN, "PCG: p.Sp <= 0"); break; }
    double alpha = rho / pi;
    for (long i = 0; i < n; i++) {
      x[i] = fma(alpha, p[i], x[i]);
      r[i] = fma(-alpha, q[i], r[i]);
    }
    if (precond) apply_B(cx, r, z); else orc_apply(cx, r, z);
    double rho1 = orc_dot(n, 3, r, z);
    *iters = it;
    if (rho1 < 0.0) { st = fail(ORC_ERR_BREAKDOWN, "PCG: r.Mr < 0"); break; }
    double rel = sqrt(rho1 / rho0);
    *relres = rel;
    if (hist) hist[it] = rel;
    if (rel < rtol) { st = ORC_OK; break; }
    double beta = rho1 / rho;
    for (long i = 0; i < n; i++) p[i] = fma(beta, p[i], z[i]);
    rho = rho1;
  }
done:
  free(r); free(z); free(p); free(q);
  return st;
}

/* ---------- introspection for tests ---------- */
/* info: [nlev, nc, nco, then per level: nodes, b, nnzb(A), nnzb(P), n_agg] */
void orc_info(orc_ctx *cx, long *out) {
  out[0] = cx->nlev; out[1] = cx->nc; out[2] = cx->nco;
  for (int l = 0; l < cx->nlev; l++) {
    level_t *L = &cx->lev[l];
    out[3 + 5 * l + 0] = L->nodes;
    out[3 + 5 * l + 1] = L->b;
    out[3 + 5 * l + 2] = bsr_nnzb(&L->A);
    out[3 + 5 * l + 3] = (l < cx->nlev - 1) ? bsr_nnzb(&L->P) : 0;
    out[3 + 5 * l + 4] = (l < cx->nlev - 1) ? L->n_agg : 0;
  }
}

int orc_nf(orc_ctx *cx) { return cx->nf; }

/* Phase wall times (s) of orc_create: {S, A_w assembly, A_w dense Cholesky, AMG hierarchy}. */
void orc_times(orc_ctx *cx, double *out) { memcpy(out, cx->t_phase, sizeof cx->t_phase); }

/* which: 0 A.ptr 1 A.col 2 A.val 3 P.ptr 4 P.col 5 P.val 6 R.ptr 7 R.col 8 R.val
 *        9 dl1 10 agg 11 Bnn 12 [lambda, omega] 13 Pt.val 14 root 15 comp
 *        20 Z 21 Aw(dense, Z order) 22 Lw(dense, pi order) 23 Ac(dense) 24 Lc(dense) 25 pi 26 bw */
int orc_get(orc_ctx *cx, int which, int level, void *dst) {
  level_t *L = &cx->lev[level];
  long nzA = bsr_nnzb(&L->A);
  switch (which) {
    case 0: memcpy(dst, L->A.ptr, ((size_t)L->nodes + 1) * sizeof(int)); return 0;
    case 1: memcpy(dst, L->A.col, (size_t)nzA * sizeof(int)); return 0;
    case 2: memcpy(dst, L->A.val, (size_t)nzA * L->b * L->b * sizeof(double)); return 0;
    case 3: memcpy(dst, L->P.ptr, ((size_t)L->nodes + 1) * sizeof(int)); return 0;
    case 4: memcpy(dst, L->P.col, (size_t)bsr_nnzb(&L->P) * sizeof(int)); return 0;
    case 5: memcpy(dst, L->P.val, (size_t)bsr_nnzb(&L->P) * L->b * 6 * sizeof(double)); return 0;
    case 6: memcpy(dst, L->R.ptr, ((size_t)L->n_agg + 1) * sizeof(int)); return 0;
    case 7: memcpy(dst, L->R.col, (size_t)bsr_nnzb(&L->R) * sizeof(int)); return 0;
    case 8: memcpy(dst, L->R.val, (size_t)bsr_nnzb(&L->R) * L->b * 6 * sizeof(double)); return 0;
    case 9: memcpy(dst, L->dl1, (size_t)L->n * sizeof(double)); return 0;
    case 10: memcpy(dst, L->agg, (size_t)L->nodes * sizeof(int)); return 0;
    case 11: memcpy(dst, L->Bnn, (size_t)L->n * 6 * sizeof(double)); return 0;
    case 12: ((double *)dst)[0] = L->lambda; ((double *)dst)[1] = L->omega; return 0;
    case 13: memcpy(dst, L->Pt.val, (size_t)bsr_nnzb(&L->Pt) * L->b * 6 * sizeof(double)); return 0;
    case 14: if (!L->root) return -1; memcpy(dst, L->root, (size_t)L->nodes * sizeof(int)); return 0;
    case 15: memcpy(dst, L->comp, (size_t)L->nodes * sizeof(int)); return 0;
    case 16: if (!L->bfac) return -1;
      memcpy(dst, L->bfac, (size_t)L->nodes * (L->b * (L->b + 1) / 2 + L->b) * sizeof(double)); return 0;
    case 20: memcpy(dst, cx->Z, (size_t)cx->nc * sizeof(int)); return 0;
    case 21: if (!cx->Aw) return -1; memcpy(dst, cx->Aw, (size_t)cx->nf * cx->nf * sizeof(double)); return 0;
    case 22: if (!cx->Lw) return -1; memcpy(dst, cx->Lw, (size_t)cx->nf * cx->nf * sizeof(double)); return 0;
    case 23: memcpy(dst, cx->Ac, (size_t)cx->nco * cx->nco * sizeof(double)); return 0;
    case 24: memcpy(dst, cx->Lc, (size_t)cx->nco * cx->nco * sizeof(double)); return 0;
    case 25: memcpy(dst, cx->pi, (size_t)cx->nf * sizeof(int)); return 0;
    case 26: ((int *)dst)[0] = cx->bw; return 0;
  }
  return -1;
}

/* Raw BSR SpMV (contract C2) for golden/pin tests on hand-written matrices. */
void orc_bsr_spmv(int nbr, int nbc, int br, int bc, int *ptr, int *col, double *val,
                  const double *x, double *y) {
  bsr_t A = {nbr, nbc, br, bc, ptr, col, val};
  bsr_spmv(&A, x, NULL, y, 0);
}
