// common.cuh -- shared declarations of libamgf.so (B200 / sm_100a, fp64).
//
// Arithmetic contract: DESIGN.md section 3.  Every kernel in this library is compiled with
// --fmad=false, so a fused multiply-add happens only where __fma_rn is written.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>
#include <vector>

#include "../../include/amgf.h"

namespace amgf {

constexpr int MAXLEV = 32;
constexpr int CTA = 256;  // CTA size of all row kernels; fixes the dot contract C14 level 1

// ------------------------------------------------------------------ errors
struct Error {
  amgf_status code;
  std::string msg;
};
void set_error(const std::string &m);
const char *get_error();

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess)                                                                       \
      throw ::amgf::Error{AMGF_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};       \
  } while (0)

#define REQUIRE(cond, code, m)                      \
  do {                                              \
    if (!(cond)) throw ::amgf::Error{(code), (m)};  \
  } while (0)

// device error flag codes (first error wins)
enum DevErr { DERR_NONE = 0, DERR_NONFINITE = 1, DERR_DOMAIN = 2, DERR_NOT_SPD = 3, DERR_RANK = 4,
              DERR_ARG = 5, DERR_LIMIT = 6, DERR_BREAKDOWN = 7 };

__device__ __forceinline__ void raise_err(int *flag, int code, int info) {
  if (atomicCAS(flag, 0, code) == 0) flag[1] = info;
}

// ------------------------------------------------------------------ storage
// Block-CSR matrix on the device: nbr block rows of br x bc row-major blocks.
struct Bsr {
  int nbr = 0, nbc = 0, br = 0, bc = 0;
  long nnzb = 0;
  int *ptr = nullptr, *col = nullptr;
  double *val = nullptr;
  // level-0 restriction only: val regrouped per row into groups of 32 consecutive blocks (the blocks one
  // warp step of k_restrict reads), component-major inside a group: block gb + l, component q at
  // ival[gb * bs + q * gs + l] with gs = min(32, row end - gb), bs = br * bc; every load instruction of the
  // warp is then one contiguous segment (C5's order is unchanged)
  double *ival = nullptr;
};

// SELL-32 block matrix: slices of 32 consecutive block rows; slot s of a slice holds the s-th block
// of each of its 32 rows, components interleaved so that one block component of the 32 rows is one
// contiguous 256-byte segment:  col[slot*32 + lane],  val[(slot*BB + e)*32 + lane].
struct Sell {
  int nrows = 0, nslices = 0, br = 0, bc = 0;
  long nslots = 0;
  int *slice_ptr = nullptr;  // [nslices+1] first slot of each slice
  int *rowlen = nullptr;     // [nrows]
  int *col = nullptr;        // [nslots*32]
  double *val = nullptr;     // [nslots*br*bc*32]
  int *src = nullptr;        // [nslots*32] index of the source BSR block (-1 padding) for refresh
  int *perm = nullptr;       // [nrows] or null: SELL row i holds matrix row perm[i] (rows sorted by length
                             // within windows to remove slot padding; prolongators and large coarse levels)
};

struct Level {
  int b = 3, nodes = 0;
  long n = 0;
  Bsr A;          // operator (level 0: S)
  Sell As;        // A in SELL-32 for the solve
  double *dl1 = nullptr, *dpt = nullptr;
  double *bfac = nullptr;  // smoother 2: per-node block factors (C24)
  int *agg = nullptr, *comp = nullptr, *root = nullptr;
  int n_agg = 0;
  Bsr Pt, P, R;   // tentative / smoothed prolongator (b x 6), restriction (6 x b)
  Sell Ps;        // P in SELL-32 for prolongation
  Bsr AP;         // A*P (b x 6), kept for numeric re-setup
  int *agg_ptr = nullptr, *agg_nodes = nullptr;  // nodes of each aggregate, ascending
  double *Bnn = nullptr;   // near-null space [n x 6]
  double lambda = 0, omega = 0;
  // solve workspace
  double *x = nullptr, *x2 = nullptr, *bv = nullptr, *r = nullptr;
  double *dir = nullptr;  // Chebyshev direction (smoother 1)
};

// Device scalars of PCG (C15) and dot results.
struct Scalars {
  double rho0, rho, pi, alpha, beta, rho1, dot, pad;
};
// Device-side PCG loop control (api.cu, k_pcg_control): the whole iteration loop is one CUDA graph with a
// conditional WHILE node; the convergence test runs on the device with the host's formula.
struct LoopState {
  int it, max_it, stop, cap;
  double rtol, rel;
  double *hist;  // [2 * cap]: alpha_k, beta_k of iteration k (PCG history, amgf_pcg_history)
};

struct Ctx {
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;        // A_w factorization overlaps the hierarchy's numeric setup
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int fork_at = -1;                   // numeric re-setup: where the A_w factorization forks (-1: not in update_D)
  // filter overlap (apply_M): the A_w solve runs on fstream (high priority) while the full residual
  // SpMV runs on the main stream; rz = r1 at the Z rows in pi order, computed first by k_resid_dofs
  cudaStream_t fstream = nullptr;
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr;
  double *rz = nullptr;
  double *nd_arena = nullptr;  // filter solve data (filter.cu) in one range
  size_t nd_arena_bytes = 0;
  int resid_sms = 0;
  cudaEvent_t ph_ev[8] = {};  // numeric re-setup phase events (setup.cu)
  double setup_ms[5] = {};    // last numeric re-setup: total, S, hierarchy, coarsest, A_w factor (side)
  double cheb_c0 = 0.0, cheb_a[33] = {}, cheb_b[33] = {};  // Chebyshev coefficients (C23)           // SMs of the residual SpMV that runs beside the A_w solve
  amgf_config cfg;
  int nodes = 0, m = 0;
  long n = 0;
  // inputs kept for update_D
  Bsr K;
  int *J_ptr = nullptr, *J_col = nullptr;
  double *J_val = nullptr;
  int nnzJ = 0;
  int *Jt_ptr = nullptr, *Jt_row = nullptr;  // J^T (per dof: constraint rows ascending)
  double *Jt_val = nullptr;
  double *D = nullptr;
  double *D_lo = nullptr, *D_up = nullptr;  // bound-constraint diagonals of A~ (n each; has_box: in use)
  bool has_box = false;
  int *S_kblk = nullptr;  // per S block: index of the K block (-1 if none)
  // filter (A_w factor in nested-dissection order, filter.cu)
  struct NdLevel { int count = 0, ngroups = 0; int *ids = nullptr, *p0 = nullptr, *len = nullptr, *sub_ptr = nullptr, *sub_list = nullptr, *groups = nullptr, *selfpairs = nullptr; };
  int nd_nblocks = 0, nd_nleaves = 0, nd_depth = 0, nd_npairs = 0, nd_nsep = 0, nd_maxsep = 0;
  int *nd_sep_blocks = nullptr;
  void *nd_blk = nullptr;                 // device NdBlk[nd_nblocks]
  int *nd_leaf_p0 = nullptr, *nd_leaf_len = nullptr, *nd_pairs = nullptr;
  NdLevel nd_lev[16];                     // separators by depth (0 = root)
  int *nd_sspairs[16][16] = {};           // (S at level l, S' at depth d) pairs
  int nd_sspairs_n[16][16] = {};
  int *pi_z = nullptr, *zpi = nullptr, *dof = nullptr, *block_of = nullptr;
  double *Loff = nullptr;                 // separator rows, row-major (factorization)
  double *fw2 = nullptr;                  // forward results shifted by one position (TMA alignment)
  long loff_size = 0;
  double *fw = nullptr;                   // filter workspace (pi order)
  int nc = 0, bw = 0;
  int nf = 0;                // filter-space dimension: nc (filter_basis 0) or m (filter_basis 1, P = J^T)
  double *fJv = nullptr;     // filter_basis 1: v = J r1 (elimination order, nf) and w = J^T y (Z order, nc)
  double *fJw = nullptr;
  int *Z = nullptr, *pos = nullptr;
  double *Lrow = nullptr;   // band, row-major: Lrow[i*W + bw - (i-k)] = L_ik, W = band_stride(bw)
  double *Lcol = nullptr;   // band, column-major: Lcol[k*W + (i-k)] = L_ik
  double *Lrev = nullptr;   // band, reversed rows: Lrev[i*W + (i-k)] = L_ik
  double *Ldinv = nullptr;  // 1/L_ii
  double *fv = nullptr;     // filter workspace (nc)
  int nthin = 0;
  int *thin_row = nullptr, *thin_ptr = nullptr, *thin_pos = nullptr, *thin_src = nullptr;
  double *thin_val = nullptr;
  // the fine rows S[dof[p], :] of the n_c filter dofs (elimination order) in a compact copy for the Z-row
  // residual (k_resid_dofs): block columns and the row's 3 values per block, in the row's block order
  int *zr_ptr = nullptr, *zr_col = nullptr, *zr_src = nullptr;
  double *zr_val = nullptr;
  long zr_nnz = 0;
  // hierarchy
  int nlev = 0;
  Level lev[MAXLEV];
  int nco = 0;
  // fused coarse tail (tail.cu): the V-cycle below level tail_level in one thread-block cluster
  int tail_level = -1, tail_ncta = 0, tail_xs = 0, tail_maxv = 0, tail_maxc = 0, tail_maxpv = 0, tail_maxpc = 0;
  size_t tail_smem = 0;
  int *tail_cta_s = nullptr;
  double *Lc_row = nullptr, *Lc_col = nullptr, *Lc_rev = nullptr, *Lc_dinv = nullptr;
  // solve workspace
  double *w_x1 = nullptr, *w_r1 = nullptr, *w_xv = nullptr;
  double *p = nullptr, *q = nullptr, *rr = nullptr, *zz = nullptr, *xx = nullptr, *bb = nullptr;
  double *dot_part = nullptr;
  double *pw_v = nullptr, *pw_w = nullptr;  // power-iteration work vectors (allocated once)
  double *pw_s = nullptr;                    // power-iteration scalars {w.w, v.v, lambda}
  double *pw_part = nullptr;                 // power-iteration C14 partials of v.v (w.w go to dot_part)
  double *pw_lev = nullptr;                  // per level {lambda, omega} on the device
  Scalars *sc = nullptr;      // device
  Scalars *sc_host = nullptr; // pinned
  int *err = nullptr;         // device [2]
  int *err_host = nullptr;    // pinned [2]
  int64_t launches = 0;
  void *setup_cache = nullptr;  // numeric re-setup data (setup.cu)
  // PCG iteration body captured once per preconditioner (0 AMGF, 1 AMG) and replayed as one graph launch
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t pcg_graph[2] = {nullptr, nullptr};
  cudaGraphExec_t pcg_loop[2] = {nullptr, nullptr};  // device-side loop (conditional WHILE node)
  bool pcg_loop_tried[2] = {false, false};
  LoopState *loop = nullptr, *loop_host = nullptr;
  double *hist = nullptr;  // device PCG coefficient history, capacity hist_cap iterations
  int hist_cap = 0, hist_n = 0;
  std::vector<double> host_hist;  // same, host-loop fallback
  int64_t graph_launches[2] = {0, 0};
  bool capturing = false;
  bool imported = false;      // built by amgf_import: no K, J, D (amgf_update_D unavailable)
  double last_setup_ms = 0;   // amgf_setup / amgf_import wall time or the last amgf_update_D device time
  std::vector<void *> allocs;

  // Debug guard zones (environment AMGF_GUARD=1): every allocation is followed by kGuardBytes of a fixed byte
  // pattern; guard_violations() counts the zones a kernel wrote into (out-of-bounds writes), see
  // amgf_debug_guard_check.  compute-sanitizer is not available on this pool, so this is the library's own
  // bounds check, used by tests/test_gpu_parity.py::test_guard_zones on every code path of a small solve.
  static constexpr size_t kGuardBytes = 4096;
  static constexpr unsigned char kGuardByte = 0xA5;
  std::vector<std::pair<void *, size_t>> guards;  // (allocation, payload bytes)
  static bool guard_enabled();

  template <class T>
  T *alloc(size_t count) {
    void *p = nullptr;
    if (count == 0) count = 1;
    const size_t bytes = count * sizeof(T), extra = guard_enabled() ? kGuardBytes : 0;
    cudaError_t e = cudaMalloc(&p, bytes + extra);
    if (e != cudaSuccess) throw Error{AMGF_ERR_OOM, "cudaMalloc " + std::to_string(bytes) + " bytes"};
    allocs.push_back(p);
    if (extra) {
      cudaMemset((char *)p + bytes, kGuardByte, extra);
      guards.emplace_back(p, bytes);
    }
    return (T *)p;
  }
  long guard_violations();
  void release(void *p);
  ~Ctx();
};

inline int nblk(long n, int t = CTA) { return (int)((n + t - 1) / t); }

// Launch with programmatic dependent launch (PDL) on c.stream: the kernel may start while the previous
// kernel of the stream is finishing; it must call pdl_wait() (devutil.cuh) before reading that kernel's
// results.  Used for the chain of small latency-bound kernels of the A_w solve.
template <typename... KArgs, typename... Args>
inline void launch_pdl(cudaStream_t st, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
  if (e != cudaSuccess) throw Error{AMGF_ERR_CUDA, std::string("cudaLaunchKernelEx (PDL): ") + cudaGetErrorString(e)};
}

// One-time per-DEVICE state of a kernel (function attributes, __constant__ setup): cudaFuncSetAttribute and
// cudaMemcpyToSymbol act on the current device only, so a process-wide static guard would skip them for a
// second device.  Returns the slot of (current device, key), 0 before its first use; thread-safe.
size_t &device_slot(const void *key);

// Post-launch bookkeeping: count the launch, surface launch errors; with AMGF_DEBUG_SYNC=1 in the
// environment also synchronise and name the kernel that faulted.
bool debug_sync();
void after_launch(Ctx &c, const char *name);
void timeline_begin(Ctx &c);                       // AMGF_LAUNCH_TIMELINE diagnostic (api.cu)
void timeline_dump(Ctx &c, cudaEvent_t origin);

// check the device error flag (synchronises the stream)
void check_dev_error(Ctx &c, const char *where);

// ------------------------------------------------------------------ solve kernels (solve.cu)
enum SpmvMode { SPMV_Y = 0, SPMV_RESID = 1, SPMV_SMOOTH = 2, SPMV_DOT = 3, SPMV_SMOOTH_ADD = 4, SPMV_CHEB1 = 6,
                SPMV_CHEB = 7, SPMV_YDIV = 9, SPMV_POW = 10 };
// power step (C18): w = (A v) / d; the fine level (3x3 SELL, one thread per block row = the C14 level-1
// mapping) also forms the C14 level-1 partials of w.w into part_w and of v.v into part_v
void launch_sell_pow(Ctx &c, const Sell &A, const double *v, const double *d, double *w, double *part_w,
                     double *part_v);
struct ChebArgs {  // Chebyshev step of the SpMV epilogue (solve.cu, contract C23)
  double ca = 0.0, cb = 0.0;
  double *dir = nullptr;
  const double *dot_r = nullptr;  // fused dot(dot_r, y) partials (C14 level 1) into dot_part, or null
  double *dot_part = nullptr;
};
void launch_sell_cheb(Ctx &c, const Sell &A, bool first, const double *x, const double *b, const double *dl1,
                      double *dir, double ca, double cb, const double *add, double *y, const double *dot_r = nullptr);
void launch_axpy2_cheb0(Ctx &c, long n, const double *p, const double *q, double *x, double *r, const double *d,
                        double c0, double *dir, double *xs);
void launch_cheb0(Ctx &c, long n, const double *b, const double *d, double c0, double *dir, double *x);
void launch_sell_spmv(Ctx &c, const Sell &A, int mode, const double *x, const double *b, const double *d,
                      const double *add, double *y, double *dot_part);
void launch_jacobi0(Ctx &c, long n, const double *b, const double *d, double *x);
// smoother 2 (C25): out = [add +] (x_in + B^{-1} v) per node, or B^{-1} v when x_in is null (start from zero)
void launch_block_smooth(Ctx &c, const Level &L, const double *v, const double *x_in, const double *add, double *out);
void launch_restrict(Ctx &c, const Bsr &R, const double *r, double *bc);
void launch_prolong(Ctx &c, const Sell &P, const double *xc, double *x);
void launch_dot(Ctx &c, long n, int b, const double *u, const double *v, int finish);
void launch_dot_finish(Ctx &c, long n_partials, int finish);  // C14 level 2 over c.dot_part
// power step (C18): C14 level-1 partials of w.w and v.v (block rows of b), and both level-2 sums into pw[0..1]
void launch_pow_dots(Ctx &c, long nb, int b, const double *w, const double *v, double *part_w, double *part_v);
void launch_pow_fin(Ctx &c, long n_partials, const double *part_w, const double *part_v, double *pw);
void launch_pow_fin_scale(Ctx &c, long n_partials, const double *part_w, const double *part_v, double *pw, long n,
                          const double *w, double *v);
void launch_axpy2(Ctx &c, long n, const double *p, const double *q, double *x, double *r);
void launch_xpby(Ctx &c, long n, const double *z, double *p);
// y = L^{-T} L^{-1} v[gather] (C10); if scatter: xout[scatter[a]] += y[a].  Band storage (row stride
// W = band_stride(bw)): Lcol[j*W + t] = L_{j+t,j}, Lrev[k*W + d] = L_{k,k-d}; zero outside the band.
void launch_band_trsv(Ctx &c, int n, int bw, const double *Lcol, const double *Lrev, const double *dinv,
                      const double *v, const int *gather, double *y, const int *scatter, double *xout,
                      double *work);
// Band storage row stride: 32*R (R = window registers per lane of the warp TRSV, zero padded so that a
// round of 32 band columns is one contiguous TMA bulk copy); wider bands use the fallback kernel.
__host__ __device__ inline int band_R(int bw) { return (bw + 31) / 32 + 1; }
__host__ __device__ inline int band_stride(int bw) { return band_R(bw) <= 8 ? 32 * band_R(bw) : ((bw + 2) & ~1); }
constexpr int BAND_PAD_ROWS = 64;
void launch_thin_resid(Ctx &c, int nthin, const int *rows, const int *ptr, const int *pos, const double *val,
                       const double *y, double *r, int nsc = 0, const int *sdof = nullptr, double *x2 = nullptr);
void launch_bsr_spmv(Ctx &c, const Bsr &A, const double *x, double *y);  // setup-side, thread per block row
void launch_copy(Ctx &c, long n, const double *src, double *dst);
void launch_zero(Ctx &c, long n, double *dst);
void launch_add(Ctx &c, long n, const double *a, const double *b, double *out);
// dot finishing kinds
enum DotFinish { DOT_PLAIN = 0, DOT_PI = 1, DOT_RHO0 = 2, DOT_RHO1 = 3 };

// ------------------------------------------------------------------ setup (setup.cu)
void setup_all(Ctx &c, const int *K_ptr, const int *K_col, const double *K_val, const int *J_ptr,
               const int *J_col, const double *J_val, const double *D, const int *Z, int nc,
               const double *B_nns);
void setup_numeric(Ctx &c, const double *D, const double *D_lo = nullptr,
                   const double *D_up = nullptr);  // update_D (+ bound-constraint diagonals)
// filter.cu
void nd_symbolic(Ctx &c);
void nd_numeric(Ctx &c);
void nd_solve(Ctx &c, const double *r1, const int *gather);  // c.fv <- A_w^{-1} r1 (pi order; r1[gather[p]])
void launch_resid_partition(Ctx &c, const Sell &A, const double *x, const double *b, double *y, int nsm,
                            size_t reserve);
void launch_resid_dofs(Ctx &c, int n, const int *dof, const double *x, const double *b, double *out);
void nd_remap_positions(Ctx &c, int *pos_z, long n);  // Z positions -> pi positions
int band_width_J(Ctx &c);                              // filter_basis 1: band width of J S J^T
// filter_basis 1: v_pi = J r1 (rz: r1 at the Z positions) if v_pi, else w_z = J^T y_pi
void filter_J_apply(Ctx &c, const double *rz, double *v_pi, const double *y_pi, double *w_z);
void band_factor_blocks(Ctx &c, int n, int nblocks, const int *d_p0, const int *d_len, int bw, double *Lrow, int tag);
void band_finish(Ctx &c, int n, int bw, const double *Lrow, double *Lcol, double *Lrev, double *dinv);
void launch_band_sweep(Ctx &c, int nblocks, const int *d_p0, const int *d_len, int max_len, int bw, bool forward,
                       const double *Lcol, const double *Lrev, const double *dinv, const double *in, const int *gather,
                       double *out, double *out_shift = nullptr);
void drop_caches(Ctx &c);
// separator rows of the A_w factor against factored blocks as warp band sweeps (solve.cu); false: band too wide
bool launch_sep_rows_sweep(Ctx &c, int np, const int *pairs, const void *blk, int maxsep, int bw, const double *Lcol,
                           double *Loff);
void build_sell(Ctx &c, const Bsr &A, Sell &S, bool alloc, bool split, bool sort_rows = false);

// pieces of setup_all reused by amgf_import (io.cu)
void build_thin(Ctx &c);
void alloc_workspaces(Ctx &c);
void r_interleave(Ctx &c, Bsr &R);
void coarsest_alloc(Ctx &c);
int band_width(Ctx &c);
// api.cu: handle basics shared by amgf_setup and amgf_import
void ctx_init(Ctx &c, void *stream);  // validates c.cfg, Chebyshev coefficients, scalars and error flags

// ------------------------------------------------------------------ solve orchestration (api.cu)
// Fusion hooks of the PCG iteration into the V-cycles (Chebyshev smoother only; bitwise unchanged):
//   prestarted  level 0's from-zero start (dir, start buffer) was written by k_axpy2_cheb0
//   dot_r       the last level-0 step also forms the C14 partials of dot(dot_r, x) into c.dot_part
struct VcOpts {
  bool prestarted = false;
  const double *dot_r = nullptr;
};
void vcycle(Ctx &c, int l, const double *b, double *x, const double *add, VcOpts o = VcOpts{});
void tail_plan(Ctx &c);                                   // after setup_all: enable the fused coarse tail
void tail_vcycle(Ctx &c, const double *b, double *x);    // V-cycle from level c.tail_level down, one launch
void apply_M(Ctx &c, const double *r, double *z, VcOpts first = VcOpts{}, const double *dot_r = nullptr);

}  // namespace amgf

// The opaque handle of the C ABI (include/amgf.h).
struct amgf_ctx : public amgf::Ctx {};

namespace amgf {
// Run f, mapping exceptions to an amgf_status (no exception crosses the ABI).
template <class F>
amgf_status guarded(F &&f) {
  try {
    return f();
  } catch (const Error &e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc &) {
    set_error("host allocation failed");
    return AMGF_ERR_OOM;
  } catch (const std::exception &e) {
    set_error(e.what());
    return AMGF_ERR_ARG;
  }
}
}  // namespace amgf
