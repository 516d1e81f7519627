// api.cu -- C-ABI entry points of libamgf.so and the solve orchestration (V-cycle, AMGF apply, PCG).
//
//   vcycle   B b: l1-Jacobi pre-sweep from zero, residual, restriction, recursion, prolongation,
//            post-sweep; dense Cholesky solve on the coarsest level.
//   apply_M  x1 = B r; r1 = r - S x1; y = A_w^{-1} r1[Z]; x2 = x1 + P y; r2 = r1 - S[:,Z] y;
//            z = x2 + B r2  (Def. AMGF; three stages SPEC.md:245; C11).
//   pcg      PAPER.md:368 (relative preconditioned residual), C15.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

#include <chrono>
#include <map>
#include <mutex>

namespace amgf {

static thread_local std::string g_last_error;
void set_error(const std::string &m) { g_last_error = m; }
const char *get_error() { return g_last_error.c_str(); }

bool Ctx::guard_enabled() {
  static const bool on = [] {
    const char *e = getenv("AMGF_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}

long Ctx::guard_violations() {
  cudaDeviceSynchronize();
  long bad = 0;
  std::vector<unsigned char> buf(kGuardBytes);
  for (auto &g : guards) {
    if (cudaMemcpy(buf.data(), (char *)g.first + g.second, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (unsigned char b : buf)
      if (b != kGuardByte) {
        bad++;
        break;
      }
  }
  return bad;
}

void Ctx::release(void *p) {
  if (!p) return;
  for (size_t i = 0; i < guards.size(); i++)
    if (guards[i].first == p) {
      guards[i] = guards.back();
      guards.pop_back();
      break;
    }
  for (size_t i = 0; i < allocs.size(); i++)
    if (allocs[i] == p) {
      cudaFree(p);
      allocs[i] = allocs.back();
      allocs.pop_back();
      return;
    }
}

Ctx::~Ctx() {
  drop_caches(*this);
  for (auto &g : pcg_graph)
    if (g) cudaGraphExecDestroy(g);
  for (auto &g : pcg_loop)
    if (g) cudaGraphExecDestroy(g);
  if (loop_host) cudaFreeHost(loop_host);
  if (gstream) cudaStreamDestroy(gstream);
  if (ev_in) cudaEventDestroy(ev_in);
  if (ev_out) cudaEventDestroy(ev_out);
  if (side) cudaStreamDestroy(side);
  if (ev_fork) cudaEventDestroy(ev_fork);
  for (auto &e : ph_ev)
    if (e) cudaEventDestroy(e);
  if (fstream) cudaStreamDestroy(fstream);
  if (ev_f0) cudaEventDestroy(ev_f0);
  if (ev_f1) cudaEventDestroy(ev_f1);
  if (ev_join) cudaEventDestroy(ev_join);
  for (void *p : allocs) cudaFree(p);
  if (sc_host) cudaFreeHost(sc_host);
  if (err_host) cudaFreeHost(err_host);
}

size_t &device_slot(const void *key) {
  static std::mutex mu;
  static std::map<std::pair<int, const void *>, size_t> slots;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  return slots[{dev, key}];  // std::map references stay valid across insertions
}

bool debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("AMGF_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// AMGF_LAUNCH_TIMELINE=1 (diagnostic): an event after every launch of the numeric re-setup, on the stream it
// went to; timeline_dump prints each kernel's completion time relative to `origin` (both streams, no profiler).
struct TimelineRec {
  const char *name;
  bool side;
  cudaEvent_t ev;
};
static std::vector<TimelineRec> g_timeline;
static std::vector<cudaEvent_t> g_timeline_pool;
static bool g_timeline_on = false;
void timeline_begin(Ctx &c) {
  static const bool en = getenv("AMGF_LAUNCH_TIMELINE") != nullptr;
  g_timeline_on = en;
  for (auto &r : g_timeline) g_timeline_pool.push_back(r.ev);
  g_timeline.clear();
}
void timeline_dump(Ctx &c, cudaEvent_t origin) {
  if (!g_timeline_on) return;
  g_timeline_on = false;
  cudaDeviceSynchronize();
  float prev[2] = {0, 0};
  for (auto &r : g_timeline) {
    float t = 0;
    cudaEventElapsedTime(&t, origin, r.ev);
    fprintf(stderr, "tl %s %-28s end %8.1f us  (+%7.1f)\n", r.side ? "side" : "main", r.name, t * 1e3,
            (t - prev[r.side]) * 1e3);
    prev[r.side] = t;
  }
}
void after_launch(Ctx &c, const char *name) {
  c.launches++;
  if (g_timeline_on && !c.capturing) {
    cudaEvent_t ev;
    if (!g_timeline_pool.empty()) {
      ev = g_timeline_pool.back();
      g_timeline_pool.pop_back();
    } else {
      cudaEventCreate(&ev);
    }
    cudaEventRecord(ev, c.stream);
    g_timeline.push_back({name, (c.side && c.stream == c.side) || (c.fstream && c.stream == c.fstream), ev});
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && debug_sync() && !c.capturing) e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) throw Error{AMGF_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e)};
}

void check_dev_error(Ctx &c, const char *where) {
  CK(cudaMemcpyAsync(c.err_host, c.err, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  const int code = c.err_host[0], info = c.err_host[1];
  if (code == DERR_NONE) return;
  CK(cudaMemsetAsync(c.err, 0, 2 * sizeof(int), c.stream));
  CK(cudaStreamSynchronize(c.stream));
  std::string w = std::string(where) + ": ";
  switch (code) {
    case DERR_NONFINITE: throw Error{AMGF_ERR_NONFINITE, w + "non-finite value at index " + std::to_string(info)};
    case DERR_DOMAIN: throw Error{AMGF_ERR_DOMAIN, w + "D must be > 0 and bound diagonals >= 0 (index " + std::to_string(info) + ")"};
    case DERR_NOT_SPD:
      throw Error{AMGF_ERR_NOT_SPD, w + "non-positive pivot " + std::to_string(info % 1000000) +
                                        (info / 1000000 == 1 ? " of A_w" : " of the coarsest operator")};
    case DERR_RANK: throw Error{AMGF_ERR_RANK, w + "rank-deficient tentative prolongator at aggregate " + std::to_string(info)};
    case DERR_LIMIT: throw Error{AMGF_ERR_LIMIT, w + "capacity limit exceeded at row " + std::to_string(info)};
    case DERR_BREAKDOWN: throw Error{AMGF_ERR_BREAKDOWN, w + (info == 1 ? "p.Sp <= 0" : "r.Mr < 0")};
    default: throw Error{AMGF_ERR_ARG, w + "invalid input (index " + std::to_string(info) + ")"};
  }
}

// ------------------------------------------------------------------ V-cycle
void vcycle(Ctx &c, int l, const double *b, double *x, const double *add, VcOpts o) {
  Level &L = c.lev[l];
  if (l == c.nlev - 1) {
    double *dst = add ? L.x2 : x;
    launch_band_trsv(c, c.nco, c.nco - 1, c.Lc_col, c.Lc_rev, c.Lc_dinv, b, nullptr, dst, nullptr, nullptr, L.r);
    if (add) launch_add(c, L.n, add, dst, x);
    return;
  }
  if (l == c.tail_level && !add) {
    tail_vcycle(c, b, x);
    return;
  }
  Level &Lc = c.lev[l + 1];
  const int pre = c.cfg.pre_sweeps, post = c.cfg.post_sweeps;
  if (c.cfg.smoother == 1) {  // Chebyshev (C23): each SpMV step writes the other buffer of {x, x2}
    const int k = c.cfg.cheb_degree;
    const int nswap = (k - 1) + (pre - 1) * k + post * k;
    double *bufs[2] = {x, L.x2};
    int ci = nswap & 1;  // so that the last step lands in x
    auto step = [&](bool first, int s, const double *addp) {
      launch_sell_cheb(c, L.As, first, bufs[ci], b, L.dl1, L.dir, first ? c.cheb_c0 : c.cheb_a[s],
                       first ? 0.0 : c.cheb_b[s], addp, bufs[1 - ci]);
      ci = 1 - ci;
    };
    if (!o.prestarted) launch_cheb0(c, L.n, b, L.dl1, c.cheb_c0, L.dir, bufs[ci]);
    for (int s = 1; s < k; s++) step(false, s, nullptr);
    for (int sw = 1; sw < pre; sw++) {
      step(true, 0, nullptr);
      for (int s = 1; s < k; s++) step(false, s, nullptr);
    }
    launch_sell_spmv(c, L.As, SPMV_RESID, bufs[ci], b, nullptr, nullptr, L.r, nullptr);
    launch_restrict(c, L.R, L.r, Lc.bv);
    vcycle(c, l + 1, Lc.bv, Lc.x, nullptr);
    launch_prolong(c, L.Ps, Lc.x, bufs[ci]);
    for (int sw = 0; sw < post; sw++)
      for (int s = 0; s < k; s++) {
        const bool last = (sw == post - 1 && s == k - 1);
        if (last && o.dot_r && s > 0) {  // final step fused with the PCG dot's level-1 partials (C14)
          launch_sell_cheb(c, L.As, false, bufs[ci], b, L.dl1, L.dir, c.cheb_a[s], c.cheb_b[s], add,
                           bufs[1 - ci], o.dot_r);
          ci = 1 - ci;
        } else {
          step(s == 0, s, (add && last) ? add : nullptr);
        }
      }
    return;
  }
  if (c.cfg.smoother == 2) {  // nodal-block l1 (C25): residual SpMV, then the per-node block solve and update
    double *bufs[2] = {x, L.x2};
    int ci = ((pre - 1) + post) & 1;  // so that the last post-sweep lands in x
    launch_block_smooth(c, L, b, nullptr, nullptr, bufs[ci]);
    for (int s = 1; s < pre; s++) {
      launch_sell_spmv(c, L.As, SPMV_RESID, bufs[ci], b, nullptr, nullptr, L.r, nullptr);
      launch_block_smooth(c, L, L.r, bufs[ci], nullptr, bufs[1 - ci]);
      ci = 1 - ci;
    }
    launch_sell_spmv(c, L.As, SPMV_RESID, bufs[ci], b, nullptr, nullptr, L.r, nullptr);
    launch_restrict(c, L.R, L.r, Lc.bv);
    vcycle(c, l + 1, Lc.bv, Lc.x, nullptr);
    launch_prolong(c, L.Ps, Lc.x, bufs[ci]);
    for (int s = 0; s < post; s++) {
      launch_sell_spmv(c, L.As, SPMV_RESID, bufs[ci], b, nullptr, nullptr, L.r, nullptr);
      launch_block_smooth(c, L, L.r, bufs[ci], (s == post - 1) ? add : nullptr, bufs[1 - ci]);
      ci = 1 - ci;
    }
    return;
  }
  double *bufs[2] = {x, L.x2};
  int ci = ((pre - 1) + post) & 1;  // so that the last post-sweep lands in x
  launch_jacobi0(c, L.n, b, L.dl1, bufs[ci]);
  for (int s = 1; s < pre; s++) {
    launch_sell_spmv(c, L.As, SPMV_SMOOTH, bufs[ci], b, L.dl1, nullptr, bufs[1 - ci], nullptr);
    ci = 1 - ci;
  }
  launch_sell_spmv(c, L.As, SPMV_RESID, bufs[ci], b, nullptr, nullptr, L.r, nullptr);
  launch_restrict(c, L.R, L.r, Lc.bv);
  vcycle(c, l + 1, Lc.bv, Lc.x, nullptr);
  launch_prolong(c, L.Ps, Lc.x, bufs[ci]);
  for (int s = 0; s < post; s++) {
    const bool last = (s == post - 1);
    launch_sell_spmv(c, L.As, (last && add) ? SPMV_SMOOTH_ADD : SPMV_SMOOTH, bufs[ci], b, L.dl1, add, bufs[1 - ci],
                     nullptr);
    ci = 1 - ci;
  }
}

// ------------------------------------------------------------------ AMGF apply (C11)
void apply_M(Ctx &c, const double *r, double *z, VcOpts first, const double *dot_r) {
  Level &L0 = c.lev[0];
  vcycle(c, 0, r, c.w_x1, nullptr, first);
  if (c.nc == 0) {
    // I_c empty: filter stage is the identity
    launch_sell_spmv(c, L0.As, SPMV_RESID, c.w_x1, r, nullptr, nullptr, c.w_r1, nullptr);
    VcOpts second;
    second.dot_r = dot_r;
    vcycle(c, 0, c.w_r1, z, c.w_x1, second);
    return;
  }
  // r1 at the Z rows first (pi order), then the A_w solve on the high-priority filter stream while the
  // full residual r1 = r - S x1 runs here; x2 = x1 + P y and the thin r2 after the join.  Same kernels
  // and arithmetic as the serial order, so the result is unchanged bitwise.
  if (!c.fstream) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c.fstream, cudaStreamNonBlocking, hi));
    // SM partition for the overlap: the residual SpMV runs on 80 of the 148 SMs (measured at cfg 3 with PDL:
    // 80 SMs -> A_w solve done at 250 us, SpMV at 257 us; 84-96 SMs -> A_w solve 278-284 us, SpMV 235-255 us;
    // the A_w solve alone takes 234 us, and 383 us next to the unpartitioned SpMV).  An L2 persistence window
    // for the A_w data was measured too and did not help (it costs the V-cycles L2 capacity).
    int dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    c.resid_sms = std::max(1, nsm * 80 / 148);
    CK(cudaEventCreateWithFlags(&c.ev_f0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_f1, cudaEventDisableTiming));
  }
  static const bool trace = getenv("AMGF_TRACE_FILTER") != nullptr;  // tools only: overlap timeline
  cudaEvent_t te[5] = {};
  if (trace && !c.capturing) {
    for (auto &e : te) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(te[0], c.stream));
  }
  launch_resid_dofs(c, c.nc, c.dof, c.w_x1, r, c.rz);
  CK(cudaEventRecord(c.ev_f0, c.stream));
  CK(cudaStreamWaitEvent(c.fstream, c.ev_f0, 0));
  const bool basisJ = c.cfg.filter_basis == 1;
  {
    cudaStream_t main = c.stream;
    c.stream = c.fstream;
    try {
      if (basisJ) {  // P = J^T: v = J r1 (rz in Z order), y = (J S J^T)^{-1} v, w = J^T y (Z order)
        filter_J_apply(c, c.rz, c.fJv, nullptr, nullptr);
        nd_solve(c, c.fJv, nullptr);
        filter_J_apply(c, nullptr, nullptr, c.fv, c.fJw);
      } else {
        nd_solve(c, c.rz, nullptr);  // y = A_w^{-1} r1[Z] (pi order, c.fv)
      }
    } catch (...) {
      c.stream = main;
      throw;
    }
    c.stream = main;
  }
  CK(cudaEventRecord(c.ev_f1, c.fstream));
  if (te[0]) CK(cudaEventRecord(te[1], c.fstream));
  static const bool no_overlap = getenv("AMGF_NO_OVERLAP") != nullptr;  // A/B experiments
  if (no_overlap) CK(cudaStreamWaitEvent(c.stream, c.ev_f1, 0));
  {
    // 180 KB of shared memory reserved per CTA: no filter CTA (>= 49 KB) fits beside it
    static const int spmv_sms = getenv("AMGF_SPMV_SMS") ? atoi(getenv("AMGF_SPMV_SMS")) : -1;  // A/B only
    const int n_sms = spmv_sms >= 0 ? spmv_sms : c.resid_sms;
    if (n_sms > 0) launch_resid_partition(c, L0.As, c.w_x1, r, c.w_r1, n_sms, 180 * 1024);
    else launch_sell_spmv(c, L0.As, SPMV_RESID, c.w_x1, r, nullptr, nullptr, c.w_r1, nullptr);
  }
  if (te[0]) CK(cudaEventRecord(te[2], c.stream));
  CK(cudaStreamWaitEvent(c.stream, c.ev_f1, 0));
  if (te[0]) {
    CK(cudaEventSynchronize(te[1]));
    CK(cudaEventSynchronize(te[2]));
    float a = 0, b = 0;
    CK(cudaEventElapsedTime(&a, te[0], te[1]));
    CK(cudaEventElapsedTime(&b, te[0], te[2]));
    fprintf(stderr, "filter overlap: filter done at %.1f us, residual SpMV done at %.1f us\n", a * 1e3, b * 1e3);
    for (auto &e : te) cudaEventDestroy(e);
  }
  // x2 = x1 + P y (scatter) and the thin residual r2 = r1 - S[:,Z] y in one launch
  launch_thin_resid(c, c.nthin, c.thin_row, c.thin_ptr, c.thin_pos, c.thin_val, basisJ ? c.fJw : c.fv, c.w_r1, c.nc,
                    c.dof, c.w_x1);
  VcOpts second;
  second.dot_r = dot_r;
  vcycle(c, 0, c.w_r1, z, c.w_x1, second);
}

// ------------------------------------------------------------------ PCG (C15)
// One PCG iteration (C15): q = S p (+ p.q partials), pi and alpha, x += alpha p, r -= alpha q, z = M r,
// rho' = r.z and beta, p = z + beta p, then the scalars and the error flag to pinned host memory.  The
// p update of the final iteration is harmless (p is not used afterwards).  All pointers are the handle's
// own buffers, so the body is captured once into a CUDA graph and replayed (values change, pointers do not).
static void pcg_body(Ctx &c, int precond, bool host_copies = true) {
  const long n = c.n;
  launch_sell_spmv(c, c.lev[0].As, SPMV_DOT, c.p, nullptr, nullptr, nullptr, c.q, c.dot_part);
  launch_dot_finish(c, nblk(c.lev[0].As.nrows), DOT_PI);  // pi = p.q, alpha = rho / pi
  // Chebyshev: the x, r update also writes the from-zero start of V-cycle #1 at level 0, and the last level-0
  // step of the last V-cycle forms the partials of r.z (both bitwise the same as the separate kernels)
  Level &L0 = c.lev[0];
  const bool pre0 = (c.cfg.smoother == 1 && c.nlev >= 2);
  const bool fdot = pre0 && c.cfg.cheb_degree >= 2;
  if (pre0) {
    const int k = c.cfg.cheb_degree, pre = c.cfg.pre_sweeps, post = c.cfg.post_sweeps;
    const int ci = ((k - 1) + (pre - 1) * k + post * k) & 1;  // vcycle's start-buffer parity
    double *xs = ci ? L0.x2 : (precond == 0 ? c.w_x1 : c.zz);
    launch_axpy2_cheb0(c, n, c.p, c.q, c.xx, c.rr, L0.dl1, c.cheb_c0, L0.dir, xs);
  } else {
    launch_axpy2(c, n, c.p, c.q, c.xx, c.rr);
  }
  VcOpts first;
  first.prestarted = pre0;
  if (precond == 0) {
    apply_M(c, c.rr, c.zz, first, fdot ? c.rr : nullptr);
  } else {
    first.dot_r = fdot ? c.rr : nullptr;
    vcycle(c, 0, c.rr, c.zz, nullptr, first);
  }
  if (fdot) launch_dot_finish(c, nblk(L0.As.nrows), DOT_RHO1);  // rho' = r.z, beta = rho'/rho, rho = rho'
  else launch_dot(c, n, 3, c.rr, c.zz, DOT_RHO1);
  launch_xpby(c, n, c.zz, c.p);
  if (host_copies) {
    CK(cudaMemcpyAsync(c.sc_host, c.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaMemcpyAsync(c.err_host, c.err, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  }
}

// End of one device-side PCG iteration: it += 1, rel = sqrt(rho1 / rho0) (the host loop's formula), stop
// on rel < rtol, on it == max_it or on a raised error flag; the WHILE node repeats the body while 1.
__global__ void k_pcg_control(cudaGraphConditionalHandle h, const Scalars *sc, LoopState *ls, const int *err) {
  const int it = ls->it + 1;
  const double rel = sqrt(sc->rho1 / sc->rho0);
  if (it <= ls->cap) {
    ls->hist[2 * (it - 1)] = sc->alpha;
    ls->hist[2 * (it - 1) + 1] = sc->beta;
  }
  const bool stop = (rel < ls->rtol) || (it >= ls->max_it) || (err[0] != 0);
  ls->it = it;
  ls->rel = rel;
  ls->stop = stop;
  cudaGraphSetConditional(h, stop ? 0u : 1u);
}

// Capture the iteration body into the body graph of a conditional WHILE node (one graph launch per solve,
// no host round trip per iteration).  Returns false (and leaves the host loop in charge) if the driver
// refuses any step.
static bool build_pcg_loop(Ctx &c, int precond) {
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  const int64_t l0 = c.launches;
  bool ok = false;
  try {
    if (!c.loop) {
      c.loop = c.alloc<LoopState>(1);
      CK(cudaMallocHost(&c.loop_host, sizeof(LoopState)));
    }
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    c.capturing = true;
    CK(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    try {
      pcg_body(c, precond, false);
      k_pcg_control<<<1, 1, 0, c.stream>>>(h, c.sc, c.loop, c.err);
      after_launch(c, "k_pcg_control");
    } catch (...) {
      cudaGraph_t tmp;
      cudaStreamEndCapture(c.stream, &tmp);
      throw;
    }
    CK(cudaStreamEndCapture(c.stream, &body));
    c.capturing = false;
    CK(cudaGraphInstantiate(&ex, g, 0));
    c.pcg_loop[precond] = ex;
    c.graph_launches[precond] = c.launches - l0;
    ok = true;
  } catch (const Error &) {
    c.capturing = false;
    cudaGetLastError();
  }
  c.launches = l0;
  if (g) cudaGraphDestroy(g);
  return ok;
}

static amgf_status pcg_impl(Ctx &c, const double *b, double *x, double rtol, int max_it, int precond,
                            amgf_report *rep) {
  const long n = c.n;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, c.stream));
  launch_zero(c, n, c.xx);
  launch_copy(c, n, b, c.rr);
  if (precond == 0) apply_M(c, c.rr, c.zz);
  else vcycle(c, 0, c.rr, c.zz, nullptr);
  launch_dot(c, n, 3, c.rr, c.zz, DOT_RHO0);
  CK(cudaMemcpyAsync(c.sc_host, c.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, c.stream));
  check_dev_error(c, "pcg");
  const double rho0 = c.sc_host->rho0;
  int it = 0;
  double rel = 0.0;
  amgf_status st = AMGF_NOT_CONVERGED;
  if (rho0 == 0.0) {
    st = AMGF_OK;
    c.hist_n = 0;  // no iterations: no history (not the previous solve's)
  } else if (!(rho0 > 0.0)) {
    throw Error{AMGF_ERR_BREAKDOWN, "pcg: r.Mr <= 0"};
  } else {
    launch_copy(c, n, c.zz, c.p);
    static const bool host_loop = getenv("AMGF_HOST_LOOP") != nullptr;  // A/B experiments
    if (!host_loop && !c.pcg_loop_tried[precond] && max_it > 0) {
      c.pcg_loop_tried[precond] = true;
      build_pcg_loop(c, precond);
    }
    if (!host_loop && c.pcg_loop[precond] && max_it > 0) {
      const int want = std::min(max_it, 100000);  // history capacity (iterations beyond it are not recorded)
      if (c.hist_cap < want) {  // history buffer (read through LoopState: the graph keeps its pointers)
        if (c.hist) c.release(c.hist);
        c.hist_cap = want;
        c.hist = c.alloc<double>(2 * (size_t)c.hist_cap);
      }
      LoopState ls = {};
      ls.max_it = max_it;
      ls.rtol = rtol;
      ls.cap = c.hist_cap;
      ls.hist = c.hist;
      *c.loop_host = ls;
      CK(cudaMemcpyAsync(c.loop, c.loop_host, sizeof(LoopState), cudaMemcpyHostToDevice, c.stream));
      CK(cudaGraphLaunch(c.pcg_loop[precond], c.stream));
      CK(cudaMemcpyAsync(c.loop_host, c.loop, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
      CK(cudaMemcpyAsync(c.err_host, c.err, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      it = c.loop_host->it;
      rel = c.loop_host->rel;
      c.hist_n = std::min(it, c.hist_cap);
      c.launches += c.graph_launches[precond] * it;
      if (c.err_host[0]) check_dev_error(c, "pcg");
      st = (rel < rtol) ? AMGF_OK : AMGF_NOT_CONVERGED;
    } else {
    c.host_hist.clear();
    if (!c.pcg_graph[precond] && max_it > 0) {
      cudaGraph_t g;
      const int64_t l0 = c.launches;
      c.capturing = true;
      CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      try {
        pcg_body(c, precond);
      } catch (...) {
        cudaStreamEndCapture(c.stream, &g);
        c.capturing = false;
        throw;
      }
      CK(cudaStreamEndCapture(c.stream, &g));
      c.capturing = false;
      CK(cudaGraphInstantiate(&c.pcg_graph[precond], g, 0));
      CK(cudaGraphDestroy(g));
      c.graph_launches[precond] = c.launches - l0;
      c.launches = l0;
    }
    for (it = 1; it <= max_it; it++) {
      CK(cudaGraphLaunch(c.pcg_graph[precond], c.stream));
      c.launches += c.graph_launches[precond];
      CK(cudaStreamSynchronize(c.stream));
      if (c.err_host[0]) check_dev_error(c, "pcg");
      const double rho1 = c.sc_host->rho1;
      rel = std::sqrt(rho1 / rho0);
      c.host_hist.push_back(c.sc_host->alpha);
      c.host_hist.push_back(c.sc_host->beta);
      if (rel < rtol) { st = AMGF_OK; break; }
      if (it == max_it) break;
    }
    if (it > max_it) it = max_it;
    c.hist_n = -(int)(c.host_hist.size() / 2);  // negative: the history is on the host
    }
  }
  if (x != c.xx) launch_copy(c, n, c.xx, x);
  CK(cudaEventRecord(e1, c.stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iterations = it;
    rep->converged = st == AMGF_OK;
    rep->rel_pres_norm = rel;
    rep->solve_ms = ms;
    rep->setup_ms = c.last_setup_ms;
    rep->n_levels = c.nlev;
    for (int l = 0; l < MAXLEV; l++) {
      rep->level_dofs[l] = l < c.nlev ? c.lev[l].n : 0;
      rep->level_nnzb[l] = l < c.nlev ? c.lev[l].A.nnzb : 0;
    }
  }
  return st;
}

// The solve runs on the handle's own (capturable, non-default) stream, ordered after and before the
// caller's stream by events.
static amgf_status pcg(Ctx &c, const double *b, double *x, double rtol, int max_it, int precond, amgf_report *rep) {
  if (!c.gstream) {
    CK(cudaStreamCreateWithFlags(&c.gstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c.ev_in, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c.ev_out, cudaEventDisableTiming));
  }
  cudaStream_t user = c.stream;
  CK(cudaEventRecord(c.ev_in, user));
  CK(cudaStreamWaitEvent(c.gstream, c.ev_in, 0));
  c.stream = c.gstream;
  amgf_status st;
  try {
    st = pcg_impl(c, b, x, rtol, max_it, precond, rep);
  } catch (...) {
    c.stream = user;
    throw;
  }
  c.stream = user;
  CK(cudaEventRecord(c.ev_out, c.gstream));
  CK(cudaStreamWaitEvent(user, c.ev_out, 0));
  return st;
}

void ctx_init(Ctx &c, void *stream) {
  c.stream = (cudaStream_t)stream;
  REQUIRE(c.cfg.pre_sweeps >= 1 && c.cfg.post_sweeps >= 1 && c.cfg.max_levels >= 1 && c.cfg.power_iters >= 1,
          AMGF_ERR_ARG, "invalid config");
  REQUIRE(c.cfg.smoother == 0 || c.cfg.smoother == 2 || (c.cfg.smoother == 1 && c.cfg.cheb_degree >= 1 && c.cfg.cheb_degree <= 32 &&
                                  c.cfg.cheb_ratio > 1.0),
          AMGF_ERR_ARG, "invalid smoother config");
  REQUIRE(c.cfg.filter_basis == 0 || c.cfg.filter_basis == 1, AMGF_ERR_ARG, "invalid filter_basis");
  if (c.cfg.smoother == 1) {  // Chebyshev coefficients (C23): same formulas, in the same order, as the oracle
    const double ratio = c.cfg.cheb_ratio;
    const double theta = (1.0 + 1.0 / ratio) / 2.0, delta = (1.0 - 1.0 / ratio) / 2.0;
    const double sigma = theta / delta;
    double rho = 1.0 / sigma;
    c.cheb_c0 = 1.0 / theta;
    for (int k = 1; k < c.cfg.cheb_degree; k++) {
      const double rn = 1.0 / (2.0 * sigma - rho);
      c.cheb_a[k] = rn * rho;
      c.cheb_b[k] = 2.0 * rn / delta;
      rho = rn;
    }
  }
  c.sc = c.alloc<Scalars>(1);
  c.err = c.alloc<int>(2);
  CK(cudaMemsetAsync(c.err, 0, 2 * sizeof(int), c.stream));
  CK(cudaMemsetAsync(c.sc, 0, sizeof(Scalars), c.stream));
  CK(cudaMallocHost(&c.sc_host, sizeof(Scalars)));
  CK(cudaMallocHost(&c.err_host, 2 * sizeof(int)));
}

}  // namespace amgf

// =================================================================== C ABI
using namespace amgf;


#ifdef AMGF_R1_TRACE
namespace amgf { int r1_trace_read(unsigned long long *h, int n); }
#endif
extern "C" {

void amgf_default_config(amgf_config *cfg) {
  cfg->pre_sweeps = 1;
  cfg->post_sweeps = 1;
  cfg->coarsest_size = 64;
  cfg->max_levels = 25;
  cfg->power_iters = 6;   // measured: DESIGN.md R19
  cfg->nd_levels = 3;
  cfg->smoother = 1;  // Chebyshev degree 2 (DESIGN R18); 0 = l1-Jacobi
  cfg->cheb_degree = 2;
  cfg->agg_seed = 0x5EED;
  cfg->cheb_ratio = 20.0;
  cfg->filter_basis = 0;
  cfg->pad_ = 0;
}

const char *amgf_last_error(void) { return get_error(); }

amgf_status amgf_setup(int32_t nodes, const int32_t *K_ptr, const int32_t *K_col, const double *K_val, int32_t m,
                       const int32_t *J_ptr, const int32_t *J_col, const double *J_val, const double *D,
                       const int32_t *Z, int32_t nc, const double *B_nns, const amgf_config *cfg, void *stream,
                       amgf_handle *out) {
  if (!out) { set_error("out is NULL"); return AMGF_ERR_ARG; }
  *out = nullptr;
  amgf_ctx *c = new amgf_ctx();
  amgf_status st = guarded([&]() -> amgf_status {
    REQUIRE(nodes > 0 && K_ptr && K_col && K_val && B_nns, AMGF_ERR_ARG, "null K / near-null space or nodes <= 0");
    REQUIRE(m >= 0 && (m == 0 || (J_ptr && J_col && J_val && D)), AMGF_ERR_ARG, "null J or D");
    REQUIRE(!Z || nc >= 0, AMGF_ERR_ARG, "negative nc");
    if (cfg) c->cfg = *cfg; else amgf_default_config(&c->cfg);
    ctx_init(*c, stream);
    c->nodes = nodes;
    c->n = 3L * nodes;
    c->m = m;
    c->dot_part = c->alloc<double>(nblk(c->n) + 1);
    const auto t0 = std::chrono::steady_clock::now();
    setup_all(*c, K_ptr, K_col, K_val, J_ptr, J_col, J_val, D, Z, nc, B_nns);
    c->last_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return AMGF_OK;
  });
  if (st != AMGF_OK) {
    cudaStreamSynchronize((cudaStream_t)stream);
    delete c;
    return st;
  }
  *out = c;
  return AMGF_OK;
}

amgf_status amgf_update_D(amgf_handle h, const double *D, void *stream) {
  if (!h) { set_error("null handle"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(!h->imported, AMGF_ERR_ARG, "update_D: an imported hierarchy has no K, J (set it up with amgf_setup)");
    REQUIRE(h->m == 0 || D, AMGF_ERR_ARG, "null D");
    h->stream = (cudaStream_t)stream;
    setup_numeric(*h, D);
    h->last_setup_ms = h->setup_ms[0];
    CK(cudaStreamSynchronize(h->stream));
    return AMGF_OK;
  });
}

amgf_status amgf_update_D_box(amgf_handle h, const double *D, const double *D_lo, const double *D_up, void *stream) {
  if (!h) { set_error("null handle"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(!h->imported, AMGF_ERR_ARG, "update_D_box: an imported hierarchy has no K, J (set it up with amgf_setup)");
    REQUIRE(h->m == 0 || D, AMGF_ERR_ARG, "null D");
    h->stream = (cudaStream_t)stream;
    setup_numeric(*h, D, D_lo, D_up);
    h->last_setup_ms = h->setup_ms[0];
    CK(cudaStreamSynchronize(h->stream));
    return AMGF_OK;
  });
}

amgf_status amgf_apply(amgf_handle h, const double *r, double *z, void *stream) {
  if (!h || !r || !z) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    h->stream = (cudaStream_t)stream;
    static const bool tl = getenv("AMGF_LAUNCH_TIMELINE") != nullptr;  // diagnostic: per-launch completion times
    static cudaEvent_t tl0 = nullptr;
    if (tl) {
      if (!tl0) CK(cudaEventCreate(&tl0));
      timeline_begin(*h);
      CK(cudaEventRecord(tl0, h->stream));
    }
    apply_M(*h, r, z);
    if (tl) timeline_dump(*h, tl0);
    return AMGF_OK;
  });
}

amgf_status amgf_vcycle(amgf_handle h, const double *b, double *x, void *stream) {
  if (!h || !b || !x) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    h->stream = (cudaStream_t)stream;
    vcycle(*h, 0, b, x, nullptr);
    return AMGF_OK;
  });
}

amgf_status amgf_spmv(amgf_handle h, int32_t level, const double *x, double *y, void *stream) {
  if (!h || !x || !y) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(level >= 0 && level < h->nlev, AMGF_ERR_ARG, "bad level");
    h->stream = (cudaStream_t)stream;
    Level &L = h->lev[level];
    if (L.As.val) launch_sell_spmv(*h, L.As, SPMV_Y, x, nullptr, nullptr, nullptr, y, nullptr);
    else launch_bsr_spmv(*h, L.A, x, y);
    return AMGF_OK;
  });
}

amgf_status amgf_spmv_K(amgf_handle h, const double *x, double *y, void *stream) {
  if (!h || !x || !y) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(!h->imported && h->K.val, AMGF_ERR_ARG, "spmv_K: the handle holds no K (imported hierarchy)");
    h->stream = (cudaStream_t)stream;
    launch_bsr_spmv(*h, h->K, x, y);
    return AMGF_OK;
  });
}

amgf_status amgf_pcg_solve(amgf_handle h, const double *b, double *x, double rtol, int32_t max_it, int32_t precond,
                           amgf_report *rep, void *stream) {
  if (!h || !b || !x) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(max_it >= 0 && rtol >= 0 && (precond == 0 || precond == 1), AMGF_ERR_ARG, "bad pcg arguments");
    h->stream = (cudaStream_t)stream;
    return pcg(*h, b, x, rtol, max_it, precond, rep);
  });
}

amgf_status amgf_pcg_solve_host(amgf_handle h, const double *b_host, double *x_host, double rtol, int32_t max_it,
                                int32_t precond, amgf_report *rep, void *stream) {
  if (!h || !b_host || !x_host) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    h->stream = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(h->bb, b_host, h->n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    amgf_status st = pcg(*h, h->bb, h->xx, rtol, max_it, precond, rep);
    CK(cudaMemcpyAsync(x_host, h->xx, h->n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return st;
  });
}

amgf_status amgf_level_info(amgf_handle h, int64_t *info) {
  if (!h || !info) { set_error("null argument"); return AMGF_ERR_ARG; }
  info[0] = h->nlev;
  info[1] = h->nc;
  info[2] = h->nco;
  info[3] = h->bw;
  for (int l = 0; l < h->nlev; l++) {
    Level &L = h->lev[l];
    const bool co = (l == h->nlev - 1);
    info[4 + 6 * l + 0] = L.nodes;
    info[4 + 6 * l + 1] = L.b;
    info[4 + 6 * l + 2] = L.A.nnzb;
    info[4 + 6 * l + 3] = co ? 0 : L.P.nnzb;
    info[4 + 6 * l + 4] = co ? 0 : L.n_agg;
    info[4 + 6 * l + 5] = L.As.nslots;
  }
  info[4 + 6 * MAXLEV + 0] = h->loff_size;
  info[4 + 6 * MAXLEV + 1] = h->nd_nblocks;
  info[4 + 6 * MAXLEV + 2] = h->tail_level;
  info[4 + 6 * MAXLEV + 3] = h->tail_ncta;
  info[4 + 6 * MAXLEV + 4] = h->nf;
  return AMGF_OK;
}

amgf_status amgf_level_get(amgf_handle h, int32_t which, int32_t level, void *dst) {
  if (!h || !dst) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    REQUIRE(level >= 0 && level < h->nlev, AMGF_ERR_ARG, "bad level");
    Level &L = h->lev[level];
    const bool co = (level == h->nlev - 1);
    auto cp = [&](const void *src, size_t bytes) {
      REQUIRE(src || bytes == 0, AMGF_ERR_ARG, "array not available at this level");
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
    };
    switch (which) {
      case 0: cp(L.A.ptr, (L.nodes + 1) * 4); break;
      case 1: cp(L.A.col, L.A.nnzb * 4); break;
      case 2: cp(L.A.val, L.A.nnzb * L.b * L.b * 8); break;
      case 3: REQUIRE(!co, AMGF_ERR_ARG, "no P"); cp(L.P.ptr, (L.nodes + 1) * 4); break;
      case 4: REQUIRE(!co, AMGF_ERR_ARG, "no P"); cp(L.P.col, L.P.nnzb * 4); break;
      case 5: REQUIRE(!co, AMGF_ERR_ARG, "no P"); cp(L.P.val, L.P.nnzb * L.b * 6 * 8); break;
      case 6: REQUIRE(!co, AMGF_ERR_ARG, "no R"); cp(L.R.ptr, (L.n_agg + 1) * 4); break;
      case 7: REQUIRE(!co, AMGF_ERR_ARG, "no R"); cp(L.R.col, L.R.nnzb * 4); break;
      case 8: REQUIRE(!co, AMGF_ERR_ARG, "no R"); cp(L.R.val, L.R.nnzb * L.b * 6 * 8); break;
      case 9: cp(L.dl1, L.n * 8); break;
      case 10: REQUIRE(!co, AMGF_ERR_ARG, "no aggregates"); cp(L.agg, L.nodes * 4); break;
      case 11: cp(L.Bnn, L.n * 6 * 8); break;
      case 12: {
        double lo[2] = {L.lambda, L.omega};
        CK(cudaStreamSynchronize(h->stream));
        std::memcpy(dst, lo, sizeof lo);
        return AMGF_OK;
      }
      case 14: REQUIRE(L.root, AMGF_ERR_ARG, "no roots"); cp(L.root, L.nodes * 4); break;
      case 15: cp(L.comp, L.nodes * 4); break;
      case 20: cp(h->Z, h->nc * 4); break;
      case 22: cp(h->Lrow, (size_t)h->nf * band_stride(h->bw) * 8); break;
      case 23: cp(h->Loff, (size_t)h->loff_size * 8); break;
      case 24: cp(h->Lc_row, (size_t)h->nco * band_stride(h->nco - 1) * 8); break;
      case 25: cp(h->pi_z, (size_t)h->nf * 4); break;
      case 27: cp(h->nd_blk, (size_t)h->nd_nblocks * 32); break;
      default: throw Error{AMGF_ERR_ARG, "unknown array id"};
    }
    CK(cudaStreamSynchronize(h->stream));
    return AMGF_OK;
  });
}

int64_t amgf_launch_count(amgf_handle h) { return h ? h->launches : -1; }

#ifdef AMGF_R1_TRACE
int amgf_debug_r1_trace(unsigned long long *h, int n) { return amgf::r1_trace_read(h, n); }
#endif
int64_t amgf_debug_guard_check(amgf_handle h) {
  if (!h) return -1;
  if (!Ctx::guard_enabled()) return -2;
  return h->guard_violations();
}

amgf_status amgf_setup_times(amgf_handle h, double *ms) {
  if (!h || !ms) { set_error("null argument"); return AMGF_ERR_ARG; }
  for (int i = 0; i < 5; i++) ms[i] = h->setup_ms[i];
  return AMGF_OK;
}

amgf_status amgf_pcg_history(amgf_handle h, int32_t n, double *alpha, double *beta) {
  if (!h || (n > 0 && (!alpha || !beta))) { set_error("null argument"); return AMGF_ERR_ARG; }
  return guarded([&]() -> amgf_status {
    const int avail = h->hist_n >= 0 ? h->hist_n : -h->hist_n;
    REQUIRE(n >= 0 && n <= avail, AMGF_ERR_ARG, "pcg_history: n exceeds the iterations of the last solve");
    std::vector<double> buf(2 * (size_t)n);
    if (n > 0) {
      if (h->hist_n >= 0) {
        CK(cudaMemcpy(buf.data(), h->hist, buf.size() * sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        std::copy(h->host_hist.begin(), h->host_hist.begin() + buf.size(), buf.begin());
      }
    }
    for (int k = 0; k < n; k++) {
      alpha[k] = buf[2 * k];
      beta[k] = buf[2 * k + 1];
    }
    return AMGF_OK;
  });
}

void amgf_destroy(amgf_handle h) {
  if (!h) return;
  cudaStreamSynchronize(h->stream);
  delete h;
}

}  // extern "C"
