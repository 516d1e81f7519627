#!/usr/bin/env python
"""bench.py -- AMGF-PCG on B200 (arxiv 2505.18576), BASELINE.json metric on configs[3].

Workload (N=1): cfg 3 = two-block elasticity, N=64 (1,647,750 dofs, 4,225 contact constraints),
the 10-system interior-point-like D sequence (D log-uniform in [1, 10^(2+10s/9)], s = 0..9).
A step = one system of the sequence: numeric re-setup for its D (amgf_update_D: S, A_w + Cholesky,
Galerkin hierarchy) + AMGF-PCG solve to rtol 1e-8 (amgf_pcg_solve).  Symbolic setup (aggregation,
patterns) is done once before timing (it does not depend on D, R5) and reported separately.

value = device time per system (ms, CUDA events, barrier + synchronize on both sides, max over
ranks, divided by the systems all ranks solved).  With --gpus N > 1 the ranks are replicas, each
solving its own systems (the sequence's D values are pre-drawn, so systems are independent): "weak".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AMGF-PCG solve ms, PCG iters, V-cycle HBM GB/s (frac of peak) @ 1.6M dofs"


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def level_bytes(g):
    """Algorithmic HBM bytes of one V-cycle, one pre- and one post-sweep: per level the
    passes of A (2 for l1-Jacobi: residual + post sweep; 2k for a degree-k Chebyshev sweep: k-1 pre steps,
    residual, k post steps), one of R and one of P (values + int32 block columns), plus the vector traffic
    of the kernels (Jacobi start 24n, residual 24n, restriction, prolongation, l1 sweep 32n; Chebyshev start
    32n, step 48n: x gather, b, d, dir read/write, new x)."""
    cheb = int(getattr(g.config, "smoother", 0)) == 1
    k = int(getattr(g.config, "cheb_degree", 1))
    tot = 0
    for l, L in enumerate(g.levels):
        b, n = L["b"], L["nodes"] * L["b"]
        if l == g.nlev - 1:
            tot += 2 * (g.nco * g.nco) * 8 // 2 + 16 * n   # coarsest dense factor read twice (lower half)
            continue
        A = L["nnzb"] * (8 * b * b + 4) + 4 * L["nodes"]
        Pb = L["nnzb_P"] * (8 * 6 * b + 4)
        nc6 = 6 * L["n_agg"]
        common = (24 * n) + (8 * n + 8 * nc6) + (8 * nc6 + 16 * n)  # residual, restriction, prolongation
        if cheb:
            tot += 2 * k * A + 2 * Pb + common + 32 * n + (2 * k - 1) * 48 * n
        else:
            tot += 2 * A + 2 * Pb + common + 24 * n + 32 * n
    return tot


def system_of(rank: int, world: int, k: int, nsys: int) -> int:
    """Replica schedule: rank r solves systems r, r+N, r+2N, ... of the sequence (mod its length)."""
    return (rank + world * k) % nsys


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a timing over all ranks (identity for one rank)."""
    if world <= 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def spmv_bytes(g):
    L = g.levels[0]
    return L["nnzb"] * 76 + 4 * L["nodes"] + 48 * L["nodes"]


def run_amgf(args, rank, world, local_rank):
    import numpy as np
    import torch
    import amgf_gen
    from paper_2505_18576_b200 import AMGF

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = amgf_gen.config(args.cfg)
    nsys = p.D_seq.shape[0]
    stream = torch.cuda.current_stream()
    D_dev = [torch.from_numpy(p.D_seq[s].copy()).to(dev) for s in range(nsys)]
    b_dev = torch.from_numpy(p.b).to(dev)
    x_dev = torch.empty_like(b_dev)

    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    cfg_over = json.loads(os.environ["AMGF_BENCH_CONFIG"]) if os.environ.get("AMGF_BENCH_CONFIG") else None
    g = AMGF.from_problem(p, D=p.D_seq[rank % nsys], stream=stream, config=cfg_over)
    t1.record(stream); t1.synchronize()
    full_setup_ms = t0.elapsed_time(t1)

    def step(k):
        s = system_of(rank, world, k, nsys)
        g.update_D(D_dev[s])
        _, rep = g.pcg(b_dev, rtol=p.rtol, max_it=5000, out=x_dev)
        return s, rep

    for k in range(args.warmup):
        step(k)
    # per-phase split (untimed probe, one system): numeric setup vs solve
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); g.update_D(D_dev[0]); e1.record(stream); e1.synchronize()
    upd_ms = e0.elapsed_time(e1)
    upd_breakdown = g.setup_times()

    launches0 = g.launches
    clocks = Clocks(local_rank)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    torch.cuda.nvtx.range_push("bench_timed")  # for ncu --nvtx-include "bench_timed/" (profiles/ launch list)
    iters, solve_ms, systems = [], [], []
    for k in range(args.steps):
        s, rep = step(args.warmup + k)
        iters.append(rep["iterations"]); solve_ms.append(rep["solve_ms"]); systems.append(s)
        if not rep["converged"]:
            raise RuntimeError(f"system {s} did not converge: {rep}")
    torch.cuda.nvtx.range_pop()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1)
    launches = g.launches - launches0
    elapsed = max_over_ranks(elapsed, world, dev)

    # ---- e2e: same metric through the public API with host buffers (pinned), copies inside the region
    D_host = [torch.from_numpy(p.D_seq[s].copy()).pin_memory() for s in range(nsys)]
    b_host = torch.from_numpy(p.b.copy()).pin_memory()
    x_host = torch.empty(p.n, dtype=torch.float64).pin_memory()
    D_stage = torch.empty(p.m, dtype=torch.float64, device=dev)
    ke = args.steps  # the same systems as the timed region (e2e is comparable with value)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ee0 = torch.cuda.Event(enable_timing=True); ee1 = torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    for k in range(ke):
        s = system_of(rank, world, args.warmup + k, nsys)
        D_stage.copy_(D_host[s], non_blocking=True)
        g.update_D(D_stage)
        g.pcg_host(b_host, x_host, rtol=p.rtol)
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1)
    e2e_ms = max_over_ranks(e2e_ms, world, dev)

    # ---- kernel-level roofline: fine-level SpMV (dominant kernel family) and whole V-cycle
    xr = torch.randn(p.n, dtype=torch.float64, device=dev)
    yr = torch.empty_like(xr)
    for _ in range(3):
        g.spmv(xr, 0, out=yr)
    nrep = 30
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(nrep):
        g.spmv(xr, 0, out=yr)
    a1.record(stream); a1.synchronize()
    spmv_ms = a0.elapsed_time(a1) / nrep
    for _ in range(2):
        g.vcycle(xr, out=yr)
    v0 = torch.cuda.Event(enable_timing=True); v1 = torch.cuda.Event(enable_timing=True)
    nv = 20
    v0.record(stream)
    for _ in range(nv):
        g.vcycle(xr, out=yr)
    v1.record(stream); v1.synchronize()
    vcycle_ms = v0.elapsed_time(v1) / nv
    ap0 = torch.cuda.Event(enable_timing=True); ap1 = torch.cuda.Event(enable_timing=True)
    ap0.record(stream)
    for _ in range(10):
        g.apply(xr, out=yr)
    ap1.record(stream); ap1.synchronize()
    apply_ms = ap0.elapsed_time(ap1) / 10

    peak, peak_src = peaks()
    sb = spmv_bytes(g)
    vb = level_bytes(g)
    filt_bytes = 2 * g.nc * (g.bw + 1) * 8
    apply_bytes = 2 * vb + sb + filt_bytes + 6 * 8 * p.n
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "spmv_traffic.json")
    if os.path.exists(tpath):
        try:
            tr = json.load(open(tpath))
            # the capture is of one workload: only report it for that workload (same algorithmic bytes)
            if tr.get("algorithmic_bytes_per_launch") == sb:
                traffic = tr.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    spmv_gbs = sb / (spmv_ms * 1e-3) / 1e9
    res = {
        "metric": METRIC,
        "value": elapsed / (args.steps * world),
        "unit": "ms/system",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed / args.steps,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (amgf_gen: seeded two-block Q1 elasticity + node-on-segment contact, DESIGN.md section 4)",
        "config": dict(bench_config(args.cfg, p, g.nc, g.config, world),
                       levels=[(L["nodes"] * L["b"]) for L in g.levels], band_width_Aw=g.bw),
        "pcg_iterations": iters,
        "systems": systems,
        "solve_ms_per_system": solve_ms,
        "numeric_setup_ms": upd_ms,
        "numeric_setup_breakdown_ms": upd_breakdown,
        "full_setup_ms": full_setup_ms,
        "vcycle_ms": vcycle_ms,
        "vcycle_gbs": vb / (vcycle_ms * 1e-3) / 1e9,
        "vcycle_frac_of_measured_peak": vb / (vcycle_ms * 1e-3) / 1e9 / peak,
        "vcycle_frac_of_8TBs": vb / (vcycle_ms * 1e-3) / 1e9 / 8000.0,
        "apply_ms": apply_ms,
        "apply_gbs": apply_bytes / (apply_ms * 1e-3) / 1e9,
        "roofline": {"kernel": "k_sell<3,3> (fine-level S SpMV, SELL-32)", "bound": "hbm",
                     "achieved": spmv_gbs, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": spmv_gbs / peak, "traffic": traffic, "algorithmic_bytes_per_launch": sb,
                     "avg_launch_ms": spmv_ms},
        "e2e": {"value": e2e_ms / (ke * world), "unit": "ms/system", "h2d_bytes_per_step": 8 * (p.m + p.n),
                "d2h_bytes_per_step": 8 * p.n},
        "gpu_launches": launches,
        "clocks": clk,
    }
    return res, p


def bench_config(cfg, p, nc, c, world):
    """The `config` object both arms print (c: the solver configuration, attribute access)."""
    return {"workload": f"cfg{cfg}: two-block N={p.N}, n={p.n} dofs, m={p.m}, n_c={nc}, "
                        f"{p.D_seq.shape[0]}-system IP-like D sequence, rtol={p.rtol}",
            "l2": (f"inputs larger than L2 (fine operator {p.K_col.size * 76 / 1e9:.2f} GB + hierarchy)"
                   if p.K_col.size * 76 > 126e6 else "L2-resident workload (parity case, not a bench line)"),
            "parallelism": f"replicas x{world}",
            "smoother": (f"chebyshev degree {c.cheb_degree} on [1/{c.cheb_ratio:g}, 1] of D_l1^-1 A (DESIGN R18)"
                         if c.smoother == 1 else "l1-jacobi"),
            "sweeps": [c.pre_sweeps, c.post_sweeps]}


def oracle_iterations(cfg, systems):
    """The oracle's OWN PCG iteration counts for these systems, from its cached full-size runs
    (tests/golden/oracle/, written by tools/oracle_golden.py with the plain oracle only)."""
    out = []
    for s in systems:
        path = os.path.join(ROOT, "tests", "golden", "oracle", f"cfg{cfg}_s{s}.json")
        if not os.path.exists(path):
            return None
        out.append(json.load(open(path))["pcg"]["iterations"])
    return out


def _chol_fma(n):
    """Fused multiply-adds of the oracle's dense left-looking Cholesky (orc_cholesky_dense) of order n:
    column j costs j for the pivot and j for each of its n-1-j sub-diagonal entries."""
    j = np.arange(n, dtype=np.float64)
    return float(np.sum(j * (n - j)))


class OracleSample:
    """Bounded timing of the oracle as it stands (one host core) on the full-size workload p.

    Measured here: the setup without the dense A_w factor (S = K + J^T D J and the AMG hierarchy, full size),
    the dense Cholesky on an n0 x n0 SPD sample (its cost is data-independent: no pivoting, no zero
    skipping), one V-cycle, one S SpMV and one dense TRSV pair of the full order n_c.  A system then costs
    setup + Cholesky(n_c) [scaled by the exact FMA count] + iterations x (2 V-cycles + 3 S-sized passes
    (S x1, the thin residual's loop over S, S p) + TRSV pair), with the oracle's own iteration count from its
    cached full-size runs -- no number from the GPU path."""

    def __init__(self, p, n0=2000):
        import oracle
        oracle.build()
        self.p = p
        t = time.perf_counter()
        self.o = oracle.Oracle.from_problem(p, factor_filter=0)
        self.t_setup = time.perf_counter() - t
        self.nc = self.o.nc
        self.bw = int(self.o.get(26)[0])
        rng = np.random.default_rng(0)
        n0 = min(n0, max(self.nc, 1))
        A = rng.standard_normal((n0, n0))
        A = A @ A.T + n0 * np.eye(n0)
        t = time.perf_counter(); oracle.cholesky(A); t_c = time.perf_counter() - t
        self.n0 = n0
        self.t_chol = t_c * _chol_fma(self.nc) / _chol_fma(n0) if self.nc else 0.0
        Lt = np.tril(rng.random((self.nc, self.nc))) + self.nc * np.eye(self.nc)
        v = rng.standard_normal(self.nc)
        t = time.perf_counter(); oracle.chol_solve(Lt, v); self.t_trsv = time.perf_counter() - t
        del Lt
        self.x = rng.standard_normal(p.n)
        self.sample_iteration()

    def sample_iteration(self):
        t = time.perf_counter(); self.o.vcycle(self.x); self.t_v = time.perf_counter() - t
        t = time.perf_counter(); self.o.spmv(self.x); self.t_s = time.perf_counter() - t
        return self.per_iteration()

    def per_iteration(self):
        return 2 * self.t_v + 3 * self.t_s + self.t_trsv

    def per_system_s(self, iters):
        return self.t_setup + self.t_chol + iters * self.per_iteration()

    def sample_text(self, iters_src):
        return (f"oracle (plain C, 1 core) on the full {self.p.name} system: measured setup without "
                f"the dense A_w factor {self.t_setup:.1f} s, Cholesky of a {self.n0}^2 SPD sample scaled by the exact "
                f"FMA count to n_c={self.nc} -> {self.t_chol:.0f} s, V-cycle {self.t_v:.2f} s, S SpMV {self.t_s:.3f} s, "
                f"TRSV pair {self.t_trsv:.2f} s; per system = setup + Cholesky + iterations x (2 V + 3 S passes + TRSV "
                f"pair) with {iters_src}.  Full-system oracle runs (tests/golden/oracle/*.json times_s) took "
                f"{_golden_full_time(self.p)}")


def _golden_full_time(p):
    cfg = p.name[3:] if p.name.startswith("cfg") else "?"
    ts = []
    cpu = "?"
    for s in range(p.D_seq.shape[0]):
        path = os.path.join(ROOT, "tests", "golden", "oracle", f"cfg{cfg}_s{s}.json")
        if os.path.exists(path):
            r = json.load(open(path))
            ts.append(r["times_s"]["setup_total"] + r["times_s"]["pcg"])
            cpu = r["host"]["cpu"]
    if not ts:
        return "n/a"
    return f"{statistics.mean(ts):.0f} s per system on average ({len(ts)} systems, {cpu}, shared with other runs)"


def cpu_baseline(p, cfg, systems):
    """GPU arm's cpu_baseline: the oracle, bounded sample (OracleSample), on the systems the timed region solved."""
    iters = oracle_iterations(cfg, systems)
    if iters is None:
        return {"value": None, "unit": "ms/system", "cores": 1, "kind": "oracle",
                "sample": "oracle iteration counts for these systems are not cached (tools/oracle_golden.py)"}
    smp = OracleSample(p)
    v = statistics.mean(smp.per_system_s(i) for i in iters) * 1e3
    return {"value": v, "unit": "ms/system", "cores": 1, "kind": "oracle",
            "sample": smp.sample_text(f"the oracle's own iteration counts (mean {statistics.mean(iters):.1f})"),
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" (nproc {os.cpu_count()})"
    except Exception:
        pass
    return f"nproc {os.cpu_count()}"


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle (this tier has no reference implementation), same metric/config.
    Each step is a bounded sample (one V-cycle and one S SpMV re-timed) of one system of the sequence, in the
    same replica schedule as the GPU arm; setup and the Cholesky sample are timed once."""
    if rank != 0:
        return None
    import amgf_gen
    import oracle
    p = amgf_gen.config(args.cfg)
    nsys = p.D_seq.shape[0]
    smp = OracleSample(p)
    for _ in range(min(args.warmup, 1)):
        smp.sample_iteration()
    vals, its = [], []
    for k in range(args.steps):
        s = system_of(0, 1, args.warmup + k, nsys)
        it = oracle_iterations(args.cfg, [s])
        if it is None:
            raise RuntimeError(f"no cached oracle run for cfg{args.cfg} system {s} (tools/oracle_golden.py)")
        smp.sample_iteration()
        vals.append(smp.per_system_s(it[0]) * 1e3)
        its.append(it[0])
    v = statistics.mean(vals)
    sample = smp.sample_text(f"the oracle's own iteration counts per system {its}")
    cfgns = types.SimpleNamespace(**oracle.DEFAULTS)
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms/system", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(bench_config(args.cfg, p, smp.nc, cfgns, world),
                           levels=[(L["nodes"] * L["b"]) for L in smp.o.levels], band_width_Aw=smp.bw),
            "pcg_iterations": its,
            "cpu_baseline": {"value": v, "unit": "ms/system", "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": _cpu_model()},
            "e2e": {"value": v, "unit": "ms/system", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="amgf", choices=["amgf", "reference"])
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3 and args.impl == "amgf":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out))
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res, p = run_amgf(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            res["cpu_baseline"] = cpu_baseline(p, args.cfg, res["systems"])
        print(json.dumps(res))
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
