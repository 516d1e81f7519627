"""Cached oracle results for the full-size parity tests (cfg 3's ten systems, cfg 4).

Runs the UNCHANGED plain oracle (oracle/, dense A_w Cholesky, default configuration) on one system of a
BASELINE config and writes tests/golden/oracle/cfg{c}_s{s}.json: digests (amgf_gen.digest) of every
hierarchy array, of the A_w matrix and of its dense Cholesky factor, of S x, B x and M x for a seeded
probe x, and the PCG result (iterations, final relative preconditioned residual, solution digest and
sampled entries), plus the oracle's own wall times per phase on this host.  Imports only oracle/ and
amgf_gen/: no value here comes from the CUDA path.

    python tools/oracle_golden.py --cfg 3 --system 0          # one system (minutes at cfg 3)
    python tools/oracle_golden.py --all --jobs 6               # cfg 4 system 0 + cfg 3 systems 0-9
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "oracle")


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_one(cfg: int, system: int) -> dict:
    import numpy as np
    import amgf_gen
    import oracle
    from amgf_gen.digest import digest, hierarchy_items, probe_vector, sample_hex

    p = amgf_gen.config(cfg)
    D = p.D_seq[system]
    t0 = time.perf_counter()
    o = oracle.Oracle.from_problem(p, D=D)
    t_setup = time.perf_counter() - t0
    rec = dict(cfg=cfg, system=system, n=p.n, m=p.m, nc=o.nc, nco=o.nco, nlev=o.nlev, levels=o.levels,
               oracle_config={k: (hex(v) if k == "agg_seed" else v) for k, v in o.cfg.items()},
               oracle_cflags=oracle.CFLAGS, D_digest=digest(D))
    arrays = {key: digest(o.get(w, l)) for key, w, l in hierarchy_items(o.nlev)}
    arrays["pi"] = digest(o.get(25))
    rec["bw"] = int(o.get(26)[0])
    if o.nc:
        arrays["A_w"] = digest(o.get(21))
        arrays["L_w"] = digest(o.get(22))
    arrays["coarsest_L"] = digest(o.get(24))
    rec["arrays"] = arrays
    seed = 1000 + 17 * cfg + system
    x = probe_vector(p.n, seed)
    rec["probe_seed"] = seed
    t = time.perf_counter(); y = o.spmv(x); t_spmv = time.perf_counter() - t
    t = time.perf_counter(); v = o.vcycle(x); t_v = time.perf_counter() - t
    t = time.perf_counter(); z = o.apply(x); t_apply = time.perf_counter() - t
    rec["probe"] = dict(spmv=digest(y), vcycle=digest(v), apply=digest(z),
                        apply_samples=sample_hex(z))
    t = time.perf_counter()
    xs, info = o.pcg(p.b, rtol=p.rtol, maxit=5000)
    t_pcg = time.perf_counter() - t
    rec["pcg"] = dict(rtol=p.rtol, iterations=info["iterations"], converged=bool(info["converged"]),
                      relres=float(info["relres"]).hex(), relres_float=float(info["relres"]),
                      x=digest(xs), x_samples=sample_hex(xs), history=digest(info["history"]))
    rec["times_s"] = dict(setup_total=t_setup, **o.times(), spmv=t_spmv, vcycle=t_v, apply=t_apply,
                          pcg=t_pcg, pcg_per_iteration=t_pcg / max(1, info["iterations"]))
    rec["host"] = dict(cpu=cpu_model(), nproc=os.cpu_count(), threads_used=1)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int)
    ap.add_argument("--system", type=int, default=0)
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--jobs", type=int, default=4)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if a.all:
        todo = [(4, 0)] + [(3, s) for s in range(9, -1, -1)]
        todo = [t for t in todo if not os.path.exists(os.path.join(OUT, f"cfg{t[0]}_s{t[1]}.json"))]
        procs = []
        while todo or procs:
            while todo and len(procs) < a.jobs:
                c, s = todo.pop(0)
                log = open(os.path.join(OUT, f".cfg{c}_s{s}.log"), "w")
                procs.append(subprocess.Popen([sys.executable, __file__, "--cfg", str(c), "--system", str(s)],
                                              stdout=log, stderr=subprocess.STDOUT))
            time.sleep(5)
            procs = [q for q in procs if q.poll() is None]
        return
    rec = run_one(a.cfg, a.system)
    path = os.path.join(OUT, f"cfg{a.cfg}_s{a.system}.json")
    with open(path + ".tmp", "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    os.replace(path + ".tmp", path)
    print(path, rec["pcg"]["iterations"], rec["times_s"])


if __name__ == "__main__":
    main()
