"""Oracle confirmation of the N2 study's AMGF-PCG iteration counts (tools/n2_study.py grid): the plain oracle
(dense A_w factor) on the same cases, one process per (N, interface), rtol 1e-8.  Writes one JSON line per
case to stdout.  Usage: python tools/n2_oracle.py N matching(0/1)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import amgf_gen  # noqa: E402
import oracle  # noqa: E402

N, matching = int(sys.argv[1]), bool(int(sys.argv[2]))
p = amgf_gen.study_case(N, matching)
for s, e in enumerate(p.meta["e_max"]):
    t = time.perf_counter()
    o = oracle.Oracle.from_problem(p, D=p.D_seq[s])
    x, info = o.pcg(p.b, rtol=1e-8)
    print(json.dumps(dict(case=p.name, N=N, matching=matching, D_max=10.0 ** e, k_amgf_oracle=info["iterations"],
                          relres=float(info["relres"]).hex(), seconds=time.perf_counter() - t)), flush=True)
    del o
