"""Bounds-check run (the pool has no compute-sanitizer): with AMGF_GUARD=1 every internal allocation gets a
4 KB guard zone; this drives every solve-side code path -- setup, update_D, V-cycle, AMGF apply, SpMV per
level, PCG (device loop; host loop with AMGF_HOST_LOOP=1), both smoothers, Z = NULL, a one-level hierarchy,
an export/import round trip -- on small configurations and prints the number of overwritten guard zones
(must be 0) as one JSON line."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402


def drive(g, p, rng):
    r = rng.standard_normal(g.n)
    z = g.apply(r).cpu().numpy()
    g.vcycle(r)
    for l in range(g.nlev):
        g.spmv(rng.standard_normal(g.levels[l]["nodes"] * g.levels[l]["b"]), l)
    g.pcg(p.b, rtol=p.rtol)
    g.pcg(p.b, rtol=p.rtol, precond="amg", max_it=50)
    return r, z


out = {}
rng = np.random.default_rng(0)
for name, p, kw in (("cfg0", amgf_gen.config(0), {}), ("cfg1", amgf_gen.config(1), {}),
                    ("cfg2", amgf_gen.config(2), {}),
                    ("cfg1_l1", amgf_gen.config(1), dict(config=dict(smoother=0))),
                    ("tiny_Znull", amgf_gen.generate(3, matching=False, e_max=[8.0], seed=7),
                     dict(Z=None, config=dict(coarsest_size=16))),
                    ("tiny_1level", amgf_gen.generate(2), dict(config=dict(coarsest_size=10 ** 6)))):
    g = AMGF.from_problem(p, **kw)
    g.update_D(p.D_seq[-1])
    r, z = drive(g, p, rng)
    with tempfile.TemporaryDirectory() as d:
        g.export(d)
        h = AMGF.import_dir(d)
        assert np.array_equal(h.apply(r).cpu().numpy(), z)
        drive(h, p, rng)
        out[name + "_import"] = h.guard_violations()
    out[name] = g.guard_violations()
torch.cuda.synchronize()
print(json.dumps(out))
