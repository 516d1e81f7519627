"""Markdown tables of the iteration study (profiles/r02_n2_grid.jsonl, r02_n2_cfg4.jsonl from tools/n2_study.py;
profiles/r02_n2_oracle.jsonl from tools/n2_oracle.py).  Prints to stdout."""
import json
import os
import sys

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def load(name):
    path = os.path.join(P, name)
    return [json.loads(l) for l in open(path)] if os.path.exists(path) else []


orc = {(d["N"], d["matching"], d["D_max"]): d["k_amgf_oracle"] for d in load("r02_n2_oracle.jsonl")}
print("| N | interface | D_max | AMGF-PCG (GPU) | oracle | AMG-PCG | kappa(MS) | contact-free AMG-PCG | beta | bound k | 2(beta+3) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for d in load("r02_n2_grid.jsonl"):
    key = (d["N"], d["matching"], d["D_max"])
    o = orc.get(key)
    amg = f"{d['k_amg']}" + ("" if d.get("amg_converged", True) else " (cap)")
    print(f"| {d['N']} | {'matching' if d['matching'] else 'offset'} | {d['D_max']:.0e} | {d['k_amgf']} | "
          f"{'=' if o == d['k_amgf'] else (o if o is not None else '-')} | {amg} | {d['kappa_MS']:.1f} | "
          f"{d['k_amg_contact_free']} | {d['beta']:.2f} | {d['k_bound']:.1f} | {2 * (d['beta'] + 3):.1f} |")
print()
print("| case | N | inclusion | rtol | D_max | AMGF-PCG | kappa(MS) | contact-free AMG-PCG | beta | bound k |")
print("|---|---|---|---|---|---|---|---|---|---|")
for d in load("r02_n2_cfg4.jsonl"):
    print(f"| {d['case']} | {d['N']} | {d['inclusion']} | {d['rtol']:.0e} | {d['D_max']:.0e} | {d['k_amgf']} | "
          f"{d['kappa_MS']:.1f} | {d['k_amg_contact_free']} | {d['beta']:.2f} | {d['k_bound']:.1f} |")
