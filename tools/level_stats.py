import sys, numpy as np
sys.path.insert(0,'/root/repo')
import amgf_gen
from paper_2505_18576_b200 import AMGF
p=amgf_gen.config(3); g=AMGF.from_problem(p)
for l in range(g.nlev-1):
    rp=g.get(6,l).astype(np.int64); ln=np.diff(rp)
    pp=g.get(3,l).astype(np.int64); lp=np.diff(pp)
    ap=g.get(0,l).astype(np.int64); la=np.diff(ap)
    print(l, "R rows", len(ln), "len mean %.1f max %d p99 %d" % (ln.mean(), ln.max(), np.percentile(ln,99)),
          "| P rows len mean %.1f max %d" % (lp.mean(), lp.max()), "| A rows mean %.1f p50 %d p90 %d p99 %d max %d" % (la.mean(), np.percentile(la,50), np.percentile(la,90), np.percentile(la,99), la.max()))
