"""Per-launch completion timeline of one cfg 3 amgf_update_D on both streams (AMGF_LAUNCH_TIMELINE=1, no profiler)."""
import json
import os
import sys

os.environ["AMGF_LAUNCH_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(3)
cfg_over = json.loads(os.environ["AMGF_TIME_CONFIG"]) if os.environ.get("AMGF_TIME_CONFIG") else None
g = AMGF.from_problem(p, D=p.D_seq[0], config=cfg_over)
D = torch.from_numpy(p.D_seq[5]).cuda()
for k in range(3):
    print(f"--- update_D {k}", file=sys.stderr, flush=True)
    g.update_D(D)
    torch.cuda.synchronize()
