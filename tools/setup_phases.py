"""Wall time of every phase of amgf_setup at a config (AMGF_SETUP_TIMING=1), second setup of the process."""
import os
import sys
import time

os.environ["AMGF_SETUP_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
for k in range(2):
    print(f"--- setup {k}", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = AMGF.from_problem(p)
    torch.cuda.synchronize()
    print(f"setup wall {1e3 * (time.perf_counter() - t):.1f} ms", file=sys.stderr, flush=True)
    g.close()
