"""Per-operation timestamps of the coarse-level executor (SR_FMG_CEXEC_PROF=1) for one C3 solve
without graph capture.  GPU box only; the times carry the synchronisation after each launch."""
import os
import sys

os.environ["SR_FMG_CEXEC_PROF"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n, M, seg, buf, K, rhs = WORKLOADS[cfg]
s = Solver(n, M, seg=seg, buffer=buf, K=K, use_graph=False)
f = torch.from_numpy(W.make_rhs(rhs, n)).cuda()
u = torch.empty_like(f)
s.solve(f, u)
torch.cuda.synchronize()
print("---- second solve ----", file=sys.stderr, flush=True)
s.solve(f, u)
torch.cuda.synchronize()
