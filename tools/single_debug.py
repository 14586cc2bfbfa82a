"""Single-GPU solve of one grid shape with SR_FMG_TRACE/SR_FMG_SYNC (GPU box debugging)."""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

n = tuple(int(v) for v in sys.argv[1].split(","))
M, seg, K = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
solves = int(sys.argv[5]) if len(sys.argv) > 5 else 1
graph = len(sys.argv) > 6 and sys.argv[6] == "graph"
faulthandler.dump_traceback_later(25, exit=True)
f = W.make_rhs("manufactured+noise", n)
with Solver(n, M, seg=seg, buffer=2, K=K, use_graph=graph) as s:
    ft = torch.from_numpy(f).cuda()
    for i in range(solves):
        u = s.solve(ft).cpu().numpy()
        print("solve", i, "finite", bool(np.isfinite(u).all()), flush=True)
print("done", np.isfinite(u).all(), flush=True)
