"""Debug driver for the fused passes (GPU box): one eager solve, optional oracle check.

    SR_FMG_SYNC=1 python tools/dbg_pass.py MODE K N [ref]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

mode, K, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = (N, N, N)
M = {128: 6, 256: 7, 512: 8}[N]
f = W.make_rhs("manufactured+noise", n)
os.environ["SR_FMG_PASS"] = mode
graph = os.environ.get("DBG_GRAPH", "0") == "1"
with Solver(n, M, seg=64, buffer=2, K=K, use_graph=graph) as s:
    ft = torch.from_numpy(f).cuda()
    for _ in range(int(os.environ.get("DBG_REPS", "1"))):
        u = s.solve(ft)
    torch.cuda.synchronize()
    u = u.double().cpu().numpy()
print("solved", sys.argv, flush=True)
if len(sys.argv) > 4:
    ref = O.solve(f, O.Config(n=n, M=M, seg=64, buffer=2, K=K))
    print("rel", np.linalg.norm(u - ref) / np.linalg.norm(ref))
