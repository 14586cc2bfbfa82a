"""Time single schedule ops (debug_op) at one level of the C3 solver with CUDA events.

    SR_FMG_CHEB2_VARIANT=1 python tools/bench_ops.py --op cheb2 --level 8
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--op", default="cheb2")
ap.add_argument("--level", type=int, default=-1)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n, M, seg, buf, K, rhs = WORKLOADS[a.config]
s = Solver(n, M, seg=seg, buffer=buf, K=K, dtype=a.dtype, use_graph=False)
f = torch.from_numpy(W.make_rhs(rhs, n).astype(np.float64 if a.dtype == "f64" else np.float32)).cuda()
u = torch.empty_like(f)
s.solve(f, u)
torch.cuda.synchronize()
l = (M - 1 if a.op == 'tau' else M) if a.level < 0 else a.level
op, deg = {"cheb1": (0, 1), "cheb2": (0, 2), "restrict": (1, 0), "tau": (2, 0),
           "prolong": (3, 0), "correct": (4, 0)}[a.op]
for _ in range(2):
    s.debug_op(op, l, deg, f)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    s.debug_op(op, l, deg, f)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
li = s.level(l)
print(f"variant={os.environ.get('SR_FMG_CHEB2_VARIANT', '0')} op={a.op} level={l} "
      f"E={li.storage_ext} {ms:.3f} ms per op")
