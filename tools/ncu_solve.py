"""Profiling driver for ncu (run under gpurun; never a bench number).

    ncu --profile-from-start off ... python tools/ncu_solve.py [--config C3] [--what solve|cheb]

Builds the C3 solver, runs two warm solves, then opens the CUDA profiler range around
either one whole solve (launch list) or one degree-2 Chebyshev smoothing of the finest
level (the dominant kernel, for `ncu --set full`).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from bench import WORKLOADS  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--what", default="solve", choices=["solve", "cheb", "restrict", "prolong", "correct"])
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--level", type=int, default=-1, help="level of the single operation (default M)")
ap.add_argument("--stencil", default="7pt")
a = ap.parse_args()
n, M, seg, buf, K, rhs = WORKLOADS[a.config]
h = 1.0 / n[0] if a.config != "P27" else 2.0 / n[0]
s = Solver(n, M, seg=seg, buffer=buf, K=K, dtype=a.dtype, use_graph=bool(a.graph), h=h,
           stencil=a.stencil)
f = torch.from_numpy(W.make_rhs(rhs, n, h=h).astype(np.float64 if a.dtype == "f64" else np.float32)).cuda()
u = torch.empty_like(f)
s.solve(f, u)
s.solve(f, u)
torch.cuda.synchronize()
lv = M if a.level < 0 else a.level
torch.cuda.profiler.start()
if a.what == "solve":
    s.solve(f, u)
elif a.what == "cheb":
    s.debug_op(0, lv, 2, f)
elif a.what == "restrict":
    s.debug_op(1, lv, 0, f)
elif a.what == "prolong":
    s.debug_op(3, lv, 0, f)
elif a.what == "correct":
    s.debug_op(4, lv, 0, f)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
