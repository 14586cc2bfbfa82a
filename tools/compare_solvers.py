"""The paper's solver comparison (Fig. conva/scaling/verrors) on one B200:
SR-FMG (C3), conventional FMG (K = 0) and the conventional V-cycle solver to a relative
residual of 1e-4, on the C3 problem (512^3, fp64, manufactured f, no noise so the error
against the manufactured u is the discretisation + algebraic error).

    python tools/compare_solvers.py [--n 512] > profiles/r1_solver_comparison.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
N = a.n
M = int(np.log2(N)) - 1
n = (N, N, N)
f = torch.from_numpy(W.make_rhs("manufactured", n)).cuda()
uex = torch.from_numpy(W.manufactured_u(n, 1.0 / N)).cuda()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps, out


res = {"grid": N, "M": M, "dtype": "f64", "rhs": "manufactured (no noise)"}
with Solver(n, M, seg=N // 8, buffer=2, K=4) as s:
    u = torch.empty_like(f)
    ms, _ = timed(lambda: s.solve(f, u))
    res["sr_fmg"] = {"K": 4, "seg": N // 8, "J": 2, "ms": ms,
                     "err_inf": float((u - uex).abs().max())}
with Solver(n, M, K=0) as s:
    u = torch.empty_like(f)
    ms, _ = timed(lambda: s.solve(f, u))
    res["conventional_fmg"] = {"ms": ms, "err_inf": float((u - uex).abs().max())}
    ms, out = timed(lambda: s.vsolve(f, u, rtol=1e-4, maxit=60))
    res["vcycle_rtol_1e-4"] = {"ms": ms, "cycles": out[1], "relres": out[2],
                               "err_inf": float((out[0] - uex).abs().max())}
print(json.dumps(res, indent=1))
