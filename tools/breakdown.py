"""In-graph device-time breakdown of one solve by (kernel class, level), via the library's
profiling events (sr_fmg_profile_select/read).  GPU box only.

    python tools/breakdown.py [--config C3] [--dtype f64]
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
from paper_1406_7808_b200 import Solver, kernel_names  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--dtype", default="f64")
ap.add_argument("--stencil", default="7pt")
a = ap.parse_args()
n, M, seg, buf, K, rhs = WORKLOADS[a.config]
h = 1.0 / n[0] if a.config != "P27" else 2.0 / n[0]
s = Solver(n, M, seg=seg, buffer=buf, K=K, dtype=a.dtype, h=h, stencil=a.stencil)
f = torch.from_numpy(W.make_rhs(rhs, n, h=h).astype(np.float64 if a.dtype == "f64" else np.float32)).cuda()
u = torch.empty_like(f)
for _ in range(3):
    s.solve(f, u)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    s.solve(f, u)
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1) / 10
names = kernel_names()
rows = []
for c in range(len(names)):
    for lvl in range(M + 1):
        s.profile_select(c, lvl)
        s.solve(f, u)
        torch.cuda.synchronize()
        ms = []
        for _ in range(3):
            s.solve(f, u)
            torch.cuda.synchronize()
            t, b, nl = s.profile_read()
            ms.append(t)
        if nl:
            rows.append((names[c], lvl, nl, min(ms), b))
s.profile_select(-1, -1)
print(f"solve {total:.3f} ms (graph replay, mean of 10)")
acc = 0.0
for name, lvl, nl, t, b in sorted(rows, key=lambda r: -r[3]):
    acc += t
    print(f"{name:14s} l={lvl} launches={nl:3d} {t:8.3f} ms  {b / 1e9:7.3f} GB  "
          f"{(b / 1e9) / (t / 1e3) if t > 0 else 0:7.0f} GB/s")
print(f"sum of kernel intervals {acc:.3f} ms; rest (gaps) {total - acc:.3f} ms")
