"""C5 at full size on one B200 (GPU box; writes gpurun_out/r2_c5_sweep.json): the SR level
count sweep K in {2, 3, 4, 5} for both segment sizes S in {32, 128} (BASELINE configs[4]:
"sweep of SR level count to expose the extra parameter's effect on accuracy").

Per (S, K): device time of one FMG+SR solve (captured graph, CUDA events, mean of 5 after 2
warm solves), fine cells/s, and the algebraic error against the exact discrete solution
u_h* = A^-1 f.  The bump rhs has no continuum solution, so u_h* is computed here by the
library's conventional V-cycle solver (sr_fmg_vsolve, K = 0) iterated to a relative residual
of 1e-12 -- a reported accuracy figure, not a parity check (parity at these parameter sets is
tests/test_gpu_parity.py at 256^3 against the oracle).  e_ratio = e_alg(SR) / e_alg(FMG)
with FMG = the conventional K = 0 solve of the same f (PAPER.md:262-264's e_r uses the
continuum error instead; the algebraic one isolates the SR error source).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

N, M, J = 1024, 9, 2
n = (N, N, N)
t0 = time.time()
f = torch.from_numpy(W.make_rhs("bumps", n)).cuda()
print(f"rhs {time.time() - t0:.1f} s", flush=True)


def timed(s, f, u, reps=5):
    for _ in range(2):
        s.solve(f, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s.solve(f, u)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def errs(u, ref):
    d = u - ref
    return float(d.abs().max()), float(torch.linalg.vector_norm(d) / torch.linalg.vector_norm(ref))


with Solver(n, M, K=0) as s:
    t0 = time.time()
    ustar, cyc, rel = s.vsolve(f, rtol=1e-12, maxit=60)
    torch.cuda.synchronize()
    print(f"u_h*: {cyc} V-cycles, relres {rel:.2e}, {time.time() - t0:.1f} s", flush=True)
    u = torch.empty_like(f)
    ms_fmg = timed(s, f, u)
    e_fmg_inf, e_fmg_l2 = errs(u, ustar)
del u
rows = [dict(S=0, K=0, pN0V=None, ms=ms_fmg, cells_per_s=N ** 3 / (ms_fmg / 1e3),
             e_alg_inf=e_fmg_inf, e_alg_rel_l2=e_fmg_l2, e_ratio_inf=1.0)]
print(f"FMG (K = 0): {ms_fmg:.2f} ms  e_alg_inf {e_fmg_inf:.3e}", flush=True)
for S in (128, 32):
    for K in (2, 3, 4, 5):
        with Solver(n, M, seg=S, buffer=J, K=K) as s:
            u = torch.empty_like(f)
            ms = timed(s, f, u)
            ei, el = errs(u, ustar)
            del u
        rows.append(dict(S=S, K=K, pN0V=S >> K, ms=ms, cells_per_s=N ** 3 / (ms / 1e3),
                         e_alg_inf=ei, e_alg_rel_l2=el, e_ratio_inf=ei / e_fmg_inf))
        print(f"S {S:3d} K {K}: {ms:7.2f} ms  {N ** 3 / (ms / 1e3):.3e} cells/s  "
              f"e_alg_inf {ei:.3e}  ratio {ei / e_fmg_inf:.2f}", flush=True)
out = dict(config="C5: 1024^3, M = 9, J = 2, f = 16 Gaussian bumps (R22), fp64, 1 B200",
           u_h_star=dict(method="sr_fmg_vsolve (K = 0) to relative residual 1e-12",
                         cycles=cyc, relres=rel),
           rows=rows)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "r2_c5_sweep.json"), "w") as fh:
    json.dump(out, fh, indent=1)
