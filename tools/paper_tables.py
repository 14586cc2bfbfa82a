"""e_r = ||e_SR||_inf / ||e_conv||_inf at the paper's Table 1-3 configurations
with the paper's 27-point operator on Omega = [0,2]x[0,1]^2 (R = (2,1,1)), the manufactured
u = prod(x_i^4 - R_i^2 x_i^2), F(1,2,2), a 4x2x2 "process" grid = 4x2x2 SR segments of
N_K = pN0V 2^K cells each (GPU box; writes profiles/r2_paper_tables.json).

Run: Table 1 column log2 pN0V = 2 (K = 4: 256x128x128) for every (A, B); Table 2 for pN0V =
4 (512x256x256); Table 3 (MBS, J_1 = 4, K = 4) for pN0V = 2, 4, 8 (up to 512x256x256).  The
other columns need 1024x512x512 with 256^3 segments or more (E > 256: not supported by
this build's 27-point kernels) or 4096x2048x2048.  Also: the Chebyshev interval's effect
on e_r (the paper does not state it; reading R28 uses [1/3, 1] lambda_max).  The coarsest grid is 2R =
4x2x2 cells (the paper's M = K + log2 pN0V + 2, would give
1x0.5x0.5 -- a garbled formula).
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

PAPER_T1 = {  # (A, B) -> [4(6), 3(5), 2(4)] (None = NA)
    (2, 0): [17, 7.2, 2.7], (2, 1): [2.9, 2.1, 1.2], (2, 2): [1.5, 1.2, None], (2, 3): [1.2, 1.1, None],
    (4, 0): [5.7, 2.6, 1.2], (4, 1): [2.0, 1.4, 1.0], (4, 2): [1.3, 1.1, None], (4, 3): [1.1, 1.0, None],
    (6, 0): [2.8, 1.4, 1.0], (6, 1): [1.5, 1.1, None], (6, 2): [1.3, 1.0, None], (6, 3): [1.1, None, None],
    (8, 0): [1.5, 1.1, 1.0], (8, 1): [1.3, 1.0, None], (8, 2): [1.1, 1.0, None], (8, 3): [1.0, None, None],
}
PAPER_T2 = {32: 1.02, 16: 1.05, 8: 1.13, 4: 1.28}     # pN0V -> e_r, A=8 B=0 K=5
PAPER_T3 = {64: 1.02, 32: 1.05, 16: 1.11, 8: 1.25, 4: 1.4, 2: 1.9}  # MBS J1=4 K=4


def grid(pn0v, K):
    NK = pn0v << K                      # fine cells per "process" per dimension
    n = (4 * NK, 2 * NK, 2 * NK)        # 4x2x2 process grid, R = (2,1,1), h = 1/(2 NK)
    M = int(np.log2(NK))                # coarsest grid 4x2x2 (2R cells): n / 2^M
    return n, M, NK, 1.0 / (2 * NK)


_cache = {}


def errors(pn0v, K, sched=None, conv=False, cheb=None):
    n, M, NK, h = grid(pn0v, K)
    key = (n, M)
    if key not in _cache:
        _cache.clear()
        torch.cuda.empty_cache()
        _cache[key] = (torch.from_numpy(W.manufactured_f(n, h)).cuda(),
                       torch.from_numpy(W.manufactured_u(n, h)).cuda())
    f, ue = _cache[key]
    kw = dict(h=h, stencil="27pt", cheb=cheb)
    if conv:
        s = Solver(n, M, K=0, **kw)
    else:
        s = Solver(n, M, seg=NK, K=K, sched=sched, **kw)
    with s:
        u = s.solve(f)
        e = float((u - ue).abs().max())
    return e


def main():
    out = {"operator": "27-point (R28), Omega = [0,2]x[0,1]^2, 4x2x2 segments, F(1,2,2)",
           "coarsest": "4x2x2 (2R)", "table1": {}, "table2": {}, "table3": {}}
    t0 = time.time()
    for pn0v, K, col in ((4, 4, 2),):
        ec = errors(pn0v, K, conv=True)
        for (A, B), pv in PAPER_T1.items():
            es = errors(pn0v, K, sched=(A, B))
            out["table1"][f"A{A}_B{B}_pN0V{pn0v}_K{K}"] = {
                "e_sr": es, "e_conv": ec, "e_r": es / ec, "paper": pv[col]}
            print(A, B, pn0v, K, es / ec, pv[col], flush=True)
    for pn0v in (4,):
        ec = errors(pn0v, 5, conv=True)
        es = errors(pn0v, 5, sched=(8, 0))
        out["table2"][f"pN0V{pn0v}"] = {"e_r": es / ec, "paper": PAPER_T2[pn0v]}
        print("T2", pn0v, es / ec, PAPER_T2[pn0v], flush=True)
    for pn0v in (2, 4, 8):
        ec = errors(pn0v, 4, conv=True)
        es = errors(pn0v, 4, sched=("mbs", 4))
        out["table3"][f"pN0V{pn0v}"] = {"e_r": es / ec, "paper": PAPER_T3[pn0v]}
        print("T3", pn0v, es / ec, PAPER_T3[pn0v], flush=True)
    out["interval"] = {}
    for lo, hi in ((1 / 3, 1.0), (1 / 4, 1.0), (1 / 2, 1.0), (0.1, 1.1), (0.2, 1.2)):
        ec = errors(4, 4, conv=True, cheb=(lo, hi))
        row = {"e_conv": ec}
        for A in (2, 8):
            row[f"e_r_A{A}_B0"] = errors(4, 4, sched=(A, 0), cheb=(lo, hi)) / ec
        out["interval"][f"{lo:.3g}-{hi:.3g}"] = row
        print("interval", lo, hi, row, flush=True)
    out["seconds"] = time.time() - t0
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "r2_paper_tables.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
