"""Accuracy of the GPU solve at the BASELINE configs (GPU box; writes
gpurun_out/r2_accuracy.json, the source of BASELINE.md §4).

Per (config, dtype): rel-L2 against the oracle run on the same f (fp64 oracle; R23), and
the north-star error ratios: e_SR = ||u_SR - u||_inf and e_FMG (K = 0)
against the manufactured u, e_disc = ||u_h* - u||_inf with u_h* = A^-1 f (DST), e_r =
e_SR / e_FMG, and the algebraic errors ||u - u_h*||_inf / e_disc.  For the bump rhs (C5)
there is no continuum solution: only the algebraic errors against u_h*.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402
from tests import pins  # noqa: E402

CASES = [  # name, n, M, seg, J, K, rhs
    ("C1", 32, 4, 16, 2, 2, "manufactured"),
    ("C2-J1", 128, 6, 32, 1, 3, "manufactured"),
    ("C2-J2", 128, 6, 32, 2, 3, "manufactured"),
    ("C2-J4", 128, 6, 32, 4, 3, "manufactured"),
    ("C3", 512, 8, 64, 2, 4, "manufactured+noise"),
    ("C5@256-S32-K2", 256, 7, 32, 2, 2, "bumps"),
    ("C5@256-S32-K3", 256, 7, 32, 2, 3, "bumps"),
    ("C5@256-S128-K4", 256, 7, 128, 2, 4, "bumps"),
    ("C5@256-S128-K5", 256, 7, 128, 2, 5, "bumps"),
]


def gpu(f, N, M, seg, J, K, dtype):
    npd = np.float64 if dtype == "f64" else np.float32
    with Solver((N,) * 3, M, seg=seg, buffer=J, K=K, dtype=dtype) as s:
        return s.solve(torch.from_numpy(f.astype(npd)).cuda()).double().cpu().numpy()


def main():
    out = {}
    for name, N, M, seg, J, K, rhs in CASES:
        t0 = time.time()
        n, h = (N,) * 3, 1.0 / N
        f = W.make_rhs(rhs, n)
        ref = O.solve(f, O.Config(n=n, M=M, seg=seg, buffer=J, K=K))
        ustar = pins.dst_solve(f, h)
        row = {"n": N, "M": M, "seg": seg, "J": J, "K": K, "rhs": rhs}
        manu = rhs.startswith("manufactured")
        if manu:
            fm = W.manufactured_f(n, h)
            ue = W.manufactured_u(n, h)
            um = pins.dst_solve(fm, h)
            row["e_disc_inf"] = float(np.abs(um - ue).max())
        for dt in ("f64", "f32"):
            u = gpu(f, N, M, seg, J, K, dt)
            d = {"rel_l2_vs_oracle": float(np.linalg.norm(u - ref) / np.linalg.norm(ref)),
                 "e_alg_inf": float(np.abs(u - ustar).max()),
                 "e_alg_rel_l2": float(np.linalg.norm(u - ustar) / np.linalg.norm(ustar))}
            if manu:
                usr = gpu(fm, N, M, seg, J, K, dt)
                ufm = gpu(fm, N, M, 0, 0, 0, dt)
                d["e_sr_inf"] = float(np.abs(usr - ue).max())
                d["e_fmg_inf"] = float(np.abs(ufm - ue).max())
                d["e_r"] = d["e_sr_inf"] / d["e_fmg_inf"]
                d["e_sr_over_disc"] = d["e_sr_inf"] / row["e_disc_inf"]
                d["e_sr_alg_over_disc"] = float(np.abs(usr - um).max()) / row["e_disc_inf"]
            row[dt] = d
        row["oracle_rel_l2_vs_dst"] = float(np.linalg.norm(ref - ustar) / np.linalg.norm(ustar))
        row["seconds"] = time.time() - t0
        out[name] = row
        print(name, json.dumps(row), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "r2_accuracy.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
