"""Robustness sweep (GPU box): every (S, J, K, dtype) combination at 256^3 (and a few non-cubic
grids) must create, solve without a CUDA error, and agree with the unfused step kernels
(SR_FMG_FUSED=0) to rounding -- the launch-configuration limits of the fused kernels (shared
memory, row widths, grid sizes) are exercised where they are actually chosen."""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

grids = [((256, 256, 256), 7), ((512, 256, 128), 6), ((128, 256, 512), 6)]
fails, n_ok = [], 0
for (n, M), dt in itertools.product(grids, ("f64", "f32")):
    npd = np.float64 if dt == "f64" else np.float32
    f = torch.from_numpy(W.make_rhs("manufactured+noise", n).astype(npd)).cuda()
    for S, J, K in itertools.product((16, 32, 64, 128), (0, 1, 2, 3, 4), (1, 2, 3, 4)):
        if S % (1 << K) or any(d % S for d in n) or K > M:
            continue
        if n != (256, 256, 256) and (J not in (1, 2) or K not in (2, 4)):
            continue
        out = []
        try:
            for fu in ("1", "0"):
                os.environ["SR_FMG_FUSED"] = fu
                with Solver(n, M, seg=S, buffer=J, K=K, dtype=dt) as s:
                    out.append(s.solve(f).double())
            rel = float(torch.linalg.vector_norm(out[0] - out[1]) / torch.linalg.vector_norm(out[1]))
            tol = 1e-12 if dt == "f64" else 1e-5
            if not rel <= tol:
                fails.append((n, S, J, K, dt, f"rel {rel:.2e}"))
            else:
                n_ok += 1
        except Exception as e:  # noqa: BLE001
            fails.append((n, S, J, K, dt, repr(e)[:200]))
            torch.cuda.synchronize()
        print(n, S, J, K, dt, "ok" if not fails or fails[-1][:5] != (n, S, J, K, dt) else fails[-1][5],
              flush=True)
print("ok", n_ok, "fail", len(fails))
for x in fails:
    print("FAIL", x)
