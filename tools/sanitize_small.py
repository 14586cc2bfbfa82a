"""Small solves for compute-sanitizer (memcheck): several configs incl. J = 0 and K = M."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

for n, M, seg, J, K, dt in [((32, 32, 32), 4, 16, 2, 2, "f64"), ((32, 32, 32), 4, 16, 0, 2, "f64"),
                            ((16, 16, 16), 3, 8, 2, 3, "f32"), ((32, 16, 16), 3, 8, 1, 2, "f64"),
                            ((32, 32, 32), 4, 0, 0, 0, "f64")]:
    f = torch.from_numpy(W.make_rhs("manufactured+noise", n).astype(
        np.float64 if dt == "f64" else np.float32)).cuda()
    with Solver(n, M, seg=seg, buffer=J, K=K, dtype=dt, use_graph=False) as s:
        u = s.solve(f)
        torch.cuda.synchronize()
        assert torch.isfinite(u).all()
print("sanitize ok")
