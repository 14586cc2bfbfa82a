"""Solve a 27-point problem (paper domain, 256x128x128, K = 2, 32^3 segments) and save u
(GPU box; bitwise comparison of two library builds)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import Solver  # noqa: E402

n, h = (256, 128, 128), 2.0 / 256
f = torch.from_numpy(W.make_rhs("manufactured+noise", n, h=h)).cuda()
with Solver(n, 6, seg=32, buffer=2, K=2, h=h, stencil="27pt") as s:
    np.save(sys.argv[1], s.solve(f).cpu().numpy())
