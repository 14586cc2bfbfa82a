"""Locate fused-vs-step mismatches of one degree-2 Chebyshev application on an SR level."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1406_7808_b200 import Solver  # noqa: E402
from tests.gpu_helpers import seg_array, storage_box, zero_outside  # noqa: E402

n, l = (32, 32, 32), 3
res = {}
for fused in ("1", "0"):
    os.environ["SR_FMG_FUSED"] = fused
    s = Solver(n, 4, seg=16, buffer=2, K=2, use_graph=False)
    li = s.level(l)
    nsegs = li.nseg[0] * li.nseg[1] * li.nseg[2]
    rng = np.random.default_rng(1)
    u = zero_outside(rng.standard_normal(nsegs * li.pitch[2]), li)
    b = zero_outside(rng.standard_normal(nsegs * li.pitch[2]), li)
    s.set_level_storage(l, 0, u)
    s.set_level_storage(l, 1, b)
    s.debug_op(0, l, 2)
    res[fused] = s.level_storage(l, 0)
    s.close()
print("E", li.storage_ext, "pitch", li.pitch)
for k in range(nsegs):
    a = seg_array(res["1"], li, k)
    c = seg_array(res["0"], li, k)
    box = storage_box(li, k)
    d = np.abs(a - c) > 1e-12
    # only cells inside the domain matter
    N = 16
    idx = np.argwhere(d)
    glob = idx + np.array(box.lo)
    ok = ((glob >= 0) & (glob < N)).all(axis=1)
    idx = idx[ok]
    print("seg", k, "box lo", box.lo, "mismatches", len(idx))
    if len(idx):
        print("   z:", sorted(set(idx[:, 0].tolist())), "y:", sorted(set(idx[:, 1].tolist())),
              "x:", sorted(set(idx[:, 2].tolist()))[:20])
