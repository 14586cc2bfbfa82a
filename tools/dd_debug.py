"""Debug driver (GPU box): one multi-rank case through the host-store backend, one thread per
rank, with SR_FMG_TRACE output and a stack dump of every thread after `--dump` seconds."""
import argparse
import faulthandler
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1406_7808_b200 import HostStore, Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="128,32,32")
ap.add_argument("--M", type=int, default=5)
ap.add_argument("--seg", type=int, default=16)
ap.add_argument("--J", type=int, default=2)
ap.add_argument("--K", type=int, default=2)
ap.add_argument("--pgrid", default="4,1,1")
ap.add_argument("--dtype", default="f32")
ap.add_argument("--dd_min", type=int, default=2)
ap.add_argument("--dump", type=float, default=60)
ap.add_argument("--idle", type=int, default=0)
a = ap.parse_args()
n = tuple(int(v) for v in a.n.split(","))
pg = tuple(int(v) for v in a.pgrid.split(","))
world = int(np.prod(pg))
faulthandler.dump_traceback_later(a.dump, exit=True)
npd = np.float64 if a.dtype == "f64" else np.float32
f = W.make_rhs("manufactured+noise", n).astype(npd)
with Solver(n, a.M, seg=a.seg, buffer=a.J, K=a.K, dtype=a.dtype) as s1:
    single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
print("single done", flush=True)
store = HostStore(world)
ranks = [Solver(n, a.M, seg=a.seg, buffer=a.J, K=a.K, dtype=a.dtype, world=world, rank=r,
                pgrid=pg, host_store=store, dd_min=a.dd_min, coarse_idle=bool(a.idle)) for r in range(world)]
print("A", ranks[0].level_A, "T", ranks[0].T, "dd", ranks[0].dd_levels(), flush=True)
fl = [torch.from_numpy(s.local_f(f)).cuda() for s in ranks]
torch.cuda.synchronize()  # the rank threads solve on streams of their own
outs = [None] * world


def work(r):
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        outs[r] = ranks[r].solve(fl[r])
    st.synchronize()
    print("rank", r, "done", flush=True)


th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
for t in th:
    t.start()
for t in th:
    t.join()
for r, s in enumerate(ranks):
    o, b = outs[r].cpu().numpy(), s.block_of(single)
    print("rank", r, "bitwise", np.array_equal(o, b), "max diff", float(np.abs(o - b).max()),
          flush=True)
