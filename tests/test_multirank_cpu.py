"""Multi-rank path on CPU (gloo): the product's partition arithmetic drives a decomposed
oracle solve -- each rank runs only its own segments; the conventional levels A < l <= T
are domain-decomposed with a halo exchange before every operator application, and level A
is all-gathered (the library's exchange points; tests/dd_oracle.py).  The
result must equal the single-process solve BITWISE (R25): SR segments are independent
(PAPER.md:44), a decomposed V-cycle replicates the serial one and the
agglomerated levels are solved redundantly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W
from oracle import Field


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    # agglomeration at T (dd_min larger than the level-T block)
    "x-split": dict(n=(32, 16, 16), M=3, seg=8, buffer=2, K=2, pgrid=(2, 1, 1), dd_min=1 << 20),
    "y-split": dict(n=(16, 32, 16), M=3, seg=8, buffer=1, K=1, pgrid=(1, 2, 1), dd_min=1 << 20),
    # decomposed conventional levels with halo exchanges
    "dd-x": dict(n=(64, 32, 32), M=5, seg=16, buffer=2, K=2, pgrid=(2, 1, 1), dd_min=4),
    "dd-xy-J3": dict(n=(32, 32, 16), M=4, seg=8, buffer=3, K=1, pgrid=(2, 2, 1), dd_min=2),
    "dd-xyz": dict(n=(32, 32, 32), M=4, seg=8, buffer=2, K=1, pgrid=(2, 2, 2), dd_min=2),
    # the idle coarse grid (levels <= A on rank 0 alone)
    "dd-x-idle": dict(n=(64, 32, 32), M=5, seg=16, buffer=2, K=2, pgrid=(2, 1, 1), dd_min=4,
                      idle=True),
    # conventional distributed FMG (K = 0): the finest level decomposed too
    "dd-K0-x": dict(n=(32, 16, 16), M=3, seg=8, buffer=2, K=0, pgrid=(2, 1, 1), dd_min=4),
    "dd-K0-xyz-idle": dict(n=(32, 32, 32), M=4, seg=8, buffer=2, K=0, pgrid=(2, 2, 2), dd_min=4,
                           idle=True),
}


def _worker(rank, world, port, case, outq):
    from paper_1406_7808_b200 import partition
    from tests.dd_oracle import DDOracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = CASES[case]
    part = partition(c["n"], c["M"], c["seg"], c["buffer"], c["K"], world, rank, c["pgrid"],
                     dd_min=c["dd_min"], coarse_idle=c.get("idle", False))
    f = W.make_rhs("manufactured+noise", c["n"])
    o = DDOracle(O.Config(n=c["n"], M=c["M"], seg=c["seg"], buffer=c["buffer"], K=c["K"]),
                 part, c["pgrid"], idle=c.get("idle", False))
    u = o.solve(f)
    bl, bn = part["block_lo"], part["block_n"]
    outq.put((rank, (u[bl[2]:bl[2] + bn[2], bl[1]:bl[1] + bn[1], bl[0]:bl[0] + bn[0]].copy(),
                     part["level_A"], o.n_exchanges)))
    dist.barrier()
    dist.destroy_process_group()


def _box(lo_xyz, n_xyz):
    from oracle import Box
    return Box((lo_xyz[2], lo_xyz[1], lo_xyz[0]),
               (lo_xyz[2] + n_xyz[2], lo_xyz[1] + n_xyz[1], lo_xyz[0] + n_xyz[0]))


@pytest.mark.parametrize("case", sorted(CASES))
def test_decomposed_solve_equals_single_process(case):
    c = CASES[case]
    world = int(np.prod(c["pgrid"]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f = W.make_rhs("manufactured+noise", c["n"])
    ref = O.solve(f, O.Config(n=c["n"], M=c["M"], seg=c["seg"], buffer=c["buffer"], K=c["K"]))
    from paper_1406_7808_b200 import partition
    T = c["M"] - c["K"]
    for r in range(world):
        part = partition(c["n"], c["M"], c["seg"], c["buffer"], c["K"], world, r, c["pgrid"],
                         dd_min=c["dd_min"])
        bl, bn = part["block_lo"], part["block_n"]
        blk = ref[bl[2]:bl[2] + bn[2], bl[1]:bl[1] + bn[1], bl[0]:bl[0] + bn[0]]
        u, A, nex = res[r]
        assert np.array_equal(u, blk), (case, r)
        assert (A < T) == case.startswith("dd"), (case, A, T)
        assert nex > 0


def test_partition_blocks_tile_the_grid():
    from paper_1406_7808_b200 import partition
    for n, seg, K, pg in [((1024, 1024, 1024), 64, 4, (2, 2, 2)), ((64, 32, 32), 8, 2, (2, 2, 1)),
                          ((128, 128, 64), 16, 3, (4, 2, 1))]:
        world = int(np.prod(pg))
        M = int(np.log2(min(n))) - 1
        cover = np.zeros((n[2] // seg, n[1] // seg, n[0] // seg), int)
        for r in range(world):
            p = partition(n, M, seg, 2, K, world, r, pg)
            assert p["f_halo"] >= 2 << (K - 1) and p["f_halo"] % 4 == 0
            assert all(p["f_dims"][d] == p["block_n"][d] + 2 * p["f_halo"] for d in range(3))
            assert all(p["level_T_n"][d] * (1 << K) == p["block_n"][d] for d in range(3))
            lo = [p["block_lo"][d] // seg for d in range(3)]
            sl = tuple(slice(lo[2 - d], lo[2 - d] + p["segs_per_rank"][2 - d]) for d in range(3))
            cover[sl] += 1
        assert np.all(cover == 1)


def test_rank_blocks_of_every_rhs_kind_equal_the_global_rhs():
    # bench.py at N > 1 evaluates each rank's haloed f block on its own (W.rhs_block); on the
    # block's in-domain cells it must equal the global array bitwise
    n, h = (64, 32, 32), 1.0 / 64
    lo, dims = (30, -2, 4), (20, 20, 20)
    for kind in ("manufactured", "bumps", "manufactured+noise"):
        full = W.make_rhs(kind, n, h=h)
        blk = W.rhs_block(kind, n, h, lo, dims)
        assert blk.shape == (20, 20, 20)
        assert np.array_equal(blk[:, 2:20, :], full[4:24, 0:18, 30:50]), kind
