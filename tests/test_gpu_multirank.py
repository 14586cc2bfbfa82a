"""The multi-GPU path of the library on ONE GPU (test comm backend, desc.comm = 1).

Every rank's handle lives in this process; its all-gathers record / replay per-rank blocks
through a shared host store, and solving all ranks exchanges_per_solve + 1 times makes every
exchange consistent.  Each rank's output block must equal the single-GPU solve BITWISE (R25:
SR segments are independent and the coarse levels are solved redundantly), and the oracle
to the parity tolerance.  Only the NCCL call itself is not exercised here.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_1406_7808_b200 import ReplayStore, Solver  # noqa: E402
from tests.gpu_helpers import rel_l2  # noqa: E402

CASES = [
    ("2x1x1", (64, 64, 64), 5, 8, 2, 2, (2, 1, 1), "f64"),
    ("2x2x1", (64, 64, 64), 5, 16, 2, 3, (2, 2, 1), "f64"),
    ("2x2x2", (64, 64, 64), 5, 8, 2, 2, (2, 2, 2), "f64"),
    ("4x1x2-f32", (128, 64, 64), 5, 16, 1, 2, (4, 1, 2), "f32"),
    # 32^3 and 64^3 segments: the fused FMG entry (pset.cu), the tau inside the coarse
    # pre-smoothing and the pyramid restriction run with nonzero segment / f offsets per rank
    ("2x1x1-S32", (128, 64, 64), 5, 32, 2, 2, (2, 1, 1), "f64"),
    ("1x2x2-S64", (128, 128, 128), 6, 64, 2, 2, (1, 2, 2), "f64"),
    ("2x1x1-S64-f32", (128, 64, 64), 5, 64, 2, 2, (2, 1, 1), "f32"),
]


@pytest.mark.parametrize("force", ["0", "1"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_replayed_ranks_equal_single_gpu(case, force, monkeypatch):
    name, n, M, seg, J, K, pgrid, dt = case
    monkeypatch.setenv("SR_FMG_FORCE_FUSED", force)
    npd = np.float64 if dt == "f64" else np.float32
    f = W.make_rhs("manufactured+noise", n).astype(npd)
    with Solver(n, M, seg=seg, buffer=J, K=K, dtype=dt) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    world = int(np.prod(pgrid))
    store = ReplayStore(world)
    ranks = [Solver(n, M, seg=seg, buffer=J, K=K, dtype=dt, world=world, rank=r, pgrid=pgrid,
                    replay_store=store) for r in range(world)]
    fl = [torch.from_numpy(s.local_f(f)).cuda() for s in ranks]
    E = ranks[0].exchanges_per_solve
    assert E == K + 1
    outs = None
    for _ in range(E + 1):
        outs = [s.solve(fl[r]).cpu().numpy() for r, s in enumerate(ranks)]
    for r, s in enumerate(ranks):
        # kernel choices follow the global level shape, so every rank runs the single-GPU
        # schedule on its segments: bitwise (R25)
        assert np.array_equal(outs[r], s.block_of(single)), (name, r)
    if dt == "f64":
        ref = O.solve(f.astype(np.float64), O.Config(n=n, M=M, seg=seg, buffer=J, K=K))
        full = np.zeros_like(ref)
        for r, s in enumerate(ranks):
            lo, nb = s.block_lo, s.block_n
            full[lo[2]:lo[2] + nb[2], lo[1]:lo[1] + nb[1], lo[0]:lo[0] + nb[0]] = outs[r]
        assert rel_l2(full, ref) <= 1e-11
    for s in ranks:
        s.close()


def test_multirank_local_f_uses_halo_only():
    # f outside a rank's haloed block must not matter: perturb it and get the same block
    n, M, seg, J, K, pgrid = (64, 64, 64), 5, 8, 2, 2, (2, 1, 1)
    f = W.make_rhs("manufactured+noise", n)
    store = ReplayStore(2)
    ranks = [Solver(n, M, seg=seg, buffer=J, K=K, world=2, rank=r, pgrid=pgrid,
                    replay_store=store) for r in range(2)]
    fl = [s.local_f(f) for s in ranks]
    assert ranks[0].f_halo > 0 and fl[0].shape == ranks[0].f_shape
    ft = [torch.from_numpy(x).cuda() for x in fl]
    for _ in range(ranks[0].exchanges_per_solve + 1):
        outs = [s.solve(ft[r]).cpu().numpy() for r, s in enumerate(ranks)]
    with Solver(n, M, seg=seg, buffer=J, K=K) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    for r, s in enumerate(ranks):
        assert np.array_equal(outs[r], s.block_of(single)), r
