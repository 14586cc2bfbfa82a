"""The multi-GPU path of the library on ONE GPU (test comm backend, desc.comm = 1).

Every rank's handle lives in this process and runs its solve in a thread of its own; the
all-gathers and halo slabs go through a host store (sr_fmg_host_store_create), so no kernel
of one rank ever waits for another.  Each rank's output block must equal the single-GPU
solve BITWISE (R25: SR segments are independent, the decomposed coarse levels exchange
their ghost rings before every operator application, the agglomerated levels are solved
redundantly), and the oracle to the parity tolerance.  Only the NCCL call itself is not
exercised here.
"""
import threading

import numpy as np
import pytest

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_1406_7808_b200 import HostStore, Solver  # noqa: E402
from tests.gpu_helpers import rel_l2  # noqa: E402


def run_ranks(n, M, seg, J, K, pgrid, f, dtype="f64", dd_min=0, solves=1, **kw):
    """Solve f on every rank of pgrid concurrently (one thread per rank); returns the
    handles (open) and each rank's output block of the last solve."""
    world = int(np.prod(pgrid))
    store = HostStore(world)
    ranks = [Solver(n, M, seg=seg, buffer=J, K=K, dtype=dtype, world=world, rank=r, pgrid=pgrid,
                    host_store=store, dd_min=dd_min, **kw) for r in range(world)]
    fl = [torch.from_numpy(s.local_f(f)).cuda() for s in ranks]
    # the ranks solve on streams of their own: the inputs' copies (default stream) must have
    # landed first (a pageable host-to-device copy can return before it has)
    torch.cuda.synchronize()
    outs, errs = [None] * world, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(solves):
                    u = ranks[r].solve(fl[r])
                st.synchronize()
            outs[r] = u.cpu().numpy()
        except Exception as e:  # reported in the main thread
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    return ranks, outs, store


CASES = [
    # name, n, M, seg, J, K, pgrid, dtype, dd_min
    ("2x1x1", (64, 64, 64), 5, 8, 2, 2, (2, 1, 1), "f64", 0),
    ("2x2x1", (64, 64, 64), 5, 16, 2, 3, (2, 2, 1), "f64", 0),
    ("2x2x2", (64, 64, 64), 5, 8, 2, 2, (2, 2, 2), "f64", 0),
    ("4x1x2-f32", (128, 64, 64), 5, 16, 1, 2, (4, 1, 2), "f32", 0),
    ("2x1x1-S32", (128, 64, 64), 5, 32, 2, 2, (2, 1, 1), "f64", 0),
    ("1x2x2-S64", (128, 128, 128), 6, 64, 2, 2, (1, 2, 2), "f64", 0),
    ("2x1x1-S64-f32", (128, 64, 64), 5, 64, 2, 2, (2, 1, 1), "f32", 0),
    # decomposed coarse levels (halo exchange) below T, agglomeration further down
    ("dd-2x1x1", (64, 64, 64), 5, 16, 2, 2, (2, 1, 1), "f64", 4),
    ("dd-2x2x2", (128, 128, 128), 6, 32, 2, 2, (2, 2, 2), "f64", 4),
    ("dd-2x2x1-J1", (128, 128, 64), 5, 32, 1, 2, (2, 2, 1), "f64", 2),
    ("dd-4x1x1-f32", (128, 32, 32), 5, 16, 2, 2, (4, 1, 1), "f32", 2),
    ("dd-1x2x2-K1", (64, 128, 128), 6, 32, 2, 1, (1, 2, 2), "f64", 4),
    ("dd-2x2x2-J3", (64, 64, 64), 5, 16, 3, 2, (2, 2, 2), "f64", 2),
]


@pytest.mark.timeout(150)
@pytest.mark.parametrize("force", ["0", "1"])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_ranks_equal_single_gpu(case, force, monkeypatch):
    name, n, M, seg, J, K, pgrid, dt, dd_min = case
    monkeypatch.setenv("SR_FMG_FORCE_FUSED", force)
    npd = np.float64 if dt == "f64" else np.float32
    f = W.make_rhs("manufactured+noise", n).astype(npd)
    with Solver(n, M, seg=seg, buffer=J, K=K, dtype=dt) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    ranks, outs, store = run_ranks(n, M, seg, J, K, pgrid, f, dt, dd_min, solves=2)
    T, A = ranks[0].T, ranks[0].level_A
    if dd_min:
        assert A < T, (name, A, T)               # the case decomposes at least level T
        assert ranks[0].dd_levels() == list(range(A + 1, T + 1))
    for r, s in enumerate(ranks):
        # kernel choices follow the global level shape, so every rank runs the single-GPU
        # arithmetic on its segments and blocks: bitwise (R25)
        assert np.array_equal(outs[r], s.block_of(single)), (name, r)
        calls = s.comm_calls()
        # zero collectives on the SR levels; the decomposed levels
        # exchange halos, the agglomeration level gathers
        assert all(calls[l] == 0 for l in range(T + 1, s.M + 1)), calls
        assert calls[A] >= 1 and all(calls[l] == 0 for l in range(A)), calls
        assert all(calls[l] > 0 for l in range(A + 1, T + 1)), calls
        assert s.exchanges_per_solve == sum(calls)
    if dt == "f64":
        ref = O.solve(f.astype(np.float64), O.Config(n=n, M=M, seg=seg, buffer=J, K=K))
        full = np.zeros_like(ref)
        for r, s in enumerate(ranks):
            lo, nb = s.block_lo, s.block_n
            full[lo[2]:lo[2] + nb[2], lo[1]:lo[1] + nb[1], lo[0]:lo[0] + nb[0]] = outs[r]
        assert rel_l2(full, ref) <= 1e-11
    for s in ranks:
        s.close()


VARIANTS = [
    # name, n, M, seg, J, K, pgrid, dtype, dd_min, idle
    # idle coarse grid (desc.coarse_idle): levels <= A on rank 0 alone
    ("idle-agg-T", (64, 64, 64), 5, 8, 2, 2, (2, 1, 1), "f64", 0, True),
    ("idle-dd-2x2x2", (128, 128, 128), 6, 32, 2, 2, (2, 2, 2), "f64", 4, True),
    ("idle-dd-4x1x1-f32", (128, 32, 32), 5, 16, 2, 2, (4, 1, 1), "f32", 2, True),
    # conventional distributed FMG (K = 0): the finest level decomposed,
    # halo exchanges on every level down to A
    ("K0-2x1x1", (64, 64, 64), 5, 0, 0, 0, (2, 1, 1), "f64", 8, False),
    ("K0-2x2x2-idle", (64, 64, 64), 5, 0, 0, 0, (2, 2, 2), "f64", 8, True),
    ("K0-4x1x1-f32", (128, 64, 64), 5, 0, 0, 0, (4, 1, 1), "f32", 8, False),
    ("K0-1x2x2-big", (128, 128, 128), 6, 0, 0, 0, (1, 2, 2), "f64", 16, False),
]


@pytest.mark.timeout(150)
@pytest.mark.parametrize("case", VARIANTS, ids=[c[0] for c in VARIANTS])
def test_idle_and_conventional_ranks_equal_single_gpu(case):
    name, n, M, seg, J, K, pgrid, dt, dd_min, idle = case
    npd = np.float64 if dt == "f64" else np.float32
    f = W.make_rhs("manufactured+noise", n).astype(npd)
    with Solver(n, M, seg=seg, buffer=J, K=K, dtype=dt) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    ranks, outs, _ = run_ranks(n, M, seg, J, K, pgrid, f, dt, dd_min, solves=2,
                               coarse_idle=idle)
    T, A = ranks[0].T, ranks[0].level_A
    if K == 0:
        assert T == M and A < M, (name, A)   # the finest level is decomposed
        assert ranks[0].f_halo == 0
    launches = [s.launches_per_solve for s in ranks]
    calls = [s.comm_calls() for s in ranks]
    for r, s in enumerate(ranks):
        assert np.array_equal(outs[r], s.block_of(single)), (name, r)
        c = calls[r]
        assert all(c[l] == 0 for l in range(T + 1, s.M + 1)), c
        assert all(c[l] > 0 for l in range(A + 1, T + 1)), c
        assert c[A] >= 1 and all(c[l] == 0 for l in range(A)), c
    if idle:
        # against the redundant coarse grid: the ranks other than 0 launch fewer kernels
        # (none of the levels <= A) and level A carries one broadcast per gather besides
        red, red_outs, _ = run_ranks(n, M, seg, J, K, pgrid, f, dt, dd_min, solves=1)
        for r, s in enumerate(red):
            assert np.array_equal(red_outs[r], outs[r]), (name, r)
            if r > 0:
                assert launches[r] < s.launches_per_solve, (launches, r)
            assert calls[r][A] > s.comm_calls()[A], (calls[r], s.comm_calls())
            s.close()
    if dt == "f64":
        ref = O.solve(f.astype(np.float64), O.Config(n=n, M=M, seg=seg, buffer=J, K=K))
        full = np.zeros_like(ref)
        for r, s in enumerate(ranks):
            lo, nb = s.block_lo, s.block_n
            full[lo[2]:lo[2] + nb[2], lo[1]:lo[1] + nb[1], lo[0]:lo[0] + nb[0]] = outs[r]
        assert rel_l2(full, ref) <= 1e-11
    for s in ranks:
        s.close()


OPS = [
    # name, n, M, seg, J, K, pgrid, dd_min, extra Solver arguments
    ("27pt-2x1x1", (64, 32, 32), 5, 16, 2, 2, (2, 1, 1), 0, dict(stencil="27pt", h=2.0 / 64)),
    ("27pt-dd-2x2x1", (128, 64, 64), 5, 32, 2, 2, (2, 2, 1), 4, dict(stencil="27pt", h=2.0 / 128)),
    ("nl-2x1x1", (64, 64, 64), 5, 16, 2, 2, (2, 1, 1), 0, dict(nl_gamma=1e4)),
    ("nl-dd-2x2x2", (128, 128, 128), 6, 32, 2, 2, (2, 2, 2), 4, dict(nl_gamma=1e4)),
    ("27pt-K0-2x1x1", (64, 32, 32), 5, 0, 0, 0, (2, 1, 1), 4, dict(stencil="27pt", h=2.0 / 64)),
]


@pytest.mark.timeout(150)
@pytest.mark.parametrize("case", OPS, ids=[c[0] for c in OPS])
def test_27pt_and_nonlinear_ranks_equal_single_gpu(case):
    # the NEXT-row operators (f1: 27-point, f4: nonlinear FAS) through the multi-GPU path:
    # the decomposed levels exchange the ghost ring (edges and corners included, which the
    # 27-point stencil reads) before every operator application -- bitwise one GPU
    name, n, M, seg, J, K, pgrid, dd_min, kw = case
    f = W.make_rhs("manufactured+noise", n, h=kw.get("h"))
    with Solver(n, M, seg=seg, buffer=J, K=K, **kw) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    ranks, outs, _ = run_ranks(n, M, seg, J, K, pgrid, f, "f64", dd_min, solves=1, **kw)
    for r, s in enumerate(ranks):
        assert np.array_equal(outs[r], s.block_of(single)), (name, r)
        s.close()


@pytest.mark.timeout(150)
def test_multirank_local_f_uses_halo_only():
    # f outside a rank's haloed block must not matter: perturb it and get the same block
    n, M, seg, J, K, pgrid = (64, 64, 64), 5, 16, 2, 2, (2, 1, 1)
    f = W.make_rhs("manufactured+noise", n)
    with Solver(n, M, seg=seg, buffer=J, K=K) as s1:
        single = s1.solve(torch.from_numpy(f).cuda()).cpu().numpy()
    for dd_min in (0, 4):
        ranks, outs, _ = run_ranks(n, M, seg, J, K, pgrid, f, dd_min=dd_min)
        fl = ranks[0].local_f(f)
        assert ranks[0].f_halo > 0 and fl.shape == ranks[0].f_shape
        for r, s in enumerate(ranks):
            assert np.array_equal(outs[r], s.block_of(single)), (dd_min, r)
            s.close()
