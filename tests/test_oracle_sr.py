r"""Pins of the oracle's segmental refinement (fig:fmgsr / fig:mgvsr).

What fixes SR independently of the oracle's own arithmetic:
  * the region definitions of PAPER.md:187-214, evaluated by brute force on cell sets;
  * equivalences: C = Omega on every level (huge buffer) and a single segment must give
    conventional FMG exactly (north_star; SPEC sr examples);
  * symmetry: a symmetric f on a symmetric segment grid gives a symmetric u;
  * the paper's trends: e_r decreases with the buffer and with larger
    transition subdomains pN0V;
  * frozen GSR cells: never changed by a smoother;
  * the SR V-cycle: u_h* (DST, tests/pins.py) in every segment is a fixed point of
    FASMGVSR; every correction increments the GSR cells by exactly
    P(w - t) (R17); the tau leaves a zero residual on C \ F and R on F (R18).  Mutations
    checked by hand to fail these: GSR corrected on C only (k = 1 or k >= 2), b = 0 on
    C \ F, b = R - A u on F, R dropped from b.
The e_r VALUES of Tables 1-3 belong to a 27-point stencil on [0,2]x[0,1]^2: parity unpinned.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from oracle import Box, Config, Oracle


def _cells(box):
    return set(box.cells())


def _linf_grow(cells, j):
    out = set()
    for c in cells:
        for o in itertools.product(range(-j, j + 1), repeat=3):
            out.add((c[0] + o[0], c[1] + o[1], c[2] + o[2]))
    return out


@pytest.mark.parametrize("J", [0, 1, 2, 3, 4])
def test_regions_match_set_definitions(J):
    cfg = Config(n=(16, 16, 16), M=4, seg=8, buffer=J, K=2)
    o = Oracle(cfg)
    for l in range(o.T + 1, o.M + 1):
        S = o.S_l(l)
        omega = _cells(o.dom[l])
        for p in o.segs:
            V = {c for c in omega if tuple(v // S for v in c) == p}
            assert V == _cells(o.V(l, p))
            C = _linf_grow(V, J) & omega
            G = _linf_grow(C, 1) - C
            GBC, GSR = G - omega, G & omega
            assert C == _cells(o.C(l, p))
            assert C | GSR == _cells(o.CG(l, p))              # range of prolongation L215
            st = _cells(o.storage(l, p))
            assert (C | G) <= st
            # F: coarse cells whose 8 children all lie in C_l^p
            omc = _cells(o.dom[l - 1])
            F = {I for I in omc
                 if all((2 * I[0] + a, 2 * I[1] + b, 2 * I[2] + c) in C
                        for a, b, c in itertools.product((0, 1), repeat=3))}
            assert F == _cells(o.F(l, p))
            # zero-communication footprint (R15): the trilinear footprint of C cup GSR lies
            # in the segment's own level-(l-1) storage (k >= 2) ...
            foot = set()
            for i in C | GSR:
                par = tuple(v // 2 for v in i)
                s = tuple(-1 if v % 2 == 0 else 1 for v in i)
                for a, b, c in itertools.product((0, 1), repeat=3):
                    foot.add((par[0] + a * s[0], par[1] + b * s[1], par[2] + c * s[2]))
            if l - 1 > o.T:
                assert foot <= _cells(o.storage(l - 1, p))
            # ... and reaches outside Omega_{l-1} only through depth-1 (reflected) ghosts
            for I in foot - omc:
                assert all(-1 <= v <= n for v, n in zip(I, o.N[l - 1]))
        # genuine regions tile Omega_l disjointly
        assert sum(o.V(l, p).volume for p in o.segs) == len(omega)


def test_huge_buffer_equals_conventional_fmg():
    # J >= N - S makes C_l^p = Omega_l on every level: SR must reproduce FMG (north_star)
    n = (32, 32, 32)
    f = W.manufactured_f(n, 1 / 32) + W.noise(n, 1e-2)
    u0 = O.solve(f, Config(n=n, M=4, K=0))
    for S, K in [(16, 2), (8, 3)]:
        u = O.solve(f, Config(n=n, M=4, seg=S, buffer=32, K=K))
        assert np.abs(u - u0).max() <= 1e-14 * np.abs(u0).max()


@pytest.mark.parametrize("J", [0, 1, 2])
def test_single_segment_equals_conventional_fmg(J):
    n = (32, 32, 32)
    f = W.manufactured_f(n, 1 / 32)
    u0 = O.solve(f, Config(n=n, M=4, K=0))
    u = O.solve(f, Config(n=n, M=4, seg=32, buffer=J, K=3))
    assert np.abs(u - u0).max() <= 1e-14 * np.abs(u0).max()


def test_all_levels_sr():
    # K = M: the transition level is the coarsest grid (T = 0)
    n = (16, 16, 16)
    f = W.manufactured_f(n, 1 / 16)
    u = O.solve(f, Config(n=n, M=3, seg=8, buffer=2, K=3))
    ue = W.manufactured_u(n, 1 / 16)
    assert np.isfinite(u).all() and np.abs(u - ue).max() < 20 * np.abs(ue).max() * 1e-2


def test_symmetric_rhs_gives_symmetric_solution():
    n = (32, 32, 32)
    f = W.random_field(n, seed=11)
    f = f + f[:, :, ::-1]                     # mirror x1
    f = f + f[:, ::-1, :]                     # mirror x2
    f = f + np.transpose(f, (0, 2, 1))        # swap x1 <-> x2 (keeps both mirrors)
    u = O.solve(f, Config(n=n, M=4, seg=8, buffer=2, K=2))
    sc = np.abs(u).max()
    assert np.abs(u - u[:, :, ::-1]).max() <= 1e-13 * sc
    assert np.abs(u - np.transpose(u, (0, 2, 1))).max() <= 1e-13 * sc


def test_deterministic():
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    cfg = Config(n=n, M=4, seg=16, buffer=2, K=2)
    assert np.array_equal(O.solve(f, cfg), O.solve(f, cfg))


def _err(n, M, S, J, K):
    f = W.manufactured_f(n, 1 / n[0])
    u = W.manufactured_u(n, 1 / n[0])
    return np.abs(O.solve(f, Config(n=n, M=M, seg=S, buffer=J, K=K)) - u).max()


def test_error_ratio_decreases_with_buffer():
    # A and B "both correlate with increased accuracy" (they increase J)
    n = (64, 64, 64)
    e_conv = _err(n, 5, 0, 0, 0)
    er = [_err(n, 5, 16, J, 3) / e_conv for J in (0, 1, 2, 4, 8)]
    assert all(a > b for a, b in zip(er, er[1:])), er
    assert er[-1] < 1.5


def test_error_ratio_grows_as_transition_subdomain_shrinks():
    # halving pN0V (at fixed K, J) increases e_r
    n = (64, 64, 64)
    e_conv = _err(n, 5, 0, 0, 0)
    er = [_err(n, 5, S, 2, 2) / e_conv for S in (32, 16, 8)]   # pN0V = 8, 4, 2
    assert er[0] < er[1] < er[2], er


def test_gsr_cells_are_never_smoothed():
    # GSR cells are set by prolongation only ("frozen")
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    o = Oracle(Config(n=n, M=4, seg=8, buffer=2, K=2))
    checked = [0]
    orig = o._cheb

    def spy(deg, u, b, X, l):
        if l > o.T:
            before = u.a.copy()
            orig(deg, u, b, X, l)
            inside = u.box.intersect(o.dom[l])
            m = np.zeros(u.box.shape, bool)
            sl = tuple(slice(a - s, c - s) for a, c, s in zip(X.lo, X.hi, u.box.lo))
            m[sl] = True
            ins = np.zeros(u.box.shape, bool)
            sl2 = tuple(slice(a - s, c - s) for a, c, s in zip(inside.lo, inside.hi, u.box.lo))
            ins[sl2] = True
            gsr = ins & ~m
            assert np.array_equal(before[gsr], u.a[gsr])
            checked[0] += 1
        else:
            orig(deg, u, b, X, l)

    o._cheb = spy
    o.solve(f)
    assert checked[0] > 0


def test_sr_error_second_order_at_fixed_segment_grid():
    # SR keeps 2nd-order accuracy; at a fixed segment grid (S = N/2) and
    # fixed K, J the SR error ratio per halving of h tends towards 4
    errs = [_err((N, N, N), M, N // 2, 2, 2) for N, M in ((32, 4), (64, 5), (128, 6))]
    q = [errs[0] / errs[1], errs[1] / errs[2]]
    assert 2.5 < q[0] and 2.5 < q[1] < 4.6, (errs, q)


def test_paper_tables_fixture_is_context_only():
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))
    # the paper's own trend: down every column, e_r does not increase with B
    for A in ("A2", "A4", "A6", "A8"):
        rows = [g["table1"][A][f"B{b}"] for b in range(4)]
        for c in range(3):
            col = [r[c] for r in rows if r[c] is not None]
            assert all(x >= y for x, y in zip(col, col[1:]))
    assert g["table2"]["e_r"] == sorted(g["table2"]["e_r"])


# ---- maximum buffer schedule (MBS) ----------------
@pytest.mark.parametrize("J1", [1, 2, 4])
def test_mbs_compute_regions_equal_F(J1):
    # "the rest of the SR buffers completely support grid k=1: pOmega^C_k = pOmega^F_k for
    # k < K", checked on cell sets: F_k from the children of C_{k+1}
    cfg = Config(n=(64, 64, 64), M=5, seg=32, K=3, sched=("mbs", J1))
    o = Oracle(cfg)
    assert [cfg.J(k) for k in (1, 2, 3)] == [J1, 2 * J1, 4 * J1]
    for l in range(o.T + 2, o.M + 1):          # coarse level l-1 = T+1 .. M-1 (k < K)
        for p in list(o.segs)[:3]:
            C = _cells(o.C(l, p))
            omc = _cells(o.dom[l - 1])
            F = {I for I in omc
                 if all((2 * I[0] + a, 2 * I[1] + b, 2 * I[2] + c) in C
                        for a, b, c in itertools.product((0, 1), repeat=3))}
            assert F == _cells(o.C(l - 1, p)), (l, p)
    # the number of buffer cells grows exponentially toward the fine grid
    assert cfg.J(3) == 4 * cfg.J(1)


def test_mbs_error_ratio_trend():
    # Table 3: with MBS (K fixed, J_1 = 4) the error ratio still grows as
    # pN0V halves, and MBS is at least as accurate as the constant buffer J = J_1
    n = (64, 64, 64)
    f = W.manufactured_f(n, 1 / n[0])
    u = W.manufactured_u(n, 1 / n[0])
    e_conv = np.abs(O.solve(f, Config(n=n, M=5)) - u).max()

    def er(S, sched=None, J=4):
        return np.abs(O.solve(f, Config(n=n, M=5, seg=S, buffer=J, K=2, sched=sched)) - u).max() / e_conv

    mbs = [er(S, ("mbs", 2)) for S in (32, 16, 8)]          # pN0V = 8, 4, 2
    assert mbs[0] < mbs[1] < mbs[2], mbs
    for S in (16, 8):
        assert er(S, ("mbs", 2)) <= er(S, None, 2) + 1e-12


# ---- 27-point operator: the SR equivalences and the paper's e_r trends on the
# paper's own domain [0,2]x[0,1]^2, R = (2,1,1) (Tables 1-2 trends)
def test_27pt_sr_huge_buffer_and_one_segment_equal_fmg():
    n, h = (64, 32, 32), 1 / 32
    f = W.manufactured_f(n, h)
    ref = O.solve(f, Config(n=n, M=4, h=h, stencil="27pt"))
    big = O.solve(f, Config(n=n, M=4, h=h, seg=16, buffer=64, K=2, stencil="27pt"))
    assert np.array_equal(big, ref)
    n1 = (32, 32, 32)
    f1 = W.manufactured_f(n1, 1 / 32)
    one = O.solve(f1, Config(n=n1, M=4, seg=32, buffer=2, K=2, stencil="27pt"))
    assert np.array_equal(one, O.solve(f1, Config(n=n1, M=4, stencil="27pt")))


def test_27pt_error_ratio_trends_on_paper_domain():
    N = 32
    n, h = (2 * N, N, N), 1.0 / N
    f = W.manufactured_f(n, h)
    u = W.manufactured_u(n, h)
    e_conv = np.abs(O.solve(f, Config(n=n, M=5, h=h, stencil="27pt")) - u).max()

    def er(S, J, K, sched=None):
        cfg = Config(n=n, M=5, h=h, seg=S, buffer=J, K=K, sched=sched, stencil="27pt")
        return np.abs(O.solve(f, cfg) - u).max() / e_conv

    by_J = [er(16, J, 2) for J in (1, 2, 4)]            # e_r falls with J
    assert by_J[0] > by_J[1] > by_J[2], by_J
    by_p = [er(S, 2, 2) for S in (32, 16, 8)]            # pN0V = 8, 4, 2
    assert by_p[0] < by_p[1] < by_p[2], by_p


def test_nl_sr_huge_buffer_and_one_segment_equal_fmg():
    # nonlinear FAS through the SR hierarchy keeps the SR equivalences
    n, h, g = (32, 32, 32), 1 / 32, 1.0e4
    u = W.manufactured_u(n, h)
    f = W.manufactured_f(n, h) + g * u ** 3
    ref = O.solve(f, Config(n=n, M=4, nl_gamma=g))
    assert np.array_equal(O.solve(f, Config(n=n, M=4, seg=16, buffer=32, K=2, nl_gamma=g)), ref)
    assert np.array_equal(O.solve(f, Config(n=n, M=4, seg=32, buffer=2, K=2, nl_gamma=g)), ref)
    sr = O.solve(f, Config(n=n, M=4, seg=16, buffer=2, K=2, nl_gamma=g))
    assert np.abs(sr - u).max() < 5 * np.abs(ref - u).max()


# ---- the SR V-cycle itself (fig:mgvsr) ---------------------------------
def _load_exact(o, f):
    """Every level and every segment holds (a restriction of) the exact discrete solution
    u_h* = A_M^{-1} f (DST, tests/pins.py -- independent of the oracle); b_M^p = f on C."""
    from tests import pins
    M = o.M
    ustar = pins.dst_solve(f, o.h[M])
    pyr = {M: ustar}
    for l in range(M, 0, -1):
        a = pyr[l]
        pyr[l - 1] = 0.125 * sum(a[i::2, j::2, k::2] for i in (0, 1) for j in (0, 1) for k in (0, 1))
    for l in range(o.T + 1):
        o.u[l][o.dom[l]] = pyr[l]
    for l in range(o.T + 1, M + 1):
        for p in o.segs:
            u = O.Field(o.storage(l, p))
            CG = o.CG(l, p)
            u[CG] = pyr[l][tuple(slice(a, b) for a, b in zip(CG.lo, CG.hi))]
            o.us[l][p] = u
            b = O.Field(o.storage(l, p))       # coarse SR levels: set by the tau (L234-236)
            if l == M:
                C = o.C(l, p)
                b[C] = f[tuple(slice(a, c) for a, c in zip(C.lo, C.hi))]
            o.bs[l][p] = b
    return ustar


@pytest.mark.parametrize("K,S", [(2, 8), (3, 16)])
def test_sr_vcycle_fixed_point_at_exact_discrete_solution(K, S):
    # with u = u_h* in every segment the fine residual vanishes, so the
    # FAS coarse problems (Eq. 4, fig:mgvsr L234-236: b = R + A u on F, A u on C \ F) have
    # zero residual on every level and the correction w - t is zero: FASMGVSR(M) leaves u
    # unchanged.  A wrong sign or a dropped term in the tau (e.g. b = 0 on C \ F, or
    # b = R - A u) makes the coarse smoothers move u, and the fixed point breaks.
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    o = Oracle(Config(n=n, M=4, seg=S, buffer=2, K=K))
    ustar = _load_exact(o, f)
    before = {p: o.us[o.M][p].copy() for p in o.segs}
    o.vsr(o.M)
    sc = np.abs(ustar).max()
    worst = 0.0
    for p in o.segs:
        CG = o.CG(o.M, p)
        worst = max(worst, np.abs(o.us[o.M][p][CG] - before[p][CG]).max())
    assert worst <= 1e-12 * sc, worst / sc
    # the coarse SR levels saw the consistent tau right-hand sides (a visit happened)
    assert all(o.counters["vsr_visits"][l] == 1 for l in range(o.T + 1, o.M + 1))


def _spy_vsr(o, on_cheb):
    """Wrap Oracle.vsr / vconv / _cheb: on_cheb(phase, l, p, u, b, X) runs before each SR
    smoothing, phase 'pre' (L232) or 'post' (L242); state['tT'] holds t_T at the k = 1
    hand-off (the level-T values right after the restriction, L234)."""
    state = {"active": {}, "tT": None}
    orig_vsr, orig_vconv, orig_cheb = o.vsr, o.vconv, o._cheb

    def vsr(l):
        state["active"][l] = {}
        orig_vsr(l)
        del state["active"][l]

    def vconv(l, b):
        if l == o.T and (o.T + 1) in state["active"]:
            state["tT"] = o.u[o.T][o.dom[o.T]].copy()
        orig_vconv(l, b)

    def cheb(deg, u, b, X, l):
        if l in state["active"]:
            p = next(q for q in o.segs if o.us[l][q] is u)
            seen = state["active"][l]
            phase = "post" if p in seen else "pre"
            seen[p] = True
            on_cheb(phase, l, p, u, b, X)
        orig_cheb(deg, u, b, X, l)

    o.vsr, o.vconv, o._cheb = vsr, vconv, cheb
    return state


def _gsr_mask(o, l, p):
    st = o.storage(l, p)
    m = np.zeros(st.shape, bool)
    for box, val in ((st.intersect(o.dom[l]), True), (o.C(l, p), False)):
        m[tuple(slice(a - s, b - s) for a, b, s in zip(box.lo, box.hi, st.lo))] = val
    return m


def test_corrections_increment_gsr_cells():
    # R17: the correction u += P(w - t) acts on C u GSR, so
    # between the pre- and post-smoothing of an SR visit every GSR cell changes by exactly
    # P(w - t) (the smoother never touches GSR).  K = 3 covers the k = 1 hand-off (w - t
    # from the conventional level T) and k >= 2 (w - t from the segment's own coarse level).
    _check_gsr_increments(Oracle)


class _CorrectCOnly(Oracle):
    """Mutant (the other reading SPEC leaves open): the corrections of the SR V-cycle act on
    C only, so GSR cells stay as the FMG interpolation set them."""

    def vsr(self, l):
        self._in_vsr = getattr(self, "_in_vsr", 0) + 1
        try:
            super().vsr(l)
        finally:
            self._in_vsr -= 1

    def CG(self, l, p):  # inside vsr CG is used by the corrections only
        return self.C(l, p) if getattr(self, "_in_vsr", 0) else super().CG(l, p)


def test_gsr_increment_pin_catches_the_correct_on_c_only_mutation():
    # the pin above is not vacuous: the mutant that corrects C only fails it
    with pytest.raises(AssertionError):
        _check_gsr_increments(_CorrectCOnly)


def _check_gsr_increments(cls):
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    o = cls(Config(n=n, M=4, seg=16, buffer=2, K=3))
    saved, checked, moved = {}, [], [0.0]

    def on_cheb(phase, l, p, u, b, X):
        m = _gsr_mask(o, l, p)
        if phase == "pre":
            saved[(l, p)] = u.a.copy()      # GSR values: unchanged by this smoothing
            return
        lc = l - 1
        if lc == o.T:
            w = o.u[o.T]
            e = O.Field(w.box, fill=0.0)
            e[o.dom[o.T]] = w[o.dom[o.T]] - st["tT"]
        else:
            e = O.Field(o.us[lc][p].box, array=o.us[lc][p].a - o.ts[lc][p].a)
        O.fill_bc_ghosts(e, o.dom[lc])
        stb = o.storage(l, p)
        inc = np.zeros(stb.shape)
        CG = Oracle.CG(o, l, p)     # the region as defined, not o's
        inc[tuple(slice(a - s, c - s) for a, c, s in zip(CG.lo, CG.hi, stb.lo))] = O.prolong(e, CG)
        got = u.a[m] - saved[(l, p)][m]
        np.testing.assert_allclose(got, inc[m], rtol=0, atol=1e-13 * np.abs(u.a[m]).max())
        moved[0] = max(moved[0], np.abs(inc[m]).max() / np.abs(u.a[m]).max())
        checked.append((l, p))

    st = _spy_vsr(o, on_cheb)
    o.solve(f)
    # every SR level and segment, over all the FMG visits, was checked
    assert {l for l, _ in checked} == set(range(o.T + 1, o.M + 1))
    assert moved[0] > 1e-6, moved        # the increments are not trivially zero


def test_tau_gives_zero_residual_on_c_minus_f():
    # R18: on C_{l-1} \ F the coarse rhs is A u (the coarse cells keep
    # their value, zero effective residual); on F it is R + A(I u), so b - A u = R there.
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    o = Oracle(Config(n=n, M=4, seg=8, buffer=4, K=3))
    seen = []

    def on_cheb(phase, l, p, u, b, X):
        if phase != "pre" or (l + 1) not in st["active"]:
            return        # (FMG visits of level l smooth against b = f_l)
        Cc, Fb = o.C(l, p), o.F(l + 1, p)
        ug = u.copy()
        r = O.residual(ug, b, Cc, o.h[l], o.dom[l])
        inF = np.zeros(Cc.shape, bool)
        inF[tuple(slice(a - s, c - s) for a, c, s in zip(Fb.lo, Fb.hi, Cc.lo))] = True
        assert (~inF).any() and inF.any()
        scale = np.abs(O.apply_A(ug, Cc, o.h[l])).max()
        assert np.abs(r[~inF]).max() <= 1e-13 * scale
        assert np.abs(r[inF]).max() > 1e-8 * scale      # R itself, not zero
        seen.append(l)

    st = _spy_vsr(o, on_cheb)
    o.solve(f)
    assert set(seen) == set(range(o.T + 1, o.M))
