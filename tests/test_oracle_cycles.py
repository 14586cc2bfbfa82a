"""Pins of the oracle's cycles (FASMGV, FMG) and of SR (FASFMGSR/FASMGVSR). CPU only."""
import itertools

import numpy as np
import pytest

import oracle as O
import workloads as W
from oracle import Box, Config, Field
from tests import pins


def _mf(N):
    n = (N, N, N)
    return n, W.manufactured_f(n, 1 / N), W.manufactured_u(n, 1 / N)


# ----------------------------------------------------------------------------- FASMGV
def test_vcycle_fixed_point_at_exact_discrete_solution():
    # u = u_h* (DST, A u = f to rounding) must be left unchanged by a V(2,2) cycle
    n, f, _ = _mf(16)
    ustar = pins.dst_solve(f, 1 / 16)
    it = O.vcycle_iterate(f, Config(n=n, M=3), 1, u0=ustar)[0]
    assert np.abs(it - ustar).max() < 1e-12 * np.abs(ustar).max()


def test_fas_equals_correction_scheme_on_linear_problem():
    # I-hat = 0 recovers CS multigrid; for a linear A and linear smoother the
    # two cycles coincide (up to rounding) from the same start
    n = (16, 16, 16)
    f = W.random_field(n, seed=5)
    u0 = W.random_field(n, seed=6)
    a = O.vcycle_iterate(f, Config(n=n, M=3, fas=True), 2, u0=u0)
    b = O.vcycle_iterate(f, Config(n=n, M=3, fas=False), 2, u0=u0)
    for x, y in zip(a, b):
        assert np.abs(x - y).max() < 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("N,M", [(16, 3), (32, 4)])
def test_vcycle_contraction_below_quarter(N, M):
    # need Gamma < 0.25 for FMG; measure the algebraic-error reduction
    n = (N, N, N)
    f = W.random_field(n, seed=7)
    ustar = pins.dst_solve(f, 1 / N)
    its = O.vcycle_iterate(f, Config(n=n, M=M), 4)
    errs = [np.abs(ustar)] + [np.abs(x - ustar) for x in its]
    ratios = [errs[i + 1].max() / errs[i].max() for i in range(1, 4)]
    assert max(ratios) < 0.25, ratios


def test_gamma_of_r_formula_values():
    # Gamma = r/(4r+3); r = 1 -> 1/7, r -> inf -> 1/4
    assert pins.gamma_of_r(1.0) == pytest.approx(1 / 7)
    assert pins.gamma_of_r(3.0) == pytest.approx(0.2)
    assert pins.gamma_of_r(1e12) == pytest.approx(0.25)


# ----------------------------------------------------------------------------- FMG (K=0)
@pytest.mark.parametrize("N,M", [(16, 3), (32, 4), (64, 5)])
def test_fmg_algebraic_error_below_discretisation_error(N, M):
    # FMG reduces the algebraic error to the ORDER of the discretisation
    # error.  PAPER.md:149-150: with a per-level reduction Gamma, the ratio r of algebraic to
    # discretisation error obeys Gamma = r/(4r+3), i.e. r <= 3 Gamma / (1 - 4 Gamma).
    # (With the measured Gamma ~ 0.2 of this V(2,2) that bound is r <= 3, approached from
    # below as N grows; e_alg < e_disc itself is NOT implied -- see DESIGN.md §3 R11.)
    n, f, u = _mf(N)
    ustar = pins.dst_solve(f, 1 / N)
    ufmg = O.solve(f, Config(n=n, M=M, K=0))
    e_alg = np.abs(ufmg - ustar).max()
    e_disc = np.abs(ustar - u).max()
    its = O.vcycle_iterate(f, Config(n=n, M=M), 3)
    g = max(np.abs(its[i + 1] - ustar).max() / np.abs(its[i] - ustar).max() for i in range(2))
    assert g < 0.25
    assert e_alg / e_disc <= 3 * g / (1 - 4 * g)


def test_discretisation_second_order():
    # PAPER.md:478 "2nd-order accuracy": the exact discrete solution's error halves twice
    # per halving of h; ratio in [3.6, 4.4] for N >= 32
    errs = {}
    for N in (32, 64, 128):
        n, f, u = _mf(N)
        errs[N] = np.abs(pins.dst_solve(f, 1 / N) - u).max()
    for a, b in [(32, 64), (64, 128)]:
        assert 3.6 <= errs[a] / errs[b] <= 4.4, errs


def test_fmg_total_error_order():
    # FMG total error converges at 2nd order asymptotically; pre-asymptotically r grows
    # towards its induction limit, so the per-halving ratio rises towards 4 from below
    errs = {}
    for N, M in [(32, 4), (64, 5), (128, 6)]:
        n, f, u = _mf(N)
        errs[N] = np.abs(O.solve(f, Config(n=n, M=M)) - u).max()
    q1, q2 = errs[32] / errs[64], errs[64] / errs[128]
    assert 2.5 < q1 < q2 < 4.4, errs


def test_fmg_ratio_bounded_as_h_shrinks():
    # asymptotic exactness: r = e_alg/e_disc stays bounded by the
    # induction limit as N doubles, and it grows towards it (monotone) rather than away
    rs = []
    for N, M in [(8, 2), (16, 3), (32, 4), (64, 5)]:
        n, f, u = _mf(N)
        ustar = pins.dst_solve(f, 1 / N)
        rs.append(np.abs(O.solve(f, Config(n=n, M=M)) - ustar).max() / np.abs(ustar - u).max())
    assert all(a < b for a, b in zip(rs, rs[1:]))
    assert rs[-1] < 3.0


def test_fmg_exact_on_coarsest_only():
    # M = 0: the solve is the exact coarsest solve (fig:fmg L137-138)
    n = (2, 4, 2)
    f = W.random_field(n, seed=8)
    u = O.solve(f, Config(n=n, M=0, K=0, h=0.5))
    assert np.abs(u - pins.dst_solve(f, 0.5)).max() < 1e-14 * np.abs(u).max()


def test_fmg_non_cubic_domain():
    # C4-style global grid (2,1,1) x 16 with R = (2,1,1): coarsest 2R cells; still O(h^2)
    errs = []
    for N in (16, 32):
        n = (2 * N, N, N)
        h = 1 / N
        f = W.manufactured_f(n, h)
        u = W.manufactured_u(n, h)
        ustar = pins.dst_solve(f, h)
        ufmg = O.solve(f, Config(n=n, M=int(np.log2(N)) - 0, K=0, h=h))
        assert np.abs(ufmg - ustar).max() < 3.0 * np.abs(ustar - u).max()
        errs.append(np.abs(ufmg - u).max())
    assert 2.5 < errs[0] / errs[1] < 4.6


# ---- conventional V-cycle solver to a relative residual tolerance
def test_vsolve_converges_to_the_exact_discrete_solution():
    # against the exact discrete solution (DST, tests/pins.py): independent of the cycle
    from tests.pins import dst_solve
    n = (32, 32, 32)
    f = W.make_rhs("manufactured+noise", n)
    ustar = dst_solve(f, 1.0 / n[0])
    u, it, hist = O.vsolve(f, Config(n=n, M=4), rtol=1e-10, maxit=40)
    assert hist[-1] <= 1e-10 and it < 40
    assert np.linalg.norm(u - ustar) / np.linalg.norm(ustar) < 1e-8
    # geometric reduction by about the measured V(2,2) contraction (Gamma < 0.25, L151)
    ratios = [b / a for a, b in zip(hist[1:], hist[2:])]
    assert max(ratios) < 0.3, ratios


def test_vsolve_tolerance_semantics():
    n = (32, 32, 32)
    f = W.make_rhs("bumps", n)
    u, it, hist = O.vsolve(f, Config(n=n, M=4), rtol=1e-4)
    assert hist[0] == pytest.approx(1.0) and hist[-1] <= 1e-4 < hist[-2]
    assert len(hist) == it + 1
    # a tolerance the zero guess already meets needs no cycle
    u0, it0, _ = O.vsolve(f, Config(n=n, M=4), rtol=1.0)
    assert it0 == 0 and np.all(u0 == 0)


# ---- 27-point operator on the paper's domain [0,2]x[0,1]^2 ----
def test_27pt_vcycle_contraction_and_fmg_accuracy():
    from tests.pins import dst_solve27
    N = 16
    n, h = (2 * N, N, N), 1.0 / N
    f = W.manufactured_f(n, h)
    cfg = Config(n=n, M=3, h=h, stencil="27pt")
    ustar = dst_solve27(f, h)
    # V(2,2) contraction from a zero guess (PAPER.md:149-151 asks Gamma < 1/4)
    its = O.vcycle_iterate(f, cfg, 4)
    e = [np.linalg.norm(u - ustar) for u in its]
    assert max(b / a for a, b in zip(e, e[1:])) < 0.25, e
    # FMG: algebraic error of the order of the discretisation error (R11 bound r <= 3)
    u = O.solve(f, cfg)
    e_alg = np.abs(u - ustar).max()
    e_disc = np.abs(ustar - W.manufactured_u(n, h)).max()
    assert e_alg < 3.0 * e_disc, (e_alg, e_disc)
    # the fixed point: the exact discrete solution is left unchanged by a V-cycle
    it = O.vcycle_iterate(f, cfg, 1, u0=ustar)[0]
    assert np.abs(it - ustar).max() < 1e-12 * np.abs(ustar).max()


# ---- nonlinear FAS (reading R29): A(u) = -Lap_h u + gamma u^3 -----------------
GAMMA = 1.0e4   # gamma u^2 ~ 2.4 against lambda_min(-Lap) ~ 3 pi^2: a visible nonlinearity


def _nl_problem(N, gamma=GAMMA):
    n, h = (N, N, N), 1.0 / N
    u = W.manufactured_u(n, h)
    return n, h, u, W.manufactured_f(n, h) + gamma * u ** 3


def test_nl_exact_coarse_solve_is_a_root():
    # Newton with the dense Jacobian reaches the root of A(u) = b; checked against the
    # operator written out independently (Kronecker assembly) and scipy's root finder
    import scipy.optimize
    shape, h = (2, 4, 4), 0.25
    rng = np.random.default_rng(5)
    b = 50.0 * rng.standard_normal(shape)
    u = O.exact_solve(b, Box((0, 0, 0), shape), h, gamma=GAMMA)
    A = pins.dense_A(shape, h)
    F = A @ u.ravel() + GAMMA * u.ravel() ** 3 - b.ravel()
    assert np.abs(F).max() < 1e-11 * np.abs(b).max()
    v = scipy.optimize.fsolve(lambda x: A @ x + GAMMA * x ** 3 - b.ravel(),
                              np.linalg.solve(A, b.ravel()), xtol=1e-14)
    assert np.abs(u.ravel() - v).max() < 1e-10 * np.abs(v).max()


def test_nl_operator_truncation_error_second_order():
    # the discrete nonlinear operator applied to the manufactured u reproduces f to O(h^2)
    errs = []
    for N in (16, 32, 64):
        n, h, u, f = _nl_problem(N)
        dom = Box((0, 0, 0), u.shape)
        uf = Field(dom.grow(1))
        uf[dom] = u
        r = O.residual(uf, Field(dom, array=f), dom, h, dom, gamma=GAMMA)
        errs.append(np.abs(r[2:-2, 2:-2, 2:-2]).max())   # interior: boundary rows are O(1)
    assert 3.5 < errs[0] / errs[1] < 4.5 and 3.5 < errs[1] / errs[2] < 4.5, errs


def test_nl_fas_vcycle_contracts_and_fmg_reaches_discretisation_accuracy():
    N, M = 32, 4
    n, h, u, f = _nl_problem(N)
    cfg = Config(n=n, M=M, nl_gamma=GAMMA)
    ustar, it, hist = O.vsolve(f, cfg, rtol=1e-12, maxit=60)   # the discrete solution
    assert hist[-1] <= 1e-12
    ratios = [b / a for a, b in zip(hist[1:], hist[2:-1])]
    assert max(ratios) < 0.25, ratios                       # FAS V(2,2) contraction
    # the FAS fixed point: a V-cycle leaves the discrete solution unchanged
    again = O.vcycle_iterate(f, cfg, 1, u0=ustar)[0]
    assert np.abs(again - ustar).max() < 1e-11 * np.abs(ustar).max()
    ufmg = O.solve(f, cfg)
    e_alg = np.abs(ufmg - ustar).max()
    e_disc = np.abs(ustar - u).max()
    assert e_alg < 3.0 * e_disc, (e_alg, e_disc)
    # and the nonlinearity matters: the linear solve of the same f is far off
    assert np.abs(O.solve(f, Config(n=n, M=M)) - ustar).max() > 4 * e_disc
