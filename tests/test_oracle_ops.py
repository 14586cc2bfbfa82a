"""Pins of the oracle's multigrid components against closed forms (CPU only)."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from oracle import Box, Field
from tests import pins

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- inputs
def test_manufactured_points_match_spec_examples():
    g = json.load(open(os.path.join(GOLD, "manufactured_points.json")))
    R = g["R"]
    for pt in g["points"]:
        assert W.manufactured_u_at(pt["x"], R) == pytest.approx(pt["u"], abs=1e-15)
        if "lap_u" in pt:
            assert W.manufactured_f_at(pt["x"], R) == pytest.approx(-pt["lap_u"], rel=1e-15)


def test_manufactured_f_is_minus_laplacian_by_finite_differences():
    # f = -Lap u: compare with a 4th-order central difference of u at random points
    rng = np.random.default_rng(0)
    R = (2.0, 1.0, 1.0)
    for _ in range(5):
        x = rng.uniform(0.1, 0.9, 3) * np.array(R)
        e = 1e-3
        lap = 0.0
        for d in range(3):
            xs = [x.copy() for _ in range(5)]
            for j, o in enumerate((-2, -1, 0, 1, 2)):
                xs[j][d] += o * e
            v = [W.manufactured_u_at(z, R) for z in xs]
            lap += (-v[0] + 16 * v[1] - 30 * v[2] + 16 * v[3] - v[4]) / (12 * e * e)
        assert W.manufactured_f_at(x, R) == pytest.approx(-lap, rel=1e-7, abs=1e-9)


def test_sampled_fields_match_point_formulas():
    n, h = (8, 4, 4), 0.25
    R = W.extents(n, h)
    u, f = W.manufactured_u(n, h), W.manufactured_f(n, h)
    for (k, j, i) in [(0, 0, 0), (3, 2, 7), (1, 3, 4)]:
        x = ((i + 0.5) * h, (j + 0.5) * h, (k + 0.5) * h)
        assert u[k, j, i] == pytest.approx(W.manufactured_u_at(x, R), rel=1e-14)
        assert f[k, j, i] == pytest.approx(W.manufactured_f_at(x, R), rel=1e-14)


def test_seeded_inputs_are_deterministic():
    assert np.array_equal(W.noise((8, 8, 8)), W.noise((8, 8, 8)))
    b1, b2 = W.gaussian_bumps((16, 16, 16), 1 / 16), W.gaussian_bumps((16, 16, 16), 1 / 16)
    assert np.array_equal(b1, b2) and np.abs(b1).max() > 0


# ----------------------------------------------------------------------------- boxes
def test_box_algebra_examples():
    b = Box((0, 0, 0), (4, 4, 4))
    assert b.grow(2) == Box((-2, -2, -2), (6, 6, 6))
    assert b.grow(0) == b
    assert b.intersect(Box((2, 2, 2), (6, 6, 6))) == Box((2, 2, 2), (4, 4, 4))
    assert b.intersect(Box((4, 4, 4), (6, 6, 6))).empty
    assert b.refine() == Box((0, 0, 0), (8, 8, 8))
    assert b.refine().coarsen_inner() == b
    assert Box((-3, 1, 2), (7, 5, 9)).coarsen_inner() == Box((-1, 1, 1), (3, 2, 4))


# ----------------------------------------------------------------------------- ghosts
def test_bc_ghosts_face_edge_corner():
    dom = Box((0, 0, 0), (3, 3, 3))
    u = Field(dom.grow(1), fill=0.0)
    u[dom] = np.arange(27.0).reshape(3, 3, 3) + 1.0
    O.fill_bc_ghosts(u, dom)
    a = u.a  # a[i+1] is cell i
    assert a[0, 2, 2] == -a[1, 2, 2]                # face: -mirror
    assert a[0, 0, 2] == +a[1, 1, 2]                # edge: (+1) * mirror
    assert a[0, 0, 0] == -a[1, 1, 1]                # corner: (-1)^3 * mirror
    assert a[4, 4, 4] == -a[3, 3, 3]
    # deeper out-of-domain cells are poisoned
    v = Field(dom.grow(2), fill=1.0)
    O.fill_bc_ghosts(v, dom)
    assert np.isnan(v.a[0, 3, 3]) and not np.isnan(v.a[1, 3, 3])


def test_bc_ghosts_leave_in_domain_cells_alone():
    dom = Box((0, 0, 0), (8, 8, 8))
    st = Box((2, -3, 4), (9, 5, 11))   # a segment storage box crossing two faces
    u = Field(st, fill=7.0)
    O.fill_bc_ghosts(u, dom)
    inside = st.intersect(dom)
    assert np.all(u[inside] == 7.0)


# ----------------------------------------------------------------------------- operator
@pytest.mark.parametrize("shape,ks", [((4, 6, 8), (1, 2, 3)), ((4, 6, 8), (4, 6, 8)),
                                      ((5, 3, 7), (2, 3, 1)), ((2, 2, 2), (1, 2, 1))])
def test_operator_eigenpairs(shape, ks):
    h = 0.37
    lam, v = pins.eigvec3(shape, ks, h)
    dom = Box((0, 0, 0), shape)
    u = Field(dom.grow(1))
    u[dom] = v
    O.fill_bc_ghosts(u, dom)
    Av = O.apply_A(u, dom, h)
    assert np.abs(Av - lam * v).max() <= 1e-13 * lam * np.abs(v).max()


def test_lambda_max_is_12_over_h2():
    # R8: lambda_max(A_l) = 12/h_l^2 exactly (1D lambda_n = 4 sin^2(pi/2) = 4)
    for n in (2, 3, 4, 8, 16):
        lam = np.linalg.eigvalsh(pins.tridiag_1d(n))
        assert lam.max() == pytest.approx(4.0 * np.sin(n * np.pi / (2 * n)) ** 2, abs=1e-13)
        assert abs(lam.max() - 4.0) < 1e-12


@pytest.mark.parametrize("deg,coef", [(2, (1.0, 0.0, 0.0)), (3, (0.5, -2.0, 1.5))])
def test_operator_exact_on_cubics_interior(deg, coef):
    # -Lap of sum_d c_d x_d^deg, evaluated at interior cells (no boundary involvement)
    h = 0.1
    dom = Box((0, 0, 0), (8, 8, 8))
    big = dom.grow(1)
    x = [(np.arange(big.lo[d], big.hi[d]) + 0.5) * h for d in range(3)]
    u = Field(big)
    u.a = (coef[0] * x[0][:, None, None] ** deg + coef[1] * x[1][None, :, None] ** deg
           + coef[2] * x[2][None, None, :] ** deg) * np.ones(big.shape)
    Au = O.apply_A(u, dom, h)  # no ghost fill: pure interior stencil on a grown box
    xs = [(np.arange(dom.lo[d], dom.hi[d]) + 0.5) * h for d in range(3)]
    exact = -deg * (deg - 1) * (coef[0] * xs[0][:, None, None] ** (deg - 2)
                                + coef[1] * xs[1][None, :, None] ** (deg - 2)
                                + coef[2] * xs[2][None, None, :] ** (deg - 2))
    assert np.abs(Au - exact).max() < 1e-9


def test_dense_operator_matches_kronecker_assembly():
    for shape in [(2, 2, 2), (2, 3, 4), (4, 4, 4)]:
        dom = Box((0, 0, 0), shape)
        h = 0.25
        assert np.abs(O.dense_operator(dom, h) - pins.dense_A(shape, h)).max() < 1e-12


@pytest.mark.parametrize("shape", [(2, 2, 2), (4, 2, 2), (4, 4, 4), (2, 4, 8)])
def test_exact_solve_matches_dst_and_kronecker(shape):
    rng = np.random.default_rng(1)
    b = rng.standard_normal(shape)
    h = 0.5
    u = O.exact_solve(b, Box((0, 0, 0), shape), h)
    u_dst = pins.dst_solve(b, h)
    u_kr = np.linalg.solve(pins.dense_A(shape, h), b.ravel()).reshape(shape)
    assert np.abs(u - u_dst).max() < 1e-13 * np.abs(u_dst).max()
    assert np.abs(u - u_kr).max() < 1e-13 * np.abs(u_kr).max()


def test_dst_solve_residual():
    n = (16, 8, 12)
    f = W.manufactured_f(n, 1 / 16)
    u = pins.dst_solve(f, 1 / 16)
    r = f - (pins.dense_A(f.shape, 1 / 16) @ u.ravel()).reshape(f.shape)
    assert np.abs(r).max() < 1e-11 * np.abs(f).max()


# ----------------------------------------------------------------------------- smoother
@pytest.mark.parametrize("deg", [1, 2, 3])
@pytest.mark.parametrize("ks", [(1, 1, 1), (3, 5, 2), (8, 8, 8), (2, 7, 8)])
def test_chebyshev_eigenvector_response(deg, ks):
    # b = 0, u = v_k  ->  S^deg u = R_deg(lambda_k) v_k  with R_d = T_d((theta-l)/delta)/T_d(sigma)
    shape, h = (8, 8, 8), 1 / 8
    lam, v = pins.eigvec3(shape, ks, h)
    dom = Box((0, 0, 0), shape)
    u = Field(dom.grow(1))
    u[dom] = v
    b = Field(dom, fill=0.0)
    O.cheb(deg, u, b, dom, h, dom, 1 / 6, 1.0)
    lm = 12 / h ** 2
    factor = pins.cheb_error_factor(deg, lam, lm / 6, lm)
    assert np.abs(u[dom] - factor * v).max() < 1e-13


def test_chebyshev_deg1_is_richardson_with_optimal_weight():
    shape, h = (6, 6, 6), 0.2
    dom = Box((0, 0, 0), shape)
    rng = np.random.default_rng(3)
    u0 = rng.standard_normal(shape)
    b = Field(dom, array=rng.standard_normal(shape))
    u = Field(dom.grow(1))
    u[dom] = u0
    O.cheb(1, u, b, dom, h, dom, 0.25, 1.0)
    lm = 12 / h ** 2
    A = pins.dense_A(shape, h)
    expect = u0.ravel() + 2.0 / (0.25 * lm + lm) * (b.a.ravel() - A @ u0.ravel())
    assert np.abs(u[dom].ravel() - expect).max() < 1e-12


def test_chebyshev_fixed_point_and_frozen_cells():
    shape, h = (8, 8, 8), 1 / 8
    dom = Box((0, 0, 0), shape)
    rng = np.random.default_rng(4)
    ustar = rng.standard_normal(shape)
    b = Field(dom, array=(pins.dense_A(shape, h) @ ustar.ravel()).reshape(shape))
    u = Field(dom.grow(1))
    u[dom] = ustar
    O.cheb(2, u, b, dom, h, dom, 1 / 6, 1.0)
    assert np.abs(u[dom] - ustar).max() < 1e-12
    # update region X strictly inside: cells of dom outside X must not change
    X = Box((2, 2, 2), (6, 6, 6))
    u2 = Field(dom.grow(1))
    u2[dom] = rng.standard_normal(shape)
    before = u2[dom].copy()
    O.cheb(2, u2, b, X, h, dom, 1 / 6, 1.0)
    mask = np.ones(shape, bool)
    mask[2:6, 2:6, 2:6] = False
    assert np.array_equal(u2[dom][mask], before[mask])


# ----------------------------------------------------------------------------- transfers
def test_restriction_mean_constant_linear():
    fine = Field(Box((0, 0, 0), (4, 4, 4)), array=np.zeros((4, 4, 4)))
    fine.a[0:2, 0:2, 0:2] = np.arange(8.0).reshape(2, 2, 2)
    assert O.restrict_avg8(fine, Box((0, 0, 0), (1, 1, 1)))[0, 0, 0] == 3.5
    fine.a[:] = 2.5
    assert np.all(O.restrict_avg8(fine, Box((0, 0, 0), (2, 2, 2))) == 2.5)
    h = 0.125
    x = (np.arange(8) + 0.5) * h
    fine = Field(Box((0, 0, 0), (8, 8, 8)),
                 array=1.0 + 2 * x[:, None, None] - 3 * x[None, :, None] + 0.5 * x[None, None, :]
                 + 0 * x[None, None, :])
    X = (np.arange(4) + 0.5) * 2 * h
    exp = 1.0 + 2 * X[:, None, None] - 3 * X[None, :, None] + 0.5 * X[None, None, :]
    assert np.abs(O.restrict_avg8(fine, Box((0, 0, 0), (4, 4, 4))) - exp).max() < 1e-14


def test_prolongation_weights_partition_of_unity_and_linear_exactness():
    H = 0.25
    cdom = Box((0, 0, 0), (4, 4, 4))
    src = Field(cdom.grow(1), fill=1.0)
    assert np.all(O.prolong(src, Box((0, 0, 0), (8, 8, 8))) == 1.0)
    # linear function vanishing on the x1 = 0 face: reflected ghosts reproduce it exactly
    Xc = (np.arange(-1, 5) + 0.5) * H
    src.a = np.broadcast_to(Xc[None, None, :], src.box.shape).copy()
    O.fill_bc_ghosts(src, cdom)      # ghosts at x1=-1 become -x_0 = x_{-1}; others reflect
    fine = O.prolong(src, Box((0, 0, 0), (8, 8, 8)))
    xf = (np.arange(8) + 0.5) * H / 2
    # exact up to and including the x1 = 0 face cell; the x1 = 1 face reflects about a
    # different zero, and the x2/x3 faces flip the (constant-in-x2,x3) function's sign, so
    # compare only rows away from those faces
    assert np.abs(fine[1:-1, 1:-1, :-1] - xf[None, None, :-1]).max() < 1e-14
    # 1D weights: left child of parent j gets 0.75 u_j + 0.25 u_{j-1}
    src.a = np.zeros(src.box.shape)
    src.a[2, 2, 2] = 1.0              # coarse cell (1,1,1)
    fine = O.prolong(src, Box((0, 0, 0), (8, 8, 8)))
    assert fine[2, 2, 2] == 27 / 64 and fine[1, 2, 2] == 9 / 64 and fine[1, 1, 1] == 1 / 64
    assert fine[4, 2, 2] == 9 / 64 and fine[0, 2, 2] == 0.0
    # sum of all child weights of one coarse cell = 8 (each fine cell's weights sum to 1)
    assert fine.sum() == pytest.approx(8.0)


# ----------------------------------------------------------------------------- 27-point
# SURVEY f1 ("27-point stencil, second order"; weights per SPEC / reading R28)
@pytest.mark.parametrize("shape,ks", [((4, 4, 4), (1, 1, 1)), ((6, 4, 8), (5, 2, 7)),
                                      ((8, 8, 8), (8, 1, 1)), ((3, 5, 2), (2, 5, 1))])
def test_27pt_operator_eigenpairs(shape, ks):
    # pins the edge/corner ghost reflection (-1)^m: A27 v_k = lam27(k) v_k on the DST basis
    h = 0.3
    lam, v = pins.eigvec3_27(shape, ks, h)
    dom = Box((0, 0, 0), shape)
    u = Field(dom.grow(1))
    u[dom] = v
    O.fill_bc_ghosts(u, dom)
    assert np.abs(O.apply_A(u, dom, h, "27pt") - lam * v).max() < 1e-12 * lam


def test_27pt_lambda_max_bound_and_high_frequency_band():
    # R28: sup of the symbol is 4/h^2 (at c = (-1, 1, 1)); over the high frequencies of
    # full coarsening (some theta_d >= pi/2) its minimum is 4/3 /h^2 (at theta = (pi,pi,pi))
    h = 1.0
    th = np.linspace(0, np.pi, 181)
    c = np.cos(th)
    L = pins.lam27(c[:, None, None], c[None, :, None], c[None, None, :], h)
    assert L.max() == pytest.approx(4.0, abs=1e-12) and L.min() == pytest.approx(0.0, abs=1e-12)
    hi = (th[:, None, None] >= np.pi / 2) | (th[None, :, None] >= np.pi / 2) | (th[None, None, :] >= np.pi / 2)
    assert L[hi].min() == pytest.approx(4.0 / 3.0, abs=1e-12)
    from oracle.ops import lambda_max
    assert lambda_max(0.5, "27pt") == 16.0 and lambda_max(0.5) == 48.0


@pytest.mark.parametrize("poly", ["x2", "xy", "yz2", "lin"])
def test_27pt_operator_exact_on_quadratics_interior(poly):
    h = 0.1
    dom = Box((0, 0, 0), (6, 6, 6))
    big = dom.grow(1)
    z, y, x = np.meshgrid(*[(np.arange(big.lo[d], big.hi[d]) + 0.5) * h for d in range(3)],
                          indexing="ij")
    f = {"x2": (x * x, -2.0), "xy": (x * y, 0.0), "yz2": (y * y + 3 * z * z, -8.0),
         "lin": (2 * x - y + 0.5 * z + 1, 0.0)}[poly]
    u = Field(big)
    u.a = f[0]
    assert np.abs(O.apply_A(u, dom, h, "27pt") - f[1]).max() < 1e-9


@pytest.mark.parametrize("shape", [(2, 2, 2), (4, 2, 2), (2, 4, 8)])
def test_27pt_exact_solve_matches_dst(shape):
    rng = np.random.default_rng(7)
    b = rng.standard_normal(shape)
    h = 0.5
    u = O.exact_solve(b, Box((0, 0, 0), shape), h, "27pt")
    assert np.abs(u - pins.dst_solve27(b, h)).max() < 1e-12 * np.abs(u).max()


def test_27pt_discretisation_second_order_on_paper_domain():
    # Omega = [0,2] x [0,1]^2, u = prod(x^4 - R^2 x^2): exact discrete
    # solutions by DST converge at second order (ratio ~4 per halving)
    errs = []
    for N in (8, 16, 32, 64):
        n = (2 * N, N, N)
        h = 1.0 / N
        f = W.manufactured_f(n, h)
        u = W.manufactured_u(n, h)
        errs.append(np.abs(pins.dst_solve27(f, h) - u).max())
    ratios = [a / b for a, b in zip(errs, errs[1:])]
    assert 3.5 < ratios[-1] < 4.5, ratios


@pytest.mark.parametrize("deg", [1, 2])
def test_27pt_chebyshev_eigenvector_response(deg):
    shape, h = (8, 8, 8), 1 / 8
    dom = Box((0, 0, 0), shape)
    lm = 4 / h ** 2
    for ks in [(1, 1, 1), (8, 1, 1), (8, 8, 8), (3, 6, 2)]:
        lam, v = pins.eigvec3_27(shape, ks, h)
        u = Field(dom.grow(1))
        u[dom] = v
        O.cheb(deg, u, Field(dom, fill=0.0), dom, h, dom, 1 / 3, 1.0, "27pt")
        factor = pins.cheb_error_factor(deg, lam, lm / 3, lm)
        assert np.abs(u[dom] - factor * v).max() < 1e-13
