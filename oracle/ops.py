"""Multigrid components of the model problem, fp64 (oracle; TEST INFRASTRUCTURE ONLY).

Every function follows one passage of PAPER.md (or a reading R<n> of SURVEY.md §8(c),
listed in DESIGN.md §3).  Plain numpy slicing; no blocking, fusion or reordering.

  fill_bc_ghosts  R3:  PAPER.md:160-161 (§3.3) "Boundary ghost cell values are set with
                  appropriate (linear) interpolation of interior values before each
                  operator application": u_ghost = -u_mirror (linear through 0 at the face),
                  per dimension sequentially => (-1)^m u_mirror at edges/corners.
  apply_A         R1/R2: A = -Lap_h, 7-point cell-centred FD on h_l (Eq. 2;
                  re-discretised coarse operators PAPER.md:91); or the
                  paper's "27-point stencil, second order" with SPEC's
                  trilinear FE/FV weights: centre 8/3, faces 0, edges -1/6, corners -1/12.
  cheb            R8: PAPER.md:133, 257 (§5.1) Chebyshev smoother of degree d on
                  [lo_frac, hi_frac] * lambda_max, lambda_max = 12/h^2 (7-point) or 4/h^2
                  (27-point: the supremum of its symbol, R28).
  restrict_avg8   R9: "simple averaging"/"piecewise constant restriction".
  prolong         R10: "linear prolongation": cell-centred trilinear,
                  1D weights 3/4 (parent) and 1/4 (neighbour on the child's side).
"""
from __future__ import annotations

import itertools

import numpy as np

from .grid import Box, Field

W1D = (0.75, 0.25)


def fill_bc_ghosts(u: Field, domain: Box) -> None:
    """Set the out-of-domain cells of u's storage (R3).

    Depth-1 ghosts (the layer just outside a face) get (-1)^m * mirror; deeper
    out-of-domain cells are set to NaN so that any read of them poisons the result.
    """
    box = u.box
    a = u.a
    # 1. every out-of-domain cell -> NaN
    inside = [(np.arange(box.lo[d], box.hi[d]) >= domain.lo[d]) &
              (np.arange(box.lo[d], box.hi[d]) < domain.hi[d]) for d in range(3)]
    mask = inside[0][:, None, None] & inside[1][None, :, None] & inside[2][None, None, :]
    a[~mask] = np.nan
    # 2. face rule, one dimension after another (sequential => (-1)^m at edges/corners)
    for d in range(3):
        for ghost, mirror in ((domain.lo[d] - 1, domain.lo[d]), (domain.hi[d], domain.hi[d] - 1)):
            if not (box.lo[d] <= ghost < box.hi[d]):
                continue
            assert box.lo[d] <= mirror < box.hi[d]
            gi = [slice(None)] * 3
            mi = [slice(None)] * 3
            gi[d] = ghost - box.lo[d]
            mi[d] = mirror - box.lo[d]
            a[tuple(gi)] = -a[tuple(mi)]


def _shift(u: Field, X: Box, o) -> np.ndarray:
    return u[Box([a + d for a, d in zip(X.lo, o)], [b + d for b, d in zip(X.hi, o)])]


def apply_A(u: Field, X: Box, h: float, stencil: str = "7pt", gamma: float = 0.0) -> np.ndarray:
    """(A u)_i on X, A = -L_h (R1, R2).

    7pt:  (6 u_i - sum_{+-e_d} u_{i+-e_d}) / h^2.
    27pt: (8/3 u_i - 1/6 sum_{12 edge neighbours} - 1/12 sum_{8 corner neighbours}) / h^2,
          face neighbours weight 0 (SPEC "Stencil weights"; R28).
    gamma > 0 (reading R29): the nonlinear FAS test operator A(u) = -L_h u +
    gamma u^3 (monotone cubic reaction term, pointwise).
    Reads u on grow(X,1) as stored (ghosts, incl. edges/corners, filled by the caller).
    """
    c = u[X]
    s = np.zeros(X.shape)
    nl = gamma * c * c * c if gamma else 0.0
    if stencil == "7pt":
        for d in range(3):
            for o in (-1, 1):
                off = [0, 0, 0]
                off[d] = o
                s = s + _shift(u, X, off)
        return (6.0 * c - s) / (h * h) + nl
    if stencil != "27pt":
        raise ValueError(f"unknown stencil {stencil!r}")
    e = np.zeros(X.shape)
    k = np.zeros(X.shape)
    for o in itertools.product((-1, 0, 1), repeat=3):
        nz = sum(1 for v in o if v)
        if nz == 2:
            e = e + _shift(u, X, o)
        elif nz == 3:
            k = k + _shift(u, X, o)
    return ((8.0 / 3.0) * c - e / 6.0 - k / 12.0) / (h * h) + nl


def residual(u: Field, b: Field, X: Box, h: float, domain: Box, stencil: str = "7pt",
             gamma: float = 0.0) -> np.ndarray:
    """r = b - A(u) on X (fig:mgv PAPER.md:113)."""
    fill_bc_ghosts(u, domain)
    return b[X] - apply_A(u, X, h, stencil, gamma)


def lambda_max(h: float, stencil: str = "7pt") -> float:
    """Largest eigenvalue bound of A_l (Appendix A of SURVEY): 12/h^2 for the 7-point
    operator (attained); for the 27-point operator the supremum of its symbol
    (8/3 - 2/3 (c1c2 + c2c3 + c1c3) - 2/3 c1c2c3)/h^2 over c_d in [-1, 1], which is 4/h^2
    at (c1, c2, c3) = (-1, 1, 1) (R28)."""
    return (12.0 if stencil == "7pt" else 4.0) / (h * h)


def cheb_constants(h: float, lo_frac: float, hi_frac: float, stencil: str = "7pt"):
    """theta, delta, sigma of the Chebyshev interval [a, b] (R8; lambda_max per stencil)."""
    lam = lambda_max(h, stencil)
    a, b = lo_frac * lam, hi_frac * lam
    theta = 0.5 * (b + a)
    delta = 0.5 * (b - a)
    return theta, delta, theta / delta


def cheb(deg: int, u: Field, b: Field, X: Box, h: float, domain: Box,
         lo_frac: float, hi_frac: float, stencil: str = "7pt", gamma: float = 0.0) -> None:
    """u <- S^deg(L, u, b) on X: one degree-`deg` Chebyshev polynomial (R8).

    Three-term Chebyshev recurrence:  x1 = x0 + r0/theta;
    x_{k+1} = x_k + rho_k rho_{k-1} (x_k - x_{k-1}) + (2 rho_k / delta) r_k,
    rho_0 = 1/sigma, rho_k = 1/(2 sigma - rho_{k-1}),  r_k = b - A x_k.
    Every operator application reads u (incl. frozen GSR cells and reflected GBC ghosts)
    from before the sweep; only cells of X are updated.
    """
    if deg <= 0:
        return
    theta, delta, sigma = cheb_constants(h, lo_frac, hi_frac, stencil)
    x_prev = u.copy()
    fill_bc_ghosts(x_prev, domain)
    x = x_prev.copy()
    x[X] = x_prev[X] + (b[X] - apply_A(x_prev, X, h, stencil, gamma)) / theta
    rho_prev = 1.0 / sigma
    for _ in range(1, deg):
        rho = 1.0 / (2.0 * sigma - rho_prev)
        fill_bc_ghosts(x, domain)
        x_new = x.copy()
        x_new[X] = (x[X] + rho * rho_prev * (x[X] - x_prev[X])
                    + (2.0 * rho / delta) * (b[X] - apply_A(x, X, h, stencil, gamma)))
        x_prev, x, rho_prev = x, x_new, rho
    u[X] = x[X]


def restrict_avg8(fine: Field, Z: Box) -> np.ndarray:
    """(1/8) * sum of the 8 children of every coarse cell of Z (R9)."""
    sub = fine[Z.refine()]
    out = np.zeros(Z.shape)
    for a, b, c in itertools.product((0, 1), repeat=3):
        out = out + sub[a::2, b::2, c::2]
    return out / 8.0


def prolong(src: Field, Y: Box) -> np.ndarray:
    """Cell-centred trilinear interpolation of `src` onto fine cells Y (R10).

    Fine cell i has parent I = floor(i/2) and, per dimension, a neighbour on the child's
    side: I-1 for an even (left) child, I+1 for an odd (right) child.  Weights 3/4 and
    1/4 per dimension (tensor products 27/64 ... 1/64).  `src` must hold valid values
    (incl. reflected ghosts) on the whole footprint.
    """
    idx = []
    for d in range(3):
        i = np.arange(Y.lo[d], Y.hi[d])
        p = np.floor_divide(i, 2)
        s = np.where(i % 2 == 0, -1, 1)
        idx.append((p - src.box.lo[d], p + s - src.box.lo[d]))
        assert idx[d][0].min() >= 0 and idx[d][1].min() >= 0
        assert idx[d][0].max() < src.box.shape[d] and idx[d][1].max() < src.box.shape[d]
    out = np.zeros(Y.shape)
    for a, b, c in itertools.product((0, 1), repeat=3):
        w = W1D[a] * W1D[b] * W1D[c]
        out = out + w * src.a[np.ix_(idx[0][a], idx[1][b], idx[2][c])]
    return out


def dense_operator(domain: Box, h: float, stencil: str = "7pt") -> np.ndarray:
    """The matrix of A on a (tiny) domain, column j = A e_j (used for the exact solve)."""
    n = domain.volume
    A = np.zeros((n, n))
    for j in range(n):
        e = Field(domain.grow(1), fill=0.0)
        e.a[1:-1, 1:-1, 1:-1].flat[j] = 1.0
        fill_bc_ghosts(e, domain)
        A[:, j] = apply_A(e, domain, h, stencil).ravel()
    return A


def exact_solve(b: np.ndarray, domain: Box, h: float, stencil: str = "7pt",
                gamma: float = 0.0) -> np.ndarray:
    """u = A^{-1} b on the coarsest grid (fig:mgv PAPER.md:121, R7): dense LU in fp64.

    gamma > 0 (R29): A(u) = A_lin u + gamma u^3 = b solved exactly by Newton's method with
    the dense Jacobian A_lin + 3 gamma diag(u^2), to rounding."""
    A = dense_operator(domain, h, stencil)
    bb = b.ravel()
    u = np.linalg.solve(A, bb)
    if gamma:
        for _ in range(50):
            F = A @ u + gamma * u ** 3 - bb
            du = np.linalg.solve(A + np.diag(3.0 * gamma * u * u), F)
            u = u - du
            if np.abs(du).max() <= 1e-16 * max(np.abs(u).max(), 1e-300):
                break
    return u.reshape(domain.shape)
