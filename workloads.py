"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no operator, smoother, transfer or cycle):
it only samples right-hand sides f at cell centres, in fp64, on the host.  Both sides of
every parity test receive the same arrays from here.

Conventions
-----------
* Arrays are numpy fp64, C-contiguous, shape ``(n3, n2, n1)`` -- i.e. x1 is the fastest
  (innermost) index, as in a ``[z][y][x]`` layout.  ``n`` tuples passed to this module are
  in the paper's dimension order ``(n1, n2, n3)``.
* Cell ``i`` of a grid with spacing ``h`` has centre ``x = i*h + h/2``
  (§2 Eq. 2).  The domain is ``prod_d [0, R_d]`` with ``R_d = n_d*h``.

Workloads (BASELINE.json configs, readings R4/R21/R22 of SURVEY.md §8(c)):
* manufactured solution ``u = prod_d (x_d^4 - R_d^2 x_d^2)`` (§5.1), which
  vanishes on every face of the box; ``f = -Lap u`` (BASELINE: "-Lap u = f"; reading R2);
* C3 noise: ``f + sigma * N(0,1)`` with sigma = 1e-3, numpy PCG64(seed), x-fastest fill;
* C5 bumps: 16 Gaussian bumps, centres U[0,1]^3, widths U[0.02,0.1], amplitudes N(0,1),
  drawn bump by bump in the order c, w, a from PCG64(seed).
"""
from __future__ import annotations

import numpy as np

SEED = 14067808  # arXiv id, used for every seeded config


def centres(n: int, h: float) -> np.ndarray:
    """Cell centres x_i = i*h + h/2, i = 0..n-1."""
    return np.arange(n, dtype=np.float64) * h + 0.5 * h


def extents(n, h):
    """Domain extents R_d = n_d * h (reading R4)."""
    return tuple(float(nd) * h for nd in n)


def manufactured_u_at(x, R):
    """u(x) = prod_d (x_d^4 - R_d^2 x_d^2) at one point x = (x1, x2, x3)."""
    return float(np.prod([x[d] ** 4 - R[d] ** 2 * x[d] ** 2 for d in range(3)]))


def manufactured_f_at(x, R):
    """f = -Lap u at one point: -sum_d (12 x_d^2 - 2 R_d^2) prod_{e != d}(x_e^4 - R_e^2 x_e^2)."""
    p = [x[d] ** 4 - R[d] ** 2 * x[d] ** 2 for d in range(3)]
    q = [12.0 * x[d] ** 2 - 2.0 * R[d] ** 2 for d in range(3)]
    return -float(q[0] * p[1] * p[2] + p[0] * q[1] * p[2] + p[0] * p[1] * q[2])


def manufactured_u(n, h, R=None) -> np.ndarray:
    """u(x) = prod_d (x_d^4 - R_d^2 x_d^2) sampled at cell centres."""
    R = extents(n, h) if R is None else R
    g = [centres(n[d], h) for d in range(3)]
    p = [g[d] ** 4 - R[d] ** 2 * g[d] ** 2 for d in range(3)]
    return p[2][:, None, None] * p[1][None, :, None] * p[0][None, None, :]


def manufactured_f(n, h, R=None) -> np.ndarray:
    """f = -Lap u for the manufactured u, analytic, sampled at cell centres.

    d^2/dx^2 (x^4 - R^2 x^2) = 12 x^2 - 2 R^2, so
    f = -sum_d (12 x_d^2 - 2 R_d^2) prod_{e != d} (x_e^4 - R_e^2 x_e^2).
    """
    R = extents(n, h) if R is None else R
    g = [centres(n[d], h) for d in range(3)]
    p = [g[d] ** 4 - R[d] ** 2 * g[d] ** 2 for d in range(3)]
    q = [12.0 * g[d] ** 2 - 2.0 * R[d] ** 2 for d in range(3)]
    f = q[2][:, None, None] * p[1][None, :, None] * p[0][None, None, :]
    f = f + p[2][:, None, None] * q[1][None, :, None] * p[0][None, None, :]
    f = f + p[2][:, None, None] * p[1][None, :, None] * q[0][None, None, :]
    return -f


def manufactured_f_block(h, R, lo, dims) -> np.ndarray:
    """f = -Lap u of the manufactured solution on the block of cells [lo, lo + dims)
    (paper order), shape (dims3, dims2, dims1) -- a multi-GPU rank's (haloed) local block;
    cells outside the domain are evaluated by the same formula (they are never used)."""
    g = [(np.arange(lo[d], lo[d] + dims[d], dtype=np.float64) + 0.5) * h for d in range(3)]
    p = [g[d] ** 4 - R[d] ** 2 * g[d] ** 2 for d in range(3)]
    q = [12.0 * g[d] ** 2 - 2.0 * R[d] ** 2 for d in range(3)]
    f = q[2][:, None, None] * p[1][None, :, None] * p[0][None, None, :]
    f = f + p[2][:, None, None] * q[1][None, :, None] * p[0][None, None, :]
    f = f + p[2][:, None, None] * p[1][None, :, None] * q[0][None, None, :]
    return -f


def noise(n, sigma=1e-3, seed=SEED) -> np.ndarray:
    """i.i.d. N(0, sigma^2), PCG64(seed), filled in x-fastest order (reading R21)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return sigma * rng.standard_normal(size=(n[2], n[1], n[0]), dtype=np.float64)


def gaussian_bumps_params(count=16, seed=SEED):
    """The bumps' (centre, width, amplitude), drawn bump by bump in the order c, w, a from
    PCG64(seed) (reading R22)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(count):
        c = rng.uniform(0.0, 1.0, size=3)
        w = rng.uniform(0.02, 0.1)
        a = rng.standard_normal()
        out.append((c, w, a))
    return out


def gaussian_bumps(n, h, count=16, seed=SEED) -> np.ndarray:
    """f(x) = sum_m a_m exp(-|x - c_m|^2 / (2 w_m^2)) (reading R22)."""
    g = [centres(n[d], h) for d in range(3)]
    f = np.zeros((n[2], n[1], n[0]), dtype=np.float64)
    for c, w, a in gaussian_bumps_params(count, seed):
        e = [np.exp(-((g[d] - c[d]) ** 2) / (2.0 * w * w)) for d in range(3)]
        f += a * (e[2][:, None, None] * e[1][None, :, None] * e[0][None, None, :])
    return f


def gaussian_bumps_block(h, lo, dims, count=16, seed=SEED) -> np.ndarray:
    """gaussian_bumps on the block of cells [lo, lo + dims) (paper order), shape (dims3,
    dims2, dims1): a multi-GPU rank's (haloed) local block; cells outside the domain are
    evaluated by the same formula (they are never used)."""
    g = [(np.arange(lo[d], lo[d] + dims[d], dtype=np.float64) + 0.5) * h for d in range(3)]
    f = np.zeros((dims[2], dims[1], dims[0]), dtype=np.float64)
    for c, w, a in gaussian_bumps_params(count, seed):
        e = [np.exp(-((g[d] - c[d]) ** 2) / (2.0 * w * w)) for d in range(3)]
        f += a * (e[2][:, None, None] * e[1][None, :, None] * e[0][None, None, :])
    return f


def rhs_block(kind: str, n, h, lo, dims, seed=SEED) -> np.ndarray:
    """make_rhs(kind, n, h) restricted to the block [lo, lo + dims) (cells outside the
    domain: the formula's value, or 0 for the sampled noise/random kinds)."""
    if kind == "manufactured":
        return manufactured_f_block(h, extents(n, h), lo, dims)
    if kind == "bumps":
        return gaussian_bumps_block(h, lo, dims, 16, seed)
    full = make_rhs(kind, n, h, seed)
    out = np.zeros((dims[2], dims[1], dims[0]), dtype=np.float64)
    src = [slice(max(lo[d], 0), min(lo[d] + dims[d], n[d])) for d in range(3)]
    dst = [slice(src[d].start - lo[d], src[d].stop - lo[d]) for d in range(3)]
    out[dst[2], dst[1], dst[0]] = full[src[2], src[1], src[0]]
    return out


def random_field(n, seed=SEED, scale=1.0) -> np.ndarray:
    """Plain N(0, scale^2) field (used for operator-level parity inputs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return scale * rng.standard_normal(size=(n[2], n[1], n[0]), dtype=np.float64)


# ---------------------------------------------------------------------------------------
# BASELINE.json configs.  `n` in paper order (n1, n2, n3).
# ---------------------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(n=(32, 32, 32), M=4, seg=16, buffer=2, K=2, rhs="manufactured"),
    "C2": dict(n=(128, 128, 128), M=6, seg=32, buffer=2, K=3, rhs="manufactured"),
    "C3": dict(n=(512, 512, 512), M=8, seg=64, buffer=2, K=4, rhs="manufactured+noise"),
    "C4": dict(n=(512, 512, 512), M=8, seg=64, buffer=2, K=4, rhs="manufactured"),
    "C5": dict(n=(1024, 1024, 1024), M=9, seg=32, buffer=2, K=4, rhs="bumps"),
}


def make_rhs(kind: str, n, h=None, seed=SEED) -> np.ndarray:
    """Right-hand side for a config kind; h defaults to 1/n1 (unit cube for cubes)."""
    h = 1.0 / n[0] if h is None else h
    if kind == "manufactured":
        return manufactured_f(n, h)
    if kind == "manufactured+noise":
        return manufactured_f(n, h) + noise(n, 1e-3, seed)
    if kind == "bumps":
        return gaussian_bumps(n, h, 16, seed)
    if kind == "random":
        return random_field(n, seed)
    raise ValueError(f"unknown rhs kind {kind!r}")
