"""Closed forms the oracle is pinned to (independent of oracle/ and of the CUDA path).

Nothing here calls the oracle.  Each value follows from the mathematics of the model
problem, not from the algorithm under test:
  * spectrum of the 1D cell-centred Dirichlet operator with reflected ghosts,
    tridiag(-1, 2, -1) with end entries 3:  lambda_k = 4 sin^2(k pi / (2n)),
    v_k(i) = sin(k pi (i + 1/2) / n), k = 1..n  (DST-II basis);
  * the exact discrete solution u_h* = A^{-1} f by DST-II diagonalisation;
  * an independently assembled Kronecker-sum matrix of A for tiny grids;
  * Chebyshev polynomials T_d via numpy.polynomial.
"""
import numpy as np
import scipy.fft


def tridiag_1d(n: int) -> np.ndarray:
    T = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    T[0, 0] = 3.0
    T[-1, -1] = 3.0
    return T


def dense_A(shape, h):
    """Kronecker sum (T_z x I x I + I x T_y x I + I x I x T_x)/h^2 for array order (z,y,x)."""
    nz, ny, nx = shape
    Iz, Iy, Ix = np.eye(nz), np.eye(ny), np.eye(nx)
    A = (np.kron(np.kron(tridiag_1d(nz), Iy), Ix) + np.kron(np.kron(Iz, tridiag_1d(ny)), Ix)
         + np.kron(np.kron(Iz, Iy), tridiag_1d(nx)))
    return A / (h * h)


def eig1d(n: int, k: int):
    i = np.arange(n)
    return 4.0 * np.sin(k * np.pi / (2 * n)) ** 2, np.sin(k * np.pi * (i + 0.5) / n)


def eigvec3(shape, ks, h):
    """Eigenpair of A: (sum of 1D eigenvalues / h^2, tensor product of 1D vectors)."""
    (lz, vz), (ly, vy), (lx, vx) = (eig1d(shape[d], ks[d]) for d in range(3))
    return (lz + ly + lx) / (h * h), vz[:, None, None] * vy[None, :, None] * vx[None, None, :]


def dst_solve(f: np.ndarray, h: float) -> np.ndarray:
    """u_h* with A u = f exactly (up to rounding), via orthonormal DST-II."""
    shape = f.shape
    lam = np.zeros(shape)
    for d in range(3):
        k = np.arange(1, shape[d] + 1)
        l1 = 4.0 * np.sin(k * np.pi / (2 * shape[d])) ** 2
        sh = [1, 1, 1]
        sh[d] = shape[d]
        lam = lam + l1.reshape(sh)
    fh = scipy.fft.dstn(f, type=2, norm="ortho", workers=-1)
    return scipy.fft.idstn(fh * (h * h) / lam, type=2, norm="ortho", workers=-1)


def cheb_T(d: int, x):
    c = np.zeros(d + 1)
    c[d] = 1.0
    return np.polynomial.chebyshev.chebval(x, c)


def cheb_error_factor(d: int, lam, a: float, b: float):
    """R_d(lambda) = T_d((theta - lambda)/delta) / T_d(theta/delta)."""
    theta, delta = 0.5 * (a + b), 0.5 * (b - a)
    return cheb_T(d, (theta - lam) / delta) / cheb_T(d, theta / delta)


def gamma_of_r(r):
    """PAPER.md:150 (§3.2): Gamma = r / (4 r + 3)."""
    return r / (4.0 * r + 3.0)


# ---- 27-point operator (SPEC weights: centre 8/3, faces 0, edges -1/6,
# corners -1/12, times 1/h^2).  With reflected ghosts it is diagonalised by the same DST-II
# basis: the 1D neighbour average (u_{i-1} + u_{i+1})/2 with reflected ends has eigenvalue
# c_k = cos(k pi / n) on v_k, and the stencil is 8/3 - 2/3 (c1 c2 + c2 c3 + c1 c3)
# - 2/3 c1 c2 c3 in those averages.
def lam27(cz, cy, cx, h):
    return (8.0 / 3.0 - (2.0 / 3.0) * (cz * cy + cy * cx + cz * cx) - (2.0 / 3.0) * cz * cy * cx) / (h * h)


def eigvec3_27(shape, ks, h):
    cs, vs = [], []
    for d in range(3):
        n, k = shape[d], ks[d]
        i = np.arange(n)
        cs.append(np.cos(k * np.pi / n))
        vs.append(np.sin(k * np.pi * (i + 0.5) / n))
    return lam27(cs[0], cs[1], cs[2], h), vs[0][:, None, None] * vs[1][None, :, None] * vs[2][None, None, :]


def dst_solve27(f: np.ndarray, h: float) -> np.ndarray:
    """u_h* with A27 u = f via orthonormal DST-II (eigenvalues lam27)."""
    c = [np.cos(np.arange(1, n + 1) * np.pi / n) for n in f.shape]
    lam = lam27(c[0][:, None, None], c[1][None, :, None], c[2][None, None, :], h)
    fh = scipy.fft.dstn(f, type=2, norm="ortho", workers=-1)
    return scipy.fft.idstn(fh / lam, type=2, norm="ortho", workers=-1)
