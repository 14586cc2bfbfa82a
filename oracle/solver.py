"""FAS-FMG with segmental refinement, transcribed step by step (oracle; TEST INFRASTRUCTURE).

Follows, in the paper's order and notation:
  fig:mgv   FASMGV     PAPER.md:108-125   -> Oracle.vconv
  fig:fmg   FMG        PAPER.md:134-146   -> Oracle.fmg_conventional
  fig:fmgsr FASFMGSR   PAPER.md:216-227   -> Oracle.solve (SR part)
  fig:mgvsr FASMGVSR   PAPER.md:229-246   -> Oracle.vsr
with the model solver of §5.1: refinement ratio 2, piecewise-constant
restriction, linear prolongation for Pi and the correction, Chebyshev F(1,2,2).

Global level index l: 0 = coarsest ... M = finest.  T = M - K is the
transition level (the paper's SR index k = 0); SR levels are l = T+1..M.
Readings where the paper is silent or ambiguous (R1..R25) are those of SURVEY.md §8(c);
DESIGN.md §3 lists them.  fp64 throughout.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .grid import Box, Field
from .ops import (apply_A, cheb, exact_solve, fill_bc_ghosts, prolong, residual,
                  restrict_avg8)


@dataclass
class Config:
    n: Tuple[int, int, int]          # fine cells per dimension, paper order (n1, n2, n3)
    M: int                           # coarsenings; coarsest grid n / 2^M
    seg: int = 0                     # S, genuine segment edge on the finest level
    buffer: int = 2                  # J (constant buffer, Eq. 5 with A = J, B = 0)
    K: int = 0                       # number of SR levels (0 = conventional FMG)
    h: Optional[float] = None        # fine cell size (default 1/n1)
    sched: Optional[Tuple] = None    # Eq. 5 (A, B), or ("mbs", J1); overrides `buffer`
    alpha: int = 1                   # F(alpha, nu1, nu2)
    nu1: int = 2
    nu2: int = 2
    lo_frac: Optional[float] = None  # Chebyshev interval as fractions of lambda_max (R8):
    hi_frac: float = 1.0             #   default 1/6 (7-point) or 1/3 (27-point, R28)
    stencil: str = "7pt"             # "7pt" (R1, BASELINE) or "27pt" (f1)
    nl_gamma: float = 0.0            # f4 (R29): A(u) = -L_h u + nl_gamma u^3 (FAS, nonlinear)
    fas: bool = True                 # False: correction scheme (I-hat = 0)

    def validate(self):
        n, M, K, S = self.n, self.M, self.K, self.seg
        if not (0 <= K <= M):
            raise ValueError("need 0 <= K <= M")
        for nd in n:
            if nd % (1 << M):
                raise ValueError("n_d must be divisible by 2^M")
            if K > 0 and (S <= 0 or nd % S):
                raise ValueError("n_d must be divisible by seg")
        if K > 0 and S % (1 << K):
            raise ValueError("seg must be divisible by 2^K")
        if self.buffer < 0:
            raise ValueError("buffer must be >= 0")

    def J(self, k: int) -> int:
        """Buffer width of SR level k (1..K): Eq. 5, PAPER.md:192 (R14); or the maximum
        buffer schedule (MBS): J_1 given and the finer buffers completely
        support grid k = 1, i.e. C_k = F_k for k < K.  With F_k = grow(V_k, floor(J_{k+1}/2))
        (R15) that is J_{k+1} = 2 J_k, so J_k = 2^(k-1) J_1."""
        if self.sched is None:
            return self.buffer
        if self.sched[0] == "mbs":
            return int(self.sched[1]) << (k - 1)
        A, B = self.sched
        return 2 * ((A + B * (self.K - k)) // 2)


class Oracle:
    """One solver instance; `solve(f)` returns u on the fine grid (array order z,y,x)."""

    def __init__(self, cfg: Config):
        cfg.validate()
        self.cfg = cfg
        self.st = cfg.stencil
        self.lo_frac = cfg.lo_frac if cfg.lo_frac is not None else (
            1.0 / 6.0 if cfg.stencil == "7pt" else 1.0 / 3.0)
        M, K = cfg.M, cfg.K
        self.M, self.K, self.T = M, K, M - K
        n_arr = (cfg.n[2], cfg.n[1], cfg.n[0])
        h = (1.0 / cfg.n[0]) if cfg.h is None else cfg.h
        self.N = [tuple(v >> (M - l) for v in n_arr) for l in range(M + 1)]
        self.h = [h * (1 << (M - l)) for l in range(M + 1)]
        self.dom = [Box((0, 0, 0), self.N[l]) for l in range(M + 1)]
        # conventional (global) fields, l <= T: storage grow(Omega_l, 1)
        self.u = {l: Field(self.dom[l].grow(1)) for l in range(self.T + 1)}
        # SR segments (R13): S_l = S / 2^(M-l); segment grid identical on every SR level
        self.nseg = tuple(v // cfg.seg for v in n_arr) if K > 0 else (0, 0, 0)
        self.segs = [tuple(p) for p in np.ndindex(*self.nseg)] if K > 0 else []
        self.us = {l: {} for l in range(self.T + 1, M + 1)}
        self.bs = {l: {} for l in range(self.T + 1, M + 1)}
        self.ts = {l: {} for l in range(self.T + 1, M + 1)}
        self.f = None
        self.counters = {"vconv_visits": [0] * (M + 1), "vsr_visits": [0] * (M + 1)}
        # decomposition hook (tests of the multi-rank path): a rank processes only its own
        # `segs`; at the k = 1 hand-off exchange_T(u_T, R_T) fills the other ranks' V_T^p
        # blocks (the levels <= T are then solved redundantly on every rank)
        self.exchange_T = None

    # ------------------------------------------------------------------------------
    # SR regions (readings R13-R15)
    # ------------------------------------------------------------------------------
    def S_l(self, l):
        return self.cfg.seg >> (self.M - l)

    def Jl(self, l):
        return self.cfg.J(l - self.T)

    def V(self, l, p) -> Box:
        """Genuine region ^p Omega^V_l: the segment's own S_l^3 cells."""
        s = self.S_l(l)
        return Box([q * s for q in p], [(q + 1) * s for q in p])

    def storage(self, l, p) -> Box:
        """Segment storage grow(V, J+1) = compute region plus its ghost layer (unclipped)."""
        return self.V(l, p).grow(self.Jl(l) + 1)

    def C(self, l, p) -> Box:
        """Compute region ^p Omega^C = grow(V, J) cap Omega."""
        return self.V(l, p).grow(self.Jl(l)).intersect(self.dom[l])

    def CG(self, l, p) -> Box:
        """C cup GSR = grow(C, 1) cap Omega: the range of prolongation."""
        return self.storage(l, p).intersect(self.dom[l])

    def F(self, l, p) -> Box:
        """Support of C_l on level l-1 (R15): coarse cells whose 8 children
        all lie in C_l^p  (= grow(V_{l-1}, floor(J/2)) cap Omega_{l-1})."""
        return self.C(l, p).coarsen_inner()

    # ------------------------------------------------------------------------------
    # Cheb helpers
    # ------------------------------------------------------------------------------
    def _cheb(self, deg, u, b, X, l):
        cheb(deg, u, b, X, self.h[l], self.dom[l], self.lo_frac, self.cfg.hi_frac, self.st,
             self.cfg.nl_gamma)

    # ------------------------------------------------------------------------------
    # fig:mgv, FASMGV(L_l, u_l, b_l) on the conventional (global) levels; u_l in place
    # ------------------------------------------------------------------------------
    def vconv(self, l: int, b: Field) -> None:
        self.counters["vconv_visits"][l] += 1
        u, dom, h = self.u[l], self.dom[l], self.h[l]
        if l == 0:
            u[dom] = exact_solve(b[dom], dom, h, self.st, self.cfg.nl_gamma)
            return
        self._cheb(self.cfg.nu1, u, b, dom, l)                        # L112
        r = Field(dom, array=residual(u, b, dom, h, dom, self.st, self.cfg.nl_gamma))  # L113
        uc, domc, hc = self.u[l - 1], self.dom[l - 1], self.h[l - 1]
        R = restrict_avg8(r, domc)                                    # L115  r_{k-1}
        if self.cfg.fas:
            uc[domc] = restrict_avg8(u, domc)                         # L114  u_{k-1}=Î u_k
        else:
            uc[domc] = 0.0                                            # Î = 0 (L127): CS
        t = uc.copy()                                                 # L116  t_{k-1}
        fill_bc_ghosts(uc, domc)
        bc = Field(domc, array=R + apply_A(uc, domc, hc, self.st, self.cfg.nl_gamma))  # L117 (Eq. 4)
        self.vconv(l - 1, bc)                                         # L117  w_{k-1}
        e = Field(uc.box, array=uc.a - t.a)
        fill_bc_ghosts(e, domc)
        u[dom] = u[dom] + prolong(e, dom)                             # L118
        self._cheb(self.cfg.nu2, u, b, dom, l)                        # L119

    # ------------------------------------------------------------------------------
    # fig:fmg on levels 0..T
    # ------------------------------------------------------------------------------
    def fmg_conventional(self) -> None:
        u0 = self.u[0]
        u0[self.dom[0]] = 0.0                                         # L137
        self.vconv(0, self.f[0])                                      # L138 (exact, R12)
        for l in range(1, self.T + 1):                                # L139
            src = self.u[l - 1]
            fill_bc_ghosts(src, self.dom[l - 1])
            self.u[l][self.dom[l]] = prolong(src, self.dom[l])        # L140 Pi
            self._cheb(self.cfg.alpha, self.u[l], self.f[l], self.dom[l], l)   # L141
            self.vconv(l, self.f[l])                                  # L142

    # ------------------------------------------------------------------------------
    # fig:mgvsr, FASMGVSR on SR level l (k = l - T >= 1), all segments
    # ------------------------------------------------------------------------------
    def vsr(self, l: int) -> None:
        self.counters["vsr_visits"][l] += 1
        T, h, dom = self.T, self.h[l], self.dom[l]
        k = l - T
        r = {}
        for p in self.segs:                                           # L232 (+ r for L235)
            C = self.C(l, p)
            self._cheb(self.cfg.nu1, self.us[l][p], self.bs[l][p], C, l)
            r[p] = Field(C, array=residual(self.us[l][p], self.bs[l][p], C, h, dom, self.st, self.cfg.nl_gamma))
        if k == 1:
            # R16: level T is conventional; each segment restricts onto V_T^p only
            uT, domT, hT = self.u[T], self.dom[T], self.h[T]
            RT = Field(domT)
            for p in self.segs:
                VT = self.V(T, p)
                if self.cfg.fas:
                    uT[VT] = restrict_avg8(self.us[l][p], VT)         # L233 Î
                else:
                    uT[VT] = 0.0
                RT[VT] = restrict_avg8(r[p], VT)                      # L235 I(r)
            if self.exchange_T is not None:
                self.exchange_T(uT, RT)
            t = uT.copy()                                             # L234
            fill_bc_ghosts(uT, domT)
            bT = Field(domT, array=RT[domT] + apply_A(uT, domT, hT, self.st, self.cfg.nl_gamma))  # L235
            self.vconv(T, bT)                                         # L237-238 FASMGV
            e = Field(uT.box, array=uT.a - t.a)
            fill_bc_ghosts(e, domT)
            for p in self.segs:                                       # L241
                CG = self.CG(l, p)
                u = self.us[l][p]
                u[CG] = u[CG] + prolong(e, CG)
        else:
            lc, hc, domc = l - 1, self.h[l - 1], self.dom[l - 1]
            for p in self.segs:
                uc = self.us[lc][p]
                Fb = self.F(l, p)
                if self.cfg.fas:
                    uc[Fb] = restrict_avg8(self.us[l][p], Fb)         # L233 on F
                else:
                    uc[Fb] = 0.0
                R = restrict_avg8(r[p], Fb)                           # L235 on F
                self.ts[lc][p] = uc.copy()                            # L234 (whole storage)
                fill_bc_ghosts(uc, domc)
                Cc = self.C(lc, p)
                bc = self.bs[lc][p]
                bc[Cc] = apply_A(uc, Cc, hc, self.st, self.cfg.nl_gamma)  # L236 on C \ F
                bc[Fb] = R + apply_A(uc, Fb, hc, self.st, self.cfg.nl_gamma)  # L235 on F
            self.vsr(lc)                                              # L240
            for p in self.segs:                                       # L241
                e = Field(self.us[lc][p].box, array=self.us[lc][p].a - self.ts[lc][p].a)
                fill_bc_ghosts(e, domc)
                CG = self.CG(l, p)
                u = self.us[l][p]
                u[CG] = u[CG] + prolong(e, CG)
        for p in self.segs:                                           # L242
            self._cheb(self.cfg.nu2, self.us[l][p], self.bs[l][p], self.C(l, p), l)

    # ------------------------------------------------------------------------------
    # fig:fmgsr, FASFMGSR; returns u on the fine grid
    # ------------------------------------------------------------------------------
    def solve(self, f_fine: np.ndarray) -> np.ndarray:
        M, T, K = self.M, self.T, self.K
        f_fine = np.asarray(f_fine, dtype=np.float64)
        assert f_fine.shape == self.N[M]
        # R6: f_{l-1} := avg8(f_l) (the ABI receives only the fine f)
        self.f = {M: Field(self.dom[M], array=f_fine.copy())}
        for l in range(M, 0, -1):
            self.f[l - 1] = Field(self.dom[l - 1], array=restrict_avg8(self.f[l], self.dom[l - 1]))
        self.fmg_conventional()                                       # L219 u_0 <- FMG
        for k in range(1, K + 1):                                     # L220
            l = T + k
            for p in self.segs:
                st = self.storage(l, p)
                u = Field(st)
                if k == 1:
                    src = self.u[T]
                    fill_bc_ghosts(src, self.dom[T])
                else:
                    src = self.us[l - 1][p]
                    fill_bc_ghosts(src, self.dom[l - 1])
                CG = self.CG(l, p)
                u[CG] = prolong(src, CG)                              # L221 on C cup GSR
                b = Field(st)
                C = self.C(l, p)
                b[C] = self.f[l][C]
                self.us[l][p], self.bs[l][p] = u, b
                if l < M:
                    self.ts[l][p] = None
                self._cheb(self.cfg.alpha, u, b, C, l)                # L222 on C
            self.vsr(l)                                               # L223
        out = np.empty(self.N[M])
        if K == 0:
            out[...] = self.u[M][self.dom[M]]
        else:
            for p in self.segs:                                       # R19: genuine cells
                V = self.V(M, p)
                sl = tuple(slice(a, b) for a, b in zip(V.lo, V.hi))
                out[sl] = self.us[M][p][V]
        return out


def solve(f: np.ndarray, cfg: Config) -> np.ndarray:
    """Convenience wrapper: one FASFMGSR solve of A u = f (array order z,y,x)."""
    return Oracle(cfg).solve(f)


def vcycle_iterate(f: np.ndarray, cfg: Config, cycles: int, u0: Optional[np.ndarray] = None):
    """Repeated conventional FASMGV(M) from u0 (default 0); returns the list of iterates.

    Used by the tests to measure the V-cycle contraction Gamma.
    """
    o = Oracle(Config(**{**cfg.__dict__, "K": 0}))
    M = o.M
    o.f = {M: Field(o.dom[M], array=np.asarray(f, dtype=np.float64).copy())}
    o.u[M][o.dom[M]] = 0.0 if u0 is None else u0
    its = []
    for _ in range(cycles):
        o.vconv(M, o.f[M])
        its.append(o.u[M][o.dom[M]].copy())
    return its


def vsolve(f: np.ndarray, cfg: Config, rtol: float = 1e-4, maxit: int = 50):
    """Conventional V-cycle solver: "the solve times for a V-cycle
    solve with a relative residual tolerance of 10^-4".  From u = 0 on
    Omega_M, repeat FASMGV(M) (fig:mgv) until ||f - A u||_2 / ||f||_2 <=
    rtol (reading R26: 2-norm over the fine grid, checked before every cycle).

    Returns (u, cycles, history of the relative residual norms, one per check).
    """
    o = Oracle(Config(**{**cfg.__dict__, "K": 0}))
    M, dom, h = o.M, o.dom[o.M], o.h[o.M]
    fM = Field(dom, array=np.asarray(f, dtype=np.float64).copy())
    o.f = {M: fM}
    u = o.u[M]
    u[dom] = 0.0
    fn = float(np.linalg.norm(fM[dom]))
    hist = []
    for it in range(maxit + 1):
        rel = float(np.linalg.norm(residual(u, fM, dom, h, dom, o.st, o.cfg.nl_gamma))) / fn
        hist.append(rel)
        if rel <= rtol or it == maxit:
            return u[dom].copy(), it, hist
        o.vconv(M, fM)
