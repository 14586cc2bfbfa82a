"""Domain-decomposed run of the oracle (TEST INFRASTRUCTURE for tests/test_multirank_cpu.py).

Mirrors the library's multi-GPU schedule on top of the plain oracle: a rank
runs only its own SR segments; the conventional levels A < l <= T are held as
the rank's block, with the ghost ring refreshed by a halo exchange (three face phases over
torch.distributed, gloo) before every operator application ("ghost
cells ... before each operator application"); level A is all-gathered and the levels <= A
run redundantly.  Each step is the oracle's own function on the block
box; the Chebyshev recurrence is the oracle's (oracle/ops.py cheb) with an exchange before
each operator application.  The partition (blocks, A) comes from the product's
sr_fmg_partition.  With exact exchanges the result equals the serial oracle bitwise.
"""
import numpy as np
import torch
import torch.distributed as dist

from oracle import Box, Field, Oracle
from oracle.ops import apply_A, cheb_constants, fill_bc_ghosts, prolong, residual, restrict_avg8


class DDOracle(Oracle):
    def __init__(self, cfg, part, pgrid, idle=False):
        super().__init__(cfg)
        self.part, self.pgrid = part, pgrid
        # idle coarse grid (desc.coarse_idle): the level-A blocks are
        # gathered onto rank 0, which alone runs the levels <= A and sends u_A (and t_A)
        # back; emulated for decomposed A < T (the agglomeration at T is the base vsr's)
        self.idle = idle
        self.A = part["level_A"]
        self.world = int(np.prod(pgrid))
        self.rank = part["rank"]
        c = part["coord"]
        lo = [c[d] * part["segs_per_rank"][d] for d in range(3)]
        hi = [lo[d] + part["segs_per_rank"][d] for d in range(3)]
        self.segs = [p for p in self.segs if all(lo[d] <= p[2 - d] < hi[d] for d in range(3))]
        self.n_exchanges = 0

    # -- partition ------------------------------------------------------------------------
    def blk(self, l, rank=None):
        """The rank's block of Omega_l (array order z, y, x)."""
        p = self.part
        s = self.M - l
        if rank is None:
            lo = [p["block_lo"][d] >> s for d in range(3)]
        else:
            c = (rank % self.pgrid[0], (rank // self.pgrid[0]) % self.pgrid[1],
                 rank // (self.pgrid[0] * self.pgrid[1]))
            lo = [c[d] * (p["block_n"][d] >> s) for d in range(3)]
        n = [p["block_n"][d] >> s for d in range(3)]
        return Box((lo[2], lo[1], lo[0]), (lo[2] + n[2], lo[1] + n[1], lo[0] + n[0]))

    def dd(self, l):
        return self.world > 1 and self.A < l <= self.T

    def _rank_of(self, c):
        return c[0] + self.pgrid[0] * (c[1] + self.pgrid[1] * c[2])

    def halo(self, u, l, w=1):
        """Three phases x, y, z: send the w boundary planes of the block to the neighbours,
        receive theirs into the ghost layers; later phases include earlier ghosts (edges,
        corners)."""
        B = self.blk(l)
        c = self.part["coord"]
        for dl in range(3):                    # library dimension (x, y, z) ...
            ad = 2 - dl                        # ... is array axis 2, 1, 0
            lo_nb, hi_nb = c[dl] > 0, c[dl] < self.pgrid[dl] - 1
            if not (lo_nb or hi_nb):
                continue
            rng = []
            N = self.dom[l].hi
            for ax in range(3):
                e = 2 - ax
                if e < dl:  # (layers beyond the domain face are the reflected ghosts)
                    rng.append((max(B.lo[ax] - w, 0), min(B.hi[ax] + w, N[ax])))
                else:
                    rng.append((B.lo[ax], B.hi[ax]))
            ops, recvs = [], []

            def box_at(a0, a1):
                r = list(rng)
                r[ad] = (a0, a1)
                return Box([x[0] for x in r], [x[1] for x in r])

            for side, ok in ((-1, lo_nb), (1, hi_nb)):
                if not ok:
                    continue
                cc = list(c)
                cc[dl] += side
                peer = self._rank_of(cc)
                if side < 0:
                    sb, rb = box_at(B.lo[ad], B.lo[ad] + w), box_at(B.lo[ad] - w, B.lo[ad])
                else:
                    sb, rb = box_at(B.hi[ad] - w, B.hi[ad]), box_at(B.hi[ad], B.hi[ad] + w)
                snd = torch.from_numpy(np.ascontiguousarray(u[sb]))
                rcv = torch.empty(rb.shape, dtype=torch.float64)
                ops.append(dist.isend(snd, peer))
                ops.append(dist.irecv(rcv, peer))
                recvs.append((rb, rcv))
            for op in ops:
                op.wait()
            for rb, rcv in recvs:
                u[rb] = rcv.numpy()
            self.n_exchanges += 1

    def gather(self, l, fields):
        """All-gather of every rank's block of level l into the global fields (idle: a
        gather onto rank 0 only)."""
        for fld in fields:
            mine = torch.from_numpy(np.ascontiguousarray(fld[self.blk(l)]))
            if self.idle:
                got = [torch.empty_like(mine) for _ in range(self.world)] if self.rank == 0 else None
                dist.gather(mine, got, dst=0)
                if self.rank != 0:
                    continue
            else:
                got = [torch.empty_like(mine) for _ in range(self.world)]
                dist.all_gather(got, mine)
            for q in range(self.world):
                fld[self.blk(l, q)] = got[q].numpy()
        self.n_exchanges += 1

    def solves_A(self):
        return not self.idle or self.rank == 0

    def bcast(self, fields):
        """Idle coarse grid: rank 0's whole arrays to every rank."""
        for fld in fields:
            buf = torch.from_numpy(np.ascontiguousarray(fld.a))
            dist.broadcast(buf, src=0)
            fld.a[...] = buf.numpy()
        self.n_exchanges += 1

    # -- the oracle's Chebyshev recurrence with an exchange before each application -------
    def _dd_cheb(self, deg, u, b, X, l):
        if deg <= 0:
            return
        h, dom = self.h[l], self.dom[l]
        theta, delta, sigma = cheb_constants(h, self.lo_frac, self.cfg.hi_frac, self.st)
        g = self.cfg.nl_gamma
        self.halo(u, l)
        x_prev = u.copy()
        fill_bc_ghosts(x_prev, dom)
        x = x_prev.copy()
        x[X] = x_prev[X] + (b[X] - apply_A(x_prev, X, h, self.st, g)) / theta
        rho_prev = 1.0 / sigma
        for _ in range(1, deg):
            rho = 1.0 / (2.0 * sigma - rho_prev)
            self.halo(x, l)
            fill_bc_ghosts(x, dom)
            x_new = x.copy()
            x_new[X] = (x[X] + rho * rho_prev * (x[X] - x_prev[X])
                        + (2.0 * rho / delta) * (b[X] - apply_A(x, X, h, self.st, g)))
            x_prev, x, rho_prev = x, x_new, rho
        u[X] = x[X]

    # -- fig:mgv on a decomposed level ------------------------------------------------------
    def vconv(self, l, b):
        if not self.dd(l):
            return super().vconv(l, b)
        self.counters["vconv_visits"][l] += 1
        u, dom, h = self.u[l], self.dom[l], self.h[l]
        B = self.blk(l)
        g = self.cfg.nl_gamma
        self._dd_cheb(self.cfg.nu1, u, b, B, l)                          # L112
        self.halo(u, l)
        r = Field(B, array=residual(u, b, B, h, dom, self.st, g))        # L113
        lc = l - 1
        uc, domc, hc, Bc = self.u[lc], self.dom[lc], self.h[lc], self.blk(lc)
        uc[Bc] = restrict_avg8(u, Bc)                                    # L114
        R = Field(domc, fill=0.0)
        R[Bc] = restrict_avg8(r, Bc)                                     # L115
        if not self.dd(lc):                                              # agglomerate A
            self.gather(lc, (uc, R))
            t = uc.copy()
            fill_bc_ghosts(uc, domc)
            bc = Field(domc, array=R[domc] + apply_A(uc, domc, hc, self.st, g))
        else:
            self.halo(uc, lc)
            t = uc.copy()                                                # L116 (with ghosts)
            fill_bc_ghosts(uc, domc)
            bc = Field(domc, fill=0.0)
            bc[Bc] = R[Bc] + apply_A(uc, Bc, hc, self.st, g)             # L117 (Eq. 4)
        if self.dd(lc) or self.solves_A():
            self.vconv(lc, bc)
        if self.idle and not self.dd(lc):
            self.bcast((uc, t))                                          # w_A, t_A
        if self.dd(lc):
            self.halo(uc, lc)                                            # w on the ghosts
        e = Field(uc.box, array=uc.a - t.a)
        fill_bc_ghosts(e, domc)
        u[B] = u[B] + prolong(e, B)                                      # L118
        self._dd_cheb(self.cfg.nu2, u, b, B, l)                          # L119

    def fmg_conventional(self):
        assert not self.idle or self.A < self.T, "idle emulated for decomposed A < T only"
        u0 = self.u[0]
        u0[self.dom[0]] = 0.0
        if self.solves_A():
            self.vconv(0, self.f[0])
        for l in range(1, self.T + 1):
            if l <= self.A and not self.solves_A():
                continue                                                 # idle rank
            if self.idle and l == self.A + 1:
                self.bcast((self.u[self.A],))                            # u_A for Pi
            src = self.u[l - 1]
            if self.dd(l - 1):
                self.halo(src, l - 1)
            fill_bc_ghosts(src, self.dom[l - 1])
            X = self.blk(l) if self.dd(l) else self.dom[l]
            self.u[l][X] = prolong(src, X)                               # L140 Pi
            if self.dd(l):
                self._dd_cheb(self.cfg.alpha, self.u[l], self.f[l], X, l)
            else:
                self._cheb(self.cfg.alpha, self.u[l], self.f[l], X, l)  # L141
            self.vconv(l, self.f[l])                                     # L142
        if self.K > 0 and self.dd(self.T):
            # the FMG interpolation into the first SR level (fig:fmgsr L221) reads u_T on
            # the segments' footprints, partly in the neighbouring blocks
            self._footprint(self.u[self.T])

    # -- the k = 1 hand-off with a decomposed level T ---------------------------------------
    def _footprint(self, fld):
        """The level-T values the segments' interpolation reads: grow(V_T^p, ceil(J/2) + 1)
        (R15), i.e. ghost layers that deep from the neighbouring blocks."""
        G = (self.Jl(self.T + 1) + 1) // 2 + 1
        self.halo(fld, self.T, G)

    def vsr(self, l):
        T = self.T
        if l - T != 1 or not self.dd(T):
            if l - T == 1 and self.world > 1:       # agglomeration at T: gather u_T, R_T
                self.exchange_T = lambda uT, RT: self.gather(T, (uT, RT))
            return super().vsr(l)
        self.counters["vsr_visits"][l] += 1
        h, dom = self.h[l], self.dom[l]
        g = self.cfg.nl_gamma
        r = {}
        for p in self.segs:                                               # L232
            C = self.C(l, p)
            self._cheb(self.cfg.nu1, self.us[l][p], self.bs[l][p], C, l)
            r[p] = Field(C, array=residual(self.us[l][p], self.bs[l][p], C, h, dom, self.st, g))
        uT, domT, hT, BT = self.u[T], self.dom[T], self.h[T], self.blk(T)
        RT = Field(domT, fill=0.0)
        for p in self.segs:
            VT = self.V(T, p)
            uT[VT] = restrict_avg8(self.us[l][p], VT)                     # L233
            RT[VT] = restrict_avg8(r[p], VT)                              # L235
        self.halo(uT, T)
        t = uT.copy()                                                     # L234
        fill_bc_ghosts(uT, domT)
        bT = Field(domT, fill=0.0)
        bT[BT] = RT[BT] + apply_A(uT, BT, hT, self.st, g)
        self.vconv(T, bT)                                                 # L237-238
        e = Field(uT.box, fill=0.0)
        e[BT] = uT[BT] - t[BT]
        self._footprint(e)
        fill_bc_ghosts(e, domT)
        for p in self.segs:                                               # L241
            CG = self.CG(l, p)
            u = self.us[l][p]
            u[CG] = u[CG] + prolong(e, CG)
        for p in self.segs:                                               # L242
            self._cheb(self.cfg.nu2, self.us[l][p], self.bs[l][p], self.C(l, p), l)
