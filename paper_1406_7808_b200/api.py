"""Thin Python front end of the SR-FMG C ABI (argument marshalling only).

PyTorch supplies device memory and streams; every step of a solve runs in the library's
CUDA kernels (paper_1406_7808_b200/csrc).  Arrays use shape (n3, n2, n1), x1 fastest,
exactly the layout include/sr_fmg.h documents.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _lib
from ._lib import Desc, Info, Partition, check, lib


@dataclass
class LevelInfo:
    n: Tuple[int, int, int]
    sr: bool
    seg: int
    buffer: int
    nseg: Tuple[int, int, int]
    storage_ext: Tuple[int, int, int]
    pitch: Tuple[int, int, int]
    compute_cells: int
    visits: int


def make_desc(n, M, seg=0, buffer=2, K=0, dtype="f64", h=None, sched=None, alpha=1, nu1=2,
              nu2=2, cheb=None, device=None, use_graph=True, world=1, rank=0,
              pgrid=(1, 1, 1), stencil="7pt", nl_gamma=0.0, dd_min=0, coarse_idle=False) -> Desc:
    if isinstance(n, int):
        n = (n, n, n)
    d = Desc()
    lib.sr_fmg_desc_init(ctypes.byref(d))
    for i in range(3):
        d.n[i] = int(n[i])
        d.pgrid[i] = int(pgrid[i])
    d.M, d.seg, d.buffer, d.sr_levels = int(M), int(seg), int(buffer), int(K)
    if sched is not None:
        if sched[0] == "mbs":  # maximum buffer schedule, J_k = 2^(k-1) J_1
            d.sched_A, d.sched_B = int(sched[1]), -2
        else:
            d.sched_A, d.sched_B = int(sched[0]), int(sched[1])
    d.dtype = {"f64": _lib.SR_F64, "f32": _lib.SR_F32}[dtype]
    d.h = 0.0 if h is None else float(h)
    d.alpha, d.nu1, d.nu2 = int(alpha), int(nu1), int(nu2)
    if cheb is not None:  # default: the stencil's interval (R8 / R28)
        d.cheb_lo, d.cheb_hi = float(cheb[0]), float(cheb[1])
    d.stencil = {"7pt": 7, "27pt": 27}[stencil]
    d.nl_gamma = float(nl_gamma)
    d.device = -1 if device is None else int(device)
    d.use_graph = 1 if use_graph else 0
    d.world, d.rank = int(world), int(rank)
    d.dd_min = int(dd_min)
    d.coarse_idle = 1 if coarse_idle else 0
    return d


def partition(n, M, seg, buffer, K, world, rank, pgrid, sched=None, dd_min=0,
              coarse_idle=False) -> dict:
    """This rank's block of a multi-GPU descriptor (host arithmetic, no GPU)."""
    d = make_desc(n, M, seg, buffer, K, sched=sched, world=world, rank=rank, pgrid=pgrid,
                  dd_min=dd_min, coarse_idle=coarse_idle)
    p = Partition()
    check(lib.sr_fmg_partition(ctypes.byref(d), ctypes.byref(p)))
    return dict(world=p.world, rank=p.rank, coord=tuple(p.coord),
                segs_per_rank=tuple(p.segs_per_rank), block_lo=tuple(p.block_lo),
                block_n=tuple(p.block_n), f_halo=p.f_halo, f_dims=tuple(p.f_dims),
                level_T_lo=tuple(p.level_T_lo), level_T_n=tuple(p.level_T_n),
                level_A=p.level_A)


def nccl_unique_id() -> bytes:
    import torch  # noqa: F401  (load PyTorch's NCCL first: the library reuses it)
    buf = ctypes.create_string_buffer(128)
    check(lib.sr_fmg_nccl_unique_id(buf))
    return buf.raw


class HostStore:
    """Test-only in-process stand-in for NCCL: the ranks' handles (one host thread each, all
    on one GPU) pass their all-gather blocks and halo slabs through host memory."""

    def __init__(self, world):
        self.ptr = ctypes.c_void_p(lib.sr_fmg_host_store_create(int(world)))

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            lib.sr_fmg_host_store_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()


class Solver:
    """One FMG+SR solver instance (a handle of the C ABI).

    Parameters mirror sr_fmg_desc_t: n (n1, n2, n3) or an int for a cube, M, seg (S),
    buffer (J), K (SR levels), dtype "f64"/"f32", h (fine cell size), sched (Eq. 5 A, B),
    F(alpha, nu1, nu2) degrees, Chebyshev interval fractions.  Multi-GPU: world, rank,
    pgrid, nccl_id (or host_store, tests), dd_min (decomposed coarse levels), coarse_idle
    (levels <= A on rank 0 alone instead of redundantly); K = 0 with
    world > 1 is the conventional distributed FMG with fine-level halo exchanges.
    """

    def __init__(self, n, M, seg=0, buffer=2, K=0, dtype="f64", h=None, sched=None,
                 alpha=1, nu1=2, nu2=2, cheb=None, device=None, use_graph=True,
                 world=1, rank=0, pgrid=(1, 1, 1), nccl_id=None, host_store=None,
                 stencil="7pt", nl_gamma=0.0, allocator=None, dd_min=0, coarse_idle=False):
        if isinstance(n, int):
            n = (n, n, n)
        d = make_desc(n, M, seg, buffer, K, dtype, h, sched, alpha, nu1, nu2, cheb, device,
                      use_graph, world, rank, pgrid, stencil, nl_gamma, dd_min, coarse_idle)
        if allocator == "torch":
            # the workspace comes from PyTorch's caching allocator (desc.alloc / desc.free);
            # the callbacks must outlive the handle
            import torch

            def _alloc(nbytes, ctx):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes))
                except RuntimeError:  # out of memory: the library reports it
                    return None

            def _free(ptr, ctx):
                torch.cuda.caching_allocator_delete(ptr)

            self._alloc_cb = _lib.ALLOC_FN(_alloc)
            self._free_cb = _lib.FREE_FN(_free)
            d.alloc, d.free = self._alloc_cb, self._free_cb
        elif allocator is not None:
            raise ValueError("allocator must be None (cudaMalloc) or 'torch'")
        if world > 1 and host_store is None:
            import torch  # noqa: F401  (PyTorch's NCCL is the one the library will reuse)
            if nccl_id is None:
                raise ValueError("world > 1 needs nccl_id (see nccl_unique_id) or host_store")
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        if host_store is not None:
            d.comm = 1
        self._h = ctypes.c_void_p()
        check(lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(self._h)))
        if host_store is not None:
            check(lib.sr_fmg_set_host_store(self._h, host_store.ptr), self._h)
            self._store = host_store
        self.n = tuple(int(v) for v in n)
        self.dtype = dtype
        self.np_dtype = np.float64 if dtype == "f64" else np.float32
        self._info = self._get_info()
        i = self._info
        self.world = i.world
        self.block_lo = tuple(i.block_lo)
        self.block_n = tuple(i.block_n)
        self.f_halo = i.f_halo
        # array shapes (x1 fastest): output block and (haloed) input block
        self.shape = (i.block_n[2], i.block_n[1], i.block_n[0])
        self.f_shape = (i.f_dims[2], i.f_dims[1], i.f_dims[0])

    # -- lifetime ------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib.sr_fmg_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- info ----------------------------------------------------------------------------
    def _get_info(self):
        inf = Info()
        check(lib.sr_fmg_get_info(self._h, ctypes.byref(inf)), self._h)
        return inf

    @property
    def M(self):
        return self._info.M

    @property
    def K(self):
        return self._info.K

    @property
    def T(self):
        return self._info.T

    def level(self, l) -> LevelInfo:
        i = self._info
        return LevelInfo(tuple(i.n_level[l]), bool(i.sr[l]), i.seg_level[l], i.buffer_level[l],
                         tuple(i.nseg[l]), tuple(i.storage_ext[l]), tuple(i.storage_pitch[l]),
                         i.compute_cells[l], i.visits[l])

    @property
    def launches_per_solve(self) -> int:
        """Kernel launches of the last solve (exact once a solve has been enqueued)."""
        return self._get_info().launches_per_solve

    @property
    def alg_bytes_per_solve(self) -> float:
        return self._info.alg_bytes_per_solve

    @property
    def workspace_bytes(self) -> int:
        return self._info.workspace_bytes

    @property
    def exchanges_per_solve(self) -> int:
        """Collective calls of the last solve (all-gathers and halo phases)."""
        return self._get_info().exchanges_per_solve

    @property
    def level_A(self) -> int:
        """Levels <= A are gathered and redundant; A < l <= T are domain-decomposed."""
        return self._info.level_A

    def comm_calls(self):
        """Collective calls per level in the last solve (index = level)."""
        i = self._get_info()
        return [int(i.comm_calls[l]) for l in range(i.M + 1)]

    def dd_levels(self):
        return [l for l in range(self._info.M + 1) if self._info.dd[l]]

    def local_f(self, f_global):
        """This rank's haloed block of a global f (numpy, shape (n3, n2, n1)); cells of the
        halo outside the domain are zero."""
        H = self.f_halo
        lo = self.block_lo
        out = np.zeros(self.f_shape, dtype=f_global.dtype)
        n = self.n
        src = [(max(lo[d] - H, 0), min(lo[d] + self.block_n[d] + H, n[d])) for d in range(3)]
        dst = [(a - (lo[d] - H), b - (lo[d] - H)) for d, (a, b) in enumerate(src)]
        out[dst[2][0]:dst[2][1], dst[1][0]:dst[1][1], dst[0][0]:dst[0][1]] = \
            f_global[src[2][0]:src[2][1], src[1][0]:src[1][1], src[0][0]:src[0][1]]
        return out

    def block_of(self, u_global):
        lo, nb = self.block_lo, self.block_n
        return u_global[lo[2]:lo[2] + nb[2], lo[1]:lo[1] + nb[1], lo[0]:lo[0] + nb[0]]

    # -- solves --------------------------------------------------------------------------
    def _check_tensor(self, t, name, shape):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{name} must be a CUDA torch.Tensor")
        want = torch.float64 if self.dtype == "f64" else torch.float32
        if t.dtype != want or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {want} tensor of shape {shape}")

    def solve(self, f, out=None):
        """u = FMG+SR solve of A u = f.  f, out: CUDA tensors of shape (n3, n2, n1).
        Ordered on torch's current stream; returns `out`."""
        import torch
        self._check_tensor(f, "f", self.f_shape)
        if out is None:
            out = torch.empty(self.shape, dtype=f.dtype, device=f.device)
        self._check_tensor(out, "out", self.shape)
        check(lib.sr_fmg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              self._h)
        check(lib.sr_fmg_solve(self._h, ctypes.c_void_p(f.data_ptr()),
                               ctypes.c_void_p(out.data_ptr())), self._h)
        return out

    def solve_host(self, f, out=None):
        """Same solve from host memory (numpy array or CPU tensor, pinned or not); copies
        happen inside the library call.  Synchronous; returns `out`."""
        import torch
        if isinstance(f, np.ndarray):
            f = torch.from_numpy(np.ascontiguousarray(f, dtype=self.np_dtype))
        if out is None:
            out = torch.empty(self.shape, dtype=f.dtype, pin_memory=f.is_pinned())
        for t, nm, shp in ((f, "f", self.f_shape), (out, "out", self.shape)):
            if t.is_cuda or tuple(t.shape) != tuple(shp) or not t.is_contiguous():
                raise ValueError(f"{nm} must be a contiguous host tensor of shape {shp}")
        check(lib.sr_fmg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              self._h)
        check(lib.sr_fmg_solve_host(self._h, ctypes.c_void_p(f.data_ptr()),
                                    ctypes.c_void_p(out.data_ptr())), self._h)
        return out

    def solve_host_async(self, f, out):
        """Enqueue a host-buffer solve (sr_fmg_solve_host_async): returns at once; the
        host->device copy of the next call, this solve and the device->host copy of the
        previous call overlap.  Neither `f` nor `out` may be touched before synchronize()."""
        import torch
        for t, nm, shp in ((f, "f", self.f_shape), (out, "out", self.shape)):
            if not isinstance(t, torch.Tensor) or t.is_cuda or tuple(t.shape) != tuple(shp) \
                    or not t.is_contiguous() or t.dtype != (torch.float64 if self.dtype == "f64"
                                                            else torch.float32):
                raise ValueError(f"{nm} must be a contiguous host tensor of shape {shp}")
        check(lib.sr_fmg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              self._h)
        check(lib.sr_fmg_solve_host_async(self._h, ctypes.c_void_p(f.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr())), self._h)

    def synchronize(self):
        check(lib.sr_fmg_synchronize(self._h), self._h)

    def vsolve(self, f, out=None, rtol=1e-4, maxit=50):
        """Conventional V-cycle solver (sr_fmg_vsolve; needs K = 0): returns
        (u, cycles, relative residual)."""
        import torch
        want = torch.float64 if self.dtype == "f64" else torch.float32
        self._check_tensor(f, "f", self.f_shape)
        if out is None:
            out = torch.empty(self.shape, dtype=want, device=f.device)
        self._check_tensor(out, "out", self.shape)
        check(lib.sr_fmg_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              self._h)
        cyc, rel = ctypes.c_int32(0), ctypes.c_double(0.0)
        check(lib.sr_fmg_vsolve(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                float(rtol), int(maxit), ctypes.byref(cyc), ctypes.byref(rel)),
              self._h)
        return out, int(cyc.value), float(rel.value)

    # -- test / profiling hooks ----------------------------------------------------------
    def level_storage(self, l, field=0) -> np.ndarray:
        """Internal storage of level l (field 0 = u, 1 = rhs, 2 = t) as an array of shape
        (nsegs, E_z, E_y, pitch_y) view-able per segment."""
        li = self.level(l)
        nsegs = li.nseg[0] * li.nseg[1] * li.nseg[2]
        buf = np.empty(nsegs * li.pitch[2], dtype=self.np_dtype)
        check(lib.sr_fmg_debug_level_io(self._h, l, field, 0, buf.ctypes.data_as(ctypes.c_void_p)),
              self._h)
        return buf

    def set_level_storage(self, l, field, arr: np.ndarray):
        arr = np.ascontiguousarray(arr, dtype=self.np_dtype)
        check(lib.sr_fmg_debug_level_io(self._h, l, field, 1, arr.ctypes.data_as(ctypes.c_void_p)),
              self._h)

    def debug_op(self, op, level, deg=0, f=None):
        ptr = ctypes.c_void_p(f.data_ptr()) if f is not None else None
        check(lib.sr_fmg_debug_op(self._h, op, level, deg, ptr), self._h)

    def profile_select(self, kernel_class: int, level: int):
        check(lib.sr_fmg_profile_select(self._h, kernel_class, level), self._h)

    def profile_ring(self, nslots: int):
        check(lib.sr_fmg_profile_ring(self._h, int(nslots)), self._h)

    def profile_read_slot(self, slot: int):
        ms, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        check(lib.sr_fmg_profile_read_slot(self._h, int(slot), ctypes.byref(ms), ctypes.byref(by),
                                           ctypes.byref(n)), self._h)
        return ms.value, by.value, n.value

    def profile_read(self):
        ms, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
        check(lib.sr_fmg_profile_read(self._h, ctypes.byref(ms), ctypes.byref(by),
                                      ctypes.byref(n)), self._h)
        return ms.value, by.value, n.value
