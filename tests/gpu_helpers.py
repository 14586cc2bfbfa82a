"""Helpers mapping the library's internal segment storage to oracle Fields (tests only)."""
import numpy as np

from oracle import Box, Field


def seg_coords(li, s):
    nx, ny, _ = li.nseg
    return (s % nx, (s // nx) % ny, s // (nx * ny))  # (px, py, pz)


def storage_box(li, s):
    """Global storage box of segment s in ARRAY order (z, y, x) as the oracle uses."""
    p = seg_coords(li, s)
    lo_xyz = [p[d] * (li.seg if li.sr else li.n[d]) - (li.buffer + 1) for d in range(3)]
    E = li.storage_ext
    return Box((lo_xyz[2], lo_xyz[1], lo_xyz[0]),
               (lo_xyz[2] + E[2], lo_xyz[1] + E[1], lo_xyz[0] + E[0]))


def seg_array(buf, li, s):
    """View (E_z, E_y, E_x) of segment s inside a flat level buffer."""
    py, pz, ss = li.pitch
    E = li.storage_ext
    a = buf[s * ss: s * ss + pz * E[2]].reshape(E[2], E[1], py)
    return a[:, :, :E[0]]


def to_fields(buf, li):
    nsegs = li.nseg[0] * li.nseg[1] * li.nseg[2]
    return [Field(storage_box(li, s), array=seg_array(buf, li, s).astype(np.float64))
            for s in range(nsegs)]


def from_fields(fields, li, dtype):
    py, pz, ss = li.pitch
    nsegs = len(fields)
    buf = np.zeros(nsegs * ss, dtype=dtype)
    for s, fld in enumerate(fields):
        seg_array(buf, li, s)[...] = fld.a
    return buf


def oracle_seg_index(li, s):
    """Oracle segment tuple (array order) of library segment s."""
    px, py, pz = seg_coords(li, s)
    return (pz, py, px)


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def zero_outside(buf, li):
    """Zero every storage cell outside Omega_l (the library's invariant: storage cells
    outside the domain are zero; kernels never write them)."""
    nsegs = li.nseg[0] * li.nseg[1] * li.nseg[2]
    for s in range(nsegs):
        box = storage_box(li, s)
        a = seg_array(buf, li, s)
        for d, ax in ((0, 2), (1, 1), (2, 0)):   # li.n is (x, y, z); array axes (z, y, x)
            g = np.arange(box.lo[ax], box.hi[ax])
            bad = (g < 0) | (g >= li.n[d])
            sl = [slice(None)] * 3
            sl[ax] = bad
            a[tuple(sl)] = 0.0
    return buf
