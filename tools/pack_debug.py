"""Debug (GPU box): packed vs scalar fp32 degree-2 pass, one launch on one level (debug_op),
random storage, against a float64 numpy model of the kernels' arithmetic on segment 0."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1406_7808_b200 import Solver  # noqa: E402

os.environ["SR_FMG_FORCE_FUSED"] = "1"
n, M, seg, K, l = (128, 128, 128), 6, 64, 2, 5
s = Solver(n, M, seg=seg, buffer=2, K=K, dtype="f32")
li = s.level(l)
E, P = li.storage_ext, li.pitch
rng = np.random.default_rng(1)
nseg = li.nseg[0] * li.nseg[1] * li.nseg[2]
u = rng.standard_normal(nseg * P[2]).astype(np.float32)
b = rng.standard_normal(nseg * P[2]).astype(np.float32)
out = {}
for pk in ("1", "0"):
    os.environ["SR_FMG_CHEB_PACK"] = pk
    s.set_level_storage(l, 0, u)
    s.set_level_storage(l, 1, b)
    s.debug_op(0, l, 2)
    out[pk] = s.level_storage(l, 0).copy()
# model: segment 0 (at the domain corner), J = 2, S = 32, N = 64
N, S, J = 64, 32, 2
h = 1.0 / N
lam = 12 / h**2
lo, hi = lam / 6, lam
theta, delta = (hi + lo) / 2, (hi - lo) / 2
sig = theta / delta
r0 = 1 / sig
r1 = 1 / (2 * sig - r0)
c0, cm, cr = 1 / theta, r1 * r0, 2 * r1 / delta


def seg0(a):
    return a[:P[2]][:E[2] * P[1]].reshape(E[2], E[1], P[0]).astype(np.float64)


U, B = seg0(u), seg0(b)
o = -(J + 1)
g = np.arange(E[0]) + o
inside = (g >= 0) & (g < N)
Cx = inside & (np.arange(E[0]) >= 1) & (np.arange(E[0]) <= E[0] - 2)
C = Cx[:, None, None] & Cx[None, :, None] & Cx[None, None, :]
Cz = np.zeros((E[2], E[1], P[0]), bool)
Cz[:, :, :E[0]] = C


def sweep(v, prev, coef_first):
    d = np.zeros_like(v)
    sm = np.zeros_like(v)
    for ax in range(3):
        for sh in (-1, 1):
            nb = np.roll(v, sh, axis=ax)
            sm += nb
    # diagonal: 6 + outside neighbours (storage ghosts assumed zero)
    gg = [g[:, None, None], g[None, :, None], g[None, None, :]]
    cnt = 6 + sum(((x == 0).astype(int) + (x == N - 1).astype(int)) for x in gg)
    cnt = np.broadcast_to(cnt, C.shape)
    dcnt = np.zeros_like(v)
    dcnt[:, :, :E[0]] = cnt
    r = B - (dcnt * v - sm) / h**2
    w = v.copy()
    if coef_first:
        w[Cz] = (v + c0 * r)[Cz]
    else:
        w[Cz] = (v + cm * (v - prev) + cr * r)[Cz]
    return w


u1 = sweep(U, None, True)
u2 = sweep(u1, U, False)
for pk in ("1", "0"):
    got = seg0(out[pk])
    err = np.abs(got - u2)[Cz]
    print("pack", pk, "max err vs model on C", float(err.max()), "rel", float(err.max() / np.abs(u2[Cz]).max()))
    bad = np.argwhere((np.abs(got - u2) > 1e-3 * np.abs(u2).max()) & Cz)
    print("  bad cells", len(bad), bad[:8].tolist())
got = seg0(out["1"])
for name, ref in [("u0", U), ("u1", u1), ("u2", u2)]:
    print(name, "max |packed - ref| on C", float(np.abs(got - ref)[Cz].max()))
# lane swap: packed at x vs model at x^1
sw = got.copy()
sw[:, :, 0::2], sw[:, :, 1::2] = got[:, :, 1::2], got[:, :, 0::2]
print("lane-swapped vs u2", float(np.abs(sw - u2)[Cz].max()))
print("sample z=3 y=3 x=3..8 packed", got[3, 3, 3:9], "model u2", u2[3, 3, 3:9], "u1", u1[3, 3, 3:9])
