// Coarse-level executor: the small conventional levels (l <= T, Omega_l as one segment with a
// one-cell ghost ring) run as a recorded list of operations inside ONE launch
// of a thread-block cluster, one cluster barrier (release/acquire at cluster scope) between
// consecutive operations.  Same arithmetic as the single-purpose kernels of kernels.cu:
//
//   CHEB      out = cur + c_mom (cur - prev) + c_res (b - A cur) on Omega     (R8)
//   RESTRICT  u_c = avg8(u_f), R_c = avg8(b - A u_f) on Omega_c                (R9, Eq. 4)
//   TAU       t = u, rhs = R + A u on Omega (F = V = Omega on these levels)    (Eq. 4)
//   PROLONG   u_f = P(w) or u_f += P(w - t), trilinear, reflected ghosts      (R10, R3)
//   COARSEST  u_0 = A_0^{-1} b_0                                              (R7)
//   PYRAMID   f_c = avg8(f_f) on dense arrays                                 (R6)
//
// A = -Lap_h with 7 points; a neighbour outside Omega is the reflected ghost -u_i (R3).
// A level may be a rank's BLOCK of a domain-decomposed conventional level (multi-GPU,
// DESIGN.md §8): the operations run over the block's cells (L.S, global offset L.so*L.S),
// read neighbours in other ranks' blocks from the ghost ring (filled by the halo exchange
// before the operation) and test the domain boundary in global coordinates -- with one
// block (S = N, so = 0) this is exactly the single-GPU operation, cell for cell.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "coarse.cuh"

namespace srfmg {

namespace {

constexpr int kCluster = 16;  // non-portable cluster size (B200 allows 16)
constexpr int kThreadsC = 512;

template <class T>
__device__ __forceinline__ long long soff(const Lvl& L, int x, int y, int z) {
  return (long long)(z + 1) * L.pz + (long long)(y + 1) * L.py + (x + 1);
}

// global index of the block's first cell in dimension d (0 with one block)
__device__ __forceinline__ int goff(const Lvl& L, int d) { return L.so[d] * L.S[d]; }

// rhs at local cell (x, y, z) / global cell (gx, gy, gz): dense views (f pyramid, user f)
// are indexed globally (virtual origin), segment-storage views locally
template <class T>
__device__ __forceinline__ T rhs_at(const View<T>& v, int x, int y, int z, int gx, int gy,
                                    int gz) {
  if (v.global) return v.p[(long long)gz * v.sz + (long long)gy * v.sy + gx];
  return v.p[(long long)(z + 1) * v.sz + (long long)(y + 1) * v.sy + (x + 1)];
}

// (A u) at global cell (x, y, z) of a conventional level (storage offset o); neighbour
// order z-, z+, y-, y+, x-, x+
template <class T>
__device__ __forceinline__ T apply_A(const Lvl& L, const T* __restrict__ u, long long o, int x,
                                     int y, int z) {
  const T c = u[o];
  T s = T(0);
  s += (z > 0) ? u[o - L.pz] : -c;
  s += (z < L.N[2] - 1) ? u[o + L.pz] : -c;
  s += (y > 0) ? u[o - L.py] : -c;
  s += (y < L.N[1] - 1) ? u[o + L.py] : -c;
  s += (x > 0) ? u[o - 1] : -c;
  s += (x < L.N[0] - 1) ? u[o + 1] : -c;
  return (T(6) * c - s) * T(L.inv_h2) + T(L.nlg) * c * c * c;
}

// Index math of the operations: every executor operation is a short dependent chain per
// thread, so the divisions by run-time extents (~15 instructions each) are a visible part of
// an operation's latency.  Extents that are powers of two (all of the BASELINE grids) take
// shifts and masks instead; the mapping is the same, so the results are too.
__device__ __forceinline__ bool pow2(int v) { return (v & (v - 1)) == 0; }
__device__ __forceinline__ int lg2(int v) { return __ffs(v) - 1; }  // v a power of two

__device__ __forceinline__ void cell_of(int i, const int n[3], int& x, int& y, int& z) {
  if (pow2(n[0]) && pow2(n[1])) {
    const int l0 = lg2(n[0]), l1 = lg2(n[1]);
    x = i & (n[0] - 1);
    y = (i >> l0) & (n[1] - 1);
    z = i >> (l0 + l1);
    return;
  }
  x = i % n[0];
  const int r = i / n[0];
  y = r % n[1];
  z = r / n[1];
}

// Thread layout of every operation: thread t owns the (x, y) column t % ncol and the z
// chunk t / ncol of ceil(nz / nchunk) planes (nchunk = max(1, nth / ncol)); the column's
// z-neighbours stay in registers and all loads of a chunk are issued before the arithmetic.
struct ColMap {
  int x, y, z0, z1;
  bool ok;
};
__device__ __forceinline__ ColMap col_map(int nx, int ny, int nz, int tid, int nth) {
  ColMap m;
  const int ncol = nx * ny;
  if (pow2(nx) && pow2(ny) && pow2(nz) && pow2(nth)) {  // (ncol, nch, per: powers of two)
    const int lx = lg2(nx), lc = lx + lg2(ny);
    const int lch = max(0, min(lg2(nz), lg2(nth) - lc));
    const int col = tid & (ncol - 1), ch = tid >> lc;
    m.x = col & (nx - 1);
    m.y = col >> lx;
    m.z0 = ch << (lg2(nz) - lch);
    m.z1 = min(nz, m.z0 + (nz >> lch));
    m.ok = tid < (ncol << lch) && m.z0 < m.z1;
    return m;
  }
  const int nch = max(1, min(nz, nth / ncol));
  const int per = (nz + nch - 1) / nch;
  const int col = tid % ncol, ch = tid / ncol;
  m.x = col % nx;
  m.y = col / nx;
  m.z0 = ch * per;
  m.z1 = min(nz, m.z0 + per);
  m.ok = tid < ncol * nch && m.z0 < m.z1;
  return m;
}
constexpr int kZC = 4;  // planes per register batch (longer chunks loop; 64 registers)

// CHEB (c_mom == 0 and prev == null: first step) and TAU share the column sweep:
// storage ghosts are zero, so the reflected ghost -u_i is +1 on the diagonal (R3)
template <class T, bool TAU>
__device__ void op_column(const Lvl& L, const COp<T>& o, int tid, int nth) {
  const ColMap m = col_map(L.S[0], L.S[1], L.S[2], tid, nth);
  if (!m.ok) return;
  const T cm = T(o.c0), cr = T(o.c1);
  const int gx = m.x + goff(L, 0), gy = m.y + goff(L, 1), gz0 = goff(L, 2);
  const bool xm = gx > 0, xp = gx < L.N[0] - 1, ym = gy > 0, yp = gy < L.N[1] - 1;
  const T dxy = T(6 + !xm + !xp + !ym + !yp);
  for (int zb = m.z0; zb < m.z1; zb += kZC) {
    const int ze = min(m.z1, zb + kZC);
    T q[kZC + 2], nb[kZC], bv[kZC], pv[kZC];
    const long long c0 = soff<T>(L, m.x, m.y, zb);
#pragma unroll
    for (int k = 0; k < kZC + 2; ++k)  // planes zb-1 .. zb+kZC (ghost planes: zero at the
      q[k] = (zb - 1 + k <= ze) ? o.a[c0 + (long long)(k - 1) * L.pz] : T(0);  // domain face)
#pragma unroll
    for (int k = 0; k < kZC; ++k) {
      if (zb + k >= ze) break;
      const long long off = c0 + (long long)k * L.pz;
      nb[k] = ((ym ? o.a[off - L.py] : T(0)) + (yp ? o.a[off + L.py] : T(0))) +
              ((xm ? o.a[off - 1] : T(0)) + (xp ? o.a[off + 1] : T(0)));
      if constexpr (TAU) {
        bv[k] = o.c[off];
      } else {
        bv[k] = rhs_at(o.v, m.x, m.y, zb + k, gx, gy, gz0 + zb + k);
        pv[k] = o.b ? o.b[off] : T(0);
      }
    }
#pragma unroll
    for (int k = 0; k < kZC; ++k) {
      const int z = zb + k;
      if (z >= ze) break;
      const T d = dxy + T((gz0 + z == 0 ? 1 : 0) + (gz0 + z == L.N[2] - 1 ? 1 : 0));
      const T c = q[k + 1];
      const T Au = (d * c - ((q[k] + q[k + 2]) + nb[k])) * T(L.inv_h2) + T(L.nlg) * c * c * c;
      const long long off = c0 + (long long)k * L.pz;
      if constexpr (TAU) {
        o.d[off] = c;           // t = u
        o.c[off] = bv[k] + Au;  // rhs = R + A u
      } else {
        const T r = bv[k] - Au;
        o.c[off] = o.b ? c + cm * (c - pv[k]) + cr * r : c + cr * r;
      }
    }
  }
}

// RESTRICT: eight lanes per coarse cell, one fine child each (residual of the child with all
// its loads in flight at once), reduced with three butterfly shuffles
// (the coarse cells are those of the fine block: local X of the fine block's coarsening,
// global X + goff(Lf)/2, written at their local index in the coarse array -- a block of a
// decomposed level, or the rank's part of a global one)
template <class T>
__device__ void op_restrict(const Lvl& Lf, const Lvl& Lc, const COp<T>& o, int tid, int nth) {
  const int nc[3] = {Lf.S[0] / 2, Lf.S[1] / 2, Lf.S[2] / 2};
  const int n = nc[0] * nc[1] * nc[2];
  const int ch = tid & 7;
  const int dx = ch & 1, dy = (ch >> 1) & 1, dz = ch >> 2;
  const int fo[3] = {goff(Lf, 0), goff(Lf, 1), goff(Lf, 2)};
  // whole warps run the loop (the shuffles need all 32 lanes), so the bound is 8 n rounded
  // up to a multiple of 32; lanes past the last coarse cell compute a copy of it
  const int nl = (8 * n + 31) & ~31;
  for (int base = tid - ch; base < nl; base += nth) {  // warp-uniform trip count
    const int c = base >> 3;
    const bool ok = c < n;
    int X, Y, Z;
    cell_of(ok ? c : n - 1, nc, X, Y, Z);
    const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
    const long long off = soff<T>(Lf, x, y, z);
    T su = o.a[off];
    T sr = rhs_at(o.v, x, y, z, x + fo[0], y + fo[1], z + fo[2]) -
           apply_A(Lf, o.a, off, x + fo[0], y + fo[1], z + fo[2]);
#pragma unroll
    for (int m = 1; m < 8; m <<= 1) {
      su += __shfl_xor_sync(0xffffffffu, su, m);
      sr += __shfl_xor_sync(0xffffffffu, sr, m);
    }
    if (ok && ch == 0) {
      const long long co = soff<T>(Lc, X + fo[0] / 2 - goff(Lc, 0), Y + fo[1] / 2 - goff(Lc, 1),
                                   Z + fo[2] / 2 - goff(Lc, 2));
      o.c[co] = su * T(0.125);
      o.d[co] = sr * T(0.125);
    }
  }
}

template <class T>
__device__ void op_prolong(const Lvl& Lf, const Lvl& Lc, const COp<T>& o, int tid, int nth) {
  const ColMap m = col_map(Lf.S[0], Lf.S[1], Lf.S[2], tid, nth);
  if (!m.ok) return;
  const T W0 = T(0.75), W1 = T(0.25);
  const int g[2] = {m.x + goff(Lf, 0), m.y + goff(Lf, 1)};
  const int co[3] = {goff(Lc, 0), goff(Lc, 1), goff(Lc, 2)};
  int P[2], Q[2];
  T sg[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    P[d] = g[d] >> 1;
    Q[d] = P[d] + ((g[d] & 1) ? 1 : -1);
    sg[d] = T(1);
    if (Q[d] < 0) { Q[d] = 0; sg[d] = T(-1); }
    if (Q[d] >= Lc.N[d]) { Q[d] = Lc.N[d] - 1; sg[d] = T(-1); }
    P[d] -= co[d];  // local coarse index (-1 or S_c: the ghost ring of a block)
    Q[d] -= co[d];
  }
  // xy-interpolant of coarse plane cz (global; weights 3/4 parent, 1/4 neighbour, signed
  // ghosts)
  auto ixy = [&](int cz) {
    T sgz = T(1);
    if (cz < 0) { cz = 0; sgz = T(-1); }
    if (cz >= Lc.N[2]) { cz = Lc.N[2] - 1; sgz = T(-1); }
    cz -= co[2];
    T py[2];
#pragma unroll
    for (int ky = 0; ky < 2; ++ky) {
      const int cy = ky ? Q[1] : P[1];
      const long long a0 = soff<T>(Lc, P[0], cy, cz), a1 = soff<T>(Lc, Q[0], cy, cz);
      const T v0 = o.flag ? o.a[a0] - o.b[a0] : o.a[a0];
      const T v1 = o.flag ? o.a[a1] - o.b[a1] : o.a[a1];
      py[ky] = W0 * v0 + (W1 * sg[0]) * v1;
    }
    return sgz * (W0 * py[0] + (W1 * sg[1]) * py[1]);
  };
  for (int z = m.z0; z < m.z1; ++z) {
    const int gz = z + goff(Lf, 2);
    const int Pz = gz >> 1, Qz = Pz + ((gz & 1) ? 1 : -1);
    const T acc = W0 * ixy(Pz) + W1 * ixy(Qz);
    const long long off = soff<T>(Lf, m.x, m.y, z);
    o.c[off] = o.flag ? o.c[off] + acc : acc;
  }
}

template <class T>
__device__ void op_pyramid(const Lvl& Lf, const COp<T>& o, int tid, int nth) {
  const int nfx = Lf.N[0], nfy = Lf.N[1];
  const int nc[3] = {Lf.N[0] / 2, Lf.N[1] / 2, Lf.N[2] / 2};
  const ColMap m = col_map(nc[0], nc[1], nc[2], tid, nth);
  if (!m.ok) return;
  for (int z = m.z0; z < m.z1; ++z) {
    T s = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          s += o.a[((long long)(2 * z + dz) * nfy + (2 * m.y + dy)) * nfx + (2 * m.x + dx)];
    o.c[((long long)z * nc[1] + m.y) * nc[0] + m.x] = s * T(0.125);
  }
}

template <class T>
__global__ void __launch_bounds__(kThreadsC, 1)
    k_coarse_exec(const __grid_constant__ COpList<T> ol) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ T bs[1024];
  __shared__ T us[1024];
  // the operation list and the level table are read from shared memory: dynamically
  // indexed kernel-parameter reads go through the constant cache and miss (~1 us per op)
  __shared__ COp<T> sop[kCoarseMaxOps];
  __shared__ Lvl sL[kCoarseMaxLevels];
  {
    const int* src = reinterpret_cast<const int*>(ol.op);
    int* dst = reinterpret_cast<int*>(sop);
    const int nw = (int)(ol.n * sizeof(COp<T>) / sizeof(int));
    for (int k = threadIdx.x; k < nw; k += blockDim.x) dst[k] = src[k];
    const int* ls = reinterpret_cast<const int*>(ol.L);
    int* ld = reinterpret_cast<int*>(sL);
    for (int k = threadIdx.x; k < (int)(sizeof(sL) / sizeof(int)); k += blockDim.x) ld[k] = ls[k];
  }
  __syncthreads();
  const int rank = (int)cl.block_rank();
  if (ol.prof && rank == 0 && threadIdx.x == 0) {
    // SM cycle counter (CTA 0 stays on one SM): %globaltimer ticks in ~1 us steps
    const unsigned long long t = (unsigned long long)clock64();
    ol.prof[0] = t;
  }
  for (int i = 0; i < ol.n; ++i) {
    const COp<T>& o = sop[i];
    // an operation on a tiny level runs on CTA 0 alone, and a run of them needs only CTA
    // barriers; the cluster barrier follows the last of the run
    const bool tiny = o.tiny != 0;
    if (tiny && rank != 0) {
      while (i + 1 < ol.n && sop[i + 1].tiny) ++i;
      cl.sync();
      continue;
    }
    const int tid = tiny ? (int)threadIdx.x : rank * kThreadsC + (int)threadIdx.x;
    const int nth = tiny ? kThreadsC : kCluster * kThreadsC;
    switch (o.code) {
      case kCopCheb: op_column<T, false>(sL[o.lf], o, tid, nth); break;
      case kCopRestrict: op_restrict(sL[o.lf], sL[o.lc], o, tid, nth); break;
      case kCopTau: op_column<T, true>(sL[o.lf], o, tid, nth); break;
      case kCopProlong: op_prolong(sL[o.lf], sL[o.lc], o, tid, nth); break;
      case kCopPyramid: op_pyramid(sL[o.lf], o, tid, nth); break;
      case kCopCoarsest:
        if (rank == 0) {  // one CTA: n0 <= 1024 (create-time check)
          const Lvl& L = sL[o.lf];
          const int n0 = L.N[0] * L.N[1] * L.N[2];
          for (int j = threadIdx.x; j < n0; j += kThreadsC) {
            int x, y, z;
            cell_of(j, L.N, x, y, z);
            bs[j] = rhs_at(o.v, x, y, z, x, y, z);
          }
          __syncthreads();
          // nonlinear (R29): Picard sweeps u <- A_lin^-1 (b - nlg u^3), as k_coarsest
          const int sweeps = L.nlg != 0.0 ? 41 : 1;
          for (int it = 0; it < sweeps; ++it) {
            for (int r = threadIdx.x; r < n0; r += kThreadsC) {
              T acc = T(0);
              for (int j = 0; j < n0; ++j) acc += o.a[(long long)r * n0 + j] * bs[j];
              us[r] = acc;
            }
            __syncthreads();
            if (it + 1 < sweeps) {
              for (int j = threadIdx.x; j < n0; j += kThreadsC) {
                int x, y, z;
                cell_of(j, L.N, x, y, z);
                bs[j] = rhs_at(o.v, x, y, z, x, y, z) - T(L.nlg) * us[j] * us[j] * us[j];
              }
              __syncthreads();
            }
          }
          for (int r = threadIdx.x; r < n0; r += kThreadsC) {
            int x, y, z;
            cell_of(r, L.N, x, y, z);
            o.c[soff<T>(L, x, y, z)] = us[r];
          }
        }
        break;
      default: break;
    }
    if (tiny && i + 1 < ol.n && sop[i + 1].tiny)
      __syncthreads();  // CTA 0 alone: block-scope visibility suffices
    else
      cl.sync();  // the operation's results are visible to every CTA of the cluster
    if (ol.prof && rank == 0 && threadIdx.x == 0) {
      const unsigned long long t = (unsigned long long)clock64();
      ol.prof[i + 1] = t;
    }
  }
}

}  // namespace

bool coarse_level_ok(const Lvl& L) {
  return L.nsegs == 1 && L.J == 0 && (long long)L.N[0] * L.N[1] * L.N[2] <= kCoarseMaxCells;
}

bool coarse_level_tiny(const Lvl& L) {
  static const long long lim = [] {  // cells up to which CTA 0 alone runs a level's ops
    const char* e = std::getenv("SR_FMG_CEXEC_TINY");
    return e ? std::atoll(e) : 512LL;
  }();
  return coarse_level_ok(L) && (long long)L.N[0] * L.N[1] * L.N[2] <= lim;
}

template <class T>
void launch_coarse_exec(const COpList<T>& ops, cudaStream_t st) {
  if (ops.n <= 0) return;
  // (per launch: the attribute is per device, and a process may drive several)
  cudaFuncSetAttribute(k_coarse_exec<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kCluster);
  cfg.blockDim = dim3(kThreadsC);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_coarse_exec<T>, ops);
}

template void launch_coarse_exec<double>(const COpList<double>&, cudaStream_t);
template void launch_coarse_exec<float>(const COpList<float>&, cudaStream_t);

}  // namespace srfmg
