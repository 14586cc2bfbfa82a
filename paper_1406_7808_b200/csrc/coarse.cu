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
#include <cooperative_groups.h>

#include <algorithm>

#include "coarse.cuh"

namespace srfmg {

namespace {

constexpr int kCluster = 8;
constexpr int kThreadsC = 1024;

template <class T>
__device__ __forceinline__ long long soff(const Lvl& L, int x, int y, int z) {
  return (long long)(z + 1) * L.pz + (long long)(y + 1) * L.py + (x + 1);
}

template <class T>
__device__ __forceinline__ T rhs_at(const View<T>& v, int x, int y, int z) {
  if (v.global) return v.p[(long long)z * v.sz + (long long)y * v.sy + x];
  return v.p[(long long)(z + 1) * v.sz + (long long)(y + 1) * v.sy + (x + 1)];
}

// (A u) at cell (x, y, z) of a conventional level; neighbour order z-, z+, y-, y+, x-, x+
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
  return (T(6) * c - s) * T(L.inv_h2);
}

__device__ __forceinline__ void cell_of(long long i, const int n[3], int& x, int& y, int& z) {
  x = (int)(i % n[0]);
  const long long r = i / n[0];
  y = (int)(r % n[1]);
  z = (int)(r / n[1]);
}

template <class T>
__device__ void op_cheb(const Lvl& L, const COp<T>& o, int tid, int nth) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  const T cm = T(o.c0), cr = T(o.c1);
  for (long long i = tid; i < n; i += nth) {
    int x, y, z;
    cell_of(i, L.N, x, y, z);
    const long long off = soff<T>(L, x, y, z);
    const T c = o.a[off];
    const T r = rhs_at(o.v, x, y, z) - apply_A(L, o.a, off, x, y, z);
    T v = c + cr * r;
    if (o.b) v = c + cm * (c - o.b[off]) + cr * r;
    o.c[off] = v;
  }
}

template <class T>
__device__ void op_restrict(const Lvl& Lf, const Lvl& Lc, const COp<T>& o, int tid, int nth) {
  const long long n = (long long)Lc.N[0] * Lc.N[1] * Lc.N[2];
  for (long long i = tid; i < n; i += nth) {
    int X, Y, Z;
    cell_of(i, Lc.N, X, Y, Z);
    T su = T(0), sr = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
          const long long off = soff<T>(Lf, x, y, z);
          su += o.a[off];
          sr += rhs_at(o.v, x, y, z) - apply_A(Lf, o.a, off, x, y, z);
        }
    const long long co = soff<T>(Lc, X, Y, Z);
    o.c[co] = su * T(0.125);
    o.d[co] = sr * T(0.125);
  }
}

template <class T>
__device__ void op_tau(const Lvl& L, const COp<T>& o, int tid, int nth) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  for (long long i = tid; i < n; i += nth) {
    int x, y, z;
    cell_of(i, L.N, x, y, z);
    const long long off = soff<T>(L, x, y, z);
    o.d[off] = o.a[off];
    o.c[off] = o.c[off] + apply_A(L, o.a, off, x, y, z);
  }
}

template <class T>
__device__ void op_prolong(const Lvl& Lf, const Lvl& Lc, const COp<T>& o, int tid, int nth) {
  const long long n = (long long)Lf.N[0] * Lf.N[1] * Lf.N[2];
  const T W0 = T(0.75), W1 = T(0.25);
  for (long long i = tid; i < n; i += nth) {
    int x, y, z;
    cell_of(i, Lf.N, x, y, z);
    const int g[3] = {x, y, z};
    int P[3], Q[3];
    T sg[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      P[d] = g[d] >> 1;
      Q[d] = P[d] + ((g[d] & 1) ? 1 : -1);
      sg[d] = T(1);
      if (Q[d] < 0) { Q[d] = 0; sg[d] = T(-1); }
      if (Q[d] >= Lc.N[d]) { Q[d] = Lc.N[d] - 1; sg[d] = T(-1); }
    }
    auto cv = [&](int cx, int cy, int cz) {
      const long long co = soff<T>(Lc, cx, cy, cz);
      return o.flag ? o.a[co] - o.b[co] : o.a[co];
    };
    // separable: x, then y, then z (weights 3/4 parent, 1/4 neighbour, signed ghosts)
    T pz[2];
#pragma unroll
    for (int kz = 0; kz < 2; ++kz) {
      const int cz = kz ? Q[2] : P[2];
      T py[2];
#pragma unroll
      for (int ky = 0; ky < 2; ++ky) {
        const int cy = ky ? Q[1] : P[1];
        py[ky] = W0 * cv(P[0], cy, cz) + (W1 * sg[0]) * cv(Q[0], cy, cz);
      }
      pz[kz] = W0 * py[0] + (W1 * sg[1]) * py[1];
    }
    const T acc = W0 * pz[0] + (W1 * sg[2]) * pz[1];
    const long long off = soff<T>(Lf, x, y, z);
    o.c[off] = o.flag ? o.c[off] + acc : acc;
  }
}

template <class T>
__device__ void op_pyramid(const Lvl& Lf, const COp<T>& o, int tid, int nth) {
  const int nfx = Lf.N[0], nfy = Lf.N[1];
  const int nc[3] = {Lf.N[0] / 2, Lf.N[1] / 2, Lf.N[2] / 2};
  const long long n = (long long)nc[0] * nc[1] * nc[2];
  for (long long i = tid; i < n; i += nth) {
    int x, y, z;
    cell_of(i, nc, x, y, z);
    T s = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          s += o.a[((long long)(2 * z + dz) * nfy + (2 * y + dy)) * nfx + (2 * x + dx)];
    o.c[i] = s * T(0.125);
  }
}

template <class T>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreadsC, 1)
    k_coarse_exec(const __grid_constant__ COpList<T> ol) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ T bs[1024];
  const int rank = (int)cl.block_rank();
  const int tid = rank * kThreadsC + (int)threadIdx.x;
  const int nth = kCluster * kThreadsC;
  for (int i = 0; i < ol.n; ++i) {
    const COp<T>& o = ol.op[i];
    switch (o.code) {
      case kCopCheb: op_cheb(ol.L[o.lf], o, tid, nth); break;
      case kCopRestrict: op_restrict(ol.L[o.lf], ol.L[o.lc], o, tid, nth); break;
      case kCopTau: op_tau(ol.L[o.lf], o, tid, nth); break;
      case kCopProlong: op_prolong(ol.L[o.lf], ol.L[o.lc], o, tid, nth); break;
      case kCopPyramid: op_pyramid(ol.L[o.lf], o, tid, nth); break;
      case kCopCoarsest:
        if (rank == 0) {  // one CTA: n0 <= 1024 (create-time check)
          const Lvl& L = ol.L[o.lf];
          const int n0 = L.N[0] * L.N[1] * L.N[2];
          for (int j = threadIdx.x; j < n0; j += kThreadsC) {
            int x, y, z;
            cell_of(j, L.N, x, y, z);
            bs[j] = rhs_at(o.v, x, y, z);
          }
          __syncthreads();
          for (int r = threadIdx.x; r < n0; r += kThreadsC) {
            T acc = T(0);
            for (int j = 0; j < n0; ++j) acc += o.a[(long long)r * n0 + j] * bs[j];
            int x, y, z;
            cell_of(r, L.N, x, y, z);
            o.c[soff<T>(L, x, y, z)] = acc;
          }
        }
        break;
      default: break;
    }
    cl.sync();  // the operation's results are visible to every CTA of the cluster
  }
}

}  // namespace

bool coarse_level_ok(const Lvl& L) {
  return L.nsegs == 1 && L.J == 0 && (long long)L.N[0] * L.N[1] * L.N[2] <= kCoarseMaxCells;
}

template <class T>
void launch_coarse_exec(const COpList<T>& ops, cudaStream_t st) {
  if (ops.n <= 0) return;
  k_coarse_exec<T><<<kCluster, kThreadsC, 0, st>>>(ops);
}

template void launch_coarse_exec<double>(const COpList<double>&, cudaStream_t);
template void launch_coarse_exec<float>(const COpList<float>&, cudaStream_t);

}  // namespace srfmg
