// Unfused reference-layout kernels of the SR-FMG schedule, sm_100a, fp64 and fp32.
//
// One thread per cell of a segment's storage (or target) box; blockIdx.y = segment.
// These are the straightforward kernels the fused passes (fused.cu) are checked against;
// they also run every level the fused passes do not cover.  Each kernel cites the step of
// the paper it implements (PAPER.md line numbers; readings R<n> in DESIGN.md §3).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace srfmg {

const char* const kKernelNames[] = {"k_cheb_step", "k_restrict", "k_tau",     "k_prolong",
                                    "k_coarsest",  "k_pyramid",  "k_gather",  "k_cheb2",
                                    "k_pass_entry", "k_pass_down", "k_pass_up", "k_coarse"};
const int kNumKernelNames = 12;

namespace {

constexpr int kThreads = 256;

// GLOBAL segment coordinates of local segment s (this rank's block starts at L.so)
__device__ __forceinline__ void seg_coords(const Lvl& L, int s, int p[3]) {
  p[0] = s % L.ns[0] + L.so[0];
  const int t = s / L.ns[0];
  p[1] = t % L.ns[1] + L.so[1];
  p[2] = t / L.ns[1] + L.so[2];
}

// storage origin (global index of local cell 0) of a segment: p*S - (J+1)
__device__ __forceinline__ void seg_origin(const Lvl& L, const int p[3], int o[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) o[d] = p[d] * L.S[d] - (L.J + 1);
}

__device__ __forceinline__ long long loc_off(const Lvl& L, int s, int ax, int ay, int az) {
  return (long long)s * L.ss + (long long)az * L.pz + (long long)ay * L.py + ax;
}

template <class T>
__device__ __forceinline__ T view_at(const View<T>& v, int s, const int a[3], const int g[3]) {
  if (v.global) return v.p[(long long)g[2] * v.sz + (long long)g[1] * v.sy + g[0]];
  return v.p[(long long)s * v.ss + (long long)a[2] * v.sz + (long long)a[1] * v.sy + a[0]];
}

// The paper's 27-point operator (reading R28; SPEC weights): (A u)_i =
// (8/3 u_i - 1/6 sum_{12 edge nbrs} - 1/12 sum_{8 corner nbrs}) / h^2, face weight 0.  A
// neighbour outside Omega is the reflected ghost (-1)^m u(mirror), mirrored per dimension
// (R3); the mirror cells are in-domain cells of the same storage box.
template <class T>
__device__ __forceinline__ T apply_A27(const Lvl& L, const T* __restrict__ u, long long off,
                                       const int g[3]) {
  const long long st[3] = {1, (long long)L.py, L.pz};
  T e = T(0), k = T(0);
#pragma unroll
  for (int oz = -1; oz <= 1; ++oz)
#pragma unroll
    for (int oy = -1; oy <= 1; ++oy)
#pragma unroll
      for (int ox = -1; ox <= 1; ++ox) {
        const int nz = (ox != 0) + (oy != 0) + (oz != 0);
        if (nz < 2) continue;
        const int o[3] = {ox, oy, oz};
        long long d = 0;
        T sg = T(1);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          int gn = g[q] + o[q];
          if (gn < 0) {
            gn = -1 - gn;
            sg = -sg;
          } else if (gn >= L.N[q]) {
            gn = 2 * L.N[q] - 1 - gn;
            sg = -sg;
          }
          d += (long long)(gn - g[q]) * st[q];
        }
        const T v = sg * u[off + d];
        if (nz == 2) e += v;
        else k += v;
      }
  const T c = u[off];
  return (T(8.0 / 3.0) * c - e * T(1.0 / 6.0) - k * T(1.0 / 12.0)) * T(L.inv_h2) +
         T(L.nlg) * c * c * c;
}

// (A u) at local cell a / global cell g of segment storage `u` (offset `off`):
// A = -Lap_h, 7 points (R1/R2); a neighbour outside Omega is the reflected ghost -u_i
// (R3).  Neighbour sum order z-, z+, y-, y+, x-, x+ (as the oracle).
template <class T>
__device__ __forceinline__ T apply_A(const Lvl& L, const T* __restrict__ u, long long off,
                                     const int g[3]) {
  if (L.st27) return apply_A27(L, u, off, g);
  const T c = u[off];
  T s = T(0);
  s += (g[2] > 0) ? u[off - L.pz] : -c;
  s += (g[2] < L.N[2] - 1) ? u[off + L.pz] : -c;
  s += (g[1] > 0) ? u[off - L.py] : -c;
  s += (g[1] < L.N[1] - 1) ? u[off + L.py] : -c;
  s += (g[0] > 0) ? u[off - 1] : -c;
  s += (g[0] < L.N[0] - 1) ? u[off + 1] : -c;
  return (T(6) * c - s) * T(L.inv_h2) + T(L.nlg) * c * c * c;
}

// ------------------------------------------------------------------------------------
// Column-marching thread layout shared by the segment kernels: a CTA covers a (bx, by)
// tile of one segment's storage plane, each thread owns one (x, y) column and marches z
// over a chunk of planes, keeping the z-neighbours of its column in registers.  No
// per-cell integer division; domain/region tests are hoisted per column.
// ------------------------------------------------------------------------------------
struct Col {
  int ax, ay;   // local storage column
  int z0, z1;   // local z chunk [z0, z1)
};

__device__ __forceinline__ bool col_index(int ex, int ey, int ez, int ntx, int zchunk, Col& c) {
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  c.ax = tx * blockDim.x + threadIdx.x;
  c.ay = ty * blockDim.y + threadIdx.y;
  c.z0 = blockIdx.z * zchunk;
  c.z1 = min(ez, c.z0 + zchunk);
  return c.ax < ex && c.ay < ey && c.z0 < c.z1;
}

// ------------------------------------------------------------------------------------
// One Chebyshev step (R8) on the compute region C = grow(V,J) ∩ Omega
// (fig:fmgsr L222, fig:mgvsr L232/L242):
//   out = cur + c_mom (cur - prev) + c_res (b - A cur)      on C
//   out = cur                                               on GSR (if copy_gsr)
// A = -Lap_h, 7 points (R1/R2); a neighbour outside Omega is the reflected ghost -u_i (R3,
// PAPER.md:161); neighbour sum order z-, z+, y-, y+, x-, x+ (as the oracle).
// prev may alias out (in-place second step: each thread reads prev at its own cell only).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_cheb_step(Lvl L, const T* __restrict__ cur,
                                                        const T* prev, View<T> b, T* out,
                                                        T c_mom, T c_res, int copy_gsr, int ntx,
                                                        int zchunk) {
  constexpr int U = 4;  // planes per batch: all loads of a batch are issued before any use
  Col c;
  if (!col_index(L.E[0], L.E[1], L.E[2], ntx, zchunk, c)) return;
  const int s = blockIdx.y;
  int p[3], o[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  const int gx = o[0] + c.ax, gy = o[1] + c.ay;
  if (gx < 0 || gx >= L.N[0] || gy < 0 || gy >= L.N[1]) return;
  const bool cxy = c.ax >= 1 && c.ax <= L.E[0] - 2 && c.ay >= 1 && c.ay <= L.E[1] - 2;
  const bool xm = gx > 0, xp = gx < L.N[0] - 1, ym = gy > 0, yp = gy < L.N[1] - 1;
  const long long col = (long long)s * L.ss + (long long)c.ay * L.py + c.ax;
  const T* cc = cur + col;
  const T* bc = b.global ? b.p + (long long)gy * b.sy + gx : b.p + (long long)s * b.ss +
                                                                 (long long)c.ay * b.sy + c.ax;
  const long long pz = L.pz, py = L.py;
  const int E2 = L.E[2], N2 = L.N[2];
  T zq[U + 2];  // zq[k] = u at local plane az - 1 + k
  zq[0] = c.z0 > 0 ? cc[(long long)(c.z0 - 1) * pz] : T(0);
  zq[1] = cc[(long long)c.z0 * pz];
  for (int az = c.z0; az < c.z1; az += U) {
    T nb[U][4], bv[U], pv[U];
    bool act[U], inn[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int zz = az + 1 + k;
      zq[k + 2] = (zz < E2) ? cc[(long long)zz * pz] : T(0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int z = az + k;
      const int gz = o[2] + z;
      act[k] = z < c.z1 && gz >= 0 && gz < N2;
      inn[k] = act[k] && cxy && z >= 1 && z <= E2 - 2;
      const long long zo = (long long)z * pz;
      if (inn[k]) {
        nb[k][0] = ym ? cc[zo - py] : T(0);
        nb[k][1] = yp ? cc[zo + py] : T(0);
        nb[k][2] = xm ? cc[zo - 1] : T(0);
        nb[k][3] = xp ? cc[zo + 1] : T(0);
        bv[k] = bc[b.global ? (long long)gz * b.sz : (long long)z * b.sz];
        pv[k] = prev != nullptr ? prev[col + zo] : T(0);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int z = az + k;
      const int gz = o[2] + z;
      const long long zo = (long long)z * pz;
      const T v0 = zq[k + 1];
      if (inn[k]) {
        T sum = (gz > 0) ? zq[k] : -v0;
        sum += (gz < N2 - 1) ? zq[k + 2] : -v0;
        sum += ym ? nb[k][0] : -v0;
        sum += yp ? nb[k][1] : -v0;
        sum += xm ? nb[k][2] : -v0;
        sum += xp ? nb[k][3] : -v0;
        const T r = bv[k] - ((T(6) * v0 - sum) * T(L.inv_h2) + T(L.nlg) * v0 * v0 * v0);
        T v = v0 + c_res * r;
        if (prev != nullptr) v = v0 + c_mom * (v0 - pv[k]) + c_res * r;
        out[col + zo] = v;
      } else if (act[k] && copy_gsr) {
        out[col + zo] = v0;
      }
    }
    zq[0] = zq[U];
    zq[1] = zq[U + 1];
  }
}

// ------------------------------------------------------------------------------------
// Residual + 8-child average restriction (fig:mgv L113-115, fig:mgvsr L233/L235, R9):
// for every coarse cell I of the target box grow(coarsen(V_f^p), jr) ∩ Omega_c
//   uc[I] = (1/8) sum_children u_f          (I-hat, solution restriction)
//   rc[I] = (1/8) sum_children (b - A u_f)  (I, residual restriction; stored in the
//                                           coarse rhs buffer until the tau kernel)
// jr = floor(J_f/2) when the coarse level is an SR level (target F, R15); 0 otherwise
// (target V_T^p at k = 1 (R16), or Omega_c on conventional levels).
// One thread per coarse (X, Y) column, marching coarse Z; the 2x2 fine child columns'
// planes 2Z-1..2Z+2 live in registers.
// ------------------------------------------------------------------------------------
// bc.p != null (bf is f_l and bc = f_{l-1} = avg8(f_l), the R6 pyramid): the residual
// average is taken as avg8(b - A u) = bc - avg8(A u), so the fine b is not read at all.
// (launch bounds without a minimum block count: the compiler's own register choice, 64 in
// fp64, measured best -- an explicit minimum of 1 lets it take 96 and the finest-level
// restriction slows from 0.43 to 0.64 ms; 4 (64, with spills) 0.48; 5 (48) 0.56 ms)
template <class T, int UNR = 1>
__global__ void __launch_bounds__(kThreads) k_restrict(Lvl Lf, const T* __restrict__ uf,
                                                       View<T> bf, Lvl Lc, T* __restrict__ uc,
                                                       T* __restrict__ rc, int jr, int ntx,
                                                       int zchunk, View<T> bc) {
  const int s = blockIdx.y;
  int B[3], lo[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) B[d] = Lf.S[d] / 2 + 2 * jr;
  Col c;
  if (!col_index(B[0], B[1], B[2], ntx, zchunk, c)) return;
  int pf[3], of[3];
  seg_coords(Lf, s, pf);
  seg_origin(Lf, pf, of);
#pragma unroll
  for (int d = 0; d < 3; ++d) lo[d] = pf[d] * (Lf.S[d] / 2) - jr;
  const int X = lo[0] + c.ax, Y = lo[1] + c.ay;
  if (X < 0 || X >= Lc.N[0] || Y < 0 || Y >= Lc.N[1]) return;
  const int Zb = max(lo[2] + c.z0, 0), Ze = min(lo[2] + c.z1, Lc.N[2]);
  if (Zb >= Ze) return;
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  int pc[3], oc[3];
  seg_coords(Lc, cs, pc);
  seg_origin(Lc, pc, oc);
  const long long fpz = Lf.pz, fpy = Lf.py;
  // fine column (2X+dx, 2Y+dy) local offsets
  const int fx = 2 * X - of[0], fy = 2 * Y - of[1];
  const long long fcol = (long long)s * Lf.ss + (long long)fy * fpy + fx;
  const T* u = uf + fcol;
  const bool xm = X > 0, xp = X < Lc.N[0] - 1, ym = Y > 0, yp = Y < Lc.N[1] - 1;
  const T* bcol;
  long long bsz;
  if (bf.global) {
    bcol = bf.p + (long long)(2 * Y) * bf.sy + 2 * X;
    bsz = bf.sz;
  } else {
    bcol = bf.p + (long long)s * bf.ss + (long long)fy * bf.sy + fx;
    bsz = bf.sz;
  }
  // q[k][j]: column j = dy*2+dx, plane 2Z-1+k (k = 0..3)
  T q[4][4];
  {
    const long long z = (long long)(2 * Zb - 1 - of[2]) * fpz;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) q[k][j] = u[z + k * fpz + (j >> 1) * fpy + (j & 1)];
  }
#pragma unroll UNR
  for (int Z = Zb; Z < Ze; ++Z) {
    const long long z0 = (long long)(2 * Z - of[2]) * fpz;
#pragma unroll
    for (int k = 2; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) q[k][j] = u[z0 + (k - 1) * fpz + (j >> 1) * fpy + (j & 1)];
    const bool zmo = Z > 0, zpo = Z < Lc.N[2] - 1;
    T su = T(0), sr = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz) {
      const long long zf = z0 + dz * fpz;
      const long long bz = bf.global ? (long long)(2 * Z + dz) * bsz
                                     : (long long)(2 * Z + dz - of[2]) * bsz;
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int j = dy * 2 + dx;
          const T v = q[dz + 1][j];
          T sum = (dz == 0) ? (zmo ? q[0][j] : -v) : q[1][j];
          sum += (dz == 0) ? q[2][j] : (zpo ? q[3][j] : -v);
          const long long yo = zf + dy * fpy + dx;
          sum += (dy == 0) ? (ym ? u[yo - fpy] : -v) : q[dz + 1][dx];
          sum += (dy == 0) ? q[dz + 1][2 + dx] : (yp ? u[yo + fpy] : -v);
          sum += (dx == 0) ? (xm ? u[yo - 1] : -v) : q[dz + 1][dy * 2];
          sum += (dx == 0) ? q[dz + 1][dy * 2 + 1] : (xp ? u[yo + 1] : -v);
          const T Au = (T(6) * v - sum) * T(Lf.inv_h2) + T(Lf.nlg) * v * v * v;
          su += v;
          if (bc.p) {
            sr -= Au;
          } else {
            const T bv = bcol[bz + dy * bf.sy + dx];
            sr += bv - Au;
          }
        }
    }
    const long long co = (long long)cs * Lc.ss + (long long)(Z - oc[2]) * Lc.pz +
                         (long long)(Y - oc[1]) * Lc.py + (X - oc[0]);
    uc[co] = su * T(0.125);
    rc[co] = bc.p ? bc.p[(long long)Z * bc.sz + (long long)Y * bc.sy + X] + sr * T(0.125)
                  : sr * T(0.125);
    // planes 2Z+1, 2Z+2 are planes 2(Z+1)-1, 2(Z+1) of the next step
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      q[0][j] = q[2][j];
      q[1][j] = q[3][j];
    }
  }
}

// ------------------------------------------------------------------------------------
// FAS coarse right-hand side and t snapshot on a coarse level (Eq. 4; fig:mgv L116-117;
// fig:mgvsr L234-236; R18):
//   t = u                              on storage ∩ Omega
//   rhs = R + A u                      on F   (R = restricted residual already in rhs)
//   rhs = A u                          on C \ F
// F = grow(V, jr) ∩ Omega (jr = floor(J_fine/2) on SR levels; 0 -> F = V = Omega on
// conventional levels).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_tau(Lvl L, const T* __restrict__ u,
                                                  T* __restrict__ rhs, T* __restrict__ t,
                                                  int jr, int ntx, int zchunk) {
  Col c;
  if (!col_index(L.E[0], L.E[1], L.E[2], ntx, zchunk, c)) return;
  const int s = blockIdx.y;
  int p[3], o[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  const int gx = o[0] + c.ax, gy = o[1] + c.ay;
  if (gx < 0 || gx >= L.N[0] || gy < 0 || gy >= L.N[1]) return;
  const bool cxy = c.ax >= 1 && c.ax <= L.E[0] - 2 && c.ay >= 1 && c.ay <= L.E[1] - 2;
  const bool fxy = gx >= p[0] * L.S[0] - jr && gx < (p[0] + 1) * L.S[0] + jr &&
                   gy >= p[1] * L.S[1] - jr && gy < (p[1] + 1) * L.S[1] + jr;
  const int fz0 = p[2] * L.S[2] - jr, fz1 = (p[2] + 1) * L.S[2] + jr;
  const bool xm = gx > 0, xp = gx < L.N[0] - 1, ym = gy > 0, yp = gy < L.N[1] - 1;
  const long long col = (long long)s * L.ss + (long long)c.ay * L.py + c.ax;
  const T* cc = u + col;
  const long long pz = L.pz, py = L.py;
  const int E2 = L.E[2], N2 = L.N[2];
  constexpr int U = 4;  // planes per batch: all loads of a batch are issued before any use
  T zq[U + 2];
  zq[0] = c.z0 > 0 ? cc[(long long)(c.z0 - 1) * pz] : T(0);
  zq[1] = cc[(long long)c.z0 * pz];
  for (int az = c.z0; az < c.z1; az += U) {
    T nb[U][4], rv[U];
    bool act[U], inn[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int zz = az + 1 + k;
      zq[k + 2] = (zz < E2) ? cc[(long long)zz * pz] : T(0);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int z = az + k;
      const int gz = o[2] + z;
      act[k] = z < c.z1 && gz >= 0 && gz < N2;
      inn[k] = act[k] && cxy && z >= 1 && z <= E2 - 2;
      const long long zo = (long long)z * pz;
      if (inn[k]) {
        nb[k][0] = ym ? cc[zo - py] : T(0);
        nb[k][1] = yp ? cc[zo + py] : T(0);
        nb[k][2] = xm ? cc[zo - 1] : T(0);
        nb[k][3] = xp ? cc[zo + 1] : T(0);
        rv[k] = (fxy && gz >= fz0 && gz < fz1) ? rhs[col + zo] : T(0);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int z = az + k;
      const int gz = o[2] + z;
      const long long zo = (long long)z * pz;
      const T v0 = zq[k + 1];
      if (act[k]) t[col + zo] = v0;
      if (inn[k]) {
        T sum = (gz > 0) ? zq[k] : -v0;
        sum += (gz < N2 - 1) ? zq[k + 2] : -v0;
        sum += ym ? nb[k][0] : -v0;
        sum += yp ? nb[k][1] : -v0;
        sum += xm ? nb[k][2] : -v0;
        sum += xp ? nb[k][3] : -v0;
        const T Au = (T(6) * v0 - sum) * T(L.inv_h2) + T(L.nlg) * v0 * v0 * v0;
        const bool inF = fxy && gz >= fz0 && gz < fz1;
        rhs[col + zo] = inF ? rv[k] + Au : Au;
      }
    }
    zq[0] = zq[U];
    zq[1] = zq[U + 1];
  }
}

// ------------------------------------------------------------------------------------
// Cell-centred trilinear prolongation onto C ∪ GSR = storage ∩ Omega (R10, PAPER.md:256;
// range fig:fmgsr L221 / fig:mgvsr L241, R17):
//   add == 0:  u_f = P(w)          (FMG interpolation Pi)
//   add == 1:  u_f += P(w - t)     (V-cycle correction)
// Coarse cells just outside Omega_c are reflected ghosts -(value at the mirror) (R3).
// The coarse source is the fine segment's own coarse storage (SR level below) or the
// single global coarse array (transition / conventional level below).
// One thread per fine (x, y) column; it marches the coarse planes P and produces the fine
// planes 2P, 2P+1 from a register queue of coarse planes P-1, P, P+1.
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_prolong(Lvl Lf, T* __restrict__ uf, Lvl Lc,
                                                      const T* __restrict__ w,
                                                      const T* __restrict__ tc, int add, int ntx,
                                                      int zchunk) {
  Col c;
  if (!col_index(Lf.E[0], Lf.E[1], Lf.E[2], ntx, zchunk, c)) return;
  const int s = blockIdx.y;
  int p[3], o[3];
  seg_coords(Lf, s, p);
  seg_origin(Lf, p, o);
  const int gx = o[0] + c.ax, gy = o[1] + c.ay;
  if (gx < 0 || gx >= Lf.N[0] || gy < 0 || gy >= Lf.N[1]) return;
  const int gz0 = max(o[2] + c.z0, 0), gz1 = min(o[2] + c.z1, Lf.N[2]);
  if (gz0 >= gz1) return;
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  int pc[3], oc[3];
  seg_coords(Lc, cs, pc);
  seg_origin(Lc, pc, oc);
  // x / y: parent (k=0) and neighbour (k=1) coarse local index and sign
  int cx[2], cy[2];
  T sx1 = T(1), sy1 = T(1);
  {
    const int P = gx >> 1, Q = P + ((gx & 1) ? 1 : -1);
    int Qm = Q;
    if (Q < 0) { Qm = 0; sx1 = T(-1); }
    if (Q >= Lc.N[0]) { Qm = Lc.N[0] - 1; sx1 = T(-1); }
    cx[0] = P - oc[0];
    cx[1] = Qm - oc[0];
  }
  {
    const int P = gy >> 1, Q = P + ((gy & 1) ? 1 : -1);
    int Qm = Q;
    if (Q < 0) { Qm = 0; sy1 = T(-1); }
    if (Q >= Lc.N[1]) { Qm = Lc.N[1] - 1; sy1 = T(-1); }
    cy[0] = P - oc[1];
    cy[1] = Qm - oc[1];
  }
  const long long cbase = (long long)cs * Lc.ss;
  long long coff[4];  // j = ky*2 + kx
#pragma unroll
  for (int j = 0; j < 4; ++j) coff[j] = cbase + (long long)cy[j >> 1] * Lc.py + cx[j & 1];
  // separable trilinear: the (x, y) interpolation of coarse plane P is shared by the two
  // fine planes 2P, 2P+1 (weights 3/4 parent, 1/4 neighbour; signs of reflected ghosts)
  const T W[2] = {T(0.75), T(0.25)};
  const T wxy[4] = {W[0] * W[0], W[0] * W[1] * sx1, W[1] * W[0] * sy1, W[1] * W[1] * (sy1 * sx1)};
  auto load_plane = [&](int P) -> T {  // xy-interpolant of coarse plane P (reflected outside)
    T sg = T(1);
    int Pm = P;
    if (P < 0) { Pm = 0; sg = T(-1); }
    if (P >= Lc.N[2]) { Pm = Lc.N[2] - 1; sg = T(-1); }
    // planes the fine chunk's first/last cell does not use may lie outside the coarse
    // storage box (small J): clamp them into it (their values are never used)
    const int lz = min(max(Pm - oc[2], 0), Lc.E[2] - 1);
    const long long zo = (long long)lz * Lc.pz;
    T v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = w[coff[j] + zo];
      if (add) v[j] = v[j] - tc[coff[j] + zo];
    }
    return sg * ((wxy[0] * v[0] + wxy[1] * v[1]) + (wxy[2] * v[2] + wxy[3] * v[3]));
  };
  // coarse planes P-1 .. P+2 (queue), fine planes 2P .. 2P+3 per batch: all loads of a
  // batch are issued before any use (memory-level parallelism)
  T q[4];
  int P = gz0 >> 1;
  q[0] = load_plane(P - 1);
  q[1] = load_plane(P);
  const long long fcol = (long long)s * Lf.ss + (long long)c.ay * Lf.py + c.ax;
  for (; 2 * P < gz1; P += 2) {
    q[2] = load_plane(P + 1);
    q[3] = load_plane(P + 2);
    T uo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gz = 2 * P + e;
      uo[e] = T(0);
      if (add && gz >= gz0 && gz < gz1) uo[e] = uf[fcol + (long long)(gz - o[2]) * Lf.pz];
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gz = 2 * P + e;
      if (gz < gz0 || gz >= gz1) continue;
      const T qp = q[1 + (e >> 1)];                            // parent plane P + e/2
      const T qn = (e & 1) ? q[2 + (e >> 1)] : q[e >> 1];      // neighbour on the child's side
      const T acc = W[0] * qp + W[1] * qn;
      const long long off = fcol + (long long)(gz - o[2]) * Lf.pz;
      uf[off] = add ? uo[e] + acc : acc;
    }
    q[0] = q[2];
    q[1] = q[3];
  }
}

// ------------------------------------------------------------------------------------
// Exact coarsest solve u_0 = A_0^{-1} b (fig:mgv L120-121; R7): dense inverse (host fp64,
// rounded to T for fp32), one CTA, one thread per coarsest cell.
// ------------------------------------------------------------------------------------
template <class T>
__global__ void k_coarsest(Lvl L, T* __restrict__ u, View<T> b, const T* __restrict__ ainv) {
  const int n0 = L.N[0] * L.N[1] * L.N[2];
  extern __shared__ unsigned char smem_raw[];
  T* bs = reinterpret_cast<T*>(smem_raw);
  for (int j = threadIdx.x; j < n0; j += blockDim.x) {
    int g[3] = {j % L.N[0], (j / L.N[0]) % L.N[1], j / (L.N[0] * L.N[1])};
    int a[3] = {g[0] + 1, g[1] + 1, g[2] + 1};
    bs[j] = view_at(b, 0, a, g);
  }
  __syncthreads();
  // nonlinear (R29): Picard iteration u <- A_lin^-1 (b - nlg u^3) from u = A_lin^-1 b; the
  // contraction 3 nlg u^2 / lambda_min(A_0) is small on the coarsest grid, 40 sweeps reach
  // the root to rounding
  T* us = bs + n0;
  const int sweeps = L.nlg != 0.0 ? 41 : 1;
  for (int it = 0; it < sweeps; ++it) {
    for (int i = threadIdx.x; i < n0; i += blockDim.x) {
      T acc = T(0);
      for (int j = 0; j < n0; ++j) acc += ainv[(long long)i * n0 + j] * bs[j];
      us[i] = acc;
    }
    __syncthreads();
    if (it + 1 < sweeps) {
      for (int j = threadIdx.x; j < n0; j += blockDim.x) {
        int g[3] = {j % L.N[0], (j / L.N[0]) % L.N[1], j / (L.N[0] * L.N[1])};
        int a[3] = {g[0] + 1, g[1] + 1, g[2] + 1};
        const T x = us[j];
        bs[j] = view_at(b, 0, a, g) - T(L.nlg) * x * x * x;
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n0; i += blockDim.x) {
    int g[3] = {i % L.N[0], (i / L.N[0]) % L.N[1], i / (L.N[0] * L.N[1])};
    u[loc_off(L, 0, g[0] + 1, g[1] + 1, g[2] + 1)] = us[i];
  }
}

// f_{l-1} = avg8(f_l) on dense arrays (R6)
template <class T>
__global__ void __launch_bounds__(kThreads) k_pyramid(const T* __restrict__ ff, int nfx, int nfy,
                                                      int nfz, T* __restrict__ fc) {
  const int ncx = nfx / 2, ncy = nfy / 2, ncz = nfz / 2;
  const long long n = (long long)ncx * ncy * ncz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = i % ncx;
    const int y = (i / ncx) % ncy;
    const int z = i / ((long long)ncx * ncy);
    T s = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          s += ff[((long long)(2 * z + dz) * nfy + (2 * y + dy)) * nfx + (2 * x + dx)];
    fc[i] = s * T(0.125);
  }
}

// ---- 27-point variants: one thread per storage cell, same regions and
// arithmetic as k_cheb_step / k_tau / k_restrict with A = apply_A27 ------------------------
__device__ __forceinline__ bool cell_of_box(const Lvl& L, long long i, int& s, int a[3],
                                            int g[3], int p[3]) {
  const long long per = (long long)L.E[0] * L.E[1] * L.E[2];
  s = (int)(i / per);
  long long r = i % per;
  a[0] = (int)(r % L.E[0]);
  r /= L.E[0];
  a[1] = (int)(r % L.E[1]);
  a[2] = (int)(r / L.E[1]);
  int o[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  bool in = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g[d] = o[d] + a[d];
    in = in && g[d] >= 0 && g[d] < L.N[d];
  }
  return in;
}

template <class T>
__global__ void __launch_bounds__(kThreads) k_cheb_step27(Lvl L, const T* __restrict__ cur,
                                                          const T* prev, View<T> b, T* out,
                                                          T c_mom, T c_res, int copy_gsr) {
  const long long n = (long long)L.nsegs * L.E[0] * L.E[1] * L.E[2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int s, a[3], g[3], p[3];
    if (!cell_of_box(L, i, s, a, g, p)) continue;
    const long long off = loc_off(L, s, a[0], a[1], a[2]);
    bool c = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) c = c && a[d] >= 1 && a[d] <= L.E[d] - 2;
    const T v0 = cur[off];
    if (c) {
      const T r = view_at(b, s, a, g) - apply_A27(L, cur, off, g);
      T v = v0 + c_res * r;
      if (prev != nullptr) v = v0 + c_mom * (v0 - prev[off]) + c_res * r;
      out[off] = v;
    } else if (copy_gsr) {
      out[off] = v0;
    }
  }
}

// Column-marching 27-point Chebyshev step: thread per (x, y) storage column and z chunk;
// the 3x3 neighbourhoods of planes z-1, z, z+1 stay in registers (9 loads per cell instead
// of 20), reflected ghosts via per-column mirrored offsets and signs (R3, R28).
template <class T, int RESID = 0>
__global__ void __launch_bounds__(kThreads) k_cheb_step27c(Lvl L, const T* __restrict__ cur,
                                                           const T* prev, View<T> b, T* out,
                                                           T c_mom, T c_res, int copy_gsr,
                                                           int ntx, int zchunk) {
  Col c;
  if (!col_index(L.E[0], L.E[1], L.E[2], ntx, zchunk, c)) return;
  const int s = blockIdx.y;
  int p[3], o[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  const int gx = o[0] + c.ax, gy = o[1] + c.ay;
  if (gx < 0 || gx >= L.N[0] || gy < 0 || gy >= L.N[1]) return;
  const bool cxy = c.ax >= 1 && c.ax <= L.E[0] - 2 && c.ay >= 1 && c.ay <= L.E[1] - 2;
  const long long col = (long long)s * L.ss + (long long)c.ay * L.py + c.ax;
  // in-plane 3x3 neighbourhood: mirrored offsets and signs (index j = (dy+1)*3 + (dx+1))
  long long xyo[9];
  T xys[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const int dx = j % 3 - 1, dy = j / 3 - 1;
    int qx = gx + dx, qy = gy + dy;
    T sg = T(1);
    if (qx < 0) { qx = -1 - qx; sg = -sg; }
    if (qx >= L.N[0]) { qx = 2 * L.N[0] - 1 - qx; sg = -sg; }
    if (qy < 0) { qy = -1 - qy; sg = -sg; }
    if (qy >= L.N[1]) { qy = 2 * L.N[1] - 1 - qy; sg = -sg; }
    xyo[j] = (long long)(qy - gy) * L.py + (qx - gx);
    // neighbours outside the storage box only belong to non-C columns (never used): no load
    const int mx = c.ax + (qx - gx), my = c.ay + (qy - gy);
    xys[j] = (mx >= 0 && mx < L.E[0] && my >= 0 && my < L.E[1]) ? sg : T(0);
    if (xys[j] == T(0)) xyo[j] = 0;
  }
  const T* bc = b.global ? b.p + (long long)gy * b.sy + gx
                         : b.p + (long long)s * b.ss + (long long)c.ay * b.sy + c.ax;
  const int N2 = L.N[2];
  // plane window w[k][j]: k = 0, 1, 2 for planes z-1, z, z+1 (signed, mirrored)
  T w[3][9];
  auto load_plane = [&](int z, T (&q)[9]) {  // storage plane z (global o[2] + z)
    int gz = o[2] + z;
    T sz = T(1);
    if (gz < 0) { gz = -1 - gz; sz = -sz; }
    if (gz >= N2) { gz = 2 * N2 - 1 - gz; sz = -sz; }
    const int mz = gz - o[2];
    if (mz < 0 || mz >= L.E[2]) {  // outside the storage box: only non-C planes use it
#pragma unroll
      for (int j = 0; j < 9; ++j) q[j] = T(0);
      return;
    }
    const long long zo = (long long)mz * L.pz;
#pragma unroll
    for (int j = 0; j < 9; ++j) q[j] = (sz * xys[j]) * cur[col + zo + xyo[j]];
  };
  const int z0 = c.z0, z1 = c.z1;
  load_plane(z0 - 1, w[0]);
  load_plane(z0, w[1]);
  for (int z = z0; z < z1; ++z) {
    load_plane(z + 1, w[2]);
    const int gz = o[2] + z;
    const long long off = col + (long long)z * L.pz;
    if (gz >= 0 && gz < N2) {
      const T v0 = w[1][4];
      if (cxy && z >= 1 && z <= L.E[2] - 2) {
        // edges: in-plane diagonals of plane z, and the 4-neighbourhood of planes z +- 1
        const T e = (w[1][0] + w[1][2] + w[1][6] + w[1][8]) +
                    ((w[0][1] + w[0][3] + w[0][5] + w[0][7]) + (w[2][1] + w[2][3] + w[2][5] + w[2][7]));
        const T k = (w[0][0] + w[0][2] + w[0][6] + w[0][8]) + (w[2][0] + w[2][2] + w[2][6] + w[2][8]);
        const T Au = (T(8.0 / 3.0) * v0 - e * T(1.0 / 6.0) - k * T(1.0 / 12.0)) * T(L.inv_h2) +
                     T(L.nlg) * v0 * v0 * v0;
        const T r = bc[b.global ? (long long)gz * b.sz : (long long)z * b.sz] - Au;
        if constexpr (RESID) {
          out[off] = r;  // residual only (restriction, first pass)
        } else {
          T v = v0 + c_res * r;
          if (prev != nullptr) v = v0 + c_mom * (v0 - prev[off]) + c_res * r;
          out[off] = v;
        }
      } else if (copy_gsr) {
        out[off] = v0;
      }
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      w[0][j] = w[1][j];
      w[1][j] = w[2][j];
    }
  }
}

template <class T>
__global__ void __launch_bounds__(kThreads) k_tau27(Lvl L, const T* __restrict__ u,
                                                    T* __restrict__ rhs, T* __restrict__ t,
                                                    int jr) {
  const long long n = (long long)L.nsegs * L.E[0] * L.E[1] * L.E[2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int s, a[3], g[3], p[3];
    if (!cell_of_box(L, i, s, a, g, p)) continue;
    const long long off = loc_off(L, s, a[0], a[1], a[2]);
    t[off] = u[off];
    bool c = true, inF = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      c = c && a[d] >= 1 && a[d] <= L.E[d] - 2;
      inF = inF && g[d] >= p[d] * L.S[d] - jr && g[d] < (p[d] + 1) * L.S[d] + jr;
    }
    if (c) {
      const T Au = apply_A27(L, u, off, g);
      rhs[off] = inF ? rhs[off] + Au : Au;
    }
  }
}

template <class T>
__global__ void __launch_bounds__(kThreads) k_restrict27(Lvl Lf, const T* __restrict__ uf,
                                                         View<T> bf, Lvl Lc, T* __restrict__ uc,
                                                         T* __restrict__ rc, int jr) {
  int B[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) B[d] = Lf.S[d] / 2 + 2 * jr;
  const long long per = (long long)B[0] * B[1] * B[2];
  const long long n = per * Lf.nsegs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / per);
    long long r = i % per;
    int pf[3], of[3], pc[3], oc[3], X[3];
    seg_coords(Lf, s, pf);
    seg_origin(Lf, pf, of);
    bool ok = true;
    X[0] = pf[0] * (Lf.S[0] / 2) - jr + (int)(r % B[0]);
    r /= B[0];
    X[1] = pf[1] * (Lf.S[1] / 2) - jr + (int)(r % B[1]);
    X[2] = pf[2] * (Lf.S[2] / 2) - jr + (int)(r / B[1]);
#pragma unroll
    for (int d = 0; d < 3; ++d) ok = ok && X[d] >= 0 && X[d] < Lc.N[d];
    if (!ok) continue;
    const int cs = (Lc.nsegs == 1) ? 0 : s;
    seg_coords(Lc, cs, pc);
    seg_origin(Lc, pc, oc);
    T su = T(0), sr = T(0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int g[3] = {2 * X[0] + (c & 1), 2 * X[1] + ((c >> 1) & 1), 2 * X[2] + (c >> 2)};
      const int a[3] = {g[0] - of[0], g[1] - of[1], g[2] - of[2]};
      const long long off = loc_off(Lf, s, a[0], a[1], a[2]);
      su += uf[off];
      sr += view_at(bf, s, a, g) - apply_A27(Lf, uf, off, g);
    }
    const long long co = loc_off(Lc, cs, X[0] - oc[0], X[1] - oc[1], X[2] - oc[2]);
    uc[co] = su * T(0.125);
    rc[co] = sr * T(0.125);
  }
}

// restriction from a precomputed fine residual r (27-point path): per coarse target cell
// uc = avg8(u_f), rc = avg8(r)
template <class T>
__global__ void __launch_bounds__(kThreads) k_avg8_ur(Lvl Lf, const T* __restrict__ uf,
                                                      const T* __restrict__ rf, Lvl Lc,
                                                      T* __restrict__ uc, T* __restrict__ rc,
                                                      int jr, View<T> bc) {
  int B[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) B[d] = Lf.S[d] / 2 + 2 * jr;
  const long long per = (long long)B[0] * B[1] * B[2];
  const long long n = per * Lf.nsegs;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / per);
    long long r = i % per;
    int pf[3], of[3], pc[3], oc[3], X[3];
    seg_coords(Lf, s, pf);
    seg_origin(Lf, pf, of);
    X[0] = pf[0] * (Lf.S[0] / 2) - jr + (int)(r % B[0]);
    r /= B[0];
    X[1] = pf[1] * (Lf.S[1] / 2) - jr + (int)(r % B[1]);
    X[2] = pf[2] * (Lf.S[2] / 2) - jr + (int)(r / B[1]);
    bool ok = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) ok = ok && X[d] >= 0 && X[d] < Lc.N[d];
    if (!ok) continue;
    const int cs = (Lc.nsegs == 1) ? 0 : s;
    seg_coords(Lc, cs, pc);
    seg_origin(Lc, pc, oc);
    const long long f0 = loc_off(Lf, s, 2 * X[0] - of[0], 2 * X[1] - of[1], 2 * X[2] - of[2]);
    T su = T(0), sr = T(0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const long long off = f0 + (c & 1) + ((c >> 1) & 1) * (long long)Lf.py + (c >> 2) * Lf.pz;
      su += uf[off];
      sr += rf[off];
    }
    const long long co = loc_off(Lc, cs, X[0] - oc[0], X[1] - oc[1], X[2] - oc[2]);
    uc[co] = su * T(0.125);
    // bc.p: rf holds -A u only, R = f_{l-1} - avg8(A u) with f_{l-1} the R6 pyramid
    rc[co] = bc.p ? bc.p[(long long)X[2] * bc.sz + (long long)X[1] * bc.sy + X[0]] + sr * T(0.125)
                  : sr * T(0.125);
  }
}

template <class T>
unsigned grid_for(long long n) {
  return (unsigned)std::max<long long>(1, std::min<long long>(148LL * 16, (n + kThreads - 1) / kThreads));
}

// sum over Omega of (b - A u)^2 on a conventional (single-segment) level, accumulated in
// fp64 into acc[0] (V-cycle solver stopping test, reading R26)
template <class T>
__global__ void __launch_bounds__(kThreads) k_resnorm(Lvl L, const T* __restrict__ u, View<T> b,
                                                      double* acc) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int g[3] = {(int)(i % L.N[0]), (int)((i / L.N[0]) % L.N[1]),
                      (int)(i / ((long long)L.N[0] * L.N[1]))};
    const int a[3] = {g[0] + 1, g[1] + 1, g[2] + 1};
    const long long off = loc_off(L, 0, a[0], a[1], a[2]);
    const double r = (double)(view_at(b, 0, a, g) - apply_A(L, u, off, g));
    s += r * r;
  }
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) atomicAdd(acc, s);
  }
}

// output: genuine cells of each segment -> user u (R19); one thread per
// genuine (x, y) column of a segment, marching z.
template <class T>
__global__ void __launch_bounds__(kThreads) k_gather(Lvl L, const T* __restrict__ useg,
                                                     T* __restrict__ out, int bo0, int bo1, int bo2,
                                                     long long osy, long long osz, int ntx,
                                                     int zchunk) {
  Col c;
  if (!col_index(L.S[0], L.S[1], L.S[2], ntx, zchunk, c)) return;
  const int s = blockIdx.y;
  int p[3];
  seg_coords(L, s, p);
  const int h = L.J + 1;
  const T* src = useg + (long long)s * L.ss + (long long)(c.ay + h) * L.py + (c.ax + h);
  T* dst = out + (long long)(p[1] * L.S[1] + c.ay - bo1) * osy + (p[0] * L.S[0] + c.ax - bo0);
  for (int z = c.z0; z < c.z1; ++z)
    dst[(long long)(p[2] * L.S[2] + z - bo2) * osz] = src[(long long)(z + h) * L.pz];
}

// box copy between a strided array and a contiguous buffer (multi-GPU packing)
template <class T>
__global__ void __launch_bounds__(kThreads) k_box_copy(T* __restrict__ base, long long sy,
                                                       long long sz, int lx, int ly, int lz,
                                                       int nx, int ny, int nz,
                                                       T* __restrict__ buf, int to_buf) {
  const long long n = (long long)nx * ny * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = i % nx;
    const int y = (i / nx) % ny;
    const int z = i / ((long long)nx * ny);
    const long long o = (long long)(lz + z) * sz + (long long)(ly + y) * sy + (lx + x);
    if (to_buf) buf[i] = base[o];
    else base[o] = buf[i];
  }
}

// f_{l-1} = avg8(f_l) (R6) over a box of coarse cells [lo, lo + n) (global indices) between
// two dense views indexed globally (virtual origins): a rank's block of a domain-decomposed
// level, read from its (haloed) local f_l, written into its local f_{l-1} block or into its
// part of a global array (multi-GPU pyramid below level T)
template <class T>
__global__ void __launch_bounds__(kThreads) k_pyramid_box(View<T> f, View<T> c, int lx, int ly,
                                                          int lz, int nx, int ny, int nz) {
  const long long n = (long long)nx * ny * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int X = lx + (int)(i % nx);
    const int Y = ly + (int)((i / nx) % ny);
    const int Z = lz + (int)(i / ((long long)nx * ny));
    T s = T(0);
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy)
#pragma unroll
        for (int dx = 0; dx < 2; ++dx)
          s += f.p[(long long)(2 * Z + dz) * f.sz + (long long)(2 * Y + dy) * f.sy + (2 * X + dx)];
    const_cast<T*>(c.p)[(long long)Z * c.sz + (long long)Y * c.sy + X] = s * T(0.125);
  }
}

// dst = a - b (b != null) or dst = a on the S^3 block cells of two storage layouts (local
// cell (x, y, z) at (z + ga) pz + (y + ga) py + x + ga): the correction footprint of the
// k = 1 hand-off, w - t (or u for the FMG interpolation), moved into the wider-ghosted
// level-T array of a domain-decomposed run
template <class T>
__global__ void __launch_bounds__(kThreads) k_block_diff(Lvl La, const T* __restrict__ a,
                                                         const T* __restrict__ b, Lvl Ld,
                                                         T* __restrict__ dst) {
  const long long n = (long long)La.S[0] * La.S[1] * La.S[2];
  const int ga = La.J + 1, gd = Ld.J + 1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % La.S[0]);
    const int y = (int)((i / La.S[0]) % La.S[1]);
    const int z = (int)(i / ((long long)La.S[0] * La.S[1]));
    const long long oa = (long long)(z + ga) * La.pz + (long long)(y + ga) * La.py + (x + ga);
    const long long od = (long long)(z + gd) * Ld.pz + (long long)(y + gd) * Ld.py + (x + gd);
    dst[od] = b ? a[oa] - b[oa] : a[oa];
  }
}

}  // namespace

// column-layout launch geometry: (bx, by) tile over an (ex, ey) plane, z split into
// chunks so that small levels still fill the GPU
struct ColCfg {
  dim3 grid, block;
  int ntx, zchunk;
};

// target: threads to aim for by splitting columns into z-chunks (more chunks = more loads in
// flight, but each chunk re-reads its two boundary planes).  SR_FMG_COL_TARGET overrides.
ColCfg col_cfg(int ex, int ey, int ez, int nsegs, long long target_default = 200000) {
  ColCfg c;
  const int bx = std::min(ex, 128);
  const int by = std::max(1, std::min(ey, kThreads / bx));
  c.ntx = (ex + bx - 1) / bx;
  const int nty = (ey + by - 1) / by;
  const long long cols = (long long)nsegs * ex * ey;
  static const long long target_env = [] {
    const char* e = std::getenv("SR_FMG_COL_TARGET");
    return e ? std::atoll(e) : 0LL;
  }();
  const long long target = target_env > 0 ? target_env : target_default;
  static const int minz = [] {  // fewest planes per z-chunk (SR_FMG_COL_MINZ, tuning)
    const char* e = std::getenv("SR_FMG_COL_MINZ");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  int zsplit = (int)std::min<long long>((target + cols - 1) / cols, std::max(1, ez / minz));
  zsplit = std::max(zsplit, 1);
  c.zchunk = (ez + zsplit - 1) / zsplit;
  zsplit = (ez + c.zchunk - 1) / c.zchunk;
  c.grid = dim3(c.ntx * nty, nsegs, zsplit);
  c.block = dim3(bx, by, 1);
  return c;
}

template <class T>
void launch_cheb_step(const Lvl& L, const T* cur, const T* prev, View<T> b, T* out, double c_mom,
                      double c_res, int copy_gsr, cudaStream_t st) {
  if (L.st27) {
    const ColCfg c = col_cfg(L.E[0], L.E[1], L.E[2], L.nsegs);
    k_cheb_step27c<T><<<c.grid, c.block, 0, st>>>(L, cur, prev, b, out, (T)c_mom, (T)c_res,
                                                  copy_gsr, c.ntx, c.zchunk);
    return;
  }
  const ColCfg c = col_cfg(L.E[0], L.E[1], L.E[2], L.nsegs);
  k_cheb_step<T><<<c.grid, c.block, 0, st>>>(L, cur, prev, b, out, (T)c_mom, (T)c_res, copy_gsr,
                                             c.ntx, c.zchunk);
}

template <class T>
void launch_restrict(const Lvl& Lf, const T* uf, View<T> bf, const Lvl& Lc, T* uc, T* rc, int jr,
                     cudaStream_t st, T* scratch, View<T> bc) {
  int B[3];
  for (int d = 0; d < 3; ++d) B[d] = Lf.S[d] / 2 + 2 * jr;
  if (Lf.st27) {
    const long long n = (long long)B[0] * B[1] * B[2] * Lf.nsegs;
    if (scratch) {  // residual by the column-marching 27-point sweep, then the averages
      const ColCfg c = col_cfg(Lf.E[0], Lf.E[1], Lf.E[2], Lf.nsegs);
      k_cheb_step27c<T, 1><<<c.grid, c.block, 0, st>>>(Lf, uf, nullptr, bf, scratch, T(0), T(0),
                                                       0, c.ntx, c.zchunk);
      k_avg8_ur<T><<<grid_for<T>(n), kThreads, 0, st>>>(Lf, uf, scratch, Lc, uc, rc, jr,
                                                        View<T>{});
    } else {
      k_restrict27<T><<<grid_for<T>(n), kThreads, 0, st>>>(Lf, uf, bf, Lc, uc, rc, jr);
    }
    return;
  }
  // 800k threads: 0.657 -> 0.616 ms at C3's finest level, 0.281 -> 0.247 ms at E = 38.
  // Two coarse planes per loop trip in fp32 (C3 finest 0.298 vs 0.318 ms, level 7 0.154 vs
  // 0.168); fp64 keeps one (0.60 vs 0.43 ms unrolled: 98 registers).  SR_FMG_RESTRICT_UNROLL
  // overrides (tuning knob)
  static const int unr_env = [] {
    const char* e = std::getenv("SR_FMG_RESTRICT_UNROLL");
    return e ? std::atoi(e) : 0;
  }();
  const int unr = unr_env ? unr_env : (sizeof(T) == 4 ? 2 : 1);
  const ColCfg c = col_cfg(B[0], B[1], B[2], Lf.nsegs, 800000);
  if (unr == 2)
    k_restrict<T, 2><<<c.grid, c.block, 0, st>>>(Lf, uf, bf, Lc, uc, rc, jr, c.ntx, c.zchunk, bc);
  else
    k_restrict<T><<<c.grid, c.block, 0, st>>>(Lf, uf, bf, Lc, uc, rc, jr, c.ntx, c.zchunk, bc);
}

template <class T>
void launch_restrict_from_resid(const Lvl& Lf, const T* uf, const T* rf, const Lvl& Lc, T* uc,
                                T* rc, int jr, cudaStream_t st, View<T> bc) {
  long long n = Lf.nsegs;
  for (int d = 0; d < 3; ++d) n *= Lf.S[d] / 2 + 2 * jr;
  k_avg8_ur<T><<<grid_for<T>(n), kThreads, 0, st>>>(Lf, uf, rf, Lc, uc, rc, jr, bc);
}

template <class T>
void launch_tau(const Lvl& Lc, const T* u, T* rhs, T* t, int jr, cudaStream_t st) {
  if (Lc.st27) {
    const long long n = (long long)Lc.nsegs * Lc.E[0] * Lc.E[1] * Lc.E[2];
    k_tau27<T><<<grid_for<T>(n), kThreads, 0, st>>>(Lc, u, rhs, t, jr);
    return;
  }
  const ColCfg c = col_cfg(Lc.E[0], Lc.E[1], Lc.E[2], Lc.nsegs);
  k_tau<T><<<c.grid, c.block, 0, st>>>(Lc, u, rhs, t, jr, c.ntx, c.zchunk);
}

template <class T>
void launch_prolong(const Lvl& Lf, T* uf, const Lvl& Lc, const T* w, const T* t, int add,
                    cudaStream_t st) {
  const ColCfg c = col_cfg(Lf.E[0], Lf.E[1], Lf.E[2], Lf.nsegs);
  k_prolong<T><<<c.grid, c.block, 0, st>>>(Lf, uf, Lc, w, t, add, c.ntx, c.zchunk);
}

template <class T>
void launch_coarsest(const Lvl& L0, T* u, View<T> b, const T* ainv, cudaStream_t st) {
  const int n0 = L0.N[0] * L0.N[1] * L0.N[2];
  const int thr = n0 < 1024 ? ((n0 + 31) / 32) * 32 : 1024;
  k_coarsest<T><<<1, thr, 2 * n0 * sizeof(T), st>>>(L0, u, b, ainv);
}

template <class T>
void launch_pyramid(const T* ff, int nfx, int nfy, int nfz, T* fc, cudaStream_t st) {
  const long long n = (long long)(nfx / 2) * (nfy / 2) * (nfz / 2);
  const long long cap = 148LL * 16;
  const unsigned g = (unsigned)std::min<long long>(cap, (n + kThreads - 1) / kThreads);
  k_pyramid<T><<<g, kThreads, 0, st>>>(ff, nfx, nfy, nfz, fc);
}

template <class T>
void launch_resnorm(const Lvl& L, const T* u, View<T> b, double* acc, cudaStream_t st) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  const unsigned g = (unsigned)std::min<long long>(148LL * 8, (n + kThreads - 1) / kThreads);
  k_resnorm<T><<<std::max(g, 1u), kThreads, 0, st>>>(L, u, b, acc);
}

template <class T>
void launch_gather(const Lvl& L, const T* useg, T* out, const int bo[3], long long sy,
                   long long sz, cudaStream_t st) {
  const ColCfg c = col_cfg(L.S[0], L.S[1], L.S[2], L.nsegs);
  k_gather<T><<<c.grid, c.block, 0, st>>>(L, useg, out, bo[0], bo[1], bo[2], sy, sz, c.ntx,
                                          c.zchunk);
}

template <class T>
void launch_pyramid_box(View<T> f, View<T> c, const int lo[3], const int n[3], cudaStream_t st) {
  const long long cnt = (long long)n[0] * n[1] * n[2];
  if (cnt <= 0) return;
  const unsigned g = (unsigned)std::min<long long>(148LL * 8, (cnt + kThreads - 1) / kThreads);
  k_pyramid_box<T><<<std::max(g, 1u), kThreads, 0, st>>>(f, c, lo[0], lo[1], lo[2], n[0], n[1],
                                                         n[2]);
}

template <class T>
void launch_block_diff(const Lvl& La, const T* a, const T* b, const Lvl& Ld, T* dst,
                       cudaStream_t st) {
  const long long cnt = (long long)La.S[0] * La.S[1] * La.S[2];
  const unsigned g = (unsigned)std::min<long long>(148LL * 8, (cnt + kThreads - 1) / kThreads);
  k_block_diff<T><<<std::max(g, 1u), kThreads, 0, st>>>(La, a, b, Ld, dst);
}

template <class T>
void launch_box_copy(T* base, long long sy, long long sz, const int lo[3], const int n[3], T* buf,
                     int to_buf, cudaStream_t st) {
  const long long cnt = (long long)n[0] * n[1] * n[2];
  if (cnt <= 0) return;
  const unsigned g = (unsigned)std::min<long long>(148LL * 8, (cnt + kThreads - 1) / kThreads);
  k_box_copy<T><<<std::max(g, 1u), kThreads, 0, st>>>(base, sy, sz, lo[0], lo[1], lo[2], n[0],
                                                      n[1], n[2], buf, to_buf);
}

#define SRFMG_INST(T)                                                                          \
  template void launch_cheb_step<T>(const Lvl&, const T*, const T*, View<T>, T*, double, double, \
                                    int, cudaStream_t);                                        \
  template void launch_restrict<T>(const Lvl&, const T*, View<T>, const Lvl&, T*, T*, int,      \
                                   cudaStream_t, T*, View<T>);                                 \
  template void launch_tau<T>(const Lvl&, const T*, T*, T*, int, cudaStream_t);                 \
  template void launch_restrict_from_resid<T>(const Lvl&, const T*, const T*, const Lvl&, T*, T*,  \
                                              int, cudaStream_t, View<T>);                       \
  template void launch_prolong<T>(const Lvl&, T*, const Lvl&, const T*, const T*, int,          \
                                  cudaStream_t);                                               \
  template void launch_coarsest<T>(const Lvl&, T*, View<T>, const T*, cudaStream_t);            \
  template void launch_pyramid<T>(const T*, int, int, int, T*, cudaStream_t);                   \
  template void launch_resnorm<T>(const Lvl&, const T*, View<T>, double*, cudaStream_t);        \
  template void launch_gather<T>(const Lvl&, const T*, T*, const int*, long long, long long,      \
                                 cudaStream_t);                                                  \
  template void launch_box_copy<T>(T*, long long, long long, const int*, const int*, T*, int,    \
                                   cudaStream_t);                                                  \
  template void launch_pyramid_box<T>(View<T>, View<T>, const int*, const int*, cudaStream_t);    \
  template void launch_block_diff<T>(const Lvl&, const T*, const T*, const Lvl&, T*, cudaStream_t);
SRFMG_INST(double)
SRFMG_INST(float)

}  // namespace srfmg
