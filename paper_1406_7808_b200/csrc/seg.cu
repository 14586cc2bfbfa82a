// Segment-resident passes for the small SR levels (storage boxes E <= 22: C3's levels 5 and
// 6), sm_100a.  One CTA owns one segment and keeps its whole storage box in shared memory,
// so a half V-cycle visit of the level is ONE launch with a handful of block barriers
// instead of 3-4 z-marching launches of one barrier per plane each (those are latency-bound
// at these sizes: 12-37 us per launch for 2-44 MB of data):
//
//   DOWN   [u = Pi(w) on C ∪ GSR, S^1]   FMG entry (fig:fmgsr L221-222)         src = PSET
//          [b = R + A u on F, A u on C \ F, t = u]   tau (Eq. 4)       tau = 1
//          S^2 on C                                 pre-smoothing (L232)
//          r = b - A u on C; u_{l-1} = avg8(u), R = avg8(r) on F (or V_T)     (L233, L235)
//   UP     u += P(w - t) on C ∪ GSR                 correction (L241, R17)
//          S^2 on C                                 post-smoothing (L242)
//
// Same arithmetic plan as the other kernels: A = -Lap_h (7 points) with reflected ghosts,
// storage cells outside Omega are zero and count +1 on the diagonal (R3); Chebyshev R8; the
// 8-child averages R9; cell-centred trilinear prolongation with reflected coarse ghosts R10.
// The thread layout is one (x, y) storage column per thread, marching z, every operator
// application reading its x / y neighbours from shared memory.
#include <algorithm>
#include <cstdio>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

template <class T>
struct SegArgs {
  Lvl L, Lc, Lw;      // fine SR level, coarse level (restriction target), coarse source of
                      // the interpolation (Lc, or the wider-ghosted footprint copy of level T)
  const T* uin;       // fine u (segment storage)
  T* uout;            // fine u written (may equal uin: one CTA owns its segment)
  FusedRhs<T> rhs;    // b: dense f_l (global == 1) or segment storage
  const T* R;         // tau: restricted residual on F (segment storage, rres)
  T* rhs_out;         // tau: rhs written (segment storage)
  T* t_out;           // tau: t = u written
  int jt;             // tau: F half-width on this level (floor(J_{l+1}/2))
  const T* w;         // PSET / UP: coarse u (segment storage or level-T array)
  const T* t;         // UP: coarse t
  T* uc;              // DOWN: coarse u (written on the restriction targets)
  T* rc;              // DOWN: coarse R
  int jr;             // DOWN: restriction half-width (0: V_T at k = 1)
  int src;            // DOWN: 0 = load u, 1 = u = Pi(w) then S^1
  int tau;            // DOWN: tau in front
  T c1;               // S^1: 1/theta
  T c0, cm, cr;       // S^2: 1/theta, rho1 rho0, 2 rho1 / delta
};

template <class T, int E, int PY>
struct SG {
  static constexpr int NT = (E * E + 31) / 32 * 32;
  static constexpr int BOX = E * E * PY;             // elements of the storage box
  static constexpr int BUF = (BOX + 31) / 32 * 32;
  // u0, u1 and (when it fits) b in shared memory
  static constexpr bool BSM = (size_t)3 * BUF * sizeof(T) <= 200 * 1024;
  static constexpr size_t SMEM = (size_t)(BSM ? 3 : 2) * BUF * sizeof(T) + 16;
};

// (A u)_i * 1/h^2 terms: r = b - (d u - sum) / h^2
template <class T, int E, int PY>
__device__ __forceinline__ T resid_at(const T* __restrict__ u, int o, T b, T d, T ih2) {
  constexpr int PZ = E * PY;
  const T c = u[o];
  const T sum = ((u[o - PZ] + u[o + PZ]) + (u[o - PY] + u[o + PY])) + (u[o - 1] + u[o + 1]);
  return b - (d * c - sum) * ih2;
}

template <class T, int E, int PY, bool UP>
__global__ void __launch_bounds__(SG<T, E, PY>::NT) k_seg(const __grid_constant__ SegArgs<T> a) {
  using G = SG<T, E, PY>;
  constexpr int PZ = E * PY;
  extern __shared__ __align__(128) unsigned char sm[];
  T* u0 = reinterpret_cast<T*>(sm);
  T* u1 = u0 + G::BUF;
  T* bs = G::BSM ? u1 + G::BUF : nullptr;
  uint64_t* bar = reinterpret_cast<uint64_t*>(u1 + (G::BSM ? 2 : 1) * G::BUF);
  const Lvl& L = a.L;
  const Lvl& Lc = a.Lc;
  const int s = blockIdx.x;
  const int p[3] = {s % L.ns[0] + L.so[0], (s / L.ns[0]) % L.ns[1] + L.so[1],
                    s / (L.ns[0] * L.ns[1]) + L.so[2]};
  const int o[3] = {p[0] * L.S[0] - (L.J + 1), p[1] * L.S[1] - (L.J + 1),
                    p[2] * L.S[2] - (L.J + 1)};
  const T* useg = a.uin + (long long)s * L.ss;
  T* oseg = a.uout + (long long)s * L.ss;
  const bool load_u = UP || a.src == 0;
  // ---- stage the box: u by one bulk copy (the segment storage is contiguous), b likewise
  // when it is segment storage, else by rows of the dense f
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const bool bseg = !a.rhs.global;
  const T* bseg_p = bseg ? a.rhs.p + (long long)s * L.ss : nullptr;
  if (threadIdx.x == 0) {
    uint32_t bytes = 0;
    if (load_u) bytes += G::BOX * sizeof(T);
    if (G::BSM && bseg && !a.tau) bytes += G::BOX * sizeof(T);
    if (G::BSM && a.tau) bytes += G::BOX * sizeof(T);  // R (the tau forms b from it)
    if (bytes) {
      mbar_expect_tx(bar, bytes);
      if (load_u) bulk_g2s(u0, useg, G::BOX * sizeof(T), bar);
      if (G::BSM && a.tau)
        bulk_g2s(bs, a.R + (long long)s * L.ss, G::BOX * sizeof(T), bar);
      else if (G::BSM && bseg)
        bulk_g2s(bs, bseg_p, G::BOX * sizeof(T), bar);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    }
  }
  // this thread's column
  const int tx = threadIdx.x % E, ty = threadIdx.x / E;
  const bool col = threadIdx.x < E * E;
  const int gx = o[0] + tx, gy = o[1] + ty;
  const bool inxy = col && gx >= 0 && gx < L.N[0] && gy >= 0 && gy < L.N[1];
  const bool cxy = inxy && tx >= 1 && tx <= E - 2 && ty >= 1 && ty <= E - 2;
  const int dxy = 6 + (gx == 0) + (gx == L.N[0] - 1) + (gy == 0) + (gy == L.N[1] - 1);
  const T ih2 = T(L.inv_h2);
  auto in_z = [&](int z) { return o[2] + z >= 0 && o[2] + z < L.N[2]; };
  auto c_z = [&](int z) { return z >= 1 && z <= E - 2 && in_z(z); };
  auto dd = [&](int z) {
    const int gz = o[2] + z;
    return T(dxy + (gz == 0) + (gz == L.N[2] - 1));
  };
  // dense rhs: virtual-origin view p (global indexing); staged into bs when it fits, one
  // column per thread with all of its loads in flight
  const long long fsy = a.rhs.dims[0], fsz = (long long)a.rhs.dims[0] * a.rhs.dims[1];
  if (!bseg && G::BSM && col) {
    T v[E];
#pragma unroll
    for (int z = 0; z < E; ++z)
      v[z] = (inxy && in_z(z)) ? a.rhs.p[(long long)(o[2] + z) * fsz + (long long)gy * fsy + gx]
                               : T(0);
#pragma unroll
    for (int z = 0; z < E; ++z) bs[z * PZ + ty * PY + tx] = v[z];
  }
  auto bval = [&](int z) -> T {  // rhs at (tx, ty, z) of a C cell
    const int oo = z * PZ + ty * PY + tx;
    if (G::BSM) return bs[oo];
    if (a.tau) return a.rhs_out[(long long)s * L.ss + oo];
    if (bseg) return bseg_p[oo];
    return a.rhs.p[(long long)(o[2] + z) * fsz + (long long)gy * fsy + gx];
  };
  mbar_wait(bar, 0);
  // coarse level: the segment's own coarse storage, or the single level-T array (block)
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  const int pc[3] = {cs % Lc.ns[0] + Lc.so[0], (cs / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
                     cs / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2]};
  const int oc[3] = {pc[0] * Lc.S[0] - (Lc.J + 1), pc[1] * Lc.S[1] - (Lc.J + 1),
                     pc[2] * Lc.S[2] - (Lc.J + 1)};
  if (UP || a.src == 1) {
    // u (+)= P(w - t) on C ∪ GSR (storage ∩ Omega); u = 0 elsewhere for PSET.  The coarse
    // footprint (parents of the box +-1, folded into the domain: R3 reflection reads mirror
    // cells) is staged first into the free u1 buffer, w - t per coarse cell, one coarse
    // column per thread with its loads in flight
    const Lvl& Lw = a.Lw;  // layout of w (Lc, or the footprint copy of level T)
    const int ow[3] = {pc[0] * Lw.S[0] - (Lw.J + 1), pc[1] * Lw.S[1] - (Lw.J + 1),
                       pc[2] * Lw.S[2] - (Lw.J + 1)};
    constexpr int CB = E / 2 + 3;
    int cb[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) cb[d] = max((o[d] >> 1) - 1, 0);
    T* cw = u1;
    if (threadIdx.x < CB * CB) {
      const int X = cb[0] + threadIdx.x % CB, Y = cb[1] + threadIdx.x / CB;
      // (cells of the staged box outside Omega or outside w's storage box are never used)
      const bool okxy = X < Lw.N[0] && Y < Lw.N[1] && X - ow[0] >= 0 && X - ow[0] < Lw.E[0] &&
                        Y - ow[1] >= 0 && Y - ow[1] < Lw.E[1];
      const long long r = (long long)cs * Lw.ss + (long long)(Y - ow[1]) * Lw.py + (X - ow[0]);
      T v[CB];
#pragma unroll
      for (int k = 0; k < CB; ++k) {
        const int Z = cb[2] + k;
        v[k] = T(0);
        if (okxy && Z < Lw.N[2] && Z - ow[2] >= 0 && Z - ow[2] < Lw.E[2]) {
          const long long q = r + (long long)(Z - ow[2]) * Lw.pz;
          v[k] = UP ? a.w[q] - a.t[q] : a.w[q];
        }
      }
#pragma unroll
      for (int k = 0; k < CB; ++k) cw[(k * CB + threadIdx.x / CB) * CB + threadIdx.x % CB] = v[k];
    }
    if (!UP)
      for (int i = threadIdx.x; i < G::BOX; i += G::NT) u0[i] = T(0);  // (incl. the padding)
    __syncthreads();
    if (col) {
      // x / y: parent and neighbour (reflected: mirror cell, negative weight), box-local
      int Px[2], Py[2];
      T sx = T(1), sy = T(1);
      {
        const int P = gx >> 1, Q = P + ((gx & 1) ? 1 : -1);
        int Qm = Q;
        if (Q < 0) { Qm = 0; sx = T(-1); }
        if (Q >= Lw.N[0]) { Qm = Lw.N[0] - 1; sx = T(-1); }
        Px[0] = P - cb[0];
        Px[1] = Qm - cb[0];
      }
      {
        const int P = gy >> 1, Q = P + ((gy & 1) ? 1 : -1);
        int Qm = Q;
        if (Q < 0) { Qm = 0; sy = T(-1); }
        if (Q >= Lw.N[1]) { Qm = Lw.N[1] - 1; sy = T(-1); }
        Py[0] = P - cb[1];
        Py[1] = Qm - cb[1];
      }
      const T W0 = T(0.75), W1 = T(0.25);
      auto ixy = [&](int Z) {  // xy-interpolant of coarse plane Z (global), reflected in z
        T sz = T(1);
        if (Z < 0) { Z = 0; sz = T(-1); }
        if (Z >= Lw.N[2]) { Z = Lw.N[2] - 1; sz = T(-1); }
        const T* pl = cw + (Z - cb[2]) * CB * CB;
        const T r0 = W0 * pl[Py[0] * CB + Px[0]] + (W1 * sx) * pl[Py[0] * CB + Px[1]];
        const T r1 = W0 * pl[Py[1] * CB + Px[0]] + (W1 * sx) * pl[Py[1] * CB + Px[1]];
        return sz * (W0 * r0 + (W1 * sy) * r1);
      };
#pragma unroll
      for (int z = 0; z < E; ++z) {
        const int oo = z * PZ + ty * PY + tx;
        if (inxy && in_z(z)) {
          const int gz = o[2] + z;
          const int Pz = gz >> 1, Qz = Pz + ((gz & 1) ? 1 : -1);
          const T v = W0 * ixy(Pz) + W1 * ixy(Qz);
          u0[oo] = UP ? u0[oo] + v : v;
        }
      }
    }
    __syncthreads();
    if (!UP) {  // S^1 (alpha = 1): u1 = u0 + (b - A u0)/theta on C, then back into u0
      if (col)
#pragma unroll
        for (int z = 0; z < E; ++z) {
          const int oo = z * PZ + ty * PY + tx;
          u1[oo] = (cxy && c_z(z)) ? u0[oo] + a.c1 * resid_at<T, E, PY>(u0, oo, bval(z), dd(z), ih2)
                                   : u0[oo];
        }
      __syncthreads();
      T* tmp = u0;
      u0 = u1;
      u1 = tmp;
    }
  }
  if (!UP && a.tau) {
    // Eq. 4: b = R + A u on F, A u on C \ F; t = u (whole box)
    const int jt = a.jt;
    const bool fxy = gx >= p[0] * L.S[0] - jt && gx < (p[0] + 1) * L.S[0] + jt &&
                     gy >= p[1] * L.S[1] - jt && gy < (p[1] + 1) * L.S[1] + jt;
    T* rg = a.rhs_out + (long long)s * L.ss;
    T* tg = a.t_out + (long long)s * L.ss;
    if (col)
      for (int z = 0; z < E; ++z) {
        const int oo = z * PZ + ty * PY + tx;
        const int gz = o[2] + z;
        T rv = G::BSM ? bs[oo] : a.R[(long long)s * L.ss + oo];
        if (cxy && c_z(z)) {
          const T Au = -resid_at<T, E, PY>(u0, oo, T(0), dd(z), ih2);
          const bool inF = fxy && gz >= p[2] * L.S[2] - jt && gz < (p[2] + 1) * L.S[2] + jt;
          rv = inF ? rv + Au : Au;
        }
        if (G::BSM) bs[oo] = rv;
        if (inxy && in_z(z)) tg[oo] = u0[oo];
        rg[oo] = rv;  // (outside C: R unchanged, as the separate tau kernel leaves it)
      }
    __syncthreads();
  }
  // ---- S^2: u1 = u0 + c0 r(u0); u2 = u1 + cm (u1 - u0) + cr r(u1), into u0 in place
  if (col)
#pragma unroll
    for (int z = 0; z < E; ++z) {
      const int oo = z * PZ + ty * PY + tx;
      u1[oo] = (cxy && c_z(z)) ? u0[oo] + a.c0 * resid_at<T, E, PY>(u0, oo, bval(z), dd(z), ih2)
                               : u0[oo];
    }
  __syncthreads();
  if (col)
#pragma unroll
    for (int z = 0; z < E; ++z) {
      const int oo = z * PZ + ty * PY + tx;
      if (cxy && c_z(z)) {
        const T c1 = u1[oo];
        u0[oo] = c1 + a.cm * (c1 - u0[oo]) + a.cr * resid_at<T, E, PY>(u1, oo, bval(z), dd(z), ih2);
      }
    }
  __syncthreads();
  // ---- u out (whole box: C smoothed, GSR unchanged, zero outside Omega), coalesced
  for (int i = threadIdx.x; i < G::BOX; i += G::NT) oseg[i] = u0[i];
  if (UP) return;
  // ---- residual on C into u1, then the 8-child averages onto the restriction targets
  if (col)
#pragma unroll
    for (int z = 0; z < E; ++z) {
      const int oo = z * PZ + ty * PY + tx;
      u1[oo] = (cxy && c_z(z)) ? resid_at<T, E, PY>(u0, oo, bval(z), dd(z), ih2) : T(0);
    }
  __syncthreads();
  const int jr = a.jr;
  const int B0 = L.S[0] / 2 + 2 * jr, B1 = L.S[1] / 2 + 2 * jr, B2 = L.S[2] / 2 + 2 * jr;
  for (int i = threadIdx.x; i < B0 * B1 * B2; i += G::NT) {
    const int X = p[0] * (L.S[0] / 2) - jr + i % B0;
    const int Y = p[1] * (L.S[1] / 2) - jr + (i / B0) % B1;
    const int Z = p[2] * (L.S[2] / 2) - jr + i / (B0 * B1);
    if (X < 0 || X >= Lc.N[0] || Y < 0 || Y >= Lc.N[1] || Z < 0 || Z >= Lc.N[2]) continue;
    const int f0 = (2 * Z - o[2]) * PZ + (2 * Y - o[1]) * PY + (2 * X - o[0]);
    T su = T(0), sr = T(0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int oo = f0 + (c >> 2) * PZ + ((c >> 1) & 1) * PY + (c & 1);
      su += u0[oo];
      sr += u1[oo];
    }
    const long long co = (long long)cs * Lc.ss + (long long)(Z - oc[2]) * Lc.pz +
                         (long long)(Y - oc[1]) * Lc.py + (X - oc[0]);
    a.uc[co] = su * T(0.125);
    a.rc[co] = sr * T(0.125);
  }
}

template <class T, int E, int PY, bool UP>
bool launch_one(const SegArgs<T>& a, cudaStream_t st) {
  using G = SG<T, E, PY>;
  if (a.L.E[0] != E || a.L.E[1] != E || a.L.E[2] != E || a.L.py != PY || a.L.pz != E * PY)
    return false;
  auto kern = k_seg<T, E, PY, UP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  kern<<<a.L.nsegs, G::NT, G::SMEM, st>>>(a);
  return true;
}

// E = 14 / 22 boxes (8^3 / 16^3 segments with J = 2): row pitch 16 / 24 in fp64 and fp32
template <class T, bool UP>
bool dispatch(const SegArgs<T>& a, cudaStream_t st) {
  return launch_one<T, 14, 16, UP>(a, st) || launch_one<T, 22, 24, UP>(a, st);
}

}  // namespace

template <class T>
bool seg_ok(const Lvl& L) {
  const bool cube = L.E[0] == L.E[1] && L.E[1] == L.E[2];
  return cube && L.pz == (long long)L.E[0] * L.py &&
         ((L.E[0] == 14 && L.py == 16) || (L.E[0] == 22 && L.py == 24)) && !L.st27 &&
         L.nlg == 0.0;
}

template <class T>
bool launch_seg_down(const Lvl& L, const Lvl& Lc, const Lvl& Lw, const T* uin, T* uout,
                     FusedRhs<T> b, const T* R, T* rhs_out, T* t_out, int jt, const T* w, T* uc,
                     T* rc, int jr, int src, double c1, double c0, double cm, double cr,
                     cudaStream_t st) {
  SegArgs<T> a{};
  a.L = L;
  a.Lc = Lc;
  a.Lw = Lw;
  a.uin = uin;
  a.uout = uout;
  a.rhs = b;
  a.R = R;
  a.rhs_out = rhs_out;
  a.t_out = t_out;
  a.jt = jt;
  a.tau = R != nullptr;
  a.w = w;
  a.uc = uc;
  a.rc = rc;
  a.jr = jr;
  a.src = src;
  a.c1 = (T)c1;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  return dispatch<T, false>(a, st);
}

template <class T>
bool launch_seg_up(const Lvl& L, const Lvl& Lc, const T* uin, T* uout, FusedRhs<T> b, const T* w,
                   const T* t, double c0, double cm, double cr, cudaStream_t st) {
  SegArgs<T> a{};
  a.L = L;
  a.Lc = Lc;
  a.Lw = Lc;
  a.uin = uin;
  a.uout = uout;
  a.rhs = b;
  a.w = w;
  a.t = t;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  return dispatch<T, true>(a, st);
}

template bool seg_ok<double>(const Lvl&);
template bool seg_ok<float>(const Lvl&);
template bool launch_seg_down<double>(const Lvl&, const Lvl&, const Lvl&, const double*, double*,
                                      FusedRhs<double>, const double*, double*, double*, int,
                                      const double*, double*, double*, int, int, double, double,
                                      double, double, cudaStream_t);
template bool launch_seg_down<float>(const Lvl&, const Lvl&, const Lvl&, const float*, float*,
                                     FusedRhs<float>,
                                     const float*, float*, float*, int, const float*, float*,
                                     float*, int, int, double, double, double, double,
                                     cudaStream_t);
template bool launch_seg_up<double>(const Lvl&, const Lvl&, const double*, double*,
                                    FusedRhs<double>, const double*, const double*, double,
                                    double, double, cudaStream_t);
template bool launch_seg_up<float>(const Lvl&, const Lvl&, const float*, float*, FusedRhs<float>,
                                   const float*, const float*, double, double, double,
                                   cudaStream_t);

}  // namespace srfmg
