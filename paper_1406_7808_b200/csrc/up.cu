// Up half of an SR V-cycle visit in one HBM pass: the coarse-grid correction
// u += P(w - t) (fig:mgvsr L241, R10) followed by the degree-2 Chebyshev post-smoothing
// S^nu2 (L242, R8), sm_100a.
//
// The plane-marching plan of k_cheb2s (fused.cu): one CTA per y-band of one segment, the u
// rows and the rhs streamed into shared-memory rings by one thread (cp.async.bulk / TMA),
// stage 1 at plane z and stage 2 at plane z-1 with register z-queues, ONE __syncthreads per
// plane.  The correction is applied to each u plane when it is consumed:
//   * the coarse rows of w and t the band needs are bulk-copied into a 2-plane ring;
//   * once per coarse plane the CTA forms Xi = the x-interpolant of (w - t) at fine x
//     resolution and coarse y (reflected ghosts as signed weights, 0 outside Omega) into a
//     3-plane shared-memory ring, two fine planes ahead of its first use;
//   * a fine plane's correction is then 4 shared-memory reads per cell (two coarse rows of
//     two coarse planes); every loaded row of the plane is corrected in place (the rows of
//     the band and its two halo rows by their owner threads, the outermost margin rows by
//     the first and last thread groups), so stage 1 sees the corrected u everywhere.
// Output as k_cheb2s: C smoothed, GSR the corrected u, or (last pass of the solve) the
// genuine cells into the user's u.
//
// Replaces prolong(ADD) + cheb(2): one read and one write of u fewer per level visit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

template <class T>
struct UpArgs {
  Lvl L, Lc;
  const T* uin;
  T* uout;
  const T* rhs_seg;  // segment-storage rhs (RG = 0)
  const T* w;        // coarse u
  const T* t;        // coarse t snapshot
  T c0, cm, cr;
  FinalOut<T> fin;
  int foff[3];
  int cpl;           // elements per staged coarse plane, per array
};

template <class T, int PY, int BH, int MAXS, int RG>
struct UGeom {
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FP = RG ? PY + kAl : PY;
  static constexpr int NG = (BH + 2 + MAXS - 1) / MAXS;
  static constexpr int NT = PY * NG;
  static constexpr int A = 128 / (int)sizeof(T);
  static constexpr int TR = NG * MAXS;
  static constexpr int U0S = ((TR + 2) * PY + A - 1) / A * A;
  static constexpr int FS = (TR * FP + A - 1) / A * A;
  static constexpr int U1S = U0S;
  static constexpr int RU = 3, RF = 4, NU1 = 3, RC = 2, NXI = 3;
  static constexpr int CROWS = (TR + 2) / 2 + 3;
  static constexpr int XIS = (CROWS * PY + A - 1) / A * A;
  static size_t smem(int cpl) {
    return (size_t)(RU * U0S + RF * FS + NU1 * U1S + NXI * XIS + RC * 2 * cpl) * sizeof(T) +
           8 * (RU + RF + RC);
  }
};

// bit k of m ? a : b as a predicated select (both operands computed first)
__device__ __forceinline__ double selp_(bool p, double a, double b) {
  double r;
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n selp.f64 %0, %1, %2, q;\n}"
      : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)p));
  return r;
}
__device__ __forceinline__ float selp_(bool p, float a, float b) {
  float r;
  asm("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n selp.f32 %0, %1, %2, q;\n}"
      : "=f"(r) : "f"(a), "f"(b), "r"((unsigned)p));
  return r;
}

template <class T, int PY, int BH, int MAXS, int RG, int FIN, int NB>
__global__ void __launch_bounds__(UGeom<T, PY, BH, MAXS, RG>::NT, NB)
    k_up2s(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ UpArgs<T> a) {
  using G = UGeom<T, PY, BH, MAXS, RG>;
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const Lvl& Lc = a.Lc;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + G::RU * G::U0S;
  T* u1s = fs + G::RF * G::FS;
  T* xis = u1s + G::NU1 * G::U1S;
  T* cws = xis + G::NXI * G::XIS;  // [RC][2][cpl]: w then t per slot
  uint64_t* bars = reinterpret_cast<uint64_t*>(cws + G::RC * 2 * a.cpl);  // u0, f, coarse

  const int px = s % L.ns[0] + L.so[0];
  const int pyy = (s / L.ns[0]) % L.ns[1] + L.so[1];
  const int pzz = s / (L.ns[0] * L.ns[1]) + L.so[2];
  const int ox = px * L.S[0] - (L.J + 1);
  const int oy = pyy * L.S[1] - (L.J + 1);
  const int oz = pzz * L.S[2] - (L.J + 1);
  const T* useg = a.uin + (long long)s * L.ss;
  T* oseg = a.uout + (long long)s * L.ss;
  const T* rseg = RG ? nullptr : a.rhs_seg + (long long)s * L.ss;
  const uint32_t u0_bytes = (uint32_t)((q1 - q0) * PY * sizeof(T));
  const int oxt = ox - a.foff[0];
  const int oxa = oxt & ~(G::kAl - 1);
  const int fsh = RG ? oxt - oxa : 0;
  const uint32_t f_bytes = RG ? (uint32_t)((BH + 2) * G::FP * sizeof(T))
                              : (uint32_t)((s1 - s0) * PY * sizeof(T));
  // coarse source (the segment's own coarse storage, or the level-T array at k = 1)
  const int cseg = Lc.nsegs == 1 ? 0 : s;
  const int cpx = cseg % Lc.ns[0] + Lc.so[0], cpy = (cseg / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
            cpz = cseg / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
  const int ocx = cpx * Lc.S[0] - (Lc.J + 1), ocy = cpy * Lc.S[1] - (Lc.J + 1),
            ocz = cpz * Lc.S[2] - (Lc.J + 1);
  const int cy_lo = max(max(((oy + q0) >> 1) - 1, 0), ocy);
  const int cy_hi = min(min(((oy + q1 - 1) >> 1) + 1, Lc.N[1] - 1), ocy + Lc.E[1] - 1);
  const int ncr = cy_hi - cy_lo + 1;
  const int gz_lo = max(oz, 0), gz_hi = min(oz + Ez, L.N[2]) - 1;
  const int cz_lo = max(max((gz_lo >> 1) - 1, 0), ocz);
  const int cz_hi = min(min((gz_hi >> 1) + 1, Lc.N[2] - 1), ocz + Lc.E[2] - 1);
  const uint32_t cbytes = (uint32_t)(ncr * Lc.py * sizeof(T));
  const long long cofs = (long long)cseg * Lc.ss + (long long)(cy_lo - ocy) * Lc.py;

  if (threadIdx.x == 0) {
    for (int i = 0; i < G::RU + G::RF + G::RC; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_u0 = [=](int z) {
    const int sl = z % G::RU;
    mbar_expect_tx(&bars[sl], u0_bytes);
    bulk_g2s(u0s + sl * G::U0S + (q0 - s0 + 1) * PY, useg + (long long)z * pz + (long long)q0 * PY,
             u0_bytes, &bars[sl]);
  };
  auto issue_f = [=, &fmap](int z) {
    const int sl = z % G::RF;
    mbar_expect_tx(&bars[G::RU + sl], f_bytes);
    if (RG)
      tma_3d(fs + sl * G::FS, &fmap, oxa, oy + s0 - a.foff[1], oz + z - a.foff[2],
             &bars[G::RU + sl]);
    else
      bulk_g2s(fs + sl * G::FS, rseg + (long long)z * pz + (long long)s0 * PY, f_bytes,
               &bars[G::RU + sl]);
  };
  uint64_t* cbar = bars + G::RU + G::RF;
  auto issue_c = [&](int c) {  // w and t rows of coarse plane c into slot (c - cz_lo) & 1
    const int n = c - cz_lo, sl = n & 1;
    if (n >= 2) mbar_wait(&cbar[sl], ((n - 2) >> 1) & 1);  // the previous copy has landed
    mbar_expect_tx(&cbar[sl], 2 * cbytes);
    const long long o = cofs + (long long)(c - ocz) * Lc.pz;
    bulk_g2s(cws + (2 * sl) * a.cpl, a.w + o, cbytes, &cbar[sl]);
    bulk_g2s(cws + (2 * sl + 1) * a.cpl, a.t + o, cbytes, &cbar[sl]);
  };
  int nc = cz_lo;  // next coarse plane to stage (thread 0)
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    for (int z = 0; z < min(3, Ez); ++z) issue_f(z);
    for (; nc <= min(cz_hi, cz_lo + 1); ++nc) issue_c(nc);
  }

  constexpr T W0 = T(0.75), W1 = T(0.25);
  // Xi of coarse plane c: x-interpolant of (w - t), rows cy_lo.., fine columns (R10, R3)
  auto build_xi = [&](int c) {
    const int n = c - cz_lo, sl = n & 1;
    mbar_wait(&cbar[sl], (n >> 1) & 1);
    const T* sw = cws + (2 * sl) * a.cpl;
    const T* st = sw + a.cpl;
    T* xi = xis + (c % G::NXI) * G::XIS;
    for (int e = threadIdx.x; e < ncr * PY; e += G::NT) {
      const int m = e / PY, x = e - m * PY;
      const int gx = ox + x;
      T v = T(0);
      if (x < Ex && gx >= 0 && gx < L.N[0]) {
        const int X = gx >> 1;
        int Xq = X + ((gx & 1) ? 1 : -1);
        T w1 = W1;
        if (Xq < 0) { Xq = 0; w1 = -W1; }
        if (Xq >= Lc.N[0]) { Xq = Lc.N[0] - 1; w1 = -W1; }
        const int o0 = m * Lc.py + min(max(X - ocx, 0), Lc.E[0] - 1);
        const int o1 = m * Lc.py + min(max(Xq - ocx, 0), Lc.E[0] - 1);
        v = W0 * (sw[o0] - st[o0]) + w1 * (sw[o1] - st[o1]);
      }
      xi[e] = v;
    }
  };

  const int tx = threadIdx.x % PY, g = threadIdx.x / PY;
  const int y0 = s0 + g * MAXS;
  const int gxv = ox + tx;
  const bool tok = tx < Ex && y0 < s1;
  const bool tin = tok && gxv >= 0 && gxv < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const int dxo = (gxv == 0 ? 1 : 0) + (gxv == L.N[0] - 1 ? 1 : 0);
  unsigned ld_mask = 0, c_mask = 0, w_mask = 0, yb_mask = 0, rw_mask = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k;
    const int gy = oy + y;
    if (y >= r0 && y < r1) rw_mask |= 1u << k;
    const bool in = tin && y < s1 && gy >= 0 && gy < L.N[1];
    if (tok && y < q1) ld_mask |= 1u << k;
    if (in && tcx && y >= 1 && y <= Ey - 2) c_mask |= 1u << k;
    if (in && y >= r0 && y < r1) w_mask |= 1u << k;
    yb_mask |= (unsigned)((gy == 0 ? 1 : 0) + (gy == L.N[1] - 1 ? 1 : 0)) << (2 * k);
  }
  // correction rows: code = m0 | m1 << 8 | neg << 16 | valid << 17 (coarse rows in Xi)
  auto ycode = [&](int y) -> unsigned {
    const int gy = oy + y;
    if (y < q0 || y >= q1 || gy < 0 || gy >= L.N[1] || tx >= PY) return 0u;
    const int Y = gy >> 1;
    int Yq = Y + ((gy & 1) ? 1 : -1);
    unsigned neg = 0;
    if (Yq < 0) { Yq = 0; neg = 1; }
    if (Yq >= Lc.N[1]) { Yq = Lc.N[1] - 1; neg = 1; }
    const unsigned m0 = (unsigned)min(max(Y - cy_lo, 0), ncr - 1);
    const unsigned m1 = (unsigned)min(max(Yq - cy_lo, 0), ncr - 1);
    return m0 | (m1 << 8) | (neg << 16) | (1u << 17);
  };
  unsigned yc[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) yc[k] = ((ld_mask >> k) & 1u) ? ycode(y0 + k) : 0u;
  // the outermost loaded rows that no thread owns: above the first thread row (group 0) and
  // below the last (group NG-1)
  const int ymarg = (g == 0) ? s0 - 1 : (g == G::NG - 1 ? s0 + G::TR : -1000);
  const unsigned mcode = (ymarg >= 0 && tx < Ex) ? ycode(ymarg) : 0u;
  const int moff = (g == 0) ? -PY : MAXS * PY;  // smem offset of the margin row from u0b
  auto corr = [&](unsigned code, const T* xp, const T* xq, T wq) -> T {
    const int m0 = code & 0xff, m1 = (code >> 8) & 0xff;
    const T wy = (code >> 16) & 1u ? -W1 : W1;
    const T ap = W0 * xp[m0 * PY] + wy * xp[m1 * PY];
    const T aq = W0 * xq[m0 * PY] + wy * xq[m1 * PY];
    const T v = W0 * ap + wq * aq;
    return selp_(((code >> 17) & 1u) != 0, v, T(0));
  };
  // Xi slots and z weight of fine plane gz (in Omega): P = gz >> 1, Q = P +- 1 (reflected)
  auto zplanes = [&](int gz, const T*& xp, const T*& xq, T& wq) {
    const int P = gz >> 1;
    int Q = P + ((gz & 1) ? 1 : -1);
    wq = W1;
    if (Q < 0) { Q = 0; wq = -W1; }
    if (Q >= Lc.N[2]) { Q = Lc.N[2] - 1; wq = -W1; }
    // (both lie in the coarse storage box for every cell of C u GSR; the clamp only keeps
    // dead cells on built planes)
    const int Pc = min(max(P, cz_lo), cz_hi), Qc = min(max(Q, cz_lo), cz_hi);
    xp = xis + (Pc % G::NXI) * G::XIS + tx;
    xq = xis + (Qc % G::NXI) * G::XIS + tx;
  };

  T dk[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) dk[k] = T(6 + dxo) + T((yb_mask >> (2 * k)) & 3u);
  unsigned gen_mask = 0;
  T* fbase = nullptr;
  if constexpr (FIN == 1) {
    const int vlo = L.J + 1;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const int y = y0 + k;
      if (((w_mask >> k) & 1u) && tx >= vlo && tx < vlo + L.S[0] && y >= vlo && y < vlo + L.S[1])
        gen_mask |= 1u << k;
    }
    fbase = a.fin.p + (long long)(oy + y0 - a.fin.bo[1]) * a.fin.sy + (gxv - a.fin.bo[0]);
  }
  T* const u0b = u0s + (y0 - s0 + 1) * PY + tx;
  const T* const fb = fs + (y0 - s0) * G::FP + tx + fsh;
  T* const u1b = u1s + (y0 - s0 + 1) * PY + tx;
  T* const ob = oseg + (long long)y0 * PY + tx;
  T u0q[MAXS][3], u1q[MAXS][3];

  // prologue: Xi of the coarse planes fine planes gz_lo, gz_lo + 1 use, then plane 0
  int built = cz_lo - 1;
  {
    const int cb0 = max(cz_lo, ((gz_lo + 1) >> 1) - 1);
    const int cb1 = min(cz_hi, (gz_lo + 2) >> 1);
    for (int c = cz_lo; c <= cb1; ++c) {
      if (c >= cb0) build_xi(c);
      __syncthreads();
      if (threadIdx.x == 0)
        for (; nc <= cz_hi && nc <= c + 2; ++nc) issue_c(nc);
      built = c;
    }
  }
  mbar_wait(&bars[0], 0);
  {
    const int gz = oz;
    const bool zin = gz >= gz_lo && gz <= gz_hi;
    const T* xp = xis;
    const T* xq = xis;
    T wq = W1;
    if (zin) zplanes(gz, xp, xq, wq);
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      T v = ((ld_mask >> k) & 1u) ? u0b[k * PY] : T(0);
      if (zin && ((ld_mask >> k) & 1u)) {
        v += corr(yc[k], xp, xq, wq);
        u0b[k * PY] = v;
      }
      u0q[k][0] = v;
      u0q[k][1] = u0q[k][2] = T(0);
      u1q[k][0] = u1q[k][1] = u1q[k][2] = T(0);
    }
    if (zin && mcode) u0b[moff] += corr(mcode, xp, xq, wq);
  }
  __syncthreads();
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0, cm = a.cm, cr = a.cr;

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;
    constexpr int IM = (R + 2) % 3, I0 = R, IP = (R + 1) % 3;
    if (z < Ez) {
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % G::RU], ((z + 1) / G::RU) & 1);
      mbar_wait(&bars[G::RU + z % G::RF], (z / G::RF) & 1);
      const T* pl = u0b + (z % G::RU) * G::U0S;
      T* pn = u0b + ((z + 1) % G::RU) * G::U0S;
      const T* fp = fb + (z % G::RF) * G::FS;
      T* u1w = u1b + R * G::U1S;
      const int gz = oz + z;
      const bool zc = gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2;
      const T dz = (gz == 0 ? T(1) : T(0)) + (gz == L.N[2] - 1 ? T(1) : T(0));
      // plane z+1: corrected in place (own rows, margin row), into the register queue
      {
        const int gn = gz + 1;
        const bool zin = z + 1 < Ez && gn >= gz_lo && gn <= gz_hi;
        const T* xp = xis;
        const T* xq = xis;
        T wq = W1;
        if (zin) zplanes(gn, xp, xq, wq);
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          T v = (z + 1 < Ez) ? pn[k * PY] : T(0);
          if (zin && ((ld_mask >> k) & 1u)) {
            v += corr(yc[k], xp, xq, wq);
            pn[k * PY] = v;
          }
          u0q[k][IP] = v;
        }
        if (zin && mcode) pn[moff] += corr(mcode, xp, xq, wq);
      }
      const unsigned act = zc ? c_mask : 0u;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        const T v0 = u0q[k][I0];
        const T ym = (k == 0) ? pl[-PY] : u0q[k > 0 ? k - 1 : 0][I0];
        const T yp = (k == MAXS - 1) ? pl[MAXS * PY] : u0q[k + 1 < MAXS ? k + 1 : k][I0];
        const T sum = ((u0q[k][IM] + u0q[k][IP]) + (ym + yp)) + (pl[k * PY - 1] + pl[k * PY + 1]);
        const T r = fp[k * G::FP] - ((dk[k] + dz) * v0 - sum) * ih2;
        const T v1 = ((act >> k) & 1u) ? v0 + c0 * r : v0;
        u1q[k][I0] = v1;
        u1w[k * PY] = v1;
      }
      // Xi two fine planes ahead: coarse planes up to (gz + 4) >> 1 (ring of three: the
      // planes this step's correction reads are never the one overwritten)
      const int want = min(cz_hi, (gz + 4) >> 1);
      for (int c = built + 1; c <= want; ++c) build_xi(c);
      built = max(built, want);
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if (z + G::RU < Ez) issue_u0(z + G::RU);
      if (z >= 1 && z + 2 < Ez) issue_f(z + 2);
      for (; nc <= cz_hi && nc <= built + 2; ++nc) issue_c(nc);
    }
    if (z >= 1) {
      const int zz = z - 1;
      const int gz = oz + zz;
      if (gz >= 0 && gz < L.N[2]) {
        const bool zc = zz >= 1 && zz <= Ez - 2;
        const T dz = (gz == 0 ? T(1) : T(0)) + (gz == L.N[2] - 1 ? T(1) : T(0));
        constexpr int J2 = (R + 1) % 3, J1 = (R + 2) % 3, J0 = R;
        const T* u1r = u1b + J1 * G::U1S;
        const T* fp = fb + (zz % G::RF) * G::FS;
        T* orow = ob + (long long)zz * pz;
        const unsigned act = zc ? c_mask : 0u;
        const unsigned gw = (FIN == 1 && zz >= L.J + 1 && zz < L.J + 1 + L.S[2]) ? gen_mask : 0u;
        T* frow = FIN == 1 ? fbase + (long long)(gz - a.fin.bo[2]) * a.fin.sz : nullptr;
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const T u0v = u0q[k][J1];
          const T c1 = u1q[k][J1];
          const T ym = (k == 0) ? u1r[-PY] : u1q[k > 0 ? k - 1 : 0][J1];
          const T yp = (k == MAXS - 1) ? u1r[MAXS * PY] : u1q[k + 1 < MAXS ? k + 1 : k][J1];
          const T sum = ((u1q[k][J2] + u1q[k][J0]) + (ym + yp)) + (u1r[k * PY - 1] + u1r[k * PY + 1]);
          const T r = fp[k * G::FP] - ((dk[k] + dz) * c1 - sum) * ih2;
          const T v2 = selp_(((act >> k) & 1u) != 0, c1 + cm * (c1 - u0v) + cr * r, u0v);
          if constexpr (FIN == 0) {
            if ((rw_mask >> k) & 1u) orow[k * PY] = ((w_mask >> k) & 1u) ? v2 : u0v;
          } else {
            if ((gw >> k) & 1u) frow[k * a.fin.sy] = v2;
          }
        }
      }
    }
  };
  for (int zb = 0; zb <= Ez; zb += 3) {
    step(std::integral_constant<int, 0>{}, zb);
    if (zb + 1 <= Ez) step(std::integral_constant<int, 1>{}, zb + 1);
    if (zb + 2 <= Ez) step(std::integral_constant<int, 2>{}, zb + 2);
  }
  if (threadIdx.x == 0)  // no bulk copy may still target this CTA's shared memory
    for (int c = max(cz_lo, nc - 2); c < nc; ++c) {
      const int n = c - cz_lo;
      mbar_wait(&cbar[n & 1], (n >> 1) & 1);
    }
}

template <class T, int PY, int BH, int MAXS, int NB>
bool try_up(const Lvl& L, const Lvl& Lc, const UpArgs<T>& a0, const FusedRhs<T>& b, bool launch,
            cudaStream_t st) {
  using G1 = UGeom<T, PY, BH, MAXS, 1>;
  if (L.py != PY || L.E[0] > PY) return false;
  const int crows = G1::CROWS;
  const int cpl = (int)(((long long)crows * Lc.py + G1::A - 1) / G1::A * G1::A);
  const int smax = (NB >= 3 ? 75 : 113) * 1024;
  if (G1::smem(cpl) > (size_t)smax) return false;
  if (!launch) return true;
  UpArgs<T> a = a0;
  a.cpl = cpl;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const bool fin = a.fin.p != nullptr;
  dim3 grid((L.E[1] + BH - 1) / BH, L.nsegs);
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    kern<<<grid, nt, smem, st>>>(map, a);
  };
  if (b.global) {
    if (!encode_dense_tmap<T>(&map, b, G1::FP, BH + 2)) return false;
    if (fin) go(k_up2s<T, PY, BH, MAXS, 1, 1, NB>, G1::smem(cpl), G1::NT);
    else go(k_up2s<T, PY, BH, MAXS, 1, 0, NB>, G1::smem(cpl), G1::NT);
  } else {
    using G0 = UGeom<T, PY, BH, MAXS, 0>;
    if (fin) go(k_up2s<T, PY, BH, MAXS, 0, 1, NB>, G0::smem(cpl), G0::NT);
    else go(k_up2s<T, PY, BH, MAXS, 0, 0, NB>, G0::smem(cpl), G0::NT);
  }
  return true;
}

template <class T>
bool up_dispatch(const Lvl& L, const Lvl& Lc, const UpArgs<T>& a, const FusedRhs<T>& b,
                 bool launch, cudaStream_t st) {
  if (L.st27 || L.nlg != 0.0 || (L.S[0] | L.S[1] | L.S[2]) & 1) return false;
  constexpr int NB = sizeof(T) == 4 ? 3 : 2;
  return try_up<T, 72, 10, 4, NB>(L, Lc, a, b, launch, st) ||
         try_up<T, 40, 10, 4, 3>(L, Lc, a, b, launch, st);
}

}  // namespace

template <class T>
bool up2_fused_ok(const Lvl& L, const Lvl& Lc) {
  UpArgs<T> a{};
  FusedRhs<T> b{};
  return up_dispatch<T>(L, Lc, a, b, false, nullptr);
}

template <class T>
bool launch_up2_fused(const Lvl& L, const Lvl& Lc, const T* u_in, T* u_out, const T* w,
                      const T* t, FusedRhs<T> b, double c0, double cm, double cr,
                      cudaStream_t st, FinalOut<T> fin) {
  UpArgs<T> a{};
  a.L = L;
  a.Lc = Lc;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.w = w;
  a.t = t;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  a.fin = fin;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  return up_dispatch<T>(L, Lc, a, b, true, st);
}

template bool up2_fused_ok<double>(const Lvl&, const Lvl&);
template bool up2_fused_ok<float>(const Lvl&, const Lvl&);
template bool launch_up2_fused<double>(const Lvl&, const Lvl&, const double*, double*,
                                       const double*, const double*, FusedRhs<double>, double,
                                       double, double, cudaStream_t, FinalOut<double>);
template bool launch_up2_fused<float>(const Lvl&, const Lvl&, const float*, float*, const float*,
                                      const float*, FusedRhs<float>, double, double, double,
                                      cudaStream_t, FinalOut<float>);

}  // namespace srfmg
