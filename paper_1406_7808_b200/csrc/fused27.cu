// TMA-fed Chebyshev pass for the paper's 27-point operator (reading R28), sm_100a.
//
// Same plan as k_cheb2s (fused.cu): one CTA per y-band of one segment, marching z; one
// thread streams the u rows (cp.async.bulk) and the rhs (tensor TMA box or bulk rows) into
// shared-memory rings on mbarriers; ONE __syncthreads per plane.  The 27-point stencil reads
// the full 3x3x3 neighbourhood, so every stage input is kept as a plane ring in shared memory
// (u0: 5 planes, the first-step result u1: 4 planes) instead of register z-queues; each
// thread's own centre values stay in registers (slot p % 3).
//
//   stage 1 at plane z      u1 = u0 + c0 (b - A u0)                       (rows s0..s1)
//   stage 2 at plane z - 2  u2 = u1 + cm (u1 - u0) + cr (b - A u1)        (rows r0..r1)
//   (degree 1: stage 1 is the result)
//
// A u = (8/3 u - 1/6 sum_edges - 1/12 sum_corners) / h^2, face weight 0.  Reflected ghosts
// (R3, (-1)^m u(mirror)): a neighbour across a domain face is read from the mirror cell
// (offset 0 in that dimension) with a sign flip -- per thread for x and y, per plane for z.
// Cells outside Omega keep their (zero) value; GSR cells are carried through.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <type_traits>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

template <class T>
struct C27Args {
  Lvl L;
  const T* uin;
  T* uout;
  const T* rhs_seg;
  T c0, cm, cr;
  FinalOut<T> fin;
  int foff[3];
  // FIN = 3: tau (Eq. 4) in front of the degree-2 pass: rhs_seg holds R (its own buffer),
  // rhs = R + A u0 on F, A u0 on C \ F and t = u0 are written (as k_cheb2s FIN = 2)
  T* rhs_out;
  T* tout;
  int jr;
  int nof;  // FIN = 2 only: write -A u (the rhs is not streamed; R6 pyramid restriction)
};

template <class T, int PY, int BH, int MAXS, int RG>
struct G27 {
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FP = RG ? PY + kAl : PY;
  static constexpr int NG = (BH + 2 + MAXS - 1) / MAXS;
  static constexpr int NT = PY * NG;
  static constexpr int TR = NG * MAXS;
  static constexpr int A = 128 / (int)sizeof(T);
  static constexpr int PL = ((TR + 2) * PY + A - 1) / A * A;  // u0 / u1 plane (+1 margin row)
  static constexpr int FS = (TR * FP + A - 1) / A * A;
  static constexpr int RU = 5, RF = 5, R1 = 4;
  static constexpr size_t SMEM = (size_t)(RU * PL + RF * FS + R1 * PL) * sizeof(T) + 8 * (RU + RF);
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
};

template <class T, int PY, int BH, int MAXS, int RG, int NST, int FIN>
__global__ void __launch_bounds__(G27<T, PY, BH, MAXS, RG>::NT, G27<T, PY, BH, MAXS, RG>::MINB)
    k_cheb27s(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ C27Args<T> a) {
  using G = G27<T, PY, BH, MAXS, RG>;
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + G::RU * G::PL;
  T* u1s = fs + G::RF * G::FS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(u1s + G::R1 * G::PL);  // [0,RU) u0, then f

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
  if (threadIdx.x == 0) {
    for (int i = 0; i < G::RU + G::RF; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_u0 = [=](int z) {
    const int sl = z % G::RU;
    mbar_expect_tx(&bars[sl], u0_bytes);
    bulk_g2s(u0s + sl * G::PL + (q0 - s0 + 1) * PY, useg + (long long)z * pz + (long long)q0 * PY,
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
  constexpr int FLAG = NST == 2 ? 2 : 0;  // iterations an rhs plane stays in use
  const bool nof = FIN == 2 && a.nof;
  if (threadIdx.x == 0) {  // fill both rings
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    if (!nof)
      for (int z = 0; z < min(G::RF, Ez); ++z) issue_f(z);
  }

  const int tx = threadIdx.x % PY, g = threadIdx.x / PY;
  const int y0 = s0 + g * MAXS;
  const int gx = ox + tx;
  const bool tok = tx < Ex;
  const bool tin = tok && gx >= 0 && gx < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  // x mirror: neighbour column offsets and signs (R3)
  const bool xlo = gx == 0, xhi = gx == L.N[0] - 1;
  // (edge columns of the storage box are never C cells: their neighbour reads are clamped
  // into the row so no load leaves the shared-memory planes)
  const int cxm = (xlo || tx == 0) ? 0 : -1, cxp = (xhi || tx >= Ex - 1) ? 0 : 1;
  const T sxm = xlo ? T(-1) : T(1), sxp = xhi ? T(-1) : T(1);
  unsigned c_mask = 0, w_mask = 0;
  int rym[MAXS], ryp[MAXS];  // row offsets (in elements) of the y-1 / y+1 neighbours
  T sym[MAXS], syp[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k, gy = oy + y;
    const bool in = tin && y < s1 && gy >= 0 && gy < L.N[1];
    if (in && tcx && y >= 1 && y <= Ey - 2) c_mask |= 1u << k;
    if (in && y >= r0 && y < r1) w_mask |= 1u << k;
    const bool ylo = gy == 0, yhi = gy == L.N[1] - 1;
    rym[k] = ylo ? 0 : -PY;
    ryp[k] = yhi ? 0 : PY;
    sym[k] = ylo ? T(-1) : T(1);
    syp[k] = yhi ? T(-1) : T(1);
  }
  // FIN = 3: slots in F = grow(V, jr) (x, y), F in z, and the rhs / t rows
  unsigned f_mask = 0;
  int fz0 = 0, fz1 = 0;
  if constexpr (FIN == 3) {
    const bool fx = gx >= px * L.S[0] - a.jr && gx < (px + 1) * L.S[0] + a.jr;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const int gy = oy + y0 + k;
      if (fx && gy >= pyy * L.S[1] - a.jr && gy < (pyy + 1) * L.S[1] + a.jr) f_mask |= 1u << k;
    }
    fz0 = pzz * L.S[2] - a.jr;
    fz1 = (pzz + 1) * L.S[2] + a.jr;
  }
  const int po = (y0 - s0 + 1) * PY + tx;  // own row 0 in a u0 / u1 plane
  const int fo = (y0 - s0) * G::FP + tx + fsh;
  T* const ob = oseg + (long long)y0 * PY + tx;
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0, cm = a.cm, cr = a.cr;
  T u0r[MAXS][3], u1r[MAXS][3];  // own centre values, plane p in slot p % 3
#pragma unroll
  for (int k = 0; k < MAXS; ++k) u0r[k][0] = u0r[k][1] = u0r[k][2] = u1r[k][0] = u1r[k][1] = u1r[k][2] = T(0);

  // 27-point A (R28) for all MAXS slots of the thread from the plane triple (pm, p0, pp) with z
  // signs (szm, szp), sharing the in-plane partial sums between neighbouring slots: per plane
  // P and row r, the x pair
  //   H(P, r) = sxm P[r, x-1] + sxp P[r, x+1]
  // is loaded once (a window over rows k-1, k, k+1 slides down the slots), and
  //   edges(z)   = sym H(p0, k-1) + syp H(p0, k+1)            (in-plane diagonals)
  //   edges(z-1) = H(pm, k) + sym pm[k-1] + syp pm[k+1]       (faces of the plane below)
  //   corners    = sym H(pm, k-1) + syp H(pm, k+1)            (and likewise for pp)
  //   A u = (8/3 u - (edges)/6 - (corners)/12) / h^2,  face weight 0
  // -- 8 shared-memory loads per slot instead of 20 for the neighbour-by-neighbour sum (P27:
  // the finest degree-2 passes 13.8 -> 11.5 ms; the interior path below: -> 10.4 ms).  The row index k-1 / k+1 becomes k itself
  // across a domain face (R3 mirror, sign in sym/syp).
  // INT (a CTA whose cells have no x or y neighbour across a domain face): every sign is +1
  // and no row is mirrored, so the products and selects drop out -- the same operations on
  // the same values otherwise (x * 1 exact, fma(1, a, b) = a + b): bitwise the general path
  auto A27w = [&](auto INTt, const T* pm, const T* p0, const T* pp, T szm, T szp,
                  const T (&cv)[MAXS], T (&Av)[MAXS]) {
    constexpr bool INT = decltype(INTt)::value;
    auto hs = [&](const T* P, int r) {
      const int o = r * PY;
      if constexpr (INT) return P[o + cxm] + P[o + cxp];
      else return sxm * P[o + cxm] + sxp * P[o + cxp];
    };
    T h0m = hs(p0, -1), h0c = hs(p0, 0), hmm = hs(pm, -1), hmc = hs(pm, 0);
    T hpm = hs(pp, -1), hpc = hs(pp, 0);
    T cmm = pm[-PY], cmc = pm[0], cpm = pp[-PY], cpc = pp[0];
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const T h0n = hs(p0, k + 1), hmn = hs(pm, k + 1), hpn = hs(pp, k + 1);
      const T cmn = pm[(k + 1) * PY], cpn = pp[(k + 1) * PY];
      T e0, em, ep, km, kp;
      if constexpr (INT) {
        e0 = h0m + h0n;
        em = hmc + cmm + cmn;
        ep = hpc + cpm + cpn;
        km = hmm + hmn;
        kp = hpm + hpn;
      } else {
        const bool ylo = rym[k] == 0, yhi = ryp[k] == 0;
        e0 = sym[k] * (ylo ? h0c : h0m) + syp[k] * (yhi ? h0c : h0n);
        em = hmc + sym[k] * (ylo ? cmc : cmm) + syp[k] * (yhi ? cmc : cmn);
        ep = hpc + sym[k] * (ylo ? cpc : cpm) + syp[k] * (yhi ? cpc : cpn);
        km = sym[k] * (ylo ? hmc : hmm) + syp[k] * (yhi ? hmc : hmn);
        kp = sym[k] * (ylo ? hpc : hpm) + syp[k] * (yhi ? hpc : hpn);
      }
      const T e = e0 + szm * em + szp * ep;
      const T kk = szm * km + szp * kp;
      Av[k] = (T(8.0 / 3.0) * cv[k] - e * T(1.0 / 6.0) - kk * T(1.0 / 12.0)) * ih2;
      h0m = h0c; h0c = h0n; hmm = hmc; hmc = hmn; hpm = hpc; hpc = hpn;
      cmm = cmc; cmc = cmn; cpm = cpc; cpc = cpn;
    }
  };
  // CTA-uniform: no thread column (x, all of the row pitch) and no thread row (y) is a domain
  // boundary cell, i.e. the box [ox, ox + PY) x [oy + s0, oy + s0 + TR) lies within the
  // cells 1 .. N - 2 (z is per plane: szm / szp)
  const bool interior = ox >= 1 && ox + PY <= L.N[0] - 1 && oy + s0 >= 1 &&
                        oy + s0 + G::TR <= L.N[1] - 1;
  // plane pointers of a ring with z mirroring at the domain faces (R3)
  auto triple = [&](const T* base, int ring, int zc, const T*& pm, const T*& p0, const T*& pp,
                    T& szm, T& szp) {
    const int gz = oz + zc;
    const bool zlo = gz == 0, zhi = gz == L.N[2] - 1;
    p0 = base + (zc % ring) * G::PL + po;
    pm = zlo ? p0 : base + ((zc + ring - 1) % ring) * G::PL + po;
    pp = zhi ? p0 : base + ((zc + 1) % ring) * G::PL + po;
    szm = zlo ? T(-1) : T(1);
    szp = zhi ? T(-1) : T(1);
  };

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3
    if (z < Ez) {  // ------------------------------------------ stage 1 at plane z
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % G::RU], ((z + 1) / G::RU) & 1);
      mbar_wait(&bars[z % G::RU], (z / G::RU) & 1);
      if (!nof) mbar_wait(&bars[G::RU + z % G::RF], (z / G::RF) & 1);
      const int gz = oz + z;
      const bool zc = gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2;
      const T* pm;
      const T* p0;
      const T* pp;
      T szm, szp;
      triple(u0s, G::RU, z, pm, p0, pp, szm, szp);
      const T* fp = fs + (z % G::RF) * G::FS + fo;
      T* u1w = u1s + (z % G::R1) * G::PL + po;
      const unsigned act = zc ? c_mask : 0u;
      const unsigned fm = (FIN == 3 && gz >= fz0 && gz < fz1) ? f_mask : 0u;
      T cv0[MAXS], Av0[MAXS];
#pragma unroll
      for (int k = 0; k < MAXS; ++k) cv0[k] = p0[k * PY];
      if (interior) A27w(std::true_type{}, pm, p0, pp, szm, szp, cv0, Av0);
      else A27w(std::false_type{}, pm, p0, pp, szm, szp, cv0, Av0);
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        const T v0 = cv0[k];
        T r;
        if constexpr (FIN == 3) {
          // tau (Eq. 4, fig:mgvsr L234-236) and the first step's residual rhs - A u0
          const T Au = Av0[k];
          const T Rv = fp[k * G::FP];
          const T bv = ((fm >> k) & 1u) ? Rv + Au : Au;
          r = bv - Au;
          const bool cc = (act >> k) & 1u;
          const_cast<T*>(fp)[k * G::FP] = cc ? bv : Rv;  // stage 2 reads the new rhs
          if (((w_mask >> k) & 1u) && gz >= 0 && gz < L.N[2]) {
            const long long o = (long long)s * L.ss + (long long)z * pz + (long long)(y0 + k) * PY + tx;
            if (cc) a.rhs_out[o] = bv;
            a.tout[o] = v0;  // t = u0
          }
        } else {
          r = (nof ? T(0) : fp[k * G::FP]) - Av0[k];
        }
        const T v1 = ((act >> k) & 1u) ? v0 + c0 * r : v0;
        if constexpr (FIN == 2) {  // residual mode: r = b - A u0 on C (restriction input)
          if (((w_mask >> k) & 1u) && gz >= 0 && gz < L.N[2]) ob[(long long)z * pz + k * PY] = r;
        } else if constexpr (NST == 2) {
          u0r[k][R] = v0;
          u1r[k][R] = v1;
          u1w[k * PY] = v1;
        } else {
          if (((w_mask >> k) & 1u) && gz >= 0 && gz < L.N[2]) {
            if constexpr (FIN == 0) {
              ob[(long long)z * pz + k * PY] = v1;
            } else {
              const int y = y0 + k, vlo = L.J + 1;
              if (tx >= vlo && tx < vlo + L.S[0] && y >= vlo && y < vlo + L.S[1] && z >= vlo &&
                  z < vlo + L.S[2])
                a.fin.p[(long long)(gz - a.fin.bo[2]) * a.fin.sz +
                        (long long)(oy + y - a.fin.bo[1]) * a.fin.sy + (gx - a.fin.bo[0])] = v1;
            }
          }
        }
      }
    }
    if constexpr (NST == 2) {  // ------------------------------ stage 2 at plane z - 2
      const int zz = z - 2;
      if (zz >= 0 && zz < Ez) {
        constexpr int J = (R + 1) % 3;  // slot of plane z - 2
        const int gz = oz + zz;
        if (gz >= 0 && gz < L.N[2]) {
          const bool zc = zz >= 1 && zz <= Ez - 2;
          const T* pm;
          const T* p0;
          const T* pp;
          T szm, szp;
          triple(u1s, G::R1, zz, pm, p0, pp, szm, szp);
          const T* fp = fs + (zz % G::RF) * G::FS + fo;
          T* orow = ob + (long long)zz * pz;
          const unsigned act = zc ? c_mask : 0u;
          T cv1[MAXS], Av1[MAXS];
#pragma unroll
          for (int k = 0; k < MAXS; ++k) cv1[k] = u1r[k][J];
          if (interior) A27w(std::true_type{}, pm, p0, pp, szm, szp, cv1, Av1);
          else A27w(std::false_type{}, pm, p0, pp, szm, szp, cv1, Av1);
#pragma unroll
          for (int k = 0; k < MAXS; ++k) {
            const T c1 = cv1[k];
            const T r = fp[k * G::FP] - Av1[k];
            const T v2 = ((act >> k) & 1u) ? c1 + cm * (c1 - u0r[k][J]) + cr * r : u0r[k][J];
            if (!((w_mask >> k) & 1u)) continue;
            if constexpr (FIN != 1) {
              orow[k * PY] = v2;
            } else {
              const int y = y0 + k, vlo = L.J + 1;
              if (tx >= vlo && tx < vlo + L.S[0] && y >= vlo && y < vlo + L.S[1] && zz >= vlo &&
                  zz < vlo + L.S[2])
                a.fin.p[(long long)(gz - a.fin.bo[2]) * a.fin.sz +
                        (long long)(oy + y - a.fin.bo[1]) * a.fin.sy + (gx - a.fin.bo[0])] = v2;
            }
          }
        }
      }
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if (z >= 1 && z - 1 + G::RU < Ez) issue_u0(z - 1 + G::RU);  // plane z-1 consumed
      if (!nof && z - FLAG >= 0 && z - FLAG + G::RF < Ez) issue_f(z - FLAG + G::RF);
    }
  };
  const int nz = Ez + (NST == 2 ? 2 : 0);
  for (int zb = 0; zb < nz; zb += 3) {
    step(std::integral_constant<int, 0>{}, zb);
    if (zb + 1 < nz) step(std::integral_constant<int, 1>{}, zb + 1);
    if (zb + 2 < nz) step(std::integral_constant<int, 2>{}, zb + 2);
  }
}

template <class T, int PY, int BH, int MAXS>
bool try27(const Lvl& L, const C27Args<T>& a, const FusedRhs<T>& b, int nst, int fin,
           cudaStream_t st, bool launch) {
  if (L.py != PY || L.E[0] > PY) return false;
  using G = G27<T, PY, BH, MAXS, 1>;
  if (G::SMEM > 227 * 1024 || G27<T, PY, BH, MAXS, 0>::SMEM > 227 * 1024) return false;
  if (!launch) return true;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  dim3 grid((L.E[1] + BH - 1) / BH, L.nsegs);
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, nt, smem, st>>>(map, a);
  };
  if (b.global && fin == 3) return false;
  if (b.global) {
    if (!encode_dense_tmap<T>(&map, b, G::FP, BH + 2)) return false;
    if (fin == 2) go(k_cheb27s<T, PY, BH, MAXS, 1, 1, 2>, G::SMEM, G::NT);
    else if (nst == 2 && fin) go(k_cheb27s<T, PY, BH, MAXS, 1, 2, 1>, G::SMEM, G::NT);
    else if (nst == 2) go(k_cheb27s<T, PY, BH, MAXS, 1, 2, 0>, G::SMEM, G::NT);
    else if (fin) go(k_cheb27s<T, PY, BH, MAXS, 1, 1, 1>, G::SMEM, G::NT);
    else go(k_cheb27s<T, PY, BH, MAXS, 1, 1, 0>, G::SMEM, G::NT);
  } else {
    using G0 = G27<T, PY, BH, MAXS, 0>;
    if (fin == 3) go(k_cheb27s<T, PY, BH, MAXS, 0, 2, 3>, G0::SMEM, G0::NT);
    else if (fin == 2) go(k_cheb27s<T, PY, BH, MAXS, 0, 1, 2>, G0::SMEM, G0::NT);
    else if (nst == 2 && fin) go(k_cheb27s<T, PY, BH, MAXS, 0, 2, 1>, G0::SMEM, G0::NT);
    else if (nst == 2) go(k_cheb27s<T, PY, BH, MAXS, 0, 2, 0>, G0::SMEM, G0::NT);
    else if (fin) go(k_cheb27s<T, PY, BH, MAXS, 0, 1, 1>, G0::SMEM, G0::NT);
    else go(k_cheb27s<T, PY, BH, MAXS, 0, 1, 0>, G0::SMEM, G0::NT);
  }
  return true;
}

template <class T>
bool dispatch27(const Lvl& L, const C27Args<T>& a, const FusedRhs<T>& b, int nst, int fin,
                cudaStream_t st, bool launch) {
  return try27<T, 72, 10, 4>(L, a, b, nst, fin, st, launch) ||
         try27<T, 40, 10, 4>(L, a, b, nst, fin, st, launch) ||
         try27<T, 24, 11, 4>(L, a, b, nst, fin, st, launch) ||
         try27<T, 16, 14, 2>(L, a, b, nst, fin, st, launch);  // E = 14 (8^3 segments)
}

}  // namespace

template <class T>
bool cheb27_fused_ok(const Lvl& L) {
  if (!L.st27 || L.nlg != 0.0 || ((long long)L.N[0] * sizeof(T)) % 16) return false;
  C27Args<T> a{};
  FusedRhs<T> b{};
  return dispatch27<T>(L, a, b, 2, 0, nullptr, false);
}

template <class T>
void launch_cheb27_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, int nst,
                         double c0, double cm, double cr, cudaStream_t st, FinalOut<T> fin) {
  C27Args<T> a{};
  a.L = L;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  a.fin = fin;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  dispatch27<T>(L, a, b, nst, fin.p != nullptr ? 1 : 0, st, true);
}

// tau (Eq. 4) fused in front of the degree-2 27-point pass: R read from its own buffer
template <class T>
bool launch_tau_cheb27_fused(const Lvl& L, const T* u_in, T* u_out, const T* R, T* rhs, T* t,
                             int jr, double c0, double cm, double cr, cudaStream_t st) {
  C27Args<T> a{};
  a.L = L;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = R;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  a.rhs_out = rhs;
  a.tout = t;
  a.jr = jr;
  FusedRhs<T> b{};
  b.p = R;
  b.global = 0;
  return dispatch27<T>(L, a, b, 2, 3, st, true);
}
template bool launch_tau_cheb27_fused<double>(const Lvl&, const double*, double*, const double*,
                                              double*, double*, int, double, double, double,
                                              cudaStream_t);
template bool launch_tau_cheb27_fused<float>(const Lvl&, const float*, float*, const float*,
                                             float*, float*, int, double, double, double,
                                             cudaStream_t);

template <class T>
void launch_resid27_fused(const Lvl& L, const T* u, T* r, FusedRhs<T> b, cudaStream_t st,
                          int nof) {
  C27Args<T> a{};
  a.L = L;
  a.uin = u;
  a.uout = r;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.nof = nof;
  a.c0 = T(1);
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  dispatch27<T>(L, a, b, 1, 2, st, true);
}
template void launch_resid27_fused<double>(const Lvl&, const double*, double*, FusedRhs<double>,
                                           cudaStream_t, int);
template void launch_resid27_fused<float>(const Lvl&, const float*, float*, FusedRhs<float>,
                                          cudaStream_t, int);

template bool cheb27_fused_ok<double>(const Lvl&);
template bool cheb27_fused_ok<float>(const Lvl&);
template void launch_cheb27_fused<double>(const Lvl&, const double*, double*, FusedRhs<double>,
                                          int, double, double, double, cudaStream_t,
                                          FinalOut<double>);
template void launch_cheb27_fused<float>(const Lvl&, const float*, float*, FusedRhs<float>, int,
                                         double, double, double, cudaStream_t, FinalOut<float>);

}  // namespace srfmg
