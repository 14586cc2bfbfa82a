// FMG entry of an SR level in one HBM pass: u = Pi(w) (fig:fmgsr L221, R10) followed by the
// degree-1 Chebyshev step S^alpha (L222, R8), sm_100a.
//
// The plan of k_cheb2s (fused.cu) with the u input produced on chip: one CTA per y-band of
// one segment, marching z; one thread streams the coarse w rows the band needs
// (cp.async.bulk from the coarse segment storage, or the level-T array at k = 1) and the
// dense rhs (tensor TMA) into shared-memory rings on mbarriers.  At plane step z every thread
// interpolates its cells of fine plane z+1 (separable trilinear: the xy-interpolant of each
// coarse plane is formed once and kept in registers, fine plane 2P uses I(P), I(P-1) and
// 2P+1 uses I(P), I(P+1); reflected coarse ghosts as signed weights) into the next u0
// shared-memory plane and its register z-queue, then applies the Chebyshev step at plane z.
// ONE __syncthreads per plane.  Storage rows are written whole: C cells smoothed, GSR cells
// the prolongated value, cells outside Omega and the padding zero.
//
// Replaces the unfused pair prolong(SET) + cheb(1): 2.65 GB instead of 5.4 GB of HBM traffic
// at C3's finest level (fp64), 0.61 ms instead of 0.53 + 0.68 ms.
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
struct PsetArgs {
  Lvl L, Lc;
  const T* w;   // coarse u
  T* uout;      // fine u (storage)
  T c0;         // 1/theta
  int foff[3];  // global index of the dense rhs array's element 0
  int cpl;      // elements per staged coarse plane
};

template <class T, int PY, int BH, int MAXS, int PW = 0>
struct GP {
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FP = PY + kAl;
  static constexpr int NG = (BH + 2 + MAXS - 1) / MAXS;
  static constexpr int NT = PY * NG;
  // PW: one producer warp after the compute threads (rounded up to whole warps) issues every
  // copy; else thread 0 issues them after each plane barrier
  static constexpr int NTC = PW ? (NT + 31) / 32 * 32 : NT;
  static constexpr int NTP = PW ? NTC + 32 : NT;
  static constexpr int TR = NG * MAXS;  // thread rows, from r0 - 1
  static constexpr int A = 128 / (int)sizeof(T);
  static constexpr int U0S = ((TR + 2) * PY + A - 1) / A * A;
  static constexpr int FS = (TR * FP + A - 1) / A * A;
  static constexpr int RF = 4, RC = 8;  // powers of two: slot/phase by shifts
  static constexpr int CROWS = TR / 2 + 3;
  static size_t smem(int cpl) {
    return (size_t)(4 * U0S + RF * FS + RC * cpl) * sizeof(T) + 8 * (2 * RF + RC);
  }
};

template <class T, int PY, int BH, int MAXS, int ZQ, int NB, int PW>
__global__ void __launch_bounds__(GP<T, PY, BH, MAXS, PW>::NTP, NB)
    k_pset1s(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ PsetArgs<T> a) {
  using G = GP<T, PY, BH, MAXS, PW>;
  constexpr int NCR = MAXS / 2 + 2;
  static_assert(MAXS % 2 == 0 && BH % 2 == 0, "row pairs");
  constexpr int YP = (ZQ + 1) & 1;  // J mod 2 (ZQ = (J + 1) mod 4)
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const Lvl& Lc = a.Lc;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int sb = r0 - 1;  // first thread row (unclamped: keeps row pairs aligned)
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + 4 * G::U0S;
  T* cs_ = fs + G::RF * G::FS;
  // [0,RF) f full, [RF,RF+RC) coarse full, [RF+RC, 2RF+RC) f empty (plane step done)
  uint64_t* bars = reinterpret_cast<uint64_t*>(cs_ + G::RC * a.cpl);
  uint64_t* fdone = bars + G::RF + G::RC;

  const int px = s % L.ns[0] + L.so[0];
  const int pyy = (s / L.ns[0]) % L.ns[1] + L.so[1];
  const int pzz = s / (L.ns[0] * L.ns[1]) + L.so[2];
  const int ox = px * L.S[0] - (L.J + 1);
  const int oy = pyy * L.S[1] - (L.J + 1);
  const int oz = pzz * L.S[2] - (L.J + 1);
  T* oseg = a.uout + (long long)s * L.ss;
  const int oxt = ox - a.foff[0];
  const int oxa = oxt & ~(G::kAl - 1);
  const int fsh = oxt - oxa;
  const uint32_t f_bytes = (uint32_t)(G::TR * G::FP * sizeof(T));
  // coarse source: the fine segment's own coarse storage, or the single level-T array
  const int cseg = Lc.nsegs == 1 ? 0 : s;
  const int cpx = cseg % Lc.ns[0] + Lc.so[0], cpy = (cseg / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
            cpz = cseg / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
  const int ocx = cpx * Lc.S[0] - (Lc.J + 1), ocy = cpy * Lc.S[1] - (Lc.J + 1),
            ocz = cpz * Lc.S[2] - (Lc.J + 1);
  const int gy_lo = oy + sb, gy_hi = oy + sb + G::TR - 1;
  const int cy_lo = max(max((gy_lo >> 1) - 1, 0), ocy);
  const int cy_hi = min(min((gy_hi >> 1) + 1, Lc.N[1] - 1), ocy + Lc.E[1] - 1);
  const int gz_lo = max(oz, 0), gz_hi = min(oz + Ez, L.N[2]) - 1;
  const int cz_lo = max(max((gz_lo >> 1) - 1, 0), ocz);
  const int cz_hi = min(min((gz_hi >> 1) + 1, Lc.N[2] - 1), ocz + Lc.E[2] - 1);
  const uint32_t cbytes = (uint32_t)((cy_hi - cy_lo + 1) * Lc.py * sizeof(T));
  const T* cw = a.w + (long long)cseg * Lc.ss + (long long)(cy_lo - ocy) * Lc.py;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * G::RF + G::RC; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_f = [=, &fmap](int z) {
    const int sl = z % G::RF;
    mbar_expect_tx(&bars[sl], f_bytes);
    tma_3d(fs + sl * G::FS, &fmap, oxa, oy + sb - a.foff[1], oz + z - a.foff[2], &bars[sl]);
  };
  auto issue_c = [&](int c) {
    const int n = c - cz_lo, sl = n % G::RC;
    if (n >= G::RC) mbar_wait(&bars[G::RF + sl], ((n - G::RC) / G::RC) & 1);  // drained
    mbar_expect_tx(&bars[G::RF + sl], cbytes);
    bulk_g2s(cs_ + sl * a.cpl, cw + (long long)(c - ocz) * Lc.pz, cbytes, &bars[G::RF + sl]);
  };
  auto wait_c = [&](int c) {
    const int n = c - cz_lo;
    mbar_wait(&bars[G::RF + (n & (G::RC - 1))], (n / G::RC) & 1);
  };
  int nc = cz_lo;  // (PW = 0: next coarse plane to issue, thread 0)
  if (!PW && threadIdx.x == 0) {
    for (int z = 0; z < min(G::RF, Ez); ++z) issue_f(z);
    for (; nc <= min(cz_hi, cz_lo + G::RC - 1); ++nc) issue_c(nc);
  }
  if (PW && threadIdx.x >= G::NTC) {  // ---- producer warp: the copy schedule, off the compute path
    if (threadIdx.x == G::NTC) {
      int nc = cz_lo;
      for (int z = 0; z < min(G::RF, Ez); ++z) issue_f(z);
      for (; nc <= min(cz_hi, cz_lo + G::RC - 1); ++nc) issue_c(nc);
      for (int z = 0; z < Ez; ++z) {
        mbar_wait(&fdone[z & (G::RF - 1)], (z / G::RF) & 1);  // plane step z done
        if (z + G::RF < Ez) issue_f(z + G::RF);  // rhs plane z is consumed
        const int live = max(cz_lo, ((oz + z + 2) >> 1) - 1);
        for (; nc <= cz_hi && nc < live + G::RC; ++nc) issue_c(nc);
      }
      for (int c = max(cz_lo, nc - G::RC); c < nc; ++c) wait_c(c);  // nothing left in flight
    }
    return;
  }
  // ---- compute threads.  The NTC - NT padding threads (PW) run the same code on the last
  // row group with every mask clear and no shared-memory stores, so that all NTC threads reach
  // each (aligned) named barrier from the same instruction
  auto csync = [] {
    if constexpr (PW) asm volatile("bar.sync 1, %0;" ::"n"(G::NTC) : "memory");
    else __syncthreads();
  };
  const bool pad = PW && threadIdx.x >= G::NT;
  const int tx = threadIdx.x % PY, g = min((int)threadIdx.x / PY, G::NG - 1);
  const int y0 = sb + g * MAXS;
  const int gx = ox + tx;
  const bool tok = tx < Ex;
  const bool tin = tok && gx >= 0 && gx < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const int dxo = (gx == 0 ? 1 : 0) + (gx == L.N[0] - 1 ? 1 : 0);
  unsigned c_mask = 0, in_mask = 0, rw_mask = 0;
  T dk[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k, gy = oy + y;
    const bool in = !pad && tin && y >= 0 && y < Ey && gy >= 0 && gy < L.N[1];
    if (in) in_mask |= 1u << k;
    if (in && tcx && y >= 1 && y <= Ey - 2) c_mask |= 1u << k;
    if (!pad && y >= r0 && y < r1) rw_mask |= 1u << k;
    dk[k] = T(6 + dxo + (gy == 0 ? 1 : 0) + (gy == L.N[1] - 1 ? 1 : 0));
  }
  // prolongation geometry (R10): x parent / neighbour column in the staged coarse rows
  constexpr T W0 = T(0.75), W1 = T(0.25);
  int cx0, cx1;
  T W1x = W1;
  {
    const int X = gx >> 1;
    int Xq = X + ((gx & 1) ? 1 : -1);
    if (Xq < 0) { Xq = 0; W1x = -W1; }
    if (Xq >= Lc.N[0]) { Xq = Lc.N[0] - 1; W1x = -W1; }
    cx0 = min(max(X - ocx, 0), Lc.E[0] - 1);
    cx1 = min(max(Xq - ocx, 0), Lc.E[0] - 1);
  }
  int cro[NCR];
  T cys[NCR];
  {
    const int Y0 = (oy + y0) >> 1;
#pragma unroll
    for (int m = 0; m < NCR; ++m) {
      int Y = Y0 - 1 + m;
      T sg = T(1);
      if (Y < 0) { Y = 0; sg = T(-1); }
      if (Y >= Lc.N[1]) { Y = Lc.N[1] - 1; sg = T(-1); }
      Y = min(max(Y, cy_lo), max(cy_hi, cy_lo));
      cro[m] = (Y - cy_lo) * Lc.py;
      cys[m] = sg;
    }
  }
  auto interp = [&](int c, T (&I)[MAXS]) {  // xy-interpolant of coarse plane c (reflected)
    int cc = min(max(c, 0), Lc.N[2] - 1);
    const T a0 = (cc != c) ? -W0 : W0, a1 = (cc != c) ? -W1 : W1;  // reflected plane: -I
    cc = min(max(cc, cz_lo), cz_hi);  // (never hit for a used plane; keeps the wait safe)
    wait_c(cc);
    const T* cp = cs_ + ((cc - cz_lo) & (G::RC - 1)) * a.cpl;
    T xi[NCR];
#pragma unroll
    for (int m = 0; m < NCR; ++m) xi[m] = cys[m] * (W0 * cp[cro[m] + cx0] + W1x * cp[cro[m] + cx1]);
    // fine row oy+y0+k: parent coarse row index m and neighbour m +- 1 in xi; the parity
    // YP of oy+y0 is J mod 2 over the whole grid (S, BH, MAXS even)
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      if constexpr (YP == 0)
        I[k] = a0 * xi[k / 2 + 1] + a1 * xi[(k & 1) ? k / 2 + 2 : k / 2];
      else
        I[k] = a0 * xi[(k + 1) / 2 + 1] + a1 * xi[(k & 1) ? (k + 1) / 2 : k / 2 + 2];
    }
  };
  // I2[P & 1] = xy-interpolant of coarse plane P; fine plane 2P uses I(P), I(P-1) and 2P+1
  // uses I(P), I(P+1): with the z loop unrolled by 4 and gz mod 4 known at compile time
  // (oz = -(J+1) mod 4, S a multiple of 4) both are fixed registers -- no rotation moves
  T I2[2][MAXS];
  T u0q[MAXS][4];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    I2[0][k] = I2[1][k] = T(0);
    u0q[k][0] = u0q[k][1] = u0q[k][2] = u0q[k][3] = T(0);
  }
  // v0 of storage plane z (residue RS = z mod 4: register slot and shared-memory slot)
  auto source = [&](auto RSC, int z) {
    constexpr int RS = decltype(RSC)::value;
    constexpr int G4 = (RS + 4 - ZQ) % 4;      // gz mod 4
    constexpr int PP = G4 >> 1, PN = 1 - PP;  // parity of P = gz >> 1 and of P +- 1
    const int gz = oz + z;
    T pv[MAXS];
    if (gz >= gz_lo && gz <= gz_hi) {
      if constexpr (G4 & 1) interp((gz >> 1) + 1, I2[PN]);  // I(P+1) replaces I(P-1)
#pragma unroll
      for (int k = 0; k < MAXS; ++k) pv[k] = W0 * I2[PP][k] + W1 * I2[PN][k];
    } else {
#pragma unroll
      for (int k = 0; k < MAXS; ++k) pv[k] = T(0);
    }
    T* up = u0s + RS * G::U0S + (y0 - sb + 1) * PY + tx;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const T v = ((in_mask >> k) & 1u) ? pv[k] : T(0);
      u0q[k][RS] = v;
      if (!pad) up[k * PY] = v;
    }
  };
  {  // the interpolants at the first in-domain plane: I(P0), and I(P0-1) if it is even
    const int P = gz_lo >> 1;
    if (P & 1) {
      interp(P, I2[1]);
      if (!(gz_lo & 1)) interp(P - 1, I2[0]);
    } else {
      interp(P, I2[0]);
      if (!(gz_lo & 1)) interp(P - 1, I2[1]);
    }
  }
  source(std::integral_constant<int, 0>{}, 0);
  csync();
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0;
  T* const ob = oseg + (long long)y0 * PY + tx;
  const int fo = (y0 - sb) * G::FP + tx + fsh;

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 4
    constexpr int IM = (R + 3) % 4, IP = (R + 1) % 4;
    if (z + 1 < Ez) source(std::integral_constant<int, IP>{}, z + 1);  // plane z+1 (slot IP)
    else {
#pragma unroll
      for (int k = 0; k < MAXS; ++k) u0q[k][IP] = T(0);
    }
    mbar_wait(&bars[z & (G::RF - 1)], (z / G::RF) & 1);
    const int gz = oz + z;
    const bool zin = gz >= gz_lo && gz <= gz_hi;
    const bool zc = zin && z >= 1 && z <= Ez - 2;
    const T dz = (gz == 0 ? T(1) : T(0)) + (gz == L.N[2] - 1 ? T(1) : T(0));
    const T* pl = u0s + R * G::U0S + (y0 - sb + 1) * PY + tx;
    const T* fp = fs + (z & (G::RF - 1)) * G::FS + fo;
    const unsigned act = zc ? c_mask : 0u;
    const unsigned wr = zin ? rw_mask : 0u;
    T* const orow = ob + (long long)z * pz;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const T v0 = u0q[k][R];
      const T ym = (k == 0) ? pl[-PY] : u0q[k > 0 ? k - 1 : 0][R];
      const T yp = (k == MAXS - 1) ? pl[MAXS * PY] : u0q[k + 1 < MAXS ? k + 1 : k][R];
      const T sum = ((u0q[k][IM] + u0q[k][IP]) + (ym + yp)) + (pl[k * PY - 1] + pl[k * PY + 1]);
      const T r = fp[k * G::FP] - ((dk[k] + dz) * v0 - sum) * ih2;
      const T v1 = ((act >> k) & 1u) ? v0 + c0 * r : v0;
      if ((wr >> k) & 1u) orow[k * PY] = v1;
    }
    csync();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if constexpr (PW) {
        mbar_arrive(&fdone[z & (G::RF - 1)]);  // to the producer
      } else {
        if (z + G::RF < Ez) issue_f(z + G::RF);  // rhs plane z is consumed
        const int live = max(cz_lo, ((oz + z + 2) >> 1) - 1);
        for (; nc <= cz_hi && nc < live + G::RC; ++nc) issue_c(nc);
      }
    }
  };
  for (int zb = 0; zb < Ez; zb += 4) {
    step(std::integral_constant<int, 0>{}, zb);
    if (zb + 1 < Ez) step(std::integral_constant<int, 1>{}, zb + 1);
    if (zb + 2 < Ez) step(std::integral_constant<int, 2>{}, zb + 2);
    if (zb + 3 < Ez) step(std::integral_constant<int, 3>{}, zb + 3);
  }
  if (!PW && threadIdx.x == 0)  // no bulk copy may still target this CTA's shared memory
    for (int c = max(cz_lo, nc - G::RC); c < nc; ++c) wait_c(c);
}

template <class T, int PY, int BH, int MAXS, int ZQ, int NB = 2, int PW = 0>
bool try_pset(const Lvl& L, const Lvl& Lc, const T* w, T* uout, const FusedRhs<T>& b, double c0,
              cudaStream_t st, bool launch) {
  using G = GP<T, PY, BH, MAXS, PW>;
  if (L.py != PY || L.E[0] > PY || !b.global) return false;
  const int cpl = (int)(((long long)G::CROWS * Lc.py + G::A - 1) / G::A * G::A);
  const size_t smem = G::smem(cpl);
  const int smax = (NB >= 4 ? 56 : NB == 3 ? 75 : NB == 2 ? 113 : 227) * 1024;  // CTAs per SM
  if (smem > (size_t)smax) return false;
  if (!launch) return true;
  PsetArgs<T> a{};
  a.L = L;
  a.Lc = Lc;
  a.w = w;
  a.uout = uout;
  a.c0 = (T)c0;
  a.cpl = cpl;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.off[d];
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (!encode_dense_tmap<T>(&map, b, G::FP, G::TR)) return false;
  auto kern = k_pset1s<T, PY, BH, MAXS, ZQ, NB, PW>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);  // per device
  kern<<<dim3((L.E[1] + BH - 1) / BH, L.nsegs), G::NTP, smem, st>>>(map, a);
  return true;
}

// band geometries (PY, BH, MAXS[, CTAs/SM]).  BH = 10 (three row groups, 216 threads) keeps
// the fp64 kernel at 2 CTAs/SM within 128 registers (BH = 14, 288 threads, caps it at 96 and
// it spills: 0.77 vs 0.67 ms at C3; 6-row bands at 3 CTAs/SM 0.68 ms, 10-row bands of 6
// cells 0.71 ms); fp32: 14-row bands of 8 cells per thread (0.365 vs 0.414 ms at C3's
// finest level).  At E = 38 (PY = 40) BH = 10 at 4 CTAs/SM: 0.115 ms vs 0.172 ms for BH = 12
// at 3 (BH = 14: slower).
template <class T, int ZQ>
bool pset_geom(const Lvl& L, const Lvl& Lc, const T* w, T* uout, const FusedRhs<T>& b,
               double c0, cudaStream_t st, bool launch) {
  constexpr int NB = sizeof(T) == 4 ? 3 : 2;
  if (sizeof(T) == 4 && try_pset<T, 72, 14, 8, ZQ, NB>(L, Lc, w, uout, b, c0, st, launch))
    return true;
  // fp64 at E = 70: a producer warp issues the copies (120 registers; SR_FMG_PSET_PW=0: thread
  // 0 after each plane barrier, as the other geometries, where the extra warp costs spills)
  static const bool pw = [] {
    const char* e = std::getenv("SR_FMG_PSET_PW");
    return !(e && e[0] == '0');
  }();
  if (sizeof(T) == 8 && pw && try_pset<T, 72, 10, 4, ZQ, NB, 1>(L, Lc, w, uout, b, c0, st, launch))
    return true;
  return try_pset<T, 72, 10, 4, ZQ, NB>(L, Lc, w, uout, b, c0, st, launch) ||
         // E = 134: 10-row bands at one CTA per SM (4.9 ms at C5; 6-row bands at two: 6.7 ms)
         try_pset<T, 136, 10, 4, ZQ, 1>(L, Lc, w, uout, b, c0, st, launch) ||
         try_pset<T, 40, 10, 4, ZQ, 4>(L, Lc, w, uout, b, c0, st, launch) ||
         // E = 22 / 14 (levels 6 and 5 of C3): 47 / 22 us against 60 / 32 us for the
         // separate prolongation and degree-1 pass
         try_pset<T, 24, 10, 4, ZQ, 4>(L, Lc, w, uout, b, c0, st, launch) ||
         try_pset<T, 16, 6, 2, ZQ, 4>(L, Lc, w, uout, b, c0, st, launch);
}

template <class T>
bool pset_dispatch(const Lvl& L, const Lvl& Lc, const T* w, T* uout, const FusedRhs<T>& b,
                   double c0, cudaStream_t st, bool launch) {
  // S_z % 4: the segment origins oz = p S - (J+1) all share one residue mod 4
  if (L.st27 || L.nlg != 0.0 || (L.S[0] | L.S[1]) & 1 || L.S[2] & 3) return false;
  switch ((L.J + 1) & 3) {
    case 0: return pset_geom<T, 0>(L, Lc, w, uout, b, c0, st, launch);
    case 1: return pset_geom<T, 1>(L, Lc, w, uout, b, c0, st, launch);
    case 2: return pset_geom<T, 2>(L, Lc, w, uout, b, c0, st, launch);
    default: return pset_geom<T, 3>(L, Lc, w, uout, b, c0, st, launch);
  }
}

}  // namespace

template <class T>
bool pset1_fused_ok(const Lvl& L, const Lvl& Lc, int rhs_global) {
  FusedRhs<T> b{};
  b.global = rhs_global;
  return pset_dispatch<T>(L, Lc, nullptr, nullptr, b, 0.0, nullptr, false);
}

template <class T>
bool launch_pset1_fused(const Lvl& L, const Lvl& Lc, const T* w, T* uout, FusedRhs<T> b,
                        double c0, cudaStream_t st) {
  return pset_dispatch<T>(L, Lc, w, uout, b, c0, st, true);
}

template bool pset1_fused_ok<double>(const Lvl&, const Lvl&, int);
template bool pset1_fused_ok<float>(const Lvl&, const Lvl&, int);
template bool launch_pset1_fused<double>(const Lvl&, const Lvl&, const double*, double*,
                                         FusedRhs<double>, double, cudaStream_t);
template bool launch_pset1_fused<float>(const Lvl&, const Lvl&, const float*, float*,
                                        FusedRhs<float>, double, cudaStream_t);

}  // namespace srfmg
