// Up half of an SR level visit in one HBM pass (sm_100a): the coarse-grid correction
// u += P(w - t) on C ∪ GSR (fig:mgvsr L241, R10, R17) followed by the degree-2 Chebyshev
// post-smoothing on C (L242, R8).  Replaces the correction kernel plus the degree-2 pass:
// one read and one write of u fewer per level visit (at C3's finest level 2.8 GB).
//
// The plan of k_cheb2s (fused.cu) -- one CTA per y-band of one segment, u rows and the rhs
// streamed into shared-memory rings by one thread (cp.async.bulk / TMA) on mbarriers, stage
// 1 at plane z and stage 2 at plane z-1 with register z-queues, ONE __syncthreads per plane
// -- with the correction applied to every u plane one step before stage 1 reads it:
//   * the coarse rows of w and t the band needs are bulk-copied per coarse plane into a
//     3-plane ring;
//   * at step z the CTA forms, for fine plane z+2, F[m][x] = the x- and z-interpolant of
//     (w - t) at coarse row m and fine column x (separable trilinear, 1D weights 3/4 and 1/4,
//     reflected coarse ghosts as signed weights, R3), two rows per thread;
//   * at step z every thread corrects its cells of fine plane z+1 (already in shared memory)
//     with two reads of F, in registers and in place: u += W0 F[m0] + wy F[m1]; the band's
//     two outermost rows (read by stage 1 only as y-neighbours) are corrected by the first and
//     the last row group.
// After the barrier of step z, plane z+1 is corrected for every reader.  Output as k_cheb2s:
// C smoothed, GSR the corrected u, cells outside Omega zero; or (last pass of the solve) the
// genuine cells into the user's u.  Shared memory stays within two CTAs per SM (fp64 10-row
// bands), the budget the issue-bound pass needs.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

template <class T>
struct UpArgs {
  Lvl L, Lc;          // fine level; layout of the coarse w / t arrays
  const T* uin;
  T* uout;
  const T* rhs_seg;   // segment-storage rhs (RG = 0)
  const T* w;         // coarse u after the recursion
  const T* t;         // coarse t (snapshot at the tau)
  T c0, cm, cr;
  FinalOut<T> fin;    // fin.p: last pass of the solve -- genuine cells to the user's u
  int foff[3];        // global index of the dense rhs array's element 0 (RG = 1)
};

template <class T, int PY, int BH, int MAXS, int RG>
struct UG {
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FP = RG ? PY + kAl : PY;
  static constexpr int NG = (BH + 2 + MAXS - 1) / MAXS;
  static constexpr int NT = PY * NG;
  static constexpr int TR = NG * MAXS;  // thread rows from s0
  static constexpr int A = 128 / (int)sizeof(T);
  static constexpr int U0S = ((TR + 2) * PY + A - 1) / A * A;
  static constexpr int FS = (TR * FP + A - 1) / A * A;
  static constexpr int U1S = U0S;
  static constexpr int RU = 3, RF = 4, NU1 = 3, RC = 3;
  static constexpr int CR = (TR + 2) / 2 + 3;  // coarse rows a band's u rows interpolate from
  static constexpr int CPY = PY / 2 + 4;       // row pitch of the coarse segment storage
  static constexpr int CPL = (CR * CPY + A - 1) / A * A;  // staged elements per plane, per array
  // X rows: coarse rows ybase .. ybase + FR - 1 with ybase = (oy + s0)/2 - 1, the first
  // parent row of the band's thread rows minus one; the rows of the band's thread and margin
  // rows (s0 - 1 .. s0 + TR) and their neighbours lie in it
  static constexpr int FR = TR / 2 + 3;
  static constexpr int XB = (FR * PY + A - 1) / A * A;
  static constexpr int RX = 3;                      // X planes in flight
  static constexpr int NFR = (FR + NG - 1) / NG;    // X rows built per thread
  static constexpr size_t smem() {
    return (size_t)(RU * U0S + RF * FS + NU1 * U1S + RX * XB + RC * 2 * CPL) * sizeof(T) +
           8 * (RU + RF + RC);
  }
};

template <class T, int PY, int BH, int MAXS, int RG, int FIN, int NB>
__global__ void __launch_bounds__(UG<T, PY, BH, MAXS, RG>::NT, NB)
    k_up2(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ UpArgs<T> a) {
  using G = UG<T, PY, BH, MAXS, RG>;
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
  T* xbuf = u1s + G::NU1 * G::U1S;       // [RX][FR][PY]: x-interpolants of w - t
  T* cws = xbuf + G::RX * G::XB;          // [RC][2][CPL]: w then t rows per coarse plane
  uint64_t* bars = reinterpret_cast<uint64_t*>(cws + G::RC * 2 * G::CPL);  // u0, f, coarse

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
  // coarse source: the fine segment's own coarse storage, or the single level-T array
  const int cseg = Lc.nsegs == 1 ? 0 : s;
  const int cpx = cseg % Lc.ns[0] + Lc.so[0], cpy = (cseg / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
            cpz = cseg / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
  const int ocx = cpx * Lc.S[0] - (Lc.J + 1), ocy = cpy * Lc.S[1] - (Lc.J + 1),
            ocz = cpz * Lc.S[2] - (Lc.J + 1);
  // coarse rows staged: parents of the band's loaded rows +-1, folded into Omega and into
  // the coarse storage box
  const int gy_lo = max(oy + q0, 0), gy_hi = min(oy + q1, L.N[1]) - 1;
  const int cy_lo = max(max((gy_lo >> 1) - 1, 0), ocy);
  const int cy_hi = min(min((gy_hi >> 1) + 1, Lc.N[1] - 1), ocy + Lc.E[1] - 1);
  const int ncr = max(cy_hi - cy_lo + 1, 1);
  const int gz_lo = max(oz, 0), gz_hi = min(oz + Ez, L.N[2]) - 1;
  // coarse planes: exactly those some F reads (P = gz/2 and its neighbour Q), so every
  // staged plane is waited on before its ring slot is reissued
  const int cz_lo = max(max((gz_lo - 1) >> 1, 0), ocz);
  const int cz_hi = min(min((gz_hi + 1) >> 1, Lc.N[2] - 1), ocz + Lc.E[2] - 1);
  const uint32_t cbytes = (uint32_t)(ncr * G::CPY * sizeof(T));
  const long long cofs = (long long)cseg * Lc.ss + (long long)(cy_lo - ocy) * G::CPY;
  uint64_t* cbar = bars + G::RU + G::RF;

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
  auto issue_c = [&](int c) {  // w and t rows of coarse plane c (global) into its ring slot
    const int sl = (c - cz_lo) % G::RC;
    mbar_expect_tx(&cbar[sl], 2 * cbytes);
    const long long o = cofs + (long long)(c - ocz) * Lc.pz;
    bulk_g2s(cws + (2 * sl) * G::CPL, a.w + o, cbytes, &cbar[sl]);
    bulk_g2s(cws + (2 * sl + 1) * G::CPL, a.t + o, cbytes, &cbar[sl]);
  };
  auto wait_c = [&](int c) {
    const int n = c - cz_lo;
    mbar_wait(&cbar[n % G::RC], (n / G::RC) & 1);
  };
  int nc = cz_lo;  // next coarse plane to stage (thread 0)
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    for (int z = 0; z < min(3, Ez); ++z) issue_f(z);
    for (; nc <= min(cz_hi, cz_lo + G::RC - 1); ++nc) issue_c(nc);
  }

  constexpr T W0 = T(0.75), W1 = T(0.25);
  const int tx = threadIdx.x % PY, g = threadIdx.x / PY;
  const int y0 = s0 + g * MAXS;
  const int gxv = ox + tx;
  const bool xin = tx < Ex && gxv >= 0 && gxv < L.N[0];
  const bool tok = tx < Ex && y0 < s1;
  const bool tin = tok && gxv >= 0 && gxv < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const int dxo = (gxv == 0 ? 1 : 0) + (gxv == L.N[0] - 1 ? 1 : 0);
  // x part of the interpolation for this column: parent X and neighbour Xq (reflected:
  // mirror cell, negative weight), offsets into a staged coarse row
  int cx0 = 0, cx1 = 0;
  T wx = W1;
  {
    const int X = gxv >> 1;
    int Xq = X + ((gxv & 1) ? 1 : -1);
    if (Xq < 0) { Xq = 0; wx = -W1; }
    if (Xq >= Lc.N[0]) { Xq = Lc.N[0] - 1; wx = -W1; }
    cx0 = min(max(X - ocx, 0), Lc.E[0] - 1);
    cx1 = min(max(Xq - ocx, 0), Lc.E[0] - 1);
  }
  // Per coarse plane c the CTA forms X_c[Y][x] = the x-interpolant of (w - t) at coarse row
  // Y and fine column x (weights 3/4, 1/4; reflected ghosts as signed weights, R3), the
  // ghost rows Y = -1 and Y = Nc as the negated rows 0 and Nc - 1.  Fine cell (x, gy, gz)
  // then gets  u += sum over (Y, wy) x (Z, wz) of wy wz X_Z[Y][x]  with Y = gy/2 (3/4) and
  // its neighbour (1/4), likewise Z: separable trilinear interpolation (fig:mgvsr L241).
  // The thread rows y0 .. y0+MAXS-1 start at the same parity in every group (MAXS even):
  // with p = (oy + s0) & 1 they read the MAXS/2 + 2 X rows from gyb/2 - 1 on, row k at
  // gyb/2 + (p + k)/2 and its neighbour.  Rows outside Omega or not loaded get none.
  const int gyb = oy + y0;
  const int ybase = ((oy + s0) >> 1) - 1;
  const bool par = ((oy + s0) & 1) != 0;
  const int fr0 = ((gyb >> 1) - 1 - ybase) * PY;  // X offset of the thread's first row
  auto rowok = [&](int y) {
    const int gy = oy + y;
    return y >= q0 && y < q1 && gy >= 0 && gy < L.N[1] && xin;
  };
  unsigned cor_mask = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k)
    if (rowok(y0 + k)) cor_mask |= 1u << k;
  const bool cor_all = cor_mask == (1u << MAXS) - 1;
  // the outermost loaded rows no thread owns: above the first thread row (group 0) and below
  // the last thread row (group NG - 1)
  const int ymarg = (g == 0) ? s0 - 1 : (g == G::NG - 1 ? s0 + G::TR : -1000);
  int mm0 = 0, mm1 = 0;
  const bool marg = ymarg > -1000 && rowok(ymarg);
  if (marg) {
    const int gy = oy + ymarg;
    mm0 = ((gy >> 1) - ybase) * PY;
    mm1 = mm0 + ((gy & 1) ? PY : -PY);
  }
  const int moff = (g == 0) ? -PY : MAXS * PY;

  // X of coarse plane c into its ring slot: this thread's column, rows g, g + NG, ...
  auto build_x = [&](int c) {
    const int sl = (c - cz_lo) % G::RC;
    const T* wr = cws + (2 * sl) * G::CPL;
    T* xr = xbuf + ((c - cz_lo) % G::RX) * G::XB + tx;
#pragma unroll
    for (int j = 0; j < G::NFR; ++j) {
      const int v = g + j * G::NG;
      if (v >= G::FR) break;
      const int Y = ybase + v;
      int src;
      T sg = T(1);
      if (Y >= cy_lo && Y <= cy_hi) src = Y - cy_lo;
      else if (Y == -1 && cy_lo == 0) { src = 0; sg = T(-1); }
      else if (Y == Lc.N[1] && cy_hi == Lc.N[1] - 1) { src = cy_hi - cy_lo; sg = T(-1); }
      else continue;
      const T* r = wr + src * G::CPY;
      const T d0 = r[cx0] - r[G::CPL + cx0], d1 = r[cx1] - r[G::CPL + cx1];
      xr[v * PY] = sg * (W0 * d0 + wx * d1);
    }
  };
  // the upper coarse plane fine plane z reads (the planes below it are built before it)
  auto need_hi = [&](int z) -> int {
    const int gz = oz + z;
    if (gz < gz_lo) return cz_lo - 1;
    if (gz > gz_hi) return cz_hi;
    const int P = gz >> 1;
    const int hi = (gz & 1) ? min(P + 1, Lc.N[2] - 1) : P;
    return min(max(hi, cz_lo), cz_hi);
  };
  int xb = cz_lo;  // next coarse plane to form X of (uniform)
  auto build_upto = [&](int z) {
    for (const int h = need_hi(z); xb <= h; ++xb) {
      wait_c(xb);
      build_x(xb);
    }
  };
  // corrections of the thread's MAXS rows of fine plane z into c[] (zero when not zon)
  auto corr_rows = [&](int z, bool zon, T (&c)[MAXS], T& cmarg) {
    const int gz = oz + z;
    const int P = gz >> 1;
    int Q = P + ((gz & 1) ? 1 : -1);
    T wz = W1;
    if (Q < 0) { Q = 0; wz = -W1; }
    if (Q >= Lc.N[2]) { Q = Lc.N[2] - 1; wz = -W1; }
    const int Pc = min(max(P, cz_lo), cz_hi), Qc = min(max(Q, cz_lo), cz_hi);
    const T* xp = xbuf + ((Pc - cz_lo) % G::RX) * G::XB + tx;
    const T* xq = xbuf + ((Qc - cz_lo) % G::RX) * G::XB + tx;
    T R[MAXS / 2 + 2];
#pragma unroll
    for (int j = 0; j < MAXS / 2 + 2; ++j) R[j] = W0 * xp[fr0 + j * PY] + wz * xq[fr0 + j * PY];
    auto rows = [&](auto PP) {
      constexpr int p = decltype(PP)::value;
      if (zon && cor_all) {
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const int ia = 1 + (p + k) / 2;                  // parent
          const int ib = ((p + k) & 1) ? ia + 1 : ia - 1;  // neighbour
          c[k] = W0 * R[ia] + W1 * R[ib];
        }
      } else {
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const int ia = 1 + (p + k) / 2;
          const int ib = ((p + k) & 1) ? ia + 1 : ia - 1;
          const bool on = zon && ((cor_mask >> k) & 1u);
          c[k] = on ? W0 * R[ia] + W1 * R[ib] : T(0);
        }
      }
    };
    if (par) rows(std::integral_constant<int, 1>{});
    else rows(std::integral_constant<int, 0>{});
    cmarg = (zon && marg) ? W0 * (W0 * xp[mm0] + wz * xq[mm0]) + W1 * (W0 * xp[mm1] + wz * xq[mm1])
                          : T(0);
  };

  unsigned c_mask = 0, w_mask = 0, yb_mask = 0, rw_mask = 0, ld_mask = 0;
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
  T dk[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) dk[k] = T(6 + dxo) + T((yb_mask >> (2 * k)) & 3u);
  T* const u0b = u0s + (y0 - s0 + 1) * PY + tx;
  const T* const fb = fs + (y0 - s0) * G::FP + tx + fsh;
  T* const u1b = u1s + (y0 - s0 + 1) * PY + tx;
  T* const ob = oseg + (long long)y0 * PY + tx;
  T u0q[MAXS][3], u1q[MAXS][3];

  // ---- prologue: X of the coarse planes fine planes 0 and 1 read, then plane 0 corrected
  build_upto(min(1, Ez - 1));
  mbar_wait(&bars[0], 0);
  __syncthreads();  // X complete
  if (threadIdx.x == 0)  // raw planes whose X is formed are free
    for (; nc <= cz_hi && nc < xb + G::RC; ++nc) issue_c(nc);
  {
    const int gz = oz;
    const bool zin = gz >= gz_lo && gz <= gz_hi;
    T cc[MAXS], cmg;
    corr_rows(0, zin, cc, cmg);
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      T v = ((ld_mask >> k) & 1u) ? u0b[k * PY] : T(0);
      const bool on = zin && ((cor_mask >> k) & 1u);
      v += cc[k];
      if (on) u0b[k * PY] = v;
      u0q[k][0] = v;
      u0q[k][1] = u0q[k][2] = T(0);
      u1q[k][0] = u1q[k][1] = u1q[k][2] = T(0);
    }
    if (zin && marg) u0b[moff] += cmg;
  }
  __syncthreads();  // plane 0 corrected for every reader
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0, cm = a.cm, cr = a.cr;

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3
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
      const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
      // correct plane z+1 (the X it reads were formed at the previous step) in registers and
      // in place
      const int gzn = gz + 1;
      const bool zn = z + 1 < Ez && gzn >= gz_lo && gzn <= gz_hi;
      T cc[MAXS], cmg;
      corr_rows(z + 1, zn, cc, cmg);
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        T v = (z + 1 < Ez) ? pn[k * PY] : T(0);
        const bool on = zn && ((cor_mask >> k) & 1u);
        v += cc[k];
        if (on) pn[k * PY] = v;
        u0q[k][IP] = v;
      }
      if (zn && marg) pn[moff] += cmg;
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
      // X of the coarse plane fine plane z+2 adds (its slot's plane is no longer read)
      if (z + 2 < Ez) build_upto(z + 2);
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      // (plane z's slot holds generic-proxy corrections: order them before the TMA write)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (z + G::RU < Ez) issue_u0(z + G::RU);
      if (z >= 1 && z + 2 < Ez) issue_f(z + 2);
      // raw planes whose X is formed are free
      for (; nc <= cz_hi && nc < xb + G::RC; ++nc) issue_c(nc);
    }
    if (z >= 1) {
      const int zz = z - 1;
      const int gz = oz + zz;
      if (gz >= 0 && gz < L.N[2]) {
        const bool zc = zz >= 1 && zz <= Ez - 2;
        const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
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
          const T v2 = ((act >> k) & 1u) ? c1 + cm * (c1 - u0v) + cr * r : u0v;
          if constexpr (FIN != 1) {
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
    for (int c = max(cz_lo, nc - G::RC); c < nc; ++c) wait_c(c);
}

template <class T, int PY, int BH, int MAXS, int NB>
bool try_up(const Lvl& L, const Lvl& Lc, const T* uin, T* uout, const T* w, const T* t,
            const FusedRhs<T>& b, double c0, double cm, double cr, FinalOut<T> fin,
            cudaStream_t st, bool launch) {
  using G1 = UG<T, PY, BH, MAXS, 1>;
  if (L.py != PY || L.E[0] > PY || Lc.py != G1::CPY || Lc.E[0] > G1::CPY) return false;
  const size_t smem = G1::smem();
  const size_t smax = (size_t)(NB >= 3 ? 75 : NB == 2 ? 113 : 227) * 1024;
  if (smem > smax) return false;
  if (!launch) return true;
  UpArgs<T> a{};
  a.L = L;
  a.Lc = Lc;
  a.uin = uin;
  a.uout = uout;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.w = w;
  a.t = t;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  a.fin = fin;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  dim3 grid((L.E[1] + BH - 1) / BH, L.nsegs);
  auto go = [&](auto kern, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, nt, smem, st>>>(map, a);
  };
  const bool f = fin.p != nullptr;
  if (b.global) {
    if (!encode_dense_tmap<T>(&map, b, UG<T, PY, BH, MAXS, 1>::FP, BH + 2)) return false;
    if (f) go(k_up2<T, PY, BH, MAXS, 1, 1, NB>, UG<T, PY, BH, MAXS, 1>::NT);
    else go(k_up2<T, PY, BH, MAXS, 1, 0, NB>, UG<T, PY, BH, MAXS, 1>::NT);
  } else {
    if (f) go(k_up2<T, PY, BH, MAXS, 0, 1, NB>, UG<T, PY, BH, MAXS, 0>::NT);
    else go(k_up2<T, PY, BH, MAXS, 0, 0, NB>, UG<T, PY, BH, MAXS, 0>::NT);
  }
  return true;
}

// band geometries: fp64 10-row bands of 4 cells per thread at E = 70 (216 threads, two CTAs
// per SM within 113 KB of shared memory), 14-row bands at E = 38; fp32 14-row bands of 8
template <class T>
bool up_dispatch(const Lvl& L, const Lvl& Lc, const T* uin, T* uout, const T* w, const T* t,
                 const FusedRhs<T>& b, double c0, double cm, double cr, FinalOut<T> fin,
                 cudaStream_t st, bool launch) {
  if (L.st27 || L.nlg != 0.0) return false;
  if constexpr (sizeof(T) == 8)
    return try_up<T, 72, 10, 4, 2>(L, Lc, uin, uout, w, t, b, c0, cm, cr, fin, st, launch) ||
           try_up<T, 40, 14, 4, 2>(L, Lc, uin, uout, w, t, b, c0, cm, cr, fin, st, launch);
  else
    return try_up<T, 72, 14, 8, 3>(L, Lc, uin, uout, w, t, b, c0, cm, cr, fin, st, launch) ||
           try_up<T, 40, 14, 8, 3>(L, Lc, uin, uout, w, t, b, c0, cm, cr, fin, st, launch);
}

}  // namespace

template <class T>
bool up2_fused_ok(const Lvl& L, const Lvl& Lc) {
  FusedRhs<T> b{};
  b.global = 1;
  return up_dispatch<T>(L, Lc, nullptr, nullptr, nullptr, nullptr, b, 0, 0, 0, FinalOut<T>{},
                        nullptr, false);
}

template <class T>
bool launch_up2_fused(const Lvl& L, const Lvl& Lc, const T* u_in, T* u_out, const T* w,
                      const T* t, FusedRhs<T> b, double c0, double cm, double cr,
                      cudaStream_t st, FinalOut<T> fin) {
  return up_dispatch<T>(L, Lc, u_in, u_out, w, t, b, c0, cm, cr, fin, st, true);
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
