// Fused multi-stage SR passes for sm_100a (see pass.cuh for the stage algebra).
//
// One pass = one HBM sweep over every segment of an SR level that chains the steps of a
// half V-cycle visit which the unfused schedule runs as separate kernels:
//
//   B      (PADD, 2, STORE|FINAL)   u += P(w - t); S^2          fig:mgvsr L241-242
//   A      (LOAD, 2, RESTRICT)      S^2; r = b - A u; restrict   fig:mgvsr L232-235
//   E      (PSET, 1|3, STORE|RESTRICT)  u = P(w); S^1 [; S^2 [; r; restrict]]
//                                                               fig:fmgsr L221-223 + L232-235
//
// Work unit: a y-band of one segment's storage box (grid = bands x segments); the CTA
// marches z.  Stage j of the chain runs one plane behind stage j-1 (register z-queues: plane
// p of every stage lives in slot p % 3) and on one row fewer on each side of the band (the
// band's halo rows are recomputed, so bands never exchange data).  Per plane, ONE thread
// streams the next planes of the fine u (cp.async.bulk), of the rhs (tensor TMA box of the
// dense f, or bulk rows of the segment rhs) and of the coarse w/t rows (cp.async.bulk) into
// shared-memory rings completing on mbarriers; each stage writes its plane to a double
// buffer for the x/y neighbours of the next stage; ONE __syncthreads per plane.
//
// Layout facts used: storage cells outside Omega are zero, so the reflected
// ghost -u_i (R3) is a +1 on the diagonal per out-of-domain neighbour; GSR cells are never
// smoothed (carried through every stage, R17); bands start at rows of even global index so
// every thread's MAXS rows hold whole 2x2 restriction/prolongation pairs, and lanes are
// rotated by the parity of the segment's x origin so that x-pairs are lane pairs (2m, 2m+1)
// of one warp (restriction sums with one shuffle).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "pass.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

template <class T>
struct PassArgs {
  Lvl L, Lc;
  const T* uin;
  T* uout;
  const T* rhs_seg;
  const T* w;
  const T* t;
  T* uc;
  T* rc;
  int jr;
  T cr[3];
  T cm;         // momentum of the last step (nstep >= 2)
  FinalOut<T> fin;
  int foff[3];  // global index of the dense rhs array's element 0 (tensor coordinates)
  int cpl;      // elements per staged coarse plane (one field)
};

constexpr long long rup(long long v, long long m) { return (v + m - 1) / m * m; }

template <class T, int PY, int BH, int MAXS, int SRC, int NSTEP, int SINK, int RG, int CL>
struct PassGeom {
  static constexpr int NS = NSTEP + (SINK == kSinkRestrict ? 1 : 0);  // stencil stages
  // CL = 0: bands recompute their halo rows (thread rows start NSE rows above the band);
  // CL = 1: the bands of a segment form a cluster and exchange halo rows through DSMEM, so
  // thread rows cover the band only (band 0 starts one row early to keep row pairs aligned)
  static constexpr int NSE = CL ? 0 : NS + (NS & 1);
  static constexpr int RW = CL ? (int)rup(BH + 1, MAXS) : (int)rup(BH + 1 + NS + NSE, MAXS);
  static constexpr int NG = RW / MAXS;
  static constexpr int NT = PY * NG;
  static constexpr int A = 128 / (int)sizeof(T);
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FPI = RG ? PY + kAl : PY;       // rhs smem row pitch
  static constexpr int PL = (int)rup((RW + 2) * PY, A);  // stage plane (one margin row each side)
  static constexpr int FPL = (int)rup(RW * FPI, A);
  static constexpr bool RING = SRC != kSrcPset;        // fine u streamed (LOAD / PADD)
  static constexpr int RU = RING ? 4 : 2;              // u ring (PSET: v0 double buffer)
  static constexpr int NBU = RING ? RU : 0;
  static constexpr int NSB = (SINK == kSinkRestrict) ? NSTEP : NSTEP - 1;  // staged step outputs
  static constexpr int RF = NS >= 4 ? NS + 1 : NS + 2;  // rhs ring
  static constexpr int FD = RF - NS;                    // rhs prefetch distance (planes)
  static constexpr int RC = (SRC == kSrcLoad) ? 0 : 5;  // coarse ring
  static constexpr int RCM = RC > 0 ? RC : 1;          // (modulus without a coarse ring)
  static constexpr int NF = (SRC == kSrcPadd) ? 2 : 1;  // coarse fields (w, t)
  static constexpr int NBAR = NBU + RF + RC;
  static constexpr int OFF_U = 0;
  static constexpr int OFF_S = OFF_U + RU * PL;
  static constexpr int OFF_F = OFF_S + 2 * NSB * PL;
  static constexpr int OFF_C = OFF_F + RF * FPL;
  static size_t smem(int cpl) { return (size_t)(OFF_C + RC * NF * cpl) * sizeof(T) + 8 * NBAR; }
  static int crows() { return RW / 2 + 2; }
  // 1 CTA per SM for the chains (2 for Pi + S^1 spills and measured no faster); the plain
  // residual + restriction pass (NSTEP = 0) fits two
  static constexpr int MINB = NSTEP == 0 ? 2 : 1;
};

template <class T, int PY, int BH, int MAXS, int SRC, int NSTEP, int SINK, int RG, int CL>
__global__ void __launch_bounds__(PassGeom<T, PY, BH, MAXS, SRC, NSTEP, SINK, RG, CL>::NT,
                                  PassGeom<T, PY, BH, MAXS, SRC, NSTEP, SINK, RG, CL>::MINB)
    k_pass(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ PassArgs<T> a) {
  using G = PassGeom<T, PY, BH, MAXS, SRC, NSTEP, SINK, RG, CL>;
  constexpr int NS = G::NS;
  constexpr bool RING = G::RING;
  constexpr bool RESTRICT = SINK == kSinkRestrict;
  constexpr bool COARSE = SRC != kSrcLoad;
  constexpr int NCR = MAXS / 2 + 2;  // coarse rows touched by a thread's MAXS fine rows
  static_assert(MAXS % 2 == 0 && MAXS <= 8, "MAXS even");
  static_assert(NSTEP >= 0 && NSTEP <= 3, "0..3 steps");
  static_assert(NSTEP >= 1 || (SRC == kSrcLoad && SINK == kSinkRestrict),
                "a pass without Chebyshev steps is the plain residual + restriction");
  extern __shared__ __align__(128) unsigned char sm[];
  T* const sbase = reinterpret_cast<T*>(sm);
  const Lvl& L = a.L;
  const Lvl& Lc = a.Lc;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int px = s % L.ns[0] + L.so[0];
  const int pyy = (s / L.ns[0]) % L.ns[1] + L.so[1];
  const int pzz = s / (L.ns[0] * L.ns[1]) + L.so[2];
  const int ox = px * L.S[0] - (L.J + 1);
  const int oy = pyy * L.S[1] - (L.J + 1);
  const int oz = pzz * L.S[2] - (L.J + 1);
  const int yal = oy & 1;
  const int r0 = blockIdx.x == 0 ? 0 : yal + (int)blockIdx.x * BH;  // output rows [r0, r1)
  const int r1 = min(Ey, yal + ((int)blockIdx.x + 1) * BH);
  const int nb = (int)gridDim.x;  // bands of a segment (= cluster size when CL)
  // first thread row; rows streamed (CL: the band plus one halo row each side)
  const int yb = CL ? (blockIdx.x == 0 ? -yal : r0) : yal + (int)blockIdx.x * BH - G::NSE;
  const int q0 = CL ? max(0, r0 - 1) : max(0, yb);
  const int q1 = CL ? min(Ey, r1 + 1) : min(Ey, yb + G::RW);
  const int fq0 = max(0, yb), fq1 = min(Ey, yb + G::RW);  // rhs rows (segment storage rhs)
  T* const bufU = sbase + G::OFF_U;
  T* const bufS = sbase + G::OFF_S;
  T* const bufF = sbase + G::OFF_F;
  T* const bufC = sbase + G::OFF_C;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(bufC + G::RC * G::NF * a.cpl);
  uint64_t* const barU = bars;
  uint64_t* const barF = bars + G::NBU;
  uint64_t* const barC = barF + G::RF;
  const T* const useg = RING ? a.uin + (long long)s * L.ss : nullptr;
  const uint32_t ubytes = (uint32_t)((q1 - q0) * PY * sizeof(T));
  const int uoff = (q0 - yb + 1) * PY;
  const T* const rseg = RG ? nullptr : a.rhs_seg + (long long)s * L.ss;
  const int oxt = ox - a.foff[0];
  const int oxa = oxt & ~(G::kAl - 1);
  const int fsh = RG ? oxt - oxa : 0;
  const uint32_t fbytes = RG ? (uint32_t)(G::RW * G::FPI * sizeof(T))
                              : (uint32_t)((fq1 - fq0) * PY * sizeof(T));
  const int foffs = RG ? 0 : (fq0 - yb) * PY;

  // coarse segment (PSET/PADD source, RESTRICT target): the fine segment's own coarse
  // storage on SR levels, the single global array at the transition level
  int cs = 0, ocx = 0, ocy = 0, ocz = 0;
  if constexpr (COARSE || RESTRICT) {
    cs = Lc.nsegs == 1 ? 0 : s;
    const int cpx = cs % Lc.ns[0] + Lc.so[0];
    const int cpy = (cs / Lc.ns[0]) % Lc.ns[1] + Lc.so[1];
    const int cpz = cs / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
    ocx = cpx * Lc.S[0] - (Lc.J + 1);
    ocy = cpy * Lc.S[1] - (Lc.J + 1);
    ocz = cpz * Lc.S[2] - (Lc.J + 1);
  }
  int cy_lo = 0, cy_hi = -1, cz_lo = 0, cz_hi = -1;
  uint32_t cbytes = 0;
  const T* cwseg = nullptr;
  const T* ctseg = nullptr;
  bool cvalid = false;
  if constexpr (COARSE) {
    // parents +-1 of the thread rows / in-domain planes, inside Omega_{l-1} and inside the
    // coarse storage box (rows beyond it belong only to dead thread rows)
    const int gy_lo = oy + yb, gy_hi = oy + yb + G::RW - 1;
    cy_lo = max(max((gy_lo >> 1) - 1, 0), ocy);
    cy_hi = min(min((gy_hi >> 1) + 1, Lc.N[1] - 1), ocy + Lc.E[1] - 1);
    const int gz_lo = max(oz, 0), gz_hi = min(oz + Ez, L.N[2]) - 1;
    cz_lo = max(max((gz_lo >> 1) - 1, 0), ocz);
    cz_hi = min(min((gz_hi >> 1) + 1, Lc.N[2] - 1), ocz + Lc.E[2] - 1);
    cvalid = cy_hi >= cy_lo && cz_hi >= cz_lo;
    cbytes = cvalid ? (uint32_t)((cy_hi - cy_lo + 1) * Lc.py * sizeof(T)) : 0u;
    cwseg = a.w + (long long)cs * Lc.ss + (long long)(cy_lo - ocy) * Lc.py;
    if constexpr (SRC == kSrcPadd) ctseg = a.t + (long long)cs * Lc.ss + (long long)(cy_lo - ocy) * Lc.py;
  }

  if (threadIdx.x == 0) {
    for (int i = 0; i < G::NBAR; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (CL)
    cooperative_groups::this_cluster().sync();  // every band's smem exists before DSMEM use
  else
    __syncthreads();
  auto issue_u = [&](int z) {
    const int sl = z % G::RU;
    mbar_expect_tx(&barU[sl], ubytes);
    bulk_g2s(bufU + sl * G::PL + uoff, useg + (long long)z * pz + (long long)q0 * PY, ubytes,
             &barU[sl]);
  };
  auto issue_f = [&](int z) {
    const int sl = z % G::RF;
    mbar_expect_tx(&barF[sl], fbytes);
    if constexpr (RG)
      tma_3d(bufF + sl * G::FPL, &fmap, oxa, oy + yb - a.foff[1], oz + z - a.foff[2], &barF[sl]);
    else
      bulk_g2s(bufF + sl * G::FPL + foffs, rseg + (long long)z * pz + (long long)fq0 * PY, fbytes,
               &barF[sl]);
  };
  auto issue_c = [&](int c) {
    const int n = c - cz_lo, sl = n % G::RCM;
    // a staged plane may never be read (the parent-1 plane of an odd first fine plane):
    // let its copy land before the slot is re-armed (one phase in flight per barrier)
    if (n >= G::RC) mbar_wait(&barC[sl], ((n - G::RC) / G::RCM) & 1);
    mbar_expect_tx(&barC[sl], G::NF * cbytes);
    const long long zo = (long long)(c - ocz) * Lc.pz;
    T* dst = bufC + sl * G::NF * a.cpl;
    bulk_g2s(dst, cwseg + zo, cbytes, &barC[sl]);
    if constexpr (SRC == kSrcPadd) bulk_g2s(dst + a.cpl, ctseg + zo, cbytes, &barC[sl]);
  };
  int nc = cz_lo;  // next coarse plane to stream (thread 0)
  if (threadIdx.x == 0) {
    if constexpr (RING)
      for (int z = 0; z < min(G::RU - 1, Ez); ++z) issue_u(z);
    for (int z = 0; z < min(G::FD, Ez); ++z) issue_f(z);
    if constexpr (COARSE)
      if (cvalid)
        for (; nc <= min(cz_hi, cz_lo + G::RC - 1); ++nc) issue_c(nc);
  }

  // ---- this thread: column tx (lanes rotated by the x-origin parity), rows y0 .. y0+MAXS-1
  const int lane = threadIdx.x % PY, g = threadIdx.x / PY;
  int tx = lane + (ox & 1);
  if (tx >= PY) tx -= PY;
  const int y0 = yb + g * MAXS;
  const int gx = ox + tx;
  const bool colok = tx < Ex;
  const bool xin = colok && gx >= 0 && gx < L.N[0];
  const bool xc = tx >= 1 && tx <= Ex - 2;
  const T six = T(6 + (gx == 0 ? 1 : 0) + (gx == L.N[0] - 1 ? 1 : 0));
  unsigned inm = 0, cmk = 0, wmk = 0, ydg = 0;
  unsigned vm[NS + 1];
#pragma unroll
  for (int j = 0; j <= NS; ++j) vm[j] = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k, gy = oy + y;
    const bool rowin = y >= 0 && y < Ey;
    const bool in = xin && rowin && gy >= 0 && gy < L.N[1];
    if (in) inm |= 1u << k;
    if (in && xc && y >= 1 && y <= Ey - 2) cmk |= 1u << k;
    if (in && y >= r0 && y < r1) wmk |= 1u << k;
    ydg |= (unsigned)((gy == 0 ? 1 : 0) + (gy == L.N[1] - 1 ? 1 : 0)) << (2 * k);
#pragma unroll
    for (int j = 0; j <= NS; ++j) {
      const int hw = CL ? 0 : NS - j;  // rows recomputed beyond the band by stage j
      if (y >= r0 - hw && y < r1 + hw) vm[j] |= 1u << k;
    }
  }
  // CL: the y-halo rows of every stage input (rows r0 - 1 and r1) live in the neighbouring
  // bands' shared memory; the two slots that need them read them through DSMEM once per
  // plane step, right after the cluster barrier that published them
  unsigned hu = 0, hd = 0;
  const T* nb_up = nullptr;
  const T* nb_dn = nullptr;
  int hoff_up = 0, hoff_dn = 0;
  if constexpr (CL) {
    const int b = (int)blockIdx.x;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const int y = y0 + k;
      if (b > 0 && y == r0 && tx < Ex) hu |= 1u << k;
      if (b < nb - 1 && y == r1 - 1 && tx < Ex) hd |= 1u << k;
    }
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    if (b > 0) nb_up = cl.map_shared_rank(sbase, b - 1);
    if (b < nb - 1) nb_dn = cl.map_shared_rank(sbase, b + 1);
    const int yb_up = (b - 1 == 0) ? -yal : yal + (b - 1) * BH;
    const int yb_dn = yal + (b + 1) * BH;
    hoff_up = (r0 - 1 - yb_up + 1) * PY + tx;
    hoff_dn = (r1 - yb_dn + 1) * PY + tx;
  }
  T hup[NS + 1], hdn[NS + 1];
#pragma unroll
  for (int j = 0; j <= NS; ++j) hup[j] = hdn[j] = T(0);
  // element offset (from the smem base) of the input plane of stage j (1..NS) at plane zj
  auto in_off = [&](int j, int zj) -> int {
    if (j == 1) return G::OFF_U + (RING ? (zj % G::RU) : (zj & 1)) * G::PL;
    return G::OFF_S + (2 * (j - 2) + (zj & 1)) * G::PL;
  };

  // diagonal of A per slot: 6 + one per reflected (out-of-domain) x/y neighbour (R3);
  // the z part is added per plane
  T dk[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) dk[k] = six + T((ydg >> (2 * k)) & 3u);
  const int po = (g * MAXS + 1) * PY + tx;  // own row 0 in a stage plane
  const int fo = g * MAXS * G::FPI + tx + fsh;
  const T ih2 = T(L.inv_h2);

  // prolongation (R10): separable trilinear, weights 3/4 (parent) and 1/4 (neighbour on
  // the child's side); reflected coarse ghosts (R3) enter as signed weights
  constexpr T W0 = T(0.75), W1 = T(0.25);
  int cx0 = 0, cx1 = 0;
  T W1x = W1;
  int cro[NCR];
  T cys[NCR];
  if constexpr (COARSE) {
    const int X = gx >> 1;
    int Xq = X + ((gx & 1) ? 1 : -1);
    if (Xq < 0) { Xq = 0; W1x = -W1; }
    if (Xq >= Lc.N[0]) { Xq = Lc.N[0] - 1; W1x = -W1; }
    cx0 = min(max(X - ocx, 0), Lc.E[0] - 1);
    cx1 = min(max(Xq - ocx, 0), Lc.E[0] - 1);
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
  auto wait_c = [&](int c) {
    const int n = c - cz_lo;
    mbar_wait(&barC[n % G::RCM], (n / G::RCM) & 1);
  };
  // xy-interpolant of staged coarse plane c for the thread's rows
  auto interp = [&](int c, T (&I)[MAXS]) {
    const T* cw = bufC + ((c - cz_lo) % G::RCM) * G::NF * a.cpl;
    T xi[NCR];
#pragma unroll
    for (int m = 0; m < NCR; ++m) {
      const T* row = cw + cro[m];
      T a0 = row[cx0], a1 = row[cx1];
      if constexpr (SRC == kSrcPadd) {
        a0 -= row[a.cpl + cx0];
        a1 -= row[a.cpl + cx1];
      }
      xi[m] = cys[m] * (W0 * a0 + W1x * a1);
    }
#pragma unroll
    for (int k = 0; k < MAXS; ++k) I[k] = W0 * xi[k / 2 + 1] + W1 * xi[(k & 1) ? k / 2 + 2 : k / 2];
  };

  // I(c) with the reflected coarse ghost planes I(-1) = -I(0), I(Nc) = -I(Nc-1) (R3)
  auto get_c = [&](int c, T (&I)[MAXS]) {
    const int cc = min(max(c, 0), Lc.N[2] - 1);
    wait_c(cc);
    interp(cc, I);
    if (cc != c) {
#pragma unroll
      for (int k = 0; k < MAXS; ++k) I[k] = -I[k];
    }
  };
  T Iprev[MAXS], Icur[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) Iprev[k] = Icur[k] = T(0);

  // restriction target box (coarse global indices): F of half-width jr around V_{l-1}^p
  bool rx = false;
  unsigned ryk = 0;
  int rzlo = 0, rzhi = 0;
  if constexpr (RESTRICT) {
    const int hx = L.S[0] / 2, hy = L.S[1] / 2, hz = L.S[2] / 2;
    const int xlo = max(px * hx - a.jr, 0), xhi = min(px * hx + hx + a.jr, Lc.N[0]);
    const int ylo = max(pyy * hy - a.jr, 0), yhi = min(pyy * hy + hy + a.jr, Lc.N[1]);
    rzlo = max(pzz * hz - a.jr, 0);
    rzhi = min(pzz * hz + hz + a.jr, Lc.N[2]);
    const int X = gx >> 1;
    rx = ((lane & 1) == 0) && xin && X >= xlo && X < xhi;
#pragma unroll
    for (int k = 0; k < MAXS; k += 2) {
      const int y = y0 + k, gy = oy + y;
      const int Y = gy >> 1;
      if (y >= r0 && y + 1 < r1 && Y >= ylo && Y < yhi) ryk |= 1u << (k / 2);
    }
  }
  // lanes present in this thread's warp (the last warp of the CTA may be partial)
  const unsigned wmask = (G::NT % 32 == 0 || (int)threadIdx.x < G::NT / 32 * 32)
                             ? 0xffffffffu
                             : ((1u << (G::NT % 32)) - 1u);

  T q[NSTEP + 1][MAXS][3];
#pragma unroll
  for (int j = 0; j <= NSTEP; ++j)
#pragma unroll
    for (int k = 0; k < MAXS; ++k) q[j][k][0] = q[j][k][1] = q[j][k][2] = T(0);
  T au[MAXS / 2], ar[MAXS / 2];
#pragma unroll
  for (int k = 0; k < MAXS / 2; ++k) au[k] = ar[k] = T(0);

  auto iter = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3
    if constexpr (CL) {
#pragma unroll
      for (int j = 1; j <= NS; ++j) {
        const int zj = z - j;
        if (zj >= 0 && zj < Ez) {
          const int o = in_off(j, zj);
          if (hu) hup[j] = nb_up[o + hoff_up];
          if (hd) hdn[j] = nb_dn[o + hoff_dn];
        }
      }
    }
    // ------------------------------------------------------------ source at plane z
    if (z < Ez) {
      const int gz = oz + z;
      [[maybe_unused]] const bool zin = gz >= 0 && gz < L.N[2];
      T* const up = bufU + (RING ? (z % G::RU) : (z & 1)) * G::PL + po;
      if constexpr (RING) mbar_wait(&barU[z % G::RU], (z / G::RU) & 1);
      T pv[MAXS];
#pragma unroll
      for (int k = 0; k < MAXS; ++k) pv[k] = T(0);
      if constexpr (COARSE) {
        // the xy-interpolant of every coarse plane is formed once and kept in registers:
        // fine plane 2P uses I(P), I(P-1); fine plane 2P+1 uses I(P), I(P+1)
        if (zin) {
          const int P = gz >> 1;
          if (gz == max(oz, 0)) {  // first in-domain plane of the segment
            get_c(P, Icur);
            if (!(gz & 1)) get_c(P - 1, Iprev);
          }
          if (gz & 1) {
            T In[MAXS];
            get_c(P + 1, In);
#pragma unroll
            for (int k = 0; k < MAXS; ++k) {
              pv[k] = W0 * Icur[k] + W1 * In[k];
              Iprev[k] = Icur[k];
              Icur[k] = In[k];
            }
          } else {
#pragma unroll
            for (int k = 0; k < MAXS; ++k) pv[k] = W0 * Icur[k] + W1 * Iprev[k];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        T v = T(0);
        if constexpr (RING) v = up[k * PY];
        if constexpr (COARSE) {
          const bool in = zin && ((inm >> k) & 1u);
          const T pw = (SRC == kSrcPadd) ? v + pv[k] : pv[k];
          v = in ? pw : v;
        }
        q[0][k][R] = v;
        if constexpr (SRC != kSrcLoad) up[k * PY] = v;
      }
    }
    // ------------------------------------------------------------ steps j = 1..NSTEP
    auto stage = [&](auto JJ) {
      constexpr int j = decltype(JJ)::value;
      const int zj = z - j;
      if (zj < 0 || zj >= Ez) return;
      constexpr int I0 = ((R - j) % 3 + 3) % 3, IM = (I0 + 2) % 3, IP = (I0 + 1) % 3;
      if (j == 1) mbar_wait(&barF[zj % G::RF], (zj / G::RF) & 1);
      const int gz = oz + zj;
      const bool zc = zj >= 1 && zj <= Ez - 2 && gz >= 0 && gz < L.N[2];
      const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
      const T* src;
      if constexpr (j == 1)
        src = bufU + (RING ? (zj % G::RU) : (zj & 1)) * G::PL + po;
      else
        src = bufS + (2 * (j - 2) + (zj & 1)) * G::PL + po;
      const T* fp = bufF + (zj % G::RF) * G::FPL + fo;
      constexpr bool STAGED = j < NSTEP || RESTRICT;
      T* dst = STAGED ? bufS + (2 * (j - 1) + (zj & 1)) * G::PL + po : nullptr;
      const unsigned act = zc ? (cmk & vm[j]) : 0u;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        // branch-free: every slot computes, the C-cell predicate selects (GSR, dead rows
        // and out-of-domain cells carry their value through)
        const T v = q[j - 1][k][I0];
        T ym = (k == 0) ? src[-PY] : q[j - 1][k > 0 ? k - 1 : 0][I0];
        T yp = (k == MAXS - 1) ? src[MAXS * PY] : q[j - 1][k + 1 < MAXS ? k + 1 : k][I0];
        if constexpr (CL) {
          ym = ((hu >> k) & 1u) ? hup[j] : ym;
          yp = ((hd >> k) & 1u) ? hdn[j] : yp;
        }
        const T sum = ((q[j - 1][k][IM] + q[j - 1][k][IP]) + (ym + yp)) +
                      (src[k * PY - 1] + src[k * PY + 1]);
        const T r = fp[k * G::FPI] - ((dk[k] + dz) * v - sum) * ih2;
        T o;
        if constexpr (j == NSTEP && NSTEP >= 2)
          o = v + a.cm * (v - q[j - 2][k][I0]) + a.cr[j - 1] * r;
        else
          o = v + a.cr[j - 1] * r;
        o = ((act >> k) & 1u) ? o : v;
        q[j][k][I0] = o;
        if constexpr (STAGED) dst[k * PY] = o;
      }
      if constexpr (j == NSTEP) {
        if (gz >= 0 && gz < L.N[2]) {
          if constexpr (SINK == kSinkFinal) {
            const int vlo = L.J + 1;
            if (tx >= vlo && tx < vlo + L.S[0] && zj >= vlo && zj < vlo + L.S[2]) {
              T* orow = a.fin.p + (long long)(gz - a.fin.bo[2]) * a.fin.sz +
                        (long long)(oy + y0 - a.fin.bo[1]) * a.fin.sy + (gx - a.fin.bo[0]);
#pragma unroll
              for (int k = 0; k < MAXS; ++k) {
                const int y = y0 + k;
                if (((wmk >> k) & 1u) && y >= vlo && y < vlo + L.S[1]) orow[k * a.fin.sy] = q[j][k][I0];
              }
            }
          } else {
            T* orow = a.uout + (long long)s * L.ss + (long long)zj * pz + (long long)y0 * PY + tx;
#pragma unroll
            for (int k = 0; k < MAXS; ++k)
              if ((wmk >> k) & 1u) orow[k * PY] = q[j][k][I0];
          }
        }
      }
    };
    if constexpr (NSTEP >= 1) stage(std::integral_constant<int, 1>{});
    if constexpr (NSTEP >= 2) stage(std::integral_constant<int, 2>{});
    if constexpr (NSTEP >= 3) stage(std::integral_constant<int, 3>{});
    // ------------------------------------------------------------ residual + restriction
    if constexpr (RESTRICT) {
      const int zr = z - NS;
      if (zr >= 0 && zr < Ez) {
        constexpr int I0 = ((R - NS) % 3 + 3) % 3, IM = (I0 + 2) % 3, IP = (I0 + 1) % 3;
        const int gz = oz + zr;
        const bool zc = zr >= 1 && zr <= Ez - 2 && gz >= 0 && gz < L.N[2];
        const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
        const T* src = sbase + in_off(NS, zr) + po;  // input of the residual stage
        const T* fp = bufF + (zr % G::RF) * G::FPL + fo;
        if (NSTEP == 0) mbar_wait(&barF[zr % G::RF], (zr / G::RF) & 1);
        const unsigned act = zc ? (cmk & vm[NS]) : 0u;
        T rv[MAXS];
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const T v = q[NSTEP][k][I0];
          T ym = (k == 0) ? src[-PY] : q[NSTEP][k > 0 ? k - 1 : 0][I0];
          T yp = (k == MAXS - 1) ? src[MAXS * PY] : q[NSTEP][k + 1 < MAXS ? k + 1 : k][I0];
          if constexpr (CL) {
            ym = ((hu >> k) & 1u) ? hup[NS] : ym;
            yp = ((hd >> k) & 1u) ? hdn[NS] : yp;
          }
          const T sum = ((q[NSTEP][k][IM] + q[NSTEP][k][IP]) + (ym + yp)) +
                        (src[k * PY - 1] + src[k * PY + 1]);
          const T r = fp[k * G::FPI] - ((dk[k] + dz) * v - sum) * ih2;
          rv[k] = ((act >> k) & 1u) ? r : T(0);
        }
        const bool zodd = (gz & 1) != 0;
        const int Z = gz >> 1;
        const bool zok = zodd && zr >= 1 && Z >= rzlo && Z < rzhi;
#pragma unroll
        for (int kk = 0; kk < MAXS / 2; ++kk) {
          T su = q[NSTEP][2 * kk][I0] + q[NSTEP][2 * kk + 1][I0];
          T sr = rv[2 * kk] + rv[2 * kk + 1];
          su += __shfl_xor_sync(wmask, su, 1);
          sr += __shfl_xor_sync(wmask, sr, 1);
          if (!zodd) {
            au[kk] = su;
            ar[kk] = sr;
          } else {
            au[kk] += su;
            ar[kk] += sr;
            if (zok && rx && ((ryk >> kk) & 1u)) {
              const int Y = (oy + y0 + 2 * kk) >> 1;
              const long long ci = (long long)cs * Lc.ss + (long long)(Z - ocz) * Lc.pz +
                                   (long long)(Y - ocy) * Lc.py + ((gx >> 1) - ocx);
              a.uc[ci] = au[kk] * T(0.125);
              a.rc[ci] = ar[kk] * T(0.125);
            }
          }
        }
      }
    }
    if constexpr (CL)
      cooperative_groups::this_cluster().sync();  // planes (and halo rows) published
    else
      __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if constexpr (RING)
        if (z + G::RU - 1 < Ez) issue_u(z + G::RU - 1);  // slot of plane z-1 is free
      if (z + G::FD < Ez) issue_f(z + G::FD);            // slot of plane z-NS is free
      if constexpr (COARSE) {
        if (cvalid) {
          const int live = max(cz_lo, ((oz + z + 1) >> 1) - 1);
          for (; nc <= cz_hi && nc < live + G::RC; ++nc) issue_c(nc);
        }
      }
    }
  };
  const int nz = Ez + NS;
  for (int zb = 0; zb < nz; zb += 3) {
    iter(std::integral_constant<int, 0>{}, zb);
    if (zb + 1 < nz) iter(std::integral_constant<int, 1>{}, zb + 1);
    if (zb + 2 < nz) iter(std::integral_constant<int, 2>{}, zb + 2);
  }
  // no bulk copy may still target this CTA's shared memory when it exits
  if constexpr (COARSE) {
    if (threadIdx.x == 0 && cvalid)
      for (int c = max(cz_lo, nc - G::RC); c < nc; ++c) wait_c(c);
  }
}

// Copy the restriction target box of every fine segment (F^p of half-width jr, or V_T^p)
// from src to dst on the coarse level: the entry pass restricts into the coarse t buffer
// because the coarse u is still being read by the same pass (Pi), see launch_pass_merge.
template <class T>
__global__ void __launch_bounds__(256) k_merge_f(Lvl L, Lvl Lc, const T* __restrict__ src,
                                                 T* __restrict__ dst, int jr) {
  const int s = blockIdx.y;
  const int p[3] = {s % L.ns[0] + L.so[0], (s / L.ns[0]) % L.ns[1] + L.so[1],
                    s / (L.ns[0] * L.ns[1]) + L.so[2]};
  const int cs = Lc.nsegs == 1 ? 0 : s;
  const int cp[3] = {cs % Lc.ns[0] + Lc.so[0], (cs / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
                     cs / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2]};
  int lo[3], n[3], oc[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int h = L.S[d] / 2;
    lo[d] = max(p[d] * h - jr, 0);
    n[d] = min(p[d] * h + h + jr, Lc.N[d]) - lo[d];
    oc[d] = cp[d] * Lc.S[d] - (Lc.J + 1);
  }
  const long long cnt = (long long)n[0] * n[1] * n[2];
  const long long base = (long long)cs * Lc.ss;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < cnt; i += (long long)gridDim.x * 256) {
    const int x = (int)(i % n[0]);
    const int y = (int)((i / n[0]) % n[1]);
    const int z = (int)(i / ((long long)n[0] * n[1]));
    const long long o = base + (long long)(lo[2] + z - oc[2]) * Lc.pz +
                        (long long)(lo[1] + y - oc[1]) * Lc.py + (lo[0] + x - oc[0]);
    dst[o] = src[o];
  }
}

// ---- host side ---------------------------------------------------------------------
template <class T, int PY, int BH, int MAXS, int SRC, int NSTEP, int SINK, int RG, int CL>
bool inst(const PassSpec<T>& ps, cudaStream_t st, bool launch) {
  using G = PassGeom<T, PY, BH, MAXS, SRC, NSTEP, SINK, RG, CL>;
  const Lvl& L = ps.L;
  if (L.py != PY || L.E[0] > PY) return false;
  PassArgs<T> a{};
  a.cpl = (SRC != kSrcLoad) ? (int)rup((long long)G::crows() * ps.Lc.py, G::A) : 0;
  const size_t smem = G::smem(a.cpl);
  if (smem > 227 * 1024) return false;
  if (!launch) return true;
  a.L = L;
  a.Lc = ps.Lc;
  a.uin = ps.uin;
  a.uout = ps.uout;
  a.rhs_seg = ps.rhs.global ? nullptr : ps.rhs.p;
  a.w = ps.w;
  a.t = ps.t;
  a.uc = ps.uc;
  a.rc = ps.rc;
  a.jr = ps.jr;
  for (int i = 0; i < 3; ++i) a.cr[i] = (T)ps.cr[i];
  a.cm = (T)(NSTEP >= 2 ? ps.cm[NSTEP >= 2 ? NSTEP - 1 : 0] : 0.0);
  a.fin = ps.fin;
  for (int d = 0; d < 3; ++d) a.foff[d] = ps.rhs.global ? ps.rhs.off[d] : 0;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (RG && !encode_dense_tmap<T>(&map, ps.rhs, G::FPI, G::RW)) return false;
  const int oy = L.so[1] * L.S[1] - (L.J + 1);  // parity of every segment's y origin
  const int yal = oy & 1;
  const int nb = (L.E[1] - yal + BH - 1) / BH;
  if (CL && (nb < 2 || nb > 8)) return false;  // one cluster per segment (portable size)
  auto kern = k_pass<T, PY, BH, MAXS, SRC, NSTEP, SINK, RG, CL>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  if constexpr (CL) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nb, L.nsegs);
    cfg.blockDim = dim3(G::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nb;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, map, a);
  } else {
    kern<<<dim3(nb, L.nsegs), G::NT, smem, st>>>(map, a);
  }
  return true;
}

int max_py() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("SR_FMG_PASS_MAXPY");
    v = e ? std::atoi(e) : 1 << 20;
  }
  return v;
}

template <class T, int SRC, int NSTEP, int SINK, int RG>
bool by_geom(const PassSpec<T>& ps, cudaStream_t st, bool launch) {
  if (ps.L.py > max_py()) return false;
  // only the E = 70 geometry (64^3 segments, J = 2): on smaller boxes the band halos and
  // the low occupancy make the fused pass slower than the separate kernels (measured)
  // SR_FMG_PASS_CL=1: the cluster/DSMEM variant (no recomputed halos; one CTA of 9 warps
  // per SM and a cluster barrier per plane: measured 1.5-1.7x slower than recomputing)
  static int cl = -1;
  if (cl < 0) {
    const char* e = std::getenv("SR_FMG_PASS_CL");
    cl = (e && e[0] == '1') ? 1 : 0;
  }
  if (cl) return inst<T, 72, 14, 4, SRC, NSTEP, SINK, RG, 1>(ps, st, launch);
  if constexpr (NSTEP == 0)  // the plain residual + restriction also on E = 38 boxes
    if (inst<T, 40, 12, 4, SRC, NSTEP, SINK, RG, 0>(ps, st, launch)) return true;
  return inst<T, 72, 14, 4, SRC, NSTEP, SINK, RG, 0>(ps, st, launch);
}

template <class T>
bool dispatch(const PassSpec<T>& ps, cudaStream_t st, bool launch) {
  const int g = ps.rhs.global;
  const int key = ps.src * 100 + ps.nstep * 10 + ps.sink;
  switch (key) {
    case kSrcPadd * 100 + 20 + kSinkStore:
      return g ? by_geom<T, kSrcPadd, 2, kSinkStore, 1>(ps, st, launch)
               : by_geom<T, kSrcPadd, 2, kSinkStore, 0>(ps, st, launch);
    case kSrcPadd * 100 + 20 + kSinkFinal:
      return g && by_geom<T, kSrcPadd, 2, kSinkFinal, 1>(ps, st, launch);
    case kSrcLoad * 100 + 0 + kSinkRestrict:
      return g ? by_geom<T, kSrcLoad, 0, kSinkRestrict, 1>(ps, st, launch)
               : by_geom<T, kSrcLoad, 0, kSinkRestrict, 0>(ps, st, launch);
    case kSrcLoad * 100 + 20 + kSinkRestrict:
      return g ? by_geom<T, kSrcLoad, 2, kSinkRestrict, 1>(ps, st, launch)
               : by_geom<T, kSrcLoad, 2, kSinkRestrict, 0>(ps, st, launch);
    case kSrcPset * 100 + 10 + kSinkStore:
      return g && by_geom<T, kSrcPset, 1, kSinkStore, 1>(ps, st, launch);
    case kSrcPset * 100 + 30 + kSinkStore:
      return g && by_geom<T, kSrcPset, 3, kSinkStore, 1>(ps, st, launch);
    case kSrcPset * 100 + 30 + kSinkRestrict:
      return g && by_geom<T, kSrcPset, 3, kSinkRestrict, 1>(ps, st, launch);
    default:
      return false;
  }
}

}  // namespace

template <class T>
bool pass_ok(int src, int nstep, int sink, const Lvl& L, const Lvl& Lc, int rhs_global) {
  if (L.S[0] % 2 || L.S[1] % 2 || L.S[2] % 2) return false;
  PassSpec<T> ps{};
  ps.src = src;
  ps.nstep = nstep;
  ps.sink = sink;
  ps.L = L;
  ps.Lc = Lc;
  ps.rhs.global = rhs_global;
  return dispatch<T>(ps, nullptr, false);
}

template <class T>
bool launch_pass(const PassSpec<T>& ps, cudaStream_t st) {
  if (ps.L.S[0] % 2 || ps.L.S[1] % 2 || ps.L.S[2] % 2) return false;
  return dispatch<T>(ps, st, true);
}

template <class T>
void launch_merge_f(const Lvl& L, const Lvl& Lc, const T* src, T* dst, int jr, cudaStream_t st) {
  long long box = 1;
  for (int d = 0; d < 3; ++d) box *= L.S[d] / 2 + 2 * jr;
  const int gx = (int)std::max<long long>(1, std::min<long long>(32, (box + 1023) / 1024));
  k_merge_f<T><<<dim3(gx, L.nsegs), 256, 0, st>>>(L, Lc, src, dst, jr);
}

template void launch_merge_f<double>(const Lvl&, const Lvl&, const double*, double*, int,
                                     cudaStream_t);
template void launch_merge_f<float>(const Lvl&, const Lvl&, const float*, float*, int,
                                    cudaStream_t);
template bool pass_ok<double>(int, int, int, const Lvl&, const Lvl&, int);
template bool pass_ok<float>(int, int, int, const Lvl&, const Lvl&, int);
template bool launch_pass<double>(const PassSpec<double>&, cudaStream_t);
template bool launch_pass<float>(const PassSpec<float>&, cudaStream_t);

}  // namespace srfmg
