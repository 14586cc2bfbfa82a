// Fused, TMA-fed degree-2 Chebyshev pass (both sweeps of R8 in one HBM pass), sm_100a.
//
// Work unit: one y-band of one segment's storage box (rows [r0, r1) of every plane).  The
// CTA marches z.  The inputs of each plane -- the band's u rows (+-2 halo rows) and the
// rhs rows (+-1) -- are contiguous in HBM (segment storage) or a box of the dense f, and
// are streamed into a 4-deep shared-memory ring by ONE thread with cp.async.bulk /
// cp.async.bulk.tensor (TMA) completing on mbarriers, so the loads of the next planes are
// in flight while the CTA computes (no register-bound memory-level parallelism).
//
// Per plane z:   stage 1 at plane z     u1 = u0 + (b - A u0)/theta          (rows r0-1..r1)
//                stage 2 at plane z-1   u2 = u1 + rho1 rho0 (u1 - u0) + (2 rho1/delta)(b - A u1)
// Each thread owns up to MAXS fixed (x, y) cells of the band and keeps their z-columns of
// u0 (z-1, z, z+1) and u1 (z-2, z-1, z) in registers; x/y neighbours come from the smem
// planes (u0 ring; u1 double buffer).  Stage 1 is recomputed on one halo row each side so
// stage 2 needs no exchange between bands.  GSR cells (frozen) are
// copied; A = -Lap_h with reflected ghosts at the domain boundary (R1-R3).
// Output goes to the other ping-pong buffer (bands of one segment run concurrently, so an
// in-place write could race with a neighbour band's halo loads).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

constexpr int kRing = 4;

template <class T>
struct Cheb2Args {
  Lvl L;
  const T* uin;
  T* uout;
  const T* rhs_seg;  // segment-storage rhs (rhs_global == 0)
  int rhs_global;
  int BH;            // output rows per band
  int u0_stride;     // elements per u0 ring plane buffer
  int s_stride;      // elements per u1 plane buffer
  int f_stride;      // elements per rhs plane buffer
  int bw;            // rhs tensor-map box width (global rhs; 16-byte aligned start)
  T c0, cm, cr;
  FinalOut<T> fin;   // fin.p non-null: write only genuine cells, to the user's u block (last pass)
  // tau fused in front (FIN = 2, rhs_seg holds the restricted residual R on F, in a buffer
  // of its own): the pass first forms rhs = R + A u0 on F, A u0 on C \ F and t = u0
  // (Eq. 4) and writes both
  T* rhs_out;
  T* tout;
  int jr;
  int foff[3];       // global index of the dense rhs array's first element (tensor coords)
};

long long round_up_ll(long long v, long long m) { return (v + m - 1) / m * m; }

// bit k of m ? a : b as a predicated select (selp): both operands are computed first
__device__ __forceinline__ double sel_bit(unsigned m, int k, double a, double b) {
  double r;
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n selp.f64 %0, %1, %2, p;\n}"
      : "=d"(r) : "d"(a), "d"(b), "r"((m >> k) & 1u));
  return r;
}
__device__ __forceinline__ float sel_bit(unsigned m, int k, float a, float b) {
  float r;
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %3, 0;\n selp.f32 %0, %1, %2, p;\n}"
      : "=f"(r) : "f"(a), "f"(b), "r"((m >> k) & 1u));
  return r;
}

template <class T, int MAXS, int NTMAX>
__global__ void __launch_bounds__(NTMAX, 1)
    k_cheb2(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ Cheb2Args<T> a) {
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const int py = L.py;
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * a.BH, r1 = min(Ey, r0 + a.BH);  // output rows
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);         // stage-1 rows
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);         // u0 rows
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + kRing * a.u0_stride;
  T* u1s = fs + kRing * a.f_stride;
  uint64_t* bars = reinterpret_cast<uint64_t*>(u1s + 2 * a.s_stride);

  const int px = s % L.ns[0] + L.so[0];
  const int pyy = (s / L.ns[0]) % L.ns[1] + L.so[1];
  const int pzz = s / (L.ns[0] * L.ns[1]) + L.so[2];
  const int ox = px * L.S[0] - (L.J + 1);
  const int oy = pyy * L.S[1] - (L.J + 1);
  const int oz = pzz * L.S[2] - (L.J + 1);
  const T* useg = a.uin + (long long)s * L.ss;
  T* oseg = a.uout + (long long)s * L.ss;
  const T* rseg = a.rhs_global ? nullptr : a.rhs_seg + (long long)s * L.ss;
  const uint32_t u0_bytes = (uint32_t)((q1 - q0) * py * sizeof(T));
  // TMA tensor loads need a 16-byte aligned start in x: load from the aligned-down
  // column and shift the smem index by fsh; the rhs buffer row pitch is then bw
  constexpr int kAl = 16 / (int)sizeof(T);
  const int oxt = ox - a.foff[0];              // x in tensor coordinates
  const int oxa = oxt & ~(kAl - 1);            // 16-byte aligned box start
  const int fpitch = a.rhs_global ? a.bw : py;
  const int fsh = a.rhs_global ? oxt - oxa : 0;
  const uint32_t f_bytes = a.rhs_global ? (uint32_t)((a.BH + 2) * a.bw * sizeof(T))
                                        : (uint32_t)((s1 - s0) * py * sizeof(T));

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kRing; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // producer (thread 0 only): plane z of u rows [q0, q1) and of rhs rows [s0, s0 + BH + 2)
#define ISSUE_U0(z)                                                                          \
  do {                                                                                       \
    const int sl_ = (z) % kRing;                                                             \
    mbar_expect_tx(&bars[sl_], u0_bytes);                                                    \
    bulk_g2s(u0s + sl_ * a.u0_stride, useg + (long long)(z) * pz + (long long)q0 * py,       \
             u0_bytes, &bars[sl_]);                                                          \
  } while (0)
#define ISSUE_F(z)                                                                           \
  do {                                                                                       \
    const int sl_ = (z) % kRing;                                                             \
    mbar_expect_tx(&bars[kRing + sl_], f_bytes);                                             \
    if (a.rhs_global)                                                                        \
      tma_3d(fs + sl_ * a.f_stride, &fmap, oxa, oy + s0 - a.foff[1], oz + (z) - a.foff[2],  \
             &bars[kRing + sl_]);                                                            \
    else                                                                                     \
      bulk_g2s(fs + sl_ * a.f_stride, rseg + (long long)(z) * pz + (long long)s0 * py,       \
               f_bytes, &bars[kRing + sl_]);                                                 \
  } while (0)
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(kRing, Ez); ++z) {
      ISSUE_U0(z);
      ISSUE_F(z);
    }
  }

  // ---- fixed cells of this thread: column tx, MAXS consecutive rows y0 .. y0+MAXS-1.
  // The y-neighbours of all but the edge slots are the register queues of the thread's
  // own neighbouring slots; x-neighbours and edge y-neighbours come from shared memory.
  // Boundary handling is branch-free: storage cells outside Omega are ZERO (invariant of
  // every kernel: none writes outside Omega; buffers are zeroed at create), so a reflected
  // ghost -u_i (R3) adds +1 to the diagonal of A instead:
  //   (A u)_i = ((6 + n_out(i)) u_i - sum of the in-domain neighbours) / h^2.
  const int NG = (s1 - s0 + MAXS - 1) / MAXS;
  const int tx = threadIdx.x % Ex, g = threadIdx.x / Ex;
  const int y0 = s0 + g * MAXS;
  const int gxv = ox + tx;
  const bool tok = g < NG;
  const bool tin = tok && gxv >= 0 && gxv < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const int dxo = (gxv == 0 ? 1 : 0) + (gxv == L.N[0] - 1 ? 1 : 0);
  // slot masks: ld (u0 row loaded), ex (stage-1 row: u1 written), c (C cell), w (output)
  unsigned ld_mask = 0, ex_mask = 0, c_mask = 0, w_mask = 0;
  T diag[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k;
    const int gy = oy + y;
    const bool in = tin && y < s1 && gy >= 0 && gy < L.N[1];
    if (tok && y < q1) ld_mask |= 1u << k;
    if (tok && y < s1) ex_mask |= 1u << k;
    if (in && tcx && y >= 1 && y <= Ey - 2) c_mask |= 1u << k;
    if (in && y >= r0 && y < r1) w_mask |= 1u << k;
    diag[k] = T(6 + dxo + (gy == 0 ? 1 : 0) + (gy == L.N[1] - 1 ? 1 : 0));
  }
  const int off0 = (y0 - s0) * py + tx;
  const T* const u0b = u0s + (s0 - q0) * py + off0;  // slot 0 of ring slot 0
  const T* const fb = fs + (y0 - s0) * fpitch + tx + fsh;
  T* const u1b = u1s + off0;
  T* const ob = oseg + (long long)y0 * py + tx;
  // register queues: plane p of u0 / u1 lives in slot p % 3 (no shifting)
  T u0q[MAXS][3], u1q[MAXS][3];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    u0q[k][0] = ((ld_mask >> k) & 1u) ? u0b[k * py] : T(0);
    u0q[k][1] = T(0);
    u0q[k][2] = T(0);
    u1q[k][0] = u1q[k][1] = u1q[k][2] = T(0);
  }
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0, cm = a.cm, cr = a.cr;

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3
    constexpr int IM = (R + 2) % 3, I0 = R, IP = (R + 1) % 3;
    // ------------------------------------------------------------ stage 1 at plane z
    if (z < Ez) {
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % kRing], ((z + 1) / kRing) & 1);
      mbar_wait(&bars[kRing + z % kRing], (z / kRing) & 1);
      const T* pl = u0b + (z % kRing) * a.u0_stride;
      const T* pn = u0b + ((z + 1) % kRing) * a.u0_stride;
      const T* fp = fb + (z % kRing) * a.f_stride;
      T* u1w = u1b + (z & 1) * a.s_stride;
      const int gz = oz + z;
      const bool zc = gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2;
      const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
      if (z + 1 < Ez) {
#pragma unroll
        for (int k = 0; k < MAXS; ++k)
          if ((ld_mask >> k) & 1u) u0q[k][IP] = pn[k * py];
      } else {
#pragma unroll
        for (int k = 0; k < MAXS; ++k) u0q[k][IP] = T(0);
      }
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        const T v0 = u0q[k][I0];
        T v1 = v0;
        if (zc && ((c_mask >> k) & 1u)) {
          const T ym = (k == 0) ? pl[-py] : u0q[k > 0 ? k - 1 : 0][I0];
          const T yp = (k == MAXS - 1) ? pl[MAXS * py] : u0q[k + 1 < MAXS ? k + 1 : k][I0];
          const T sum = ((u0q[k][IM] + u0q[k][IP]) + (ym + yp)) + (pl[k * py - 1] + pl[k * py + 1]);
          const T r = fp[k * fpitch] - ((diag[k] + dz) * v0 - sum) * ih2;
          v1 = v0 + c0 * r;
        }
        u1q[k][I0] = v1;
        if ((ex_mask >> k) & 1u) u1w[k * py] = v1;
      }
    }
    __syncthreads();  // (A) u1 plane z complete; u0 plane z no longer read
    if (threadIdx.x == 0 && z < Ez && z + kRing < Ez) ISSUE_U0(z + kRing);
    // ------------------------------------------------------------ stage 2 at plane z-1
    if (z >= 1) {
      const int zz = z - 1;
      const int gz = oz + zz;
      if (gz >= 0 && gz < L.N[2]) {
        const bool zc = zz >= 1 && zz <= Ez - 2;
        const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
        const T* u1r = u1b + (zz & 1) * a.s_stride;
        const T* fp = fb + (zz % kRing) * a.f_stride;
        T* orow = ob + (long long)zz * pz;
        // u1 planes z-2, z-1, z are in slots (R+1)%3, (R+2)%3, R; u0 plane z-1 in (R+2)%3
        constexpr int J2 = (R + 1) % 3, J1 = (R + 2) % 3, J0 = R;
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          if (!((w_mask >> k) & 1u)) continue;
          const T u0v = u0q[k][J1];
          T v2 = u0v;
          if (zc && ((c_mask >> k) & 1u)) {
            const T c1 = u1q[k][J1];
            const T ym = (k == 0) ? u1r[-py] : u1q[k > 0 ? k - 1 : 0][J1];
            const T yp = (k == MAXS - 1) ? u1r[MAXS * py] : u1q[k + 1 < MAXS ? k + 1 : k][J1];
            const T sum = ((u1q[k][J2] + u1q[k][J0]) + (ym + yp)) + (u1r[k * py - 1] + u1r[k * py + 1]);
            const T r = fp[k * fpitch] - ((diag[k] + dz) * c1 - sum) * ih2;
            v2 = c1 + cm * (c1 - u0v) + cr * r;
          }
          orow[k * py] = v2;
        }
      }
    }
    __syncthreads();  // (B) u1 buffer and f plane z-1 free
    if (threadIdx.x == 0 && z >= 1 && z - 1 + kRing < Ez) ISSUE_F(z - 1 + kRing);
  };
  for (int zb = 0; zb <= Ez; zb += 3) {
    step(std::integral_constant<int, 0>{}, zb);
    if (zb + 1 <= Ez) step(std::integral_constant<int, 1>{}, zb + 1);
    if (zb + 2 <= Ez) step(std::integral_constant<int, 2>{}, zb + 2);
  }
#undef ISSUE_U0
#undef ISSUE_F
}

// =====================================================================================
// Geometry-specialised variant: compile-time row pitch PY and band height BH, so every
// smem/register offset is an immediate; ONE barrier per plane (u1 triple-buffered, u0 ring
// of 3 planes indexed by z % 3, rhs ring of 4).  RG = 1: rhs is a dense global array
// (tensor TMA, smem pitch PY + 16 B so the 16-byte aligned box start fits); RG = 0: rhs
// is segment storage (1-D bulk copies, pitch PY).  Same arithmetic as k_cheb2.
// =====================================================================================
template <class T, int PY, int BH, int MAXS, int RG, int NST = 2>
struct SpecGeom {
  static constexpr int kAl = 16 / (int)sizeof(T);
  static constexpr int FP = RG ? PY + kAl : PY;
  static constexpr int NG = (BH + 2 + MAXS - 1) / MAXS;
  static constexpr int NT = PY * NG;
  static constexpr int A = 128 / (int)sizeof(T);
  // thread rows (NG * MAXS >= BH + 2): the branch-free plane steps read and write every
  // thread row, so the buffers cover them all (+1 row above and below for u0)
  static constexpr int TR = NG * MAXS;
  static constexpr int U0S = ((TR + 2) * PY + A - 1) / A * A;
  static constexpr int FS = (TR * FP + A - 1) / A * A;
  static constexpr int U1S = ((TR + 2) * PY + A - 1) / A * A;
  // rings: the degree-1 pass has half the arithmetic per plane, so it streams 4 planes
  // ahead (in the smem the u1 planes of the degree-2 pass would take)
  static constexpr int RU = NST == 1 ? 5 : 3, RF = NST == 1 ? 5 : 4, NU1 = NST == 1 ? 0 : 3;
  static constexpr size_t SMEM =
      (size_t)(RU * U0S + RF * FS + NU1 * U1S) * sizeof(T) + 8 * (RU + RF);
  // CTAs per SM the smem allows (capped at 3: registers; more measured no faster -- fp32
  // at 4 CTAs of <72,14,8> caps the lean pass at 96 registers: 0.56 vs 0.45 ms)
  static constexpr int MINB = SMEM <= 75 * 1024 ? 3 : SMEM <= 113 * 1024 ? 2 : 1;
};

template <class T, int PY, int BH, int MAXS, int RG, int NST, int FIN = 0>
__global__ void __launch_bounds__(SpecGeom<T, PY, BH, MAXS, RG, NST>::NT,
                                  SpecGeom<T, PY, BH, MAXS, RG, NST>::MINB)
    k_cheb2s(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ Cheb2Args<T> a) {
  using G = SpecGeom<T, PY, BH, MAXS, RG, NST>;
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + G::RU * G::U0S;
  T* u1s = fs + G::RF * G::FS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(u1s + G::NU1 * G::U1S);  // [0,RU) u0, then f

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
  const int oxt = ox - a.foff[0];              // x in tensor coordinates
  const int oxa = oxt & ~(G::kAl - 1);         // 16-byte aligned box start
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
    bulk_g2s(u0s + sl * G::U0S + (q0 - s0 + 1) * PY, useg + (long long)z * pz + (long long)q0 * PY,
             u0_bytes,
             &bars[sl]);
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
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    for (int z = 0; z < min(NST == 1 ? G::RF : 3, Ez); ++z) issue_f(z);
  }

  const int tx = threadIdx.x % PY, g = threadIdx.x / PY;
  const int y0 = s0 + g * MAXS;
  const int gxv = ox + tx;
  const bool tok = tx < Ex && y0 < s1;
  const bool tin = tok && gxv >= 0 && gxv < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const int dxo = (gxv == 0 ? 1 : 0) + (gxv == L.N[0] - 1 ? 1 : 0);
  // rw_mask: the band's storage rows -- written whole (every column of the pitch, cells
  // outside Omega and the padding with their unchanged value) so no DRAM sector is written
  // partially (no read-for-ownership)
  unsigned ld_mask = 0, ex_mask = 0, c_mask = 0, w_mask = 0, yb_mask = 0, rw_mask = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k;
    const int gy = oy + y;
    if (y >= r0 && y < r1) rw_mask |= 1u << k;
    const bool in = tin && y < s1 && gy >= 0 && gy < L.N[1];
    if (tok && y < q1) ld_mask |= 1u << k;
    if (tok && y < s1) ex_mask |= 1u << k;
    if (in && tcx && y >= 1 && y <= Ey - 2) c_mask |= 1u << k;
    if (in && y >= r0 && y < r1) w_mask |= 1u << k;
    yb_mask |= (unsigned)((gy == 0 ? 1 : 0) + (gy == L.N[1] - 1 ? 1 : 0)) << (2 * k);
  }
  // FIN: the genuine (x, y) cells of the band's output rows and their column in the user's u
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
  // FIN = 2: the slots in F = grow(V, jr) (x, y) and the rows of the rhs / t outputs
  unsigned f_mask = 0;
  int fz0 = 0, fz1 = 0;
  T* rob = nullptr;
  T* tob = nullptr;
  if constexpr (FIN == 2) {
    const bool fx = gxv >= px * L.S[0] - a.jr && gxv < (px + 1) * L.S[0] + a.jr;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      const int gy = oy + y0 + k;
      if (fx && gy >= pyy * L.S[1] - a.jr && gy < (pyy + 1) * L.S[1] + a.jr) f_mask |= 1u << k;
    }
    fz0 = pzz * L.S[2] - a.jr;
    fz1 = (pzz + 1) * L.S[2] + a.jr;
    rob = a.rhs_out + (long long)s * L.ss + (long long)y0 * PY + tx;
    tob = a.tout + (long long)s * L.ss + (long long)y0 * PY + tx;
  }
  // diagonal of A per slot (6 + reflected x/y neighbours, R3); the z part is per plane
  T dk[MAXS];
#pragma unroll
  for (int k = 0; k < MAXS; ++k) dk[k] = T(6 + dxo) + T((yb_mask >> (2 * k)) & 3u);
  // smem row = storage row - s0 + 1 (one margin row above every thread row, for u0 and u1)
  const T* const u0b = u0s + (y0 - s0 + 1) * PY + tx;
  const T* const fb = fs + (y0 - s0) * G::FP + tx + fsh;
  T* const u1b = u1s + (y0 - s0 + 1) * PY + tx;
  T* const ob = oseg + (long long)y0 * PY + tx;
  T u0q[MAXS][3], u1q[MAXS][3];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    u0q[k][0] = ((ld_mask >> k) & 1u) ? u0b[k * PY] : T(0);
    u0q[k][1] = u0q[k][2] = T(0);
    u1q[k][0] = u1q[k][1] = u1q[k][2] = T(0);
  }
  const T ih2 = T(L.inv_h2);
  const T c0 = a.c0, cm = a.cm, cr = a.cr;
  const T six = T(6 + dxo);

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3: u0 ring slot, u1 buffer, queue slot
    constexpr int IM = (R + 2) % 3, I0 = R, IP = (R + 1) % 3;
    if (z < Ez) {
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % G::RU], ((z + 1) / G::RU) & 1);
      mbar_wait(&bars[G::RU + z % G::RF], (z / G::RF) & 1);
      const T* pl = u0b + (z % G::RU) * G::U0S;
      const T* pn = u0b + ((z + 1) % G::RU) * G::U0S;
      const T* fp = fb + (z % G::RF) * G::FS;
      T* u1w = u1b + R * G::U1S;
      const int gz = oz + z;
      const bool zc = gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2;
      const T dz = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0));
      // rows outside the loaded range hold stale smem: they only feed dead slots
#pragma unroll
      for (int k = 0; k < MAXS; ++k) u0q[k][IP] = (z + 1 < Ez) ? pn[k * PY] : T(0);
      const unsigned act = zc ? c_mask : 0u;
      // FIN = 2: this plane's rhs / t rows (in-domain planes only), and F in z
      const bool zin = gz >= 0 && gz < L.N[2];
      const unsigned fm = (FIN == 2 && gz >= fz0 && gz < fz1) ? f_mask : 0u;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        // branch-free: every slot computes, the C-cell predicate selects
        const T v0 = u0q[k][I0];
        const T ym = (k == 0) ? pl[-PY] : u0q[k > 0 ? k - 1 : 0][I0];
        const T yp = (k == MAXS - 1) ? pl[MAXS * PY] : u0q[k + 1 < MAXS ? k + 1 : k][I0];
        const T sum = ((u0q[k][IM] + u0q[k][IP]) + (ym + yp)) + (pl[k * PY - 1] + pl[k * PY + 1]);
        T r;
        if constexpr (FIN == 2) {
          // tau (Eq. 4, fig:mgvsr L234-236): rhs = R + A u0 on F, A u0 on C \ F; then the
          // first step's residual rhs - A u0 as the unfused pair computes it
          const T Au = ((dk[k] + dz) * v0 - sum) * ih2;
          const T Rv = fp[k * G::FP];
          const T bv = ((fm >> k) & 1u) ? Rv + Au : Au;
          r = bv - Au;
          const bool cc = (act >> k) & 1u;
          const_cast<T*>(fp)[k * G::FP] = cc ? bv : Rv;  // stage 2 reads the new rhs
          if (zin && ((rw_mask >> k) & 1u)) {
            rob[(long long)z * pz + k * PY] = cc ? bv : Rv;  // whole rows: others unchanged
            tob[(long long)z * pz + k * PY] = v0;           // t = u0 (0 outside Omega)
          }
        } else {
          r = fp[k * G::FP] - ((dk[k] + dz) * v0 - sum) * ih2;
        }
        const T v1 = ((act >> k) & 1u) ? v0 + c0 * r : v0;
        if constexpr (NST == 2) {
          u1q[k][I0] = v1;
          u1w[k * PY] = v1;
        } else {
          // degree 1: the first step is the result (C updated, GSR copied)
          if (((rw_mask >> k) & 1u) && gz >= 0 && gz < L.N[2])
            ob[(long long)z * pz + k * PY] = ((w_mask >> k) & 1u) ? v1 : v0;
        }
      }
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if (z + G::RU < Ez) issue_u0(z + G::RU);  // u0 slot of plane z is free
      if (NST == 1) {
        if (z + G::RF < Ez) issue_f(z + G::RF);  // rhs plane z is consumed
      } else if (z >= 1 && z + 2 < Ez) {
        issue_f(z + 2);  // rhs slot of plane z-2 (stage 2 finished it) is free
      }
    }
    if (NST == 2 && z >= 1) {
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
        // last pass: genuine cells of a genuine plane go to the user's u (R19)
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
          // wide bands: a select, not a branch (the compiler would sink the stencil loads into
          // one); the E = 22 / 14 boxes measure faster with the branch
          T v2;
          if constexpr (PY >= 40) v2 = sel_bit(act, k, c1 + cm * (c1 - u0v) + cr * r, u0v);
          else v2 = ((act >> k) & 1u) ? c1 + cm * (c1 - u0v) + cr * r : u0v;
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
}

// =====================================================================================
// Lean degree-2 pass (same geometry, rings and arithmetic plan as k_cheb2s; FIN = 0 / 1):
// the per-cell region masks are folded into per-slot coefficients, so a plane step is
// branch- and select-free.  A slot that is not a C cell (GSR ring, out-of-domain row or
// column, padding) gets c0 = cr = 0: u1 = fma(0, r, u0) = u0 and u2 = c1 + cm (c1 - u0) + 0
// = u0 exactly, provided r is finite -- so every shared-memory word a dead slot reads is
// zeroed once at the start (margin rows, rows beyond the loaded range).  Planes outside
// C in z are uniform per CTA (a uniform branch copies them).  The diagonal (6 + reflected
// neighbours, R3) is kept per slot, pre-multiplied by 1/h^2:
//   r = f - (d u - sum) / h^2 = fma(1/h^2, sum, fma(-d/h^2, u, f)).
// =====================================================================================
template <class T, int PY, int BH, int MAXS, int RG, int FIN = 0>
__global__ void __launch_bounds__(SpecGeom<T, PY, BH, MAXS, RG, 2>::NT,
                                  SpecGeom<T, PY, BH, MAXS, RG, 2>::MINB)
    k_cheb2l(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ Cheb2Args<T> a) {
  using G = SpecGeom<T, PY, BH, MAXS, RG, 2>;
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);
  T* u0s = reinterpret_cast<T*>(sm);
  T* fs = u0s + G::RU * G::U0S;
  T* u1s = fs + G::RF * G::FS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(u1s + G::NU1 * G::U1S);

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
  // zero every buffer once: dead slots read margin rows and rows no copy fills
  {
    const int nw = (int)((G::RU * G::U0S + G::RF * G::FS + G::NU1 * G::U1S) * sizeof(T) / 16);
    uint4* z4 = reinterpret_cast<uint4*>(sm);
    for (int i = threadIdx.x; i < nw; i += G::NT) z4[i] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < G::RU + G::RF; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // generic-proxy zero stores before the async-proxy (TMA) writes into the same buffers
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    for (int z = 0; z < min(3, Ez); ++z) issue_f(z);
  }

  const int tx = threadIdx.x % PY, g = threadIdx.x / PY;
  const int y0 = s0 + g * MAXS;
  const int gxv = ox + tx;
  const bool tin = tx < Ex && gxv >= 0 && gxv < L.N[0];
  const bool tcx = tx >= 1 && tx <= Ex - 2;
  const T ih2 = T(L.inv_h2);
  // per slot: the two step coefficients (0 on dead slots), the scaled diagonal, and the
  // rows of the band's output (written whole, padding and dead cells unchanged)
  T c0k[MAXS], crk[MAXS], dkh[MAXS];
  bool wr[MAXS];
  unsigned gen_mask = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k;
    const int gy = oy + y;
    const bool c = tin && tcx && y < s1 && y >= 1 && y <= Ey - 2 && gy >= 0 && gy < L.N[1];
    c0k[k] = c ? a.c0 : T(0);
    crk[k] = c ? a.cr : T(0);
    const int nb = 6 + (gxv == 0) + (gxv == L.N[0] - 1) + (gy == 0) + (gy == L.N[1] - 1);
    dkh[k] = T(nb) * ih2;
    wr[k] = y >= r0 && y < r1 && y0 < s1;
    if constexpr (FIN == 1) {
      const int vlo = L.J + 1;
      if (wr[k] && tin && gy >= 0 && gy < L.N[1] && tx >= vlo && tx < vlo + L.S[0] && y >= vlo &&
          y < vlo + L.S[1])
        gen_mask |= 1u << k;
    }
  }
  T* fbase = nullptr;
  if constexpr (FIN == 1)
    fbase = a.fin.p + (long long)(oy + y0 - a.fin.bo[1]) * a.fin.sy + (gxv - a.fin.bo[0]);
  const T* const u0b = u0s + (y0 - s0 + 1) * PY + tx;
  const T* const fb = fs + (y0 - s0) * G::FP + tx + fsh;
  T* const u1b = u1s + (y0 - s0 + 1) * PY + tx;
  T* const ob = oseg + (long long)y0 * PY + tx;
  T u0q[MAXS][3], u1q[MAXS][3];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    u0q[k][0] = u0b[k * PY];
    u0q[k][1] = u0q[k][2] = T(0);
    u1q[k][0] = u1q[k][1] = u1q[k][2] = T(0);
  }
  const T cm = a.cm;

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3: u0 ring slot, u1 buffer, queue slot
    constexpr int IM = (R + 2) % 3, I0 = R, IP = (R + 1) % 3;
    if (z < Ez) {
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % G::RU], ((z + 1) / G::RU) & 1);
      mbar_wait(&bars[G::RU + z % G::RF], (z / G::RF) & 1);
      const T* pl = u0b + (z % G::RU) * G::U0S;
      const T* pn = u0b + ((z + 1) % G::RU) * G::U0S;
      const T* fp = fb + (z % G::RF) * G::FS;
      T* u1w = u1b + R * G::U1S;
      const int gz = oz + z;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) u0q[k][IP] = (z + 1 < Ez) ? pn[k * PY] : T(0);
      if (gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2) {  // uniform: C planes
        const T dzh = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0)) * ih2;
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const T v0 = u0q[k][I0];
          const T ym = (k == 0) ? pl[-PY] : u0q[k > 0 ? k - 1 : 0][I0];
          const T yp = (k == MAXS - 1) ? pl[MAXS * PY] : u0q[k + 1 < MAXS ? k + 1 : k][I0];
          const T sum = ((u0q[k][IM] + u0q[k][IP]) + (ym + yp)) + (pl[k * PY - 1] + pl[k * PY + 1]);
          const T r = fma(ih2, sum, fma(-(dkh[k] + dzh), v0, fp[k * G::FP]));
          const T v1 = fma(c0k[k], r, v0);
          u1q[k][I0] = v1;
          u1w[k * PY] = v1;
        }
      } else {
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          u1q[k][I0] = u0q[k][I0];
          u1w[k * PY] = u0q[k][I0];
        }
      }
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if (z + G::RU < Ez) issue_u0(z + G::RU);  // u0 slot of plane z is free
      if (z >= 1 && z + 2 < Ez) issue_f(z + 2);  // rhs slot of plane z-2 is free
    }
    if (z >= 1) {
      const int zz = z - 1;
      const int gz = oz + zz;
      if (gz >= 0 && gz < L.N[2]) {
        constexpr int J2 = (R + 1) % 3, J1 = (R + 2) % 3, J0 = R;
        T v2[MAXS];
        if (zz >= 1 && zz <= Ez - 2) {  // uniform: C planes
          const T dzh = T((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0)) * ih2;
          const T* u1r = u1b + J1 * G::U1S;
          const T* fp = fb + (zz % G::RF) * G::FS;
#pragma unroll
          for (int k = 0; k < MAXS; ++k) {
            const T u0v = u0q[k][J1];
            const T c1 = u1q[k][J1];
            const T ym = (k == 0) ? u1r[-PY] : u1q[k > 0 ? k - 1 : 0][J1];
            const T yp = (k == MAXS - 1) ? u1r[MAXS * PY] : u1q[k + 1 < MAXS ? k + 1 : k][J1];
            const T sum = ((u1q[k][J2] + u1q[k][J0]) + (ym + yp)) + (u1r[k * PY - 1] + u1r[k * PY + 1]);
            const T r = fma(ih2, sum, fma(-(dkh[k] + dzh), c1, fp[k * G::FP]));
            v2[k] = fma(crk[k], r, fma(cm, c1 - u0v, c1));
          }
        } else {
#pragma unroll
          for (int k = 0; k < MAXS; ++k) v2[k] = u0q[k][J1];
        }
        if constexpr (FIN != 1) {
          T* orow = ob + (long long)zz * pz;
#pragma unroll
          for (int k = 0; k < MAXS; ++k)
            if (wr[k]) orow[k * PY] = v2[k];
        } else {
          // last pass: genuine cells of a genuine plane go to the user's u (R19)
          if (zz >= L.J + 1 && zz < L.J + 1 + L.S[2]) {
            T* frow = fbase + (long long)(gz - a.fin.bo[2]) * a.fin.sz;
#pragma unroll
            for (int k = 0; k < MAXS; ++k)
              if ((gen_mask >> k) & 1u) frow[k * a.fin.sy] = v2[k];
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
}

// =====================================================================================
// Packed fp32 degree-2 pass: k_cheb2l's plan, coefficients and rounding, with TWO
// x-adjacent cells per thread (x0 = 2 t, x0 + 1) and the arithmetic of both in sm_100's
// paired fp32 instructions (FADD2 / FFMA2 on float2).  The centre, next-plane, y-neighbour
// and u1 accesses are 8-byte shared-memory words; the x-neighbours outside the pair, and
// the rhs of a dense f (its TMA box starts at an odd column on the SR levels), are single
// loads.  Per lane the operations and their order are exactly k_cheb2l's:
//   sum = ((z- + z+) + (y- + y+)) + (x- + x+),  r = fma(ih2, sum, fma(-(d + dz), u, f)),
//   u1 = fma(c0, r, u0),  u2 = fma(cr, r, fma(cm, u1 - u0, u1))
// so the result is bitwise k_cheb2l's (c1 - u0 as fma(-1, u0, c1): exact, one rounding).
// =====================================================================================
__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 ld2(const float* p) { return *reinterpret_cast<const float2*>(p); }
__device__ __forceinline__ void st2(float* p, float2 v) { *reinterpret_cast<float2*>(p) = v; }

template <int PY, int BH, int MAXS, int RG>
struct PackGeom {
  using G = SpecGeom<float, PY, BH, MAXS, RG, 2>;
  static constexpr int PX = PY / 2;        // threads per row group
  static constexpr int NT = PX * G::NG;
  static_assert(PY % 2 == 0, "pair layout needs an even row pitch");
};

template <int PY, int BH, int MAXS, int RG, int FIN = 0>
__global__ void __launch_bounds__(PackGeom<PY, BH, MAXS, RG>::NT,
                                  SpecGeom<float, PY, BH, MAXS, RG, 2>::MINB)
    k_cheb2p(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ Cheb2Args<float> a) {
  using G = SpecGeom<float, PY, BH, MAXS, RG, 2>;
  using P = PackGeom<PY, BH, MAXS, RG>;
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& L = a.L;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const long long pz = L.pz;
  const int s = blockIdx.y;
  const int r0 = blockIdx.x * BH, r1 = min(Ey, r0 + BH);
  const int s0 = max(0, r0 - 1), s1 = min(Ey, r1 + 1);
  const int q0 = max(0, r0 - 2), q1 = min(Ey, r1 + 2);
  float* u0s = reinterpret_cast<float*>(sm);
  float* fs = u0s + G::RU * G::U0S;
  float* u1s = fs + G::RF * G::FS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(u1s + G::NU1 * G::U1S);

  const int px = s % L.ns[0] + L.so[0];
  const int pyy = (s / L.ns[0]) % L.ns[1] + L.so[1];
  const int pzz = s / (L.ns[0] * L.ns[1]) + L.so[2];
  const int ox = px * L.S[0] - (L.J + 1);
  const int oy = pyy * L.S[1] - (L.J + 1);
  const int oz = pzz * L.S[2] - (L.J + 1);
  const float* useg = a.uin + (long long)s * L.ss;
  float* oseg = a.uout + (long long)s * L.ss;
  const float* rseg = RG ? nullptr : a.rhs_seg + (long long)s * L.ss;
  const uint32_t u0_bytes = (uint32_t)((q1 - q0) * PY * sizeof(float));
  const int oxt = ox - a.foff[0];
  const int oxa = oxt & ~(G::kAl - 1);
  const int fsh = RG ? oxt - oxa : 0;
  const uint32_t f_bytes = RG ? (uint32_t)((BH + 2) * G::FP * sizeof(float))
                              : (uint32_t)((s1 - s0) * PY * sizeof(float));
  {  // zero every buffer once: dead slots read margin rows and rows no copy fills
    const int nw = (int)((G::RU * G::U0S + G::RF * G::FS + G::NU1 * G::U1S) * sizeof(float) / 16);
    uint4* z4 = reinterpret_cast<uint4*>(sm);
    for (int i = threadIdx.x; i < nw; i += P::NT) z4[i] = make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < G::RU + G::RF; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  if (threadIdx.x == 0) {
    for (int z = 0; z < min(G::RU, Ez); ++z) issue_u0(z);
    for (int z = 0; z < min(3, Ez); ++z) issue_f(z);
  }

  const int x0 = 2 * (threadIdx.x % P::PX), g = threadIdx.x / P::PX;
  const int y0 = s0 + g * MAXS;
  const float ih2 = float(L.inv_h2);
  // per slot and lane: the step coefficients (0 on dead cells), minus the scaled diagonal
  float2 c0k[MAXS], crk[MAXS], ndk[MAXS];
  bool wr[MAXS];
  unsigned gen_mask = 0;  // FIN: bit 2k + j = genuine cell (slot k, lane j)
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = y0 + k;
    const int gy = oy + y;
    float cc[2], rr[2], dd[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int x = x0 + j, gx = ox + x;
      const bool tin = x < Ex && gx >= 0 && gx < L.N[0];
      const bool c = tin && x >= 1 && x <= Ex - 2 && y < s1 && y >= 1 && y <= Ey - 2 && gy >= 0 &&
                     gy < L.N[1];
      cc[j] = c ? a.c0 : 0.f;
      rr[j] = c ? a.cr : 0.f;
      const int nb = 6 + (gx == 0) + (gx == L.N[0] - 1) + (gy == 0) + (gy == L.N[1] - 1);
      dd[j] = -(float(nb) * ih2);
      if constexpr (FIN == 1) {
        const int vlo = L.J + 1;
        if (y >= r0 && y < r1 && y0 < s1 && tin && gy >= 0 && gy < L.N[1] && x >= vlo &&
            x < vlo + L.S[0] && y >= vlo && y < vlo + L.S[1])
          gen_mask |= 1u << (2 * k + j);
      }
    }
    c0k[k] = make_float2(cc[0], cc[1]);
    crk[k] = make_float2(rr[0], rr[1]);
    ndk[k] = make_float2(dd[0], dd[1]);
    wr[k] = y >= r0 && y < r1 && y0 < s1;
  }
  float* fbase = nullptr;
  if constexpr (FIN == 1)
    fbase = a.fin.p + (long long)(oy + y0 - a.fin.bo[1]) * a.fin.sy + (ox + x0 - a.fin.bo[0]);
  const float* const u0b = u0s + (y0 - s0 + 1) * PY + x0;
  const float* const fb = fs + (y0 - s0) * G::FP + x0 + fsh;
  float* const u1b = u1s + (y0 - s0 + 1) * PY + x0;
  float* const ob = oseg + (long long)y0 * PY + x0;
  auto ldf = [&](const float* p) {  // rhs pair: 8-byte aligned only for segment storage
    if constexpr (RG) return make_float2(p[0], p[1]);
    else return ld2(p);
  };
  float2 u0q[MAXS][3], u1q[MAXS][3];
  mbar_wait(&bars[0], 0);
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    u0q[k][0] = ld2(u0b + k * PY);
    u0q[k][1] = u0q[k][2] = make_float2(0.f, 0.f);
    u1q[k][0] = u1q[k][1] = u1q[k][2] = make_float2(0.f, 0.f);
  }
  const float2 cm2 = make_float2(a.cm, a.cm), ih2v = make_float2(ih2, ih2);
  const float2 mone = make_float2(-1.f, -1.f);

  auto step = [&](auto RR, int z) {
    constexpr int R = decltype(RR)::value;  // z % 3: u0 ring slot, u1 buffer, queue slot
    constexpr int IM = (R + 2) % 3, I0 = R, IP = (R + 1) % 3;
    if (z < Ez) {
      if (z + 1 < Ez) mbar_wait(&bars[(z + 1) % G::RU], ((z + 1) / G::RU) & 1);
      mbar_wait(&bars[G::RU + z % G::RF], (z / G::RF) & 1);
      const float* pl = u0b + (z % G::RU) * G::U0S;
      const float* pn = u0b + ((z + 1) % G::RU) * G::U0S;
      const float* fp = fb + (z % G::RF) * G::FS;
      float* u1w = u1b + R * G::U1S;
      const int gz = oz + z;
#pragma unroll
      for (int k = 0; k < MAXS; ++k)
        u0q[k][IP] = (z + 1 < Ez) ? ld2(pn + k * PY) : make_float2(0.f, 0.f);
      if (gz >= 0 && gz < L.N[2] && z >= 1 && z <= Ez - 2) {  // uniform: C planes
        const float ndz = -(float((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0)) * ih2);
        const float2 ndz2 = make_float2(ndz, ndz);
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          const float2 v0 = u0q[k][I0];
          const float2 ym = (k == 0) ? ld2(pl - PY) : u0q[k > 0 ? k - 1 : 0][I0];
          const float2 yp = (k == MAXS - 1) ? ld2(pl + MAXS * PY) : u0q[k + 1 < MAXS ? k + 1 : k][I0];
          const float2 xs = f2add(make_float2(pl[k * PY - 1], v0.x), make_float2(v0.y, pl[k * PY + 2]));
          const float2 sum = f2add(f2add(f2add(u0q[k][IM], u0q[k][IP]), f2add(ym, yp)), xs);
          const float2 r = f2fma(ih2v, sum, f2fma(f2add(ndk[k], ndz2), v0, ldf(fp + k * G::FP)));
          const float2 v1 = f2fma(c0k[k], r, v0);
          u1q[k][I0] = v1;
          st2(u1w + k * PY, v1);
        }
      } else {
#pragma unroll
        for (int k = 0; k < MAXS; ++k) {
          u1q[k][I0] = u0q[k][I0];
          st2(u1w + k * PY, u0q[k][I0]);
        }
      }
    }
    __syncthreads();  // the only barrier of the plane step
    if (threadIdx.x == 0) {
      if (z + G::RU < Ez) issue_u0(z + G::RU);  // u0 slot of plane z is free
      if (z >= 1 && z + 2 < Ez) issue_f(z + 2);  // rhs slot of plane z-2 is free
    }
    if (z >= 1) {
      const int zz = z - 1;
      const int gz = oz + zz;
      if (gz >= 0 && gz < L.N[2]) {
        constexpr int J2 = (R + 1) % 3, J1 = (R + 2) % 3, J0 = R;
        float2 v2[MAXS];
        if (zz >= 1 && zz <= Ez - 2) {  // uniform: C planes
          const float ndz = -(float((gz == 0 ? 1 : 0) + (gz == L.N[2] - 1 ? 1 : 0)) * ih2);
          const float2 ndz2 = make_float2(ndz, ndz);
          const float* u1r = u1b + J1 * G::U1S;
          const float* fp = fb + (zz % G::RF) * G::FS;
#pragma unroll
          for (int k = 0; k < MAXS; ++k) {
            const float2 u0v = u0q[k][J1];
            const float2 c1 = u1q[k][J1];
            const float2 ym = (k == 0) ? ld2(u1r - PY) : u1q[k > 0 ? k - 1 : 0][J1];
            const float2 yp = (k == MAXS - 1) ? ld2(u1r + MAXS * PY) : u1q[k + 1 < MAXS ? k + 1 : k][J1];
            const float2 xs =
                f2add(make_float2(u1r[k * PY - 1], c1.x), make_float2(c1.y, u1r[k * PY + 2]));
            const float2 sum = f2add(f2add(f2add(u1q[k][J2], u1q[k][J0]), f2add(ym, yp)), xs);
            const float2 r = f2fma(ih2v, sum, f2fma(f2add(ndk[k], ndz2), c1, ldf(fp + k * G::FP)));
            v2[k] = f2fma(crk[k], r, f2fma(cm2, f2fma(mone, u0v, c1), c1));
          }
        } else {
#pragma unroll
          for (int k = 0; k < MAXS; ++k) v2[k] = u0q[k][J1];
        }
        if constexpr (FIN != 1) {
          float* orow = ob + (long long)zz * pz;
#pragma unroll
          for (int k = 0; k < MAXS; ++k)
            if (wr[k]) st2(orow + k * PY, v2[k]);
        } else {
          // last pass: genuine cells of a genuine plane go to the user's u (R19); the user
          // row's column parity is arbitrary, so the two lanes store separately
          if (zz >= L.J + 1 && zz < L.J + 1 + L.S[2]) {
            float* frow = fbase + (long long)(gz - a.fin.bo[2]) * a.fin.sz;
#pragma unroll
            for (int k = 0; k < MAXS; ++k) {
              if ((gen_mask >> (2 * k)) & 1u) frow[k * a.fin.sy] = v2[k].x;
              if ((gen_mask >> (2 * k + 1)) & 1u) frow[k * a.fin.sy + 1] = v2[k].y;
            }
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
}

// ---- host side ---------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// generic kernel (levels without a geometry-specialised instantiation): cells per thread
// and the thread cap
struct Variant {
  int maxs, nt;
};
template <class T>
Variant variant() {
  return sizeof(T) == 8 ? Variant{6, 512} : Variant{8, 512};
}

struct Plan {
  int BH, nbands, NT, maxs;
  size_t smem;
  int u0_stride, s_stride, f_stride, bw;
};

template <class T>
Plan make_plan(const Lvl& L, int MAXS, int NTMAX) {
  Plan pl{};
  pl.maxs = MAXS;
  const int Ey = L.E[1], Ex = L.E[0];
  constexpr int kAl = 16 / (int)sizeof(T);
  const int bw = (int)round_up_ll(Ex + kAl - 1, kAl);  // covers [align_down(ox), ox + Ex)
  for (int nb = 1; nb <= Ey; ++nb) {
    const int BH = (Ey + nb - 1) / nb;
    const long long u0s = round_up_ll((long long)(BH + 4) * L.py * sizeof(T), 128) / sizeof(T);
    const long long ss = round_up_ll((long long)(BH + 2) * L.py * sizeof(T), 128) / sizeof(T);
    const long long fsz =
        round_up_ll((long long)(BH + 2) * std::max(bw, L.py) * sizeof(T), 128) / sizeof(T);
    const size_t smem = (size_t)(kRing * u0s + kRing * fsz + 2 * ss) * sizeof(T) + 2 * kRing * 8;
    const int rows = std::min(Ey, BH + 2);  // stage-1 rows of a band (upper bound)
    const int NT = (int)round_up_ll((long long)Ex * ((rows + MAXS - 1) / MAXS), 32);
    if (smem <= 227 * 1024 && NT <= NTMAX && BH + 2 <= 256 && bw <= 256) {
      pl.BH = BH;
      pl.nbands = (Ey + BH - 1) / BH;
      pl.NT = NT;
      pl.smem = smem;
      pl.u0_stride = (int)u0s;
      pl.s_stride = (int)ss;
      pl.f_stride = (int)fsz;
      pl.bw = bw;
      return pl;
    }
  }
  pl.BH = 0;
  return pl;
}

}  // namespace

template <class T>
bool cheb2_fused_ok(const Lvl& L) {
  if (L.py > 256 || L.E[0] > 256) return false;
  if (((long long)L.N[0] * sizeof(T)) % 16) return false;
  if (!get_encode()) return false;
  const Variant v = variant<T>();
  return make_plan<T>(L, v.maxs, v.nt).BH > 0;
}

namespace {

template <class T>
bool encode_rhs_map(CUtensorMap* map, const FusedRhs<T>& rb, int bw, int rows) {
  const T* p = rb.base;
  const cuuint64_t dims[3] = {(cuuint64_t)rb.dims[0], (cuuint64_t)rb.dims[1],
                              (cuuint64_t)rb.dims[2]};
  const cuuint64_t strides[2] = {(cuuint64_t)rb.dims[0] * sizeof(T),
                                 (cuuint64_t)rb.dims[0] * rb.dims[1] * sizeof(T)};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = get_encode()(
      map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
      const_cast<T*>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fprintf(stderr, "sr_fmg: cuTensorMapEncodeTiled failed (%d)\n", (int)r);
  return r == CUDA_SUCCESS;
}

// lean plane steps (k_cheb2l) for the plain and last degree-2 passes.  Measured at C3's
// finest level (ncu, one pass): fp32 0.45 vs 0.50 ms (lean faster); fp64 0.752 vs 0.720 ms
// (the masked k_cheb2s faster: 414 vs 437 M instructions, but 96 registers and more
// short-scoreboard stalls).  SR_FMG_CHEB_LEAN=0/1 forces one for both (A/B).
template <class T>
bool lean() {
  static const int v = [] {
    const char* e = std::getenv("SR_FMG_CHEB_LEAN");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return v < 0 ? sizeof(T) == 4 : v == 1;
}

// geometry-specialised launch if (T, row pitch) has an instantiation
template <class T, int PY, int BH, int MAXS>
bool try_spec(const Lvl& L, const Cheb2Args<T>& a, FusedRhs<T> b, int nst, cudaStream_t st) {
  if (L.py != PY || L.E[0] > PY) return false;
  if (SpecGeom<T, PY, BH, MAXS, 1>::SMEM > 227 * 1024) return false;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  dim3 grid((L.E[1] + BH - 1) / BH, L.nsegs);
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, nt, smem, st>>>(map, a);
  };
  const bool fin = a.fin.p != nullptr;
  if (b.global && a.tout) return false;
  if (b.global) {
    using G2 = SpecGeom<T, PY, BH, MAXS, 1, 2>;
    using G1 = SpecGeom<T, PY, BH, MAXS, 1, 1>;
    if (!encode_rhs_map<T>(&map, b, G2::FP, BH + 2)) return false;
    if (nst == 2 && fin && lean<T>()) go(k_cheb2l<T, PY, BH, MAXS, 1, 1>, G2::SMEM, G2::NT);
    else if (nst == 2 && lean<T>()) go(k_cheb2l<T, PY, BH, MAXS, 1, 0>, G2::SMEM, G2::NT);
    else if (nst == 2 && fin) go(k_cheb2s<T, PY, BH, MAXS, 1, 2, 1>, G2::SMEM, G2::NT);
    else if (nst == 2) go(k_cheb2s<T, PY, BH, MAXS, 1, 2>, G2::SMEM, G2::NT);
    else go(k_cheb2s<T, PY, BH, MAXS, 1, 1>, G1::SMEM, G1::NT);
  } else {
    using G2 = SpecGeom<T, PY, BH, MAXS, 0, 2>;
    using G1 = SpecGeom<T, PY, BH, MAXS, 0, 1>;
    if (a.tout) {  // tau fused in front (FIN = 2)
      if (nst != 2 || fin) return false;
      go(k_cheb2s<T, PY, BH, MAXS, 0, 2, 2>, G2::SMEM, G2::NT);
    } else if (nst == 2 && fin && lean<T>()) go(k_cheb2l<T, PY, BH, MAXS, 0, 1>, G2::SMEM, G2::NT);
    else if (nst == 2 && lean<T>()) go(k_cheb2l<T, PY, BH, MAXS, 0, 0>, G2::SMEM, G2::NT);
    else if (nst == 2 && fin) go(k_cheb2s<T, PY, BH, MAXS, 0, 2, 1>, G2::SMEM, G2::NT);
    else if (nst == 2) go(k_cheb2s<T, PY, BH, MAXS, 0, 2>, G2::SMEM, G2::NT);
    else go(k_cheb2s<T, PY, BH, MAXS, 0, 1>, G1::SMEM, G1::NT);
  }
  return true;
}

// packed fp32 pass (k_cheb2p) for the plain and last degree-2 passes; SR_FMG_CHEB_PACK=0
// restores the scalar lean pass (A/B; the results are bitwise the same)
bool packed() {  // read per launch (a captured solve keeps the choice it was captured with)
  const char* e = std::getenv("SR_FMG_CHEB_PACK");
  return !(e && e[0] == '0');
}
template <int PY, int BH, int MAXS>
bool try_pack(const Lvl& L, const Cheb2Args<float>& a, FusedRhs<float> b, int nst, cudaStream_t st) {
  if (!packed() || nst != 2 || a.tout || L.py != PY || L.E[0] > PY) return false;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  dim3 grid((L.E[1] + BH - 1) / BH, L.nsegs);
  auto go = [&](auto kern, size_t smem, int nt) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, nt, smem, st>>>(map, a);
  };
  const bool fin = a.fin.p != nullptr;
  if (b.global) {
    using G = SpecGeom<float, PY, BH, MAXS, 1, 2>;
    using P = PackGeom<PY, BH, MAXS, 1>;
    if (!encode_rhs_map<float>(&map, b, G::FP, BH + 2)) return false;
    if (fin) go(k_cheb2p<PY, BH, MAXS, 1, 1>, G::SMEM, P::NT);
    else go(k_cheb2p<PY, BH, MAXS, 1, 0>, G::SMEM, P::NT);
  } else {
    using G = SpecGeom<float, PY, BH, MAXS, 0, 2>;
    using P = PackGeom<PY, BH, MAXS, 0>;
    if (fin) go(k_cheb2p<PY, BH, MAXS, 0, 1>, G::SMEM, P::NT);
    else go(k_cheb2p<PY, BH, MAXS, 0, 0>, G::SMEM, P::NT);
  }
  return true;
}

template <class T>
bool launch_spec(const Lvl& L, const Cheb2Args<T>& a, FusedRhs<T> b, int nst, cudaStream_t st) {
  // Band shapes per row pitch, measured (C3, DESIGN.md §9 keeps the losing ones):
  //  E = 70 (64^3 segments): 14-row bands; fp64 4 cells per thread (0.77 vs 0.85 ms for 2
  //    bands of 35), fp32 8 cells per thread (finest pair 0.991 vs 1.032 ms for 10 of 4);
  //  E = 38 (32^3): fp64 19-row bands of 3 cells (0.60 ms; 22 of 6: 0.71, 16 of 6: 0.73,
  //    22 of 8: 0.76; level 7 per solve, session 2: 19 of 3 0.616-0.631, 19 of 4 0.70-0.71,
  //    13 of 3 0.67-0.68, 10 of 4 0.60-0.64 ms), fp32 22 of 8 (0.38; 14 of 8: 0.45, 38 of 8: 0.57);
  //  E = 134 (128^3, C5): 14-row bands of 544 threads, one CTA per SM (6-row bands slower);
  //  E = 22 / 14: one band per segment (two bands of 11 / 7 rows: level 6 0.213 -> 0.299 ms,
  //    level 5 0.139 -> 0.158 ms per solve; fp32 likewise slower).
  if constexpr (sizeof(T) == 8)
    return try_spec<T, 72, 14, 4>(L, a, b, nst, st) || try_spec<T, 40, 19, 3>(L, a, b, nst, st) ||
           try_spec<T, 136, 14, 4>(L, a, b, nst, st) || try_spec<T, 24, 22, 3>(L, a, b, nst, st) ||
           try_spec<T, 16, 14, 2>(L, a, b, nst, st);
  else
    // packed fp32 pass at E = 70 (C3 finest pair 0.903 -> 0.862 ms); at E = 38 the 20-thread
    // row groups straddle warps more often and it measures no faster (0.376 vs 0.373 ms)
    return try_pack<72, 14, 4>(L, a, b, nst, st) ||
           try_spec<T, 72, 14, 8>(L, a, b, nst, st) || try_spec<T, 40, 22, 8>(L, a, b, nst, st) ||
           try_spec<T, 136, 14, 4>(L, a, b, nst, st) || try_spec<T, 24, 22, 3>(L, a, b, nst, st) ||
           try_spec<T, 16, 14, 2>(L, a, b, nst, st);
}

}  // namespace

template <class T>
bool encode_dense_tmap(CUtensorMap* map, const FusedRhs<T>& rb, int bw, int rows) {
  return get_encode() && encode_rhs_map<T>(map, rb, bw, rows);
}
template bool encode_dense_tmap<double>(CUtensorMap*, const FusedRhs<double>&, int, int);
template bool encode_dense_tmap<float>(CUtensorMap*, const FusedRhs<float>&, int, int);

// tau + degree-2 pass (FIN = 2): rhs holds R on F on entry and the tau rhs on exit
template <class T>
bool launch_tau_cheb2_fused(const Lvl& L, const T* u_in, T* u_out, const T* R, T* rhs, T* t,
                            int jr, double c0, double cm, double cr, cudaStream_t st) {
  Cheb2Args<T> a{};
  a.L = L;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = R;
  a.rhs_global = 0;
  a.rhs_out = rhs;
  a.tout = t;
  a.jr = jr;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  FusedRhs<T> b{};
  b.p = R;
  b.global = 0;
  return launch_spec<T>(L, a, b, 2, st);
}
template bool launch_tau_cheb2_fused<double>(const Lvl&, const double*, double*, const double*,
                                             double*, double*, int, double, double, double,
                                             cudaStream_t);
template bool launch_tau_cheb2_fused<float>(const Lvl&, const float*, float*, const float*, float*,
                                            float*, int, double, double, double, cudaStream_t);

template <class T>
bool cheb2_final_ok(const Lvl& L) {
  return cheb_spec_ok<T>(L);
}
template bool cheb2_final_ok<double>(const Lvl&);
template bool cheb2_final_ok<float>(const Lvl&);

template <class T>
void launch_cheb2_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, double c0, double cm,
                        double cr, cudaStream_t st, FinalOut<T> fin) {
  {
    Cheb2Args<T> a{};
    a.fin = fin;
    for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
    a.L = L;
    a.uin = u_in;
    a.uout = u_out;
    a.rhs_seg = b.global ? nullptr : b.p;
    a.rhs_global = b.global;
    a.c0 = (T)c0;
    a.cm = (T)cm;
    a.cr = (T)cr;
    if (launch_spec<T>(L, a, b, 2, st)) return;
  }
  const Variant v = variant<T>();
  const Plan pl = make_plan<T>(L, v.maxs, v.nt);
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (b.global) encode_rhs_map<T>(&map, b, pl.bw, pl.BH + 2);
  Cheb2Args<T> a{};
  a.L = L;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.rhs_global = b.global;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  a.BH = pl.BH;
  a.u0_stride = pl.u0_stride;
  a.s_stride = pl.s_stride;
  a.f_stride = pl.f_stride;
  a.bw = pl.bw;
  a.c0 = (T)c0;
  a.cm = (T)cm;
  a.cr = (T)cr;
  dim3 grid(pl.nbands, L.nsegs);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
    kern<<<grid, pl.NT, pl.smem, st>>>(map, a);
  };
  go(k_cheb2<T, sizeof(T) == 8 ? 6 : 8, 512>);
}

template <class T>
bool cheb_spec_ok(const Lvl& L) {
  if (!get_encode() || ((long long)L.N[0] * sizeof(T)) % 16) return false;
  const int pys[5] = {136, 72, 40, 24, 16};
  for (int p : pys)
    if (L.py == p && L.E[0] <= p) return true;
  return false;
}
template bool cheb_spec_ok<double>(const Lvl&);
template bool cheb_spec_ok<float>(const Lvl&);

template <class T>
bool launch_cheb1_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, double c0,
                        cudaStream_t st) {
  if (!get_encode()) return false;
  Cheb2Args<T> a{};
  a.L = L;
  a.uin = u_in;
  a.uout = u_out;
  a.rhs_seg = b.global ? nullptr : b.p;
  a.rhs_global = b.global;
  for (int d = 0; d < 3; ++d) a.foff[d] = b.global ? b.off[d] : 0;
  a.c0 = (T)c0;
  return launch_spec<T>(L, a, b, 1, st);
}

template bool launch_cheb1_fused<double>(const Lvl&, const double*, double*, FusedRhs<double>,
                                         double, cudaStream_t);
template bool launch_cheb1_fused<float>(const Lvl&, const float*, float*, FusedRhs<float>, double,
                                        cudaStream_t);
template void launch_cheb2_fused<double>(const Lvl&, const double*, double*, FusedRhs<double>,
                                         double, double, double, cudaStream_t, FinalOut<double>);
template void launch_cheb2_fused<float>(const Lvl&, const float*, float*, FusedRhs<float>, double,
                                        double, double, cudaStream_t, FinalOut<float>);
template bool cheb2_fused_ok<double>(const Lvl&);
template bool cheb2_fused_ok<float>(const Lvl&);

}  // namespace srfmg
