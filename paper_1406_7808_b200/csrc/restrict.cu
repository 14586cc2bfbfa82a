// Residual + 8-child average restriction on the SR levels, fed by bulk copies (sm_100a):
// the same operation as k_restrict (kernels.cu; fig:mgv L113-115, fig:mgvsr L233/L235, R9)
//   uc[I] = (1/8) sum_children u_f,   rc[I] = (1/8) sum_children (b - A u_f)
// on the coarse target box grow(coarsen(V_f^p), jr) of every segment, with the restricted
// residual taken from the R6 pyramid when b is f_l (bc = avg8(f_l): rc = bc - avg8(A u)).
//
// k_restrict marches coarse columns with plain global loads and is load-latency bound
// (72 % long-scoreboard stalls at C3's finest level, 4.6 TB/s).  Here one CTA takes a band
// of BHc coarse rows of one segment and marches coarse Z: the fine u rows of the band
// (2 BHc + 2 rows, the stencil's y halo included) arrive one plane per bulk copy into a
// 6-plane ring two planes per step ahead, the segment-storage rhs (no pyramid) likewise into
// a 4-plane ring.  Thread (tx, ty) owns fine column 2X + (tx & 1) of coarse row Y = Ya + ty:
// the 2 x 2 (y, z) children of that column, their z neighbours in a register queue, the y
// neighbours from the same column, the x neighbours from the two adjacent columns in shared
// memory; the x pair is summed with one shuffle.  One __syncthreads per coarse plane.
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "kernels.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

constexpr int kRU = 6;  // u planes in the ring (4 read per step, 2 in flight)
constexpr int kRB = 6;  // rhs planes (2 read per step, 4 in flight): both rings cycle in 3 steps

template <class T>
struct RsArgs {
  Lvl Lf, Lc;
  const T* uf;
  const T* bseg;   // segment-storage rhs (SEGB = 1)
  View<T> bc;      // coarse pyramid f_{l-1} (SEGB = 0)
  T* uc;
  T* rc;
  int jr;
  int upl, bpl;    // elements per staged plane (u, rhs)
};

template <class T, int PY, int SEGB, int NL>
__global__ void __launch_bounds__(512, 2) k_restrict_s(const __grid_constant__ RsArgs<T> a) {
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& Lf = a.Lf;
  const Lvl& Lc = a.Lc;
  const int BHc = blockDim.y;
  const int s = blockIdx.y;
  int pf[3], of[3], lo[3];
  pf[0] = s % Lf.ns[0] + Lf.so[0];
  pf[1] = (s / Lf.ns[0]) % Lf.ns[1] + Lf.so[1];
  pf[2] = s / (Lf.ns[0] * Lf.ns[1]) + Lf.so[2];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    of[d] = pf[d] * Lf.S[d] - (Lf.J + 1);
    lo[d] = pf[d] * (Lf.S[d] / 2) - a.jr;
  }
  const int B = Lf.S[0] / 2 + 2 * a.jr;
  const int Xa = max(lo[0], 0), Xb = min(lo[0] + B, Lc.N[0]);
  const int Ya = max(lo[1], 0) + blockIdx.x * BHc, Yb = min(min(lo[1] + B, Lc.N[1]), Ya + BHc);
  const int Za = max(lo[2], 0), Zb = min(lo[2] + B, Lc.N[2]);
  if (Ya >= Yb || Za >= Zb || Xa >= Xb) return;  // (uniform per CTA)
  T* us = reinterpret_cast<T*>(sm);
  T* bs = us + kRU * a.upl;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bs + (SEGB ? kRB * a.bpl : 0));
  const long long fpz = Lf.pz;
  // u: fine rows 2Ya - 1 .. 2Yb (local row 0 = 2Ya - 1), planes 2Za - 1 .. 2Zb (index i)
  const int nrow = 2 * (Yb - Ya) + 2;
  const uint32_t ubytes = (uint32_t)(nrow * PY * sizeof(T));
  const T* usrc = a.uf + (long long)s * Lf.ss + (long long)(2 * Ya - 1 - of[1]) * PY +
                  (long long)(2 * Za - 1 - of[2]) * fpz;
  const int nu = 2 * (Zb - Za) + 2;
  // rhs (SEGB): fine rows 2Ya .. 2Yb - 1, planes 2Za .. 2Zb - 1 (index j)
  const uint32_t bbytes = (uint32_t)((nrow - 2) * PY * sizeof(T));
  const T* bsrc = SEGB ? a.bseg + (long long)s * Lf.ss + (long long)(2 * Ya - of[1]) * PY +
                             (long long)(2 * Za - of[2]) * fpz
                       : nullptr;
  const int nb = 2 * (Zb - Za);
  const bool lead = threadIdx.x == 0 && threadIdx.y == 0;
  if (lead) {
    for (int i = 0; i < kRU + (SEGB ? kRB : 0); ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_u = [&](int i) {
    const int sl = i % kRU;
    mbar_expect_tx(&bars[sl], ubytes);
    bulk_g2s(us + sl * a.upl, usrc + (long long)i * fpz, ubytes, &bars[sl]);
  };
  auto issue_b = [&](int j) {
    const int sl = j % kRB;
    mbar_expect_tx(&bars[kRU + sl], bbytes);
    bulk_g2s(bs + sl * a.bpl, bsrc + (long long)j * fpz, bbytes, &bars[kRU + sl]);
  };
  if (lead) {
    for (int i = 0; i < min(kRU, nu); ++i) issue_u(i);
    if (SEGB)
      for (int j = 0; j < min(kRB, nb); ++j) issue_b(j);
  }
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int dx = tx & 1;
  const int X = Xa + (tx >> 1), Y = Ya + ty;
  const bool valid = X < Xb && Y < Yb;
  // fine local column and the first of the four u rows (2Y - 1 .. 2Y + 2) this thread reads
  const int fxl = valid ? 2 * X + dx - of[0] : 1;
  const int r0 = valid ? 2 * ty : 0;
  const T* const uc0 = us + r0 * PY + fxl;
  const T* const bc0 = bs + r0 * PY + fxl;
  // A u = ((6 + n_out) v - sum of the six neighbours) / h^2: cells outside Omega hold zero in
  // the storage (as k_cheb2s relies on), so the reflected ghost -v (R3) is the diagonal's
  // count of outside neighbours -- x and y per thread and fine row, z per coarse plane
  const int bx = (dx == 0 && X == 0) + (dx == 1 && X == Lc.N[0] - 1);
  const T d1 = T(6 + bx + (Y == 0)), d2 = T(6 + bx + (Y == Lc.N[1] - 1));  // rows 2Y, 2Y+1
  const T ih2 = T(Lf.inv_h2), nlg = T(Lf.nlg);
  const int cs = Lc.nsegs == 1 ? 0 : s;
  int oc[3];
  {
    const int pc0 = cs % Lc.ns[0] + Lc.so[0], pc1 = (cs / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
              pc2 = cs / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
    oc[0] = pc0 * Lc.S[0] - (Lc.J + 1);
    oc[1] = pc1 * Lc.S[1] - (Lc.J + 1);
    oc[2] = pc2 * Lc.S[2] - (Lc.J + 1);
  }
  const bool writer = valid && dx == 0;
  const long long cpz = Lc.pz;
  const long long co0 = writer ? (long long)cs * Lc.ss + (long long)(Za - oc[2]) * cpz +
                                     (long long)(Y - oc[1]) * Lc.py + (X - oc[0])
                               : 0;
  T* ucp = a.uc + co0;
  T* rcp = a.rc + co0;
  const T* bcp = SEGB ? nullptr : a.bc.p + (long long)Za * a.bc.sz + (long long)Y * a.bc.sy + X;
  const long long bsz = SEGB ? 0 : a.bc.sz;
  T bcn = T(0);  // pyramid value of the next coarse plane (loaded one plane ahead)
  if (!SEGB && writer) bcn = *bcp;

  // c[p][r]: u of this column at fine plane 2Z - 1 + p, fine row 2Y - 1 + r
  T c[4][4];
  mbar_wait(&bars[0], 0);
  mbar_wait(&bars[1], 0);
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int r = 0; r < 4; ++r) c[p][r] = uc0[p * a.upl + r * PY];

  // coarse plane Z = Za + 3m + R: u planes i = 2k .. 2k+3 in slots 2R .. 2R+3 (mod 6), the
  // rhs planes j = 2k, 2k+1 in slots 2R, 2R+1; ring phase m (+1 past the wrap)
  auto step = [&](auto RR, int m) {
    constexpr int R = decltype(RR)::value;
    constexpr int S1 = 2 * R + 1, S2 = (2 * R + 2) % kRU, S3 = (2 * R + 3) % kRU;
    const int k = 3 * m + R;
    const int Z = Za + k;
    T bcv = T(0);
    if (!SEGB && writer) {
      bcv = bcn;
      if (Z + 1 < Zb) bcn = bcp[(long long)(k + 1) * bsz];
    }
    const uint32_t ph = (uint32_t)(m & 1);
    mbar_wait(&bars[S2], 2 * R + 2 >= kRU ? ph ^ 1u : ph);
    mbar_wait(&bars[S3], 2 * R + 3 >= kRU ? ph ^ 1u : ph);
    if (SEGB) {
      mbar_wait(&bars[kRU + 2 * R], ph);
      mbar_wait(&bars[kRU + 2 * R + 1], ph);
    }
    const T* p1 = uc0 + S1 * a.upl;
    const T* p2 = uc0 + S2 * a.upl;
    const T* p3 = uc0 + S3 * a.upl;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      c[2][r] = p2[r * PY];
      c[3][r] = p3[r * PY];
    }
    const T dz1 = T(Z == 0), dz2 = T(Z == Lc.N[2] - 1);  // planes 2Z, 2Z+1
    T su = T(0), sa = T(0), sb = T(0);
#pragma unroll
    for (int p = 1; p <= 2; ++p) {
      const T* pl = p == 1 ? p1 : p2;
      const T* bp = bc0 + (2 * R + p - 1) * a.bpl;
#pragma unroll
      for (int r = 1; r <= 2; ++r) {
        const T v = c[p][r];
        const T sum = ((c[p - 1][r] + c[p + 1][r]) + (c[p][r - 1] + c[p][r + 1])) +
                      (pl[r * PY - 1] + pl[r * PY + 1]);
        const T dg = (r == 1 ? d1 : d2) + (p == 1 ? dz1 : dz2);
        su += v;
        if (NL) {  // f4 (R29): A(u) = -L_h u + nlg u^3
          const T Au = (dg * v - sum) * ih2 + nlg * v * v * v;
          if (SEGB) sa += bp[(r - 1) * PY] - Au;
          else sa -= Au;
        } else {   // linear: the 1/h^2 is applied once to the sum of the four cells
          sa += sum - dg * v;
          if (SEGB) sb += bp[(r - 1) * PY];
        }
      }
    }
    if (!NL) sa = SEGB ? sb + sa * ih2 : sa * ih2;
    // (the block's thread count is even and rows are 2B wide: x pairs share a warp; a
    // partial last warp shuffles among its existing lanes)
    const unsigned am = __activemask();
    su += __shfl_xor_sync(am, su, 1);
    sa += __shfl_xor_sync(am, sa, 1);
    if (writer) {
      *ucp = su * T(0.125);
      *rcp = SEGB ? sa * T(0.125) : bcv + sa * T(0.125);
      ucp += cpz;
      rcp += cpz;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      c[0][r] = c[2][r];
      c[1][r] = c[3][r];
    }
    __syncthreads();  // u planes 2k, 2k+1 and rhs planes 2k, 2k+1 free
    if (lead) {
      if (2 * k + kRU < nu) issue_u(2 * k + kRU);
      if (2 * k + 1 + kRU < nu) issue_u(2 * k + 1 + kRU);
      if (SEGB) {
        if (2 * k + kRB < nb) issue_b(2 * k + kRB);
        if (2 * k + 1 + kRB < nb) issue_b(2 * k + 1 + kRB);
      }
    }
  };
  const int nz = Zb - Za;
  for (int m = 0; 3 * m < nz; ++m) {
    step(std::integral_constant<int, 0>{}, m);
    if (3 * m + 1 < nz) step(std::integral_constant<int, 1>{}, m);
    if (3 * m + 2 < nz) step(std::integral_constant<int, 2>{}, m);
  }
}

template <class T, int PY>
bool try_rs(const Lvl& Lf, const Lvl& Lc, const T* uf, View<T> bf, View<T> bc, T* uc, T* rc,
            int jr, cudaStream_t st, bool launch) {
  if (Lf.py != PY) return false;
  const bool segb = bc.p == nullptr;
  if (segb && (bf.global || bf.p == nullptr || bf.sy != Lf.py || bf.sz != Lf.pz || bf.ss != Lf.ss))
    return false;
  if (!segb && !bc.global) return false;
  const int B = Lf.S[0] / 2 + 2 * jr;
  if (Lf.S[1] / 2 + 2 * jr != B || 2 * B > 1024) return false;
  // the fine rows / planes read lie in the storage box: 2 jr <= J
  if (2 * jr > Lf.J) return false;
  // band height: at most 512 threads (two CTAs per SM at <= 64 registers), bands balanced
  const int bhmax = std::max(1, std::min(B, 512 / (2 * B)));
  const int nb = (B + bhmax - 1) / bhmax;
  const int bh = (B + nb - 1) / nb;
  constexpr int A = 128 / (int)sizeof(T);
  const int upl = ((2 * bh + 2) * PY + A - 1) / A * A;
  const int bpl = ((2 * bh) * PY + A - 1) / A * A;
  const size_t smem = (size_t)(kRU * upl + (segb ? kRB * bpl : 0)) * sizeof(T) + 8 * (kRU + kRB);
  if (smem > 200 * 1024) return false;
  if (!launch) return true;
  RsArgs<T> a{};
  a.Lf = Lf;
  a.Lc = Lc;
  a.uf = uf;
  a.bseg = segb ? bf.p : nullptr;
  a.bc = bc;
  a.uc = uc;
  a.rc = rc;
  a.jr = jr;
  a.upl = upl;
  a.bpl = bpl;
  dim3 grid(nb, Lf.nsegs), block(2 * B, bh);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, block, smem, st>>>(a);
  };
  const bool nl = Lf.nlg != 0.0;
  if (segb) {
    if (nl) go(k_restrict_s<T, PY, 1, 1>);
    else go(k_restrict_s<T, PY, 1, 0>);
  } else {
    if (nl) go(k_restrict_s<T, PY, 0, 1>);
    else go(k_restrict_s<T, PY, 0, 0>);
  }
  return true;
}

template <class T>
bool rs_dispatch(const Lvl& Lf, const Lvl& Lc, const T* uf, View<T> bf, View<T> bc, T* uc, T* rc,
                 int jr, cudaStream_t st, bool launch) {
  if (Lf.st27 || Lf.nsegs < 1) return false;
  return try_rs<T, 72>(Lf, Lc, uf, bf, bc, uc, rc, jr, st, launch) ||
         try_rs<T, 40>(Lf, Lc, uf, bf, bc, uc, rc, jr, st, launch) ||
         try_rs<T, 24>(Lf, Lc, uf, bf, bc, uc, rc, jr, st, launch) ||
         try_rs<T, 16>(Lf, Lc, uf, bf, bc, uc, rc, jr, st, launch);
}

}  // namespace

template <class T>
bool launch_restrict_seg(const Lvl& Lf, const T* uf, View<T> bf, const Lvl& Lc, T* uc, T* rc,
                         int jr, cudaStream_t st, View<T> bc) {
  return rs_dispatch<T>(Lf, Lc, uf, bf, bc, uc, rc, jr, st, true);
}

template bool launch_restrict_seg<double>(const Lvl&, const double*, View<double>, const Lvl&,
                                          double*, double*, int, cudaStream_t, View<double>);
template bool launch_restrict_seg<float>(const Lvl&, const float*, View<float>, const Lvl&,
                                         float*, float*, int, cudaStream_t, View<float>);

}  // namespace srfmg
