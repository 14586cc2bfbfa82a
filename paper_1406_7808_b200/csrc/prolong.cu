// TMA-fed trilinear prolongation onto C ∪ GSR (R10; fig:fmgsr L221 SET, fig:mgvsr L241 ADD).
//
// Work unit: a y-band of one fine segment.  The coarse source rows the band needs (its
// parents +-1, coarse storage is contiguous per plane) are streamed plane by plane into a
// 4-deep shared-memory ring with cp.async.bulk (w and, for ADD, t); for ADD the fine u rows
// of the band are streamed the same way.  Each thread owns MAXS consecutive fine rows of one
// column and keeps, per row, the (x, y)-interpolant I(P) of the last three coarse planes in
// registers (separable trilinear: the xy part of coarse plane P is shared by the fine planes
// 2P and 2P+1).  Reflected coarse ghosts (R3) enter as signed weights (x, y) and signed
// interpolants (z).  Output is written straight from registers (coalesced rows).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <type_traits>

#include "fused.cuh"
#include "tma.cuh"

namespace srfmg {

namespace {

constexpr int kRC = 4;  // coarse plane ring
constexpr int kRF = 4;  // fine plane ring (ADD)

template <class T>
struct ProlongArgs {
  Lvl Lf, Lc;
  T* uf;
  const T* w;
  const T* t;
  int add;
  int BH;       // fine rows per band
  int cstride;  // elements per coarse smem plane (one field)
  int fstride;  // elements per fine smem plane
};

// PYC != 0: the fine row pitch (and the coarse one, PYC/2 + 4, as the segment storage of
// the next coarser SR level has) at compile time; ADD: the correction (fig:mgvsr L241)
template <class T, int MAXS, int ADD, int PYC>
// (6 rows per thread: at most 72 x 4 threads, registers up to 128 -- no spills)
__global__ void __launch_bounds__(MAXS == 6 ? 512 : 1024, 1)
    k_prolong_tma(const __grid_constant__ ProlongArgs<T> a) {
  extern __shared__ __align__(128) unsigned char sm[];
  const Lvl& Lf = a.Lf;
  const Lvl& Lc = a.Lc;
  const int s = blockIdx.y;
  const int Ey = Lf.E[1], Ez = Lf.E[2], Ex = Lf.E[0];
  const int fpy = PYC ? PYC : Lf.py;
  const int cpyc = PYC ? PYC / 2 + 4 : Lc.py;
  const int r0 = blockIdx.x * a.BH, r1 = min(Ey, r0 + a.BH);
  // fine segment geometry
  const int px = s % Lf.ns[0] + Lf.so[0], py_ = (s / Lf.ns[0]) % Lf.ns[1] + Lf.so[1],
            pz_ = s / (Lf.ns[0] * Lf.ns[1]) + Lf.so[2];
  const int ox = px * Lf.S[0] - (Lf.J + 1), oy = py_ * Lf.S[1] - (Lf.J + 1),
            oz = pz_ * Lf.S[2] - (Lf.J + 1);
  // coarse segment: the fine segment's own coarse storage, or the single global array
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  const int cpx = cs % Lc.ns[0] + Lc.so[0], cpy = (cs / Lc.ns[0]) % Lc.ns[1] + Lc.so[1],
            cpz = cs / (Lc.ns[0] * Lc.ns[1]) + Lc.so[2];
  const int ocx = cpx * Lc.S[0] - (Lc.J + 1), ocy = cpy * Lc.S[1] - (Lc.J + 1),
            ocz = cpz * Lc.S[2] - (Lc.J + 1);
  // fine rows / planes inside Omega
  const int gy_lo = max(oy + r0, 0), gy_hi = min(oy + r1, Lf.N[1]);
  const int gz_lo = max(oz, 0), gz_hi = min(oz + Ez, Lf.N[2]);
  if (gy_lo >= gy_hi || gz_lo >= gz_hi) return;
  // coarse rows / planes staged (parents +-1, reflected rows fold onto 0 / N-1)
  const int cy_lo = max((gy_lo >> 1) - 1, 0), cy_hi = min(((gy_hi - 1) >> 1) + 1, Lc.N[1] - 1);
  const int cz_lo = max((gz_lo >> 1) - 1, 0), cz_hi = min(((gz_hi - 1) >> 1) + 1, Lc.N[2] - 1);
  const int crows = cy_hi - cy_lo + 1;
  const uint32_t cbytes = (uint32_t)(crows * cpyc * sizeof(T));
  const uint32_t fbytes = (uint32_t)((r1 - r0) * fpy * sizeof(T));
  T* cw = reinterpret_cast<T*>(sm);               // kRC planes of w
  T* ct = cw + kRC * a.cstride;                   // kRC planes of t (ADD)
  T* fu = ct + kRC * a.cstride;                   // kRF planes of fine u (ADD)
  uint64_t* bars = reinterpret_cast<uint64_t*>(fu + kRF * a.fstride);  // [0,kRC) coarse, then fine
  const T* wseg = a.w + (long long)cs * Lc.ss + (long long)(cy_lo - ocy) * cpyc;
  const T* tseg = ADD ? a.t + (long long)cs * Lc.ss + (long long)(cy_lo - ocy) * cpyc : nullptr;
  T* useg = a.uf + (long long)s * Lf.ss;
  const int P0 = gz_lo >> 1, P1 = (gz_hi - 1) >> 1;  // parent planes looped over
  const int fz0 = 2 * P0;                            // first fine plane of the loop (global)

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRC + kRF; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue_c = [&](int c) {  // coarse plane c (global), c in [cz_lo, cz_hi]
    const int sl = (c - cz_lo) % kRC;
    mbar_expect_tx(&bars[sl], ADD ? 2 * cbytes : cbytes);
    const long long zo = (long long)(c - ocz) * Lc.pz;
    bulk_g2s(cw + sl * a.cstride, wseg + zo, cbytes, &bars[sl]);
    if (ADD) bulk_g2s(ct + sl * a.cstride, tseg + zo, cbytes, &bars[sl]);
  };
  auto issue_f = [&](int gz) {  // fine plane gz (global), ADD only
    const int sl = (gz - gz_lo) % kRF;
    mbar_expect_tx(&bars[kRC + sl], fbytes);
    bulk_g2s(fu + sl * a.fstride, useg + (long long)(gz - oz) * Lf.pz + (long long)r0 * fpy,
             fbytes, &bars[kRC + sl]);
  };
  int nc = cz_lo, nf = gz_lo;  // next coarse / fine plane to issue (thread 0)
  if (threadIdx.x == 0) {
    for (; nc <= min(cz_hi, cz_lo + kRC - 1); ++nc) issue_c(nc);
    if (ADD)
      for (; nf < min(gz_lo + kRF, gz_hi); ++nf) issue_f(nf);
  }

  // ---- this thread: column tx, rows r0 + g*MAXS + k
  const int tx = threadIdx.x % fpy, g = threadIdx.x / fpy;
  const int gx = ox + tx;
  const bool xin = tx < Ex && gx >= 0 && gx < Lf.N[0];
  int cxo[2];
  T sx = T(1);
  {
    const int P = gx >> 1, Q = P + ((gx & 1) ? 1 : -1);
    int Qm = Q;
    if (Q < 0) { Qm = 0; sx = T(-1); }
    if (Q >= Lc.N[0]) { Qm = Lc.N[0] - 1; sx = T(-1); }
    cxo[0] = min(max(P - ocx, 0), Lc.E[0] - 1);
    cxo[1] = min(max(Qm - ocx, 0), Lc.E[0] - 1);
  }
  const T W0 = T(0.75), W1 = T(0.25);
  const T W1x = W1 * sx;
  int yo[MAXS][2];     // coarse smem row offsets (parent, neighbour)
  T sy[MAXS];          // sign of the y neighbour (-1: reflected ghost)
  unsigned out_mask = 0;
#pragma unroll
  for (int k = 0; k < MAXS; ++k) {
    const int y = r0 + g * MAXS + k;
    const int gy = oy + y;
    sy[k] = T(1);
    int P = gy >> 1, Q = P + ((gy & 1) ? 1 : -1);
    if (Q < 0) { Q = 0; sy[k] = T(-1); }
    if (Q >= Lc.N[1]) { Q = Lc.N[1] - 1; sy[k] = T(-1); }
    const bool ok = xin && y < r1 && gy >= 0 && gy < Lf.N[1];
    if (ok) out_mask |= 1u << k;
    P = min(max(P, cy_lo), cy_hi);
    Q = min(max(Q, cy_lo), cy_hi);
    yo[k][0] = (P - cy_lo) * cpyc;
    yo[k][1] = (Q - cy_lo) * cpyc;
  }
  auto interp = [&](int c, T* I) {  // xy-interpolants of real coarse plane c for all slots
    const int sl = (c - cz_lo) % kRC;
    const T* pw = cw + sl * a.cstride;
    const T* pt = ct + sl * a.cstride;
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      T v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int o = yo[k][j >> 1] + cxo[j & 1];
        v[j] = pw[o];
        if (ADD) v[j] = v[j] - pt[o];
      }
      // I = W0 (W0 v_pp + W1 sx v_pn) + W1 sy (W0 v_np + W1 sx v_nn)
      I[k] = W0 * (W0 * v[0] + W1x * v[1]) + W1 * sy[k] * (W0 * v[2] + W1x * v[3]);
    }
  };
  auto wait_c = [&](int c) {
    const int n = c - cz_lo;
    mbar_wait(&bars[n % kRC], (n / kRC) & 1);
  };
  // interpolant of coarse plane c (global, may be -1 or N: reflected)
  T Im[MAXS], I0[MAXS], Ip[MAXS];
  auto get = [&](int c, T* I) {
    T sg = T(1);
    if (c < 0) { c = 0; sg = T(-1); }
    if (c >= Lc.N[2]) { c = Lc.N[2] - 1; sg = T(-1); }
    interp(c, I);
#pragma unroll
    for (int k = 0; k < MAXS; ++k) I[k] *= sg;
  };
  wait_c(max(P0 - 1, 0));
  wait_c(P0);
  get(P0 - 1, Im);
  get(P0, I0);
  T* const ucol = useg + (long long)(r0 + g * MAXS) * fpy + tx;
  const long long pzf = Lf.pz;
  for (int P = P0; P <= P1; ++P) {
    const int cn = min(P + 1, Lc.N[2] - 1);
    if (P + 1 < Lc.N[2]) wait_c(cn);
    get(P + 1, Ip);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gz = 2 * P + e;
      if (gz < gz_lo || gz >= gz_hi) continue;
      const T* uin = nullptr;
      if (ADD) {
        const int n = gz - gz_lo;
        mbar_wait(&bars[kRC + n % kRF], (n / kRF) & 1);
        uin = fu + (n % kRF) * a.fstride + (g * MAXS) * fpy + tx;
      }
      T* orow = ucol + (long long)(gz - oz) * pzf;
#pragma unroll
      for (int k = 0; k < MAXS; ++k) {
        if (!((out_mask >> k) & 1u)) continue;
        const T acc = W0 * I0[k] + W1 * (e ? Ip[k] : Im[k]);
        orow[k * fpy] = ADD ? uin[k * fpy] + acc : acc;
      }
    }
    __syncthreads();  // coarse plane P-1 and fine planes 2P, 2P+1 are free
    if (threadIdx.x == 0) {
      // planes P..P+3 may now be resident (the slot of P-1 is free); fine 2P+2..2P+5
      for (; nc <= min(cz_hi, P + 3); ++nc) issue_c(nc);
      if (ADD)
        for (; nf <= min(gz_hi - 1, 2 * P + 5); ++nf) issue_f(nf);
    }
#pragma unroll
    for (int k = 0; k < MAXS; ++k) {
      Im[k] = I0[k];
      I0[k] = Ip[k];
    }
  }
}

}  // namespace

// band plan of the TMA prolongation: rows per thread, band height, shared memory
struct TmaBandPlan {
  int maxs, nb, BH;
  long long cstride, fstride;
  size_t smem;
};
template <class T>
TmaBandPlan prolong_plan(const Lvl& Lf, const Lvl& Lc) {
  // measured at C3: 18-row bands at E = 70 (0.55 ms; 10: 0.61, 24: 0.66), two 19-row bands at
  // E = 38 (0.22 ms for the level's two launches; three of 13: 0.24).  SR_FMG_PROLONG_MAXS
  // (3 or 6 rows per thread) and SR_FMG_PROLONG_BH (target band height): tuning knobs
  static const int maxs_env = [] {
    const char* e = std::getenv("SR_FMG_PROLONG_MAXS");
    return e ? std::atoi(e) : 0;
  }();
  static const int bh_env = [] {
    const char* e = std::getenv("SR_FMG_PROLONG_BH");
    return e ? std::atoi(e) : 0;
  }();
  TmaBandPlan p{};
  // 6 rows per thread from E = 22 on (C3, fp64: finest correction 0.515 vs 0.538 ms, level 7
  // 0.207 vs 0.221; fp32 finest 0.311 vs 0.416 ms), 3 on the E = 14 boxes (0.074 vs 0.090)
  p.maxs = maxs_env ? (maxs_env == 6 ? 6 : 3) : (Lf.E[1] >= 22 ? 6 : 3);
  // (two bands on the E <= 22 boxes: slower, level 6 0.088 -> 0.111 ms per solve)
  const int tgt = bh_env > 0 ? bh_env : (Lf.E[1] <= 40 ? 24 : 18);
  p.nb = (Lf.E[1] + tgt - 1) / tgt;
  p.BH = (Lf.E[1] + p.nb - 1) / p.nb;
  const int crows = p.BH / 2 + 3;
  const int A = 128 / (int)sizeof(T);
  p.cstride = ((long long)crows * Lc.py + A - 1) / A * A;
  p.fstride = ((long long)p.BH * Lf.py + A - 1) / A * A;
  p.smem = (size_t)(2 * kRC * p.cstride + kRF * p.fstride) * sizeof(T) + 8 * (kRC + kRF);
  return p;
}

template <class T>
bool prolong_tma_fits(const Lvl& Lf, const Lvl& Lc) {
  return Lf.py <= 136 && prolong_plan<T>(Lf, Lc).smem <= 227 * 1024;
}

template <class T>
bool prolong_tma_ok(const Lvl& Lf, const Lvl& Lc) {
  // enough bands to fill the GPU, counted over the GLOBAL segment grid so that every world
  // size picks the same kernel (R25)
  long long g = 1;
  for (int i = 0; i < 3; ++i) g *= Lf.N[i] / Lf.S[i];
  // one thread per row column and MAXS rows: rows up to 136 wide keep a band within the
  // 1024-thread CTA limit (E = 262 boxes, e.g. 256^3 segments, take the column kernel); the
  // coarse rows are staged whole, so a wide coarse level (the first SR level over a large
  // conventional level T, e.g. C5 with K = 2) can exceed shared memory: column kernel
  return g * ((Lf.E[1] + 17) / 18) >= 148 && prolong_tma_fits<T>(Lf, Lc);
}

template <class T>
void launch_prolong_tma(const Lvl& Lf, T* uf, const Lvl& Lc, const T* w, const T* t, int add,
                        cudaStream_t st) {
  const TmaBandPlan pp = prolong_plan<T>(Lf, Lc);
  const int MAXS = pp.maxs, nb = pp.nb, BH = pp.BH;
  ProlongArgs<T> a{};
  a.Lf = Lf;
  a.Lc = Lc;
  a.uf = uf;
  a.w = w;
  a.t = t;
  a.add = add;
  a.BH = BH;
  a.cstride = (int)pp.cstride;
  a.fstride = (int)pp.fstride;
  const size_t smem = pp.smem;
  const int NT = Lf.py * ((BH + MAXS - 1) / MAXS);
  // compile-time pitches for the C3-type boxes (E = 70, 38 over a coarse SR level)
  const int pyc = (Lf.py == 72 || Lf.py == 40) && Lc.py == Lf.py / 2 + 4 ? Lf.py : 0;
  auto pick = [&](auto MS) {
    constexpr int M = decltype(MS)::value;
    if (add) {
      if (pyc == 72) return k_prolong_tma<T, M, 1, 72>;
      if (pyc == 40) return k_prolong_tma<T, M, 1, 40>;
      return k_prolong_tma<T, M, 1, 0>;
    }
    if (pyc == 72) return k_prolong_tma<T, M, 0, 72>;
    if (pyc == 40) return k_prolong_tma<T, M, 0, 40>;
    return k_prolong_tma<T, M, 0, 0>;
  };
  auto kern = MAXS == 6 ? pick(std::integral_constant<int, 6>{}) : pick(std::integral_constant<int, 3>{});
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<dim3(nb, Lf.nsegs), NT, smem, st>>>(a);
}

template bool prolong_tma_ok<double>(const Lvl&, const Lvl&);
template bool prolong_tma_fits<double>(const Lvl&, const Lvl&);
template bool prolong_tma_fits<float>(const Lvl&, const Lvl&);
template bool prolong_tma_ok<float>(const Lvl&, const Lvl&);
template void launch_prolong_tma<double>(const Lvl&, double*, const Lvl&, const double*,
                                         const double*, int, cudaStream_t);
template void launch_prolong_tma<float>(const Lvl&, float*, const Lvl&, const float*, const float*,
                                        int, cudaStream_t);

}  // namespace srfmg
