// Unfused reference-layout kernels of the SR-FMG schedule, sm_100a, fp64 and fp32.
//
// One thread per cell of a segment's storage (or target) box; blockIdx.y = segment.
// These are the straightforward kernels the fused passes (fused.cu) are checked against;
// they also run every level the fused passes do not cover.  Each kernel cites the step of
// the paper it implements (PAPER.md line numbers; readings R<n> in DESIGN.md §3).
#include <algorithm>

#include "kernels.cuh"

namespace srfmg {

const char* const kKernelNames[] = {"k_cheb_step", "k_restrict", "k_tau", "k_prolong",
                                    "k_coarsest", "k_pyramid", "k_gather"};
const int kNumKernelNames = 7;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void seg_coords(const Lvl& L, int s, int p[3]) {
  p[0] = s % L.ns[0];
  const int t = s / L.ns[0];
  p[1] = t % L.ns[1];
  p[2] = t / L.ns[1];
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

// (A u) at local cell a / global cell g of segment storage `u` (offset `off`):
// A = -Lap_h, 7 points (R1/R2); a neighbour outside Omega is the reflected ghost -u_i
// (R3).  Neighbour sum order z-, z+, y-, y+, x-, x+ (as the oracle).
template <class T>
__device__ __forceinline__ T apply_A(const Lvl& L, const T* __restrict__ u, long long off,
                                     const int g[3]) {
  const T c = u[off];
  T s = T(0);
  s += (g[2] > 0) ? u[off - L.pz] : -c;
  s += (g[2] < L.N[2] - 1) ? u[off + L.pz] : -c;
  s += (g[1] > 0) ? u[off - L.py] : -c;
  s += (g[1] < L.N[1] - 1) ? u[off + L.py] : -c;
  s += (g[0] > 0) ? u[off - 1] : -c;
  s += (g[0] < L.N[0] - 1) ? u[off + 1] : -c;
  return (T(6) * c - s) * T(L.inv_h2);
}

// ------------------------------------------------------------------------------------
// One Chebyshev step (R8) on the compute region C = grow(V,J) ∩ Omega
// (fig:fmgsr L222, fig:mgvsr L232/L242):
//   out = cur + c_mom (cur - prev) + c_res (b - A cur)      on C
//   out = cur                                               on GSR (if copy_gsr)
// prev may alias out (in-place second step: each thread reads prev at its own cell only).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_cheb_step(Lvl L, const T* __restrict__ cur,
                                                        const T* prev, View<T> b, T* out,
                                                        T c_mom, T c_res, int copy_gsr) {
  const int s = blockIdx.y;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ex * Ey * Ez) return;
  int a[3];
  a[0] = idx % Ex;
  const int t = idx / Ex;
  a[1] = t % Ey;
  a[2] = t / Ey;
  int p[3], o[3], g[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  bool in = true, interior = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g[d] = o[d] + a[d];
    in = in && (g[d] >= 0) && (g[d] < L.N[d]);
    interior = interior && (a[d] >= 1) && (a[d] <= L.E[d] - 2);
  }
  if (!in) return;
  const long long off = loc_off(L, s, a[0], a[1], a[2]);
  if (!interior) {
    if (copy_gsr) out[off] = cur[off];
    return;
  }
  const T c = cur[off];
  const T r = view_at(b, s, a, g) - apply_A(L, cur, off, g);
  T v = c + c_res * r;
  if (prev != nullptr) v = c + c_mom * (c - prev[off]) + c_res * r;
  out[off] = v;
}

// ------------------------------------------------------------------------------------
// Residual + 8-child average restriction (fig:mgv L113-115, fig:mgvsr L233/L235, R9):
// for every coarse cell I of the target box grow(coarsen(V_f^p), jr) ∩ Omega_c
//   uc[I] = (1/8) sum_children u_f          (I-hat, solution restriction)
//   rc[I] = (1/8) sum_children (b - A u_f)  (I, residual restriction; stored in the
//                                           coarse rhs buffer until the tau kernel)
// jr = floor(J_f/2) when the coarse level is an SR level (target F, R15); 0 otherwise
// (target V_T^p at k = 1 (R16), or Omega_c on conventional levels).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_restrict(Lvl Lf, const T* __restrict__ uf,
                                                       View<T> bf, Lvl Lc, T* __restrict__ uc,
                                                       T* __restrict__ rc, int jr) {
  const int s = blockIdx.y;
  int pf[3], of[3];
  seg_coords(Lf, s, pf);
  seg_origin(Lf, pf, of);
  int B[3], lo[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    B[d] = Lf.S[d] / 2 + 2 * jr;
    lo[d] = pf[d] * (Lf.S[d] / 2) - jr;
  }
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B[0] * B[1] * B[2]) return;
  int I[3];
  I[0] = lo[0] + idx % B[0];
  const int t = idx / B[0];
  I[1] = lo[1] + t % B[1];
  I[2] = lo[2] + t / B[1];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    if (I[d] < 0 || I[d] >= Lc.N[d]) return;
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  int pc[3], oc[3];
  seg_coords(Lc, cs, pc);
  seg_origin(Lc, pc, oc);
  T su = T(0), sr = T(0);
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy)
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        int g[3] = {2 * I[0] + dx, 2 * I[1] + dy, 2 * I[2] + dz};
        int a[3] = {g[0] - of[0], g[1] - of[1], g[2] - of[2]};
        const long long off = loc_off(Lf, s, a[0], a[1], a[2]);
        su += uf[off];
        sr += view_at(bf, s, a, g) - apply_A(Lf, uf, off, g);
      }
  const long long co = loc_off(Lc, cs, I[0] - oc[0], I[1] - oc[1], I[2] - oc[2]);
  uc[co] = su * T(0.125);
  rc[co] = sr * T(0.125);
}

// ------------------------------------------------------------------------------------
// FAS coarse right-hand side and t snapshot on a coarse level (Eq. 4; fig:mgv L116-117;
// fig:mgvsr L234-236; R18):
//   t = u                              on the whole storage box
//   rhs = R + A u                      on F   (R = restricted residual already in rhs)
//   rhs = A u                          on C \ F
// F = grow(V, jr) ∩ Omega (jr = floor(J_fine/2) on SR levels; 0 -> F = V = Omega on
// conventional levels).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_tau(Lvl L, const T* __restrict__ u,
                                                  T* __restrict__ rhs, T* __restrict__ t,
                                                  int jr) {
  const int s = blockIdx.y;
  const int Ex = L.E[0], Ey = L.E[1], Ez = L.E[2];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ex * Ey * Ez) return;
  int a[3];
  a[0] = idx % Ex;
  const int tt = idx / Ex;
  a[1] = tt % Ey;
  a[2] = tt / Ey;
  int p[3], o[3], g[3];
  seg_coords(L, s, p);
  seg_origin(L, p, o);
  const long long off = loc_off(L, s, a[0], a[1], a[2]);
  t[off] = u[off];
  bool in = true, interior = true, inF = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g[d] = o[d] + a[d];
    in = in && (g[d] >= 0) && (g[d] < L.N[d]);
    interior = interior && (a[d] >= 1) && (a[d] <= L.E[d] - 2);
    const int vlo = p[d] * L.S[d];
    inF = inF && (g[d] >= vlo - jr) && (g[d] < vlo + L.S[d] + jr);
  }
  if (!in || !interior) return;
  const T Au = apply_A(L, u, off, g);
  rhs[off] = inF ? rhs[off] + Au : Au;
}

// ------------------------------------------------------------------------------------
// Cell-centred trilinear prolongation onto C ∪ GSR = storage ∩ Omega (R10, PAPER.md:256;
// range fig:fmgsr L221 / fig:mgvsr L241, R17):
//   add == 0:  u_f = P(w)          (FMG interpolation Pi)
//   add == 1:  u_f += P(w - t)     (V-cycle correction)
// Coarse cells just outside Omega_c are reflected ghosts -(value at the mirror) (R3).
// The coarse source is the fine segment's own coarse storage (SR level below) or the
// single global coarse array (transition / conventional level below).
// ------------------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(kThreads) k_prolong(Lvl Lf, T* __restrict__ uf, Lvl Lc,
                                                      const T* __restrict__ w,
                                                      const T* __restrict__ tc, int add) {
  const int s = blockIdx.y;
  const int Ex = Lf.E[0], Ey = Lf.E[1], Ez = Lf.E[2];
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Ex * Ey * Ez) return;
  int a[3];
  a[0] = idx % Ex;
  const int tt = idx / Ex;
  a[1] = tt % Ey;
  a[2] = tt / Ey;
  int p[3], o[3], g[3];
  seg_coords(Lf, s, p);
  seg_origin(Lf, p, o);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    g[d] = o[d] + a[d];
    if (g[d] < 0 || g[d] >= Lf.N[d]) return;
  }
  const int cs = (Lc.nsegs == 1) ? 0 : s;
  int pc[3], oc[3];
  seg_coords(Lc, cs, pc);
  seg_origin(Lc, pc, oc);
  // per dimension: coarse local index and sign of the parent (k=0) and neighbour (k=1)
  int ci[3][2];
  T sg[3][2];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int P = g[d] >> 1;
    const int Q = P + ((g[d] & 1) ? 1 : -1);
    int Qm = Q;
    T sq = T(1);
    if (Q < 0) { Qm = 0; sq = T(-1); }
    if (Q >= Lc.N[d]) { Qm = Lc.N[d] - 1; sq = T(-1); }
    ci[d][0] = P - oc[d];
    ci[d][1] = Qm - oc[d];
    sg[d][0] = T(1);
    sg[d][1] = sq;
  }
  const T W[2] = {T(0.75), T(0.25)};
  const long long base = (long long)cs * Lc.ss;
  T acc = T(0);
#pragma unroll
  for (int kz = 0; kz < 2; ++kz)
#pragma unroll
    for (int ky = 0; ky < 2; ++ky)
#pragma unroll
      for (int kx = 0; kx < 2; ++kx) {
        const long long co = base + (long long)ci[2][kz] * Lc.pz + (long long)ci[1][ky] * Lc.py +
                             ci[0][kx];
        T v = w[co];
        if (add) v = v - tc[co];
        acc += (W[kz] * W[ky] * W[kx]) * ((sg[2][kz] * sg[1][ky] * sg[0][kx]) * v);
      }
  const long long off = loc_off(Lf, s, a[0], a[1], a[2]);
  uf[off] = add ? uf[off] + acc : acc;
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
  for (int i = threadIdx.x; i < n0; i += blockDim.x) {
    T acc = T(0);
    for (int j = 0; j < n0; ++j) acc += ainv[(long long)i * n0 + j] * bs[j];
    int g[3] = {i % L.N[0], (i / L.N[0]) % L.N[1], i / (L.N[0] * L.N[1])};
    u[loc_off(L, 0, g[0] + 1, g[1] + 1, g[2] + 1)] = acc;
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

// output: genuine cells of each segment -> user u (R19)
template <class T>
__global__ void __launch_bounds__(kThreads) k_gather(Lvl L, const T* __restrict__ useg,
                                                     T* __restrict__ out) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int g[3];
    g[0] = i % L.N[0];
    g[1] = (i / L.N[0]) % L.N[1];
    g[2] = i / ((long long)L.N[0] * L.N[1]);
    int p[3], a[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      p[d] = g[d] / L.S[d];
      a[d] = g[d] - (p[d] * L.S[d] - (L.J + 1));
    }
    const int s = (p[2] * L.ns[1] + p[1]) * L.ns[0] + p[0];
    out[i] = useg[loc_off(L, s, a[0], a[1], a[2])];
  }
}

inline unsigned nblk(long long n) { return (unsigned)((n + kThreads - 1) / kThreads); }
inline long long ecount(const Lvl& L) { return (long long)L.E[0] * L.E[1] * L.E[2]; }

}  // namespace

template <class T>
void launch_cheb_step(const Lvl& L, const T* cur, const T* prev, View<T> b, T* out, double c_mom,
                      double c_res, int copy_gsr, cudaStream_t st) {
  dim3 grid(nblk(ecount(L)), L.nsegs);
  k_cheb_step<T><<<grid, kThreads, 0, st>>>(L, cur, prev, b, out, (T)c_mom, (T)c_res, copy_gsr);
}

template <class T>
void launch_restrict(const Lvl& Lf, const T* uf, View<T> bf, const Lvl& Lc, T* uc, T* rc, int jr,
                     cudaStream_t st) {
  long long B = 1;
  for (int d = 0; d < 3; ++d) B *= (Lf.S[d] / 2 + 2 * jr);
  dim3 grid(nblk(B), Lf.nsegs);
  k_restrict<T><<<grid, kThreads, 0, st>>>(Lf, uf, bf, Lc, uc, rc, jr);
}

template <class T>
void launch_tau(const Lvl& Lc, const T* u, T* rhs, T* t, int jr, cudaStream_t st) {
  dim3 grid(nblk(ecount(Lc)), Lc.nsegs);
  k_tau<T><<<grid, kThreads, 0, st>>>(Lc, u, rhs, t, jr);
}

template <class T>
void launch_prolong(const Lvl& Lf, T* uf, const Lvl& Lc, const T* w, const T* t, int add,
                    cudaStream_t st) {
  dim3 grid(nblk(ecount(Lf)), Lf.nsegs);
  k_prolong<T><<<grid, kThreads, 0, st>>>(Lf, uf, Lc, w, t, add);
}

template <class T>
void launch_coarsest(const Lvl& L0, T* u, View<T> b, const T* ainv, cudaStream_t st) {
  const int n0 = L0.N[0] * L0.N[1] * L0.N[2];
  const int thr = n0 < 1024 ? ((n0 + 31) / 32) * 32 : 1024;
  k_coarsest<T><<<1, thr, n0 * sizeof(T), st>>>(L0, u, b, ainv);
}

template <class T>
void launch_pyramid(const T* ff, int nfx, int nfy, int nfz, T* fc, cudaStream_t st) {
  const long long n = (long long)(nfx / 2) * (nfy / 2) * (nfz / 2);
  const long long cap = 148LL * 16;
  const unsigned g = (unsigned)std::min<long long>(cap, (n + kThreads - 1) / kThreads);
  k_pyramid<T><<<g, kThreads, 0, st>>>(ff, nfx, nfy, nfz, fc);
}

template <class T>
void launch_gather(const Lvl& L, const T* useg, T* out, cudaStream_t st) {
  const long long n = (long long)L.N[0] * L.N[1] * L.N[2];
  const long long cap = 148LL * 16;
  const unsigned g = (unsigned)std::min<long long>(cap, (n + kThreads - 1) / kThreads);
  k_gather<T><<<g, kThreads, 0, st>>>(L, useg, out);
}

#define SRFMG_INST(T)                                                                          \
  template void launch_cheb_step<T>(const Lvl&, const T*, const T*, View<T>, T*, double, double, \
                                    int, cudaStream_t);                                        \
  template void launch_restrict<T>(const Lvl&, const T*, View<T>, const Lvl&, T*, T*, int,      \
                                   cudaStream_t);                                              \
  template void launch_tau<T>(const Lvl&, const T*, T*, T*, int, cudaStream_t);                 \
  template void launch_prolong<T>(const Lvl&, T*, const Lvl&, const T*, const T*, int,          \
                                  cudaStream_t);                                               \
  template void launch_coarsest<T>(const Lvl&, T*, View<T>, const T*, cudaStream_t);            \
  template void launch_pyramid<T>(const T*, int, int, int, T*, cudaStream_t);                   \
  template void launch_gather<T>(const Lvl&, const T*, T*, cudaStream_t);
SRFMG_INST(double)
SRFMG_INST(float)

}  // namespace srfmg
