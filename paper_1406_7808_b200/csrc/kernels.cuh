// Internal kernel interface of the SR-FMG library (not part of the C ABI).
//
// Every level l of the hierarchy is described by a `Lvl`: a grid of segments, each with a
// private storage box grow(V, J+1) (SURVEY §8(a) layouts).  Conventional
// levels (l <= T) are the special case of ONE segment with V = Omega_l and J = 0, whose
// storage box is Omega_l plus a one-cell ghost ring ("Omega_h^{+1}").
// Dimension order inside the library is (x, y, z) = (x1, x2, x3), x fastest.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace srfmg {

struct Lvl {
  int N[3];          // cells of Omega_l per dimension
  int S[3];          // genuine segment edge per dimension (N on conventional levels)
  int J;             // buffer width (0 on conventional levels)
  int ns[3];         // segments per dimension (of this rank's block)
  int so[3];         // global segment coordinates of this rank's first segment (0 on 1 GPU)
  int E[3];          // storage extent per dimension: S + 2J + 2
  int py;            // row pitch in elements
  long long pz;      // plane pitch in elements
  long long ss;      // segment stride in elements
  int nsegs;
  double inv_h2;     // 1 / h_l^2
  int st27;          // 1: the paper's 27-point operator; 0: 7-point (R1)
  double nlg;        // f4 (R29): A(u) = -L_h u + nlg u^3 (0: linear)
};

// Read-only right-hand-side view: either a dense global array over Omega_l without ghosts
// (user f or an f-pyramid level) or a level's segment storage (tau right-hand sides).
// Dense arrays may be a rank's haloed local block: `p` then points at the (virtual)
// global origin, so that p[g.z*sz + g.y*sy + g.x] is valid for the block's global cells.
template <class T>
struct View {
  const T* p;
  int global;        // 1: dense global array, index g.z*sz + g.y*sy + g.x
  long long sy, sz;  // strides (row, plane)
  long long ss;      // segment stride (segment storage only)
  // dense arrays only (host side, for TMA tensor maps): the real array
  const T* base;     // element 0
  int dims[3];       // array dims
  int off[3];        // global index of element 0
};

// Launchers (kernels.cu).  All asynchronous on `st`.
template <class T>
void launch_cheb_step(const Lvl& L, const T* cur, const T* prev, View<T> b, T* out, double c_mom,
                      double c_res, int copy_gsr, cudaStream_t st);
// scratch (optional, 27-point levels): a fine-level buffer the residual may be written to
// (the free Chebyshev ping-pong buffer); without it a per-cell kernel is used
// bc (optional, 7-point): the coarse f_{l-1} = avg8(bf) when bf is f_l (R6 pyramid); the
// restricted residual is then bc - avg8(A u) and the fine b is not read
template <class T>
void launch_restrict(const Lvl& Lf, const T* uf, View<T> bf, const Lvl& Lc, T* uc, T* rc, int jr,
                     cudaStream_t st, T* scratch = nullptr, View<T> bc = View<T>{});
// the same restriction on an SR level through bulk-copy-fed bands (restrict.cu): bc = the
// pyramid f_{l-1} (bf unused), or bc.p = null and bf the level's segment-storage rhs; false
// when no instantiation fits the level (nothing launched)
template <class T>
bool launch_restrict_seg(const Lvl& Lf, const T* uf, View<T> bf, const Lvl& Lc, T* uc, T* rc,
                         int jr, cudaStream_t st, View<T> bc);
template <class T>
void launch_tau(const Lvl& Lc, const T* u, T* rhs, T* t, int jr, cudaStream_t st);
// uc = avg8(uf), rc = avg8(rf) on the restriction targets (rf: precomputed fine residual)
template <class T>
void launch_restrict_from_resid(const Lvl& Lf, const T* uf, const T* rf, const Lvl& Lc, T* uc,
                                T* rc, int jr, cudaStream_t st, View<T> bc = View<T>{});
template <class T>
void launch_prolong(const Lvl& Lf, T* uf, const Lvl& Lc, const T* w, const T* t, int add,
                    cudaStream_t st);
template <class T>
void launch_coarsest(const Lvl& L0, T* u, View<T> b, const T* ainv, cudaStream_t st);
template <class T>
void launch_pyramid(const T* ff, int nfx, int nfy, int nfz, T* fc, cudaStream_t st);
// acc[0] += sum over Omega of (b - A u)^2 (single-segment level, fp64 accumulation)
template <class T>
void launch_resnorm(const Lvl& L, const T* u, View<T> b, double* acc, cudaStream_t st);
// out: this rank's dense output block; (bo, sy, sz): its global origin and strides
template <class T>
void launch_gather(const Lvl& L, const T* useg, T* out, const int bo[3], long long sy,
                   long long sz, cudaStream_t st);
// copy the box [lo, lo+n) of a strided array (element (x,y,z) at base[z*sz + y*sy + x]) to
// (to_buf = 1) or from (0) a contiguous buffer -- packing for the multi-GPU all-gathers
template <class T>
void launch_box_copy(T* base, long long sy, long long sz, const int lo[3], const int n[3], T* buf,
                     int to_buf, cudaStream_t st);

// f_{l-1} = avg8(f_l) over the coarse box [lo, lo + n) (global indices) of two globally
// indexed dense views (virtual origins): the pyramid of a rank's block below level T
template <class T>
void launch_pyramid_box(View<T> f, View<T> c, const int lo[3], const int n[3], cudaStream_t st);
// dst = a - b (or a when b == null) on the S^3 block cells of two storage layouts La, Ld
// (ghost widths La.J + 1, Ld.J + 1): the k = 1 footprint array of a decomposed level T
template <class T>
void launch_block_diff(const Lvl& La, const T* a, const T* b, const Lvl& Ld, T* dst,
                       cudaStream_t st);

extern const char* const kKernelNames[];
extern const int kNumKernelNames;

}  // namespace srfmg
