// Fused, TMA-fed multi-sweep kernels of the SR-FMG schedule (see fused.cu).
#pragma once
#include <cuda.h>

#include "kernels.cuh"

namespace srfmg {

// A right-hand side the fused kernels can stream with TMA: either a dense global array
// (tensor map built per launch from `p`) or a level's segment storage (1-D bulk copies).
template <class T>
struct FusedRhs {
  const T* p;     // segment storage (global == 0) or unused
  int global;     // 1: dense array (x fastest), 0: segment storage of the level
  const T* base;  // dense array: first element of the (possibly haloed, local) array
  int dims[3];    // dense array dims
  int off[3];     // global index of base[0] (tensor coordinate = global - off)
};

// Dense output of the last pass: the rank's block of u, global origin bo, strides sy, sz.
template <class T>
struct FinalOut {
  T* p;
  int bo[3];
  long long sy, sz;
};

// One degree-2 Chebyshev application (two sweeps, R8) on C of every segment of level L,
// in ONE pass over HBM: u_in (complete: C and GSR) -> u_out (C updated, GSR copied).
// c0 = 1/theta (first step), cm = rho1 rho0, cr = 2 rho1 / delta (second step).
// ufinal != nullptr: the last smoothing of the solve -- write only the genuine cells, to the
// user's dense u (R19), and not the segment storage (only for cheb2_final_ok levels).
template <class T>
void launch_cheb2_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, double c0, double cm,
                        double cr, cudaStream_t st, FinalOut<T> fin = FinalOut<T>{});
template <class T>
bool cheb2_final_ok(const Lvl& L);
// tau (Eq. 4: rhs = R + A u on F, A u on C \ F; t = u) fused in front of the degree-2 pass.
// R (restricted residual) is read from its own buffer: the pass writes rhs while the
// neighbouring bands still read their halo rows of R.  false: nothing launched.
template <class T>
bool launch_tau_cheb2_fused(const Lvl& L, const T* u_in, T* u_out, const T* R, T* rhs, T* t,
                            int jr, double c0, double cm, double cr, cudaStream_t st);

// One degree-1 Chebyshev step (single stencil stage) with the same TMA pipeline; returns
// false (nothing launched) when no geometry-specialised instantiation matches the level.
template <class T>
bool launch_cheb1_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, double c0,
                        cudaStream_t st);

// 3-D tensor map of a dense rhs array, box (bw, rows, 1), element type T (fused.cu).
template <class T>
bool encode_dense_tmap(CUtensorMap* map, const FusedRhs<T>& rb, int bw, int rows);

// TMA-fed Chebyshev pass for the 27-point operator (fused27.cu): nst = 1 (degree 1) or 2
// (both steps of degree 2) in one HBM pass; fin.p: last pass, genuine cells -> user u.
template <class T>
bool cheb27_fused_ok(const Lvl& L);
template <class T>
void launch_cheb27_fused(const Lvl& L, const T* u_in, T* u_out, FusedRhs<T> b, int nst,
                         double c0, double cm, double cr, cudaStream_t st, FinalOut<T> fin);

// tau (Eq. 4) fused in front of the degree-2 27-point pass (R in its own buffer; rhs and t
// written); false: no instantiation, nothing launched
template <class T>
bool launch_tau_cheb27_fused(const Lvl& L, const T* u_in, T* u_out, const T* R, T* rhs, T* t,
                             int jr, double c0, double cm, double cr, cudaStream_t st);
// r = b - A u (27-point) on the C cells of every segment into r (same layout as u)
// nof = 1: r = -A u (the rhs is not streamed; the restriction adds f_{l-1} from the pyramid)
template <class T>
void launch_resid27_fused(const Lvl& L, const T* u, T* r, FusedRhs<T> b, cudaStream_t st,
                          int nof = 0);

// A geometry-specialised instantiation exists for this level's row pitch.
template <class T>
bool cheb_spec_ok(const Lvl& L);

// Fused-kernel availability for a level (smem budget etc.); false -> use the step kernels.
template <class T>
bool cheb2_fused_ok(const Lvl& L);

// TMA-fed prolongation (prolong.cu): u_f = P(w) (add = 0) or u_f += P(w - t) (add = 1)
template <class T>
bool prolong_tma_ok(const Lvl& Lf, const Lvl& Lc);
// the TMA prolongation's band plan fits (row width, shared memory for the coarse rows)
template <class T>
bool prolong_tma_fits(const Lvl& Lf, const Lvl& Lc);
template <class T>
void launch_prolong_tma(const Lvl& Lf, T* uf, const Lvl& Lc, const T* w, const T* t, int add,
                        cudaStream_t st);

// FMG entry in one pass (pset.cu): u_out = Pi(w) on the storage of every segment of level L
// (R10), then one degree-1 Chebyshev step on C (R8, c0 = 1/theta); GSR keeps Pi(w).
// The rhs must be a dense global array.  false: no instantiation fits (nothing launched).
template <class T>
bool pset1_fused_ok(const Lvl& L, const Lvl& Lc, int rhs_global);
template <class T>
bool launch_pset1_fused(const Lvl& L, const Lvl& Lc, const T* w, T* uout, FusedRhs<T> b,
                        double c0, cudaStream_t st);

// Up half of an SR level visit in one pass (up.cu): u += P(w - t) on C ∪ GSR (R10, R17),
// then the degree-2 Chebyshev smoothing on C (R8); fin.p: the last pass of the solve, the
// genuine cells into the user's u.  Lc / w / t: the coarse level's layout and arrays.
template <class T>
bool up2_fused_ok(const Lvl& L, const Lvl& Lc);
template <class T>
bool launch_up2_fused(const Lvl& L, const Lvl& Lc, const T* u_in, T* u_out, const T* w,
                      const T* t, FusedRhs<T> b, double c0, double cm, double cr,
                      cudaStream_t st, FinalOut<T> fin);

}  // namespace srfmg
