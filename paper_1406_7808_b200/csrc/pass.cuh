// Fused multi-stage SR passes (pass.cu): one HBM pass per half V-cycle visit of an SR level.
//
//   source   LOAD  v0 = u                    (segment storage)
//            PSET  v0 = P(w)                 FMG interpolation Pi (fig:fmgsr L221)
//            PADD  v0 = u + P(w - t)         correction (fig:mgvsr L241)
//   steps    v_j = v_{j-1} + cm_j (v_{j-1} - v_{j-2}) + cr_j (b - A v_{j-1})  on C, j = 1..nstep
//            (Chebyshev R8: degree-1 step cm = 0, cr = 1/theta; degree-2 = (1/theta, 0) then
//            (rho1 rho0, 2 rho1/delta); momentum only on the last step when nstep >= 2)
//   sink     STORE     v_nstep -> segment storage (C updated, GSR carried through)
//            FINAL     genuine cells of v_nstep -> the user's dense u (R19)
//            RESTRICT  STORE + r = b - A v_nstep on C, u_{l-1}[F] = avg8(v), R[F] = avg8(r)
//                      (fig:mgvsr L232-235 / fig:mgv L112-115; F of half-width jr, or V_T)
#pragma once
#include "fused.cuh"

namespace srfmg {

enum { kSrcLoad = 0, kSrcPset = 1, kSrcPadd = 2 };
enum { kSinkStore = 0, kSinkFinal = 1, kSinkRestrict = 2 };

template <class T>
struct PassSpec {
  int src, nstep, sink;
  Lvl L;              // fine level (the level the pass runs on)
  Lvl Lc;             // coarse level l-1 (PSET/PADD source, RESTRICT target)
  const T* uin;       // LOAD/PADD: current fine u (complete: C and GSR)
  T* uout;            // STORE/RESTRICT: the other fine u buffer
  FusedRhs<T> rhs;    // b of the Chebyshev steps and the residual
  const T* w;         // PSET/PADD: coarse u
  const T* t;         // PADD: coarse t snapshot
  T* uc;              // RESTRICT: coarse u (written on F)
  T* rc;              // RESTRICT: coarse R (written on F)
  int jr;             // RESTRICT: F half-width on the coarse level (0: V_T)
  double cm[3], cr[3];
  FinalOut<T> fin;    // FINAL
};

// An instantiation exists for this (mode, level geometry, rhs kind).
template <class T>
bool pass_ok(int src, int nstep, int sink, const Lvl& L, const Lvl& Lc, int rhs_global);

// Enqueue the pass on `st` (returns false and launches nothing if !pass_ok).
template <class T>
bool launch_pass(const PassSpec<T>& ps, cudaStream_t st);

// dst[F^p] = src[F^p] on the coarse level for every segment p of the fine level L (the
// restriction target boxes of RESTRICT with half-width jr).  The FMG-entry pass
// (PSET, 3, RESTRICT) reads the coarse u for Pi while it restricts, so it restricts into
// the coarse t buffer and this copy moves the result into u before the tau step.
template <class T>
void launch_merge_f(const Lvl& L, const Lvl& Lc, const T* src, T* dst, int jr, cudaStream_t st);

}  // namespace srfmg
