// Coarse-level executor (coarse.cu): the operations of the conventional levels l <= T that
// are too small to fill the GPU (fig:mgv / fig:fmg on Omega_l with at most kCoarseMaxCells
// cells) are recorded as a list and run by ONE launch of a thread-block cluster that
// executes them in order, with a cluster barrier between consecutive operations.  This
// replaces ~190 latency-bound launches per C3 solve by a handful.
#pragma once
#include "kernels.cuh"

namespace srfmg {

enum { kCopCheb = 0, kCopRestrict, kCopTau, kCopProlong, kCopCoarsest, kCopPyramid };

constexpr int kCoarseMaxOps = 48;
constexpr int kCoarseMaxLevels = 16;
constexpr long long kCoarseMaxCells = 48LL * 48 * 48;  // conventional levels up to ~48^3

template <class T>
struct COp {
  int code;
  int lf, lc;      // level indices into COpList::L (fine, coarse)
  int flag;        // PROLONG: add
  int tiny;        // level small enough for one CTA (set by the recorder)
  const T* a;      // CHEB cur | RESTRICT u_f | TAU u | PROLONG w | COARSEST A0^-1 | PYRAMID f_f
  const T* b;      // CHEB prev (may alias c, or null) | PROLONG t
  T* c;            // CHEB out | RESTRICT u_c | TAU rhs | PROLONG u_f | COARSEST u | PYRAMID f_c
  T* d;            // RESTRICT R_c | TAU t
  View<T> v;       // CHEB / RESTRICT / COARSEST: right-hand side
  double c0, c1;   // CHEB: c_mom, c_res
};

template <class T>
struct COpList {
  int n;
  unsigned long long* prof;  // optional: SM clock64 after every operation (debug)
  Lvl L[kCoarseMaxLevels];
  COp<T> op[kCoarseMaxOps];
};

// Conventional single-segment level small enough for the executor.
bool coarse_level_ok(const Lvl& L);
// ... and small enough for one CTA of it (no cluster barrier needed around its operations)
bool coarse_level_tiny(const Lvl& L);

template <class T>
void launch_coarse_exec(const COpList<T>& ops, cudaStream_t st);

}  // namespace srfmg
