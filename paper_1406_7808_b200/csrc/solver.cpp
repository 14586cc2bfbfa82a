// Host side of the SR-FMG library: validation, level plan, workspace, the solve schedule
// (fig:fmg / fig:fmgsr / fig:mgv / fig:mgvsr as one recursion over level descriptors),
// CUDA-graph capture, and the C ABI of include/sr_fmg.h.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "fused.cuh"
#include "kernels.cuh"
#include "coarse.cuh"
#include "sr_fmg.h"

using srfmg::Lvl;
using srfmg::View;

namespace {

thread_local std::string g_tls_err = "no error";

// indices into srfmg::kKernelNames (sr_fmg_kernel_name)
enum KernelClass { KC_CHEB = 0, KC_RESTRICT, KC_TAU, KC_PROLONG, KC_COARSEST, KC_PYRAMID,
                   KC_GATHER, KC_CHEB_FUSED, KC_PASS_ENTRY, KC_PASS_DOWN, KC_PASS_UP, KC_COARSE,
                   KC_COUNT };

struct LevelBufs {
  void* u[2] = {nullptr, nullptr};  // two solution buffers (Chebyshev ping-pong)
  int cur = 0;                      // which one holds the current iterate
  void* rhs = nullptr;              // tau right-hand side (levels < M)
  void* t = nullptr;                // t snapshot (levels < M)
  void* fpyr = nullptr;             // dense f_l over Omega_l (levels <= T, and < M on 1 GPU)
  void* floc = nullptr;             // multi-GPU: this rank's haloed block of f_l, T <= l < M
  void* rres = nullptr;             // SR levels T < l < M: restricted residual R when the tau
                                    // is fused into the next pass (read there, rhs written)
  void* dwt = nullptr;              // decomposed levels < T: w - t with exchanged ghosts
};

// collectives of the multi-GPU path: all-gather of equal per-rank blocks
// (agglomeration of a coarse level), and groups of point-to-point transfers (one phase of a
// halo exchange on a domain-decomposed level)
struct Xfer {
  int peer;      // rank
  int recv;      // 0: send buf to peer, 1: receive buf from peer
  void* buf;     // device
  size_t bytes;
};
struct Comm {
  virtual ~Comm() {}
  virtual sr_status_t allgather(sr_fmg* h, const void* send, void* recv, size_t bytes,
                                cudaStream_t st) = 0;
  virtual sr_status_t group(sr_fmg* h, const Xfer* xs, int n, cudaStream_t st) = 0;
};

struct ProfRec {
  cudaEvent_t a, b;
  double bytes;
};

struct CellCounts {
  long long compute = 0;   // sum_p |C^p|
  long long cg = 0;        // sum_p |storage ∩ Omega| (C ∪ GSR)
  long long storage = 0;   // sum_p |storage box|
};

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

}  // namespace

struct sr_fmg {
  sr_fmg_desc_t d{};
  int M = 0, K = 0, T = 0;
  int esize = 8;
  double h = 0;
  std::vector<Lvl> L;
  std::vector<LevelBufs> B;
  std::vector<CellCounts> cells;
  std::vector<double> theta, delta, sigma;
  void* ainv = nullptr;
  cudaStream_t stream = nullptr;   // user stream (solves are ordered on it)
  cudaStream_t cap = nullptr;      // private stream used for graph capture
  std::string err = "no error";
  sr_status_t sticky = SR_OK;
  // captured solves, keyed by the (f, u) device pointers (two: the host-buffer pipeline
  // alternates two staging slots)
  struct GraphEnt {
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;     // kept while profiled: the event nodes below live in it
    std::vector<cudaGraphNode_t> na, nb;  // event-record nodes of prof[i].a / prof[i].b
    const void* f = nullptr;
    void* u = nullptr;
    long long used = 0;
  };
  GraphEnt graphs[2];
  long long gclock = 0;
  // host-buffer pipeline (sr_fmg_solve_host_async): two device staging slots; H2D on one
  // copy stream, the solve on the handle's stream, D2H on another, chained with events, so
  // consecutive calls overlap the two PCIe directions with each other and with the solves
  void* host_f[2] = {nullptr, nullptr};
  void* host_u[2] = {nullptr, nullptr};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_solve[2] = {nullptr, nullptr},
              ev_d2h[2] = {nullptr, nullptr};
  long long hcalls = 0;
  long long launches = 0;
  bool sync_debug = false;
  bool trace = false;  // SR_FMG_TRACE=1: print every launch, operation and collective
  bool cexec_one = false;  // SR_FMG_CEXEC_ONE=1: one executor launch per operation (debug)
  bool fused = true;  // SR_FMG_FUSED=0 disables the fused TMA kernels
  bool force = false; // SR_FMG_FORCE_FUSED=1: use them even on levels too small to fill the GPU
  int fused_min_e = 0; // SR_FMG_FUSED_MIN_E: smallest storage extent given to the TMA kernels
  bool pset1 = true;  // Pi + S^1 in one TMA pass at the FMG entry (pset.cu); SR_FMG_PSET1=0 off
  bool restrict_pyr = true;  // restriction of f-visits via the pyramid; SR_FMG_RESTRICT_PYR=0 off
  bool restrict_seg = true;  // bulk-copy-fed restriction on SR levels (restrict.cu);
                             // SR_FMG_RESTRICT_SEG=0 off
  bool tau_fuse = true;      // tau inside the next pre-smoothing pass; SR_FMG_TAU_FUSE=0 off
  bool up_fuse = false;      // correction + post-smoothing in one pass (up.cu): measured
                             // slower than the two passes; SR_FMG_UP_FUSE=1 on
  // coarse-level executor (coarse.cu) for the small conventional levels; SR_FMG_CEXEC=0
  // disables it.  flush_fn: enqueue the recorded operations (called before every launch)
  bool cexec = true;
  void (*flush_fn)(void*) = nullptr;
  void* flush_ctx = nullptr;
  int prof_cls = -1, prof_level = -1;
  std::vector<ProfRec> prof;
  size_t prof_used = 0;
  // profiling ring (sr_fmg_profile_ring): graph solve i records its profiled launches into
  // event set i % ring_n, so K solves run back to back and are read after one sync
  int ring_n = 0;
  long long ring_pos = 0;
  std::vector<std::vector<ProfRec>> ring;
  long long workspace = 0;
  std::vector<long long> visits;
  // ---- partition (multi-GPU); world = 1: one block = the whole grid, halo 0
  int world = 1, rank = 0, coord[3] = {0, 0, 0};
  int nsr[3] = {0, 0, 0};                   // SR segments per rank per dimension
  int blk_lo[3] = {0, 0, 0}, blk_n[3] = {0, 0, 0};  // fine genuine block
  std::vector<int> H;                       // f halo per level (levels >= T)
  std::vector<std::array<int, 3>> flo, fdim;  // local f array: global origin, dims (levels >= T)
  int blkT_lo[3] = {0, 0, 0}, blkT_n[3] = {0, 0, 0};  // this rank's block of level T
  Comm* comm = nullptr;
  void* xsend = nullptr;                    // exchange buffers (device)
  void* xrecv = nullptr;
  size_t xbytes = 0;                        // bytes per rank of the largest exchange
  long long exch = 0;                       // exchanges in the current solve
  long long exch_per_solve = 0;
  // domain decomposition of the conventional levels: levels A < l <= T are
  // held as this rank's block (Omega_l block + one ghost ring, refreshed by a halo exchange
  // before every operator application); levels l <= A are gathered once and solved
  // redundantly on every rank (the paper's redundant coarse grid)
  int A = 0;
  bool idle = false;                        // levels <= A on rank 0 only (desc.coarse_idle)
  int dd_min = 0;                           // a level stays decomposed while every block
                                            // dimension has at least dd_min cells
  srfmg::Lvl LT2{};                         // level T block with the k = 1 footprint ghosts
  void* wT2 = nullptr;                      // w - t (or u) of level T on LT2 storage
  void* zT2 = nullptr;                      // zeros on LT2 storage (the correction's t)
  void* hsend = nullptr;                    // halo staging buffers (device)
  void* hrecv = nullptr;
  size_t hbytes = 0;
  std::vector<long long> comm_calls;        // collective calls per level, last solve
};

namespace {

sr_status_t fail(sr_fmg* h, sr_status_t st, const std::string& msg) {
  if (h) {
    h->err = msg;
    if (st == SR_ERR_CUDA || st == SR_ERR_NCCL) h->sticky = st;
  } else {
    g_tls_err = msg;
  }
  return st;
}

#define CU(h, call)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail((h), SR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------------------------
// validation (create-time, before any allocation)
// ------------------------------------------------------------------------------------
sr_status_t validate(const sr_fmg_desc_t* d, std::string& msg) {
  auto bad = [&](const char* m) { msg = m; return SR_ERR_INVALID_ARGUMENT; };
  if (d->M < 0 || d->M >= SR_FMG_MAX_LEVELS) return bad("M out of range");
  for (int i = 0; i < 3; ++i) {
    if (d->n[i] <= 0) return bad("n[d] must be positive");
    if (d->n[i] % (1LL << d->M)) return bad("n[d] must be divisible by 2^M");
    if (d->n[i] > (1LL << 30)) return bad("n[d] too large");
  }
  if (d->sr_levels < 0 || d->sr_levels > d->M) return bad("need 0 <= sr_levels <= M");
  if (d->sr_levels > 0) {
    if (d->seg <= 0) return bad("seg must be positive when sr_levels > 0");
    for (int i = 0; i < 3; ++i)
      if (d->n[i] % d->seg) return bad("n[d] must be divisible by seg");
    if (d->seg % (1 << d->sr_levels)) return bad("seg must be divisible by 2^sr_levels");
  }
  if (d->buffer < 0) return bad("buffer must be >= 0");
  if (d->sched_B == -2) {
    if (d->sched_A < 0) return bad("maximum buffer schedule (sched_B = -2) needs sched_A = J_1 >= 0");
  } else if ((d->sched_A < 0) != (d->sched_B < 0)) {
    return bad("sched_A/sched_B: both or neither");
  }
  if (d->dtype != SR_F64 && d->dtype != SR_F32) return bad("dtype must be SR_F64 or SR_F32");
  if (d->h < 0 || !std::isfinite(d->h)) return bad("h must be >= 0 and finite");
  if (d->alpha < 0 || d->nu1 < 0 || d->nu2 < 0) return bad("Chebyshev degrees must be >= 0");
  if (!(d->cheb_lo >= 0) || !(d->cheb_hi > d->cheb_lo) || !(d->cheb_hi > 0))
    return bad("need 0 <= cheb_lo < cheb_hi (cheb_lo = 0: the stencil's default)");
  if (d->stencil != 7 && d->stencil != 27) return bad("stencil must be 7 or 27");
  if (!(d->nl_gamma >= 0) || !std::isfinite(d->nl_gamma)) return bad("nl_gamma must be >= 0");
  if (d->dd_min < 0 || d->dd_min == 1) return bad("dd_min must be 0 (default) or >= 2");
  if (d->world < 1) return bad("world must be >= 1");
  for (int i = 0; i < 3; ++i)
    if (d->pgrid[i] < 1 || d->pgrid[i] > d->world) return bad("need 1 <= pgrid[d] <= world");
  if ((long long)d->pgrid[0] * d->pgrid[1] * d->pgrid[2] != d->world) return bad("world != prod(pgrid)");
  if (d->rank < 0 || d->rank >= d->world) return bad("rank out of range");
  if (d->coarse_idle != 0 && d->coarse_idle != 1) return bad("coarse_idle must be 0 or 1");
  if (d->world > 1) {
    for (int i = 0; i < 3; ++i) {
      if (d->sr_levels > 0 && (d->n[i] / d->seg) % d->pgrid[i])
        return bad("world > 1 needs pgrid dividing the segment grid");
      // sr_levels = 0 (conventional distributed FMG): the rank blocks tile the fine grid and
      // coarsen evenly onto level M-1 at least
      if (d->sr_levels == 0 && (d->n[i] % d->pgrid[i] || (d->n[i] / d->pgrid[i]) % 2))
        return bad("world > 1 with sr_levels = 0 needs pgrid dividing n into even blocks");
    }
  }
  // supported-config checks
  if (d->world > 1 && d->comm != 0 && d->comm != 1) {
    msg = "comm must be 0 (NCCL) or 1 (host store, tests)";
    return SR_ERR_UNSUPPORTED_CONFIG;
  }
  if (d->sr_levels > 0) {  // every launch puts a rank's segments in gridDim.y (<= 65535)
    long long ns = 1;
    for (int i = 0; i < 3; ++i) ns *= (d->n[i] / d->seg) / d->pgrid[i];
    if (ns > 65535) {
      msg = "more than 65535 segments per rank; use larger segments or more ranks";
      return SR_ERR_UNSUPPORTED_CONFIG;
    }
  }
  long long n0 = 1;
  for (int i = 0; i < 3; ++i) n0 *= d->n[i] >> d->M;
  if (n0 > 1024) {
    msg = "coarsest grid has more than 1024 cells (dense exact solve); increase M";
    return SR_ERR_UNSUPPORTED_CONFIG;
  }
  return SR_OK;
}

int buffer_of(const sr_fmg_desc_t* d, int k) {  // Eq. 5
  if (d->sched_B == -2) return d->sched_A << (k - 1);  // MBS: J_k = 2^(k-1) J_1
  if (d->sched_A < 0) return d->buffer;
  return 2 * ((d->sched_A + d->sched_B * (d->sr_levels - k)) / 2);
}

// ------------------------------------------------------------------------------------
// level plan
// ------------------------------------------------------------------------------------
void make_plan(sr_fmg* h) {
  const sr_fmg_desc_t* d = &h->d;
  h->M = d->M;
  h->K = d->sr_levels;
  h->T = d->M - d->sr_levels;
  h->esize = d->dtype == SR_F64 ? 8 : 4;
  h->h = d->h > 0 ? d->h : 1.0 / (double)d->n[0];
  const int pitch_mult = 32 / h->esize;  // rows start on 32-byte sectors
  h->L.assign(h->M + 1, Lvl{});
  h->cells.assign(h->M + 1, CellCounts{});
  h->theta.assign(h->M + 1, 0);
  h->delta.assign(h->M + 1, 0);
  h->sigma.assign(h->M + 1, 0);
  // partition: rank r owns a pgrid block of the SR segment grid
  h->world = d->world;
  h->rank = d->rank;
  h->coord[0] = d->rank % d->pgrid[0];
  h->coord[1] = (d->rank / d->pgrid[0]) % d->pgrid[1];
  h->coord[2] = d->rank / (d->pgrid[0] * d->pgrid[1]);
  for (int i = 0; i < 3; ++i) {
    if (h->K > 0) {
      h->nsr[i] = (int)(d->n[i] / d->seg) / d->pgrid[i];
      h->blk_n[i] = h->nsr[i] * d->seg;
    } else {  // conventional FMG: a pgrid block of the fine grid (world 1: the whole grid)
      h->nsr[i] = 0;
      h->blk_n[i] = (int)(d->n[i] / d->pgrid[i]);
    }
    h->blk_lo[i] = h->coord[i] * h->blk_n[i];
    h->blkT_n[i] = h->blk_n[i] >> h->K;
    h->blkT_lo[i] = h->blk_lo[i] >> h->K;
  }
  // f halos: SR level l reads f_l on C = V grown by J_l; a halo H_l >= J_l, halved per
  // coarsening (the pyramid is local), kept a multiple of 4 cells above level T
  h->H.assign(h->M + 1, 0);
  h->flo.assign(h->M + 1, {0, 0, 0});
  h->fdim.assign(h->M + 1, {0, 0, 0});
  // (sr_levels = 0: every level reads f_l on the rank's block only -- no halo)
  if (h->world > 1 && h->K > 0) {
    int h1 = 0;
    for (int l = h->T + 1; l <= h->M; ++l) {
      const int j = buffer_of(d, l - h->T);
      const int need = (j + (1 << (l - h->T - 1)) - 1) >> (l - h->T - 1);  // ceil(j/2^(l-T-1))
      h1 = std::max(h1, need);
    }
    h1 = (int)round_up(std::max(h1, 1), 4);
    for (int l = h->T; l <= h->M; ++l)
      h->H[l] = l == h->T ? h1 / 2 : h1 << (l - h->T - 1);
  }
  for (int l = h->T; l <= h->M; ++l)
    for (int i = 0; i < 3; ++i) {
      h->flo[l][i] = (h->blk_lo[i] >> (h->M - l)) - h->H[l];
      h->fdim[l][i] = (h->blk_n[i] >> (h->M - l)) + 2 * h->H[l];
    }
  // domain decomposition below the SR levels: level l <= T stays decomposed while every
  // dimension of the rank's block has at least dd_min cells (and the block coarsens evenly
  // onto level l-1); the first level that does not is gathered (A), and every level <= A is
  // solved redundantly
  h->dd_min = d->dd_min > 0 ? d->dd_min : 32;
  h->idle = h->world > 1 && d->coarse_idle == 1;
  h->A = h->T;
  if (h->world > 1) {
    while (h->A >= 1) {
      bool ok = true;
      for (int i = 0; i < 3; ++i)
        ok = ok && (h->blk_n[i] >> (h->M - h->A)) >= h->dd_min &&
             h->blk_n[i] % (1LL << (h->M - h->A + 1)) == 0;
      if (!ok) break;
      --h->A;
    }
  }
  for (int l = 0; l <= h->M; ++l) {
    Lvl& L = h->L[l];
    const bool sr = l > h->T;
    const bool ddl = h->world > 1 && l > h->A && l <= h->T;  // this rank's block of Omega_l
    for (int i = 0; i < 3; ++i) L.N[i] = (int)(d->n[i] >> (h->M - l));
    L.J = sr ? buffer_of(d, l - h->T) : 0;
    for (int i = 0; i < 3; ++i) {
      L.S[i] = sr ? (d->seg >> (h->M - l)) : ddl ? (h->blk_n[i] >> (h->M - l)) : L.N[i];
      L.ns[i] = sr ? h->nsr[i] : 1;
      L.so[i] = sr ? h->coord[i] * h->nsr[i] : ddl ? h->coord[i] : 0;
      L.E[i] = L.S[i] + 2 * L.J + 2;
    }
    L.nsegs = L.ns[0] * L.ns[1] * L.ns[2];
    L.py = (int)round_up(L.E[0], pitch_mult);
    L.pz = (long long)L.py * L.E[1];
    L.ss = round_up(L.pz * L.E[2], 32);
    const double hl = h->h * (double)(1LL << (h->M - l));
    L.inv_h2 = 1.0 / (hl * hl);
    L.st27 = d->stencil == 27 ? 1 : 0;
    L.nlg = d->nl_gamma;
    // R8: lambda_max(A_l) = 12/h_l^2 (7-point); R28: 4/h_l^2 (27-point, symbol supremum)
    const double lam = (L.st27 ? 4.0 : 12.0) / (hl * hl);
    const double lo = d->cheb_lo > 0 ? d->cheb_lo : (L.st27 ? 1.0 / 3.0 : 1.0 / 6.0);
    const double a = lo * lam, b = d->cheb_hi * lam;
    h->theta[l] = 0.5 * (b + a);
    h->delta[l] = 0.5 * (b - a);
    h->sigma[l] = h->theta[l] / h->delta[l];
    // cell counts (region arithmetic of PAPER.md:187-210 on boxes)
    CellCounts& c = h->cells[l];
    for (int s = 0; s < L.nsegs; ++s) {
      const int p[3] = {s % L.ns[0] + L.so[0], (s / L.ns[0]) % L.ns[1] + L.so[1],
                        s / (L.ns[0] * L.ns[1]) + L.so[2]};
      long long vc = 1, vcg = 1;
      for (int i = 0; i < 3; ++i) {
        const int lo = p[i] * L.S[i], hi = lo + L.S[i];
        vc *= std::min(hi + L.J, L.N[i]) - std::max(lo - L.J, 0);
        vcg *= std::min(hi + L.J + 1, L.N[i]) - std::max(lo - L.J - 1, 0);
      }
      c.compute += vc;
      c.cg += vcg;
      c.storage += (long long)L.E[0] * L.E[1] * L.E[2];
    }
  }
  h->visits.assign(h->M + 1, 0);
  for (int l = 0; l <= h->M; ++l) h->visits[l] = h->M - l + 1;
  h->comm_calls.assign(h->M + 1, 0);
  // a decomposed level T also keeps a copy of its block with the ghost width of the k = 1
  // footprint, grow(V_T^p, ceil(J/2) + 1) (R15): the interpolation and the correction of the
  // first SR level read up to that far into the neighbouring ranks' blocks
  h->LT2 = h->L[h->T];
  if (h->world > 1 && h->A < h->T && h->K > 0) {
    Lvl& L2 = h->LT2;
    L2.J = std::max(0, (h->L[h->T + 1].J + 1) / 2);  // ghost width J + 1 = ceil(J_{T+1}/2) + 1
    for (int i = 0; i < 3; ++i) L2.E[i] = L2.S[i] + 2 * L2.J + 2;
    L2.py = (int)round_up(L2.E[0], pitch_mult);
    L2.pz = (long long)L2.py * L2.E[1];
    L2.ss = round_up(L2.pz * L2.E[2], 32);
  }
}

// checks that need the plan: the conventional distributed FMG (sr_levels = 0, world > 1)
// decomposes the finest level itself, so its rank blocks must not fall under dd_min
bool plan_ok(const sr_fmg* h, std::string& msg) {
  if (h->world > 1 && h->K == 0 && h->A >= h->M) {
    msg = "world > 1 with sr_levels = 0: the finest rank block has fewer than dd_min cells in "
          "some dimension (lower dd_min or use fewer ranks)";
    return false;
  }
  return true;
}

// dense inverse of A_0 (7-point, reflected ghosts) by Gauss-Jordan in fp64 (R7)
std::vector<double> coarsest_inverse(const Lvl& L0) {
  const int nx = L0.N[0], ny = L0.N[1], nz = L0.N[2];
  const int n = nx * ny * nz;
  std::vector<double> A((size_t)n * n, 0.0), I((size_t)n * n, 0.0);
  auto id = [&](int x, int y, int z) { return (z * ny + y) * nx + x; };
  if (L0.st27) {  // 27-point (R28): reflected edge/corner ghosts (-1)^m u(mirror), per dim
    const int N[3] = {nx, ny, nz};
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
          const int i = id(x, y, z);
          A[(size_t)i * n + i] += (8.0 / 3.0) * L0.inv_h2;
          for (int oz = -1; oz <= 1; ++oz)
            for (int oy = -1; oy <= 1; ++oy)
              for (int ox = -1; ox <= 1; ++ox) {
                const int nzc = (ox != 0) + (oy != 0) + (oz != 0);
                if (nzc < 2) continue;
                const int c[3] = {x + ox, y + oy, z + oz};
                int q[3];
                double sg = 1.0;
                for (int dd = 0; dd < 3; ++dd) {
                  q[dd] = c[dd];
                  if (q[dd] < 0) { q[dd] = -1 - q[dd]; sg = -sg; }
                  if (q[dd] >= N[dd]) { q[dd] = 2 * N[dd] - 1 - q[dd]; sg = -sg; }
                }
                const double wgt = nzc == 2 ? 1.0 / 6.0 : 1.0 / 12.0;
                A[(size_t)i * n + id(q[0], q[1], q[2])] -= sg * wgt * L0.inv_h2;
              }
        }
  }
  for (int z = 0; z < nz && !L0.st27; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) {
        const int i = id(x, y, z);
        double diag = 6.0;
        const int c[3] = {x, y, z}, N[3] = {nx, ny, nz};
        for (int dd = 0; dd < 3; ++dd)
          for (int o = -1; o <= 1; o += 2) {
            int q[3] = {c[0], c[1], c[2]};
            q[dd] += o;
            if (q[dd] < 0 || q[dd] >= N[dd]) {
              diag += 1.0;  // ghost = -u_i
            } else {
              A[(size_t)i * n + id(q[0], q[1], q[2])] -= L0.inv_h2;
            }
          }
        A[(size_t)i * n + i] += diag * L0.inv_h2;
      }
  for (int i = 0; i < n; ++i) I[(size_t)i * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(A[(size_t)r * n + col]) > std::fabs(A[(size_t)piv * n + col])) piv = r;
    if (piv != col)
      for (int k = 0; k < n; ++k) {
        std::swap(A[(size_t)piv * n + k], A[(size_t)col * n + k]);
        std::swap(I[(size_t)piv * n + k], I[(size_t)col * n + k]);
      }
    const double inv = 1.0 / A[(size_t)col * n + col];
    for (int k = 0; k < n; ++k) {
      A[(size_t)col * n + k] *= inv;
      I[(size_t)col * n + k] *= inv;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double fct = A[(size_t)r * n + col];
      if (fct == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        A[(size_t)r * n + k] -= fct * A[(size_t)col * n + k];
        I[(size_t)r * n + k] -= fct * I[(size_t)col * n + k];
      }
    }
  }
  return I;
}

// ------------------------------------------------------------------------------------
// launch bookkeeping: count launches, optional CUDA-event profiling of one (class, level)
// ------------------------------------------------------------------------------------
struct Launch {
  sr_fmg* h;
  cudaStream_t st;
  ProfRec* rec = nullptr;
  Launch(sr_fmg* h_, cudaStream_t st_, int cls, int level, double bytes) : h(h_), st(st_) {
    if (h->flush_fn) h->flush_fn(h->flush_ctx);  // recorded coarse-level operations first
    h->launches++;
    if (h->trace)
      fprintf(stderr, "sr_fmg[rank %d]: launch %s level %d\n", h->rank, srfmg::kKernelNames[cls],
              level);
    if (cls == h->prof_cls && level == h->prof_level) {
      if (h->prof_used == h->prof.size()) {
        ProfRec r{};
        cudaEventCreate(&r.a);
        cudaEventCreate(&r.b);
        h->prof.push_back(r);
      }
      rec = &h->prof[h->prof_used++];
      rec->bytes = bytes;
      cudaEventRecordWithFlags(rec->a, st, cudaEventRecordExternal);
    }
  }
  ~Launch() {
    if (rec) cudaEventRecordWithFlags(rec->b, st, cudaEventRecordExternal);
    if (h->sync_debug) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) {
        fprintf(stderr, "sr_fmg: kernel failed: %s\n", cudaGetErrorString(e));
        h->sticky = SR_ERR_CUDA;
        h->err = std::string("kernel failed: ") + cudaGetErrorString(e);
      }
    }
  }
};

// ------------------------------------------------------------------------------------
// the schedule
// ------------------------------------------------------------------------------------
template <class T>
struct Schedule {
  sr_fmg* h;
  cudaStream_t st;
  const T* f;  // user fine rhs (device)
  double w;    // element size

  T* U(int l) { return (T*)h->B[l].u[h->B[l].cur]; }

  // f_l as a dense view: the user's (haloed) block at l = M, the rank's haloed local
  // pyramid block on SR levels (multi-GPU), the global f_l otherwise
  // sr_read: the view an SR level's restriction reads (f_{l} near its segments' F regions):
  // on multi-GPU the rank's haloed local f_T even when level T is gathered -- an idle rank
  // (desc.coarse_idle) never assembles the global f_T
  View<T> fview(int l, bool sr_read = false) {
    View<T> v{};
    v.global = 1;
    const bool local = l > h->T || (l == h->M) || (h->world > 1 && l > h->A) ||
                       (sr_read && h->world > 1 && l == h->T);
    if (local && (l == h->M || l >= h->T)) {
      v.base = (l == h->M) ? f : (const T*)(h->world > 1 ? h->B[l].floc : h->B[l].fpyr);
      for (int i = 0; i < 3; ++i) {
        v.dims[i] = h->fdim[l][i];
        v.off[i] = h->flo[l][i];
      }
    } else if (local) {  // decomposed level below T: the rank's block of f_l, no halo
      v.base = (const T*)h->B[l].fpyr;
      for (int i = 0; i < 3; ++i) {
        v.dims[i] = h->L[l].S[i];
        v.off[i] = h->blk_lo[i] >> (h->M - l);
      }
    } else {
      v.base = (const T*)h->B[l].fpyr;
      for (int i = 0; i < 3; ++i) {
        v.dims[i] = h->L[l].N[i];
        v.off[i] = 0;
      }
    }
    v.sy = v.dims[0];
    v.sz = (long long)v.dims[0] * v.dims[1];
    v.p = v.base - (v.off[0] + v.off[1] * v.sy + v.off[2] * v.sz);  // virtual global origin
    v.ss = 0;
    return v;
  }
  static srfmg::FusedRhs<T> frhs(const View<T>& v) {
    srfmg::FusedRhs<T> r{};
    r.p = v.p;
    r.global = v.global;
    r.base = v.base;
    for (int i = 0; i < 3; ++i) {
      r.dims[i] = v.dims[i];
      r.off[i] = v.off[i];
    }
    return r;
  }
  static bool tma_rhs_ok(const View<T>& v) {  // tensor-map strides must be 16-byte multiples
    return !v.global || ((long long)v.dims[0] * sizeof(T)) % 16 == 0;
  }
  View<T> sview(int l) {
    const Lvl& L = h->L[l];
    View<T> v{};
    v.p = (const T*)h->B[l].rhs;
    v.global = 0;
    v.sy = L.py;
    v.sz = L.pz;
    v.ss = L.ss;
    return v;
  }

  // ---- coarse-level executor: operations on small conventional levels are recorded and
  // enqueued as one cluster launch right before the next ordinary launch (Launch ctor)
  srfmg::COpList<T> cops{};
  bool flushing = false;
  int cops_top = 0;
  double cops_bytes = 0;
  bool cx(int l) const {
    return h->cexec && !h->L[l].st27 && srfmg::coarse_level_ok(h->L[l]);
  }
  void emit(const srfmg::COp<T>& o, double bytes) {
    if (cops.n == srfmg::kCoarseMaxOps) flush();
    if (cops.n == 0) {
      for (int i = 0; i <= std::min(h->M, srfmg::kCoarseMaxLevels - 1); ++i) cops.L[i] = h->L[i];
      cops_top = 0;
      cops_bytes = 0;
    }
    cops.op[cops.n] = o;
    // tiny: every level the operation touches fits one CTA
    cops.op[cops.n].tiny = srfmg::coarse_level_tiny(h->L[o.lf]) && srfmg::coarse_level_tiny(h->L[o.lc]);
    cops.n++;
    cops_top = std::max(cops_top, o.lf);
    cops_bytes += bytes;
    if (h->trace)
      fprintf(stderr, "sr_fmg[rank %d]:   op %d code %d lf %d lc %d tiny %d\n", h->rank,
              cops.n - 1, o.code, o.lf, o.lc, cops.op[cops.n - 1].tiny);
    if (h->cexec_one) flush();  // debugging: one launch per operation
  }
  void flush() {
    if (cops.n == 0 || flushing) return;
    flushing = true;
    {
      Launch g(h, st, KC_COARSE, cops_top, cops_bytes);
      static const char* pe = std::getenv("SR_FMG_CEXEC_PROF");
      cops.prof = nullptr;
      if (pe && pe[0] == '1') {  // debug: per-operation timestamps, printed after the launch
        static unsigned long long* buf = nullptr;
        // mapped pinned host memory: a managed buffer page-faults on the first write of every
        // launch and inflates the first operation by ~35 us
        if (!buf)
          cudaHostAlloc((void**)&buf, sizeof(unsigned long long) * (srfmg::kCoarseMaxOps + 1),
                        cudaHostAllocMapped);
        cops.prof = buf;
        srfmg::launch_coarse_exec<T>(cops, st);
        cudaStreamSynchronize(st);
        for (int i = 0; i < cops.n; ++i) {
          const srfmg::COp<T>& o = cops.op[i];
          fprintf(stderr, "cexec op %2d code %d lf %d lc %d tiny %d  %8llu cycles\n", i, o.code,
                  o.lf, o.lc, o.tiny, buf[i + 1] - buf[i]);
        }
      } else {
        srfmg::launch_coarse_exec<T>(cops, st);
      }
    }
    cops.n = 0;
    flushing = false;
  }
  static void flush_cb(void* p) { static_cast<Schedule*>(p)->flush(); }
  void bind() {
    h->flush_fn = &Schedule::flush_cb;
    h->flush_ctx = this;
  }
  void unbind() {
    flush();
    h->flush_fn = nullptr;
    h->flush_ctx = nullptr;
  }
  static srfmg::COp<T> cop(int code, int lf, int lc) {
    srfmg::COp<T> o{};
    o.code = code;
    o.lf = lf;
    o.lc = lc;
    return o;
  }

  // The fused kernels march z inside a CTA: they are used when segments x bands of `rows`
  // fill the GPU; tiny levels are latency-bound and run faster as z-chunked step kernels.
  // The count is over the GLOBAL segment grid, so every world size picks the same kernels
  // and the result does not depend on the partition (R25, bitwise).
  bool fills(const Lvl& L, int rows) const {
    long long g = 1;
    for (int i = 0; i < 3; ++i) g *= L.N[i] / L.S[i];
    return h->force || g * ((L.E[1] + rows - 1) / rows) >= 148;
  }

  // S^deg(L_l, u_l, b) on C_l of every segment (R8): ping-pong between the two buffers
  T* final_out = nullptr;  // user u: the last level-M smoothing writes it directly (R19)
  bool pyr = false;        // the f pyramid f_l (R6) of this solve is built
  int pend_tau = -1;       // level whose tau is deferred into its first Chebyshev pass
  int pend_jr = 0;
  bool final_done = false;

  void cheb(int l, int deg, View<T> b, bool last = false) {
    if (pend_tau == l && deg != 2) {  // (safety net: tau_fuse_ok asked for nu1 = 2)
      pend_tau = -1;
      tau_from_rres(l, pend_jr);
    }
    if (deg <= 0) return;
    const Lvl& L = h->L[l];
    LevelBufs& bb = h->B[l];
    const CellCounts& c = h->cells[l];
    // the fused pass marches z inside a CTA: use it only when segments x bands fill the
    // GPU; tiny levels are latency-bound and run faster as z-chunked step kernels
    if (deg == 2 && l > h->T && h->fused && !L.st27 && L.nlg == 0.0 &&
        (fills(L, 40) && (h->force || L.E[1] >= h->fused_min_e)) &&
        tma_rhs_ok(b) && srfmg::cheb2_fused_ok<T>(L)) {
      // both sweeps in one HBM pass: read u, b; write u (C) and copy GSR
      const double rho0 = 1.0 / h->sigma[l];
      const double rho1 = 1.0 / (2.0 * h->sigma[l] - rho0);
      const bool fin = last && final_out != nullptr && srfmg::cheb2_final_ok<T>(L);
      const double nv = (double)L.N[0] * L.N[1] * L.N[2];
      if (pend_tau == l && !fin) {  // tau (Eq. 4) fused in front of the pre-smoothing pass
        pend_tau = -1;
        bool done;
        {
          Launch g(h, st, KC_CHEB_FUSED, l,
                   w * (3.0 * c.compute + 2.0 * (c.cg - c.compute) + c.compute + c.storage));
          done = srfmg::launch_tau_cheb2_fused<T>(
              L, (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur], (const T*)bb.rres, (T*)bb.rhs,
              (T*)bb.t, pend_jr, 1.0 / h->theta[l], rho1 * rho0, 2.0 * rho1 / h->delta[l], st);
        }
        if (done) {
          bb.cur = 1 - bb.cur;
          return;
        }
        tau_from_rres(l, pend_jr);  // no instantiation: the separate kernel, then the pass
      }
      Launch g(h, st, KC_CHEB_FUSED, l,
               fin ? w * (2.0 * c.compute + nv)
                   : w * (3.0 * c.compute + 2.0 * (c.cg - c.compute)));
      srfmg::FinalOut<T> fo{};
      if (fin) {
        fo.p = final_out;
        for (int i = 0; i < 3; ++i) fo.bo[i] = h->blk_lo[i];
        fo.sy = h->blk_n[0];
        fo.sz = (long long)h->blk_n[0] * h->blk_n[1];
      }
      srfmg::launch_cheb2_fused<T>(L, (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur], frhs(b),
                                   1.0 / h->theta[l], rho1 * rho0, 2.0 * rho1 / h->delta[l], st,
                                   fo);
      bb.cur = 1 - bb.cur;
      if (fin) final_done = true;
      return;
    }
    if (deg == 1 && l > h->T && h->fused && !L.st27 && L.nlg == 0.0 &&
        (fills(L, 40) && (h->force || L.E[1] >= h->fused_min_e)) &&
        tma_rhs_ok(b) && srfmg::cheb_spec_ok<T>(L)) {
      Launch g(h, st, KC_CHEB_FUSED, l, w * (3.0 * c.compute + 2.0 * (c.cg - c.compute)));
      srfmg::launch_cheb1_fused<T>(L, (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur], frhs(b),
                                   1.0 / h->theta[l], st);
      bb.cur = 1 - bb.cur;
      return;
    }
    if ((deg == 1 || deg == 2) && l > h->T && h->fused && L.st27 && L.nlg == 0.0 && tma_rhs_ok(b) &&
        fills(L, 10) &&
        srfmg::cheb27_fused_ok<T>(L)) {
      // 27-point operator: the whole polynomial in one TMA-fed pass (fused27.cu)
      const double rho0 = 1.0 / h->sigma[l];
      const double rho1 = 1.0 / (2.0 * h->sigma[l] - rho0);
      const bool fin = last && final_out != nullptr;
      srfmg::FinalOut<T> fo{};
      if (fin) {
        fo.p = final_out;
        for (int i = 0; i < 3; ++i) fo.bo[i] = h->blk_lo[i];
        fo.sy = h->blk_n[0];
        fo.sz = (long long)h->blk_n[0] * h->blk_n[1];
      }
      if (pend_tau == l && deg == 2 && !fin) {  // tau (Eq. 4) in front of the pass
        pend_tau = -1;
        bool done;
        {
          Launch g(h, st, KC_CHEB_FUSED, l,
                   w * (3.0 * c.compute + 2.0 * (c.cg - c.compute) + c.compute + c.storage));
          done = srfmg::launch_tau_cheb27_fused<T>(
              L, (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur], (const T*)bb.rres, (T*)bb.rhs,
              (T*)bb.t, pend_jr, 1.0 / h->theta[l], rho1 * rho0, 2.0 * rho1 / h->delta[l], st);
        }
        if (done) {
          bb.cur = 1 - bb.cur;
          return;
        }
        tau_from_rres(l, pend_jr);
      }
      Launch g(h, st, KC_CHEB_FUSED, l, w * (3.0 * c.compute + 2.0 * (c.cg - c.compute)));
      srfmg::launch_cheb27_fused<T>(L, (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur], frhs(b), deg,
                                    1.0 / h->theta[l], rho1 * rho0, 2.0 * rho1 / h->delta[l], st,
                                    fo);
      bb.cur = 1 - bb.cur;
      if (fin) final_done = true;
      return;
    }
    if (pend_tau == l) {  // (safety net: the fused pass did not apply)
      pend_tau = -1;
      tau_from_rres(l, pend_jr);
    }
    int lat = bb.cur, oth = 1 - bb.cur;
    if (cx(l)) {  // recorded for the coarse-level executor (same steps, same ping-pong)
      double rho_prev = 1.0 / h->sigma[l];
      for (int k = 0; k < deg; ++k) {
        if (dd(l)) halo(l, L, (T*)bb.u[lat]);  // every step reads the neighbours' cells
        srfmg::COp<T> o = cop(srfmg::kCopCheb, l, l);
        o.a = (const T*)bb.u[lat];
        o.b = k == 0 ? nullptr : (const T*)bb.u[oth];
        o.c = (T*)bb.u[oth];
        o.v = b;
        if (k == 0) {
          o.c0 = 0.0;
          o.c1 = 1.0 / h->theta[l];
        } else {
          const double rho = 1.0 / (2.0 * h->sigma[l] - rho_prev);
          o.c0 = rho * rho_prev;
          o.c1 = 2.0 * rho / h->delta[l];
          rho_prev = rho;
        }
        emit(o, w * (k == 0 ? 3.0 : 4.0) * c.compute);
        std::swap(lat, oth);
      }
      bb.cur = lat;
      return;
    }
    if (dd(l)) halo(l, L, (T*)bb.u[lat]);
    {
      Launch g(h, st, KC_CHEB, l, w * (3.0 * c.compute + 2.0 * (c.cg - c.compute)));
      srfmg::launch_cheb_step<T>(L, (const T*)bb.u[lat], nullptr, b, (T*)bb.u[oth], 0.0,
                                 1.0 / h->theta[l], 1, st);
    }
    std::swap(lat, oth);
    double rho_prev = 1.0 / h->sigma[l];
    for (int k = 1; k < deg; ++k) {
      const double rho = 1.0 / (2.0 * h->sigma[l] - rho_prev);
      if (dd(l)) halo(l, L, (T*)bb.u[lat]);
      {
        Launch g(h, st, KC_CHEB, l, w * 4.0 * c.compute);
        srfmg::launch_cheb_step<T>(L, (const T*)bb.u[lat], (const T*)bb.u[oth], b,
                                   (T*)bb.u[oth], rho * rho_prev, 2.0 * rho / h->delta[l], 0,
                                   st);
      }
      std::swap(lat, oth);
      rho_prev = rho;
    }
    bb.cur = lat;
  }

  int jr_for(int l) {  // restriction / F half-width for fine level l -> coarse l-1
    return (l - 1 > h->T) ? h->L[l].J / 2 : 0;
  }

  void coarsest(View<T> b) {
    if (cx(0)) {
      srfmg::COp<T> o = cop(srfmg::kCopCoarsest, 0, 0);
      o.a = (const T*)h->ainv;
      o.c = U(0);
      o.v = b;
      emit(o, 0.0);
      return;
    }
    Launch g(h, st, KC_COARSEST, 0, 0.0);
    srfmg::launch_coarsest<T>(h->L[0], U(0), b, (const T*)h->ainv, st);
  }

  void prolong(int l, int add) {
    const CellCounts& c = h->cells[l];
    // a decomposed coarse level: the interpolation reads one ghost layer of the source (the
    // neighbours' cells).  The correction's source is w - t, formed on the block and then
    // exchanged (t is snapshotted on the block only); P(d - 0) == P(w - t) cell for cell
    const bool dwt = dd(l - 1) && add && l - 1 < h->T;
    if (dd(l - 1)) {
      if (l - 1 == h->T) {
        footprint_T(add != 0);  // k = 1: w - t (or u) with the footprint ghosts
      } else if (dwt) {
        const Lvl& Lc = h->L[l - 1];
        {
          Launch g(h, st, KC_PROLONG, l - 1, 0.0);
          srfmg::launch_block_diff<T>(Lc, U(l - 1), (const T*)h->B[l - 1].t, Lc,
                                      (T*)h->B[l - 1].dwt, st);
        }
        halo(l - 1, Lc, (T*)h->B[l - 1].dwt);
      } else {
        halo_u(l - 1);  // Pi reads u
      }
    }
    const T* wsrc = dwt ? (const T*)h->B[l - 1].dwt : U(l - 1);
    const T* tsrc = dwt ? (const T*)h->zT2 : (const T*)h->B[l - 1].t;
    // the k = 1 source of a decomposed level T: the footprint copy, P(d - 0) == P(w - t)
    const bool fp = dd(l - 1) && l - 1 == h->T;
    if (cx(l) && cx(l - 1)) {
      srfmg::COp<T> o = cop(srfmg::kCopProlong, l, l - 1);
      o.flag = add;
      o.a = wsrc;
      o.b = tsrc;
      o.c = U(l);
      if (fp) {  // (an SR level is never an executor level; kept for completeness)
        h->sticky = SR_ERR_UNSUPPORTED_CONFIG;
        h->err = "executor interpolation from the footprint copy";
      }
      emit(o, w * (add ? 2.0 : 1.0) * c.cg);
      return;
    }
    const Lvl& Lc = fp ? h->LT2 : h->L[l - 1];
    const T* wc = fp ? (const T*)h->wT2 : wsrc;
    const T* tc = fp ? (const T*)h->zT2 : tsrc;
    Launch g(h, st, KC_PROLONG, l,
             w * (add ? 2.0 : 1.0) * c.cg + w * (add ? 2.0 : 1.0) * h->cells[l - 1].cg / 8.0);
    // (decided on the single-GPU shape of the coarse level, R25; the rank's block must fit too)
    const Lvl Lg = glob(l - 1);
    if (h->fused && srfmg::prolong_tma_fits<T>(h->L[l], Lg) && srfmg::prolong_tma_fits<T>(h->L[l], Lc) &&
        (h->force || (srfmg::prolong_tma_ok<T>(h->L[l], Lg) && h->L[l].E[1] >= h->fused_min_e)))
      srfmg::launch_prolong_tma<T>(h->L[l], U(l), Lc, wc, tc, add, st);
    else
      srfmg::launch_prolong<T>(h->L[l], U(l), Lc, wc, tc, add, st);
  }

  // FMG entry Pi + S^1 (alpha = 1) in one TMA pass (pset.cu), on the levels the fused
  // Chebyshev pass takes (enough segments x bands to fill the GPU).  The choice uses the
  // single-GPU shape of the coarse level, so every partition makes the same one.
  bool pset1_on(int l, const View<T>& b) {
    const Lvl& L = h->L[l];
    return h->pset1 && h->fused && h->d.alpha == 1 && l > h->T && !cx(l) && !L.st27 &&
           L.nlg == 0.0 && b.global && tma_rhs_ok(b) &&
           (fills(L, 40) && (h->force || L.E[1] >= h->fused_min_e)) &&
           srfmg::pset1_fused_ok<T>(L, glob(l - 1), 1);
  }
  void pset1(int l, const View<T>& b) {
    const Lvl& L = h->L[l];
    const CellCounts& c = h->cells[l];
    const bool fp = dd(l - 1) && l - 1 == h->T;
    if (fp) footprint_T(false);
    // algorithmic words: u written (storage), rhs read (C), coarse u read (1/8 of storage)
    Launch g(h, st, KC_PASS_ENTRY, l, w * (c.cg + c.compute + h->cells[l - 1].cg / 8.0));
    LevelBufs& bb = h->B[l];
    const bool ok = srfmg::launch_pset1_fused<T>(L, fp ? h->LT2 : h->L[l - 1],
                                                 fp ? (const T*)h->wT2 : U(l - 1),
                                                 (T*)bb.u[bb.cur], frhs(b), 1.0 / h->theta[l], st);
    if (!ok) {  // (pset1_on checked the single-GPU fit; a block never needs more)
      h->sticky = SR_ERR_UNSUPPORTED_CONFIG;
      h->err = "fused FMG entry: no instantiation for this rank's level-T block";
    }
  }

  // ---- multi-GPU.  Levels A < l <= T are decomposed: the rank holds its
  // block of Omega_l with a ghost ring that a halo exchange refreshes before every operator
  // application.  Level A is agglomerated: its blocks are all-gathered into a global array on
  // every rank, and the levels <= A are solved redundantly.
  bool dd(int l) const { return h->world > 1 && l > h->A && l <= h->T; }
  int rank_of(const int c[3]) const {
    return c[0] + h->d.pgrid[0] * (c[1] + h->d.pgrid[1] * c[2]);
  }
  // halo exchange of a decomposed level's array `base` (storage layout L, ghost width
  // g = L.J + 1): three phases x, y, z; phase d sends the g boundary planes of the block to
  // the two neighbours in d and receives their planes into the ghost ring.  A phase covers
  // the ghost cells of the dimensions already exchanged, so edges and corners arrive too
  // (the trilinear interpolation reads them).  One NCCL group per phase.
  void halo(int lvl, const Lvl& L, T* base) {
    flush();
    if (h->trace) fprintf(stderr, "sr_fmg[rank %d]: halo level %d (width %d)\n", h->rank, lvl, L.J + 1);
    const int g = L.J + 1;
    T* snd = (T*)h->hsend;
    T* rcv = (T*)h->hrecv;
    for (int d = 0; d < 3; ++d) {
      const bool lo_nb = h->coord[d] > 0, hi_nb = h->coord[d] < h->d.pgrid[d] - 1;
      if (!lo_nb && !hi_nb) continue;
      int lo[3], n[3];
      for (int e = 0; e < 3; ++e) {
        lo[e] = e < d ? 0 : g;
        n[e] = e < d ? L.E[e] : L.S[e];
      }
      n[d] = g;
      const long long cnt = (long long)n[0] * n[1] * n[2];
      const size_t bytes = (size_t)cnt * sizeof(T);
      Xfer xs[4];
      int nx = 0;
      int c[3] = {h->coord[0], h->coord[1], h->coord[2]};
      if (lo_nb) {
        lo[d] = g;
        srfmg::launch_box_copy<T>(base, L.py, L.pz, lo, n, snd, 1, st);
        c[d] = h->coord[d] - 1;
        xs[nx++] = Xfer{rank_of(c), 0, snd, bytes};
        xs[nx++] = Xfer{rank_of(c), 1, rcv, bytes};
      }
      if (hi_nb) {
        lo[d] = L.S[d];
        srfmg::launch_box_copy<T>(base, L.py, L.pz, lo, n, snd + cnt, 1, st);
        c[d] = h->coord[d] + 1;
        xs[nx++] = Xfer{rank_of(c), 0, snd + cnt, bytes};
        xs[nx++] = Xfer{rank_of(c), 1, rcv + cnt, bytes};
      }
      const sr_status_t r = h->comm->group(h, xs, nx, st);
      if (r != SR_OK) h->sticky = r;
      h->comm_calls[lvl]++;
      h->exch++;
      if (lo_nb) {
        lo[d] = 0;
        srfmg::launch_box_copy<T>(base, L.py, L.pz, lo, n, rcv, 0, st);
      }
      if (hi_nb) {
        lo[d] = g + L.S[d];
        srfmg::launch_box_copy<T>(base, L.py, L.pz, lo, n, rcv + cnt, 0, st);
      }
      h->launches += 2 * ((lo_nb ? 1 : 0) + (hi_nb ? 1 : 0));
    }
  }
  void halo_u(int l) { halo(l, h->L[l], U(l)); }

  // all-gather of the rank blocks of level lvl: field k of this rank's block is read at
  // slo[k] (local coordinates) of (sbase, ssy, ssz) and every rank's block is written at its
  // global origin into the global array (dbase, dsy, dsz)
  void gather(int lvl, int nf, T* const* sbase, const long long* ssy, const long long* ssz,
              const int (*slo)[3], T* const* dbase, const long long* dsy, const long long* dsz) {
    flush();
    if (h->trace) fprintf(stderr, "sr_fmg[rank %d]: all-gather level %d\n", h->rank, lvl);
    int nb3[3];
    for (int i = 0; i < 3; ++i) nb3[i] = h->blk_n[i] >> (h->M - lvl);
    const long long nb = (long long)nb3[0] * nb3[1] * nb3[2];
    T* snd = (T*)h->xsend;
    T* rcv = (T*)h->xrecv;
    for (int k = 0; k < nf; ++k)
      srfmg::launch_box_copy<T>(sbase[k], ssy[k], ssz[k], slo[k], nb3, snd + k * nb, 1, st);
    const size_t bytes = (size_t)nf * nb * sizeof(T);
    sr_status_t r = SR_OK;
    if (!h->idle) {
      r = h->comm->allgather(h, snd, rcv, bytes, st);
    } else {
      // idle coarse grid: the blocks go to rank 0 alone, one NCCL group
      std::vector<Xfer> xs;
      if (h->rank == 0) {
        for (int q = 1; q < h->world; ++q) xs.push_back(Xfer{q, 1, rcv + q * nf * nb, bytes});
      } else {
        xs.push_back(Xfer{0, 0, snd, bytes});
      }
      r = h->comm->group(h, xs.data(), (int)xs.size(), st);
    }
    if (r != SR_OK) h->sticky = r;
    h->comm_calls[lvl]++;
    h->exch++;
    h->launches += nf;
    if (h->idle && h->rank != 0) return;  // only rank 0 assembles level A
    for (int q = 0; q < h->world; ++q) {
      const int c[3] = {q % h->d.pgrid[0], (q / h->d.pgrid[0]) % h->d.pgrid[1],
                        q / (h->d.pgrid[0] * h->d.pgrid[1])};
      int lo[3];
      for (int i = 0; i < 3; ++i) lo[i] = c[i] * nb3[i];
      if (q == h->rank && sbase[0] == dbase[0]) continue;  // already in place
      // (the rank's own block from its send buffer: a gather to rank 0 receives no copy)
      T* from = q == h->rank ? snd : rcv + q * nf * nb;
      for (int k = 0; k < nf; ++k)
        srfmg::launch_box_copy<T>(dbase[k], dsy[k], dsz[k], lo, nb3, from + k * nb, 0, st);
      h->launches += nf;
    }
  }
  // idle coarse grid: rank 0 alone runs the levels <= A (redundant: every rank)
  bool solves_A() const { return !h->idle || h->rank == 0; }
  // idle coarse grid: rank 0 sends its level-A solution u_A (and the tau snapshot t_A for a
  // correction) to every other rank, whole storage arrays, one NCCL group
  void bcast_A(bool with_t) {
    flush();
    const int a = h->A;
    const Lvl& LA = h->L[a];
    const size_t bytes = (size_t)LA.ss * LA.nsegs * sizeof(T);
    std::vector<Xfer> xs;
    for (int q = 1; q < h->world; ++q) {
      if (h->rank != 0 && q != h->rank) continue;
      const int peer = h->rank == 0 ? q : 0, rcv = h->rank == 0 ? 0 : 1;
      xs.push_back(Xfer{peer, rcv, U(a), bytes});
      if (with_t) xs.push_back(Xfer{peer, rcv, h->B[a].t, bytes});
    }
    if (h->trace) fprintf(stderr, "sr_fmg[rank %d]: broadcast level %d\n", h->rank, a);
    const sr_status_t r = h->comm->group(h, xs.data(), (int)xs.size(), st);
    if (r != SR_OK) h->sticky = r;
    h->comm_calls[a]++;
    h->exch++;
  }
  // u_A and R_A: the blocks written by this rank's restriction into the global level-A
  // arrays (k = 1 restriction when A = T, else the restriction from the decomposed A + 1)
  void gather_uR() {
    const int a = h->A;
    const Lvl& LA = h->L[a];
    T* base[2] = {U(a) + LA.pz + LA.py + 1, (T*)h->B[a].rhs + LA.pz + LA.py + 1};
    const long long sy[2] = {LA.py, LA.py}, sz[2] = {LA.pz, LA.pz};
    int lo[2][3];
    for (int i = 0; i < 3; ++i) lo[0][i] = lo[1][i] = h->blk_lo[i] >> (h->M - a);
    gather(a, 2, base, sy, sz, lo, base, sy, sz);
  }
  // f_A: this rank's block (the interior of the haloed local f_T when A = T, else the part of
  // the global f_A its block pyramid wrote), all-gathered into the global f_A
  void gather_f() {
    const int a = h->A;
    const Lvl& LA = h->L[a];
    T* dst[1] = {(T*)h->B[a].fpyr};
    const long long dsy[1] = {LA.N[0]}, dsz[1] = {(long long)LA.N[0] * LA.N[1]};
    if (a == h->T) {
      const int HT = h->H[h->T];
      const auto& d = h->fdim[h->T];
      T* src[1] = {(T*)h->B[h->T].floc};
      const long long ssy[1] = {d[0]}, ssz[1] = {(long long)d[0] * d[1]};
      const int lo[1][3] = {{HT, HT, HT}};
      gather(a, 1, src, ssy, ssz, lo, dst, dsy, dsz);
    } else {
      int lo[1][3];
      for (int i = 0; i < 3; ++i) lo[0][i] = h->blk_lo[i] >> (h->M - a);
      gather(a, 1, dst, dsy, dsz, lo, dst, dsy, dsz);
    }
  }
  // the k = 1 footprint of a decomposed level T (R15: grow(V_T^p, ceil(J/2) + 1)) on the
  // wider-ghosted copy LT2: w - t for the correction (t = the zero array), u for the
  // interpolation; the same values the single-GPU kernels read from the global level T
  void footprint_T(bool diff) {
    const int t = h->T;
    {
      Launch g(h, st, KC_PROLONG, t, 0.0);
      srfmg::launch_block_diff<T>(h->L[t], U(t), diff ? (const T*)h->B[t].t : nullptr, h->LT2,
                                  (T*)h->wT2, st);
    }
    halo(t, h->LT2, (T*)h->wT2);
  }
  // single-GPU shape of a conventional level: the kernel choices are made on it, so every
  // partition runs the same kernels (R25)
  Lvl glob(int l) const {
    Lvl L = h->L[l];
    if (l > h->T) return L;
    for (int i = 0; i < 3; ++i) {
      L.S[i] = L.N[i];
      L.so[i] = 0;
      L.E[i] = L.N[i] + 2;
    }
    const int pm = 32 / (int)sizeof(T);
    L.py = (L.E[0] + pm - 1) / pm * pm;
    L.pz = (long long)L.py * L.E[1];
    L.ss = (L.pz * L.E[2] + 31) / 32 * 32;
    return L;
  }

  void restrict_std(int l, View<T> b) {
    const int jr = jr_for(l);
    if (dd(l)) halo_u(l);  // the residual reads the neighbours' cells
    if (cx(l) && cx(l - 1)) {
      srfmg::COp<T> o = cop(srfmg::kCopRestrict, l, l - 1);
      o.a = U(l);
      o.c = U(l - 1);
      o.d = (T*)h->B[l - 1].rhs;
      o.v = b;
      emit(o, w * 2.25 * h->cells[l].compute);
      return;
    }
    const Lvl& Lf = h->L[l];
    double tgt = h->L[l].nsegs;
    for (int i = 0; i < 3; ++i) tgt *= (Lf.S[i] / 2 + 2 * jr);
    const Lvl& L = h->L[l];
    // b = f_l (an FMG visit, or the finest level): its average f_{l-1} is the R6 pyramid, so
    // the restricted residual is f_{l-1} - avg8(A u) and f_l need not be read (7-point)
    const bool use_pyr = pyr && b.global && !L.st27 && h->restrict_pyr;
    Launch g(h, st, KC_RESTRICT, l, w * (use_pyr ? 8.0 + 1.0 + 2.0 : 16.0 + 2.0) * tgt);
    // R goes to the level's rres buffer when its tau rides in the next pass (that pass
    // writes rhs while neighbouring bands still read R)
    T* rc = tau_fuse_ok(l - 1) ? (T*)h->B[l - 1].rres : (T*)h->B[l - 1].rhs;
    if (l > h->T && L.st27 && L.nlg == 0.0 && h->fused && tma_rhs_ok(b) &&
        srfmg::cheb27_fused_ok<T>(L) && fills(L, 10)) {
      // 27-point: TMA-fed residual pass into the free ping-pong buffer, then the averages
      T* scratch = (T*)h->B[l].u[1 - h->B[l].cur];
      // f-visit: R = f_{l-1} - avg8(A u) from the R6 pyramid, f_l not streamed
      const bool pyr27 = pyr && b.global && h->restrict_pyr;
      srfmg::launch_resid27_fused<T>(L, U(l), scratch, frhs(b), st, pyr27 ? 1 : 0);
      srfmg::launch_restrict_from_resid<T>(L, U(l), scratch, h->L[l - 1], U(l - 1), rc, jr, st,
                                           pyr27 ? fview(l - 1, l > h->T) : View<T>{});
      return;
    }
    // SR levels (segment storage; per segment, so every partition runs it, R25): the
    // bulk-copy-fed bands when an instantiation fits
    if (l > h->T && h->restrict_seg && !L.st27 && (use_pyr || !b.global) &&
        srfmg::launch_restrict_seg<T>(h->L[l], U(l), b, h->L[l - 1], U(l - 1), rc, jr, st,
                                      use_pyr ? fview(l - 1, l > h->T) : View<T>{}))
      return;
    // the free ping-pong buffer of level l is scratch for the 27-point residual
    srfmg::launch_restrict<T>(h->L[l], U(l), b, h->L[l - 1], U(l - 1), rc, jr, st,
                              (T*)h->B[l].u[1 - h->B[l].cur],
                              use_pyr ? fview(l - 1, l > h->T) : View<T>{});  // L113-115 / L233, L235
  }

  void tau_from_rres(int lc, int jr) {  // the separate tau on R parked in rres
    const Lvl& L = h->L[lc];
    flush();
    cudaMemcpyAsync(h->B[lc].rhs, h->B[lc].rres, (size_t)L.ss * L.nsegs * sizeof(T),
                    cudaMemcpyDeviceToDevice, st);
    tau_std(lc, jr);
  }
  void tau_std(int lc, int jr) {
    const CellCounts& c = h->cells[lc];
    Launch g(h, st, KC_TAU, lc, w * (2.0 * c.storage + 2.0 * c.compute));
    srfmg::launch_tau<T>(h->L[lc], U(lc), (T*)h->B[lc].rhs, (T*)h->B[lc].t, jr, st);
  }
  // the tau of SR level lc can ride in the first pass of vcycle(lc): the same conditions
  // as the fused degree-2 pre-smoothing with the segment-storage rhs
  bool tau_fuse_ok(int lc) const {
    const Lvl& L = h->L[lc];
    const bool base = h->tau_fuse && h->B[lc].rres && lc > h->T && h->fused &&
                      h->d.nu1 == 2 && L.nlg == 0.0;
    if (L.st27)  // the 27-point pass (fused27.cu) under the conditions cheb() uses
      return base && fills(L, 10) &&
             srfmg::cheb27_fused_ok<T>(L);
    return base &&
           (fills(L, 40) && (h->force || L.E[1] >= h->fused_min_e)) &&
           srfmg::cheb2_fused_ok<T>(L) && srfmg::cheb_spec_ok<T>(L);
  }

  // fig:mgv (l <= T) and fig:mgvsr (l > T) are the same recursion over level descriptors.
  // entry = the FMG visit of level l (fig:fmg L139-141 / fig:fmgsr L221-223): Pi and S^alpha
  // run first, fused with the V-cycle's first half where a pass exists.
  void vcycle(int l, View<T> b, bool entry = false) {
    if (l == 0) {  // L120-121: exact solve
      coarsest(b);
      return;
    }
    if (entry) {
      if (pset1_on(l, b)) {
        pset1(l, b);                 // Pi onto C ∪ GSR and S^1, one pass
      } else {
        prolong(l, 0);               // Pi onto C ∪ GSR
        cheb(l, h->d.alpha, b);      // S^alpha
      }
    }
    cheb(l, h->d.nu1, b);  // L112 / L232
    restrict_std(l, b);
    const int jr = jr_for(l);
    // a8: the level-T hand-off (R16).  Multi-GPU: the blocks of the agglomeration level A
    // (T, or below a decomposed T) are all-gathered; a decomposed coarse level refreshes its
    // ghost ring for the tau instead
    if (h->world > 1 && l - 1 == h->A) gather_uR();
    if (dd(l - 1)) halo_u(l - 1);
    // an idle rank (l - 1 == A, desc.coarse_idle) skips the tau and the coarse V-cycle:
    // rank 0 runs them and sends w_A and t_A back
    if (!solves_A() && l - 1 == h->A) {
      // (nothing here: rank 0 forms the tau rhs and t_A)
    } else if (cx(l - 1)) {  // conventional level: F = V = Omega (jr = 0)
      srfmg::COp<T> o = cop(srfmg::kCopTau, l - 1, l - 1);
      o.a = U(l - 1);
      o.c = (T*)h->B[l - 1].rhs;
      o.d = (T*)h->B[l - 1].t;
      emit(o, w * 4.0 * h->cells[l - 1].compute);
    } else if (tau_fuse_ok(l - 1)) {
      pend_tau = l - 1;  // L234-236 inside the first pass of vcycle(l - 1)
      pend_jr = jr;
    } else {
      tau_std(l - 1, jr);  // L116-117 / L234-236
    }
    if (solves_A() || l - 1 > h->A) vcycle(l - 1, sview(l - 1));  // L117 / L237-240
    if (h->idle && l - 1 == h->A) bcast_A(true);  // w_A and t_A to the idle ranks
    if (up_on(l, b)) {
      up2(l, b, l == h->M);  // L241-242 in one pass (at l = M: the solve's last pass)
      return;
    }
    prolong(l, 1);                    // L118 / L241
    cheb(l, h->d.nu2, b, l == h->M);  // L119 / L242 (at l = M: the solve's last pass)
  }

  // correction + degree-2 post-smoothing in one pass (up.cu) on the SR levels the fused
  // Chebyshev pass takes; the choice uses the single-GPU shape of the coarse level (R25)
  bool up_on(int l, const View<T>& b) const {
    const Lvl& L = h->L[l];
    // (l - 1 > T: the coarse w and t in segment storage, whose row pitch the pass fixes)
    return h->up_fuse && h->fused && l - 1 > h->T && h->d.nu2 == 2 && !L.st27 && L.nlg == 0.0 &&
           tma_rhs_ok(b) && fills(L, 40) && (h->force || L.E[1] >= h->fused_min_e) &&
           srfmg::up2_fused_ok<T>(L, glob(l - 1));
  }
  void up2(int l, const View<T>& b, bool last) {
    const Lvl& L = h->L[l];
    LevelBufs& bb = h->B[l];
    const CellCounts& c = h->cells[l];
    const bool fp = dd(l - 1) && l - 1 == h->T;
    if (fp) footprint_T(true);  // k = 1 from a decomposed level T: w - t with its ghosts
    const double rho0 = 1.0 / h->sigma[l];
    const double rho1 = 1.0 / (2.0 * h->sigma[l] - rho0);
    const bool fin = last && final_out != nullptr;
    srfmg::FinalOut<T> fo{};
    const double nv = (double)h->blk_n[0] * h->blk_n[1] * h->blk_n[2];
    if (fin) {
      fo.p = final_out;
      for (int i = 0; i < 3; ++i) fo.bo[i] = h->blk_lo[i];
      fo.sy = h->blk_n[0];
      fo.sz = (long long)h->blk_n[0] * h->blk_n[1];
    }
    bool ok;
    {
      // algorithmic words: u read (C u GSR), rhs (C), w and t (1/8 each), u or user u written
      Launch g(h, st, KC_PASS_UP, l, w * (c.cg + c.compute + c.cg / 4.0 + (fin ? nv : c.cg)));
      ok = srfmg::launch_up2_fused<T>(
          L, fp ? h->LT2 : h->L[l - 1], (const T*)bb.u[bb.cur], (T*)bb.u[1 - bb.cur],
          fp ? (const T*)h->wT2 : U(l - 1), fp ? (const T*)h->zT2 : (const T*)h->B[l - 1].t,
          frhs(b), 1.0 / h->theta[l], rho1 * rho0, 2.0 * rho1 / h->delta[l], st, fo);
    }
    if (!ok) {  // (up_on checked the single-GPU fit; a rank's block never needs more)
      h->sticky = SR_ERR_UNSUPPORTED_CONFIG;
      h->err = "fused up pass: no instantiation for this level";
      return;
    }
    bb.cur = 1 - bb.cur;
    if (fin) final_done = true;
  }

  void run(T* uout) {
    bind();
    run_body(uout);
    unbind();
  }
  void run_body(T* uout) {
    const int M = h->M;
    final_out = uout;
    final_done = false;
    // R6: f pyramid -- the rank's haloed blocks down to level T (multi-GPU), then the
    // global levels below (after assembling f_T)
    for (int l = M; l > h->T; --l) {
      const auto& d = h->fdim[l];
      const T* src = (l == M) ? f : (const T*)(h->world > 1 ? h->B[l].floc : h->B[l].fpyr);
      T* dst = (T*)(h->world > 1 ? h->B[l - 1].floc : h->B[l - 1].fpyr);
      Launch g(h, st, KC_PYRAMID, l, w * (double)d[0] * d[1] * d[2] * (1.0 + 1.0 / 8));
      srfmg::launch_pyramid<T>(src, d[0], d[1], d[2], dst, st);
    }
    if (h->world > 1) {
      // decomposed levels: each rank averages its own block (f_T from the haloed local
      // f_T) down to level A, whose blocks are then all-gathered (the rank's own part is
      // written straight into the global f_A)
      for (int l = h->T; l > h->A; --l) {
        int lo[3], n[3];
        for (int i = 0; i < 3; ++i) {
          n[i] = h->blk_n[i] >> (M - l + 1);
          lo[i] = h->blk_lo[i] >> (M - l + 1);
        }
        Launch g(h, st, KC_PYRAMID, l, w * (double)n[0] * n[1] * n[2] * 9.0);
        srfmg::launch_pyramid_box<T>(fview(l), fview(l - 1), lo, n, st);
      }
      gather_f();
    }
    for (int l = h->A; l >= 1 && solves_A(); --l) {
      const Lvl& L = h->L[l];
      if (l < M && cx(l)) {
        srfmg::COp<T> o = cop(srfmg::kCopPyramid, l, l - 1);
        o.a = (const T*)h->B[l].fpyr;
        o.c = (T*)h->B[l - 1].fpyr;
        emit(o, w * (double)L.N[0] * L.N[1] * L.N[2] * (1.0 + 1.0 / 8));
        continue;
      }
      Launch g(h, st, KC_PYRAMID, l, w * (double)L.N[0] * L.N[1] * L.N[2] * (1.0 + 1.0 / 8));
      srfmg::launch_pyramid<T>(l == M ? f : (const T*)h->B[l].fpyr, L.N[0], L.N[1], L.N[2],
                               (T*)h->B[l - 1].fpyr, st);
    }
    pyr = true;
    if (solves_A()) coarsest(fview(0));  // fig:fmg L137-138
    for (int l = 1; l <= M; ++l) {  // fig:fmg L139-142 (l <= T), fig:fmgsr L220-223 (l > T)
      if (l <= h->A && !solves_A()) continue;  // idle rank
      if (h->idle && l == h->A + 1) bcast_A(false);  // u_A for the interpolation
      vcycle(l, fview(l), /*entry=*/true);
    }
    if (!final_done) {
      const Lvl& L = h->L[M];
      Launch g(h, st, KC_GATHER, M, w * 2.0 * h->blk_n[0] * (double)h->blk_n[1] * h->blk_n[2]);
      srfmg::launch_gather<T>(L, U(M), uout, h->blk_lo, h->blk_n[0],
                              (long long)h->blk_n[0] * h->blk_n[1], st);  // R19
    }
  }
};

sr_status_t enqueue_solve(sr_fmg* h, const void* f, void* u, cudaStream_t st) {
  h->launches = 0;
  h->exch = 0;
  std::fill(h->comm_calls.begin(), h->comm_calls.end(), 0LL);
  h->prof_used = 0;
  for (int l = 0; l <= h->M; ++l) h->B[l].cur = 0;
  if (h->esize == 8) {
    Schedule<double> s{h, st, (const double*)f, 8.0};
    s.run((double*)u);
  } else {
    Schedule<float> s{h, st, (const float*)f, 4.0};
    s.run((float*)u);
  }
  h->exch_per_solve = h->exch;
  if (h->sticky != SR_OK) return h->sticky;
  CU(h, cudaGetLastError());
  return SR_OK;
}

double alg_bytes(const sr_fmg* h) {
  // B_alg: 5.5 words per compute cell per level visit, the f pyramid
  // (8/7 N^3 words) and the output (N^3 words)
  double words = 0;
  for (int l = 1; l <= h->M; ++l) words += 5.5 * (double)h->visits[l] * h->cells[l].compute;
  const Lvl& L = h->L[h->M];
  const double n = (double)L.N[0] * L.N[1] * L.N[2];
  words += n * (8.0 / 7.0) + n;
  return words * h->esize;
}

// ---- NCCL, loaded at run time from the libnccl.so.2 the process already uses (torch's)
struct NcclApi {
  typedef struct { char internal[128]; } UniqueId;
  typedef void* CommT;
  int (*getUniqueId)(UniqueId*) = nullptr;
  int (*commInitRank)(CommT*, int, UniqueId, int) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, CommT, cudaStream_t) = nullptr;
  int (*send)(const void*, size_t, int, int, CommT, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, CommT, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  int (*commDestroy)(CommT) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    // prefer the NCCL the process already uses (e.g. PyTorch's, loaded by `import torch`):
    // loading a second, older libnccl.so.2 first would shadow it for later loads; else an
    // explicit SR_FMG_NCCL_LIB, else the loader's libnccl.so.2
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib)
      if (const char* e = std::getenv("SR_FMG_NCCL_LIB")) lib = dlopen(e, RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!lib) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return api;
    }
    api.getUniqueId = (int (*)(NcclApi::UniqueId*))dlsym(lib, "ncclGetUniqueId");
    api.commInitRank =
        (int (*)(NcclApi::CommT*, int, NcclApi::UniqueId, int))dlsym(lib, "ncclCommInitRank");
    api.allGather = (int (*)(const void*, void*, size_t, int, NcclApi::CommT, cudaStream_t))dlsym(
        lib, "ncclAllGather");
    api.send = (int (*)(const void*, size_t, int, int, NcclApi::CommT, cudaStream_t))dlsym(
        lib, "ncclSend");
    api.recv = (int (*)(void*, size_t, int, int, NcclApi::CommT, cudaStream_t))dlsym(
        lib, "ncclRecv");
    api.groupStart = (int (*)())dlsym(lib, "ncclGroupStart");
    api.groupEnd = (int (*)())dlsym(lib, "ncclGroupEnd");
    api.commDestroy = (int (*)(NcclApi::CommT))dlsym(lib, "ncclCommDestroy");
    api.getErrorString = (const char* (*)(int))dlsym(lib, "ncclGetErrorString");
    api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.send && api.recv &&
             api.groupStart && api.groupEnd && api.commDestroy;
    if (!api.ok) api.why = "libnccl.so.2 lacks the expected symbols";
  }
  return api;
}

struct NcclComm : Comm {
  NcclApi::CommT comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().commDestroy(comm);
  }
  sr_status_t allgather(sr_fmg* h, const void* send, void* recv, size_t bytes,
                        cudaStream_t st) override {
    const int r = nccl().allGather(send, recv, bytes, /*ncclInt8*/ 0, comm, st);
    if (r != 0) return fail(h, SR_ERR_NCCL, std::string("ncclAllGather: ") +
                                                (nccl().getErrorString ? nccl().getErrorString(r) : "error"));
    return SR_OK;
  }
  // one halo phase: the sends and receives with the (up to two) neighbours of one dimension
  // in one NCCL group (matched per peer in issue order; one transfer per direction and pair)
  sr_status_t group(sr_fmg* h, const Xfer* xs, int n, cudaStream_t st) override {
    NcclApi& api = nccl();
    int r = api.groupStart();
    for (int i = 0; i < n && r == 0; ++i)
      r = xs[i].recv ? api.recv(xs[i].buf, xs[i].bytes, /*ncclInt8*/ 0, xs[i].peer, comm, st)
                     : api.send(xs[i].buf, xs[i].bytes, 0, xs[i].peer, comm, st);
    const int e = api.groupEnd();
    if (r == 0) r = e;
    if (r != 0) return fail(h, SR_ERR_NCCL, std::string("ncclSend/ncclRecv: ") +
                                                (api.getErrorString ? api.getErrorString(r) : "error"));
    return SR_OK;
  }
};

// ---- test backend: the ranks of one process (one host thread each, all on one GPU) pass
// their messages through host memory.  Every transfer is synchronous on the host (device ->
// host copy, mailbox, host -> device copy); a receive blocks until its sender has posted, so
// the ranks must run concurrently.  No kernel of one rank ever waits for another rank.
struct HostStore {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<std::vector<char>>> box;  // (src, dst) -> FIFO
  bool aborted = false;
};

struct HostComm : Comm {
  HostStore* store = nullptr;
  sr_status_t post(sr_fmg* h, int peer, const void* buf, size_t bytes, cudaStream_t st) {
    std::vector<char> msg(bytes);
    CU(h, cudaMemcpyAsync(msg.data(), buf, bytes, cudaMemcpyDeviceToHost, st));
    CU(h, cudaStreamSynchronize(st));
    {
      std::lock_guard<std::mutex> g(store->mu);
      store->box[{h->rank, peer}].push_back(std::move(msg));
    }
    store->cv.notify_all();
    return SR_OK;
  }
  sr_status_t take(sr_fmg* h, int peer, void* buf, size_t bytes, cudaStream_t st) {
    std::vector<char> msg;
    {
      std::unique_lock<std::mutex> g(store->mu);
      auto& q = store->box[{peer, h->rank}];
      const bool got = store->cv.wait_for(g, std::chrono::seconds(30),
                                          [&] { return !q.empty() || store->aborted; });
      if (!got || q.empty()) {
        store->aborted = true;
        store->cv.notify_all();
        return fail(h, SR_ERR_NCCL, "host store: no message from rank " + std::to_string(peer));
      }
      msg = std::move(q.front());
      q.pop_front();
    }
    if (msg.size() != bytes) return fail(h, SR_ERR_NCCL, "host store: message size mismatch");
    CU(h, cudaMemcpyAsync(buf, msg.data(), bytes, cudaMemcpyHostToDevice, st));
    CU(h, cudaStreamSynchronize(st));
    return SR_OK;
  }
  sr_status_t allgather(sr_fmg* h, const void* send, void* recv, size_t bytes,
                        cudaStream_t st) override {
    if (!store) return fail(h, SR_ERR_INVALID_ARGUMENT, "host comm without a store");
    for (int q = 0; q < store->world; ++q)
      if (q != h->rank) {
        sr_status_t r = post(h, q, send, bytes, st);
        if (r != SR_OK) return r;
      }
    CU(h, cudaMemcpyAsync((char*)recv + (size_t)h->rank * bytes, send, bytes,
                          cudaMemcpyDeviceToDevice, st));
    for (int q = 0; q < store->world; ++q)
      if (q != h->rank) {
        sr_status_t r = take(h, q, (char*)recv + (size_t)q * bytes, bytes, st);
        if (r != SR_OK) return r;
      }
    return SR_OK;
  }
  sr_status_t group(sr_fmg* h, const Xfer* xs, int n, cudaStream_t st) override {
    if (!store) return fail(h, SR_ERR_INVALID_ARGUMENT, "host comm without a store");
    for (int i = 0; i < n; ++i)  // all sends first: posting never blocks
      if (!xs[i].recv) {
        sr_status_t r = post(h, xs[i].peer, xs[i].buf, xs[i].bytes, st);
        if (r != SR_OK) return r;
      }
    for (int i = 0; i < n; ++i)
      if (xs[i].recv) {
        sr_status_t r = take(h, xs[i].peer, xs[i].buf, xs[i].bytes, st);
        if (r != SR_OK) return r;
      }
    return SR_OK;
  }
};

// device memory of a handle: the descriptor's allocator hooks, else cudaMalloc / cudaFree
cudaError_t dev_alloc(sr_fmg* h, void** p, size_t bytes) {
  if (h->d.alloc) {
    *p = h->d.alloc(bytes, h->d.alloc_ctx);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMalloc(p, bytes);
}
void dev_free(sr_fmg* h, void* p) {
  if (!p) return;
  if (h->d.free) h->d.free(p, h->d.alloc_ctx);
  else cudaFree(p);
}

void drop_graph(sr_fmg::GraphEnt& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  if (g.graph) cudaGraphDestroy(g.graph);
  g.exec = nullptr;
  g.graph = nullptr;
  g.na.clear();
  g.nb.clear();
}

void free_ring(sr_fmg* h) {
  for (auto& set : h->ring)
    for (auto& r : set) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  h->ring.clear();
  h->ring_n = 0;
  h->ring_pos = 0;
}

void free_all(sr_fmg* h) {
  for (auto& g : h->graphs) drop_graph(g);
  free_ring(h);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
    if (h->ev_solve[i]) cudaEventDestroy(h->ev_solve[i]);
    if (h->ev_d2h[i]) cudaEventDestroy(h->ev_d2h[i]);
  }
  if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
  if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
  for (auto& b : h->B) {
    dev_free(h, b.u[0]);
    dev_free(h, b.u[1]);
    dev_free(h, b.rres);
    dev_free(h, b.rhs);
    dev_free(h, b.t);
    dev_free(h, b.fpyr);
    dev_free(h, b.floc);
    dev_free(h, b.dwt);
  }
  dev_free(h, h->xsend);
  dev_free(h, h->xrecv);
  dev_free(h, h->wT2);
  dev_free(h, h->zT2);
  dev_free(h, h->hsend);
  dev_free(h, h->hrecv);
  delete h->comm;
  h->comm = nullptr;
  dev_free(h, h->ainv);
  for (int i = 0; i < 2; ++i) {
    dev_free(h, h->host_f[i]);
    dev_free(h, h->host_u[i]);
  }
  for (auto& r : h->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (h->cap) cudaStreamDestroy(h->cap);
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

size_t sr_fmg_desc_size(void) { return sizeof(sr_fmg_desc_t); }

void sr_fmg_desc_init(sr_fmg_desc_t* d) {
  if (!d) return;
  std::memset(d, 0, sizeof(*d));
  d->buffer = 2;
  d->sched_A = -1;
  d->sched_B = -1;
  d->dtype = SR_F64;
  d->alpha = 1;
  d->nu1 = 2;
  d->nu2 = 2;
  d->cheb_lo = 0.0;  // the stencil's default: 1/6 (7-point, R8) or 1/3 (27-point, R28)
  d->cheb_hi = 1.0;
  d->stencil = 7;
  d->nl_gamma = 0.0;
  d->world = 1;
  d->pgrid[0] = d->pgrid[1] = d->pgrid[2] = 1;
  d->device = -1;
  d->use_graph = 1;
}

sr_status_t sr_fmg_create(int64_t N, int32_t M, int32_t seg, int32_t buffer, int32_t sr_levels,
                          sr_fmg_t** out) {
  sr_fmg_desc_t d;
  sr_fmg_desc_init(&d);
  d.n[0] = d.n[1] = d.n[2] = N;
  d.M = M;
  d.seg = seg;
  d.buffer = buffer;
  d.sr_levels = sr_levels;
  return sr_fmg_create_ex(&d, out);
}

sr_status_t sr_fmg_create_ex(const sr_fmg_desc_t* d, sr_fmg_t** out) {
  if (!out) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!d) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "descriptor is NULL");
  std::string msg;
  sr_status_t st = validate(d, msg);
  if (st != SR_OK) return fail(nullptr, st, msg);

  sr_fmg* h = new sr_fmg();
  h->d = *d;
  make_plan(h);
  if (!plan_ok(h, msg)) {
    delete h;
    return fail(nullptr, SR_ERR_UNSUPPORTED_CONFIG, msg);
  }
  for (int l = 1; l <= h->M; ++l) {
    const Lvl &Lf = h->L[l], &Lc = h->L[l - 1];
    if (l - 1 > h->T && Lc.J < (Lf.J + 1) / 2) {
      delete h;
      return fail(nullptr, SR_ERR_UNSUPPORTED_CONFIG,
                  "buffer schedule violates J_{l-1} >= ceil(J_l/2) (prolongation footprint)");
    }
    if ((long long)Lf.E[0] * Lf.E[1] * Lf.E[2] >= (1LL << 31)) {
      delete h;
      return fail(nullptr, SR_ERR_UNSUPPORTED_CONFIG, "segment storage box too large");
    }
  }
  {
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      delete h;
      return fail(nullptr, SR_ERR_CUDA,
                  std::string("no CUDA device: ") + (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    }
  }
  const char* sd = std::getenv("SR_FMG_SYNC");
  h->sync_debug = sd && sd[0] == '1';
  const char* tr = std::getenv("SR_FMG_TRACE");
  h->trace = tr && tr[0] == '1';
  if (const char* e = std::getenv("SR_FMG_CEXEC_ONE")) h->cexec_one = e[0] == '1';
  const char* fu = std::getenv("SR_FMG_FUSED");
  h->fused = !(fu && fu[0] == '0');
  const char* ff = std::getenv("SR_FMG_FORCE_FUSED");
  h->force = ff && ff[0] == '1';
  if (const char* e = std::getenv("SR_FMG_FUSED_MIN_E")) h->fused_min_e = std::atoi(e);
  const char* ce = std::getenv("SR_FMG_CEXEC");
  h->cexec = !(ce && ce[0] == '0');
  if (const char* e = std::getenv("SR_FMG_PSET1")) h->pset1 = std::atoi(e) != 0;
  if (const char* e = std::getenv("SR_FMG_RESTRICT_PYR")) h->restrict_pyr = std::atoi(e) != 0;
  if (const char* e = std::getenv("SR_FMG_RESTRICT_SEG")) h->restrict_seg = std::atoi(e) != 0;
  if (const char* e = std::getenv("SR_FMG_TAU_FUSE")) h->tau_fuse = std::atoi(e) != 0;
  if (const char* e = std::getenv("SR_FMG_UP_FUSE")) h->up_fuse = std::atoi(e) != 0;
  if (d->device >= 0) {
    cudaError_t e = cudaSetDevice(d->device);
    if (e != cudaSuccess) {
      delete h;
      return fail(nullptr, SR_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
  }
  h->stream = (cudaStream_t)d->stream;
  h->B.assign(h->M + 1, LevelBufs{});
  auto alloc = [&](void** p, size_t bytes) -> bool {
    if (bytes == 0) bytes = 16;
    if (dev_alloc(h, p, bytes) != cudaSuccess) return false;
    h->workspace += (long long)bytes;
    return cudaMemset(*p, 0, bytes) == cudaSuccess;
  };
  bool ok = true;
  for (int l = 0; l <= h->M && ok; ++l) {
    const Lvl& L = h->L[l];
    const size_t bytes = (size_t)L.ss * L.nsegs * h->esize;
    ok = ok && alloc(&h->B[l].u[0], bytes) && alloc(&h->B[l].u[1], bytes);
    if (l < h->M) {
      ok = ok && alloc(&h->B[l].rhs, bytes) && alloc(&h->B[l].t, bytes);
      if (l > h->T && h->tau_fuse) ok = ok && alloc(&h->B[l].rres, bytes);
      if (h->world == 1 || l <= h->A)
        ok = ok && alloc(&h->B[l].fpyr, (size_t)L.N[0] * L.N[1] * L.N[2] * h->esize);
      else if (l < h->T)  // decomposed level below T: the rank's block of f_l, and w - t
        ok = ok && alloc(&h->B[l].fpyr, (size_t)L.S[0] * L.S[1] * L.S[2] * h->esize) &&
             alloc(&h->B[l].dwt, bytes);
      if (h->world > 1 && l >= h->T) {
        const auto& fd = h->fdim[l];
        ok = ok && alloc(&h->B[l].floc, (size_t)fd[0] * fd[1] * fd[2] * h->esize);
      }
    }
  }
  if (h->world > 1) {
    // all-gather of the agglomeration level's blocks (u and R), and halo staging for the
    // decomposed levels: both sides of the largest face slab, ghost width deep
    long long nbA = 1;
    for (int i = 0; i < 3; ++i) nbA *= h->blk_n[i] >> (h->M - h->A);
    h->xbytes = (size_t)2 * nbA * h->esize;
    ok = ok && alloc(&h->xsend, h->xbytes) && alloc(&h->xrecv, h->xbytes * h->world);
    long long face = 0;
    auto slab = [&](const Lvl& L) {
      for (int i = 0; i < 3; ++i)
        face = std::max(face, 2LL * (L.J + 1) * L.E[(i + 1) % 3] * L.E[(i + 2) % 3]);
    };
    for (int l = h->A + 1; l <= h->T; ++l) slab(h->L[l]);
    if (h->A < h->T && h->K > 0) slab(h->LT2);
    h->hbytes = (size_t)std::max(face, 1LL) * h->esize;
    if (h->A < h->T) ok = ok && alloc(&h->hsend, h->hbytes) && alloc(&h->hrecv, h->hbytes);
  }
  if (h->world > 1 && h->A < h->T) {
    // zT2: the zero t of the corrections from w - t copies (dwt on the decomposed levels
    // below T, the footprint copy wT2 of level T); wT2 only with SR levels above T
    long long zs = 0;
    for (int l = h->A + 1; l < h->T; ++l) zs = std::max(zs, h->L[l].ss);
    if (h->K > 0) {
      zs = std::max(zs, h->LT2.ss);
      ok = ok && alloc(&h->wT2, (size_t)h->LT2.ss * h->esize);
    }
    ok = ok && alloc(&h->zT2, (size_t)std::max(zs, 1LL) * h->esize);
  }
  std::vector<double> inv = coarsest_inverse(h->L[0]);
  const size_t n0sq = inv.size();
  ok = ok && alloc(&h->ainv, n0sq * h->esize);
  if (ok) {
    if (h->esize == 8) {
      ok = cudaMemcpy(h->ainv, inv.data(), n0sq * 8, cudaMemcpyHostToDevice) == cudaSuccess;
    } else {
      std::vector<float> f32(inv.begin(), inv.end());
      ok = cudaMemcpy(h->ainv, f32.data(), n0sq * 4, cudaMemcpyHostToDevice) == cudaSuccess;
    }
  }
  if (ok) ok = cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    free_all(h);
    delete h;
    return fail(nullptr, SR_ERR_OUT_OF_MEMORY, "device allocation failed");
  }
  if (h->world > 1) {
    if (d->comm == 1) {
      h->comm = new HostComm();
      h->d.use_graph = 0;  // host round trips inside the solve
    } else {
      NcclApi& api = nccl();
      if (!api.ok || !d->nccl_id) {
        const std::string why = !api.ok ? api.why : "world > 1 needs desc.nccl_id";
        free_all(h);
        delete h;
        return fail(nullptr, api.ok ? SR_ERR_INVALID_ARGUMENT : SR_ERR_NCCL, why);
      }
      NcclComm* c = new NcclComm();
      NcclApi::UniqueId id;
      std::memcpy(&id, d->nccl_id, sizeof(id));
      const int r = api.commInitRank(&c->comm, d->world, id, d->rank);
      h->comm = c;
      if (r != 0) {
        const std::string why = std::string("ncclCommInitRank: ") +
                                (api.getErrorString ? api.getErrorString(r) : "error");
        free_all(h);
        delete h;
        return fail(nullptr, SR_ERR_NCCL, why);
      }
    }
  }
  *out = h;
  return SR_OK;
}

sr_status_t sr_fmg_set_stream(sr_fmg_t* h, void* stream) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->stream = (cudaStream_t)stream;
  return SR_OK;
}

sr_status_t sr_fmg_solve(sr_fmg_t* h, const void* f, void* u) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->sticky != SR_OK) return h->sticky;
  if (!f || !u) return fail(h, SR_ERR_INVALID_ARGUMENT, "f or u is NULL");
  if (((uintptr_t)f & 15) || ((uintptr_t)u & 15))
    return fail(h, SR_ERR_INVALID_ARGUMENT, "f and u must be 16-byte aligned");
  const bool graph = h->d.use_graph && !h->sync_debug;
  if (!graph) return enqueue_solve(h, f, u, h->stream);
  sr_fmg::GraphEnt* ge = nullptr;
  for (auto& g : h->graphs)
    if (g.exec && g.f == f && g.u == u) ge = &g;
  if (!ge) {  // capture for these pointers, replacing the least recently used graph
    ge = &h->graphs[0];
    for (auto& g : h->graphs)
      if (!g.exec || g.used < ge->used) ge = &g;
    drop_graph(*ge);
    CU(h, cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    sr_status_t st = enqueue_solve(h, f, u, h->cap);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    if (st != SR_OK) return st;
    if (e != cudaSuccess) return fail(h, SR_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&ge->exec, g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      return fail(h, SR_ERR_CUDA, std::string("instantiate: ") + cudaGetErrorString(e));
    }
    if (h->prof_used > 0) {  // profiled: find the event-record nodes of every ProfRec
      size_t nn = 0;
      CU(h, cudaGraphGetNodes(g, nullptr, &nn));
      std::vector<cudaGraphNode_t> nodes(nn);
      CU(h, cudaGraphGetNodes(g, nodes.data(), &nn));
      ge->na.assign(h->prof_used, nullptr);
      ge->nb.assign(h->prof_used, nullptr);
      for (cudaGraphNode_t n : nodes) {
        cudaGraphNodeType ty;
        cudaEvent_t ev = nullptr;
        if (cudaGraphNodeGetType(n, &ty) != cudaSuccess || ty != cudaGraphNodeTypeEventRecord ||
            cudaGraphEventRecordNodeGetEvent(n, &ev) != cudaSuccess)
          continue;
        for (size_t i = 0; i < h->prof_used; ++i) {
          if (h->prof[i].a == ev) ge->na[i] = n;
          if (h->prof[i].b == ev) ge->nb[i] = n;
        }
      }
      ge->graph = g;
    } else {
      cudaGraphDestroy(g);
    }
    ge->f = f;
    ge->u = u;
  }
  ge->used = ++h->gclock;
  if (h->ring_n > 0 && ge->graph) {  // this solve's events: ring slot ring_pos % ring_n
    auto& set = h->ring[(size_t)(h->ring_pos++ % h->ring_n)];
    while (set.size() < h->prof_used) {
      ProfRec r{};
      CU(h, cudaEventCreate(&r.a));
      CU(h, cudaEventCreate(&r.b));
      set.push_back(r);
    }
    for (size_t i = 0; i < h->prof_used; ++i) {
      set[i].bytes = h->prof[i].bytes;
      if (!ge->na[i] || !ge->nb[i]) return fail(h, SR_ERR_CUDA, "profiling ring: event node missing");
      CU(h, cudaGraphExecEventRecordNodeSetEvent(ge->exec, ge->na[i], set[i].a));
      CU(h, cudaGraphExecEventRecordNodeSetEvent(ge->exec, ge->nb[i], set[i].b));
    }
  }
  CU(h, cudaGraphLaunch(ge->exec, h->stream));
  return SR_OK;
}

// Conventional V-cycle solver: u = 0, then FASMGV(M) until
// ||f - A u||_2 / ||f||_2 <= rtol (reading R26), at most maxit cycles.  Eager launches; one
// host synchronisation per cycle for the stopping test.
sr_status_t sr_fmg_vsolve(sr_fmg_t* h, const void* f, void* u, double rtol, int32_t maxit,
                          int32_t* cycles, double* relres) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->sticky != SR_OK) return h->sticky;
  if (!f || !u) return fail(h, SR_ERR_INVALID_ARGUMENT, "f or u is NULL");
  if (!(rtol >= 0) || maxit < 0) return fail(h, SR_ERR_INVALID_ARGUMENT, "need rtol >= 0, maxit >= 0");
  if (h->K != 0 || h->world != 1)
    return fail(h, SR_ERR_UNSUPPORTED_CONFIG,
                "the V-cycle solver runs on a conventional (sr_levels = 0) single-GPU handle");
  cudaStream_t st = h->stream;
  double* acc = nullptr;
  CU(h, cudaMalloc(&acc, 2 * sizeof(double)));
  auto body = [&](auto tag) -> sr_status_t {
    using T = decltype(tag);
    Schedule<T> s{h, st, (const T*)f, (double)sizeof(T)};
    s.bind();
    const int M = h->M;
    const Lvl& L = h->L[M];
    LevelBufs& bb = h->B[M];
    for (int l = 0; l <= M; ++l) h->B[l].cur = 0;
    CU(h, cudaMemsetAsync(bb.u[0], 0, (size_t)L.ss * L.nsegs * sizeof(T), st));
    CU(h, cudaMemsetAsync(bb.u[1], 0, (size_t)L.ss * L.nsegs * sizeof(T), st));
    // the R6 pyramid is not used: the coarse rhs are the tau right-hand sides
    auto norm2 = [&](double& out) -> sr_status_t {
      s.flush();
      CU(h, cudaMemsetAsync(acc, 0, sizeof(double), st));
      srfmg::launch_resnorm<T>(L, s.U(M), s.fview(M), acc, st);
      h->launches++;
      double hv = 0;
      CU(h, cudaMemcpyAsync(&hv, acc, sizeof(double), cudaMemcpyDeviceToHost, st));
      CU(h, cudaStreamSynchronize(st));
      out = std::sqrt(hv);
      return SR_OK;
    };
    double fn = 0, rn = 0;
    sr_status_t r = norm2(fn);  // u = 0: the residual is f
    if (r != SR_OK) return r;
    int it = 0;
    double rel = !std::isfinite(fn) ? fn : (fn > 0 ? 1.0 : 0.0);
    for (;; ++it) {
      if (it > 0) {
        r = norm2(rn);
        if (r != SR_OK) return r;
        rel = fn > 0 ? rn / fn : 0.0;
      }
      if (!std::isfinite(rel)) {  // diverged (or a non-finite f): stop, report
        s.unbind();
        if (cycles) *cycles = it;
        if (relres) *relres = rel;
        return fail(h, SR_ERR_NONFINITE, "vsolve: the residual norm is not finite");
      }
      if (rel <= rtol || it == maxit) break;
      s.vcycle(M, s.fview(M));  // fig:mgv from level M
    }
    s.flush();
    srfmg::launch_gather<T>(L, s.U(M), (T*)u, h->blk_lo, h->blk_n[0],
                            (long long)h->blk_n[0] * h->blk_n[1], st);
    h->launches++;
    s.unbind();
    if (cycles) *cycles = it;
    if (relres) *relres = rel;
    return SR_OK;
  };
  sr_status_t r = h->esize == 8 ? body(double{}) : body(float{});
  cudaFree(acc);
  if (r != SR_OK) return r;
  CU(h, cudaGetLastError());
  return SR_OK;
}

sr_status_t sr_fmg_solve_host_async(sr_fmg_t* h, const void* f_host, void* u_host) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  if (h->sticky != SR_OK) return h->sticky;
  if (!f_host || !u_host) return fail(h, SR_ERR_INVALID_ARGUMENT, "f or u is NULL");
  const auto& fd = h->fdim[h->M];
  const size_t fbytes = (size_t)fd[0] * fd[1] * fd[2] * h->esize;
  const size_t ubytes = (size_t)h->blk_n[0] * h->blk_n[1] * h->blk_n[2] * h->esize;
  if (!h->s_h2d) {
    CU(h, cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    CU(h, cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CU(h, cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming));
      CU(h, cudaEventCreateWithFlags(&h->ev_solve[i], cudaEventDisableTiming));
      CU(h, cudaEventCreateWithFlags(&h->ev_d2h[i], cudaEventDisableTiming));
      // "already completed" initial state for the first two calls' waits
      CU(h, cudaEventRecord(h->ev_solve[i], h->stream));
      CU(h, cudaEventRecord(h->ev_d2h[i], h->stream));
    }
  }
  const int k = (int)(h->hcalls & 1);
  if (!h->host_f[k]) {
    CU(h, dev_alloc(h, &h->host_f[k], fbytes));
    CU(h, dev_alloc(h, &h->host_u[k], ubytes));
  }
  // f -> slot k once the solve two calls back has finished reading it
  CU(h, cudaStreamWaitEvent(h->s_h2d, h->ev_solve[k], 0));
  CU(h, cudaMemcpyAsync(h->host_f[k], f_host, fbytes, cudaMemcpyHostToDevice, h->s_h2d));
  CU(h, cudaEventRecord(h->ev_h2d[k], h->s_h2d));
  // the solve once f has landed and the copy-out two calls back has drained u of slot k
  CU(h, cudaStreamWaitEvent(h->stream, h->ev_h2d[k], 0));
  CU(h, cudaStreamWaitEvent(h->stream, h->ev_d2h[k], 0));
  sr_status_t st = sr_fmg_solve(h, h->host_f[k], h->host_u[k]);
  if (st != SR_OK) return st;
  CU(h, cudaEventRecord(h->ev_solve[k], h->stream));
  CU(h, cudaStreamWaitEvent(h->s_d2h, h->ev_solve[k], 0));
  CU(h, cudaMemcpyAsync(u_host, h->host_u[k], ubytes, cudaMemcpyDeviceToHost, h->s_d2h));
  CU(h, cudaEventRecord(h->ev_d2h[k], h->s_d2h));
  h->hcalls++;
  return SR_OK;
}

sr_status_t sr_fmg_synchronize(sr_fmg_t* h) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  CU(h, cudaStreamSynchronize(h->stream));
  if (h->s_h2d) CU(h, cudaStreamSynchronize(h->s_h2d));
  if (h->s_d2h) CU(h, cudaStreamSynchronize(h->s_d2h));
  return h->sticky;
}

sr_status_t sr_fmg_solve_host(sr_fmg_t* h, const void* f_host, void* u_host) {
  sr_status_t st = sr_fmg_solve_host_async(h, f_host, u_host);
  if (st != SR_OK) return st;
  return sr_fmg_synchronize(h);
}

void sr_fmg_destroy(sr_fmg_t* h) {
  if (!h) return;
  // every stream of the handle: a copy of the host pipeline may still read a staging slot,
  // which an allocator hook could hand out again as soon as it is freed
  cudaStreamSynchronize(h->stream);
  if (h->s_h2d) cudaStreamSynchronize(h->s_h2d);
  if (h->s_d2h) cudaStreamSynchronize(h->s_d2h);
  free_all(h);
  delete h;
}

sr_status_t sr_fmg_partition(const sr_fmg_desc_t* d, sr_fmg_partition_t* out) {
  if (!d || !out) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  std::string msg;
  const sr_status_t st = validate(d, msg);
  if (st != SR_OK) return fail(nullptr, st, msg);
  sr_fmg tmp;
  tmp.d = *d;
  make_plan(&tmp);
  if (!plan_ok(&tmp, msg)) return fail(nullptr, SR_ERR_UNSUPPORTED_CONFIG, msg);
  std::memset(out, 0, sizeof(*out));
  out->world = tmp.world;
  out->rank = tmp.rank;
  for (int i = 0; i < 3; ++i) {
    out->coord[i] = tmp.coord[i];
    out->segs_per_rank[i] = tmp.nsr[i];
    out->block_lo[i] = tmp.blk_lo[i];
    out->block_n[i] = tmp.blk_n[i];
    out->f_dims[i] = tmp.fdim[tmp.M][i];
    out->level_T_lo[i] = tmp.blkT_lo[i];
    out->level_T_n[i] = tmp.blkT_n[i];
  }
  out->f_halo = tmp.H[tmp.M];
  out->level_A = tmp.A;
  return SR_OK;
}

sr_status_t sr_fmg_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  NcclApi& api = nccl();
  if (!api.ok) return fail(nullptr, SR_ERR_NCCL, api.why);
  NcclApi::UniqueId id;
  const int r = api.getUniqueId(&id);
  if (r != 0) return fail(nullptr, SR_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, sizeof(id));
  return SR_OK;
}

void* sr_fmg_host_store_create(int32_t world) {
  HostStore* s = new HostStore();
  s->world = world;
  return s;
}

void sr_fmg_host_store_destroy(void* store) { delete (HostStore*)store; }

sr_status_t sr_fmg_set_host_store(sr_fmg_t* h, void* store) {
  if (!h || !store) return fail(h, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  HostComm* c = dynamic_cast<HostComm*>(h->comm);
  if (!c) return fail(h, SR_ERR_INVALID_ARGUMENT, "handle was not created with comm = 1");
  c->store = (HostStore*)store;
  return SR_OK;
}

sr_status_t sr_fmg_get_info(const sr_fmg_t* h, sr_fmg_info_t* info) {
  if (!h || !info) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->M = h->M;
  info->K = h->K;
  info->T = h->T;
  info->dtype = h->d.dtype;
  for (int l = 0; l <= h->M; ++l) {
    const Lvl& L = h->L[l];
    for (int i = 0; i < 3; ++i) {
      info->n_level[l][i] = L.N[i];
      info->nseg[l][i] = L.ns[i];
      info->storage_ext[l][i] = L.E[i];
    }
    info->storage_pitch[l][0] = L.py;
    info->storage_pitch[l][1] = L.pz;
    info->storage_pitch[l][2] = L.ss;
    info->sr[l] = l > h->T;
    info->seg_level[l] = L.S[0];
    info->buffer_level[l] = L.J;
    info->compute_cells[l] = h->cells[l].compute;
    info->visits[l] = h->visits[l];
  }
  info->workspace_bytes = h->workspace;
  // count launches of one solve without enqueuing: dry count from the schedule shape
  long long n = 0;
  {
    // pyramid M, coarsest 1, per FMG level l: prolong + alpha + vcycle(l)
    auto cheb_n = [&](int deg) { return deg > 0 ? deg : 0; };
    std::vector<long long> vc(h->M + 1, 0);
    vc[0] = 1;
    for (int l = 1; l <= h->M; ++l)
      vc[l] = cheb_n(h->d.nu1) + 2 + vc[l - 1] + 1 + cheb_n(h->d.nu2);
    n = h->M + 1 + 1;
    for (int l = 1; l <= h->M; ++l) n += 1 + cheb_n(h->d.alpha) + vc[l];
  }
  // launches of the last enqueued solve (exact), else the unfused schedule's count
  info->launches_per_solve = h->launches > 0 ? h->launches : n;
  info->world = h->world;
  info->rank = h->rank;
  for (int i = 0; i < 3; ++i) {
    info->block_lo[i] = h->blk_lo[i];
    info->block_n[i] = h->blk_n[i];
    info->f_dims[i] = h->fdim[h->M][i];
  }
  info->f_halo = h->H[h->M];
  info->exchanges_per_solve = h->exch_per_solve;
  info->level_A = h->A;
  for (int l = 0; l <= h->M; ++l) {
    info->dd[l] = (h->world > 1 && l > h->A && l <= h->T) ? 1 : 0;
    info->comm_calls[l] = h->comm_calls[l];
  }
  info->alg_bytes_per_solve = alg_bytes(h);
  return SR_OK;
}

const char* sr_fmg_last_error(const sr_fmg_t* h) {
  if (h) return h->err.c_str();
  return g_tls_err.c_str();
}

int32_t sr_fmg_kernel_count(void) { return srfmg::kNumKernelNames; }
const char* sr_fmg_kernel_name(int32_t i) {
  if (i < 0 || i >= srfmg::kNumKernelNames) return "";
  return srfmg::kKernelNames[i];
}

// ---- profiling (used by bench.py): CUDA events around every launch of one kernel class
// at one level, recorded inside the captured graph of the next solves.
sr_status_t sr_fmg_profile_select(sr_fmg_t* h, int32_t kernel_class, int32_t level) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "handle is NULL");
  h->prof_cls = kernel_class;
  h->prof_level = level;
  for (auto& g : h->graphs) drop_graph(g);
  free_ring(h);
  return SR_OK;
}

sr_status_t sr_fmg_profile_ring(sr_fmg_t* h, int32_t nslots) {
  if (!h || nslots < 0) return fail(h, SR_ERR_INVALID_ARGUMENT, "NULL handle or nslots < 0");
  free_ring(h);
  h->ring_n = nslots;
  h->ring.resize((size_t)nslots);
  return SR_OK;
}

sr_status_t sr_fmg_profile_read_slot(sr_fmg_t* h, int32_t slot, double* ms, double* bytes,
                                     int32_t* launches) {
  if (!h || !ms || !bytes || !launches) return fail(h, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  if (slot < 0 || slot >= h->ring_n) return fail(h, SR_ERR_INVALID_ARGUMENT, "slot out of range");
  double t = 0, b = 0;
  const auto& set = h->ring[(size_t)slot];
  for (const auto& r : set) {
    float x = 0;
    CU(h, cudaEventElapsedTime(&x, r.a, r.b));
    t += x;
    b += r.bytes;
  }
  *ms = t;
  *bytes = b;
  *launches = (int32_t)set.size();
  return SR_OK;
}

// After a solve has completed: total device time (ms), algorithmic bytes and the number
// of profiled launches of that solve.
sr_status_t sr_fmg_profile_read(sr_fmg_t* h, double* ms, double* bytes, int32_t* launches) {
  if (!h || !ms || !bytes || !launches) return fail(h, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  double t = 0, b = 0;
  for (size_t i = 0; i < h->prof_used; ++i) {
    float x = 0;
    CU(h, cudaEventElapsedTime(&x, h->prof[i].a, h->prof[i].b));
    t += x;
    b += h->prof[i].bytes;
  }
  *ms = t;
  *bytes = b;
  *launches = (int32_t)h->prof_used;
  return SR_OK;
}

sr_status_t sr_fmg_debug_level_io(sr_fmg_t* h, int32_t level, int32_t field, int32_t write,
                                  void* host) {
  if (!h || !host) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "NULL argument");
  if (level < 0 || level > h->M) return fail(h, SR_ERR_INVALID_ARGUMENT, "bad level");
  LevelBufs& b = h->B[level];
  void* p = field == 0 ? b.u[b.cur] : field == 1 ? b.rhs : field == 2 ? b.t : nullptr;
  if (!p) return fail(h, SR_ERR_INVALID_ARGUMENT, "field not present on this level");
  const Lvl& L = h->L[level];
  const size_t bytes = (size_t)L.ss * L.nsegs * h->esize;
  CU(h, cudaStreamSynchronize(h->stream));
  if (write) {
    CU(h, cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice));
    if (field == 0) CU(h, cudaMemcpy(b.u[1 - b.cur], host, bytes, cudaMemcpyHostToDevice));
  } else {
    CU(h, cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost));
  }
  return SR_OK;
}

sr_status_t sr_fmg_debug_op(sr_fmg_t* h, int32_t op, int32_t level, int32_t deg,
                            const void* f_dev) {
  if (!h) return fail(nullptr, SR_ERR_INVALID_ARGUMENT, "NULL handle");
  if (level < 0 || level > h->M) return fail(h, SR_ERR_INVALID_ARGUMENT, "bad level");
  if ((op == 1 || op == 3 || op == 4) && level < 1)
    return fail(h, SR_ERR_INVALID_ARGUMENT, "op needs level >= 1");
  if (op == 2 && level >= h->M) return fail(h, SR_ERR_INVALID_ARGUMENT, "tau needs level < M");
  cudaStream_t st = h->stream;
  auto body = [&](auto tag) -> sr_status_t {
    using T = decltype(tag);
    Schedule<T> s{h, st, (const T*)f_dev, (double)sizeof(T)};
    auto rhs = [&](int l) { return (l == h->M) ? s.fview(l) : s.sview(l); };
    s.bind();
    switch (op) {
      case 0: s.cheb(level, deg, rhs(level)); break;
      case 1:
        srfmg::launch_restrict<T>(h->L[level], s.U(level), rhs(level), h->L[level - 1],
                                  s.U(level - 1), (T*)h->B[level - 1].rhs, s.jr_for(level), st);
        break;
      case 2:
        srfmg::launch_tau<T>(h->L[level], s.U(level), (T*)h->B[level].rhs, (T*)h->B[level].t,
                             s.jr_for(level + 1), st);
        break;
      case 3: s.prolong(level, 0); break;
      case 4: s.prolong(level, 1); break;
      case 5: s.coarsest(s.sview(0)); break;
      default: s.unbind(); return fail(h, SR_ERR_INVALID_ARGUMENT, "unknown op");
    }
    s.unbind();
    return SR_OK;
  };
  if (op == 0 && level == h->M && !f_dev)
    return fail(h, SR_ERR_INVALID_ARGUMENT, "level M smoothing needs f_dev");
  sr_status_t r = h->esize == 8 ? body(double{}) : body(float{});
  if (r != SR_OK) return r;
  CU(h, cudaGetLastError());
  CU(h, cudaStreamSynchronize(st));
  return SR_OK;
}

}  // extern "C"
