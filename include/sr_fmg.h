/*
 * sr_fmg.h -- C ABI of the B200 segmental-refinement full-multigrid solver.
 *
 * Operation (the paper's problem statement, §2 Eq. 1-2):
 *   solve  L_h u_h = f_h  on the cell-centred grid Omega_h, u = 0 on the boundary, with
 *   L_h = -Lap_h the 7-point operator (readings R1/R2 of DESIGN.md §3), by one FAS full
 *   multigrid F(alpha, nu1, nu2) solve (fig:fmg) whose finest
 *   `sr_levels` levels are segmental-refinement levels (fig:fmgsr / fig:mgvsr,
 *   PAPER.md:216-246): every segment of seg^3 genuine fine cells plus `buffer` buffer
 *   cells is smoothed, residual-evaluated, restricted and prolongated on its own, with no
 *   exchange between segments; the levels at and below the transition level
 *   T = M - sr_levels run a conventional FAS V-cycle down to an exact coarsest solve.
 *   The result is an APPROXIMATION (FMG algebraic error O(discretisation error), plus the
 *   SR buffer perturbation) -- not the exact discrete solution.
 *
 * Layout.  f and u are dense arrays of n[0]*n[1]*n[2] elements, x1 fastest:
 *   element (i1, i2, i3) at offset (i3*n[1] + i2)*n[0] + i1, cell centre
 *   x_d = (i_d + 1/2) h.  Element type: double (SR_F64) or float (SR_F32).
 *
 * Ownership.  The caller owns f and u; the library never retains them after a call
 *   returns.  The library owns its device workspace (allocated in create, freed in
 *   destroy) and, when it captures one, the CUDA graph of a solve.
 *
 * Execution.  sr_fmg_solve is asynchronous and ordered on the handle's stream (the
 *   legacy default stream unless one is given).  Device pointers must be 16-byte aligned
 *   and must not overlap.  sr_fmg_solve_host is synchronous.
 *
 * Errors.  Every call returns SR_OK or an error code; sr_fmg_last_error() gives a
 *   message.  create validates everything before allocating; on failure *out = NULL.
 *   A CUDA error makes the handle sticky-failed: that call and every later call on the
 *   handle return SR_ERR_CUDA until destroy.  A handle is not thread-safe.
 *
 * Determinism.  Results are bitwise reproducible for a fixed (descriptor, f).
 */
#ifndef SR_FMG_H
#define SR_FMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SR_FMG_MAX_LEVELS 24

typedef struct sr_fmg sr_fmg_t; /* opaque */

typedef enum {
  SR_OK = 0,
  SR_ERR_INVALID_ARGUMENT = 1,  /* arithmetically impossible descriptor / null pointer */
  SR_ERR_UNSUPPORTED_CONFIG = 2,/* valid, but outside what this build supports          */
  SR_ERR_OUT_OF_MEMORY = 3,
  SR_ERR_CUDA = 4,
  SR_ERR_NCCL = 5,
  SR_ERR_NONFINITE = 6          /* sr_fmg_vsolve: the residual norm became NaN or Inf    */
} sr_status_t;

typedef enum { SR_F64 = 0, SR_F32 = 1 } sr_dtype_t;

/* Full descriptor.  Initialise with sr_fmg_desc_init() and override fields. */
typedef struct {
  int64_t n[3];       /* fine cells per dimension (x1, x2, x3); each divisible by 2^M   */
  int32_t M;          /* number of coarsenings: levels 0..M, coarsest grid n/2^M (>= 1) */
  int32_t seg;        /* S: genuine segment edge on the finest level; n_d % S == 0,      */
                      /*    S % 2^sr_levels == 0 (ignored when sr_levels == 0)           */
  int32_t buffer;     /* J: buffer cells on every SR level (Eq. 5 with A = J, B = 0)     */
  int32_t sr_levels;  /* K: number of SR levels, 0 <= K <= M (0 = conventional FMG)      */
  int32_t sched_A;    /* Eq. 5 buffer schedule J_k = 2 floor((A + B (K-k))/2)            */
  int32_t sched_B;    /*   (PAPER.md:192); (-1, -1) = constant `buffer`; sched_B = -2:    */
                      /*   maximum buffer schedule J_k = 2^(k-1) J_1 with J_1 = sched_A  */
                      /*   (C_k = F_k for k < K)                        */
  int32_t dtype;      /* sr_dtype_t                                                       */
  double h;           /* fine cell size; 0 = 1/n[0] (unit cube for cubic grids)          */
  int32_t alpha;      /* F(alpha, nu1, nu2) Chebyshev degrees;       */
  int32_t nu1;        /*   default (1, 2, 2)                                             */
  int32_t nu2;
  double cheb_lo;     /* Chebyshev interval [lo, hi] * lambda_max (12/h_l^2, 7-point;    */
  double cheb_hi;     /*   4/h_l^2, 27-point); lo = 0: default 1/6 (7-pt) / 1/3 (27-pt)  */
  int32_t world;      /* number of ranks (GPUs); 1 = single GPU                          */
  int32_t rank;
  int32_t pgrid[3];   /* rank grid; world == pgrid[0]*pgrid[1]*pgrid[2]                  */
  const void *nccl_id;/* 128-byte ncclUniqueId (world > 1)                               */
  int32_t device;     /* CUDA device ordinal; -1 = current device                        */
  void *stream;       /* cudaStream_t; NULL = legacy default stream                      */
  int32_t use_graph;  /* 1 (default): capture a solve into a CUDA graph and replay it    */
  int32_t comm;       /* world > 1: 0 = NCCL (default), 1 = test host store (see below)   */
  int32_t stencil;    /* 7 (default): 7-point FD, A = -Lap_h (BASELINE); 27: the paper's    */
                      /*   27-point operator (weights centre 8/3, edges     */
                      /*   -1/6, corners -1/12, faces 0, /h^2), lambda_max = 4/h^2; runs  */
                      /*   on the unfused kernels                                        */
  double nl_gamma;    /* >= 0: nonlinear FAS test operator A(u) = -L_h u + nl_gamma u^3     */
                      /*   (SURVEY f4); 0 (default) = linear.  Unfused kernels; Picard    */
                      /*   iterations with A_lin^-1 for the exact coarsest solve          */
  /* Optional device allocator for the workspace (e.g. a framework's caching allocator):  */
  /* alloc(bytes, ctx) returns device memory or NULL; free(p, ctx) releases it.  Both NULL */
  /* (default): cudaMalloc / cudaFree.  Used for every device buffer the handle owns, from */
  /* create (and the host-pipeline slots, on first use) to destroy.                         */
  void *(*alloc)(size_t bytes, void *ctx);
  void (*free)(void *p, void *ctx);
  void *alloc_ctx;
  /* world > 1: the conventional levels l <= T stay domain-decomposed (each rank holds its  */
  /* block, a halo exchange of grouped ncclSend/ncclRecv before every operator application, */
  /* PAPER.md:157-168) while every dimension of the rank's block has at least dd_min cells; */
  /* the first level below is all-gathered once per visit and it and the coarser levels    */
  /* are solved redundantly on every rank.  0 = default (32); a value    */
  /* larger than the level-T block agglomerates at T (no decomposed coarse levels).         */
  /* sr_levels = 0 with world > 1 is the paper's non-SR baseline: every  */
  /* level down to A is decomposed, the finest included (fine-level halo exchanges); the   */
  /* finest rank block must then have at least dd_min cells per dimension.                  */
  int32_t dd_min;
  /* world > 1: how the levels <= A are solved.  0 (default) = redundant: */
  /* level A is all-gathered and every rank solves the levels <= A.  1 = idle: the blocks of */
  /* level A are gathered onto rank 0 alone, rank 0 solves the levels <= A while the other   */
  /* ranks idle, and rank 0 sends u_A (and the tau snapshot t_A) back to every rank.  Same   */
  /* arithmetic, bitwise the same result.                                                    */
  int32_t coarse_idle;
} sr_fmg_desc_t;

typedef struct {
  int32_t M, K, T;                         /* levels 0..M; transition level T = M-K    */
  int32_t dtype;
  int64_t n_level[SR_FMG_MAX_LEVELS][3];   /* cells of Omega_l per dimension           */
  int32_t sr[SR_FMG_MAX_LEVELS];           /* 1 if level l is an SR level              */
  int32_t seg_level[SR_FMG_MAX_LEVELS];    /* S_l (SR levels) or n_l[0] (conventional) */
  int32_t buffer_level[SR_FMG_MAX_LEVELS]; /* J_l (0 on conventional levels)           */
  int32_t nseg[SR_FMG_MAX_LEVELS][3];      /* segments per dimension (1 if conventional) */
  int32_t storage_ext[SR_FMG_MAX_LEVELS][3];/* storage box extent per segment            */
  int64_t storage_pitch[SR_FMG_MAX_LEVELS][3]; /* element strides: row, plane, segment  */
  int64_t compute_cells[SR_FMG_MAX_LEVELS];/* sum_p |C_l^p|                             */
  int64_t visits[SR_FMG_MAX_LEVELS];       /* level visits per solve (smoothing passes)  */
  int64_t workspace_bytes;
  int64_t launches_per_solve;              /* kernel launches in one solve               */
  double alg_bytes_per_solve;              /* B_alg of DESIGN.md §6 (fused-design bytes) */
  int32_t world, rank;                     /* multi-GPU: this rank's block (see partition) */
  int64_t block_lo[3], block_n[3];         /* fine cells owned (output block of u)        */
  int32_t f_halo;                          /* halo width of the local f block             */
  int64_t f_dims[3];                       /* local f array dims = block_n + 2 f_halo     */
  int64_t exchanges_per_solve;             /* collective calls of the last solve (all-    */
                                           /* gathers + halo phases; 0 before a solve)    */
  int32_t level_A;                         /* levels <= A gathered / redundant; levels    */
                                           /* A < l <= T decomposed (A = T: none)         */
  int32_t dd[SR_FMG_MAX_LEVELS];           /* 1 if level l is domain-decomposed           */
  int64_t comm_calls[SR_FMG_MAX_LEVELS];   /* collective calls (NCCL groups / all-gathers) */
                                           /* per level in the last solve: 0 on SR levels */
} sr_fmg_info_t;

/* Multi-GPU partition of a descriptor (pure host arithmetic, no GPU needed).  The
 * segment grid (n_d/seg per dimension) is split into pgrid blocks; rank r has block
 * coordinates (r % P1, (r / P1) % P2, r / (P1 P2)).  Each rank solves the SR levels of its
 * own segments with no communication.  The conventional levels A < l <= T
 * are domain-decomposed: rank r owns block (its fine block) / 2^(M-l) of Omega_l and
 * exchanges halos with its face neighbours; the levels <= A are
 * all-gathered and solved redundantly on every rank. */
typedef struct {
  int32_t world, rank, coord[3];
  int32_t segs_per_rank[3];          /* SR segments per dimension owned by this rank     */
  int64_t block_lo[3], block_n[3];   /* fine genuine cells owned: [lo, lo + n)           */
  int32_t f_halo;                    /* f must be given on [lo - halo, lo + n + halo)     */
  int64_t f_dims[3];                 /* = block_n + 2 f_halo (x1 fastest)                 */
  int64_t level_T_lo[3], level_T_n[3]; /* this rank's block of the transition level T     */
  int32_t level_A;                   /* levels A < l <= T decomposed, l <= A redundant      */
} sr_fmg_partition_t;

/* Fill *d with defaults: cube 0, M 0, seg 0, buffer 2, K 0, sched (-1,-1), fp64,
 * h 0, F(1,2,2), interval [1/6, 1], world 1, device -1, stream NULL, use_graph 1. */
void sr_fmg_desc_init(sr_fmg_desc_t *d);

/* sizeof(sr_fmg_desc_t) as compiled into the library: bindings check their struct layout
 * against it before passing a descriptor (the struct grew with stencil and nl_gamma). */
size_t sr_fmg_desc_size(void);

/* North-star form: cube N^3, fp64, constant buffer, current device, default stream. */
sr_status_t sr_fmg_create(int64_t N, int32_t M, int32_t seg, int32_t buffer,
                          int32_t sr_levels, sr_fmg_t **out);
sr_status_t sr_fmg_create_ex(const sr_fmg_desc_t *d, sr_fmg_t **out);

/* One FMG+SR solve.  f: device pointer to the fine right-hand side; u: device pointer to
 * the output (every cell written).  Asynchronous on the handle's stream.
 * world > 1: f is this rank's block WITH a halo of f_halo cells on every side
 * (sr_fmg_partition; halo cells outside the domain are ignored), u is the rank's block
 * without halo.  Collective: every rank must call it (NCCL all-gathers inside). */
sr_status_t sr_fmg_solve(sr_fmg_t *h, const void *f, void *u);

/* The same solve from HOST buffers: copies f to the device, solves, copies u back,
 * synchronises.  Pinned host memory makes the copies asynchronous DMA. */
sr_status_t sr_fmg_solve_host(sr_fmg_t *h, const void *f_host, void *u_host);

/* Asynchronous host-buffer solve for a stream of right-hand sides.  Enqueues: copy f_host
 * (layout of sr_fmg_solve's f) into one of two internal device slots on a copy stream, the
 * solve on the handle's stream, and the copy of u back to u_host on a second copy stream,
 * chained with events.  Consecutive calls alternate the slots, so the host->device copy of
 * call i+1, the solve of call i and the device->host copy of call i-1 overlap (PCIe is full
 * duplex; the copy engines run beside the SMs).  Returns immediately: the caller must not
 * modify f_host nor read u_host before sr_fmg_synchronize(h).  f_host/u_host should be
 * pinned (cudaHostAlloc / cudaHostRegister); pageable memory works but serialises. */
sr_status_t sr_fmg_solve_host_async(sr_fmg_t *h, const void *f_host, void *u_host);

/* Wait for every solve and copy enqueued on the handle; returns its sticky status. */
sr_status_t sr_fmg_synchronize(sr_fmg_t *h);

/* Conventional multigrid V-cycle solver, the paper's comparison solver ("V-cycle solve
 * with a relative residual tolerance of 10^-4"): u = 0 on the fine grid,
 * then V(nu1, nu2)-cycles (fig:mgv) until ||f - A u||_2 <= rtol ||f||_2 or maxit cycles.
 * f, u: device pointers as in sr_fmg_solve.  Needs a handle with sr_levels = 0 and
 * world = 1 (SR_ERR_UNSUPPORTED_CONFIG otherwise).  Synchronous (one device->host read of
 * the residual norm per cycle).  *cycles = cycles run, *relres = final relative residual
 * (either may be NULL). */
sr_status_t sr_fmg_vsolve(sr_fmg_t *h, const void *f, void *u, double rtol, int32_t maxit,
                          int32_t *cycles, double *relres);

/* Change the stream later solves are ordered on (a captured graph is reused). */
sr_status_t sr_fmg_set_stream(sr_fmg_t *h, void *stream);

void sr_fmg_destroy(sr_fmg_t *h); /* NULL-safe; synchronises the handle's stream */

/* Partition arithmetic of a (validated) descriptor; no GPU needed. */
sr_status_t sr_fmg_partition(const sr_fmg_desc_t *d, sr_fmg_partition_t *out);

/* 128-byte ncclUniqueId for sr_fmg_desc_t.nccl_id (call on rank 0, broadcast). */
sr_status_t sr_fmg_nccl_unique_id(void *out128);

sr_status_t sr_fmg_get_info(const sr_fmg_t *h, sr_fmg_info_t *info);

/* Message of the last error on h (or of the calling thread's last failed create when
 * h == NULL).  Never NULL; valid until the next call on the same handle/thread. */
const char *sr_fmg_last_error(const sr_fmg_t *h);

/* Number of distinct kernels the library can launch, and their names (for launch lists). */
int32_t sr_fmg_kernel_count(void);
const char *sr_fmg_kernel_name(int32_t i);

/* ---- test-only hooks (not part of the solver contract) ---------------------------------
 * sr_fmg_debug_level_io: copy the internal storage of (level, field) of ALL segments
 * between the device and a host buffer of nseg*storage_pitch[level][2] elements; cells
 * outside the domain must be written as zero (the kernels rely on that invariant)
 * (field 0 = current u, 1 = rhs, 2 = t; write != 0 copies host -> device).
 * sr_fmg_debug_op: run one kernel of the schedule on the internal buffers:
 *   op 0 = CHEB(deg) on level with rhs = internal rhs buffer (or user f when level == M),
 *   op 1 = residual + restriction level -> level-1,  op 2 = tau-rhs + t snapshot on level
 *          (support from level+1),  op 3 = prolongation SET level-1 -> level,
 *   op 4 = prolongation ADD of (u - t) level-1 -> level,  op 5 = exact coarsest solve. */
sr_status_t sr_fmg_debug_level_io(sr_fmg_t *h, int32_t level, int32_t field, int32_t write,
                                  void *host);
sr_status_t sr_fmg_debug_op(sr_fmg_t *h, int32_t op, int32_t level, int32_t deg,
                            const void *f_dev);

/* Test-only comm backend (desc.comm = 1): instead of NCCL, the handles of all ranks live in
 * one process, one host thread each (all on one GPU), and pass every all-gather block and
 * halo slab through a host-side store (device -> host copy, mailbox, host -> device copy;
 * a receive blocks until the sending rank has posted, at most 30 s, then SR_ERR_NCCL).
 * The rank threads must call sr_fmg_solve concurrently.  No kernel waits for another rank.
 * Forces eager (non-graph) execution. */
void *sr_fmg_host_store_create(int32_t world);
void sr_fmg_host_store_destroy(void *store);
sr_status_t sr_fmg_set_host_store(sr_fmg_t *h, void *store);

/* Profiling hooks used by bench.py: select one kernel class (index into
 * sr_fmg_kernel_name) at one level; later solves record a CUDA event pair around every
 * such launch (inside the captured graph).  profile_read, after the solve completed,
 * returns the summed device time (ms), the summed algorithmic bytes and
 * the number of profiled launches of the last solve.  kernel_class -1 disables. */
sr_status_t sr_fmg_profile_select(sr_fmg_t *h, int32_t kernel_class, int32_t level);
sr_status_t sr_fmg_profile_read(sr_fmg_t *h, double *ms, double *bytes, int32_t *launches);
/* Profiling ring (graph solves only): after profile_select and one capturing solve,
 * profile_ring(h, n) makes graph solve number i (counted from this call) record its
 * profiled launches into event set i % n, so n solves can run back to back with no host
 * synchronisation between them; profile_read_slot(h, i, ...) reads set i once they have
 * completed (same outputs as profile_read).  n = 0 turns the ring off. */
sr_status_t sr_fmg_profile_ring(sr_fmg_t *h, int32_t nslots);
sr_status_t sr_fmg_profile_read_slot(sr_fmg_t *h, int32_t slot, double *ms, double *bytes,
                                     int32_t *launches);

#ifdef __cplusplus
}
#endif
#endif /* SR_FMG_H */
