/*
 * trmcr.h — C ABI of the B200-native TRMC-R hot path (arXiv:1009.2768).
 *
 * One call of trmcr_step() advances every cell by one time step of the
 * recursive Time-Relaxed Monte Carlo scheme:
 *   (shock only) A1 free transport x <- x + v_x dt with inflow/outflow
 *                reservoirs (splitting; boundary states P:971-988)
 *   (shock only) A2 stable counting sort of the particles by cell
 *   A3 per-cell moments and majorant Sigma = sigma(2 dv)
 *   A4 split into collision sets, Alg 4.2 with IR rounding
 *   A5 recursive collision trees of Alg 4.3/4.4, flattened into a
 *      level-synchronous work list
 *   A6 binary (dummy) collisions, eq. Maxwell_coll/n3d
 *   A7 adaptive truncation TRMC-RAD
 *   A8 conservative Maxwellian resampling of the truncated set
 * Paper line numbers "P:nnn" refer to PAPER.md; readings "[Rnn]" to DESIGN.md §2.
 *
 * Conventions (all calls):
 *   - Every call returns trmcr_status; nothing throws across the ABI.
 *   - Argument errors return TRMCR_EINVAL and set trmcr_last_error(ctx).
 *   - CUDA failures are sticky: the context returns TRMCR_ESTATE afterwards.
 *   - A context owns all device buffers it allocates; caller memory passed to
 *     trmcr_init is COPIED (the caller keeps ownership).  Output pointers
 *     belong to the caller.
 *   - One context per device and stream; calls are not thread safe.
 *   - trmcr_step is asynchronous on the context's stream; calls that return
 *     host data synchronise that stream.
 *   - Units: K = 1/(4 pi) [R4]; homogeneous cells have rho = 1.
 */
#ifndef TRMCR_H
#define TRMCR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct trmcr_ctx trmcr_ctx;

typedef enum {
  TRMCR_OK = 0,
  TRMCR_EINVAL = 1,     /* bad argument (message in trmcr_last_error)              */
  TRMCR_ENOMEM = 2,     /* device allocation failed                                */
  TRMCR_ECUDA = 3,      /* CUDA runtime error                                      */
  TRMCR_ENCCL = 4,      /* reserved: collective error                              */
  TRMCR_ECAPACITY = 5,  /* particles or per-cell tree exceeded the capacity        */
  TRMCR_ESTATE = 6      /* context unusable after an earlier sticky error          */
} trmcr_status;

/* B(|q|, .) = K |q|^alpha, K = 1/(4 pi): Maxwell alpha = 0, hard spheres
 * alpha = 1, VHS any alpha in [0, 1] (trmcr_kernel.alpha; dummy collisions with
 * Sigma = sigma(2 dv), sec. VHS). */
typedef enum { TRMCR_MAXWELL = 0, TRMCR_HARD_SPHERE = 1, TRMCR_VHS = 2 } trmcr_model;
typedef enum { TRMCR_F32 = 0, TRMCR_F64 = 1 } trmcr_dtype;
typedef enum { TRMCR_HOMOGENEOUS = 0, TRMCR_SHOCK_1D = 1 } trmcr_geometry;
typedef enum { TRMCR_IND_PXX = 0, TRMCR_IND_M4 = 1 } trmcr_indicator;  /* RAD indicator S */

/* Particle ensemble handed to trmcr_init.  Structure of arrays of length n
 * in `dtype`; device pointers unless `host` = 1.  x (positions) only for the
 * shock geometry.  Homogeneous: particles must be grouped by cell as
 * described by trmcr_cells.offsets.  Shock: positions inside [x_min, x_max)
 * and sorted by cell (non-decreasing cell index; validated, EINVAL if not). */
typedef struct {
  int32_t dtype;             /* trmcr_dtype                                          */
  int32_t host;              /* 1: pointers are host memory, 0: device memory        */
  int64_t n;                 /* number of particles                                  */
  int64_t capacity;          /* particle capacity (shock inflow headroom); 0: auto   */
  const void *vx, *vy, *vz;  /* velocities                                           */
  const void *x;             /* positions (shock) or NULL                            */
} trmcr_particles;

/* Cell geometry.
 * HOMOGENEOUS: n_cells independent space-homogeneous gases (rho = 1), cell c
 *   holding particles [offsets[c], offsets[c+1]) (host array of n_cells+1,
 *   non-decreasing, offsets[0] = 0).
 * SHOCK_1D: n_cells uniform cells on [x_min, x_max); weight = mass per
 *   particle; reservoir states (rho,u,T)_{L,R} from Rankine-Hugoniot
 *   (P:975-985).  offsets must be NULL.
 * cell_base: global id of local cell 0 (keys the RNG: results do not depend
 *   on how cells are split across devices).
 * SHOCK_1D slabs: the context owns global cells [cell_base, cell_base +
 *   n_cells) of an n_cells_global grid on the GLOBAL domain [x_min, x_max);
 *   neighbors = bit 0 (a slab on the left), bit 1 (a slab on the right); the
 *   reservoir of a side exists only without a neighbour there.  A slab with
 *   neighbours steps with trmcr_shock_begin / (exchange) / trmcr_shock_finish. */
typedef struct {
  int32_t geometry;          /* trmcr_geometry                                       */
  int32_t n_cells;
  int32_t cell_base;
  int32_t pad;
  const int64_t *offsets;    /* HOMOGENEOUS: host [n_cells+1]; SHOCK_1D: NULL        */
  double x_min, x_max, weight;
  double rho_L, u_L, T_L, rho_R, u_R, T_R;
  int32_t n_cells_global;    /* SHOCK_1D: cells of the whole domain (0: = n_cells)   */
  int32_t neighbors;         /* SHOCK_1D: bit 0 left slab, bit 1 right slab          */
} trmcr_cells;

/* Collision kernel and truncation control. */
typedef struct {
  int32_t model;             /* trmcr_model                                          */
  int32_t adaptive;          /* 0: fixed truncation m_fixed (TRMC-R); 1: TRMC-RAD     */
  int32_t m_fixed;           /* e.g. 64                                              */
  int32_t m_init;            /* RAD initial m_max (paper: 2)                   */
  int32_t m_cap;             /* RAD largest m_max (<= 16384)                          */
  int32_t indicator;         /* trmcr_indicator                                       */
  double delta1, delta2;     /* RAD interval, 0 < delta1 < delta2 (paper 0.005, 0.01) */
  uint64_t seed;             /* Philox4x32-10 key                                     */
  double alpha;              /* TRMCR_VHS exponent in [0, 1] (ignored otherwise)      */
  int32_t wb;                /* TRMC-WB (sec. 4.4, Alg 4.6): 0 off; tree length 1 = 1 + min
                                (eq. def:2), 2 = 1 + mean (eq. def:3), 3 = level (def:1);
                                requires adaptive = 0                                  */
  int32_t wb_max;            /* TRMC-WB m_max: final samples with longer trees are
                                resampled from the local Maxwellian                   */
  int32_t sigma_update;      /* majorant variant (remark after Alg 4.4):
                                0 = Sigma' frozen for the step (default); 1 = raised
                                to sigma_ij after every proposal, in the canonical
                                order (level ascending, index ascending, RAD attempts
                                in order).  tau (and mu) still come from the pre-step
                                Sigma'; the stats row reports the pre-step Sigma'.     */
  int32_t literal;           /* 1: the paper's own layout instead of the level-synchronous
                                plan: Alg 4.3/4.4 literally (recursive builds, stored
                                siblings, one sequential keyed stream per cell), one
                                thread per cell (for measuring the
                                LS reformulation).  Homogeneous cells, fixed m <= 128,
                                no RAD / TRMC-WB; TRMCR_ECAPACITY if a cell's trees
                                need more f_0 particles than it holds.                */
} trmcr_kernel;

/* Per-cell statistics row (doubles), trmcr_stats(): */
enum {
  TRMCR_ST_N = 0, TRMCR_ST_P, TRMCR_ST_MU, TRMCR_ST_SIGMA, TRMCR_ST_S0, TRMCR_ST_SEST,
  TRMCR_ST_E1, TRMCR_ST_MUSED, TRMCR_ST_MNEXT, TRMCR_ST_DEPTH, TRMCR_ST_ATTEMPTS,
  TRMCR_ST_LEAVES, TRMCR_ST_UNTOUCHED, TRMCR_ST_THERMALISED, TRMCR_ST_PROPOSALS,
  TRMCR_ST_ACCEPTED, TRMCR_ST_VIOLATIONS, TRMCR_ST_MAXW,
  TRMCR_ST_PX, TRMCR_ST_PY, TRMCR_ST_PZ, TRMCR_ST_ENERGY,   /* sum v, sum |v|^2 (conserved by the step) */
  TRMCR_NSTATS
};
/* Global sums over this context's cells, trmcr_global_moments(): */
enum {
  TRMCR_GM_N = 0, TRMCR_GM_PX, TRMCR_GM_PY, TRMCR_GM_PZ, TRMCR_GM_ENERGY, TRMCR_GM_NPXX,
  TRMCR_GM_PROPOSALS, TRMCR_GM_ACCEPTED, TRMCR_GM_MAXW, TRMCR_GM_COST, TRMCR_NGLOBAL
};
/* Per-cell moment row (doubles), trmcr_moments(): */
enum {
  TRMCR_MO_N = 0, TRMCR_MO_RHO, TRMCR_MO_UX, TRMCR_MO_UY, TRMCR_MO_UZ, TRMCR_MO_T,
  TRMCR_MO_E, TRMCR_MO_P, TRMCR_MO_PXX, TRMCR_MO_M4, TRMCR_MO_M4C, TRMCR_MO_MMAX,
  TRMCR_NMOMENTS
};

/* Collision decision record (trmcr_get_log), one per tree node. */
typedef struct {
  int32_t cell, attempt, level, accepted;
  int64_t j, slot_i, slot_k;
} trmcr_coll_rec;

/* Create a context on the current CUDA device, bound to `cuda_stream`
 * (a cudaStream_t, NULL = legacy default stream).  eps: Knudsen number
 * (P:127-129), dt: time step, both > 0.  Copies the particles (and builds
 * the cell offsets for the shock).
 * Multi-GPU: one context per rank of one simulation.  nccl_id:
 * the 128-byte NCCL unique id from trmcr_get_nccl_id on one rank, moved to every
 * rank by the caller (e.g. a torch.distributed broadcast); rank in [0, nranks).
 * NULL with nranks = 1 for a single GPU.  The context then owns an NCCL
 * communicator (ncclCommInitRank: collective, every rank must call) and uses it
 * for the global moments (trmcr_global_moments all_ranks, trmcr_global_sums,
 * trmcr_moments global) and, for a shock slab with neighbours, for the
 * neighbour exchange inside trmcr_step (rank r must own the r-th slab).
 * Errors: EINVAL (bad sizes/arguments, eps or dt <= 0, delta1 >= delta2, offsets
 * not monotone, particle outside the shock domain, rank/slab mismatch), ENOMEM,
 * ECUDA, ENCCL. */
trmcr_status trmcr_init(trmcr_ctx **out, const trmcr_particles *particles,
                        const trmcr_cells *cells, double eps, double dt,
                        const trmcr_kernel *kernel, void *cuda_stream,
                        const void *nccl_id, int32_t rank, int32_t nranks);

/* Write a fresh NCCL unique id (128 bytes) to out128 (host memory). ENCCL on failure. */
trmcr_status trmcr_get_nccl_id(void *out128);

/* Ranks of the context's communicator (1 without one). */
int32_t trmcr_comm_size(const trmcr_ctx *ctx);

/* Advance n_steps >= 0 time steps (asynchronous).  A shock slab with neighbours
 * needs the NCCL communicator (else: trmcr_shock_begin / exchange / finish). */
trmcr_status trmcr_step(trmcr_ctx *ctx, int32_t n_steps);

/* Per-cell moments of the current state, host
 * out[cells * TRMCR_NMOMENTS]: this context's cells (global = 0), or every
 * rank's cells in global cell order (global = 1; collective over the
 * communicator; out sized for the whole grid).  Syncs. */
trmcr_status trmcr_moments(trmcr_ctx *ctx, double *host_out, int32_t global);

/* Per-cell statistics of the last step, host out[n_cells * TRMCR_NSTATS]. Syncs. */
trmcr_status trmcr_stats(trmcr_ctx *ctx, double *host_out);

/* Global sums (TRMCR_NGLOBAL doubles) of the last step's per-cell statistics,
 * written asynchronously to DEVICE memory `dev_out`; cost = proposals + maxw/2
 * (P:829-832, 878-879).  all_ranks = 1 with a communicator: the sums are then
 * all-reduced over the ranks on the context's communication stream, overlapping
 * the following steps (a later call on the same buffer, or trmcr_comm_wait,
 * orders the context stream after it).  The all-reduced sums depend on the
 * rank count in the last bits; trmcr_global_sums is partition independent. */
trmcr_status trmcr_global_moments(trmcr_ctx *ctx, double *dev_out, int32_t all_ranks);

/* Make the context stream wait for every all-reduce in flight (asynchronous). */
trmcr_status trmcr_comm_wait(trmcr_ctx *ctx);

/* Partition-independent global sums (TRMCR_NGLOBAL doubles, host out) of the last
 * step's statistics over every rank: the per-cell rows are all-gathered and each
 * column is summed exactly rounded (Shewchuk's algorithm), so the result is
 * bitwise the same for any number of GPUs.  Collective; syncs. */
trmcr_status trmcr_global_sums(trmcr_ctx *ctx, double *host_out);

/* Current particle count (shock: changes with inflow/outflow). Syncs. */
trmcr_status trmcr_num_particles(trmcr_ctx *ctx, int64_t *n);

/* Copy the current state out (cell-sorted).  Pointers are host (host = 1) or
 * device memory of capacity >= trmcr_num_particles(); x may be NULL;
 * offsets (n_cells+1 int64, same memory kind) may be NULL. Syncs. */
trmcr_status trmcr_copy_particles(trmcr_ctx *ctx, void *vx, void *vy, void *vz, void *x,
                                  int64_t *offsets, int32_t host);

/* Overwrite the velocities (same count and cell layout as the current
 * state) from host (host = 1) or device memory. Asynchronous. */
trmcr_status trmcr_set_velocities(trmcr_ctx *ctx, const void *vx, const void *vy,
                                  const void *vz, int32_t host);

/* Host-buffer step (the e2e path): upload velocities from host memory,
 * advance one step, download per-cell moments to host_moments
 * [n_cells * TRMCR_NMOMENTS].  Homogeneous geometry only.  Syncs. */
trmcr_status trmcr_step_host(trmcr_ctx *ctx, const void *vx, const void *vy, const void *vz,
                             double *host_moments);

/* Replace the whole particle state (any geometry) from host (host = 1) or
 * device memory: n particles, SoA in the context dtype.  HOMOGENEOUS: x must be
 * NULL and n equal to the context's count (same cell layout; = set_velocities).
 * SHOCK_1D: positions inside this slab and sorted by cell (validated); the
 * cell offsets are rebuilt (count + scan on the device).  Synchronises.
 * Errors: EINVAL (bad arrays, particle outside the slab or not sorted: the
 * context then holds no particles until the next successful call, but stays
 * usable), ECAPACITY (n > capacity). */
trmcr_status trmcr_set_particles(trmcr_ctx *ctx, const void *x, const void *vx, const void *vy, const void *vz,
                                 int64_t n, int32_t host);

/* Host-buffer step for any geometry (the e2e path of the shock):
 * trmcr_set_particles(host) + one step + per-cell moments to host_moments
 * [n_cells * TRMCR_NMOMENTS].  A slab with neighbours returns EINVAL (it steps
 * with trmcr_shock_begin / exchange / trmcr_shock_finish).  Syncs. */
trmcr_status trmcr_step_host_particles(trmcr_ctx *ctx, const void *x, const void *vx, const void *vy,
                                       const void *vz, int64_t n, double *host_moments);

/* ---- 1D shock slab decomposition (multi-GPU) ----
 * Exchange buffer of `capacity` particles, trmcr_exchange_bytes() bytes, layout
 * [int32 count | pad to 16 B][capacity x][vx][vy][vz][capacity int32 global dest],
 * reals in the context dtype.  trmcr_shock_begin (reservoirs, transport, counts)
 * packs, in canonical order, the particles that moved into the left/right slab
 * into send_left/send_right; the caller moves send_left to the left rank's
 * recv_right and send_right to the right rank's recv_left (e.g. NCCL
 * send/recv on the context stream); trmcr_shock_finish merges the immigrants
 * as virtual source segments (the global canonical order of §3.3 of DESIGN.md,
 * so results do not depend on the partition) and runs the collision step.
 * Buffers are caller memory (device) and must outlive the context.
 * Errors: EINVAL (not a shock context, missing buffer for a neighbour),
 * ECAPACITY at the next sync if more than `capacity` particles emigrate or a
 * particle crosses a whole slab. */
int64_t trmcr_exchange_bytes(int32_t dtype, int64_t capacity);
/* Sort diagnostics of the last shock step (syncs): out[0] = W, a bound of the
 * cell displacement of every local particle (per transport tile: its
 * destinations against its source-cell range), out[1] = emigrant scan width, out[2] = 1
 * when the scatter sort could not be used and the collision
 * kernels gathered instead (a tile's destinations spanned more than 256 cells
 * or an edge particle landed more than 4096 cells from its edge), out[3] = 1
 * when the scatter sort is enabled for this context.  EINVAL for a
 * homogeneous context. */
trmcr_status trmcr_shock_sort_info(trmcr_ctx *ctx, int64_t *out4);
/* 1 when this shock context steps with the fused pass (transport,
 * sort and collisions in one pass over the particles, 33 B per fp32 particle
 * instead of 68; enabled at init by TRMCR_SHOCK_FUSED=1 when particles move less
 * than a cell per step, =2 always), 0 for the three-pass step (the default: it
 * is faster on B200) or a homogeneous context.  Results are
 * bitwise identical. */
int32_t trmcr_shock_fused(const trmcr_ctx *ctx);
trmcr_status trmcr_shock_set_exchange(trmcr_ctx *ctx, void *send_left, void *send_right,
                                      void *recv_left, void *recv_right, int64_t capacity);
trmcr_status trmcr_shock_begin(trmcr_ctx *ctx);
trmcr_status trmcr_shock_finish(trmcr_ctx *ctx);

/* Decision log for parity tests: capacity records (0 disables). */
trmcr_status trmcr_set_log(trmcr_ctx *ctx, int64_t capacity);
/* Copies min(count, capacity) records to host `out`, *count = records produced
 * during the last step (may exceed the capacity). Syncs. */
trmcr_status trmcr_get_log(trmcr_ctx *ctx, trmcr_coll_rec *out, int64_t *count);

/* Number of kernel launches issued by this context so far. */
int64_t trmcr_launch_count(const trmcr_ctx *ctx);

/* Per-kernel device timing (CUDA events recorded around every launch on the
 * context stream while enabled).  Kernel ids: */
enum {
  TRMCR_K_CELL_SMEM = 0, TRMCR_K_CELL_GMEM, TRMCR_K_MOMENTS, TRMCR_K_GHOST_COUNT, TRMCR_K_GHOST_GEN,
  TRMCR_K_TRANSPORT, TRMCR_K_SCAN, TRMCR_K_SHOCK_SMEM, TRMCR_K_SHOCK_GMEM, TRMCR_K_THERMAL,
  TRMCR_K_CELL_WARP, TRMCR_K_SHOCK_WARP, TRMCR_K_SCATTER, TRMCR_K_LITERAL, TRMCR_NKERNELS
};
trmcr_status trmcr_set_profiling(trmcr_ctx *ctx, int32_t on);
/* Same, restricted to the kernel ids whose bit is set in `mask` (fewer events
 * in the stream: bracket only the kernel being measured). */
trmcr_status trmcr_set_profiling_mask(trmcr_ctx *ctx, uint32_t mask);
/* Sums, per kernel id, the device time (ms) and launch count recorded since
 * the previous call (or since profiling was enabled), then resets. Syncs.
 * ms and launches are host arrays of TRMCR_NKERNELS entries. */
trmcr_status trmcr_kernel_times(trmcr_ctx *ctx, double *ms, int64_t *launches);

/* Debug builds (-DTRMCR_PHASE_TIMING) only: CTA cycles spent per phase of the
 * general kernels since the last call (16 doubles); EINVAL otherwise. */
trmcr_status trmcr_debug_phase_cycles(double *out16);

/* Last error message of ctx (or of the last failed trmcr_init when ctx is NULL). */
const char *trmcr_last_error(const trmcr_ctx *ctx);

/* Library version / build string. */
const char *trmcr_version(void);

/* Release every resource of ctx (NULL is a no-op). */
void trmcr_destroy(trmcr_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* TRMCR_H */
