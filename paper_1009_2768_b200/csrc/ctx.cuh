// ctx.cuh — host-side context of a TRMC-R simulation and shared helpers.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/trmcr.h"
#include "cell_step.cuh"
#include "cell_warp.cuh"
#include "batch.cuh"

namespace trmcr {

constexpr int kSmemThreads = 256;
constexpr int kGmemThreads = 1024;

// ---- shared-memory layout of cell_step_smem ----
struct SmemLayout {
  int n_cap, K_cap, L_cap, wb;
  size_t real_size;
  size_t off_v, off_ctype, off_crank, off_cslot, off_ints, off_rk, off_mask, off_red, off_wlen, off_wused, total;
  void build(int n, int K, int L, size_t rs, int wb_on = 0) {
    n_cap = n; K_cap = K; L_cap = L; real_size = rs; wb = wb_on;
    size_t o = 0;
    auto al = [&](size_t a) { o = (o + a - 1) / a * a; };
    off_red = o; o += 32 * 8 * sizeof(double);
    al(16); off_rk = o; o += (size_t)(L + 1) * sizeof(uint4);
    al(16); off_v = o; o += 3 * (size_t)n * rs;
    al(16); off_ctype = o; o += (size_t)K * 4;
    off_crank = o; o += (size_t)K * 4;
    off_cslot = o; o += (size_t)K * 8;
    off_ints = o; o += 6 * (size_t)(L + 1) * 4;
    off_mask = o; o += (size_t)((n + 31) / 32) * 4;
    al(16); off_wlen = o; if (wb) o += (size_t)K * 8;
    off_wused = o; if (wb) o += (size_t)K * 2;
    al(16); total = o;
  }
};

template <typename Real>
__device__ __forceinline__ void bind_smem(CellBuf<Real> &B, unsigned char *base, const SmemLayout &Lay) {
  B.red = reinterpret_cast<double *>(base + Lay.off_red);
  B.rk = reinterpret_cast<uint4 *>(base + Lay.off_rk);
  Real *v = reinterpret_cast<Real *>(base + Lay.off_v);
  B.vx = v; B.vy = v + Lay.n_cap; B.vz = v + 2 * Lay.n_cap;
  B.ctype = reinterpret_cast<uint32_t *>(base + Lay.off_ctype);
  B.crank = reinterpret_cast<uint32_t *>(base + Lay.off_crank);
  B.cslot = reinterpret_cast<uint32_t *>(base + Lay.off_cslot);
  int32_t *ints = reinterpret_cast<int32_t *>(base + Lay.off_ints);
  const int Lp = Lay.L_cap + 1;
  B.Q = ints; B.C = ints + Lp; B.S = ints + 2 * Lp; B.cons = ints + 3 * Lp;
  B.base = ints + 4 * Lp; B.cnt = ints + 5 * Lp;
  B.mask = reinterpret_cast<uint32_t *>(base + Lay.off_mask);
  B.pdom = nullptr;
  B.wlen = Lay.wb ? reinterpret_cast<double *>(base + Lay.off_wlen) : nullptr;
  B.wused = Lay.wb ? reinterpret_cast<uint8_t *>(base + Lay.off_wused) : nullptr;
  B.n_cap = Lay.n_cap; B.K_cap = Lay.K_cap; B.L_cap = Lay.L_cap;
}

struct GmemScratch {
  unsigned char *base;
  size_t stride;
  int n_cap, K_cap, L_cap, wb;
};

// Bind the plan arrays of CTA blockIdx.x to its slab of global scratch.
template <typename Real>
__device__ __forceinline__ void bind_gmem(CellBuf<Real> &B, const GmemScratch &G, double *red) {
  unsigned char *p = G.base + (size_t)blockIdx.x * G.stride;
  const int Lp = G.L_cap + 1;
  B.red = red;
  B.rk = reinterpret_cast<uint4 *>(p); p += (size_t)Lp * sizeof(uint4);
  B.ctype = reinterpret_cast<uint32_t *>(p); p += (size_t)G.K_cap * 4;
  B.crank = reinterpret_cast<uint32_t *>(p); p += (size_t)G.K_cap * 4;
  B.cslot = reinterpret_cast<uint32_t *>(p); p += (size_t)G.K_cap * 8;
  int32_t *ints = reinterpret_cast<int32_t *>(p); p += 6 * (size_t)Lp * 4;
  B.Q = ints; B.C = ints + Lp; B.S = ints + 2 * Lp; B.cons = ints + 3 * Lp;
  B.base = ints + 4 * Lp; B.cnt = ints + 5 * Lp;
  B.mask = reinterpret_cast<uint32_t *>(p); p += (size_t)((G.n_cap + 31) / 32) * 4;
  B.pdom = nullptr;
  p = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  B.wlen = G.wb ? reinterpret_cast<double *>(p) : nullptr;
  B.wused = G.wb ? reinterpret_cast<uint8_t *>(p + (size_t)G.K_cap * 8) : nullptr;
  B.n_cap = G.n_cap; B.K_cap = G.K_cap; B.L_cap = G.L_cap;
}

inline size_t gmem_stride(int n_cap, int64_t K_cap, int L_cap, int wb = 0) {
  size_t s = (size_t)(L_cap + 1) * 16 + (size_t)K_cap * 16 + 6 * (size_t)(L_cap + 1) * 4 +
             (size_t)((n_cap + 31) / 32) * 4 + 256 + (wb ? (size_t)K_cap * 10 + 16 : 0);
  return (s + 255) / 256 * 256;
}

struct QueueArgs {
  int *ovf_count;
  int *ovf_list;
  int *err;
  trmcr_coll_rec *log;
  unsigned long long *log_count;
  int64_t log_cap;
  int *zero_next;          // step-parity counter set of the next step: zeroed by block 0 (nullable)
};

// Last statement of every step kernel (late-trigger variant).
// Triggering at the end (not the start) measured faster on C3: an early
// trigger lets the successor's CTAs take SM slots while this kernel runs.
__device__ __forceinline__ void step_kernel_epilogue() {
#ifndef TRMCR_PDL_EARLY
  trmcr::pdl_trigger();
#endif
}

// First statements of every step kernel: wait for the predecessor (PDL), let
// the successor be scheduled, re-arm the next step's counters.
__device__ __forceinline__ void step_kernel_prologue(int *zero_next) {
  trmcr::pdl_wait();
#ifdef TRMCR_PDL_EARLY
  trmcr::pdl_trigger();
#endif
  if (zero_next && blockIdx.x == 0 && threadIdx.x < 4) zero_next[threadIdx.x] = 0;
}

// Shock geometry state (A1, A2): see shock.cuh.
struct ShockState {
  int C = 0, Cg = 0, cbase = 0, has_left = 0, has_right = 0;
  void *xsend[2] = {nullptr, nullptr}, *xrecv[2] = {nullptr, nullptr};   // slab exchange (caller memory)
  int xcap = 0;
  double x_min = 0, x_max = 1, inv_dx = 1, weight = 1;
  double rho[2] = {1, 1}, u[2] = {0, 0}, T[2] = {1, 1}, Lg[2] = {0, 0};
  int cap_g = 0;
  int64_t *d_off[2] = {nullptr, nullptr};   // offsets double buffer
  int32_t *d_dest = nullptr;                // [cap] destination cell (-1: left the domain)
  int32_t *d_gdest[2] = {nullptr, nullptr}; // [cap_g] per side
  void *gx[2] = {nullptr, nullptr};         // ghost positions (after transport)
  void *gv[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  int32_t *d_counts = nullptr;              // [C] particles per destination cell
  int *d_ng = nullptr;                      // [2] ghosts generated this step
  int *d_W = nullptr;                       // [3] max local displacement, emigrant scan width, scatter overflow
  int32_t *d_tileH = nullptr;               // [ntiles][kHist] destination histogram of each transport tile
  int2 *d_tile_meta = nullptr;              // [ntiles] (first histogram cell dmin, last source cell)
  int32_t *d_lcnt = nullptr;                // [kEdgeBins] left-edge (ghost + immigrant) particles per cell
  int ntiles = 0;
  int tile_ng = 4;                          // transport / sort tile = 1024 * tile_ng particles (1 or 4)
  unsigned long long *d_scan_status = nullptr;   // [ceil(C / 4096)] look-back status words of scan_offsets_lb
  uint32_t scan_epoch = 0;                  // per-call stamp of those words (30 bits used)
  int scan_lb = 1;                          // multi-CTA look-back scan (else the one-CTA scan)
  int scatter = 1;                          // sort by scatter (TRMCR_SHOCK_SCATTER=0: gather in the collide kernel)
  unsigned long long *d_acct = nullptr;     // [4] injected L, injected R, dropped, generated
  // fused step (fused.cuh): move codes of each buffer, per-cell code counts,
  // far-mover lists (parity = the buffer described)
  int fused = 0;                            // this context steps with the fused pass
  int codes_ok = 0;                         // the codes of buffer cur are current
  int8_t *d_code[2] = {nullptr, nullptr};
  int32_t *d_nlsr[2] = {nullptr, nullptr};
  int32_t *d_far_src[2] = {nullptr, nullptr}, *d_far_dst[2] = {nullptr, nullptr};
  int *d_far_cnt = nullptr;
  int far_cap = 0;
  size_t xbytes = 0;                        // bytes of one exchange buffer (library-owned buffers)
  int own_xbuf = 0;                         // the exchange buffers belong to the context (NCCL path)
};

constexpr int kCommSlots = 4;               // global-moments buffers with an all-reduce in flight

thread_local inline std::string g_init_error;

}  // namespace trmcr


// ======================================================================
// context
// ======================================================================
struct trmcr_ctx {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int dtype = TRMCR_F32, geometry = TRMCR_HOMOGENEOUS;
  size_t rs = 4;
  int64_t n = 0, cap = 0;
  int ncells = 0, cell_base = 0;
  double eps = 1, dt = 0.1;
  trmcr_kernel kern{};
  // particle state (double buffered for the shock)
  void *v[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  void *x[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t *d_offsets = nullptr;
  std::vector<int64_t> h_offsets;
  int32_t *d_mstate = nullptr;
  double *d_stats = nullptr, *d_moments = nullptr;
  int *d_ovf_count = nullptr, *d_ovf_list = nullptr, *d_err = nullptr;
  // thermal fast path (thermal.cuh): cells it defers go to the general kernel
  int *d_cnt = nullptr;            // [2][4] step-parity counter sets {defer, ovf, defer2, -}
  int use_pdl = 1;                 // programmatic dependent launch (TRMCR_PDL=0 disables)
  int *d_defer_count = nullptr, *d_defer_list = nullptr;
  int *d_defer2_count = nullptr, *d_defer2_list = nullptr;   // warp kernel -> CTA kernel
  trmcr::WarpSlabLayout wlay{};
  int warp_smem = 0, warp_grid = 1, warp_wpc = 1;
  int *h_defer = nullptr;          // pinned copy of the last defer count
  double *d_gm_partial = nullptr;  // global-moments partial sums
  unsigned *d_gm_done = nullptr;
  cudaEvent_t ev_defer = nullptr;
  int thermal_prefetch = 1;
  trmcr::BatchLayout blay{};
  int batch_grid = 0;                 // pooled-batch collision kernel (batch.cuh; 0: off)
  int lock_grid = 0, lock_smem = 0;   // shock lock-step collision kernel (0: free-running warps)   // L2 prefetch of each warp's next cell (TRMCR_THERMAL_PREFETCH=0 disables)
  int fast_ok = 1, fast_pending = 0, fast_grid = 0, smem_grid = 0, last_defer = -1, last_ovf = -1;
  unsigned char *d_scratch = nullptr;
  int literal = 0;                         // Alg 4.3/4.4 literally, one thread per cell (literal.cuh)
  uint8_t *d_lit_flag = nullptr;           // [cap] Theta membership (literal mode)
  double *d_lit_g = nullptr;               // [3 cap] Gaussian draws of Theta (literal mode)
  int giant_min = 0, giant_grid = 0;       // cells with n >= giant_min: cell_step_giant (0: off)
  trmcr::CellShared *d_gsh = nullptr;
  double *d_gpart = nullptr;
  int32_t *d_ghbuf = nullptr;
  int64_t ghcap = 0;
  trmcr::GmemScratch gs{};
  int G = 1;
  int gmem_threads = trmcr::kGmemThreads;
  int smem_threads = 128;
  trmcr::SmemLayout lay{};
  trmcr::StepParams P{};
  uint32_t step = 0;
  trmcr_coll_rec *d_log = nullptr;
  unsigned long long *d_log_count = nullptr;
  int64_t log_cap = 0;
  int64_t launches = 0;
  // per-kernel timing (trmcr_set_profiling)
  int prof = 0;
  uint32_t prof_mask = 0xFFFFFFFFu;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_kid;
  trmcr::ShockState shock{};
  // multi-GPU (comm.cuh): NCCL communicator over the ranks of one simulation
  struct ncclComm *comm = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_xchg = nullptr;   // shock slabs: emigrants packed / exchange done
  cudaEvent_t ev_comm_ready = nullptr;
  cudaEvent_t ev_comm_done[trmcr::kCommSlots] = {nullptr, nullptr, nullptr, nullptr};
  const void *comm_ptr[trmcr::kCommSlots] = {nullptr, nullptr, nullptr, nullptr};
  int comm_busy[trmcr::kCommSlots] = {0, 0, 0, 0};
  int comm_next = 0;
  std::vector<void *> allocs;
  std::string err;
  int sticky = 0;
};

namespace trmcr {

inline trmcr_status fail(trmcr_ctx *c, trmcr_status s, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (s == TRMCR_ECUDA || s == TRMCR_ENOMEM) c->sticky = 1;
  } else {
    g_init_error = msg;
  }
  return s;
}

#define CUDA_TRY(ctx, call)                                                               \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, TRMCR_ECUDA, std::string(#call " failed: ") + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
inline trmcr_status dalloc(trmcr_ctx *c, T **p, size_t bytes) {
  void *q = nullptr;
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, TRMCR_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + ") failed");
  }
  c->allocs.push_back(q);
  *p = reinterpret_cast<T *>(q);
  return TRMCR_OK;
}

// Profiling brackets around a launch: prof_begin records the start event,
// check_launch (with kid >= 0) records the stop event.
inline void prof_event(trmcr_ctx *c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  cudaEventRecord(c->ev_pool[c->ev_used++], c->stream);
}
// Kernel launch, with the programmatic-stream-serialization attribute when
// PDL is on (the kernel must begin with step_kernel_prologue / pdl_wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(const trmcr_ctx *c, void (*k)(KArgs...), dim3 grid, int block, size_t smem, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->use_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// The warp / lock-step kernels come in two instantiations: the plain one and
// the extended one (TRMC-WB and/or the majorant-update variant), so that the
// default path carries none of their code.
inline bool ext_variant(const trmcr_ctx *c) { return c->P.wb != 0 || c->P.sigma_update != 0; }

inline void prof_begin(trmcr_ctx *c, int kid) {
  if (!c->prof || !((c->prof_mask >> kid) & 1u)) return;
  c->ev_kid.push_back(kid);
  prof_event(c);
}

inline trmcr_status check_launch(trmcr_ctx *c, const char *what, int kid = -1) {
  if (c->prof && kid >= 0 && ((c->prof_mask >> kid) & 1u)) prof_event(c);
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, TRMCR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TRMCR_OK;
}

// Device-side errors corrupt or drop part of the state: they are sticky (the
// context returns TRMCR_ESTATE afterwards).
inline trmcr_status sync_check(trmcr_ctx *c) {
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  int err = 0;
  CUDA_TRY(c, cudaMemcpy(&err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err & ~12) c->sticky = 1;
  if (err & 1) return fail(c, TRMCR_ECAPACITY, "a cell's collision tree exceeded the global-memory plan capacity");
  if (err & 2) return fail(c, TRMCR_ECAPACITY, "particle capacity exceeded (shock inflow)");
  if (err & 16) return fail(c, TRMCR_ECUDA, "internal fault: tree index out of range");
  if (err & 32) return fail(c, TRMCR_ECAPACITY, "a particle crossed more than one slab in a step");
  if (err & 64) return fail(c, TRMCR_ECAPACITY, "literal mode: the trees needed more f_0 particles than the cell holds");
  if (err & 256) return fail(c, TRMCR_ECAPACITY, "a particle left its slab from more than 64 cells inside it in one step (lower dt)");
  if (err & 128) return fail(c, TRMCR_ECAPACITY, "fused shock step: too many particles moved two or more cells in one step (far-mover list full; lower dt or set TRMCR_SHOCK_FUSED=0)");
  return TRMCR_OK;
}

}  // namespace trmcr

