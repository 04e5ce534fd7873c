// trmcr.cu — kernels and host runtime behind include/trmcr.h (sm_100a).
//
// Step pipeline (homogeneous geometry), all on the context stream:
//   cell_step_smem<Real>   one CTA per cell, working set in shared memory;
//                          cells larger than n_cap, or whose tree overflows the
//                          shared-memory plan, are queued (nothing written)
//   cell_step_gmem<Real>   persistent CTAs drain that queue with the working
//                          set in global memory (L2-resident for C1/C2 sizes)
// Shock geometry adds transport/binning kernels (shock.cuh) in front.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/trmcr.h"
#include "cell_step.cuh"
#include "ctx.cuh"
#include "shock.cuh"
#include "comm.cuh"
#include "thermal.cuh"
#include "literal.cuh"

using namespace trmcr;

#define TRMCR_VERSION "trmcr 0.1 (sm_100a)"

namespace {

template <typename Real, int THREADS>
__global__ void __launch_bounds__(THREADS, 768 / THREADS)
cell_step_smem(StepParams P, SmemLayout Lay, const int64_t *__restrict__ offsets, int ncells,
               const int *list_count, const int *list, Real *vx, Real *vy, Real *vz, int32_t *m_state,
               double *stats, QueueArgs Q, GmemScratch GS, int inline_gmem) {
  step_kernel_prologue(Q.zero_next);
  BlockTeam team;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CellShared sh;
  CellBuf<Real> B;
  bind_smem(B, smem, Lay);
  const int count = list ? *list_count : ncells;
  for (int k = blockIdx.x; k < count; k += gridDim.x) {
    const int c = list ? list[k] : k;
    const int64_t off = offsets[c];
    const int n = (int)(offsets[c + 1] - off);
    const int rc = process_cell<Real, true, true>(team, P, B, sh, vx + off, vy + off, vz + off, vx + off,
                                                  vy + off, vz + off, n, P.cell_base + (uint32_t)c,
                                                  m_state + c, stats + (size_t)c * TRMCR_NSTATS, Q.log,
                                                  Q.log_count, Q.log_cap);
    if (rc != kOk && inline_gmem) {
      // single-CTA (idle) launch: redo the cell here with the global-memory
      // plan of scratch slab 0 (no separate global-memory kernel launch)
      __syncthreads();
      CellBuf<Real> BG;
      bind_gmem(BG, GS, B.red);
      BG.vx = vx + off; BG.vy = vy + off; BG.vz = vz + off;
      const int rg = process_cell<Real, false, false>(team, P, BG, sh, vx + off, vy + off, vz + off, vx + off,
                                                      vy + off, vz + off, n, P.cell_base + (uint32_t)c,
                                                      m_state + c, stats + (size_t)c * TRMCR_NSTATS, Q.log,
                                                      Q.log_count, Q.log_cap);
      if (rg != kOk && threadIdx.x == 0) atomicOr(Q.err, 1);
    } else if (rc != kOk && threadIdx.x == 0) {
      const int j = atomicAdd(Q.ovf_count, 1);
      Q.ovf_list[j] = c;
    }
    __syncthreads();
  }
  step_kernel_epilogue();
}

template <typename Real>
__global__ void __launch_bounds__(kGmemThreads)
cell_step_gmem(StepParams P, GmemScratch G, const int64_t *__restrict__ offsets, Real *vx, Real *vy,
               Real *vz, int32_t *m_state, double *stats, QueueArgs Q, int giant_min) {
  step_kernel_prologue(Q.zero_next);
  BlockTeam team;
  __shared__ CellShared sh;
  __shared__ double red[32 * 8];
  const int count = *Q.ovf_count;
  CellBuf<Real> B;
  bind_gmem(B, G, red);
  for (int k = blockIdx.x; k < count; k += gridDim.x) {
    const int c = Q.ovf_list[k];
    const int64_t off = offsets[c];
    const int n = (int)(offsets[c + 1] - off);
    if (giant_min > 0 && n >= giant_min) continue;   // cell_step_giant (whole grid) takes it
    B.vx = vx + off; B.vy = vy + off; B.vz = vz + off;
    const int rc = process_cell<Real, false, false>(team, P, B, sh, vx + off, vy + off, vz + off, vx + off,
                                             vy + off, vz + off, n, P.cell_base + (uint32_t)c,
                                             m_state + c, stats + (size_t)c * TRMCR_NSTATS, Q.log,
                                             Q.log_count, Q.log_cap);
    if (rc != kOk && threadIdx.x == 0) atomicOr(Q.err, 1);
    __syncthreads();
  }
  step_kernel_epilogue();
}


// Giant cells (n >= giant_min, e.g. config 2's single 10^6-particle cell):
// one cell at a time on the whole grid of a cooperative launch - the CTA step
// code with a GridTeam (grid barriers, two-level deterministic reductions,
// the cell's plan in global scratch slab 0, its shared scalars in global memory).
constexpr int kGiantThreads = 256;
template <typename Real>
__global__ void __launch_bounds__(kGiantThreads)
cell_step_giant(StepParams P, GmemScratch G, CellShared *gsh, double *part, int32_t *hbuf, int64_t hcap,
                const int64_t *__restrict__ offsets, Real *vx, Real *vy, Real *vz, int32_t *m_state,
                double *stats, QueueArgs Q, int giant_min) {
  GridTeam team{part, hbuf, hcap, 0};
  __shared__ double red[32 * 8];
  CellBuf<Real> B;
  G.stride = 0;                                   // every block binds the same plan slab
  bind_gmem(B, G, red);
  const int count = *Q.ovf_count;
  for (int k = 0; k < count; ++k) {
    const int c = Q.ovf_list[k];
    const int64_t off = offsets[c];
    const int n = (int)(offsets[c + 1] - off);
    if (n < giant_min) continue;
    B.vx = vx + off; B.vy = vy + off; B.vz = vz + off;
    const int rc = process_cell<Real, false, false>(team, P, B, *gsh, vx + off, vy + off, vz + off, vx + off,
                                                    vy + off, vz + off, n, P.cell_base + (uint32_t)c,
                                                    m_state + c, stats + (size_t)c * TRMCR_NSTATS, Q.log,
                                                    Q.log_count, Q.log_cap);
    if (rc != kOk && team.tid() == 0) atomicOr(Q.err, 1);
    team.sync();
  }
}

// General cells, one warp each (cell_warp.cuh), over the thermal kernel's
// defer list (or every cell); cells that do not fit go to list2 (CTA kernel).
template <typename Real, bool WB, int MOD = -1>
__global__ void __launch_bounds__(kWarpCellWarps * 32, TRMCR_WARP_MINB)
cell_step_warp(StepParams P, WarpSlabLayout Lay, const int64_t *__restrict__ offsets, int ncells,
               const int *list_count, const int *list, Real *vx, Real *vy, Real *vz, int32_t *m_state,
               double *stats, int *list2_count, int *list2, QueueArgs Q) {
  step_kernel_prologue(Q.zero_next);
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *slab = smem + (size_t)warp * Lay.per_warp;
  WarpShared &sh = *reinterpret_cast<WarpShared *>(slab + Lay.off_sh);
  CellBuf<Real> B;
  double *usplit;
  bind_warp_slab(B, slab, Lay, usplit);
  const int count = list ? *list_count : ncells;
  const int nw = gridDim.x * (blockDim.x >> 5);
  for (int k = blockIdx.x * (blockDim.x >> 5) + warp; k < count; k += nw) {
    const int c = list ? list[k] : k;
    const int64_t off = offsets[c];
    const int n = (int)(offsets[c + 1] - off);
    int rc = kOverflow;
    if (n > 0 && n <= Lay.n_cap) {
      double sx = 0, sy = 0, sz = 0;
      warp_cell_fori<Real>(vx + off, vy + off, vz + off, n, [&](int i, Real a, Real b, Real d) {
        B.vx[i] = a; B.vy[i] = b; B.vz[i] = d;
        sx += a; sy += b; sz += d;
      });
      __syncwarp();
      rc = process_cell_warp<Real, WB, MOD>(P, B, sh, usplit, sx, sy, sz, vx + off, vy + off, vz + off, n,
                                   P.cell_base + (uint32_t)c, m_state + c, stats + (size_t)c * TRMCR_NSTATS,
                                   Q.log, Q.log_count, Q.log_cap);
    }
    if (rc != kOk && lane == 0) list2[atomicAdd(list2_count, 1)] = c;
    __syncwarp();
  }
  step_kernel_epilogue();
}

// A9: per-cell moments, one warp per cell (two passes: the second reads the
// cell from L1), fp64 sums of the lane partials.
constexpr int kMomWarps = 8;
template <typename Real>
__global__ void __launch_bounds__(kMomWarps * 32)
moments_kernel(const int64_t *__restrict__ offsets, int ncells, const Real *__restrict__ vx,
               const Real *__restrict__ vy, const Real *__restrict__ vz,
               const int32_t *__restrict__ m_state, int shock, double w_over_dx, double *out) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * kMomWarps + (threadIdx.x >> 5);
  if (c >= ncells) return;
  const int64_t off = offsets[c];
  const int n = (int)(offsets[c + 1] - off);
  const Real *X = vx + off, *Y = vy + off, *Z = vz + off;
  double s0 = 0, s1 = 0, s2 = 0;
  warp_cell_for<Real>(X, Y, Z, n, [&](Real x, Real y, Real z) { s0 += (double)x; s1 += (double)y; s2 += (double)z; });
  s0 = warp_sum(s0); s1 = warp_sum(s1); s2 = warp_sum(s2);
  const double ux = n ? s0 / n : 0.0, uy = n ? s1 / n : 0.0, uz = n ? s2 / n : 0.0;
  double t0 = 0, t1 = 0, t2 = 0, t3 = 0;
  warp_cell_for<Real>(X, Y, Z, n, [&](Real xr, Real yr, Real zr) {
    const double x = xr, y = yr, z = zr;
    const double dx = x - ux, dy = y - uy, dz = z - uz;
    const double c2 = dx * dx + dy * dy + dz * dz, v2 = x * x + y * y + z * z;
    t0 += c2; t1 += dx * dx; t2 += v2 * v2; t3 += c2 * c2;
  });
  t0 = warp_sum(t0); t1 = warp_sum(t1); t2 = warp_sum(t2); t3 = warp_sum(t3);
  if (lane == 0) {
    double *r = out + (size_t)c * TRMCR_NMOMENTS;
    const double rho = shock ? n * w_over_dx : 1.0;
    const double T = n ? t0 / (3.0 * n) : 0.0;
    r[TRMCR_MO_N] = n; r[TRMCR_MO_RHO] = rho;
    r[TRMCR_MO_UX] = ux; r[TRMCR_MO_UY] = uy; r[TRMCR_MO_UZ] = uz; r[TRMCR_MO_T] = T;
    r[TRMCR_MO_E] = 0.5 * rho * (ux * ux + uy * uy + uz * uz + 3.0 * T);
    r[TRMCR_MO_P] = rho * T;
    r[TRMCR_MO_PXX] = n ? t1 / n : 0.0;
    r[TRMCR_MO_M4] = n ? t2 / n : 0.0;
    r[TRMCR_MO_M4C] = n ? t3 / n : 0.0;
    r[TRMCR_MO_MMAX] = m_state[c];
  }
}

// Global sums of the per-cell statistics rows: kGmBlocks CTAs of kGmThreads
// write partial sums of contiguous cell ranges (one row per thread per round,
// warp sums then the CTA's warps in order), the last CTA to finish adds the
// partials in block order with one warp (deterministic), writes `out` and
// re-arms the counter.  Few, wide CTAs: the kernel is a short latency chain.
#ifndef TRMCR_GM_BLOCKS
#define TRMCR_GM_BLOCKS 64
#endif
#ifndef TRMCR_GM_THREADS
#define TRMCR_GM_THREADS 256     // C3 step (blocks x threads): 64 x 512 0.1055 ms, 64 x 256 0.1032, 128 x 128 0.1033, 32 x 512 0.1035, 16 x 1024 0.1054
#endif
constexpr int kGmBlocks = TRMCR_GM_BLOCKS, kGmThreads = TRMCR_GM_THREADS;
__global__ void __launch_bounds__(kGmThreads) global_moments_kernel(const double *__restrict__ stats, int ncells,
                                                                    double *partial, unsigned *done, double *out) {
  step_kernel_prologue(nullptr);
  constexpr int NW = kGmThreads / 32, NV = 9;
  __shared__ double red[NW][NV];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int per = (ncells + gridDim.x - 1) / gridDim.x;
  const int lo = blockIdx.x * per, hi = min(ncells, lo + per);
  double v[NV] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    const double *r = stats + (size_t)c * TRMCR_NSTATS;
    const double n = r[TRMCR_ST_N];
    v[0] += n; v[1] += r[TRMCR_ST_PX]; v[2] += r[TRMCR_ST_PY]; v[3] += r[TRMCR_ST_PZ];
    v[4] += r[TRMCR_ST_ENERGY]; v[5] += n * r[TRMCR_ST_S0];
    v[6] += r[TRMCR_ST_PROPOSALS]; v[7] += r[TRMCR_ST_ACCEPTED]; v[8] += r[TRMCR_ST_MAXW];
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[warp][k] = v[k];
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    if (lane < NV)
      for (int w = 0; w < NW; ++w) t += red[w][lane];
    if (lane < NV) partial[blockIdx.x * 10 + lane] = t;
    __threadfence();
    __syncwarp();
    if (lane == 0) last = (atomicAdd(done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last && warp == 0) {         // uniform per CTA: the last CTA adds the partials
    __threadfence();
    double w[NV] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = lane; b < (int)gridDim.x; b += 32)
#pragma unroll
      for (int k = 0; k < NV; ++k) w[k] += ((volatile double *)partial)[b * 10 + k];
#pragma unroll
    for (int k = 0; k < NV; ++k) w[k] = warp_sum(w[k]);
    if (lane == 0) {
      for (int k = 0; k < NV; ++k) out[k] = w[k];
      out[TRMCR_GM_COST] = w[TRMCR_GM_PROPOSALS] + 0.5 * w[TRMCR_GM_MAXW];
      *done = 0u;
    }
  }
  step_kernel_epilogue();
}

__global__ void fill_i32(int32_t *a, int n, int32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

}  // namespace

namespace {


template <typename Real>
trmcr_status launch_collide(trmcr_ctx *c) {
  Real *vx = (Real *)c->v[c->cur][0], *vy = (Real *)c->v[c->cur][1], *vz = (Real *)c->v[c->cur][2];
  // step-parity counter sets: this step's are zero (re-armed by the previous
  // step's kernels, or at init); this step's kernels re-arm the other set
  int *cnt = c->d_cnt + 4 * (c->step & 1), *nxt = c->d_cnt + 4 * ((c->step + 1) & 1);
  c->d_defer_count = cnt; c->d_ovf_count = cnt + 1; c->d_defer2_count = cnt + 2;
  QueueArgs Q{c->d_ovf_count, c->d_ovf_list, c->d_err, c->d_log, c->d_log_count, c->log_cap, nxt};
  c->P.step = c->step;
  if (c->literal) {   // the paper's layout: Alg 4.3/4.4 literally, one thread per cell
    if (c->ncells == 0) return TRMCR_OK;
    prof_begin(c, TRMCR_K_LITERAL);
    literal_step_kernel<Real><<<(c->ncells + kLitThreads - 1) / kLitThreads, kLitThreads, 0, c->stream>>>(
        c->P, c->d_offsets, c->ncells, vx, vy, vz, c->d_stats, c->d_lit_flag, c->d_lit_g);
    return check_launch(c, "literal_step_kernel", TRMCR_K_LITERAL);
  }
  if (c->ncells > 0) {
    // Counts of the last observed step (pinned async copy, read when ready):
    // the thermal fast path runs while it handles most cells (re-tried every
    // 16 steps); when nothing was deferred the general kernels are launched
    // with one CTA (they still drain whatever this step queues: correct, and
    // re-sized once the counts are seen).
    if (c->fast_pending && cudaEventQuery(c->ev_defer) == cudaSuccess) {
      c->fast_ok = (c->h_defer[0] <= c->ncells / 2);
      c->last_defer = c->h_defer[0];
      c->last_ovf = c->h_defer[1];
      c->fast_pending = 0;
    } else if (c->fast_pending) {
      cudaGetLastError();   // cudaErrorNotReady is not an error here
    }
    const bool fast = c->fast_ok || (c->step % 16 == 0);
    if (fast) {
      prof_begin(c, TRMCR_K_THERMAL);
      KeySched ks;
      for (int r = 0; r < 10; ++r) {
        ks.k0[r] = c->P.k0 + (uint32_t)r * 0x9E3779B9u;
        ks.k1[r] = c->P.k1 + (uint32_t)r * 0xBB67AE85u;
      }
      launch_k(c, thermal_warp_kernel<Real>, c->fast_grid, kThermalWarps * 32,
               kThermalWarps * 3 * ThermalCap<Real>::value * sizeof(Real), c->P, ks, (const int64_t *)c->d_offsets,
               c->ncells, vx, vy, vz, c->d_mstate, c->d_stats, c->d_defer_count, c->d_defer_list,
               c->thermal_prefetch, nxt);
      if (auto s = check_launch(c, "thermal_warp_kernel", TRMCR_K_THERMAL)) return s;
    }
    const bool idle = fast && c->fast_ok && c->last_defer == 0 && c->last_ovf == 0 && c->giant_min == 0;
    // idle (nothing deferred lately): skip the warp kernel, the CTA kernel
    // (one CTA) drains whatever this step defers
    const bool use_warp = c->wlay.n_cap > 0 && !idle;
    const int *l1c = fast ? c->d_defer_count : nullptr, *l1 = fast ? c->d_defer_list : nullptr;
    if (use_warp) {
      prof_begin(c, TRMCR_K_CELL_WARP);
      launch_k(c, ext_variant(c) ? cell_step_warp<Real, true>
                                 : (c->P.model == TRMCR_HARD_SPHERE ? cell_step_warp<Real, false, TRMCR_HARD_SPHERE>
                                                                    : cell_step_warp<Real, false>),
               idle ? 1 : c->warp_grid, c->warp_wpc * 32, (size_t)c->warp_smem, c->P,
               c->wlay, (const int64_t *)c->d_offsets, c->ncells, l1c, l1, vx, vy, vz, c->d_mstate, c->d_stats,
               c->d_defer2_count, c->d_defer2_list, Q);
      if (auto s = check_launch(c, "cell_step_warp", TRMCR_K_CELL_WARP)) return s;
      l1c = c->d_defer2_count;
      l1 = c->d_defer2_list;
    }
    prof_begin(c, TRMCR_K_CELL_SMEM);
    auto kern = c->smem_threads == 64 ? cell_step_smem<Real, 64>
                : (c->smem_threads == 128 ? cell_step_smem<Real, 128> : cell_step_smem<Real, 256>);
    launch_k(c, kern, idle ? 1 : c->smem_grid, c->smem_threads, (size_t)c->lay.total, c->P, c->lay,
             (const int64_t *)c->d_offsets, c->ncells, l1c, l1, vx, vy, vz, c->d_mstate, c->d_stats, Q, c->gs,
             idle ? 1 : 0);
    if (auto s = check_launch(c, "cell_step_smem", TRMCR_K_CELL_SMEM)) return s;
    if (!idle) {   // idle: the single CTA above handled overflowing cells itself
      prof_begin(c, TRMCR_K_CELL_GMEM);
      launch_k(c, cell_step_gmem<Real>, c->G, c->gmem_threads, 0, c->P, c->gs, (const int64_t *)c->d_offsets, vx,
               vy, vz, c->d_mstate, c->d_stats, Q, c->giant_min);
      if (auto s = check_launch(c, "cell_step_gmem", TRMCR_K_CELL_GMEM)) return s;
      if (c->giant_min > 0) {
        StepParams Pg = c->P;
        GmemScratch gs = c->gs;
        CellShared *gsh = c->d_gsh;
        double *gpart = c->d_gpart;
        int32_t *ghb = c->d_ghbuf;
        int64_t ghc = c->ghcap;
        const int64_t *offs = c->d_offsets;
        int32_t *ms = c->d_mstate;
        double *st = c->d_stats;
        int gmin = c->giant_min;
        void *args[] = {&Pg, &gs, &gsh, &gpart, &ghb, &ghc, &offs, &vx, &vy, &vz, &ms, &st, &Q, &gmin};
        CUDA_TRY(c, cudaLaunchCooperativeKernel((const void *)cell_step_giant<Real>, dim3(c->giant_grid),
                                                dim3(kGiantThreads), args, 0, c->stream));
        if (auto s = check_launch(c, "cell_step_giant", TRMCR_K_CELL_GMEM)) return s;
      }
    }
    // sample the counts only of a step that ran the thermal kernel (otherwise
    // nothing was deferred to count, and a zero would read as "all thermal")
    if (!c->fast_pending && fast && (c->step % 8 == 0 || !c->fast_ok)) {
      CUDA_TRY(c, cudaMemcpyAsync(c->h_defer, c->d_defer_count, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaEventRecord(c->ev_defer, c->stream));
      c->fast_pending = 1;
    }
  }
  return TRMCR_OK;
}

template <typename Real>
trmcr_status launch_moments(trmcr_ctx *c) {
  if (c->ncells == 0) return TRMCR_OK;
  prof_begin(c, TRMCR_K_MOMENTS);
  moments_kernel<Real><<<(c->ncells + kMomWarps - 1) / kMomWarps, kMomWarps * 32, 0, c->stream>>>(
      c->d_offsets, c->ncells, (const Real *)c->v[c->cur][0], (const Real *)c->v[c->cur][1],
      (const Real *)c->v[c->cur][2], c->d_mstate, c->P.shock, c->P.w_over_dx, c->d_moments);
  return check_launch(c, "moments_kernel", TRMCR_K_MOMENTS);
}

// Allow the device maximum of dynamic shared memory (minus the kernel's static
// shared memory): the attribute is per function and process-wide.
cudaError_t allow_max_dyn_smem(const void *f, int smem_optin) {
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, f);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - (int)a.sharedSizeBytes);
}

trmcr_status do_step(trmcr_ctx *c) {
  const bool slab = c->geometry == TRMCR_SHOCK_1D && (c->shock.has_left || c->shock.has_right);
  if (slab && !c->comm)
    return fail(c, TRMCR_EINVAL, "a slab with neighbours steps with trmcr_shock_begin / exchange / trmcr_shock_finish "
                                 "(or give trmcr_init an NCCL id)");
  if (c->log_cap > 0)
    CUDA_TRY(c, cudaMemsetAsync(c->d_log_count, 0, sizeof(unsigned long long), c->stream));
  trmcr_status s;
  if (slab) {                        // begin, NCCL neighbour exchange on the context stream, finish
    s = c->dtype == TRMCR_F64 ? shock_begin<double>(c) : shock_begin<float>(c);
    if (!s) s = comm_shock_exchange(c);
    if (!s) s = c->dtype == TRMCR_F64 ? shock_finish<double>(c) : shock_finish<float>(c);
  } else if (c->geometry == TRMCR_SHOCK_1D)
    s = c->dtype == TRMCR_F64 ? shock_step<double>(c) : shock_step<float>(c);
  else
    s = c->dtype == TRMCR_F64 ? launch_collide<double>(c) : launch_collide<float>(c);
  if (s) return s;
  c->step++;
  return TRMCR_OK;
}

}  // namespace

// ======================================================================
// ABI
// ======================================================================
extern "C" {

const char *trmcr_version(void) { return TRMCR_VERSION; }

const char *trmcr_last_error(const trmcr_ctx *ctx) {
  return ctx ? ctx->err.c_str() : g_init_error.c_str();
}

int64_t trmcr_launch_count(const trmcr_ctx *ctx) { return ctx ? ctx->launches : 0; }

trmcr_status trmcr_global_moments(trmcr_ctx *c, double *dev_out, int32_t all_ranks) {
  if (!c || !dev_out) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  const bool ar = all_ranks && c->comm;
  int slot = -1;
  if (ar) {                 // the buffer's previous all-reduce must be done before it is rewritten
    slot = comm_slot(c, dev_out);
    if (c->comm_busy[slot]) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_comm_done[slot], 0));
  }
  const int blocks = std::max(1, std::min(kGmBlocks, c->ncells));
  launch_k(c, global_moments_kernel, blocks, kGmThreads, 0, (const double *)c->d_stats, c->ncells, c->d_gm_partial,
           c->d_gm_done, dev_out);
  if (trmcr_status e = check_launch(c, "global_moments_kernel")) return e;
  if (ar) {                 // all-reduce on the communication stream, overlapping the next step
    CUDA_TRY(c, cudaEventRecord(c->ev_comm_ready, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_comm_ready, 0));
    NCCL_TRY(c, ncclAllReduce(dev_out, dev_out, TRMCR_NGLOBAL, ncclDouble, ncclSum, c->comm, c->comm_stream));
    CUDA_TRY(c, cudaEventRecord(c->ev_comm_done[slot], c->comm_stream));
    c->comm_busy[slot] = 1;
  }
  return TRMCR_OK;
}

trmcr_status trmcr_comm_wait(trmcr_ctx *c) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  for (int k = 0; k < kCommSlots; ++k)
    if (c->comm_busy[k]) {
      CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_comm_done[k], 0));
      c->comm_busy[k] = 0;
    }
  return TRMCR_OK;
}

trmcr_status trmcr_get_nccl_id(void *out128) {
  if (!out128) return fail(nullptr, TRMCR_EINVAL, "null argument");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, TRMCR_ENCCL, std::string("ncclGetUniqueId failed: ") + ncclGetErrorString(r));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  memcpy(out128, &id, sizeof(id));
  return TRMCR_OK;
}

int32_t trmcr_comm_size(const trmcr_ctx *c) { return c ? c->nranks : 0; }

trmcr_status trmcr_global_sums(trmcr_ctx *c, double *host_out) {
  if (!c || !host_out) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  if (trmcr_status s = sync_check(c)) return s;
  // per-cell rows of the summed quantities (the statistics rows of the last step)
  std::vector<double> st((size_t)c->ncells * TRMCR_NSTATS), rows((size_t)c->ncells * TRMCR_NGLOBAL);
  CUDA_TRY(c, cudaMemcpy(st.data(), c->d_stats, sizeof(double) * st.size(), cudaMemcpyDeviceToHost));
  for (int i = 0; i < c->ncells; ++i) {
    const double *r = &st[(size_t)i * TRMCR_NSTATS];
    double *o = &rows[(size_t)i * TRMCR_NGLOBAL];
    o[TRMCR_GM_N] = r[TRMCR_ST_N]; o[TRMCR_GM_PX] = r[TRMCR_ST_PX]; o[TRMCR_GM_PY] = r[TRMCR_ST_PY];
    o[TRMCR_GM_PZ] = r[TRMCR_ST_PZ]; o[TRMCR_GM_ENERGY] = r[TRMCR_ST_ENERGY];
    o[TRMCR_GM_NPXX] = r[TRMCR_ST_N] * r[TRMCR_ST_S0];
    o[TRMCR_GM_PROPOSALS] = r[TRMCR_ST_PROPOSALS]; o[TRMCR_GM_ACCEPTED] = r[TRMCR_ST_ACCEPTED];
    o[TRMCR_GM_MAXW] = r[TRMCR_ST_MAXW];
    o[TRMCR_GM_COST] = r[TRMCR_ST_PROPOSALS] + 0.5 * r[TRMCR_ST_MAXW];
  }
  double *d_rows = nullptr;
  if (dalloc(c, &d_rows, sizeof(double) * std::max<size_t>(rows.size(), 1))) return TRMCR_ENOMEM;
  CUDA_TRY(c, cudaMemcpy(d_rows, rows.data(), sizeof(double) * rows.size(), cudaMemcpyHostToDevice));
  std::vector<double> all;
  int64_t total = 0;
  trmcr_status s = comm_allgather_rows(c, d_rows, TRMCR_NGLOBAL, all, total);
  c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void *)d_rows), c->allocs.end());
  cudaFree(d_rows);
  if (s) return s;
  for (int k = 0; k < TRMCR_NGLOBAL; ++k) host_out[k] = exact_sum(all.data() + k, (size_t)total, TRMCR_NGLOBAL);
  return TRMCR_OK;
}

// Debug builds only: per-phase CTA cycles of the general kernels (reset on read).
trmcr_status trmcr_debug_phase_cycles(double *out16) {
#ifdef TRMCR_PHASE_TIMING
  unsigned long long h[16];
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(h, g_phase_cycles, sizeof(h));
  for (int k = 0; k < 16; ++k) out16[k] = (double)h[k];
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  return TRMCR_OK;
#else
  (void)out16;
  return TRMCR_EINVAL;
#endif
}

trmcr_status trmcr_set_profiling(trmcr_ctx *c, int32_t on) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->prof = on ? 1 : 0;
  c->prof_mask = 0xFFFFFFFFu;
  c->ev_used = 0;
  c->ev_kid.clear();
  return TRMCR_OK;
}

trmcr_status trmcr_set_profiling_mask(trmcr_ctx *c, uint32_t mask) {
  if (trmcr_status s = trmcr_set_profiling(c, mask != 0)) return s;
  c->prof_mask = mask;
  return TRMCR_OK;
}

trmcr_status trmcr_kernel_times(trmcr_ctx *c, double *ms, int64_t *launches) {
  if (!c || !ms || !launches) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int k = 0; k < TRMCR_NKERNELS; ++k) { ms[k] = 0.0; launches[k] = 0; }
  for (size_t i = 0; i < c->ev_kid.size(); ++i) {
    float t = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&t, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
    ms[c->ev_kid[i]] += t;
    launches[c->ev_kid[i]] += 1;
  }
  c->ev_used = 0;
  c->ev_kid.clear();
  return TRMCR_OK;
}

void trmcr_destroy(trmcr_ctx *ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
  comm_destroy(ctx);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ev_defer) cudaEventDestroy(ctx->ev_defer);
  if (ctx->h_defer) cudaFreeHost(ctx->h_defer);
  for (void *p : ctx->allocs) cudaFree(p);
  delete ctx;
}

trmcr_status trmcr_init(trmcr_ctx **out, const trmcr_particles *pp, const trmcr_cells *cc, double eps,
                        double dt, const trmcr_kernel *kk, void *cuda_stream, const void *nccl_id, int32_t rank,
                        int32_t nranks) {
  if (!out || !pp || !cc || !kk) return fail(nullptr, TRMCR_EINVAL, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(nullptr, TRMCR_EINVAL, "need 0 <= rank < nranks");
  if (!(eps > 0) || !(dt > 0)) return fail(nullptr, TRMCR_EINVAL, "eps and dt must be > 0");
  if (pp->dtype != TRMCR_F32 && pp->dtype != TRMCR_F64) return fail(nullptr, TRMCR_EINVAL, "bad dtype");
  if (pp->n < 0 || pp->n > 0x7FFFFFFFLL) return fail(nullptr, TRMCR_EINVAL, "bad particle count");
  if (pp->n > 0 && (!pp->vx || !pp->vy || !pp->vz)) return fail(nullptr, TRMCR_EINVAL, "null velocity pointer");
  if (kk->model != TRMCR_MAXWELL && kk->model != TRMCR_HARD_SPHERE && kk->model != TRMCR_VHS)
    return fail(nullptr, TRMCR_EINVAL, "bad model");
  if (kk->model == TRMCR_VHS && !(kk->alpha >= 0.0 && kk->alpha <= 1.0))
    return fail(nullptr, TRMCR_EINVAL, "VHS alpha must lie in [0, 1]");
  if (kk->wb < 0 || kk->wb > 3 || (kk->wb && (kk->adaptive || kk->wb_max < 0)))
    return fail(nullptr, TRMCR_EINVAL, "TRMC-WB: wb in 0..3, wb_max >= 0, not with adaptive (RAD)");
  if (kk->indicator != TRMCR_IND_PXX && kk->indicator != TRMCR_IND_M4) return fail(nullptr, TRMCR_EINVAL, "bad indicator");
  if (kk->literal && (kk->adaptive || kk->wb || cc->geometry != TRMCR_HOMOGENEOUS || kk->m_fixed < 1 ||
                      kk->m_fixed > kLitMaxLevel))
    return fail(nullptr, TRMCR_EINVAL, "literal mode: homogeneous cells, fixed 1 <= m <= 128, no RAD, no TRMC-WB");
  if (kk->adaptive) {
    if (kk->m_init < 1 || kk->m_cap < kk->m_init || kk->m_cap > 16384)
      return fail(nullptr, TRMCR_EINVAL, "need 1 <= m_init <= m_cap <= 16384");
    if (!(kk->delta1 > 0) || !(kk->delta1 < kk->delta2)) return fail(nullptr, TRMCR_EINVAL, "need 0 < delta1 < delta2");
  } else if (kk->m_fixed < 0 || kk->m_fixed > 16384) {
    return fail(nullptr, TRMCR_EINVAL, "need 0 <= m_fixed <= 16384");
  }
  if (cc->geometry != TRMCR_HOMOGENEOUS && cc->geometry != TRMCR_SHOCK_1D)
    return fail(nullptr, TRMCR_EINVAL, "bad geometry");
  if (cc->n_cells < 0 || cc->cell_base < 0) return fail(nullptr, TRMCR_EINVAL, "bad cell count");

  trmcr_ctx *c = new trmcr_ctx();
  c->stream = (cudaStream_t)cuda_stream;
  cudaGetDevice(&c->dev);
  c->dtype = pp->dtype;
  c->rs = pp->dtype == TRMCR_F64 ? 8 : 4;
  c->geometry = cc->geometry;
  c->n = pp->n;
  c->ncells = cc->n_cells;
  c->cell_base = cc->cell_base;
  c->eps = eps; c->dt = dt; c->kern = *kk;
  auto bail = [&](trmcr_status s) { g_init_error = c->err; trmcr_destroy(c); return s; };

  int max_cell = 0;
  if (c->geometry == TRMCR_HOMOGENEOUS) {
    if (!cc->offsets) { fail(c, TRMCR_EINVAL, "homogeneous geometry needs offsets"); return bail(TRMCR_EINVAL); }
    c->h_offsets.assign(cc->offsets, cc->offsets + c->ncells + 1);
    if (c->h_offsets[0] != 0 || c->h_offsets[c->ncells] != c->n) {
      fail(c, TRMCR_EINVAL, "offsets must start at 0 and end at n");
      return bail(TRMCR_EINVAL);
    }
    for (int i = 0; i < c->ncells; ++i) {
      const int64_t d = c->h_offsets[i + 1] - c->h_offsets[i];
      if (d < 0) { fail(c, TRMCR_EINVAL, "offsets not monotone"); return bail(TRMCR_EINVAL); }
      max_cell = (int)std::max<int64_t>(max_cell, d);
    }
    c->cap = c->n;
  } else {
    if (cc->offsets) { fail(c, TRMCR_EINVAL, "shock geometry takes no offsets"); return bail(TRMCR_EINVAL); }
    if (!pp->x && pp->n > 0) { fail(c, TRMCR_EINVAL, "shock geometry needs positions"); return bail(TRMCR_EINVAL); }
    if (!(cc->x_max > cc->x_min) || !(cc->weight > 0) || c->ncells < 1) {
      fail(c, TRMCR_EINVAL, "bad shock domain");
      return bail(TRMCR_EINVAL);
    }
    if (!(cc->rho_L > 0) || !(cc->rho_R > 0) || !(cc->T_L > 0) || !(cc->T_R > 0)) {
      fail(c, TRMCR_EINVAL, "reservoir states need rho, T > 0");
      return bail(TRMCR_EINVAL);
    }
    c->cap = pp->capacity > 0 ? pp->capacity : c->n + c->n / 4 + 65536;
    if (c->cap < c->n || c->cap > 0x7FFFFFFFLL) { fail(c, TRMCR_EINVAL, "bad capacity"); return bail(TRMCR_EINVAL); }
  }

  // ---- parameters ----
  StepParams &P = c->P;
  P.model = kk->model; P.alpha = kk->model == TRMCR_VHS ? kk->alpha : (kk->model == TRMCR_HARD_SPHERE ? 1.0 : 0.0);
  P.adaptive = kk->adaptive;
  P.wb = kk->wb; P.wb_max = kk->wb_max; P.sigma_update = kk->sigma_update != 0 && kk->model != TRMCR_MAXWELL; P.m_fixed = kk->m_fixed; P.m_cap = kk->m_cap;
  P.indicator = kk->indicator; P.log_on = 0;
  P.delta1 = kk->delta1; P.delta2 = kk->delta2; P.dt = dt; P.eps = eps;
  P.k0 = (uint32_t)kk->seed; P.k1 = (uint32_t)(kk->seed >> 32);
  P.step = 0; P.cell_base = (uint32_t)cc->cell_base;
  P.shock = c->geometry == TRMCR_SHOCK_1D;
  P.err = nullptr;   // set once d_err exists
  P.debug_stop = getenv("TRMCR_DEBUG_STOP") ? atoi(getenv("TRMCR_DEBUG_STOP")) : 0;
  P.w_over_dx = P.shock ? cc->weight / ((cc->x_max - cc->x_min) /
                                        (cc->n_cells_global > 0 ? cc->n_cells_global : cc->n_cells))
                        : 0.0;

  // ---- buffers ----
  const int nbuf = c->geometry == TRMCR_SHOCK_1D ? 2 : 1;
  for (int b = 0; b < nbuf; ++b) {
    for (int k = 0; k < 3; ++k)
      if (dalloc(c, &c->v[b][k], (size_t)c->cap * c->rs)) return bail(TRMCR_ENOMEM);
    if (c->geometry == TRMCR_SHOCK_1D && dalloc(c, &c->x[b], (size_t)c->cap * c->rs)) return bail(TRMCR_ENOMEM);
  }
  if (dalloc(c, &c->d_offsets, sizeof(int64_t) * (c->ncells + 1)) ||
      dalloc(c, &c->d_mstate, sizeof(int32_t) * std::max(c->ncells, 1)) ||
      dalloc(c, &c->d_stats, sizeof(double) * TRMCR_NSTATS * std::max(c->ncells, 1)) ||
      dalloc(c, &c->d_moments, sizeof(double) * TRMCR_NMOMENTS * std::max(c->ncells, 1)) ||

      dalloc(c, &c->d_ovf_list, sizeof(int) * std::max(c->ncells, 1)) ||
      dalloc(c, &c->d_err, sizeof(int)) || dalloc(c, &c->d_log_count, sizeof(unsigned long long)) ||
      dalloc(c, &c->d_cnt, 8 * sizeof(int)) ||
      dalloc(c, &c->d_defer2_list, sizeof(int) * std::max(c->ncells, 1)) || dalloc(c, &c->d_gm_partial, sizeof(double) * 10 * kGmBlocks) ||
      dalloc(c, &c->d_gm_done, sizeof(unsigned)) || dalloc(c, &c->d_defer_list, sizeof(int) * std::max(c->ncells, 1)))
    return bail(TRMCR_ENOMEM);
  c->literal = kk->literal != 0;
  if (c->literal && (dalloc(c, &c->d_lit_flag, (size_t)c->cap) || dalloc(c, &c->d_lit_g, sizeof(double) * 3 * (size_t)c->cap)))
    return bail(TRMCR_ENOMEM);
  c->d_defer_count = c->d_cnt; c->d_ovf_count = c->d_cnt + 1; c->d_defer2_count = c->d_cnt + 2;
  if (const char *pe = getenv("TRMCR_PDL")) c->use_pdl = atoi(pe) != 0;
  if (cudaMallocHost(&c->h_defer, 2 * sizeof(int)) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_defer, cudaEventDisableTiming) != cudaSuccess) {
    fail(c, TRMCR_ENOMEM, "pinned host / event allocation failed");
    return bail(TRMCR_ENOMEM);
  }
  c->h_defer[0] = c->h_defer[1] = 0;
  c->last_defer = c->last_ovf = -1;
  c->P.err = c->d_err;
  if (cudaMemsetAsync(c->d_gm_done, 0, sizeof(unsigned), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->d_err, 0, sizeof(int), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->d_cnt, 0, 8 * sizeof(int), c->stream) != cudaSuccess ||
      cudaMemsetAsync(c->d_stats, 0, sizeof(double) * TRMCR_NSTATS * std::max(c->ncells, 1), c->stream) != cudaSuccess) {
    fail(c, TRMCR_ECUDA, "memset failed");
    return bail(TRMCR_ECUDA);
  }
  const int m0 = kk->adaptive ? kk->m_init : kk->m_fixed;
  if (c->ncells > 0) {
    fill_i32<<<(c->ncells + 255) / 256, 256, 0, c->stream>>>(c->d_mstate, c->ncells, m0);
    if (check_launch(c, "fill_i32")) return bail(TRMCR_ECUDA);
  }

  // ---- copy particles in ----
  const cudaMemcpyKind kind = pp->host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const void *src[3] = {pp->vx, pp->vy, pp->vz};
  for (int k = 0; k < 3 && c->n > 0; ++k)
    if (cudaMemcpyAsync(c->v[0][k], src[k], (size_t)c->n * c->rs, kind, c->stream) != cudaSuccess) {
      fail(c, TRMCR_ECUDA, "particle copy failed");
      return bail(TRMCR_ECUDA);
    }
  if (c->geometry == TRMCR_SHOCK_1D && c->n > 0)
    if (cudaMemcpyAsync(c->x[0], pp->x, (size_t)c->n * c->rs, kind, c->stream) != cudaSuccess) {
      fail(c, TRMCR_ECUDA, "position copy failed");
      return bail(TRMCR_ECUDA);
    }
  if (c->geometry == TRMCR_HOMOGENEOUS) {
    if (cudaMemcpyAsync(c->d_offsets, c->h_offsets.data(), sizeof(int64_t) * (c->ncells + 1),
                        cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
      fail(c, TRMCR_ECUDA, "offsets copy failed");
      return bail(TRMCR_ECUDA);
    }
  }

  if (c->geometry == TRMCR_SHOCK_1D) {
    trmcr_status s = shock_init(c, cc, &max_cell);
    if (s) return bail(s);
    // per-cell capacities from the domain's densest state (cells of
    // max(rho_L, rho_R) dx / w particles, + 6 sigma), not from this slab's
    // initial data: every slab of a domain then sizes its plans alike, so a
    // cell takes the same kernel (and the same rounding) in any partition
    const double dx = (cc->x_max - cc->x_min) / (double)c->shock.Cg;
    const double nd = std::max(cc->rho_L, cc->rho_R) * dx / cc->weight;
    if (nd > 0.0 && nd < 1e7) max_cell = (int)ceil(nd + 6.0 * sqrt(nd) + 8.0);
  }

  // ---- shared-memory plan capacity ----
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
  if (smem_max <= 0) smem_max = 227 * 1024;
  const int budget = std::min(smem_max - 4096, 160 * 1024);
  int n_cap = 0;
  if (c->geometry == TRMCR_HOMOGENEOUS) n_cap = std::max(32, (max_cell + 31) / 32 * 32);
  else n_cap = std::max(64, (max_cell + max_cell / 4 + 31) / 32 * 32);   // shock cells fluctuate; rarer giants go to gmem
  const int L_cap = 64;
  // debug knobs: TRMCR_FORCE_GMEM=1 routes every cell through the global-memory
  // path; TRMCR_SMEM_KCAP overrides the shared-memory tree capacity.
  const char *force_g = getenv("TRMCR_FORCE_GMEM");
  const char *kcap_env = getenv("TRMCR_SMEM_KCAP");
  for (;;) {
    const int K_cap = kcap_env ? atoi(kcap_env)
                               : (c->geometry == TRMCR_SHOCK_1D ? std::max(256, n_cap / 4) : std::max(256, n_cap));
    c->lay.build(n_cap, K_cap, L_cap, c->rs, c->P.wb != 0);
    if ((int)c->lay.total <= budget || n_cap <= 32) break;
    n_cap = std::max(32, n_cap / 2 / 32 * 32);
  }
  if (force_g && atoi(force_g)) c->lay.n_cap = 0;
  if (const char *gt = getenv("TRMCR_GMEM_THREADS")) c->gmem_threads = std::max(32, std::min(1024, atoi(gt)));
  const int dyn = (int)c->lay.total;
  if (const char *st = getenv("TRMCR_SMEM_THREADS")) c->smem_threads = atoi(st);
  if (c->smem_threads != 64 && c->smem_threads != 256) c->smem_threads = 128;
  cudaError_t ea = cudaSuccess;
  {
    const void *fns[] = {
        (const void *)shock_collide_smem<double, 64>, (const void *)shock_collide_smem<double, 128>,
        (const void *)shock_collide_smem<double, 256>, (const void *)shock_collide_smem<float, 64>,
        (const void *)shock_collide_smem<float, 128>, (const void *)shock_collide_smem<float, 256>,
        (const void *)cell_step_smem<double, 64>, (const void *)cell_step_smem<double, 128>,
        (const void *)cell_step_smem<double, 256>, (const void *)cell_step_smem<float, 64>,
        (const void *)cell_step_smem<float, 128>, (const void *)cell_step_smem<float, 256>};
    // the attribute is per function (process-wide): set the device maximum so
    // that contexts with different layouts can coexist
    for (const void *f : fns) {
      cudaError_t e = allow_max_dyn_smem(f, smem_max);
      if (e != cudaSuccess) ea = e;
    }
    (void)dyn;
  }
  if (ea != cudaSuccess) { fail(c, TRMCR_ECUDA, "cudaFuncSetAttribute failed"); return bail(TRMCR_ECUDA); }
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
    const int tsm = kThermalWarps * 3 * (c->dtype == TRMCR_F64 ? 512 * 8 : 1024 * 4);
    cudaError_t e2 = c->dtype == TRMCR_F64
        ? allow_max_dyn_smem((const void *)thermal_warp_kernel<double>, smem_max)
        : allow_max_dyn_smem((const void *)thermal_warp_kernel<float>, smem_max);
    if (e2 != cudaSuccess) { fail(c, TRMCR_ECUDA, "cudaFuncSetAttribute(thermal) failed"); return bail(TRMCR_ECUDA); }
    int occ_t = 1, occ_s = 1;
    if (c->dtype == TRMCR_F64) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, thermal_warp_kernel<double>, kThermalWarps * 32, tsm);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, cell_step_smem<double, 256>, 256, dyn);
      occ_s = occ_s * 256 / c->smem_threads;
    } else {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, thermal_warp_kernel<float>, kThermalWarps * 32, tsm);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, cell_step_smem<float, 256>, 256, dyn);
      occ_s = occ_s * 256 / c->smem_threads;
    }
    if (const char *pe = getenv("TRMCR_THERMAL_PREFETCH")) c->thermal_prefetch = atoi(pe);
    c->fast_grid = std::max(1, std::min((c->ncells + kThermalWarps - 1) / kThermalWarps, nsm * std::max(occ_t, 1)));
    c->smem_grid = std::max(1, std::min(c->ncells, nsm * std::max(occ_s, 1)));
    if (c->geometry == TRMCR_SHOCK_1D) c->fast_ok = 0;
  }

  // ---- warp-per-cell general kernel slab (0 disables) ----
  {
    const char *wenv = getenv("TRMCR_WARP_PATH");
    const bool want = !(wenv && atoi(wenv) == 0);
    int wn = c->geometry == TRMCR_SHOCK_1D ? std::max(64, (2 * max_cell + 31) / 32 * 32)
                                           : std::max(32, (max_cell + 31) / 32 * 32);
    // tree capacity: collisions per cell ~ n x / 2 untruncated, and deep trees
    // (x > 1 at fixed m) reach ~0.75 n: homogeneous slabs hold n collisions
    // (a shock cell's slab is sized for twice its particles, its trees are shallow)
    const int wK = c->geometry == TRMCR_SHOCK_1D ? std::max(256, std::min(512, wn / 4)) : std::max(256, wn);
    // shock: velocities are gathered into the output buffer and processed in
    // place (a deferred cell is re-gathered); homogeneous: staged in the slab
    // (in place would corrupt the input of a deferred cell)
    const int v_smem = c->geometry == TRMCR_SHOCK_1D ? 0 : 1;
    if (!v_smem) wn = std::max(wn, 4096);
    wn = std::min(wn, 65504);   // slots are 16-bit in the warp plan; larger cells take the CTA path
    c->wlay.build(wn, wK, 64, c->rs, v_smem, c->P.wb != 0);
    const size_t slab = c->wlay.per_warp;
    c->warp_wpc = (int)std::max<size_t>(1, std::min<size_t>(kWarpCellWarps, (48 * 1024) / slab));
    c->warp_smem = (int)(slab * c->warp_wpc);
    if (const char *pe = getenv("TRMCR_WARP_SMEM_PAD")) c->warp_smem += std::max(0, atoi(pe));   // occupancy experiments
    if (!want || c->warp_smem > smem_max - 2048) {
      c->wlay.n_cap = 0;     // disabled: the CTA kernel takes every general cell
    } else {
      const void *fns[] = {(const void *)cell_step_warp<float, false>, (const void *)cell_step_warp<double, false>,
                           (const void *)shock_collide_warp<float, false>, (const void *)shock_collide_warp<double, false>,
                           (const void *)cell_step_warp<float, true>, (const void *)cell_step_warp<double, true>,
                           (const void *)cell_step_warp<float, false, TRMCR_HARD_SPHERE>,
                           (const void *)cell_step_warp<double, false, TRMCR_HARD_SPHERE>,
                           (const void *)shock_collide_warp<float, true>, (const void *)shock_collide_warp<double, true>};
      for (const void *f : fns)
        if (allow_max_dyn_smem(f, smem_max) != cudaSuccess) {
          fail(c, TRMCR_ECUDA, "cudaFuncSetAttribute(warp) failed");
          return bail(TRMCR_ECUDA);
        }
      int occ = 1, nsm = 148;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
      if (c->dtype == TRMCR_F64)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, shock_collide_warp<double, true>, c->warp_wpc * 32, c->warp_smem);
      else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, shock_collide_warp<float, true>, c->warp_wpc * 32, c->warp_smem);
      c->warp_grid = std::max(1, std::min((c->ncells + c->warp_wpc - 1) / c->warp_wpc, nsm * std::max(occ, 1)));
      // shock: lock-step kernel (TRMCR_SHOCK_LOCKSTEP=0 disables)
      const char *le = getenv("TRMCR_SHOCK_LOCKSTEP");
      const size_t lsm = slab * kLockWarps;
      if (c->geometry == TRMCR_SHOCK_1D && !v_smem && !(le && atoi(le) == 0) && lsm <= (size_t)smem_max - 1024) {
        const bool wbk = ext_variant(c);
        const void *lf = c->dtype == TRMCR_F64
                             ? (wbk ? (const void *)shock_collide_lock<double, true> : (const void *)shock_collide_lock<double, false>)
                             : (wbk ? (const void *)shock_collide_lock<float, true> : (const void *)shock_collide_lock<float, false>);
        int occ_l = 0;
        const void *lfh = c->dtype == TRMCR_F64 ? (const void *)shock_collide_lock<double, false, TRMCR_HARD_SPHERE>
                                                : (const void *)shock_collide_lock<float, false, TRMCR_HARD_SPHERE>;
        if (allow_max_dyn_smem(lfh, smem_max) != cudaSuccess) cudaGetLastError();
        if (allow_max_dyn_smem(lf, smem_max) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_l, lf, kLockWarps * 32, lsm) == cudaSuccess &&
            occ_l > 0) {
          c->lock_smem = (int)lsm;
          c->lock_grid = std::max(1, std::min((c->ncells + kLockWarps - 1) / kLockWarps, nsm * occ_l));
        } else {
          cudaGetLastError();
        }
      }
    }
  }

  // ---- shock: the scatter sort stages fp32 tiles (4 x 16 KB) in dynamic shared memory ----
  if (c->geometry == TRMCR_SHOCK_1D && c->dtype == TRMCR_F32) {
    const void *f1 = (const void *)scatter_sorted<float, 1>, *f4 = (const void *)scatter_sorted<float, kTransportGroups>;
    if (allow_max_dyn_smem(f1, smem_max) != cudaSuccess || allow_max_dyn_smem(f4, smem_max) != cudaSuccess) {
      fail(c, TRMCR_ECUDA, "cudaFuncSetAttribute(scatter_sorted) failed");
      return bail(TRMCR_ECUDA);
    }
  }

  // ---- shock: pooled-batch collision kernel (batch.cuh; TRMCR_SHOCK_BATCH=0 disables) ----
  if (c->geometry == TRMCR_SHOCK_1D && c->wlay.n_cap > 0 && !c->wlay.v_smem && !ext_variant(c) && c->P.debug_stop == 0) {
    // off by default: on C5 it measured 1.90-2.30 ms against the lock-step
    // kernel's 1.29; TRMCR_SHOCK_BATCH=1 enables it
    const char *be = getenv("TRMCR_SHOCK_BATCH");
    if (be && atoi(be) != 0) {
      int nsm = 148, smem_sm = 0;
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
      cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, c->dev);
      const void *bf = c->dtype == TRMCR_F64 ? (const void *)collide_batch<double, QueueArgs> : (const void *)collide_batch<float, QueueArgs>;
      cudaFuncAttributes a;
      int occ_b = 0;
      if (cudaFuncGetAttributes(&a, bf) == cudaSuccess) {
        // two CTAs per SM: one stages its batch while the other computes
        const size_t per = (size_t)smem_sm / kBatchCtas - 1024 - a.sharedSizeBytes - 64;
        c->blay.build(c->rs, std::min(per, (size_t)smem_max - a.sharedSizeBytes));
        if (c->blay.vcap >= 1024 && c->blay.kcap >= 512 &&
            cudaFuncSetAttribute(bf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->blay.total) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, bf, kBatchThreads, c->blay.total) == cudaSuccess &&
            occ_b > 0)
          c->batch_grid = std::max(1, std::min((c->ncells + kBatchCells - 1) / kBatchCells, nsm * occ_b));
      }
      cudaGetLastError();
    }
  }

  if (c->geometry == TRMCR_SHOCK_1D)
    if (trmcr_status s = shock_fused_setup(c)) return bail(s);

  // ---- global-memory plan scratch for large / overflowing cells ----
  const int n_cap_g = c->geometry == TRMCR_HOMOGENEOUS
                          ? std::max(max_cell, 32)
                          : (int)std::min<int64_t>(c->cap, std::max(16 * max_cell, 65536));
  const int L_cap_g = std::max(kk->adaptive ? kk->m_cap : kk->m_fixed, 64) + 1;
  const int64_t K_cap_g = std::min<int64_t>(4LL * n_cap_g + 65536, 0x3FFFFFFFLL);
  const size_t stride = gmem_stride(n_cap_g, K_cap_g, L_cap_g, c->P.wb != 0);
  // CTAs of the global-memory kernel: one per SM (2 per SM when the scratch is
  // small) - many cells can overflow the shared-memory plans at once (deep
  // trees); bounded by 4 GB of scratch
  int G = c->geometry == TRMCR_SHOCK_1D ? 16 : ((double)stride * 296 <= 1e9 ? 296 : 148);   // shock: rare
  G = std::max(1, std::min(c->ncells, G));
  while (G > 1 && (double)G * stride > 4e9) G /= 2;
  c->G = G;
  if (dalloc(c, &c->d_scratch, stride * G)) return bail(TRMCR_ENOMEM);
  c->gs = GmemScratch{c->d_scratch, stride, n_cap_g, (int)K_cap_g, L_cap_g, c->P.wb != 0 ? 1 : 0};

  // ---- giant cells: the whole grid per cell (cooperative launch) ----
  {
    const char *ge = getenv("TRMCR_GIANT");
    const int gmin = ge ? atoi(ge) : 32768;       // 0 disables
    int coop = 0, nsm = 148, occ_g = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
    if (gmin > 0 && c->geometry == TRMCR_HOMOGENEOUS && max_cell >= gmin && coop) {
      const void *gf = c->dtype == TRMCR_F64 ? (const void *)cell_step_giant<double> : (const void *)cell_step_giant<float>;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_g, gf, kGiantThreads, 0) == cudaSuccess && occ_g > 0) {
        // 32 blocks: the step is bound by its grid barriers, whose cost grows
        // with the block count (C2: 148 blocks 2.19 ms, 64 1.42, 32 1.17, 16 1.20)
        c->giant_grid = std::min(32, nsm * occ_g);
        if (const char *gg = getenv("TRMCR_GIANT_GRID")) c->giant_grid = std::max(1, std::min(nsm * occ_g, atoi(gg)));
        c->ghcap = (int64_t)c->giant_grid * (kGiantThreads / 32) * 64;
        if (dalloc(c, &c->d_gsh, sizeof(CellShared)) ||
            dalloc(c, &c->d_gpart, sizeof(double) * kGridSlots * 8 * (size_t)c->giant_grid) ||
            dalloc(c, &c->d_ghbuf, sizeof(int32_t) * (size_t)c->ghcap))
          return bail(TRMCR_ENOMEM);
        c->giant_min = gmin;
      } else {
        cudaGetLastError();
      }
    }
  }

  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    fail(c, TRMCR_ECUDA, "init synchronisation failed");
    return bail(TRMCR_ECUDA);
  }
  if (trmcr_status s = comm_init(c, nccl_id, rank, nranks)) return bail(s);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    fail(c, TRMCR_ECUDA, "init synchronisation failed");
    return bail(TRMCR_ECUDA);
  }
  *out = c;
  return TRMCR_OK;
}

int64_t trmcr_exchange_bytes(int32_t dtype, int64_t capacity) {
  if (capacity < 0) return -1;
  return dtype == TRMCR_F64 ? (int64_t)XBuf<double>::bytes((int)capacity) : (int64_t)XBuf<float>::bytes((int)capacity);
}

trmcr_status trmcr_shock_sort_info(trmcr_ctx *c, int64_t *out4) {
  if (!c || !out4) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->geometry != TRMCR_SHOCK_1D) return fail(c, TRMCR_EINVAL, "not a shock context");
  int w[3] = {0, 0, 0};
  CUDA_TRY(c, cudaMemcpyAsync(w, c->shock.d_W, sizeof(w), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  out4[0] = w[0]; out4[1] = w[1]; out4[2] = w[2];
  out4[3] = c->shock.scatter && c->wlay.n_cap > 0 && !c->wlay.v_smem;
  return TRMCR_OK;
}

int32_t trmcr_shock_fused(const trmcr_ctx *c) {
  return (c && c->geometry == TRMCR_SHOCK_1D) ? c->shock.fused : 0;
}

trmcr_status trmcr_shock_set_exchange(trmcr_ctx *c, void *send_left, void *send_right, void *recv_left,
                                      void *recv_right, int64_t capacity) {
  if (!c || capacity <= 0 || capacity > (1 << 28)) return fail(c, TRMCR_EINVAL, "bad argument");
  if (c->geometry != TRMCR_SHOCK_1D) return fail(c, TRMCR_EINVAL, "not a shock context");
  ShockState &s = c->shock;
  if ((s.has_left && (!send_left || !recv_left)) || (s.has_right && (!send_right || !recv_right)))
    return fail(c, TRMCR_EINVAL, "missing exchange buffer for an existing neighbour");
  s.xsend[0] = send_left; s.xsend[1] = send_right; s.xrecv[0] = recv_left; s.xrecv[1] = recv_right;
  s.xcap = (int)capacity;
  s.xbytes = c->dtype == TRMCR_F64 ? XBuf<double>::bytes(s.xcap) : XBuf<float>::bytes(s.xcap);
  s.own_xbuf = 0;
  return TRMCR_OK;
}

trmcr_status trmcr_shock_begin(trmcr_ctx *c) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  if (c->geometry != TRMCR_SHOCK_1D) return fail(c, TRMCR_EINVAL, "not a shock context");
  if (c->log_cap > 0) CUDA_TRY(c, cudaMemsetAsync(c->d_log_count, 0, sizeof(unsigned long long), c->stream));
  return c->dtype == TRMCR_F64 ? shock_begin<double>(c) : shock_begin<float>(c);
}

trmcr_status trmcr_shock_finish(trmcr_ctx *c) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  if (c->geometry != TRMCR_SHOCK_1D) return fail(c, TRMCR_EINVAL, "not a shock context");
  trmcr_status s = c->dtype == TRMCR_F64 ? shock_finish<double>(c) : shock_finish<float>(c);
  if (s) return s;
  c->step++;
  return TRMCR_OK;
}

trmcr_status trmcr_step(trmcr_ctx *c, int32_t n_steps) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  if (n_steps < 0) return fail(c, TRMCR_EINVAL, "n_steps < 0");
  for (int k = 0; k < n_steps; ++k)
    if (trmcr_status s = do_step(c)) return s;
  return TRMCR_OK;
}

trmcr_status trmcr_moments(trmcr_ctx *c, double *host_out, int32_t global) {
  if (!c || !host_out) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  trmcr_status s = c->dtype == TRMCR_F64 ? launch_moments<double>(c) : launch_moments<float>(c);
  if (s) return s;
  if ((s = sync_check(c))) return s;
  if (global && c->comm) {   // every rank's rows, in global cell order
    std::vector<double> all;
    int64_t total = 0;
    if ((s = comm_allgather_rows(c, c->d_moments, TRMCR_NMOMENTS, all, total))) return s;
    memcpy(host_out, all.data(), sizeof(double) * all.size());
    return TRMCR_OK;
  }
  CUDA_TRY(c, cudaMemcpy(host_out, c->d_moments, sizeof(double) * TRMCR_NMOMENTS * c->ncells,
                         cudaMemcpyDeviceToHost));
  return TRMCR_OK;
}

trmcr_status trmcr_stats(trmcr_ctx *c, double *host_out) {
  if (!c || !host_out) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  if (trmcr_status s = sync_check(c)) return s;
  CUDA_TRY(c, cudaMemcpy(host_out, c->d_stats, sizeof(double) * TRMCR_NSTATS * c->ncells,
                         cudaMemcpyDeviceToHost));
  return TRMCR_OK;
}

trmcr_status trmcr_num_particles(trmcr_ctx *c, int64_t *n) {
  if (!c || !n) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  if (trmcr_status s = sync_check(c)) return s;
  if (c->geometry == TRMCR_SHOCK_1D) {
    int64_t last = 0;
    CUDA_TRY(c, cudaMemcpy(&last, c->d_offsets + c->ncells, sizeof(int64_t), cudaMemcpyDeviceToHost));
    c->n = last;
  }
  *n = c->n;
  return TRMCR_OK;
}

trmcr_status trmcr_copy_particles(trmcr_ctx *c, void *vx, void *vy, void *vz, void *x, int64_t *offsets,
                                  int32_t host) {
  if (!c || !vx || !vy || !vz) return fail(c, TRMCR_EINVAL, "null argument");
  int64_t n = 0;
  if (trmcr_status s = trmcr_num_particles(c, &n)) return s;
  const cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  void *dst[3] = {vx, vy, vz};
  for (int k = 0; k < 3; ++k)
    if (n > 0) CUDA_TRY(c, cudaMemcpyAsync(dst[k], c->v[c->cur][k], (size_t)n * c->rs, kind, c->stream));
  if (x && c->geometry == TRMCR_SHOCK_1D && n > 0)
    CUDA_TRY(c, cudaMemcpyAsync(x, c->x[c->cur], (size_t)n * c->rs, kind, c->stream));
  if (offsets)
    CUDA_TRY(c, cudaMemcpyAsync(offsets, c->d_offsets, sizeof(int64_t) * (c->ncells + 1), kind, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return TRMCR_OK;
}

trmcr_status trmcr_set_velocities(trmcr_ctx *c, const void *vx, const void *vy, const void *vz, int32_t host) {
  if (!c || !vx || !vy || !vz) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->sticky) return TRMCR_ESTATE;
  if (c->geometry == TRMCR_SHOCK_1D) {
    int64_t n = 0;
    if (trmcr_status s = trmcr_num_particles(c, &n)) return s;
  }
  const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const void *src[3] = {vx, vy, vz};
  for (int k = 0; k < 3; ++k)
    if (c->n > 0) CUDA_TRY(c, cudaMemcpyAsync(c->v[c->cur][k], src[k], (size_t)c->n * c->rs, kind, c->stream));
  c->shock.codes_ok = 0;   // the fused shock step recomputes the move codes
  return TRMCR_OK;
}

trmcr_status trmcr_set_particles(trmcr_ctx *c, const void *x, const void *vx, const void *vy, const void *vz,
                                 int64_t n, int32_t host) {
  if (!c) return fail(nullptr, TRMCR_EINVAL, "null ctx");
  if (c->sticky) return TRMCR_ESTATE;
  if (n < 0 || (n > 0 && (!vx || !vy || !vz))) return fail(c, TRMCR_EINVAL, "bad particle arrays");
  if (c->geometry == TRMCR_HOMOGENEOUS) {
    if (x) return fail(c, TRMCR_EINVAL, "homogeneous geometry takes no positions");
    if (n != c->n) return fail(c, TRMCR_EINVAL, "homogeneous geometry: n must equal the context's particle count");
    return n > 0 ? trmcr_set_velocities(c, vx, vy, vz, host) : TRMCR_OK;
  }
  if (n > 0 && !x) return fail(c, TRMCR_EINVAL, "shock geometry needs positions");
  if (n > c->cap) return fail(c, TRMCR_ECAPACITY, "more particles than the context capacity");
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));   // the previous step may still read the buffers
  const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const void *src[4] = {x, vx, vy, vz};
  void *dst[4] = {c->x[c->cur], c->v[c->cur][0], c->v[c->cur][1], c->v[c->cur][2]};
  for (int k = 0; k < 4; ++k)
    if (n > 0) CUDA_TRY(c, cudaMemcpyAsync(dst[k], src[k], (size_t)n * c->rs, kind, c->stream));
  c->n = n;
  return shock_rebin(c, nullptr);
}

trmcr_status trmcr_step_host_particles(trmcr_ctx *c, const void *x, const void *vx, const void *vy,
                                       const void *vz, int64_t n, double *host_moments) {
  if (!c || !host_moments) return fail(c, TRMCR_EINVAL, "null argument");
  if (trmcr_status s = trmcr_set_particles(c, x, vx, vy, vz, n, 1)) return s;
  if (trmcr_status s = do_step(c)) return s;
  return trmcr_moments(c, host_moments, 0);
}

trmcr_status trmcr_step_host(trmcr_ctx *c, const void *vx, const void *vy, const void *vz, double *host_moments) {
  if (!c || !host_moments) return fail(c, TRMCR_EINVAL, "null argument");
  if (c->geometry != TRMCR_HOMOGENEOUS) return fail(c, TRMCR_EINVAL, "trmcr_step_host: homogeneous geometry only");
  if (trmcr_status s = trmcr_set_velocities(c, vx, vy, vz, 1)) return s;
  if (trmcr_status s = do_step(c)) return s;
  return trmcr_moments(c, host_moments, 0);
}

trmcr_status trmcr_set_log(trmcr_ctx *c, int64_t capacity) {
  if (!c || capacity < 0) return fail(c, TRMCR_EINVAL, "bad argument");
  if (c->sticky) return TRMCR_ESTATE;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->d_log && capacity > 0 && capacity <= c->log_cap) {   // reuse the buffer
    c->log_cap = capacity;
    c->P.log_on = 1;
    CUDA_TRY(c, cudaMemset(c->d_log_count, 0, sizeof(unsigned long long)));
    return TRMCR_OK;
  }
  if (c->d_log) {                                              // release the old buffer
    c->allocs.erase(std::remove(c->allocs.begin(), c->allocs.end(), (void *)c->d_log), c->allocs.end());
    cudaFree(c->d_log);
  }
  c->d_log = nullptr;
  c->log_cap = 0;
  c->P.log_on = 0;
  if (capacity > 0) {
    if (dalloc(c, &c->d_log, sizeof(trmcr_coll_rec) * (size_t)capacity)) return TRMCR_ENOMEM;
    c->log_cap = capacity;
    c->P.log_on = 1;
  }
  CUDA_TRY(c, cudaMemset(c->d_log_count, 0, sizeof(unsigned long long)));
  return TRMCR_OK;
}

trmcr_status trmcr_get_log(trmcr_ctx *c, trmcr_coll_rec *out, int64_t *count) {
  if (!c || !count) return fail(c, TRMCR_EINVAL, "null argument");
  if (trmcr_status s = sync_check(c)) return s;
  unsigned long long k = 0;
  CUDA_TRY(c, cudaMemcpy(&k, c->d_log_count, sizeof(k), cudaMemcpyDeviceToHost));
  *count = (int64_t)k;
  const int64_t m = std::min<int64_t>((int64_t)k, c->log_cap);
  if (out && m > 0)
    CUDA_TRY(c, cudaMemcpy(out, c->d_log, sizeof(trmcr_coll_rec) * (size_t)m, cudaMemcpyDeviceToHost));
  return TRMCR_OK;
}

}  // extern "C"
