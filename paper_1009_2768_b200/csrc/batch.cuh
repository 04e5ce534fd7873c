// batch.cuh — pooled-batch collision kernel for cell-sorted particles (A3-A8).
//
// The same computation as the warp-per-cell general step (cell_warp.cuh: same
// keyed draws, same per-lane reduction orders, so results are bitwise those of
// shock_collide_lock / the oracle's canonical definition), laid
// out for the GPU differently: a CTA stages a BATCH of consecutive cells
// (<= kBatchCells cells, <= vcap particles) in shared memory with bulk async
// copies (cp.async.bulk + mbarrier) and runs every phase of the step POOLED
// over the batch's cells:
//   moments + split (A3, A4)        warp per cell, from shared memory
//   plan (A5, top-down)              per level: the counts of every cell, then
//                                    the type draws of all cells' collisions
//                                    flat over the CTA
//   demand indices (A5 pass 1)       warp per cell
//   keyed permutations (A5 pass 2)   flat over every demand of the batch
//   collisions (A6, bottom-up)       per level, flat over the batch
//   RAD estimate + decision (A7)     warp per cell; cells that retry go round
//                                    again (the others sit the round out)
//   Maxwellian (A8), write-back      warp per cell / flat
// so lanes are not left idle by small levels and cells, a cell's latency
// chains overlap other cells' work, and no warp waits at a barrier for the
// slowest cell of a lock-step group (shock.cuh shock_collide_lock: 19.5 % of
// its stall samples).  A cell the batch cannot hold (plan pool or level
// capacity, TRMC-WB / majorant variants) is deferred untouched to the CTA
// kernel: velocities live in shared memory until the write-back, so a cell
// can be given up at any point of its step.
#pragma once
#include "cell_warp.cuh"

namespace trmcr {

#ifndef TRMCR_BATCH_WARPS
#define TRMCR_BATCH_WARPS 8
#endif
#ifndef TRMCR_BATCH_CTAS
#define TRMCR_BATCH_CTAS 2         // CTAs per SM the shared-memory stage is sized for
#endif
#ifndef TRMCR_BATCH_CELLS
#define TRMCR_BATCH_CELLS 16
#endif
constexpr int kBatchThreads = 32 * TRMCR_BATCH_WARPS;
constexpr int kBatchWarps = TRMCR_BATCH_WARPS;
constexpr int kBatchCtas = TRMCR_BATCH_CTAS;
constexpr int kBatchCells = TRMCR_BATCH_CELLS;    // cells per chunk (and at most per batch)
constexpr int kBatchLevels = 32;   // levels 0..31 per cell; deeper quotas: deferred
constexpr int kBatchLcap = kBatchLevels - 1;
enum : int { kBDone = 8 };         // cell finished (n == 0 or every attempt run)

struct BatchCell {
  double ux, uy, uz, S0, sigma, p, mu, S_est, E1, c2;
  double cind, dS;     // pre-step indicator sum (n S0), its change by the collisions so far
  double sums[4];
  uint4 pk;            // key of pi0
  PermDom D0;          // domain of pi0 ([0, n))
  int n, vb;           // particles; index of slot 0 in the staged arrays
  int m_cur, m_next, d, top, lo, hi, r, flag, rem;
  int L, Ltot, U, nT, budget, leaf_off;
  int plan;            // 1 while this round's plan of the cell is being built
  unsigned prop, acc, viol;
};

struct BatchLayout {
  int vcap, kcap;      // staged particles (incl. alignment slack), plan pool entries
  size_t off_cells, off_Q, off_C, off_S, off_cons, off_rk, off_pd, off_pre, off_ws, off_ctype, off_ccell,
      off_clev, off_crank, off_cslot, off_dsv, off_v, total;
  // rs = sizeof(Real); smem = bytes available to one CTA
  void build(size_t rs, size_t smem) {
    auto al = [](size_t o, size_t a) { return (o + a - 1) / a * a; };
    size_t o = 0;
    off_cells = o; o += sizeof(BatchCell) * kBatchCells;
    o = al(o, 16); off_rk = o; o += sizeof(uint4) * kBatchCells * kBatchLevels;
    off_pd = o; o += sizeof(PermDom) * kBatchCells * kBatchLevels;
    off_Q = o; o += 4 * kBatchCells * kBatchLevels;
    off_C = o; o += 4 * kBatchCells * kBatchLevels;
    off_S = o; o += 4 * kBatchCells * kBatchLevels;
    off_cons = o; o += 4 * kBatchCells * kBatchLevels;
    off_pre = o; o += 4 * (kBatchCells + 1) * (kBatchLevels + 1);
    off_ws = o; o += 4 * 3 * 32 * kBatchWarps;      // pass-1 scratch: base, cnt, tmp per warp
    const size_t fixed = al(o, 16);
    // the rest: plan pool (9 B + rs per entry) and the staged velocities (3 rs
    // per particle), pool sized for ~1/3 collision per particle (C5: 0.15)
    const size_t rest = smem > fixed + 4096 ? smem - fixed - 4096 : 0;
    int v = (int)(rest / (3 * rs + (9.0 + rs) / 3.0));
    v = v / 16 * 16;
    if (v > 65520) v = 65520;
    int k = (int)((rest - (size_t)v * 3 * rs) / (9 + rs));
    if (k > 65535) k = 65535;
    vcap = v; kcap = k;
    o = fixed;
    off_cslot = o; o += 4 * (size_t)kcap;
    off_crank = o; o += 2 * (size_t)kcap;
    off_ctype = o; o += (size_t)kcap;
    off_ccell = o; o += (size_t)kcap;
    off_clev = o; o += (size_t)kcap;
    o = al(o, 16); off_dsv = o; o += rs * (size_t)kcap;
    o = al(o, 128); off_v = o; o += 3 * rs * (size_t)vcap;
    total = al(o, 16);
  }
};

// ---- bulk async copy global -> shared (TMA 1-D) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Split continued to level m (Alg 4.2, as wsplit_extend) with the whole warp
// executing it redundantly (uniform values); lane l holds the uniform of
// level l < 32, deeper levels draw theirs.  Lane 0 stores the quotas.
__device__ __forceinline__ void bsplit_extend(const RngKey &K, BatchCell &cl, int m, int32_t *Q, double ul, int &d,
                                              int &rem, int &flag) {
  const int lane = threadIdx.x & 31;
  while (rem > 0 && d < m) {
    const double y = cl.p * (double)rem;
    if (y < 0x1p-53) {
      if (lane == 0)
        for (int q = d + 1; q <= m && q <= kBatchLcap; ++q) Q[q] = 0;
      d = m;
      break;
    }
    d++;
    double u = __shfl_sync(0xffffffffu, ul, d & 31);
    if (d >= 32) {
      const uint4 w = K(kSplit, 0, (uint32_t)d, 0);
      u = u53(w.x, w.y);
    }
    const double fl = floor(y);
    int64_t q = (int64_t)fl + ((u < y - fl) ? 1 : 0);
    if (q > rem) q = rem;
    if (d <= kBatchLcap) { if (lane == 0) Q[d] = (int32_t)q; }
    else if (q > 0) flag = kOverflow;
    rem -= (int)q;
  }
}

template <typename Real>
struct BatchSmem {
  BatchCell *cells;
  int32_t *Q, *Cl, *Sl, *cons, *pre, *ws;
  uint4 *rk;
  PermDom *pd;
  uint32_t *cslot32;   // unused (alignment)
  uint16_t *cslot, *crank;
  uint8_t *ctype, *ccell, *clev;
  Real *vx, *vy, *vz;
  Real *dsv;           // [kcap] indicator change of each collision (RAD)
};

// Per-cell level arrays: [cell][level].
#define BQ(i, d) S.Q[(i) * kBatchLevels + (d)]
#define BC(i, d) S.Cl[(i) * kBatchLevels + (d)]
#define BS(i, d) S.Sl[(i) * kBatchLevels + (d)]
#define BCONS(i, d) S.cons[(i) * kBatchLevels + (d)]
#define BRK(i, d) S.rk[(i) * kBatchLevels + (d)]
#define BPD(i, d) S.pd[(i) * kBatchLevels + (d)]
#define BPRE(d, i) S.pre[(d) * (kBatchCells + 1) + (i)]

// Optional per-phase wall cycles of the batch kernel (thread 0 of each CTA,
// between barriers; debug builds: -DTRMCR_PHASE_TIMING).
#ifdef TRMCR_PHASE_TIMING
#define BPHASE_MARK() long long t_bph = clock64()
#define BPHASE_ADD(k)                                                                            \
  do {                                                                                           \
    if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[k], (unsigned long long)(clock64() - t_bph)); \
    t_bph = clock64();                                                                           \
  } while (0)
#else
#define BPHASE_MARK()
#define BPHASE_ADD(k)
#endif

// The cell of flat index f of level d's pooled work: pre[d][i] <= f < pre[d][i+1].
__device__ __forceinline__ int batch_find(const int32_t *pre, int nc, int f) {
  int i = 0;
  while (i + 1 < nc && pre[i + 1] <= f) ++i;
  return i;
}

template <typename Real, class QueueArgsT>
__global__ void __launch_bounds__(kBatchThreads, kBatchCtas)
collide_batch(StepParams P, BatchLayout Lay, int C, int64_t cap, const int64_t *__restrict__ off, Real *gvx,
              Real *gvy, Real *gvz, int32_t *m_state, double *stats, int *defer_count, int *defer_list, QueueArgsT Qa) {
  pdl_wait();   // programmatic dependent launch: the predecessor's writes are visible
  if (off[C] > cap) { pdl_trigger(); return; }   // capacity exceeded (err set by the scan): no stores
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t mbar;
  __shared__ int s_sub[4];       // sub-batch: first cell, end cell, skip
  __shared__ int s_nact, s_pool, s_dmax, s_replan, s_dmax2, s_kill;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int E = 16 / (int)sizeof(Real);   // elements per 16 bytes
  BatchSmem<Real> S;
  S.cells = reinterpret_cast<BatchCell *>(smem + Lay.off_cells);
  S.Q = reinterpret_cast<int32_t *>(smem + Lay.off_Q);
  S.Cl = reinterpret_cast<int32_t *>(smem + Lay.off_C);
  S.Sl = reinterpret_cast<int32_t *>(smem + Lay.off_S);
  S.cons = reinterpret_cast<int32_t *>(smem + Lay.off_cons);
  S.pre = reinterpret_cast<int32_t *>(smem + Lay.off_pre);
  S.ws = reinterpret_cast<int32_t *>(smem + Lay.off_ws);
  S.rk = reinterpret_cast<uint4 *>(smem + Lay.off_rk);
  S.pd = reinterpret_cast<PermDom *>(smem + Lay.off_pd);
  S.cslot = reinterpret_cast<uint16_t *>(smem + Lay.off_cslot);
  S.crank = reinterpret_cast<uint16_t *>(smem + Lay.off_crank);
  S.ctype = smem + Lay.off_ctype;
  S.ccell = smem + Lay.off_ccell;
  S.clev = smem + Lay.off_clev;
  S.dsv = reinterpret_cast<Real *>(smem + Lay.off_dsv);
  S.vx = reinterpret_cast<Real *>(smem + Lay.off_v);
  S.vy = S.vx + Lay.vcap;
  S.vz = S.vy + Lay.vcap;
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  BPHASE_MARK();
  const int nchunks = (C + kBatchCells - 1) / kBatchCells;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const int c_lo = chunk * kBatchCells, c_hi = min(C, c_lo + kBatchCells);
    int s = c_lo;
    while (s < c_hi) {
      // ---- the batch: the longest run of cells from s whose staged range fits ----
      if (warp == 0) {
        const int c = s + lane;
        int n = 0;
        if (c < c_hi) n = (int)(off[c + 1] - off[c]);
        int inc = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += t;
        }
        const bool fits = c < c_hi && inc + (E - 1) <= Lay.vcap;
        const int cnt = __popc(__ballot_sync(0xffffffffu, fits));
        if (lane == 0) {
          if (cnt == 0) {                       // one cell larger than the stage: the CTA kernel's
            defer_list[atomicAdd(defer_count, 1)] = s;
            s_sub[0] = s; s_sub[1] = s + 1; s_sub[2] = 1;
          } else {
            s_sub[0] = s; s_sub[1] = s + cnt; s_sub[2] = 0;
          }
        }
      }
      __syncthreads();
      const int e_cell = s_sub[1];
      const bool skip = s_sub[2] != 0;
      __syncthreads();                          // s_sub is rewritten by the next batch
      if (skip) { s = e_cell; continue; }
#ifdef TRMCR_PHASE_TIMING
      if (tid == 0) atomicAdd(&g_phase_cycles[14], 1ull);
#endif
      const int nc = e_cell - s;
      const int64_t ga = off[s], gb = off[e_cell];
      const int64_t a_al = ga & ~(int64_t)(E - 1), b_al = gb & ~(int64_t)(E - 1);
      // ---- stage: bulk copies of [a_al, b_al), scalar tail [max(b_al, ga), gb) ----
      if (tid == 0) {
        fence_proxy_async();                    // earlier generic accesses of the stage before the async writes
        const uint32_t bytes = b_al > a_al ? (uint32_t)((b_al - a_al) * (int64_t)sizeof(Real)) : 0u;
        mbar_expect_tx(&mbar, 3u * bytes);
        if (bytes) {
          bulk_g2s(S.vx, gvx + a_al, bytes, &mbar);
          bulk_g2s(S.vy, gvy + a_al, bytes, &mbar);
          bulk_g2s(S.vz, gvz + a_al, bytes, &mbar);
        }
      }
      {
        const int64_t t0 = b_al > ga ? b_al : ga;
        const int64_t g = t0 + tid;
        if (g < gb) {
          S.vx[g - a_al] = gvx[g]; S.vy[g - a_al] = gvy[g]; S.vz[g - a_al] = gvz[g];
        }
      }
      if (tid < nc) {
        BatchCell &cl = S.cells[tid];
        const int c = s + tid;
        const int64_t b0 = off[c];
        cl.n = (int)(off[c + 1] - b0);
        cl.vb = (int)(b0 - a_al);
        cl.m_cur = P.adaptive ? m_state[c] : P.m_fixed;
        cl.flag = kOk;
        cl.prop = 0; cl.acc = 0; cl.viol = 0;
      }
      mbar_wait(&mbar, phase);
      phase ^= 1u;
      __syncthreads();
      BPHASE_ADD(0);
      // ---- A3 moments + A4 split: warp per cell ----
      for (int i = warp; i < nc; i += kBatchWarps) {
        BatchCell &cl = S.cells[i];
        const int n = cl.n;
        const uint32_t gcell = P.cell_base + (uint32_t)(s + i);
        const RngKey K{P.k0, P.k1, gcell, P.step};
        if (n == 0) {
          if (lane == 0) {
            double *st = stats + (size_t)(s + i) * TRMCR_NSTATS;
            for (int k = 0; k < TRMCR_NSTATS; ++k) st[k] = 0.0;
            st[TRMCR_ST_MUSED] = cl.m_cur; st[TRMCR_ST_MNEXT] = cl.m_cur;
            cl.flag = kBDone;
          }
          continue;
        }
        const Real *vx = S.vx + cl.vb, *vy = S.vy + cl.vb, *vz = S.vz + cl.vb;
        double sx, sy, sz;
        if constexpr (sizeof(Real) == 4) {
          warp_cell_sums(vx, vy, vz, n, sx, sy, sz);
        } else {
          sx = 0; sy = 0; sz = 0;
          for (int q = lane; q < n; q += 32) { sx += vx[q]; sy += vy[q]; sz += vz[q]; }
        }
        const double Sx = warp_sum(sx), Sy = warp_sum(sy), Sz = warp_sum(sz);
        const double ux = Sx / n, uy = Sy / n, uz = Sz / n;
        double c0 = 0, c1 = 0, c2 = 0, dv2 = 0;
        if constexpr (sizeof(Real) == 4) {
          const float fux = (float)ux, fuy = (float)uy, fuz = (float)uz;
          warp_cell_central(vx, vy, vz, n, fux, fuy, fuz, c0, c1, c2, dv2);
        } else {
          for (int q = lane; q < n; q += 32) {
            const double x = vx[q], y = vy[q], z = vz[q];
            const double dx = x - ux, dy = y - uy, dz = z - uz;
            const double r2 = sq3(dx, dy, dz);       // the oracle's rounding (Sigma' ties |q|)
            dv2 = fmax(dv2, r2);
            c0 += dx * dx;
            const double v2 = x * x + y * y + z * z;
            c1 += v2 * v2;
            c2 += r2;
          }
        }
        const uint4 wl = K(kSplit, 0, (uint32_t)lane, 0);   // split uniform of level `lane`
        const double ul = u53(wl.x, wl.y);
        c0 = warp_sum(c0); c1 = warp_sum(c1); c2 = warp_sum(c2); dv2 = warp_max(dv2);
        // scalars (every lane computes the same values; lane 0 stores)
        const double rho_c = P.shock ? n * P.w_over_dx : 1.0;
        double sigma, mu;
        if (P.model == TRMCR_HARD_SPHERE) { sigma = 2.0 * sqrt(dv2); mu = rho_c * sigma; }
        else if (P.model == TRMCR_VHS) { sigma = vhs_majorant(dv2, P.alpha); mu = rho_c * sigma; }
        else { sigma = 0.0; mu = rho_c; }
        const double p = exp(-(mu * P.dt / P.eps));
        if (lane == 0) {
          cl.ux = ux; cl.uy = uy; cl.uz = uz; cl.c2 = c2;
          cl.sums[0] = Sx; cl.sums[1] = Sy; cl.sums[2] = Sz; cl.sums[3] = c2 + n * (ux * ux + uy * uy + uz * uz);
          cl.cind = P.indicator == TRMCR_IND_PXX ? c0 : c1;
          cl.dS = 0.0;
          cl.S0 = cl.cind / n;
          cl.sigma = sigma; cl.mu = mu; cl.p = p;
          cl.pk = K(kPerm, 0, 0, 0);
          cl.D0 = perm_dom((uint32_t)n);
        }
        __syncwarp();
        // split: N0 = IR(p n), then levels 1.. until rem == 0 or m
        int flag = kOk, d = 0, rem;
        {
          const double y = p * (double)n;
          int64_t N0 = 0;
          if (!(y < 0x1p-53)) {
            const double fl = floor(y);
            N0 = (int64_t)fl + ((__shfl_sync(0xffffffffu, ul, 0) < y - fl) ? 1 : 0);
          }
          if (lane == 0) BQ(i, 0) = (int32_t)N0;
          rem = n - (int)N0;
        }
        bsplit_extend(K, cl, cl.m_cur, &BQ(i, 0), ul, d, rem, flag);
        if (lane == 0) {
          cl.d = d; cl.rem = rem; cl.flag = flag;
          cl.r = 0; cl.lo = 1; cl.hi = d < kBatchLcap ? d : kBatchLcap;
          cl.budget = n; cl.leaf_off = 0;
          cl.Ltot = 0; cl.nT = 0; cl.U = 0;
          cl.m_next = cl.m_cur; cl.S_est = cl.S0; cl.E1 = 0.0;
        }
      }
      __syncthreads();
      BPHASE_ADD(1);
      // ---- attempt rounds: every cell still running takes part ----
      for (;;) {
        if (tid == 0) { s_nact = 0; s_pool = 0; s_dmax = 0; s_kill = 0; }
        __syncthreads();
        if (tid < nc) {
          BatchCell &cl = S.cells[tid];
          cl.plan = 0;
          if (cl.flag == kOk) {
            int top = cl.hi;
            while (top >= cl.lo && BQ(tid, top) == 0) top--;
            if (top < cl.lo || top < 1) top = 0;
            cl.top = top;
            cl.L = 0;
            atomicAdd(&s_nact, 1);
            if (top >= 1) {
              cl.plan = 1;
              atomicMax(&s_dmax, top);
              for (int q = 0; q <= top; ++q) { BCONS(tid, q) = 0; BC(tid, q) = 0; }
            }
          }
        }
        __syncthreads();
        BPHASE_ADD(2);
        if (s_nact == 0) break;
#ifdef TRMCR_PHASE_TIMING
        if (tid == 0) atomicAdd(&g_phase_cycles[15], 1ull);
#endif
        // ---- A5 plan, top-down, pooled; guard re-plans (drop the top quota level) ----
        for (;;) {
          const int dmax = s_dmax;
          for (int d = dmax; d >= 1; --d) {
            if (warp == 0) {
              int Cd = 0;
              bool part = false;
              if (lane < nc) {
                const BatchCell &cl = S.cells[lane];
                if (cl.plan && d <= cl.top) {
                  part = true;
                  const int Qd = d >= cl.lo ? BQ(lane, d) : 0;
                  Cd = (Qd + BCONS(lane, d) + 1) >> 1;
                }
              }
              int inc = Cd;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
              }
              const int excl = inc - Cd;
              const int tot = __shfl_sync(0xffffffffu, inc, 31);
              const int base = s_pool;
              __syncwarp();
              if (part) {
                int Cs = Cd;
                if (base + inc > Lay.kcap) {        // plan pool full: the cell goes to the CTA kernel
                  S.cells[lane].flag = kOverflow;
                  S.cells[lane].plan = 0;
                  Cs = 0;
                }
                BC(lane, d) = Cs;
                BS(lane, d) = base + excl;
              }
              if (lane <= nc) BPRE(d, lane) = excl;    // lane nc: the level's total
              if (lane == 0) s_pool = base + tot < Lay.kcap ? base + tot : Lay.kcap;
            }
            __syncthreads();
            const int tot = BPRE(d, nc);
            for (int f = tid; f < tot; f += kBatchThreads) {
              const int i = batch_find(&BPRE(d, 0), nc, f);
              const BatchCell &cl = S.cells[i];
              const int j = f - BPRE(d, i);
              const int e = BS(i, d) + j;
              if (!cl.plan || j >= BC(i, d)) {      // reserved for a cell the pool could not hold
                if (e < Lay.kcap) S.ccell[e] = 0xFF;
                continue;
              }
              const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)(s + i), P.step};
              const uint32_t w = K(kType, cl.r, d, j).x;
              const uint32_t a = __umulhi(w, (uint32_t)d);
              S.ctype[e] = (uint8_t)a; S.ccell[e] = (uint8_t)i; S.clev[e] = (uint8_t)d;
              atomicAdd(&BCONS(i, a), 1);
              atomicAdd(&BCONS(i, d - 1 - a), 1);
            }
            __syncthreads();
          }
          if (tid == 0) { s_replan = 0; s_dmax2 = 0; }
          __syncthreads();
          BPHASE_ADD(3);
          if (tid < nc) {
            BatchCell &cl = S.cells[tid];
            if (cl.plan) {
              if (BCONS(tid, 0) <= cl.budget) {
                cl.L = BCONS(tid, 0);
                cl.plan = 0;
              } else {                              // guard: drop the top quota level
                for (int q = 1; q <= cl.top; ++q) {  // abandon the entries of this plan
                  for (int j = 0; j < BC(tid, q); ++j) S.ccell[BS(tid, q) + j] = 0xFF;
                  BC(tid, q) = 0;
                }
                int t = cl.top - 1;
                while (t >= cl.lo && BQ(tid, t) == 0) t--;
                if (t < cl.lo || t < 1) {
                  cl.top = 0; cl.L = 0; cl.plan = 0;
                } else {
                  cl.top = t;
                  for (int q = 0; q <= t; ++q) BCONS(tid, q) = 0;
                  s_replan = 1;
                  atomicMax(&s_dmax2, t);
                }
              }
            }
          }
          __syncthreads();
          if (!s_replan) break;
          if (tid == 0) s_dmax = s_dmax2;
          __syncthreads();
          BPHASE_ADD(4);
        }
        // ---- A5 pass 1 (warp per cell): in-level ranks, demand indices, pool keys ----
        int dtop = 0;
        for (int i = warp; i < nc; i += kBatchWarps) {
          BatchCell &cl = S.cells[i];
          if (cl.flag != kOk || cl.top < 1) continue;
          const int top = cl.top;
          int32_t *base = S.ws + warp * 96, *cnt = base + 32, *tmp = base + 64;
          const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)(s + i), P.step};
          for (int q = lane; q <= top; q += 32) {
            base[q] = 0; cnt[q] = 0;
            if (q >= 1) {
              BRK(i, q) = K(kPerm, cl.r, q, 0);
              BPD(i, q) = perm_dom(2u * (uint32_t)BC(i, q));
            }
          }
          __syncwarp();
          const int leaf_off = cl.leaf_off;
          int pd = 0;
          for (int d = 1; d <= top; ++d) {
            const int Cd = BC(i, d), Sd = BS(i, d);
            if (Cd == 0) continue;
            if (pd > 0) {
              for (int p = lane; p < pd; p += 32) tmp[p] = base[p] + cnt[p] + cnt[pd - 1 - p];
              __syncwarp();
              for (int p = lane; p < pd; p += 32) { base[p] = tmp[p]; cnt[p] = 0; }
              __syncwarp();
            }
            for (int j0 = 0; j0 < Cd; j0 += 32) {
              const int j = j0 + lane;
              const bool valid = j < Cd;
              const uint32_t a = valid ? (uint32_t)S.ctype[Sd + j] : 0xFFFFFFFFu;
              const unsigned peers = __match_any_sync(0xffffffffu, a);
              const unsigned lt = (1u << lane) - 1u;
              int c0 = 0;
              if (valid) c0 = cnt[a];
              __syncwarp();
              if (valid) {
                S.crank[Sd + j] = (uint16_t)(c0 + __popc(peers & lt));
                if ((peers & lt) == 0u) cnt[a] = c0 + __popc(peers);
              }
              __syncwarp();
            }
            pd = d;
            for (int j = lane; j < Cd; j += 32) {
              const uint32_t a = S.ctype[Sd + j], b = (uint32_t)d - 1u - a;
              const uint32_t rank = S.crank[Sd + j];
              const uint32_t t0 = (uint32_t)base[a] + rank, t1 = (uint32_t)(base[b] + cnt[b]) + rank;
              S.cslot[2 * (Sd + j)] = (uint16_t)(a == 0 ? (uint32_t)leaf_off + t0 : t0);
              S.cslot[2 * (Sd + j) + 1] = (uint16_t)(b == 0 ? (uint32_t)leaf_off + t1 : t1);
            }
            __syncwarp();
          }
          dtop = max(dtop, top);
        }
        if (lane == 0 && dtop > 0) atomicMax(&s_kill, dtop);   // (reused: the round's deepest level)
        __syncthreads();
        BPHASE_ADD(5);
        const int dexec = s_kill;
        const int npool = s_pool;
        // ---- A5 pass 2: every keyed permutation of the round, flat ----
        for (int e = tid; e < npool; e += kBatchThreads) {
          const int i = S.ccell[e];
          if (i == 0xFF || S.cells[i].flag != kOk) continue;
          const BatchCell &cl = S.cells[i];
          const uint32_t a = S.ctype[e], d = S.clev[e], b = d - 1u - a;
          const uint32_t x0 = S.cslot[2 * e], x1 = S.cslot[2 * e + 1];
          uint32_t y0, y1;
          perm_eval2(x0, a == 0 ? cl.pk : BRK(i, a), a == 0 ? cl.D0 : BPD(i, a), x1, b == 0 ? cl.pk : BRK(i, b),
                     b == 0 ? cl.D0 : BPD(i, b), y0, y1);
          S.cslot[2 * e] = (uint16_t)(y0 == 0xFFFFFFFFu ? 0xFFFFu : y0);
          S.cslot[2 * e + 1] = (uint16_t)(y1 == 0xFFFFFFFFu ? 0xFFFFu : y1);
        }
        // per-level prefixes of the execution (cells whose plan survived)
        if (warp == 0) {
          for (int d = 1; d <= dexec; ++d) {
            int Cd = 0;
            if (lane < nc) {
              const BatchCell &cl = S.cells[lane];
              if (cl.flag == kOk && d <= cl.top) Cd = BC(lane, d);
            }
            int inc = Cd;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= o) inc += t;
            }
            if (lane <= nc) BPRE(d, lane) = inc - Cd;
          }
        }
        __syncthreads();
        BPHASE_ADD(6);
        // ---- A5 pass 3 + A6: slots and collisions, level by level, flat ----
        for (int d = 1; d <= dexec; ++d) {
          const int tot = BPRE(d, nc);
          for (int f = tid; f < tot; f += kBatchThreads) {
            const int i = batch_find(&BPRE(d, 0), nc, f);
            BatchCell &cl = S.cells[i];
            const int j = f - BPRE(d, i);
            const int e = BS(i, d) + j;
            const uint32_t a = S.ctype[e], b = (uint32_t)d - 1u - a;
            const uint32_t pool[2] = {a, b};
            uint32_t slot[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const uint32_t y = S.cslot[2 * e + q];
              slot[q] = (pool[q] == 0 || y == 0xFFFFu) ? y : (uint32_t)S.cslot[2u * (uint32_t)BS(i, pool[q]) + y];
              if (slot[q] >= (uint32_t)cl.n) { atomicOr(P.err, kErrInternal); slot[q] = 0; }
            }
            S.cslot[2 * e] = (uint16_t)slot[0];
            S.cslot[2 * e + 1] = (uint16_t)slot[1];
            const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)(s + i), P.step};
            CellBuf<Real> B;
            B.vx = S.vx + cl.vb; B.vy = S.vy + cl.vb; B.vz = S.vz + cl.vb;
            unsigned viol = 0;
            double dse = 0.0;
            const int ok = tree_collision<Real>(P, K, B, (Real)cl.sigma, cl.r, d, (uint32_t)j, slot[0], slot[1], viol,
                                                P.adaptive ? &dse : nullptr, (Real)cl.ux);
            S.dsv[e] = (Real)dse;
            if (ok) atomicAdd(&cl.acc, 1u);
            if (viol) atomicAdd(&cl.viol, viol);
            log_collision(P, K, Qa.log, Qa.log_count, Qa.log_cap, cl.r, d, j, ok, slot[0], slot[1]);
          }
          __syncthreads();
          BPHASE_ADD(7);
        }
        // ---- after the attempt: bookkeeping, A7 estimate and decision (warp per cell) ----
        for (int i = warp; i < nc; i += kBatchWarps) {
          BatchCell &cl = S.cells[i];
          if (cl.flag != kOk) continue;
          const int n = cl.n;
          if (lane == 0) {
            unsigned pr = 0;
            for (int q = 1; q <= cl.top; ++q) pr += (unsigned)BC(i, q);
            cl.prop += pr;
            if (cl.r == 0) {
              cl.Ltot = cl.L;
              cl.U = BQ(i, 0) < n - cl.Ltot ? BQ(i, 0) : n - cl.Ltot;
              cl.nT = n - cl.Ltot - cl.U;
              cl.m_next = cl.m_cur;
              cl.S_est = cl.S0; cl.E1 = 0.0;
            } else {
              cl.Ltot += cl.L; cl.nT -= cl.L;
            }
          }
          __syncwarp();
          if (!P.adaptive) { if (lane == 0) cl.flag = kBDone; continue; }
          const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)(s + i), P.step};
          Perm pi0;
          pi0.rk = cl.pk; pi0.D = cl.D0;
          const Real *vx = S.vx + cl.vb, *vy = S.vy + cl.vb, *vz = S.vz + cl.vb;
          // estimate (as wrad_estimate): all slots minus Theta's, plus Theta analytically
          const bool pxx = P.indicator == TRMCR_IND_PXX;
          const double ux = cl.ux;
          const int nT = cl.nT, Ltot = cl.Ltot;
          double v1 = 0, tx = 0, ty = 0, tz = 0, t2 = 0;
          {                                 // the round's indicator change, in the warp kernel's lane order
            double ds = 0.0;
            for (int q = 1; q <= cl.top; ++q)
              for (int j = lane; j < BC(i, q); j += 32) ds += (double)S.dsv[BS(i, q) + j];
            ds = warp_sum(ds);
            if (lane == 0) cl.dS += ds;
            __syncwarp();
          }
          for (int q = lane; q < nT; q += 32) {
            const uint32_t sl = pi0((uint32_t)(Ltot + q));
            if (sl >= (uint32_t)n) { atomicOr(P.err, kErrInternal); continue; }
            const double x = vx[sl], y = vy[sl], z = vz[sl];
            if (pxx) { const double dx = x - ux; v1 += dx * dx; }
            else { const double v2 = x * x + y * y + z * z; v1 += v2 * v2; }
            tx += x; ty += y; tz += z; t2 += x * x + y * y + z * z;
          }
          if (__any_sync(0xffffffffu, nT > 0)) {
            v1 = warp_sum(v1); tx = warp_sum(tx); ty = warp_sum(ty); tz = warp_sum(tz);
            t2 = warp_sum(t2);
          }
          double sest = (cl.cind + cl.dS) - v1;
          if (nT > 0) {
            tx /= nT; ty /= nT; tz /= nT;
            const double T = fmax(0.0, t2 / nT - (tx * tx + ty * ty + tz * tz)) / 3.0;
            if (pxx) {
              sest += (double)nT * (T + (tx - ux) * (tx - ux));
            } else {
              const double u2 = tx * tx + ty * ty + tz * tz;
              sest += (double)nT * (u2 * u2 + 10.0 * u2 * T + 15.0 * T * T);
            }
          }
          sest = sest / n;
          const double S0 = cl.S0;
          const double E1 = S0 != 0.0 ? fabs(sest - S0) / fabs(S0) : (sest == 0.0 ? 0.0 : INFINITY);
          // decision (R21); retries whose plan would be empty (no quota in the
          // new levels) are run here at once: nothing changes, E1 stays
          int m_cur = cl.m_cur, r = cl.r, d = cl.d, rem = cl.rem, flag = kOk, lo = cl.lo, hi = cl.hi;
          int budget = cl.budget, leaf_off = cl.leaf_off, m_next = cl.m_next;
          bool retry = false;
          const uint4 wl = K(kSplit, 0, (uint32_t)lane, 0);
          const double ul = u53(wl.x, wl.y);
          for (;;) {
            if (E1 > P.delta2 && m_cur < P.m_cap) {
              const int m_new = 2 * m_cur < P.m_cap ? 2 * m_cur : P.m_cap;
              bsplit_extend(K, cl, m_new, &BQ(i, 0), ul, d, rem, flag);
              __syncwarp();
              r += 1;
              lo = m_cur + 1;
              hi = d < kBatchLcap ? d : kBatchLcap;
              budget = nT;
              leaf_off = Ltot;
              m_cur = m_new;
              if (flag != kOk) break;
              int top = hi;
              while (top >= lo && BQ(i, top) == 0) top--;
              if (top >= lo && top >= 1) { retry = true; break; }   // a real plan: next round
            } else {
              m_next = (E1 < P.delta1) ? (m_cur / 2 > 1 ? m_cur / 2 : 1) : m_cur;
              break;
            }
          }
          if (lane == 0) {
            cl.S_est = sest; cl.E1 = E1;
            cl.m_cur = m_cur; cl.r = r; cl.d = d; cl.rem = rem; cl.lo = lo; cl.hi = hi;
            cl.budget = budget; cl.leaf_off = leaf_off; cl.m_next = m_next;
            cl.flag = flag != kOk ? flag : (retry ? kOk : kBDone);
          }
          __syncwarp();
        }
        __syncthreads();
        BPHASE_ADD(8);
      }
      // ---- A8 Maxwellian of Theta, statistics (warp per cell) ----
      for (int i = warp; i < nc; i += kBatchWarps) {
        BatchCell &cl = S.cells[i];
        if (cl.flag != kBDone || cl.n == 0) continue;
        const int n = cl.n, nT = cl.nT;
        const RngKey K{P.k0, P.k1, P.cell_base + (uint32_t)(s + i), P.step};
        Real *vx = S.vx + cl.vb, *vy = S.vy + cl.vb, *vz = S.vz + cl.vb;
        if (nT >= 2) {
          Perm pi0;
          pi0.rk = cl.pk; pi0.D = cl.D0;
          const bool full = (nT == n);
          double ux, uy, uz;
          if (full) {
            ux = cl.ux; uy = cl.uy; uz = cl.uz;
          } else {
            double a = 0, b = 0, c = 0;
            for (int q = lane; q < nT; q += 32) {
              const uint32_t sl = pi0((uint32_t)(cl.Ltot + q));
              if (sl >= (uint32_t)n) { atomicOr(P.err, kErrInternal); continue; }
              a += (double)vx[sl]; b += (double)vy[sl]; c += (double)vz[sl];
            }
            ux = warp_sum(a) / nT; uy = warp_sum(b) / nT; uz = warp_sum(c) / nT;
          }
          double g0s = 0, g1s = 0, g2s = 0, gg = 0, ec = 0;
          for (int q = lane; q < nT; q += 32) {
            uint32_t sl = (uint32_t)q;
            if (!full) sl = pi0((uint32_t)(cl.Ltot + q));
            if (sl >= (uint32_t)n) continue;
            if (!full) {
              const double dx = vx[sl] - ux, dy = vy[sl] - uy, dz = vz[sl] - uz;
              ec += dx * dx + dy * dy + dz * dz;
            }
            Real g0, g1, g2;
            gauss3<Real>(K, sl, g0, g1, g2);
            vx[sl] = g0; vy[sl] = g1; vz[sl] = g2;
            g0s += g0; g1s += g1; g2s += g2;
            gg += (double)g0 * g0 + (double)g1 * g1 + (double)g2 * g2;
          }
          g0s = warp_sum(g0s); g1s = warp_sum(g1s); g2s = warp_sum(g2s); gg = warp_sum(gg);
          ec = full ? cl.c2 : warp_sum(ec);
          const double gx = g0s / nT, gy = g1s / nT, gz = g2s / nT;
          const double D = gg - nT * (gx * gx + gy * gy + gz * gz);
          const double sc = (D > 0.0 && ec > 0.0) ? sqrt(ec / D) : 0.0;
          const Real rsc = (Real)sc, rgx = (Real)gx, rgy = (Real)gy, rgz = (Real)gz;
          const Real rux = (Real)ux, ruy = (Real)uy, ruz = (Real)uz;
          __syncwarp();
          for (int q = lane; q < nT; q += 32) {
            uint32_t sl = (uint32_t)q;
            if (!full) sl = pi0((uint32_t)(cl.Ltot + q));
            if (sl >= (uint32_t)n) continue;
            vx[sl] = rux + rsc * (vx[sl] - rgx);
            vy[sl] = ruy + rsc * (vy[sl] - rgy);
            vz[sl] = ruz + rsc * (vz[sl] - rgz);
          }
        }
        if (lane == 0) {
          const int c = s + i;
          if (P.adaptive) m_state[c] = cl.m_next;
          double *st = stats + (size_t)c * TRMCR_NSTATS;
          st[TRMCR_ST_N] = n; st[TRMCR_ST_P] = cl.p; st[TRMCR_ST_MU] = cl.mu; st[TRMCR_ST_SIGMA] = cl.sigma;
          st[TRMCR_ST_S0] = cl.S0; st[TRMCR_ST_SEST] = cl.S_est; st[TRMCR_ST_E1] = cl.E1;
          st[TRMCR_ST_MUSED] = cl.m_cur; st[TRMCR_ST_MNEXT] = cl.m_next; st[TRMCR_ST_DEPTH] = cl.d;
          st[TRMCR_ST_ATTEMPTS] = cl.r + 1; st[TRMCR_ST_LEAVES] = cl.Ltot; st[TRMCR_ST_UNTOUCHED] = cl.U;
          st[TRMCR_ST_THERMALISED] = nT; st[TRMCR_ST_PROPOSALS] = (double)cl.prop;
          st[TRMCR_ST_ACCEPTED] = (double)cl.acc; st[TRMCR_ST_VIOLATIONS] = (double)cl.viol;
          st[TRMCR_ST_MAXW] = nT >= 2 ? nT : 0;
          st[TRMCR_ST_PX] = cl.sums[0]; st[TRMCR_ST_PY] = cl.sums[1]; st[TRMCR_ST_PZ] = cl.sums[2];
          st[TRMCR_ST_ENERGY] = cl.sums[3];
        }
      }
      __syncthreads();
      BPHASE_ADD(9);
      // ---- write-back of the finished cells; deferred cells to the CTA kernel ----
      if (tid < nc) {
        const BatchCell &cl = S.cells[tid];
        if (cl.flag != kBDone) defer_list[atomicAdd(defer_count, 1)] = s + tid;
      }
      for (int i = warp; i < nc; i += kBatchWarps) {
        const BatchCell &cl = S.cells[i];
        if (cl.flag != kBDone) continue;
        const int64_t g0 = off[s + i];
        for (int q = lane; q < cl.n; q += 32) {
          gvx[g0 + q] = S.vx[cl.vb + q]; gvy[g0 + q] = S.vy[cl.vb + q]; gvz[g0 + q] = S.vz[cl.vb + q];
        }
      }
      __syncthreads();   // the stage is refilled by the next batch
      BPHASE_ADD(10);
      s = e_cell;
    }
  }
  pdl_trigger();
}

#undef BQ
#undef BC
#undef BS
#undef BCONS
#undef BRK
#undef BPD
#undef BPRE

}  // namespace trmcr
